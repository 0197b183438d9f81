// tests/cpp/doctest_main.cpp — runner for tests/cpp/doctest.h.  Prints one line per test case
// and a summary; exit status 0 only when every assertion passed.
#include "doctest.h"

#include <cstdio>
#include <exception>

int main() {
    using namespace doctest::detail;
    int failed_cases = 0;
    for (const auto& tc : registry()) {
        const int before = assertion_failures();
        bool ok = true;
        try {
            tc.fn();
        } catch (const RequireFailed&) {
            ok = false;
        } catch (const std::exception& e) {
            std::fprintf(stderr, "%s:%d: unexpected exception: %s\n", tc.file, tc.line, e.what());
            ++assertion_failures();
            ok = false;
        }
        ok = ok && assertion_failures() == before;
        failed_cases += ok ? 0 : 1;
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", tc.name);
    }
    std::printf("test cases: %zu | %d passed | %d failed | assertion failures: %d\n",
                registry().size(), static_cast<int>(registry().size()) - failed_cases,
                failed_cases, assertion_failures());
    return failed_cases == 0 ? 0 : 1;
}
