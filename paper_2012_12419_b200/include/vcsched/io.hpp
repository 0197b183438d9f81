// vcsched/io.hpp — B200 drop-in of the instance input format only
// (reference: core/include/vcsched/io.hpp:18-40; the simulator/metrics writers are out of
// scope for the solver path).  Parsing runs in libvcs_gpu.so (vcs_instance_parse).
#pragma once

#include "vcsched/greedy.hpp"
#include "vcsched/parallel_vi.hpp"
#include "vcsched/workload.hpp"

#include <iosfwd>
#include <stdexcept>
#include <string>
#include <vector>

namespace vcsched {

class ConfigError : public std::runtime_error {
    using std::runtime_error::runtime_error;
};

class IoError : public std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct ParsedInstance {
    VccModel vcc;
    std::vector<BagOfTasks> bots;
};

ParsedInstance parse_instance(std::istream& in);
ParsedInstance load_instance(const std::string& path);

} // namespace vcsched
