// vcsched_cli.cpp — the `schedule` and `speedup` subcommands of the reference CLI
// (tools/cli.cpp:43-61 run_scheduler, :100-118 run_schedule, :199-212 run_speedup) over the B200
// drop-in shim, with one more scheduler: mdp-gpu (--gpus N), whose SolverDiagnostics carry the
// device path (io.hpp SolverDiagnostics::solver/gpus/device_ms/build_ms).  Exit codes as the
// reference (tools/cli.hpp:30-33): 0 ok, 2 config, 3 state cap, 4 io.  `simulate` / `benchmark`
// drive the DSRC simulator, which is not part of the solver path: exit 2 with a message.
//
//   vcsched-b200 schedule --instance F [--scheduler greedy|mdp|mdp-parallel|mdp-gpu]
//                [--workers N] [--gpus N] [--epsilon E] [--state-cap N] [--out F] [--format csv|json]
//   vcsched-b200 speedup --instance F [--workers N] [--epsilon E] [--state-cap N] [--out F]
//   vcsched-b200 e2e --instance F [--workers REPEAT] [--gpus N]   (timing of the API call path)
#include "vcsched/greedy.hpp"
#include "vcsched/io.hpp"
#include "vcsched/mdp.hpp"
#include "vcsched/parallel_vi.hpp"

#include "../../include/vcs_gpu.h"

#include <algorithm>
#include <chrono>
#include <iostream>
#include <map>
#include <optional>
#include <string>
#include <vector>

using namespace vcsched;

namespace {

constexpr int kOk = 0, kConfigError = 2, kCapExceeded = 3, kIoError = 4;

struct Config {
    std::string sub, instance, out, format = "csv", scheduler = "greedy";
    int workers = 1, gpus = 1;
    double epsilon = 1e-6;
    std::size_t state_cap = 5'000'000;
};

Config parse(const std::vector<std::string>& a) {
    if (a.empty()) throw ConfigError("usage: vcsched-b200 <schedule|speedup> --instance FILE [...]");
    Config c;
    c.sub = a[0];
    for (std::size_t i = 1; i < a.size(); ++i) {
        const std::string& k = a[i];
        auto val = [&]() -> const std::string& {
            if (i + 1 >= a.size()) throw ConfigError("missing value for " + k);
            return a[++i];
        };
        try {
            if (k == "--instance") c.instance = val();
            else if (k == "--out") c.out = val();
            else if (k == "--format") c.format = val();
            else if (k == "--scheduler") c.scheduler = val();
            else if (k == "--workers") c.workers = std::stoi(val());
            else if (k == "--gpus") c.gpus = std::stoi(val());
            else if (k == "--epsilon") c.epsilon = std::stod(val());
            else if (k == "--state-cap") c.state_cap = static_cast<std::size_t>(std::stoull(val()));
            else throw ConfigError("unknown option '" + k + "'");
        } catch (const std::logic_error&) { // std::stoi / stod / stoull
            throw ConfigError("bad value for " + k);
        }
    }
    if (c.format != "csv" && c.format != "json")
        throw ConfigError("unknown format '" + c.format + "' (expected csv or json)");
    if (c.instance.empty()) throw ConfigError("--instance is required");
    if (c.workers < 1) throw ConfigError("--workers must be >= 1");
    if (c.gpus < 1) throw ConfigError("--gpus must be >= 1");
    return c;
}

int run_schedule(const Config& c) {
    const ParsedInstance instance = load_instance(c.instance);
    ScheduleResult result;
    std::optional<SolverDiagnostics> diag;
    if (c.scheduler == "greedy") {
        result = greedy_schedule(instance.vcc, instance.bots);
    } else if (c.scheduler == "mdp" || c.scheduler == "mdp-parallel" || c.scheduler == "mdp-gpu") {
        const auto mdp = MdpInstance::from_workload(instance.vcc, instance.bots);
        ViOptions options;
        options.epsilon = c.epsilon;
        options.state_cap = c.state_cap;
        const int n = c.scheduler == "mdp" ? 1 : c.scheduler == "mdp-parallel" ? c.workers : c.gpus;
        const auto t0 = std::chrono::steady_clock::now();
        auto space = StateSpace::build(mdp, options.state_cap);
        const auto t1 = std::chrono::steady_clock::now();
        vcs_solve_report rep{};
        const ViResult vi = detail::run_value_iteration(space, options, n, &rep);
        result = rollout(vi.policy, mdp);
        SolverDiagnostics d{vi.values.epsilon(), vi.values.sweeps(), vi.values.states_explored()};
        if (c.scheduler == "mdp-gpu") {
            d.solver = rep.method == VCS_METHOD_CERTIFIED ? "b200-certified"
                       : rep.method == VCS_METHOD_WAVEFRONT ? "b200-wavefront"
                                                            : "b200-jacobi";
            int n_dev = vcs_device_count();
            d.gpus = std::min(n, std::max(1, n_dev));
            d.device_ms = rep.sweep_ms + rep.extract_ms;
            d.build_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        }
        diag = d;
    } else {
        throw ConfigError("unknown scheduler '" + c.scheduler + "'");
    }
    if (!c.out.empty())
        write_file(c.out, c.format == "json" ? schedule_json(result, instance.vcc, diag)
                                            : schedule_csv(result, instance.vcc, diag));
    const double total = instance.vcc.reward_per_vc_vm * static_cast<double>(result.vc_placed_vms()) -
                         instance.vcc.cost_per_tcc_vm * static_cast<double>(result.paid_vms) -
                         instance.vcc.penalty_per_idle_vm * static_cast<double>(result.unused_vms);
    std::cout << "scheduler=" << c.scheduler << " vc_placed=" << result.vc_placed_vms()
              << " paid=" << result.paid_vms << " unused=" << result.unused_vms
              << " total_reward=" << total << "\n";
    if (diag) {
        std::cout << "epsilon=" << diag->epsilon << " sweeps=" << diag->sweeps
                  << " states_explored=" << diag->states_explored << "\n";
        if (!diag->solver.empty())
            std::cout << "solver=" << diag->solver << " gpus=" << diag->gpus
                      << " device_ms=" << diag->device_ms << " build_ms=" << diag->build_ms << "\n";
    }
    return kOk;
}

// `e2e`: the reference API call path end to end, repeated in one process (the CUDA context is
// created once, outside the timing): load_instance + MdpInstance::from_workload +
// StateSpace::build + detail::run_value_iteration (results into the ValueTable / Policy host
// storage) + rollout.  Prints one JSON object with the per-repetition wall times (ms).
int run_e2e(const Config& c, int repeat) {
    std::vector<double> ms, build_ms, solve_ms, rollout_ms;
    double v0 = 0.0;
    int sweeps = 0;
    long paid = 0;
    for (int i = 0; i < repeat + 2; ++i) {
        const auto t0 = std::chrono::steady_clock::now();
        const ParsedInstance instance = load_instance(c.instance);
        const auto mdp = MdpInstance::from_workload(instance.vcc, instance.bots);
        ViOptions options;
        options.epsilon = c.epsilon;
        options.state_cap = c.state_cap;
        auto space = StateSpace::build(mdp, options.state_cap);
        const auto t1 = std::chrono::steady_clock::now();
        const ViResult vi = detail::run_value_iteration(space, options, c.gpus);
        const auto t2 = std::chrono::steady_clock::now();
        const ScheduleResult r = rollout(vi.policy, mdp);
        const auto t3 = std::chrono::steady_clock::now();
        auto d = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        if (i >= 2) { // two warm-up repetitions (the device memory pool reaches its size)
            ms.push_back(d(t0, t3));
            build_ms.push_back(d(t0, t1));
            solve_ms.push_back(d(t1, t2));
            rollout_ms.push_back(d(t2, t3));
        }
        v0 = vi.values.raw_values()[0];
        sweeps = vi.values.sweeps();
        paid = r.paid_vms;
    }
    auto med = [](std::vector<double> v) {
        std::sort(v.begin(), v.end());
        return v.empty() ? 0.0 : v[v.size() / 2];
    };
    std::cout.precision(17);
    std::cout << "{\"ms_per_step\": " << med(ms) << ", \"load_and_build_ms\": " << med(build_ms)
              << ", \"solve_ms\": " << med(solve_ms) << ", \"rollout_ms\": " << med(rollout_ms)
              << ", \"steps\": " << ms.size() << ", \"sweeps\": " << sweeps
              << ", \"v0\": " << v0 << ", \"rollout_paid\": " << paid << "}\n";
    return kOk;
}

int run_speedup(const Config& c) {
    const ParsedInstance instance = load_instance(c.instance);
    const auto mdp = MdpInstance::from_workload(instance.vcc, instance.bots);
    ViOptions options;
    options.epsilon = c.epsilon;
    options.state_cap = c.state_cap;
    std::vector<int> counts = {1, 2, 4, 8}; // workers = GPUs of this process (parallel_vi.hpp)
    if (c.workers > 1) counts = {1, c.workers};
    const auto rows = measure_speedup(mdp, counts, options);
    const std::string text = speedup_csv(rows);
    if (!c.out.empty()) write_file(c.out, text);
    std::cout << text;
    return kOk;
}

} // namespace

int main(int argc, char** argv) {
    std::vector<std::string> args(argv + 1, argv + argc);
    try {
        const Config c = parse(args);
        if (c.sub == "schedule") return run_schedule(c);
        if (c.sub == "speedup") return run_speedup(c);
        if (c.sub == "e2e") return run_e2e(c, std::max(1, c.workers));
        if (c.sub == "simulate" || c.sub == "benchmark")
            throw ConfigError("subcommand '" + c.sub + "' drives the DSRC simulator, which is not "
                              "part of the B200 solver build");
        throw ConfigError("unknown subcommand '" + c.sub + "'");
    } catch (const ConfigError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kConfigError;
    } catch (const StateCapacityError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kCapExceeded;
    } catch (const IoError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kIoError;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kConfigError;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
