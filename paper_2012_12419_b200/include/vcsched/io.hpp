// vcsched/io.hpp — B200 drop-in of the solver-path I/O (reference: core/include/vcsched/io.hpp):
// the instance input format (:18-40), the schedule writers with SolverDiagnostics (:58-68) and
// the speedup table (:75).  The simulator / metrics writers are out of scope for the solver
// path.  Parsing runs in libvcs_gpu.so (vcs_instance_parse).
#pragma once

#include "vcsched/greedy.hpp"
#include "vcsched/parallel_vi.hpp"
#include "vcsched/workload.hpp"

#include <iosfwd>
#include <optional>
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
std::string instance_text(const ParsedInstance& instance);

/// The reference's three fields, plus (when `solver` is set) how the B200 path ran.
struct SolverDiagnostics {
    double epsilon = 0.0;
    int sweeps = 0;
    std::size_t states_explored = 0;
    std::string solver;     // e.g. "b200-certified" / "b200-wavefront"; empty: reference fields only
    int gpus = 0;           // GPUs the solve ran on
    double device_ms = 0.0; // device time of the solve (CUDA events)
    double build_ms = 0.0;  // device time of StateSpace::build
};

/// io.cpp:203-242 formats (summary rows / keys in the reference's order; the B200 fields follow
/// when SolverDiagnostics::solver is set).
std::string schedule_csv(const ScheduleResult& result, const VccModel& vcc,
                         const std::optional<SolverDiagnostics>& diag = std::nullopt);
std::string schedule_json(const ScheduleResult& result, const VccModel& vcc,
                          const std::optional<SolverDiagnostics>& diag = std::nullopt);
/// io.cpp:351-357.
std::string speedup_csv(const std::vector<SpeedupRow>& rows);
std::string read_file(const std::string& path);
void write_file(const std::string& path, const std::string& content);

} // namespace vcsched
