// vcsched_b200.cpp — the C++ drop-in shim (libvcsched_b200.so): the reference's public solver
// API (namespace vcsched, headers under paper_2012_12419_b200/include/vcsched/) implemented over
// the C ABI of include/vcs_gpu.h.  A C++ caller of the reference (tools/cli.cpp run_scheduler,
// the doctest suites, benchmarks/) relinks against this library unchanged.
//
// Status codes of the C ABI become the reference's exception types and messages:
//   VCS_ECAP -> StateCapacityError(cap); VCS_EINVAL -> std::invalid_argument (ConfigError in
//   io); VCS_EIO -> IoError; VCS_ERANGE -> std::out_of_range; VCS_ECUDA -> std::runtime_error.
#include "vcsched/io.hpp"
#include "vcsched/mdp.hpp"
#include "vcsched/parallel_vi.hpp"

#include "../../include/vcs_gpu.h"

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <istream>
#include <iterator>
#include <limits>
#include <sstream>

namespace vcsched {

using detail::PinnedVector;

namespace {

[[noreturn]] void rethrow(int rc, std::size_t cap = 0, bool io = false) {
    const std::string msg = vcs_last_error();
    switch (rc) {
    case VCS_ECAP: throw StateCapacityError(cap);
    case VCS_EINVAL:
        if (io) throw ConfigError(msg);
        throw std::invalid_argument(msg);
    case VCS_EIO: throw IoError(msg);
    case VCS_ERANGE: throw std::out_of_range(msg);
    default: throw std::runtime_error("vcs_gpu: " + msg);
    }
}

void check(int rc, std::size_t cap = 0, bool io = false) {
    if (rc != VCS_OK) rethrow(rc, cap, io);
}

int default_device() {
    static const int dev = [] {
        const char* env = std::getenv("VCS_DEVICE");
        return env ? std::atoi(env) : 0;
    }();
    return dev;
}

// SoA staging of an instance for the C ABI (arrays live as long as this object).
struct Soa {
    std::vector<int32_t> cid, ctot, cfree, tid, tdem, bid, boff;
    std::vector<double> cthr, cdel, tdel, tthr;
    vcs_instance v{};

    Soa(const VccModel& vcc, const std::vector<Task>& tasks, std::span<const BagOfTasks> bots) {
        for (const auto& c : vcc.clouds) {
            cid.push_back(c.id);
            ctot.push_back(c.vm_total);
            cfree.push_back(c.vm_free);
            cthr.push_back(c.vm_throughput_kbps);
            cdel.push_back(c.v2i_delay_ms);
        }
        for (const auto& t : tasks) {
            tid.push_back(t.id);
            tdem.push_back(t.vm_demand);
            tdel.push_back(t.max_delay_ms);
            tthr.push_back(t.min_vm_throughput_kbps);
        }
        boff.push_back(0);
        for (const auto& b : bots) {
            bid.push_back(b.id);
            boff.push_back(boff.back() + static_cast<int32_t>(b.tasks.size()));
        }
        v.n_clouds = static_cast<int32_t>(cid.size());
        v.cloud_id = cid.data();
        v.cloud_vm_total = ctot.data();
        v.cloud_vm_free = cfree.data();
        v.cloud_thr_kbps = cthr.data();
        v.cloud_delay_ms = cdel.data();
        v.n_tasks = static_cast<int32_t>(tid.size());
        v.task_id = tid.data();
        v.task_demand = tdem.data();
        v.task_max_delay_ms = tdel.data();
        v.task_min_thr_kbps = tthr.data();
        v.n_bots = static_cast<int32_t>(bid.size());
        v.bot_id = bid.data();
        v.bot_task_offset = boff.data();
        v.beta_vc = vcc.reward_per_vc_vm;
        v.beta_tc = vcc.cost_per_tcc_vm;
        v.gamma_vc = vcc.penalty_per_idle_vm;
    }
};

bool cloud_feasible_in_state(const MdpInstance& instance, const MdpState& s, int i) {
    const auto& cloud = instance.vcc.clouds[static_cast<std::size_t>(i)];
    const auto& task = instance.tasks[static_cast<std::size_t>(s.next_task_index)];
    return s.free_vms[static_cast<std::size_t>(i)] >= task.vm_demand &&
           cloud.v2i_delay_ms <= task.max_delay_ms &&
           cloud.vm_throughput_kbps >= task.min_vm_throughput_kbps;
}

struct StateArrays {
    std::vector<int32_t> free_vms;
    int32_t t = 0;
    uint8_t terminal = 0;
};

StateArrays state_arrays(const StateSpace& sp, const MdpState& s) {
    const int t = s.terminal ? sp.task_count() : s.next_task_index;
    if (t < 0 || t > sp.task_count()) throw std::invalid_argument("task index outside horizon");
    if (s.free_vms.size() != sp.instance().vcc.clouds.size())
        throw std::invalid_argument("state has wrong cloud count");
    StateArrays a;
    a.free_vms.assign(s.free_vms.begin(), s.free_vms.end());
    a.t = s.next_task_index;
    a.terminal = s.terminal ? 1 : 0;
    return a;
}

ParsedInstance from_owned(vcs_instance_owned* h) {
    const vcs_instance* v = vcs_instance_view(h);
    ParsedInstance p;
    p.vcc.reward_per_vc_vm = v->beta_vc;
    p.vcc.cost_per_tcc_vm = v->beta_tc;
    p.vcc.penalty_per_idle_vm = v->gamma_vc;
    for (int i = 0; i < v->n_clouds; ++i)
        p.vcc.clouds.push_back({v->cloud_id[i], v->cloud_vm_total[i], v->cloud_vm_free[i],
                                v->cloud_thr_kbps[i], v->cloud_delay_ms[i]});
    for (int b = 0; b < v->n_bots; ++b) {
        BagOfTasks bot;
        bot.id = v->bot_id[b];
        for (int j = v->bot_task_offset[b]; j < v->bot_task_offset[b + 1]; ++j)
            bot.tasks.push_back({v->task_id[j], v->task_demand[j], v->task_max_delay_ms[j],
                                 v->task_min_thr_kbps[j]});
        p.bots.push_back(std::move(bot));
    }
    vcs_instance_free(h);
    return p;
}

} // namespace

// ---- workload.hpp ---------------------------------------------------------------------------

long total_demand(std::span<const BagOfTasks> bots) {
    long sum = 0;
    for (const auto& b : bots)
        for (const auto& t : b.tasks) sum += t.vm_demand;
    return sum;
}

long total_capacity(const VccModel& vcc) {
    long sum = 0;
    for (const auto& c : vcc.clouds) sum += c.vm_total;
    return sum;
}

bool feasible(const VehicularCloud& cloud, const Task& task) {
    return cloud.vm_free >= task.vm_demand && cloud.v2i_delay_ms <= task.max_delay_ms &&
           cloud.vm_throughput_kbps >= task.min_vm_throughput_kbps;
}

std::vector<Task> flatten_tasks(std::span<const BagOfTasks> bots) {
    std::vector<Task> out;
    for (const auto& b : bots) out.insert(out.end(), b.tasks.begin(), b.tasks.end());
    return out;
}

void validate(const VccModel& vcc) {
    // vcs_instance_copy runs the library's validate(); only the model part is populated here.
    Soa soa(vcc, {}, {});
    vcs_instance_owned* h = nullptr;
    const int rc = vcs_instance_copy(&soa.v, &h);
    if (h) vcs_instance_free(h);
    check(rc);
}

void validate(std::span<const BagOfTasks> bots) {
    VccModel empty;
    Soa soa(empty, flatten_tasks(bots), bots);
    vcs_instance_owned* h = nullptr;
    const int rc = vcs_instance_copy(&soa.v, &h);
    if (h) vcs_instance_free(h);
    check(rc);
}

// ---- greedy.hpp -----------------------------------------------------------------------------

ScheduleResult greedy_schedule(const VccModel& vcc, std::span<const BagOfTasks> bots) {
    const auto tasks = flatten_tasks(bots);
    Soa soa(vcc, tasks, bots);
    std::vector<int32_t> target(std::max<std::size_t>(1, tasks.size()));
    std::vector<int64_t> used(std::max<std::size_t>(1, vcc.clouds.size()));
    int64_t paid = 0, unused = 0;
    check(vcs_greedy(&soa.v, default_device(), target.data(), used.data(), &paid, &unused));
    ScheduleResult r;
    for (const auto& c : vcc.clouds) r.per_vc_used[c.id] = 0;
    for (std::size_t i = 0; i < vcc.clouds.size(); ++i) r.per_vc_used[vcc.clouds[i].id] += used[i];
    for (std::size_t j = 0; j < tasks.size(); ++j) {
        const int t = target[j];
        r.placements.push_back(
            {tasks[j].id, t >= 0 ? vcc.clouds[static_cast<std::size_t>(t)].id : kPaidCloud,
             tasks[j].vm_demand});
    }
    r.paid_vms = paid;
    r.unused_vms = unused;
    return r;
}

double greedy_reward(const ScheduleResult& result, const VccModel& vcc) {
    return vcc.reward_per_vc_vm * static_cast<double>(result.vc_placed_vms()) -
           vcc.cost_per_tcc_vm * static_cast<double>(result.paid_vms) -
           vcc.penalty_per_idle_vm * static_cast<double>(result.unused_vms);
}

// ---- mdp.hpp --------------------------------------------------------------------------------

MdpInstance MdpInstance::from_workload(const VccModel& vcc, std::span<const BagOfTasks> bots) {
    return MdpInstance{vcc, flatten_tasks(bots)};
}

MdpState initial_state(const MdpInstance& instance) {
    MdpState s;
    for (const auto& c : instance.vcc.clouds) s.free_vms.push_back(c.vm_free);
    s.terminal = instance.tasks.empty();
    return s;
}

std::vector<MdpAction> legal_actions(const MdpInstance& instance, const MdpState& s) {
    std::vector<MdpAction> out;
    if (s.terminal) return out;
    for (int i = 0; i < static_cast<int>(instance.vcc.clouds.size()); ++i)
        if (cloud_feasible_in_state(instance, s, i)) out.push_back(MdpAction{i});
    out.push_back(MdpAction{kPaidCloud});
    return out;
}

MdpState transition(const MdpState& s, MdpAction a, const MdpInstance& instance) {
    if (s.terminal) throw std::invalid_argument("transition from terminal state");
    MdpState next = s;
    if (!a.is_paid()) {
        if (a.target < 0 || a.target >= static_cast<int>(instance.vcc.clouds.size()))
            throw std::invalid_argument("action targets unknown cloud");
        if (!cloud_feasible_in_state(instance, s, a.target))
            throw std::invalid_argument("action targets infeasible cloud");
        next.free_vms[static_cast<std::size_t>(a.target)] -=
            instance.tasks[static_cast<std::size_t>(s.next_task_index)].vm_demand;
    }
    next.next_task_index = s.next_task_index + 1;
    next.terminal = next.next_task_index == static_cast<int>(instance.tasks.size());
    return next;
}

double step_reward(const MdpState& s, MdpAction a, const MdpState&, const MdpInstance& instance) {
    const double n =
        static_cast<double>(instance.tasks[static_cast<std::size_t>(s.next_task_index)].vm_demand);
    return a.is_paid() ? -instance.vcc.cost_per_tcc_vm * n : instance.vcc.reward_per_vc_vm * n;
}

std::shared_ptr<const StateSpace> StateSpace::build(const MdpInstance& instance,
                                                    std::size_t state_cap) {
    auto sp = std::make_shared<StateSpace>();
    sp->instance_ = std::make_shared<const MdpInstance>(instance);
    sp->device_ = default_device();
    Soa soa(instance.vcc, instance.tasks, {});
    vcs_space* h = nullptr;
    check(vcs_space_build(&soa.v, state_cap, sp->device_, &h), state_cap);
    sp->handle_ = h;
    vcs_space_info info{};
    check(vcs_space_info_get(h, &info));
    sp->n_states_ = info.n_states;
    sp->horizon_ = info.horizon;
    std::vector<uint64_t> lo(static_cast<std::size_t>(info.horizon) + 2);
    check(vcs_space_layer_offsets(h, lo.data()));
    sp->layer_offset_.assign(lo.begin(), lo.end());
    return sp;
}

StateSpace::~StateSpace() {
    if (handle_) vcs_space_free(handle_);
}

std::size_t StateSpace::locate(const MdpState& s) const {
    auto a = state_arrays(*this, s);
    int64_t idx = -1;
    check(vcs_space_locate(handle_, 1, a.free_vms.data(), &a.t, &a.terminal, &idx));
    if (idx < 0) throw std::out_of_range("state not reachable in enumerated space");
    return static_cast<std::size_t>(idx);
}

double StateSpace::hidden_penalty(const MdpState& s) const {
    auto a = state_arrays(*this, s);
    double out = 0.0;
    check(vcs_space_hidden_penalty(handle_, 1, a.free_vms.data(), &a.t, &a.terminal, &out));
    return out;
}

double StateSpace::backup(std::size_t s, const double* prev, std::int32_t* best_action) const {
    std::call_once(csr_once_, [&] {
        vcs_space_info info{};
        check(vcs_space_info_get(handle_, &info));
        row_ptr_.resize(info.n_states + 1);
        succ_.resize(std::max<uint64_t>(1, info.n_edges));
        reward_.resize(std::max<uint64_t>(1, info.n_edges));
        action_.resize(std::max<uint64_t>(1, info.n_edges));
        check(vcs_space_csr(handle_, row_ptr_.data(), succ_.data(), reward_.data(),
                            action_.data()));
    });
    const std::size_t first = row_ptr_[s], last = row_ptr_[s + 1];
    if (first == last) {
        if (best_action) *best_action = kPaidCloud;
        return 0.0;
    }
    double best = -std::numeric_limits<double>::infinity();
    std::int32_t act = kPaidCloud;
    for (std::size_t e = first; e < last; ++e) {
        const double q = reward_[e] + prev[succ_[e]];
        if (q > best) {
            best = q;
            act = action_[e];
        }
    }
    if (best_action) *best_action = act;
    return best;
}

double ValueTable::value_of(const MdpState& s) const {
    return values_[space_->locate(s)] - space_->hidden_penalty(s);
}

double ValueTable::initial_value() const { return value_of(initial_state(space_->instance())); }

MdpAction Policy::action_for(const MdpState& s) const {
    if (s.terminal || s.next_task_index >= space_->task_count())
        throw std::out_of_range("terminal states carry no action");
    return MdpAction{actions_[space_->locate(s)]};
}

namespace {
// The GPUs n_workers maps to: the reference's workers are threads over row blocks
// (parallel_vi.cpp:68-107); here they are GPUs over one state space (vcs_solve_multi), as many as
// are visible.  VCS_EMULATE_RANKS=1 runs n_workers ranks even on fewer GPUs (round robin; the
// emulated-rank test mode of the multi-GPU path).
std::vector<int32_t> worker_devices(int first, int n_workers) {
    int n_dev = vcs_device_count();
    if (n_dev < 1) n_dev = 1;
    const bool emulate = std::getenv("VCS_EMULATE_RANKS") != nullptr;
    const int n = emulate ? n_workers : std::min(n_workers, n_dev);
    std::vector<int32_t> devs(static_cast<std::size_t>(n));
    for (int r = 0; r < n; ++r) devs[static_cast<std::size_t>(r)] = (first + r) % n_dev;
    return devs;
}
} // namespace

namespace detail {
ViResult run_value_iteration(std::shared_ptr<const StateSpace> space, const ViOptions& options,
                             int n_workers) {
    vcs_solve_report rep{};
    return run_value_iteration(std::move(space), options, n_workers, &rep);
}

ViResult run_value_iteration(std::shared_ptr<const StateSpace> space, const ViOptions& options,
                             int n_workers, vcs_solve_report* report) {
    if (n_workers < 1) throw std::invalid_argument("n_workers must be >= 1");
    // page-locked results: the solve streams them to the host behind the layer pass
    PinnedVector<double> values(space->size());
    PinnedVector<std::int32_t> actions(space->size());
    vcs_solve_opts opts{options.epsilon, 1, 0, 1.0, VCS_METHOD_AUTO};
    vcs_solve_report& rep = *report;
    const auto devs = worker_devices(space->device(), n_workers);
    if (devs.size() == 1)
        check(vcs_solve(space->handle(), &opts, values.data(), actions.data(), &rep));
    else
        check(vcs_solve_multi(space->handle(), &opts, static_cast<int32_t>(devs.size()), devs.data(),
                              VCS_EXCHANGE_HALO, values.data(), actions.data(), &rep));
    const std::uint64_t gen = vcs_space_result_generation(space->handle());
    ValueTable table(space, std::move(values), rep.sweeps, options.epsilon);
    Policy policy(std::move(space), std::move(actions), gen);
    return ViResult{std::move(table), std::move(policy)};
}
} // namespace detail

ViResult value_iteration(const MdpInstance& instance, const ViOptions& options) {
    return detail::run_value_iteration(StateSpace::build(instance, options.state_cap), options, 1);
}

std::pair<double, MdpAction> bellman_backup(const MdpState& s, const ValueTable& values,
                                            const MdpInstance& instance) {
    if (s.terminal) throw std::invalid_argument("bellman backup of a terminal state");
    double best = -std::numeric_limits<double>::infinity();
    MdpAction best_action{kPaidCloud};
    for (const MdpAction a : legal_actions(instance, s)) {
        const MdpState next = transition(s, a, instance);
        const double q = step_reward(s, a, next, instance) + values.value_of(next);
        if (q > best) {
            best = q;
            best_action = a;
        }
    }
    return {best, best_action};
}

// rollout (mdp.cpp:305-324).  The policy walk runs on the device (vcs_rollout: one kernel
// follows the H decisions through the device key index) when the space still holds this policy's
// results; a policy whose space has solved again since walks with one device locate per step
// against its own actions.  The ScheduleResult bookkeeping is the reference's.
ScheduleResult rollout(const Policy& policy, const MdpInstance& instance) {
    ScheduleResult result;
    for (const auto& c : instance.vcc.clouds) result.per_vc_used[c.id] = 0;
    const StateSpace& space = policy.space();
    const std::size_t H = instance.tasks.size();
    std::vector<int32_t> targets;
    if (policy.generation() == vcs_space_result_generation(space.handle())) {
        targets.resize(std::max<std::size_t>(H, 1));
        Soa soa(instance.vcc, instance.tasks, {});
        check(vcs_rollout(space.handle(), &soa.v, targets.data(), nullptr));
        targets.resize(H);
    } else {
        MdpState s = initial_state(instance);
        while (!s.terminal) {
            const MdpAction a = policy.action_for(s);
            targets.push_back(a.target);
            s = transition(s, a, instance);
        }
    }
    for (std::size_t t = 0; t < H; ++t) {
        const auto& task = instance.tasks[t];
        const int a = targets[t];
        if (a == kPaidCloud) {
            result.paid_vms += task.vm_demand;
            result.placements.push_back({task.id, kPaidCloud, task.vm_demand});
        } else {
            const int id = instance.vcc.clouds[static_cast<std::size_t>(a)].id;
            result.per_vc_used[id] += task.vm_demand;
            result.placements.push_back({task.id, id, task.vm_demand});
        }
    }
    result.unused_vms = total_capacity(instance.vcc) - result.vc_placed_vms();
    return result;
}

// ---- parallel_vi.hpp ------------------------------------------------------------------------

BlockPartition BlockPartition::even(std::size_t n_states, int n_blocks) {
    if (n_blocks < 1) throw std::invalid_argument("n_blocks must be >= 1");
    BlockPartition part;
    part.n_blocks = n_blocks;
    const std::size_t base = n_states / static_cast<std::size_t>(n_blocks);
    const std::size_t extra = n_states % static_cast<std::size_t>(n_blocks);
    std::size_t begin = 0;
    for (int b = 0; b < n_blocks; ++b) {
        const std::size_t len = base + (static_cast<std::size_t>(b) < extra ? 1 : 0);
        part.ranges.emplace_back(begin, begin + len);
        begin += len;
    }
    return part;
}

int BlockPartition::block_of(std::size_t state) const {
    for (int b = 0; b < n_blocks; ++b)
        if (state >= ranges[static_cast<std::size_t>(b)].first &&
            state < ranges[static_cast<std::size_t>(b)].second)
            return b;
    return -1;
}

void SweepBarrier::arrive_and_wait() {
    std::unique_lock lock(mutex_);
    const std::uint64_t gen = generation_;
    if (++waiting_ == participants_) {
        waiting_ = 0;
        ++generation_;
        cv_.notify_all();
    } else {
        cv_.wait(lock, [&] { return generation_ != gen; });
    }
}

ViResult parallel_value_iteration(const MdpInstance& instance, const ViOptions& options,
                                  int n_workers) {
    if (n_workers < 1) throw std::invalid_argument("n_workers must be >= 1");
    return detail::run_value_iteration(StateSpace::build(instance, options.state_cap), options,
                                       n_workers);
}

std::vector<SpeedupRow> measure_speedup(const MdpInstance& instance,
                                        std::span<const int> worker_counts,
                                        const ViOptions& options) {
    std::vector<SpeedupRow> rows;
    auto space = StateSpace::build(instance, options.state_cap);
    for (int workers : worker_counts) {
        const auto t0 = std::chrono::steady_clock::now();
        auto result = detail::run_value_iteration(space, options, workers);
        const auto t1 = std::chrono::steady_clock::now();
        (void)result;
        SpeedupRow row;
        row.workers = workers;
        row.wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        rows.push_back(row);
    }
    double baseline = rows.empty() ? 0.0 : rows.front().wall_ms;
    for (const auto& r : rows)
        if (r.workers == 1) baseline = r.wall_ms;
    for (auto& r : rows) r.speedup_vs_one = r.wall_ms > 0.0 ? baseline / r.wall_ms : 1.0;
    return rows;
}

// ---- io.hpp (instance format) ---------------------------------------------------------------

ParsedInstance parse_instance(std::istream& in) {
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    vcs_instance_owned* h = nullptr;
    check(vcs_instance_parse(text.c_str(), &h), 0, true);
    return from_owned(h);
}

ParsedInstance load_instance(const std::string& path) {
    vcs_instance_owned* h = nullptr;
    check(vcs_instance_load(path.c_str(), &h), 0, true);
    return from_owned(h);
}

// ---- io.hpp writers (io.cpp:103-118, 203-242, 351-357 formats) -------------------------------

namespace {
std::string fmt17(double v) { // io.cpp fmt: %.17g
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}
std::string json_num(double v) { // nlohmann::json's shortest round-trip form
    if (std::isnan(v) || std::isinf(v)) return "null";
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, v);
    std::string s(buf, r.ptr);
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}
std::string target_name(int target) { return target == kPaidCloud ? "tcc" : "vc:" + std::to_string(target); }
double reward_total(const ScheduleResult& r, const VccModel& vcc) { // metrics.cpp:32-39
    const double gain = vcc.reward_per_vc_vm * static_cast<double>(r.vc_placed_vms());
    const double cost = vcc.cost_per_tcc_vm * static_cast<double>(r.paid_vms);
    const double idle = vcc.penalty_per_idle_vm * static_cast<double>(r.unused_vms);
    return gain - cost - idle;
}
} // namespace

std::string instance_text(const ParsedInstance& instance) {
    std::ostringstream out;
    out << "beta_vc " << fmt17(instance.vcc.reward_per_vc_vm) << "\n";
    out << "beta_tc " << fmt17(instance.vcc.cost_per_tcc_vm) << "\n";
    out << "gamma_vc " << fmt17(instance.vcc.penalty_per_idle_vm) << "\n";
    for (const auto& c : instance.vcc.clouds)
        out << "cloud " << c.id << ' ' << c.vm_total << ' ' << fmt17(c.vm_throughput_kbps) << ' '
            << fmt17(c.v2i_delay_ms) << "\n";
    for (const auto& bot : instance.bots) {
        out << "bot " << bot.id << "\n";
        for (const auto& t : bot.tasks)
            out << "task " << t.id << ' ' << t.vm_demand << ' ' << fmt17(t.max_delay_ms) << ' '
                << fmt17(t.min_vm_throughput_kbps) << "\n";
    }
    return out.str();
}

std::string schedule_csv(const ScheduleResult& result, const VccModel& vcc,
                         const std::optional<SolverDiagnostics>& diag) {
    std::ostringstream out;
    out << "task_id,target,vms_used\n";
    for (const auto& p : result.placements)
        out << p.task_id << ',' << target_name(p.target) << ',' << p.vms_used << "\n";
    out << "\n";
    out << "summary,key,value\n";
    out << "summary,vc_placed_vms," << result.vc_placed_vms() << "\n";
    out << "summary,paid_vms," << result.paid_vms << "\n";
    out << "summary,unused_vms," << result.unused_vms << "\n";
    out << "summary,total_reward," << fmt17(reward_total(result, vcc)) << "\n";
    if (diag) {
        out << "summary,epsilon," << fmt17(diag->epsilon) << "\n";
        out << "summary,sweeps," << diag->sweeps << "\n";
        out << "summary,states_explored," << diag->states_explored << "\n";
        if (!diag->solver.empty()) {
            out << "summary,solver," << diag->solver << "\n";
            out << "summary,gpus," << diag->gpus << "\n";
            out << "summary,device_ms," << fmt17(diag->device_ms) << "\n";
            out << "summary,build_ms," << fmt17(diag->build_ms) << "\n";
        }
    }
    return out.str();
}

std::string schedule_json(const ScheduleResult& result, const VccModel& vcc,
                          const std::optional<SolverDiagnostics>& diag) {
    // the layout of nlohmann::json::dump(2) (io.cpp:228-242): object keys in sorted order
    std::ostringstream out;
    out << "{\n  \"placements\": [";
    for (std::size_t i = 0; i < result.placements.size(); ++i) {
        const auto& p = result.placements[i];
        out << (i ? ",\n" : "\n") << "    {\n      \"target\": \"" << target_name(p.target)
            << "\",\n      \"task_id\": " << p.task_id << ",\n      \"vms_used\": " << p.vms_used
            << "\n    }";
    }
    out << (result.placements.empty() ? "]" : "\n  ]") << ",\n  \"summary\": {\n";
    std::vector<std::pair<std::string, std::string>> kv = {
        {"paid_vms", std::to_string(result.paid_vms)},
        {"total_reward", json_num(reward_total(result, vcc))},
        {"unused_vms", std::to_string(result.unused_vms)},
        {"vc_placed_vms", std::to_string(result.vc_placed_vms())}};
    if (diag) {
        kv.push_back({"epsilon", json_num(diag->epsilon)});
        kv.push_back({"sweeps", std::to_string(diag->sweeps)});
        kv.push_back({"states_explored", std::to_string(diag->states_explored)});
        if (!diag->solver.empty()) {
            kv.push_back({"solver", "\"" + diag->solver + "\""});
            kv.push_back({"gpus", std::to_string(diag->gpus)});
            kv.push_back({"device_ms", json_num(diag->device_ms)});
            kv.push_back({"build_ms", json_num(diag->build_ms)});
        }
    }
    std::sort(kv.begin(), kv.end());
    for (std::size_t i = 0; i < kv.size(); ++i)
        out << "    \"" << kv[i].first << "\": " << kv[i].second << (i + 1 < kv.size() ? ",\n" : "\n");
    out << "  }\n}\n";
    return out.str();
}

std::string speedup_csv(const std::vector<SpeedupRow>& rows) {
    std::ostringstream out;
    out << "workers,wall_ms,speedup_vs_one\n";
    for (const auto& r : rows)
        out << r.workers << ',' << fmt17(r.wall_ms) << ',' << fmt17(r.speedup_vs_one) << "\n";
    return out.str();
}

std::string read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw IoError("cannot read file: " + path);
    return std::string((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
}

void write_file(const std::string& path, const std::string& content) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw IoError("cannot write file: " + path);
    out << content;
    if (!out) throw IoError("write failed: " + path);
}

} // namespace vcsched
