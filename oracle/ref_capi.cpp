// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A plain-C shim over the UNMODIFIED reference C++ library (compiled from
// /root/reference/proj/core/src/*.cpp by oracle/Makefile into oracle/_ref/libvcsref.so).
// It lets the Python tests and bench.py's reference arm drive the reference solver through
// its own public API:
//   StateSpace::build            core/src/mdp.cpp:81-214
//   detail::run_value_iteration  core/src/parallel_vi.cpp:48-116
//   ValueTable / Policy / rollout core/src/mdp.cpp:269-324
//   greedy_schedule / greedy_reward core/src/greedy.cpp:5-36
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) load it.
#include "vcsched/greedy.hpp"
#include "vcsched/io.hpp"
#include "vcsched/metrics.hpp"
#include "vcsched/sim.hpp"
#include "vcsched/mdp.hpp"
#include "vcsched/parallel_vi.hpp"

#include "../include/vcs_gpu.h"

#include <chrono>
#include <cstring>
#include <memory>
#include <optional>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

using namespace vcsched;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const StateCapacityError& e) {
        return fail(VCS_ECAP, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(VCS_EINVAL, e.what());
    } catch (const ConfigError& e) {
        return fail(VCS_EINVAL, e.what());
    } catch (const IoError& e) {
        return fail(VCS_EIO, e.what());
    } catch (const std::out_of_range& e) {
        return fail(VCS_ERANGE, e.what());
    } catch (const std::exception& e) {
        return fail(1, e.what());
    }
}

struct Converted {
    VccModel vcc;
    std::vector<BagOfTasks> bots;
};

Converted convert(const vcs_instance* in) {
    Converted c;
    for (int i = 0; i < in->n_clouds; ++i) {
        VehicularCloud cl;
        cl.id = in->cloud_id[i];
        cl.vm_total = in->cloud_vm_total[i];
        cl.vm_free = in->cloud_vm_free[i];
        cl.vm_throughput_kbps = in->cloud_thr_kbps[i];
        cl.v2i_delay_ms = in->cloud_delay_ms[i];
        c.vcc.clouds.push_back(cl);
    }
    c.vcc.reward_per_vc_vm = in->beta_vc;
    c.vcc.cost_per_tcc_vm = in->beta_tc;
    c.vcc.penalty_per_idle_vm = in->gamma_vc;
    auto task_at = [&](int j) {
        Task t;
        t.id = in->task_id[j];
        t.vm_demand = in->task_demand[j];
        t.max_delay_ms = in->task_max_delay_ms[j];
        t.min_vm_throughput_kbps = in->task_min_thr_kbps[j];
        return t;
    };
    if (in->n_bots > 0 && in->bot_task_offset) {
        for (int b = 0; b < in->n_bots; ++b) {
            BagOfTasks bot;
            bot.id = in->bot_id ? in->bot_id[b] : b + 1;
            for (int j = in->bot_task_offset[b]; j < in->bot_task_offset[b + 1]; ++j)
                bot.tasks.push_back(task_at(j));
            c.bots.push_back(std::move(bot));
        }
    } else if (in->n_tasks > 0) {
        BagOfTasks bot;
        bot.id = 1;
        for (int j = 0; j < in->n_tasks; ++j) bot.tasks.push_back(task_at(j));
        c.bots.push_back(std::move(bot));
    }
    return c;
}

struct RefSpace {
    MdpInstance inst;
    std::shared_ptr<const StateSpace> space;
};

struct RefResult {
    MdpInstance inst;
    ViResult vi;
};

MdpState make_state(const int32_t* free_vms, int n_clouds, int32_t t, uint8_t terminal) {
    MdpState s;
    s.free_vms.assign(free_vms, free_vms + n_clouds);
    s.next_task_index = t;
    s.terminal = terminal != 0;
    return s;
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_hardware_threads(void) {
    const unsigned n = std::thread::hardware_concurrency();
    return n == 0 ? 1 : static_cast<int>(n);
}

int ref_space_build(const vcs_instance* in, uint64_t cap, void** out, double* build_ms) {
    return guarded([&] {
        auto c = convert(in);
        auto h = std::make_unique<RefSpace>();
        h->inst = MdpInstance::from_workload(c.vcc, c.bots);
        const auto t0 = std::chrono::steady_clock::now();
        h->space = StateSpace::build(h->inst, static_cast<std::size_t>(cap));
        const auto t1 = std::chrono::steady_clock::now();
        if (build_ms) *build_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        *out = h.release();
        return VCS_OK;
    });
}

void ref_space_free(void* h) { delete static_cast<RefSpace*>(h); }

uint64_t ref_space_size(void* h) { return static_cast<RefSpace*>(h)->space->size(); }

int32_t ref_space_horizon(void* h) { return static_cast<RefSpace*>(h)->space->task_count(); }

void ref_space_layers(void* h, uint64_t* off) {
    const auto& sp = *static_cast<RefSpace*>(h)->space;
    for (int t = 0; t <= sp.task_count(); ++t) off[t] = sp.layer_begin(t);
    off[sp.task_count() + 1] = sp.layer_end(sp.task_count());
}

// detail::run_value_iteration on the prebuilt space (the reference's own timing convention,
// parallel_vi.cpp:126-147: build excluded, sweeps + extraction timed with steady_clock).
int ref_vi(void* h, double eps, int workers, void** res_out, int32_t* sweeps, double* ms) {
    return guarded([&] {
        auto* rs = static_cast<RefSpace*>(h);
        ViOptions opts;
        opts.epsilon = eps;
        const auto t0 = std::chrono::steady_clock::now();
        ViResult r = detail::run_value_iteration(rs->space, opts, workers);
        const auto t1 = std::chrono::steady_clock::now();
        if (ms) *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        if (sweeps) *sweeps = r.values.sweeps();
        *res_out = new RefResult{rs->inst, std::move(r)};
        return VCS_OK;
    });
}

void ref_res_free(void* r) { delete static_cast<RefResult*>(r); }

void ref_res_values(void* r, double* out) {
    const auto v = static_cast<RefResult*>(r)->vi.values.raw_values();
    std::memcpy(out, v.data(), v.size() * sizeof(double));
}

void ref_res_actions(void* r, int32_t* out) {
    const auto a = static_cast<RefResult*>(r)->vi.policy.raw_actions();
    std::memcpy(out, a.data(), a.size() * sizeof(int32_t));
}

int ref_res_initial_value(void* r, double* out) {
    return guarded([&] {
        *out = static_cast<RefResult*>(r)->vi.values.initial_value();
        return VCS_OK;
    });
}

int ref_res_value_of(void* r, const int32_t* free_vms, int32_t t, uint8_t terminal, double* out) {
    return guarded([&] {
        auto* rr = static_cast<RefResult*>(r);
        const int n = static_cast<int>(rr->inst.vcc.clouds.size());
        *out = rr->vi.values.value_of(make_state(free_vms, n, t, terminal));
        return VCS_OK;
    });
}

int ref_res_action_for(void* r, const int32_t* free_vms, int32_t t, uint8_t terminal,
                       int32_t* out) {
    return guarded([&] {
        auto* rr = static_cast<RefResult*>(r);
        const int n = static_cast<int>(rr->inst.vcc.clouds.size());
        *out = rr->vi.policy.action_for(make_state(free_vms, n, t, terminal)).target;
        return VCS_OK;
    });
}

// rollout (mdp.cpp:305-324); targets are cloud INDICES (or -1) so they compare with the
// product's vcs_greedy/rollout output; per_cloud_used is indexed by cloud position.
int ref_res_rollout(void* r, int32_t* targets, int64_t* per_cloud_used, int64_t* paid,
                    int64_t* unused, double* reward) {
    return guarded([&] {
        auto* rr = static_cast<RefResult*>(r);
        const auto res = rollout(rr->vi.policy, rr->inst);
        const auto& clouds = rr->inst.vcc.clouds;
        // The reference reports cloud ids; re-derive the index by replaying the policy.
        MdpState s = initial_state(rr->inst);
        std::size_t i = 0;
        while (!s.terminal) {
            const MdpAction a = rr->vi.policy.action_for(s);
            targets[i++] = a.target;
            s = transition(s, a, rr->inst);
        }
        if (per_cloud_used)
            for (std::size_t c = 0; c < clouds.size(); ++c)
                per_cloud_used[c] = res.per_vc_used.at(clouds[c].id);
        *paid = res.paid_vms;
        *unused = res.unused_vms;
        *reward = greedy_reward(res, rr->inst.vcc);
        return VCS_OK;
    });
}

// greedy_schedule + greedy_reward (greedy.cpp:5-36).  targets receive cloud IDS as the
// reference's PlacementRecord::target does (kPaidCloud for paid).
int ref_greedy(const vcs_instance* in, int32_t* target_ids, int32_t* vms_used, int64_t* paid,
               int64_t* unused, int64_t* placed, double* reward, double* ms) {
    return guarded([&] {
        auto c = convert(in);
        const auto t0 = std::chrono::steady_clock::now();
        const auto r = greedy_schedule(c.vcc, c.bots);
        const auto t1 = std::chrono::steady_clock::now();
        if (ms) *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        for (std::size_t i = 0; i < r.placements.size(); ++i) {
            target_ids[i] = r.placements[i].target;
            if (vms_used) vms_used[i] = r.placements[i].vms_used;
        }
        *paid = r.paid_vms;
        *unused = r.unused_vms;
        *placed = r.vc_placed_vms();
        *reward = greedy_reward(r, c.vcc);
        return VCS_OK;
    });
}

// ---- instance handles for bench.py's reference arm ------------------------------------------
// The reference arm must not load the product library, so it reads (or generates) its instance
// here, through the reference's own io.cpp parser, and builds/solves/places from the handle.
struct RefInstance {
    ParsedInstance p;
};

int ref_instance_load(const char* path, void** out) {
    return guarded([&] {
        auto h = std::make_unique<RefInstance>();
        h->p = load_instance(path); // io.cpp:97-101
        *out = h.release();
        return VCS_OK;
    });
}

int ref_instance_parse(const char* text, void** out) {
    return guarded([&] {
        auto h = std::make_unique<RefInstance>();
        std::istringstream in(text);
        h->p = parse_instance(in); // io.cpp:51-95
        *out = h.release();
        return VCS_OK;
    });
}

// The bench's seeded families, restated here for the reference arm (the product's generator is
// paper_2012_12419_b200/csrc/vcs_host.cpp gen_homog / gen_greedy; tests/test_host.py checks that
// both produce the same instance text).  kind 1 = HOMOG, 2 = GREEDY (C2).
int ref_instance_generate(int kind, uint64_t seed, int32_t a, int32_t b, int32_t c, int32_t d,
                          void** out) {
    return guarded([&] {
        auto h = std::make_unique<RefInstance>();
        std::mt19937_64 rng(seed);
        auto draw = [&](int lo, int hi) { return std::uniform_int_distribution<int>(lo, hi)(rng); };
        auto& vcc = h->p.vcc;
        if (kind == VCS_GEN_HOMOG) {
            for (int i = 0; i < a; ++i) {
                VehicularCloud cl;
                cl.id = i + 1;
                cl.vm_total = cl.vm_free = b;
                cl.vm_throughput_kbps = 100.0;
                cl.v2i_delay_ms = 10.0;
                vcc.clouds.push_back(cl);
            }
            const int n_bots = std::max(1, a);
            h->p.bots.resize(static_cast<std::size_t>(n_bots));
            for (int bi = 0; bi < n_bots; ++bi) h->p.bots[static_cast<std::size_t>(bi)].id = bi + 1;
            for (int t = 0; t < c; ++t) {
                Task task;
                task.id = t + 1;
                task.vm_demand = draw(1, d);
                task.max_delay_ms = 100.0;
                task.min_vm_throughput_kbps = 50.0;
                h->p.bots[static_cast<std::size_t>(t % n_bots)].tasks.push_back(task);
            }
        } else if (kind == VCS_GEN_GREEDY) {
            for (int i = 0; i < a; ++i) {
                VehicularCloud cl;
                cl.id = i + 1;
                cl.vm_total = cl.vm_free = draw(50, 150);
                cl.vm_throughput_kbps = draw(60, 160);
                cl.v2i_delay_ms = draw(5, 50);
                vcc.clouds.push_back(cl);
            }
            int id = 0;
            for (int bi = 0; bi < b; ++bi) {
                BagOfTasks bot;
                bot.id = bi + 1;
                for (int k = 0; k < c; ++k) {
                    Task task;
                    task.vm_demand = draw(1, d);
                    task.max_delay_ms = draw(5, 60);
                    task.min_vm_throughput_kbps = draw(50, 170);
                    task.id = ++id;
                    bot.tasks.push_back(task);
                }
                h->p.bots.push_back(std::move(bot));
            }
        } else {
            throw std::invalid_argument("unknown generator kind");
        }
        *out = h.release();
        return VCS_OK;
    });
}

void ref_instance_free(void* h) { delete static_cast<RefInstance*>(h); }

void ref_instance_counts(void* h, int32_t* n_clouds, int32_t* n_tasks) {
    const auto& p = static_cast<RefInstance*>(h)->p;
    *n_clouds = static_cast<int32_t>(p.vcc.clouds.size());
    *n_tasks = static_cast<int32_t>(flatten_tasks(p.bots).size());
}

// io.cpp:103-118 instance_text; returns the length, copies at most cap bytes.
uint64_t ref_instance_text(void* h, char* buf, uint64_t cap) {
    const std::string s = instance_text(static_cast<RefInstance*>(h)->p);
    if (buf) std::memcpy(buf, s.data(), std::min<std::size_t>(cap, s.size()));
    return s.size();
}

int ref_space_build_inst(void* inst, uint64_t cap, void** out, double* build_ms) {
    return guarded([&] {
        const auto& p = static_cast<RefInstance*>(inst)->p;
        auto h = std::make_unique<RefSpace>();
        h->inst = MdpInstance::from_workload(p.vcc, p.bots);
        const auto t0 = std::chrono::steady_clock::now();
        h->space = StateSpace::build(h->inst, static_cast<std::size_t>(cap));
        const auto t1 = std::chrono::steady_clock::now();
        if (build_ms) *build_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        *out = h.release();
        return VCS_OK;
    });
}

// greedy_schedule (greedy.cpp:5-30) timed with steady_clock; targets as cloud IDS.
int ref_greedy_inst(void* inst, int32_t* target_ids, int64_t* paid, int64_t* unused,
                    double* ms) {
    return guarded([&] {
        const auto& p = static_cast<RefInstance*>(inst)->p;
        const auto t0 = std::chrono::steady_clock::now();
        const auto r = greedy_schedule(p.vcc, p.bots);
        const auto t1 = std::chrono::steady_clock::now();
        if (ms) *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        for (std::size_t i = 0; i < r.placements.size(); ++i) target_ids[i] = r.placements[i].target;
        *paid = r.paid_vms;
        *unused = r.unused_vms;
        return VCS_OK;
    });
}

// The reference's DSRC simulator (sim.cpp run_simulation + vc_throughput, metrics.cpp:8-11
// per_vehicle_throughput): the per-vehicle service-channel share at a coverage density, used
// once by tools/c5_channel_table.py to tabulate tests/golden/c5_channel.json (the C5 sweep's
// channel-availability variants).  scheme 0 = static1609, 1 = aaa.
int ref_per_vehicle_kbps(int32_t n_vehicles, int32_t scheme, uint64_t seed, int64_t duration_ms,
                         double* out) {
    return guarded([&] {
        VanetScenario sc;
        sc.n_vehicles = n_vehicles;
        sc.scheme = scheme ? Scheme::kAaa : Scheme::kStatic1609;
        sc.rng_seed = seed;
        sc.sim_duration_ms = duration_ms;
        const SimTrace tr = run_simulation(sc);
        *out = per_vehicle_throughput(vc_throughput(tr), n_vehicles);
        return VCS_OK;
    });
}

// The reference CLI's run_schedule output file (tools/cli.cpp:43-61, 100-118; io.cpp:203-242)
// for scheduler 0 = greedy, 1 = mdp; format 0 = csv, 1 = json.  Returns the text length.
uint64_t ref_schedule_text(const char* path, int scheduler, double eps, int format, char* buf,
                           uint64_t cap) {
    std::string text;
    const int rc = guarded([&] {
        const auto p = load_instance(path);
        ScheduleResult res;
        std::optional<SolverDiagnostics> diag;
        if (scheduler == 0) {
            res = greedy_schedule(p.vcc, p.bots);
        } else {
            const auto mdp = MdpInstance::from_workload(p.vcc, p.bots);
            ViOptions o;
            o.epsilon = eps;
            const ViResult vi = value_iteration(mdp, o);
            res = rollout(vi.policy, mdp);
            diag = SolverDiagnostics{vi.values.epsilon(), vi.values.sweeps(),
                                     vi.values.states_explored()};
        }
        text = format == 1 ? schedule_json(res, p.vcc, diag) : schedule_csv(res, p.vcc, diag);
        return VCS_OK;
    });
    if (rc != VCS_OK) return 0;
    if (buf) std::memcpy(buf, text.data(), std::min<std::size_t>(cap, text.size()));
    return text.size();
}

// The reference's own parser (io.cpp:51-101), for cross-checking the product parser.
int ref_load_counts(const char* path, int32_t* n_clouds, int32_t* n_tasks, int32_t* n_bots) {
    return guarded([&] {
        const auto p = load_instance(path);
        *n_clouds = static_cast<int32_t>(p.vcc.clouds.size());
        *n_tasks = static_cast<int32_t>(flatten_tasks(p.bots).size());
        *n_bots = static_cast<int32_t>(p.bots.size());
        return VCS_OK;
    });
}

} // extern "C"

// ---- the reference's own test oracles (tests/testutil.hpp, compiled from /root/reference) ----
#include "testutil.hpp"

extern "C" {

// testutil::random_instance(rng, {a,b,c,d}) drawn `trial`+1 times from one rng(seed).  Writes the
// FLATTENED instance (flatten_tasks order) into caller buffers of capacity a clouds / c tasks.
int ref_random_instance(uint64_t seed, int32_t trial, int32_t a, int32_t b, int32_t c, int32_t d,
                        int32_t* n_clouds, int32_t* cloud_cap, double* cloud_delay,
                        double* cloud_thr, int32_t* n_tasks, int32_t* task_id,
                        int32_t* task_demand, double* task_delay, double* task_thr,
                        int32_t* n_bots, int32_t* bot_sizes) {
    std::mt19937_64 rng(seed);
    testutil::RandomInstance r;
    for (int i = 0; i <= trial; ++i) r = testutil::random_instance(rng, {a, b, c, d});
    *n_clouds = static_cast<int32_t>(r.vcc.clouds.size());
    for (std::size_t i = 0; i < r.vcc.clouds.size(); ++i) {
        cloud_cap[i] = r.vcc.clouds[i].vm_total;
        cloud_delay[i] = r.vcc.clouds[i].v2i_delay_ms;
        cloud_thr[i] = r.vcc.clouds[i].vm_throughput_kbps;
    }
    const auto tasks = flatten_tasks(r.bots);
    *n_tasks = static_cast<int32_t>(tasks.size());
    for (std::size_t j = 0; j < tasks.size(); ++j) {
        task_id[j] = tasks[j].id;
        task_demand[j] = tasks[j].vm_demand;
        task_delay[j] = tasks[j].max_delay_ms;
        task_thr[j] = tasks[j].min_vm_throughput_kbps;
    }
    *n_bots = static_cast<int32_t>(r.bots.size());
    for (std::size_t b = 0; b < r.bots.size(); ++b)
        bot_sizes[b] = static_cast<int32_t>(r.bots[b].tasks.size());
    return VCS_OK;
}

// testutil::brute_force_optimum: exhaustive search, independent of the solver.
int ref_brute_force(const vcs_instance* in, double* out) {
    return guarded([&] {
        auto c = convert(in);
        *out = testutil::brute_force_optimum(MdpInstance::from_workload(c.vcc, c.bots));
        return VCS_OK;
    });
}

// testutil::FullStateReference value/action of a full state (memoised full-state recursion).
int ref_full_state(const vcs_instance* in, const int32_t* free_vms, int32_t t, double* value,
                   int32_t* action) {
    return guarded([&] {
        auto c = convert(in);
        const auto inst = MdpInstance::from_workload(c.vcc, c.bots);
        testutil::FullStateReference fr(inst);
        MdpState s = make_state(free_vms, static_cast<int>(c.vcc.clouds.size()), t,
                                t == static_cast<int>(inst.tasks.size()));
        *value = fr.value(s);
        *action = fr.best_action(s);
        return VCS_OK;
    });
}

} // extern "C"
