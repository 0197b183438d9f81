/*
 * vcs_gpu.h — C ABI of the B200-native vehicular-cloud placement solver.
 *
 * This is the drop-in boundary for the reference's solver path
 * (reference: /root/reference/proj/core/include/vcsched/{workload,mdp,parallel_vi,greedy}.hpp).
 * Every entry point below names the reference interface it replaces (file:line, relative to
 * /root/reference/proj).  Plain C types only: the caller owns every input and output buffer,
 * the library owns the device memory behind a `vcs_space` handle.
 *
 * Status codes mirror the reference CLI exit codes (tools/cli.hpp:30-33, tools/cli.cpp:225-240):
 *   VCS_OK 0, VCS_EINVAL 2 (std::invalid_argument / ConfigError), VCS_ECAP 3 (StateCapacityError),
 *   VCS_EIO 4 (IoError), VCS_ECUDA 5 (CUDA runtime / device failure), VCS_ERANGE 6 (std::out_of_range).
 * The message of the last failure on the calling thread is returned by vcs_last_error(); the
 * messages of the reference exceptions are reproduced verbatim (e.g. "reachable state space
 * exceeds cap of N states", mdp.hpp:58-68).
 *
 * Threading: every call is synchronous and re-entrant.  The solve, query and rollout entry points
 * serialise on a per-space lock, so threads may share one handle (as the reference's
 * shared_ptr<const StateSpace> allows); a vcs_solve_enqueue / vcs_solve_collect PAIR is two
 * calls, and a caller interleaving pairs from several threads must order them itself.
 */
#ifndef VCS_GPU_H
#define VCS_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VCS_OK 0
#define VCS_EINVAL 2
#define VCS_ECAP 3
#define VCS_EIO 4
#define VCS_ECUDA 5
#define VCS_ERANGE 6

/* Sentinel target for the paid traditional cloud (workload.hpp:46 kPaidCloud). */
#define VCS_PAID_CLOUD (-1)

/*
 * A placement problem in canonical order (mdp.hpp:18-23 MdpInstance; workload.hpp:12-43).
 * Structure-of-arrays view; nothing is copied until a call needs it.
 *   clouds: VehicularCloud{id, vm_total, vm_free, vm_throughput_kbps, v2i_delay_ms}
 *   tasks : the FLATTENED task sequence (workload.cpp:28-33 flatten_tasks): bags in order,
 *           tasks in order.  bot_task_offset (n_bots+1 entries, may be NULL) records the bag
 *           boundaries for round trips; the solver and greedy only need the flat order.
 *   beta_vc / beta_tc / gamma_vc: reward_per_vc_vm, cost_per_tcc_vm, penalty_per_idle_vm.
 */
typedef struct vcs_instance {
    int32_t n_clouds;
    const int32_t* cloud_id;
    const int32_t* cloud_vm_total;
    const int32_t* cloud_vm_free;
    const double* cloud_thr_kbps;
    const double* cloud_delay_ms;
    int32_t n_tasks;
    const int32_t* task_id;
    const int32_t* task_demand;
    const double* task_max_delay_ms;
    const double* task_min_thr_kbps;
    int32_t n_bots;
    const int32_t* bot_id;          /* may be NULL when n_bots == 0 */
    const int32_t* bot_task_offset; /* n_bots + 1 entries, may be NULL when n_bots == 0 */
    double beta_vc;
    double beta_tc;
    double gamma_vc;
} vcs_instance;

/* ------------------------------------------------------------------------------------------ */
/* Instance ingestion (host)                                                                   */
/* ------------------------------------------------------------------------------------------ */

/* An instance owned by the library (parsed or generated).  vcs_instance_view() returns a view
 * whose pointers stay valid until vcs_instance_free(). */
typedef struct vcs_instance_owned vcs_instance_owned;

/* Replaces io.cpp:51-95 parse_instance (grammar of io.hpp:33-40; vm_free = vm_total, io.cpp:71;
 * validate() of workload.cpp:35-57).  Errors: VCS_EINVAL with the ConfigError text. */
int vcs_instance_parse(const char* text, vcs_instance_owned** out);
/* Replaces io.cpp:97-101 load_instance.  Errors: VCS_EIO "cannot read instance file: <path>". */
int vcs_instance_load(const char* path, vcs_instance_owned** out);
/* Build an owned copy of a caller view (runs validate()). */
int vcs_instance_copy(const vcs_instance* in, vcs_instance_owned** out);
const vcs_instance* vcs_instance_view(const vcs_instance_owned* inst);
void vcs_instance_free(vcs_instance_owned* inst);

/* Seeded synthetic instances (std::mt19937_64 + libstdc++ uniform_int_distribution, so the
 * same seed yields the same instance as the reference's generators).
 *   kind VCS_GEN_RANDOM : tests/testutil.hpp:28-65 random_instance(rng, {a,b,c,d}); the
 *                         `trial`-th instance drawn from one rng seeded with `seed`.
 *   kind VCS_GEN_HOMOG  : SURVEY §8(d) C3/C4 family: a clouds {vm_total b, thr 100, delay 10},
 *                         c tasks {demand U[1,d], max_delay 100, min_thr 50}, a bags round-robin.
 *   kind VCS_GEN_GREEDY : SURVEY §8(d) C2: a clouds {U[50,150] VMs, thr U[60,160], delay U[5,50]},
 *                         b bags x c tasks {demand U[1,d], max_delay U[5,60], min_thr U[50,170]}. */
#define VCS_GEN_RANDOM 0
#define VCS_GEN_HOMOG 1
#define VCS_GEN_GREEDY 2
int vcs_instance_generate(int kind, uint64_t seed, int32_t trial, int32_t a, int32_t b, int32_t c,
                          int32_t d, vcs_instance_owned** out);

/* ------------------------------------------------------------------------------------------ */
/* State space (device)                                                                        */
/* ------------------------------------------------------------------------------------------ */

typedef struct vcs_space vcs_space;

typedef struct vcs_space_info {
    uint64_t n_states;  /* StateSpace::size() (mdp.hpp:88) */
    uint64_t n_edges;
    int32_t horizon;    /* StateSpace::task_count() (mdp.hpp:89) */
    int32_t key_words;  /* 64-bit words per packed reduced key */
    uint64_t max_layer; /* largest layer, states */
    int32_t max_degree; /* largest out-degree */
    int32_t device;
    double build_ms;    /* device build time (CUDA events) */
    uint64_t device_bytes; /* resident bytes of the CSR + value buffers */
} vcs_space_info;

/* Replaces mdp.cpp:81-214 StateSpace::build.  The layered reachable-state enumeration runs on
 * `device`; the CSR (row_ptr, succ, reward, action) and the per-layer packed keys stay resident
 * in HBM.  Enumeration order, edge order (clouds ascending then paid), successor indices and
 * fp64 reward bits equal the reference's.  Errors: VCS_ECAP "reachable state space exceeds cap
 * of N states"; VCS_EINVAL "cloud free counts above 65535 are not supported". */
int vcs_space_build(const vcs_instance* inst, uint64_t state_cap, int device, vcs_space** out);
/* Test seam: upload an externally built CSR (e.g. the oracle's) instead of building it, so the
 * solver can be validated independently of the builder.  row_ptr has n_states+1 entries,
 * layer_offset horizon+2 entries (mdp.hpp:119-128 layout). */
int vcs_space_from_csr(uint64_t n_states, uint64_t n_edges, int32_t horizon,
                       const uint64_t* layer_offset, const uint64_t* row_ptr, const uint32_t* succ,
                       const double* reward, const int32_t* action, int device, vcs_space** out);
int vcs_space_info_get(const vcs_space* sp, vcs_space_info* info);
/* layer_offset: horizon+2 entries (StateSpace::layer_begin/layer_end, mdp.hpp:90-91). */
int vcs_space_layer_offsets(const vcs_space* sp, uint64_t* layer_offset);
/* Download the CSR (any pointer may be NULL to skip that array). */
int vcs_space_csr(const vcs_space* sp, uint64_t* row_ptr, uint32_t* succ, double* reward,
                  int32_t* action);
/* Replaces mdp.cpp:227-234 StateSpace::locate for a batch of full states.  free_vms is
 * n x n_clouds (row-major), task_index the next_task_index, terminal 0/1.  idx_out[i] receives
 * the flat state index, or -1 when the state is not reachable (the reference throws
 * std::out_of_range "state not reachable in enumerated space"). */
int vcs_space_locate(vcs_space* sp, int64_t n, const int32_t* free_vms, const int32_t* task_index,
                     const uint8_t* terminal, int64_t* idx_out);
/* Batched policy queries: ValueTable::value_of and Policy::action_for
 * (mdp.cpp:227-282) for n full states at once, served from the device-resident results of the
 * last collected solve on this space (vcs_solve, or vcs_solve_enqueue + vcs_solve_collect).
 * Keys are packed, located and the hidden penalty applied on the device.  value_out[i] =
 * V(locate(s)) - hidden_penalty(s), NaN when s is unreachable (the reference throws
 * std::out_of_range); action_out[i] = the cloud index or VCS_PAID_CLOUD, VCS_NO_ACTION for
 * unreachable or terminal states (action_for throws); idx_out[i] = the flat index or -1.  Every
 * array may live in host or device memory (device arrays are used in place); any output may be
 * NULL.  Returns after the outputs are complete when any of them is in host memory. */
#define VCS_NO_ACTION (-2)
int vcs_policy_query(vcs_space* sp, int64_t n, const int32_t* free_vms, const int32_t* task_index,
                     const uint8_t* terminal, double* value_out, int32_t* action_out,
                     int64_t* idx_out, void* stream);
/* Replaces mdp.cpp:305-324 rollout's policy walk: applies the last collected solve's policy on
 * this space from the initial state (inst = the instance the space was built from), on the
 * device — one kernel walks the H decisions through the device key index.  target_per_task[t]
 * receives the cloud index chosen for flattened task t, or VCS_PAID_CLOUD.  VCS_ERANGE when a
 * visited state is not enumerated (the reference throws std::out_of_range). */
int vcs_rollout(vcs_space* sp, const vcs_instance* inst, int32_t* target_per_task, void* stream);
/* Incremented whenever a collected solve replaces the device-resident results that
 * vcs_policy_query / vcs_rollout read (callers holding older host results compare it). */
uint64_t vcs_space_result_generation(const vcs_space* sp);
/* Replaces mdp.cpp:236-243 StateSpace::hidden_penalty for a batch of full states. */
int vcs_space_hidden_penalty(const vcs_space* sp, int64_t n, const int32_t* free_vms,
                             const int32_t* task_index, const uint8_t* terminal, double* out);
void vcs_space_free(vcs_space* sp);

/* ------------------------------------------------------------------------------------------ */
/* Value iteration (device)                                                                    */
/* ------------------------------------------------------------------------------------------ */

typedef struct vcs_solve_opts {
    double epsilon;         /* ViOptions::epsilon (mdp.hpp:131-134), default 1e-6 */
    int32_t skip_converged; /* 1: skip layers proven exact (bit-identical) */
    int32_t max_sweeps;     /* 0 = no cap (the reference has none) */
    double discount;        /* 1.0 = the reference's undiscounted backup (mdp.cpp:255).  Any
                               other value is the labelled EXTENSION q = r + discount*V(s')
                               (BASELINE.json configs[0] "gamma=0.9"); it has no reference
                               counterpart and is checked against the C oracle only. */
    int32_t method;         /* VCS_METHOD_AUTO (= VCS_METHOD_CERTIFIED when the wavefront's version
                               store fits in half of the HBM, else Jacobi), VCS_METHOD_JACOBI (one
                               kernel per sweep), VCS_METHOD_WAVEFRONT (all truncation horizons,
                               one pass) or VCS_METHOD_CERTIFIED (one backward pass with the two
                               top versions of every state; when it proves that no sweep k <= H
                               reaches delta < epsilon the result is final, otherwise the
                               wavefront runs).  All give identical bits. */
} vcs_solve_opts;

#define VCS_METHOD_AUTO 0
#define VCS_METHOD_JACOBI 1
#define VCS_METHOD_WAVEFRONT 2
#define VCS_METHOD_CERTIFIED 3

typedef struct vcs_solve_report {
    int32_t sweeps;            /* ValueTable::sweeps() */
    int32_t launches;          /* device kernel launches issued by the solve */
    uint64_t backups_ref;      /* reference-equivalent backups = n_states * sweeps */
    uint64_t backups_done;     /* backups actually performed (layer skip) */
    double sweep_ms;           /* sweeps only, CUDA events */
    double extract_ms;         /* policy extraction, CUDA events */
    double alg_bytes;          /* SURVEY §8(d) algorithmic bytes of the sweeps: (24+12 d) per backup_ref */
    double alg_bytes_done;     /* same formula over the performed backups */
    int32_t method;            /* the method that ran: VCS_METHOD_JACOBI, _WAVEFRONT, or _CERTIFIED
                                  (the certificate held: one backward pass was the whole solve) */
    int32_t fallback_deferred; /* 1: the certificate failed on an implicit-form space and the
                                  wavefront fallback ran inside vcs_solve_collect (see
                                  vcs_solve_enqueue); 0 otherwise */
    double model_bytes;        /* minimum HBM bytes of the method that ran: Jacobi = alg_bytes_done
                                  with the u32 row_ptr layout; wavefront = CSR once + every
                                  version written and read once + the extraction pass */
} vcs_solve_report;

/* Replaces parallel_vi.cpp:48-116 detail::run_value_iteration (the sweep loop, the sup-norm
 * residual `delta < epsilon`, buffer parity, and the argmax extraction of
 * parallel_vi.cpp:109-111).  values_out (n_states f64) and actions_out (n_states i32) may be
 * NULL.  Bit-identical to the reference for every epsilon (same sweep count).
 * With PINNED (cudaHostAlloc) outputs the results stream to the host while the layer pass runs;
 * for spaces of <= 127 clouds the action column crosses PCIe as int8 and is widened into
 * actions_out by library-owned host threads (VCS_HOST_WORKERS, default 7; VCS_NO_NARROW=1
 * disables it).  The call returns after every output byte is written. */
int vcs_solve(vcs_space* sp, const vcs_solve_opts* opts, double* values_out, int32_t* actions_out,
              vcs_solve_report* report);
/* The same solve split in two for callers that overlap or time it on their own stream
 * (a cudaStream_t; NULL = the space's stream): vcs_solve_enqueue launches the solve (one CUDA
 * graph) without synchronising; vcs_solve_collect waits for it, downloads the results of the
 * LAST enqueued solve and fills the report.  vcs_solve = enqueue + collect.
 * What enqueue launches: Jacobi / wavefront: the whole solve.  Certified pass on an explicit
 * CSR: the pass plus, as a graph IF node, the wavefront fallback (the whole solve).  Certified
 * pass on the IMPLICIT form (the default for dense spaces) and the multi-GPU pass: the pass and
 * its certificate only; when the certificate fails (an early stop is possible, or a sweep cap
 * below horizon+1), collect materialises the explicit CSR and runs the wavefront before it
 * returns, and sets report->fallback_deferred = 1.  Timing enqueue alone is therefore exact
 * only when the report says method == VCS_METHOD_CERTIFIED. */
int vcs_solve_enqueue(vcs_space* sp, const vcs_solve_opts* opts, void* stream);
int vcs_solve_collect(vcs_space* sp, double* values_out, int32_t* actions_out,
                      vcs_solve_report* report, void* stream);

/* Multi-GPU certified solve: ONE state space sharded across n_ranks GPUs of this
 * process — the B200 replacement of the block-parallel driver (parallel_vi.cpp:68-107,
 * BlockPartition::even :11-24, SweepBarrier :34-44): GPUs instead of std::threads, contiguous
 * shares of every large layer's pair index space (key space, or BFS rows of an explicit CSR)
 * instead of row blocks of the whole space, and per-layer peer copies over NVLink instead of the
 * shared-memory flush + barriers.  devices[r] is rank r's CUDA device (NULL = space device,
 * then the next ones); a device may repeat (several ranks on one GPU: the emulated-rank test
 * mode).  exchange: VCS_EXCHANGE_HALO pulls only the successor window a rank reads (forward halo
 * on non-retiring transitions of the key space), VCS_EXCHANGE_ALLGATHER every layer in full (the
 * north-star all-gather, kept for comparison).  Values, actions and sweeps are bit-identical to
 * vcs_solve for every n_ranks; the results land in the space's device (the primary), and
 * vcs_solve_collect downloads them (and runs the single-GPU fallback when the certificate does
 * not hold).  n_ranks == 1 on the space's device is vcs_solve_enqueue.  Methods AUTO/CERTIFIED
 * only (VCS_EINVAL otherwise). */
#define VCS_EXCHANGE_HALO 0
#define VCS_EXCHANGE_ALLGATHER 1
int vcs_solve_multi_enqueue(vcs_space* sp, const vcs_solve_opts* opts, int32_t n_ranks,
                            const int32_t* devices, int32_t exchange, void* stream);
/* = vcs_solve_multi_enqueue + vcs_solve_collect (values_out / actions_out host or NULL). */
int vcs_solve_multi(vcs_space* sp, const vcs_solve_opts* opts, int32_t n_ranks,
                    const int32_t* devices, int32_t exchange, double* values_out,
                    int32_t* actions_out, vcs_solve_report* report);
typedef struct vcs_multi_report {
    int32_t n_ranks;
    int32_t split_layers;      /* layers divided between the ranks */
    int32_t replicated_layers; /* small / sparse layers every rank computes whole */
    int32_t exchange;
    double halo_bytes;         /* pair bytes copied between ranks per solve */
    double max_share;          /* largest rank share of the divided work (1/n_ranks = balanced) */
    int32_t graph;             /* 1: the pass is one CUDA graph; 0: direct launches */
    int32_t pad;
} vcs_multi_report;
int vcs_multi_info(const vcs_space* sp, vcs_multi_report* out);

/* The same pass with one rank per PROCESS (torchrun, one GPU each; the caller moves the windows
 * between processes, e.g. torch.distributed over NCCL — paper_2012_12419_b200/sharded.py
 * run_cert_sharded).  Every rank holds the whole space:
 *   begin(opts, world, rank, exchange)   zero this rank's pairs / bounds / outputs (enqueued)
 *   for t = horizon-1 .. 0:
 *       layer(t)                          this rank's range of layer t (or all of a replicated one)
 *       if plan(t).split and t > 0:       rank q sends [max(need_lo_h, lo_q), min(need_hi_h, hi_q))
 *                                         of pairs(t) (2 doubles per index) to every rank h
 *   all-reduce(lb, MAX); finish(lb) -> certified
 *   certified: SUM-all-reduce the int64 view of values and the actions (every element is written
 *              by exactly one rank, the others hold 0) = vcs_solve's result, sweeps = horizon+1;
 *   otherwise: run vcs_solve (the fallback) on any rank.
 * plan(t, q) out[6] = {split, lo_q, hi_q, need_lo_q, need_hi_q, index-space size of layer t}. */
int vcs_cert_shard_begin(vcs_space* sp, const vcs_solve_opts* opts, int32_t world, int32_t rank,
                         int32_t exchange, void* stream);
int vcs_cert_shard_plan(const vcs_space* sp, int32_t t, int32_t q, uint64_t* out);
int vcs_cert_shard_layer(vcs_space* sp, int32_t t, void* stream);
int vcs_cert_shard_pairs(const vcs_space* sp, int32_t t, double** pairs);
int vcs_cert_shard_buffers(const vcs_space* sp, double** lb, double** values, int32_t** actions);
int vcs_cert_shard_finish(const vcs_space* sp, const double* lb_max, int32_t* certified);

/* Sharded (multi-GPU) building blocks.  One process per GPU; the host runtime owns the value
 * buffers and the collectives (torch.distributed / NCCL over NVLink), these calls only enqueue
 * device work on `stream` (a cudaStream_t; NULL = the space's own stream) and never synchronise
 * except vcs_shard_finish.  Together they replace the block-parallel worker of
 * parallel_vi.cpp:68-107 (BlockPartition + SweepBarrier + per-block residual fold).
 *   vcs_shard_plan   : host-only.  Row block [row_begin,row_end) of `rank` (contiguous, balanced
 *                      on the per-layer edge/state cost; skip_weighted also weights a layer by
 *                      the number of sweeps that visit it) and the forward halo
 *                      [halo_begin,halo_end) of successor rows owned by later ranks.
 *   vcs_shard_begin  : adopt caller-owned device buffers v0/v1 (n_states f64 each) and delta
 *                      (n_delta >= horizon+3 f64: slot k = residual of sweep k); zero them.
 *   vcs_shard_sweep  : sweep k (1-based) over [row_begin,row_end) reading v[(k-1)&1], writing
 *                      v[k&1] and the block residual into delta[k] (atomic max).  The host
 *                      all-reduces delta[k] (MAX) and exchanges the halo before sweep k+1, whose
 *                      prologue evaluates `delta[k] < eps` on the device (no host round trip).
 *   vcs_shard_finish : policy extraction over [row_begin,row_end) from the converged buffer and
 *                      download of that block's values/actions into the host arrays (indexed by
 *                      flat state); *sweeps_out = the converged sweep count. */
int vcs_shard_plan(const uint64_t* layer_offset, const uint64_t* layer_edges, int32_t horizon,
                   int32_t world, int32_t rank, int32_t skip_weighted, uint64_t* row_begin,
                   uint64_t* row_end, uint64_t* halo_begin, uint64_t* halo_end);
int vcs_space_layer_edges(const vcs_space* sp, uint64_t* layer_edges); /* horizon+1 entries */
int vcs_shard_begin(vcs_space* sp, double* v0, double* v1, double* delta, int32_t n_delta,
                    void* stream);
int vcs_shard_sweep(vcs_space* sp, int32_t k, uint64_t row_begin, uint64_t row_end,
                    const vcs_solve_opts* opts, void* stream);
int vcs_shard_finish(vcs_space* sp, int32_t n_sweeps, uint64_t row_begin, uint64_t row_end,
                     const vcs_solve_opts* opts, double* values_out, int32_t* actions_out,
                     int32_t* sweeps_out, void* stream);

/* Version-band sharding of the layer wavefront (the multi-GPU form of VCS_METHOD_WAVEFRONT).
 * Rank r of `world` computes versions [lo_t, hi_t) = [1 + r*m_t/world, 1 + (r+1)*m_t/world) of
 * every layer t (m_t = horizon - t, integer division).  Its band of layer t needs only its own
 * band of layer t+1 plus ONE column below it (version lo_{t+1}-1, owned by a lower rank), so
 * the per-layer exchange is one n_t-double column per rank.  Host driver (one process per GPU):
 *   begin(world, rank, opts, delta)      delta: caller-owned device array of horizon+3 doubles
 *   for t = horizon-1 .. 0:
 *       layer(t)                          the rank's band of layer t
 *       for every rank d with lo_t(d) > 1: owner q of version lo_t(d)-1 packs it (pack) and
 *                                         sends n_t doubles to d, which unpacks it (unpack)
 *   all-reduce(delta, MAX); K* = first k with delta[k] < eps (else horizon+1)
 *   finish(K*)                            early-stop fix-up + this rank's rows to the host
 * The results are bit-identical to vcs_solve for every world size.  Replaces the same
 * block-parallel worker (parallel_vi.cpp:68-107) as vcs_shard_*, with the wavefront's work. */
int vcs_wave_shard_begin(vcs_space* sp, int32_t world, int32_t rank, const vcs_solve_opts* opts,
                         double* delta, void* stream);
int vcs_wave_shard_band(const vcs_space* sp, int32_t t, int32_t* lo, int32_t* hi);
int vcs_wave_shard_layer(vcs_space* sp, int32_t t, void* stream);
int vcs_wave_shard_pack(vcs_space* sp, int32_t t, int32_t version, double* dst, void* stream);
int vcs_wave_shard_unpack(vcs_space* sp, int32_t t, const double* src, void* stream);
/* values_out / actions_out: host arrays of n_states; this rank writes exactly the rows it is
 * responsible for (every row is written by one rank), the rest is left untouched. */
int vcs_wave_shard_finish(vcs_space* sp, int32_t K, double* values_out, int32_t* actions_out,
                          void* stream);

/* ------------------------------------------------------------------------------------------ */
/* Greedy placement (device)                                                                   */
/* ------------------------------------------------------------------------------------------ */

/* Replaces greedy.cpp:5-30 greedy_schedule (Alg. 2 first-fit).  target_per_task[i] receives the
 * cloud INDEX (position in the cloud list) of flattened task i, or VCS_PAID_CLOUD;
 * per_cloud_used (n_clouds entries, may be NULL) the VMs placed per cloud index; *paid and
 * *unused as ScheduleResult::paid_vms / unused_vms (unused = total_capacity - placed,
 * greedy.cpp:28).  Placements are bit-exact against the reference. */
int vcs_greedy(const vcs_instance* inst, int device, int32_t* target_per_task,
               int64_t* per_cloud_used, int64_t* paid, int64_t* unused);
/* n independent instances in one launch (one warp each). */
int vcs_greedy_batch(int32_t n, const vcs_instance* insts, int device, int32_t** target_per_task,
                     int64_t* paid, int64_t* unused);
/* greedy.cpp:32-36 greedy_reward. */
double vcs_greedy_reward(const vcs_instance* inst, int64_t placed, int64_t paid, int64_t unused);

/* ------------------------------------------------------------------------------------------ */
/* Host memory                                                                                 */
/* ------------------------------------------------------------------------------------------ */

/* Page-locked host memory from the library's recycled pool (cudaHostAlloc costs milliseconds per
 * call; blocks are reused across calls).  Outputs of vcs_solve in such memory stream to the host
 * while the layer pass runs.  NULL on failure.  The C++ drop-in keeps ValueTable / Policy
 * storage here. */
void* vcs_host_alloc(uint64_t bytes);
void vcs_host_free(void* p);

/* ------------------------------------------------------------------------------------------ */
/* Diagnostics                                                                                 */
/* ------------------------------------------------------------------------------------------ */

const char* vcs_last_error(void);
/* Number of device kernels this library launched on the calling process so far. */
uint64_t vcs_kernel_launches(void);
/* 1 when a CUDA device is usable, else 0 (no kernel is launched). */
int vcs_device_count(void);

#ifdef __cplusplus
}
#endif
#endif /* VCS_GPU_H */
