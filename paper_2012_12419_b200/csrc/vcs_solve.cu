// vcs_solve.cu — fp64 Jacobi value iteration on the device (replaces
// detail::run_value_iteration, parallel_vi.cpp:48-116, and StateSpace::backup, mdp.cpp:245-263).
//
// One sweep = one kernel.  A warp owns 32 consecutive rows: it stages the rows' contiguous edge
// range with coalesced, streaming (evict-first) loads of succ/reward, gathers V_prev[succ]
// (L2-resident: successors of layer t live in layer t+1), writes q = r + V into shared memory,
// then every lane scans ITS row in edge order with the reference's strict '>' (first maximum
// wins — exact action AND value bits, incl. signed zero).  The sup-norm residual is reduced
// warp -> block -> one atomicMax per block on the u64 image of the (non-negative) double.
//
// The whole solve (zeroing, up to H+1 sweeps, extraction) is one CUDA graph; the convergence
// test `delta < eps` (parallel_vi.cpp:66) is evaluated ON THE DEVICE in the prologue of the
// next sweep kernel, which turns every later sweep into a no-op — no host round trip per sweep.
//
// Converged-layer skip (opts.skip_converged): the state graph is a layered DAG
// (edges go t -> t+1, mdp.cpp:190/201) and V starts at 0, so after sweep k every layer
// t >= H-k holds its exact value and recomputing it reproduces identical bits with zero
// residual.  Sweep k therefore only visits layers 0..min(H, H-k+1) (the +1 keeps both ping-pong
// buffers exact).  Values, actions and the sweep count are bit-identical with and without it.
#include "vcs_device.cuh"

#include <algorithm>
#include <cmath>

namespace vcs {

namespace {

constexpr int kWarpsMax = 8;

struct SweepArgs {
    const uint32_t* __restrict__ row_ptr;
    const uint32_t* __restrict__ succ;
    const double* __restrict__ reward;
    const int32_t* __restrict__ action;
    const double* v0;
    double* v1;
    double* delta;
    SolveCtrl* ctrl;
    uint32_t row_begin;
    uint32_t row_end;
    int k;         // sweep number (1-based); for extraction: sweeps launched
    int qcap;      // q slots per row (max out-degree)
    double eps;
    double discount;
    int32_t* act_out;
};

__device__ __forceinline__ double qval(double r, double v, double disc, bool discounted) {
    return discounted ? __dadd_rn(r, __dmul_rn(disc, v)) : __dadd_rn(r, v);
}

// Processes rows [a.row_begin, a.row_end) reading `vprev`.  SWEEP: writes vnext + residual.
// EXTRACT: writes the argmax action (mdp.cpp:256-258 tie-break) to a.act_out.
template <bool EXTRACT, bool DISC>
__device__ __forceinline__ double process_rows(const SweepArgs& a, const double* __restrict__ vprev,
                                               double* __restrict__ vnext, double* qw) {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int U = 8;
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t n_warps = (gridDim.x * blockDim.x) >> 5;
    double dmax = 0.0;
    for (uint64_t r0 = static_cast<uint64_t>(a.row_begin) + static_cast<uint64_t>(warp) * 32;
         r0 < a.row_end; r0 += static_cast<uint64_t>(n_warps) * 32) {
        const uint32_t r = static_cast<uint32_t>(r0) + lane;
        const bool valid = r < a.row_end;
        const uint32_t eb = __ldg(a.row_ptr + (valid ? r : a.row_end));
        uint32_t ee = __shfl_down_sync(FULL, eb, 1);
        if (lane == 31) ee = valid ? __ldg(a.row_ptr + r + 1) : eb;
        const uint32_t w0 = __shfl_sync(FULL, eb, 0);
        const uint32_t w1 = __shfl_sync(FULL, ee, 31);
        // Stage q = r + V_prev[succ] for the warp's whole edge range (coalesced).
        for (uint32_t base = w0; base < w1; base += 32 * U) {
            uint32_t sidx[U];
            double rw[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t e = base + u * 32 + lane;
                if (e < w1) {
                    sidx[u] = __ldcs(a.succ + e);
                    rw[u] = __ldcs(a.reward + e);
                }
            }
            double v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t e = base + u * 32 + lane;
                if (e < w1) v[u] = __ldg(vprev + sidx[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t e = base + u * 32 + lane;
                if (e < w1) qw[e - w0] = qval(rw[u], v[u], a.discount, DISC);
            }
        }
        __syncwarp();
        if (valid) {
            double best;
            uint32_t best_e = 0xffffffffu;
            if (eb == ee) {
                best = 0.0; // terminal (mdp.cpp:248-251)
            } else {
                best = -INFINITY;
                for (uint32_t e = eb; e < ee; ++e) {
                    const double q = qw[e - w0];
                    if (q > best) { // strict: the first maximal edge wins
                        best = q;
                        best_e = e;
                    }
                }
            }
            if constexpr (EXTRACT) {
                a.act_out[r] = best_e == 0xffffffffu ? -1 : __ldg(a.action + best_e);
            } else {
                const double d = fabs(best - vprev[r]);
                dmax = dmax < d ? d : dmax;
                vnext[r] = best;
            }
        }
        __syncwarp();
    }
    return dmax;
}

__device__ __forceinline__ void reduce_residual(double dmax, double* slot) {
    __shared__ double red[kWarpsMax];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(0xffffffffu, dmax, o);
        dmax = dmax < other ? other : dmax;
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[w] = dmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = red[0];
        for (int i = 1; i < static_cast<int>(blockDim.x >> 5); ++i) m = m < red[i] ? red[i] : m;
        // residuals are >= 0, so the u64 image orders like the double
        if (m > 0.0)
            atomicMax(reinterpret_cast<unsigned long long*>(slot),
                      static_cast<unsigned long long>(__double_as_longlong(m)));
    }
}

template <bool DISC>
__global__ void __launch_bounds__(kWarpsMax * 32) k_sweep(SweepArgs a) {
    extern __shared__ double qbuf[];
    // Device-side convergence test of the previous sweep (parallel_vi.cpp:61/66): once a
    // residual fell below eps, this and every later sweep is a no-op.
    if (a.ctrl->stop) return;
    if (a.k > 1) {
        const double prev_delta = a.delta[a.k - 1];
        if (prev_delta < a.eps) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                a.ctrl->stop = 1;
                a.ctrl->sweeps = a.k - 1;
            }
            return;
        }
    }
    const double* vprev = ((a.k - 1) & 1) ? a.v1 : a.v0;
    double* vnext = (a.k & 1) ? a.v1 : const_cast<double*>(a.v0);
    double* qw = qbuf + (threadIdx.x >> 5) * 32 * a.qcap;
    const double dmax = process_rows<false, DISC>(a, vprev, vnext, qw);
    reduce_residual(dmax, a.delta + a.k);
}

template <bool DISC>
__global__ void __launch_bounds__(kWarpsMax * 32) k_extract(SweepArgs a) {
    extern __shared__ double qbuf[];
    // K* = the sweep that converged (or the last one launched, parallel_vi.cpp:106 parity).
    int K = a.k;
    if (a.ctrl->stop) {
        K = a.ctrl->sweeps;
    } else if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.ctrl->sweeps = a.k;
    }
    const double* vprev = (K & 1) ? a.v1 : a.v0;
    double* qw = qbuf + (threadIdx.x >> 5) * 32 * a.qcap;
    process_rows<true, DISC>(a, vprev, nullptr, qw);
}

struct LaunchShape {
    int threads;
    size_t smem;
    int max_blocks;
};

LaunchShape shape_for(const vcs_space* sp, bool discounted, bool extract) {
    const int qcap = std::max(1, sp->max_degree);
    const size_t per_warp = static_cast<size_t>(32) * qcap * sizeof(double);
    int warps = kWarpsMax;
    while (warps > 1 && per_warp * warps > 96 * 1024) --warps;
    if (per_warp > 200 * 1024) raise(VCS_EINVAL, "out-degree too large for the sweep kernel");
    LaunchShape s{warps * 32, per_warp * warps, 0};
    const void* fn = extract ? (discounted ? reinterpret_cast<const void*>(k_extract<true>)
                                           : reinterpret_cast<const void*>(k_extract<false>))
                             : (discounted ? reinterpret_cast<const void*>(k_sweep<true>)
                                           : reinterpret_cast<const void*>(k_sweep<false>));
    VCS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(s.smem)));
    int per_sm = 0;
    VCS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, s.threads, s.smem));
    s.max_blocks = std::max(1, per_sm) * sp->num_sms;
    return s;
}

unsigned grid_for(const LaunchShape& sh, uint64_t rows) {
    const uint64_t chunks = (rows + 31) / 32;
    const uint64_t warps = static_cast<uint64_t>(sh.threads / 32);
    uint64_t blocks = (chunks + warps - 1) / warps;
    blocks = std::max<uint64_t>(1, std::min<uint64_t>(blocks, static_cast<uint64_t>(sh.max_blocks)));
    return static_cast<unsigned>(blocks);
}

// Row end of sweep k under the converged-layer skip: layers 0..min(H, H-k+1).
uint64_t sweep_row_end(const vcs_space* sp, int k, bool skip) {
    if (!skip) return sp->S;
    const int last = std::min(sp->H, sp->H - k + 1);
    if (last < 0) return 0;
    return sp->layer_off[static_cast<size_t>(last) + 1];
}

void launch_sweep(const vcs_space* sp, const SweepArgs& a, const LaunchShape& sh, bool disc,
                  cudaStream_t s) {
    const unsigned g = grid_for(sh, a.row_end > a.row_begin ? a.row_end - a.row_begin : 1);
    if (disc)
        k_sweep<true><<<g, sh.threads, sh.smem, s>>>(a);
    else
        k_sweep<false><<<g, sh.threads, sh.smem, s>>>(a);
    VCS_LAUNCHED();
}

void launch_extract(const vcs_space* sp, const SweepArgs& a, const LaunchShape& sh, bool disc,
                    cudaStream_t s) {
    const unsigned g = grid_for(sh, a.row_end > a.row_begin ? a.row_end - a.row_begin : 1);
    if (disc)
        k_extract<true><<<g, sh.threads, sh.smem, s>>>(a);
    else
        k_extract<false><<<g, sh.threads, sh.smem, s>>>(a);
    VCS_LAUNCHED();
}

SweepArgs base_args(vcs_space* sp, const double* v0, double* v1, double* delta, double eps,
                    double discount) {
    SweepArgs a{};
    a.row_ptr = sp->row_ptr.p;
    a.succ = sp->succ.p;
    a.reward = sp->reward.p;
    a.action = sp->action.p;
    a.v0 = v0;
    a.v1 = v1;
    a.delta = delta;
    a.ctrl = sp->ctrl.p;
    a.qcap = std::max(1, sp->max_degree);
    a.eps = eps;
    a.discount = discount;
    a.act_out = sp->actions_dev.p;
    return a;
}

bool is_discounted(double d) { return !(d == 0.0 || d == 1.0); }

CachedGraph& solve_graph(vcs_space* sp, const GraphKey& key) {
    auto it = sp->graphs.find(key);
    if (it != sp->graphs.end()) return it->second;
    CachedGraph g;
    cudaStream_t s = sp->stream;
    const bool disc = is_discounted(key.discount);
    const LaunchShape sw = shape_for(sp, disc, false);
    const LaunchShape ex = shape_for(sp, disc, true);
    for (auto& e : g.ev) VCS_CUDA(cudaEventCreate(&e));
    SweepArgs a = base_args(sp, sp->v[0].p, sp->v[1].p, sp->delta.p, key.eps, key.discount);
    VCS_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
        VCS_CUDA(cudaMemsetAsync(sp->v[0].p, 0, sp->S * sizeof(double), s));
        VCS_CUDA(cudaMemsetAsync(sp->delta.p, 0, (key.max_sweeps + 2) * sizeof(double), s));
        VCS_CUDA(cudaMemsetAsync(sp->ctrl.p, 0, sizeof(SolveCtrl), s));
        VCS_CUDA(cudaEventRecordWithFlags(g.ev[0], s, cudaEventRecordExternal));
        for (int k = 1; k <= key.max_sweeps; ++k) {
            a.k = k;
            a.row_begin = 0;
            a.row_end = static_cast<uint32_t>(sweep_row_end(sp, k, key.skip != 0));
            launch_sweep(sp, a, sw, disc, s);
        }
        VCS_CUDA(cudaEventRecordWithFlags(g.ev[1], s, cudaEventRecordExternal));
        a.k = key.max_sweeps;
        a.row_begin = 0;
        a.row_end = static_cast<uint32_t>(sp->S);
        launch_extract(sp, a, ex, disc, s);
        VCS_CUDA(cudaEventRecordWithFlags(g.ev[2], s, cudaEventRecordExternal));
    } catch (...) {
        cudaGraph_t dummy = nullptr;
        cudaStreamEndCapture(s, &dummy);
        if (dummy) cudaGraphDestroy(dummy);
        throw;
    }
    cudaGraph_t graph = nullptr;
    VCS_CUDA(cudaStreamEndCapture(s, &graph));
    const cudaError_t ierr = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ierr != cudaSuccess)
        raise(VCS_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ierr));
    g.n_sweeps = key.max_sweeps;
    g.launches = key.max_sweeps + 1;
    return sp->graphs.emplace(key, g).first->second;
}

void ensure_solve_buffers(vcs_space* sp, int max_sweeps) {
    sp->v[0].exact(sp->S);
    sp->v[1].exact(sp->S);
    sp->delta.exact(static_cast<size_t>(max_sweeps) + 2);
    sp->ctrl.exact(1);
    sp->actions_dev.exact(sp->S);
}

} // namespace
} // namespace vcs

using vcs::guarded;
using vcs::raise;

extern "C" {

int vcs_solve_enqueue(vcs_space* sp, const vcs_solve_opts* opts, void* stream) {
    return guarded([&] {
        vcs_solve_opts o{1e-6, 1, 0, 1.0};
        if (opts) o = *opts;
        if (!(o.epsilon > 0.0))
            raise(VCS_EINVAL, "epsilon must be > 0 (value iteration would never terminate)");
        vcs::bind_device(sp->device);
        int M = sp->H + 1; // delta_{H+1} == 0 on the layered DAG, so this is never binding
        if (o.max_sweeps > 0) M = std::min(M, o.max_sweeps);
        vcs::ensure_solve_buffers(sp, sp->H + 1); // fixed size: cached graphs keep addresses
        const vcs::GraphKey key{o.epsilon, o.discount, o.skip_converged ? 1 : 0, M};
        auto& g = vcs::solve_graph(sp, key);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : sp->stream;
        VCS_CUDA(cudaGraphLaunch(g.exec, s));
        vcs::note_launch(static_cast<uint64_t>(g.launches));
        sp->last_graph = &g;
        sp->last_key_skip = key.skip;
        return VCS_OK;
    });
}

int vcs_solve(vcs_space* sp, const vcs_solve_opts* opts, double* values_out, int32_t* actions_out,
              vcs_solve_report* report) {
    const int rc = vcs_solve_enqueue(sp, opts, nullptr);
    if (rc != VCS_OK) return rc;
    return vcs_solve_collect(sp, values_out, actions_out, report, nullptr);
}

int vcs_solve_collect(vcs_space* sp, double* values_out, int32_t* actions_out,
                      vcs_solve_report* report, void* stream) {
    return guarded([&] {
        if (!sp->last_graph) raise(VCS_EINVAL, "no solve was enqueued on this space");
        vcs::bind_device(sp->device);
        auto& g = *sp->last_graph;
        const vcs::GraphKey key{0.0, 0.0, sp->last_key_skip, 0};
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : sp->stream;
        vcs::SolveCtrl ctrl{};
        VCS_CUDA(cudaMemcpyAsync(&ctrl, sp->ctrl.p, sizeof ctrl, cudaMemcpyDeviceToHost, s));
        VCS_CUDA(cudaStreamSynchronize(s));
        const int K = ctrl.sweeps;
        if (values_out)
            VCS_CUDA(cudaMemcpyAsync(values_out, sp->v[K & 1].p, sp->S * sizeof(double),
                                     cudaMemcpyDeviceToHost, s));
        if (actions_out)
            VCS_CUDA(cudaMemcpyAsync(actions_out, sp->actions_dev.p, sp->S * sizeof(int32_t),
                                     cudaMemcpyDeviceToHost, s));
        VCS_CUDA(cudaStreamSynchronize(s));
        if (report) {
            float ms_sweep = 0.f, ms_ext = 0.f;
            VCS_CUDA(cudaEventElapsedTime(&ms_sweep, g.ev[0], g.ev[1]));
            VCS_CUDA(cudaEventElapsedTime(&ms_ext, g.ev[1], g.ev[2]));
            report->sweeps = K;
            report->launches = g.launches;
            report->backups_ref = sp->S * static_cast<uint64_t>(K);
            uint64_t done = 0;
            for (int k = 1; k <= K; ++k) done += vcs::sweep_row_end(sp, k, key.skip != 0);
            report->backups_done = done;
            report->sweep_ms = ms_sweep;
            report->extract_ms = ms_ext;
            const double dbar = sp->S ? static_cast<double>(sp->E) / static_cast<double>(sp->S) : 0.0;
            report->alg_bytes = (24.0 + 12.0 * dbar) * static_cast<double>(report->backups_ref);
            report->alg_bytes_done = (24.0 + 12.0 * dbar) * static_cast<double>(done);
        }
        return VCS_OK;
    });
}

int vcs_shard_begin(vcs_space* sp, double* v0, double* v1, double* delta, int32_t n_delta,
                    void* stream) {
    return guarded([&] {
        vcs::bind_device(sp->device);
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : sp->stream;
        sp->ctrl.exact(1);
        sp->actions_dev.exact(sp->S);
        sp->shard_v0 = v0;
        sp->shard_v1 = v1;
        sp->shard_delta = delta;
        sp->shard_n_delta = n_delta;
        VCS_CUDA(cudaMemsetAsync(v0, 0, sp->S * sizeof(double), s));
        VCS_CUDA(cudaMemsetAsync(delta, 0, static_cast<size_t>(n_delta) * sizeof(double), s));
        VCS_CUDA(cudaMemsetAsync(sp->ctrl.p, 0, sizeof(vcs::SolveCtrl), s));
        return VCS_OK;
    });
}

int vcs_shard_sweep(vcs_space* sp, int32_t k, uint64_t row_begin, uint64_t row_end,
                    const vcs_solve_opts* opts, void* stream) {
    return guarded([&] {
        if (!sp->shard_v0) raise(VCS_EINVAL, "vcs_shard_begin was not called");
        if (k < 1 || k + 1 > sp->shard_n_delta) raise(VCS_EINVAL, "sweep index out of range");
        vcs_solve_opts o{1e-6, 1, 0, 1.0};
        if (opts) o = *opts;
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : sp->stream;
        const bool disc = vcs::is_discounted(o.discount);
        const vcs::LaunchShape sh = vcs::shape_for(sp, disc, false);
        vcs::SweepArgs a =
            vcs::base_args(sp, sp->shard_v0, sp->shard_v1, sp->shard_delta, o.epsilon, o.discount);
        a.k = k;
        const uint64_t lim = std::min<uint64_t>(row_end, vcs::sweep_row_end(sp, k, o.skip_converged != 0));
        a.row_begin = static_cast<uint32_t>(row_begin);
        a.row_end = static_cast<uint32_t>(std::max<uint64_t>(lim, row_begin));
        vcs::launch_sweep(sp, a, sh, disc, s);
        return VCS_OK;
    });
}

int vcs_shard_finish(vcs_space* sp, int32_t n_sweeps, uint64_t row_begin, uint64_t row_end,
                     const vcs_solve_opts* opts, double* values_out, int32_t* actions_out,
                     int32_t* sweeps_out, void* stream) {
    return guarded([&] {
        if (!sp->shard_v0) raise(VCS_EINVAL, "vcs_shard_begin was not called");
        vcs_solve_opts o{1e-6, 1, 0, 1.0};
        if (opts) o = *opts;
        cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : sp->stream;
        const bool disc = vcs::is_discounted(o.discount);
        const vcs::LaunchShape sh = vcs::shape_for(sp, disc, true);
        vcs::SweepArgs a =
            vcs::base_args(sp, sp->shard_v0, sp->shard_v1, sp->shard_delta, o.epsilon, o.discount);
        a.k = n_sweeps;
        a.row_begin = static_cast<uint32_t>(row_begin);
        a.row_end = static_cast<uint32_t>(row_end);
        vcs::launch_extract(sp, a, sh, disc, s);
        vcs::SolveCtrl ctrl{};
        VCS_CUDA(cudaMemcpyAsync(&ctrl, sp->ctrl.p, sizeof ctrl, cudaMemcpyDeviceToHost, s));
        VCS_CUDA(cudaStreamSynchronize(s));
        const int K = ctrl.stop ? ctrl.sweeps : n_sweeps;
        const double* vsrc = (K & 1) ? sp->shard_v1 : sp->shard_v0;
        const uint64_t n = row_end > row_begin ? row_end - row_begin : 0;
        if (values_out && n)
            VCS_CUDA(cudaMemcpyAsync(values_out + row_begin, vsrc + row_begin, n * sizeof(double),
                                     cudaMemcpyDeviceToHost, s));
        if (actions_out && n)
            VCS_CUDA(cudaMemcpyAsync(actions_out + row_begin, sp->actions_dev.p + row_begin,
                                     n * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        VCS_CUDA(cudaStreamSynchronize(s));
        if (sweeps_out) *sweeps_out = K;
        return VCS_OK;
    });
}

} // extern "C"
