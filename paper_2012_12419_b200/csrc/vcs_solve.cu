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
#include "vcs_keys.cuh"


#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <thread>

#include <unistd.h>

namespace vcs {

namespace {

constexpr int kWarpsMax = 8;
// 4 blocks of 8 warps per SM (64 registers, no spills): C4 Jacobi 8.9 ms vs 10.9 at 3 blocks
// (74 registers); 5 blocks spill and measured 12.1 ms
constexpr int kSweepMinBlocks = 4;

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
__global__ void __launch_bounds__(kWarpsMax * 32, kSweepMinBlocks) k_sweep(SweepArgs a) {
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

// =============================================================================================
// Layer wavefront ("all truncation horizons") solver.
//
// On the layered DAG the Jacobi iterate of a layer-t state is the optimal k-step truncated
// return: V_k(s) = max_e ( r_e + V_{k-1}(succ_e) ), succ_e in layer t+1, V_0 = 0, and it is
// exact (constant) for k >= m_t = H - t.  So every Jacobi iterate V_1..V_{H+1} of every state is
// determined by the version vectors  W_t(s) = (V_1(s), ..., V_{m_t}(s)).  Processing the layers
// from t = H-1 down to 0, layer t's version vectors need only layer t+1's — the CSR is streamed
// ONCE per solve instead of once per sweep, and each V_k(s) is computed with exactly the
// reference's arithmetic (same adds, same strict '>' edge order), so the bits are identical.
// The residual of Jacobi sweep k is max over (s,k) of |V_k(s) - V_{k-1}(s)|, reduced per k
// (shared-memory atomics, then one global atomicMax per block and k).  The convergence sweep
// K* = min{k : delta_k < eps} is then known on the device; the extraction kernel outputs
// V_{K*} = W_t(s)[min(K*, m_t)] and the argmax action against V_{K*} of the successors — the
// reference's extraction (parallel_vi.cpp:109-111) bit for bit.
// Layout: W_t is state-major (state i of layer t at ver + ver_off[t] + i*m_t), so the lanes
// that compute the versions of one state read the successor's version vector contiguously.
// =============================================================================================

constexpr int kWaveWarps = 8;

// Version vectors are stored as V_0..V_m (V_0 = 0, the initial iterate) with the stride padded
// to a multiple of 4 doubles, so a thread's 4 consecutive versions load as two aligned double2.
__host__ __device__ __forceinline__ int wave_stride(int m) { return (m + 1 + 3) & ~3; }

struct WaveArgs {
    const uint32_t* __restrict__ row_ptr;
    const uint32_t* __restrict__ succ;
    const double* __restrict__ reward;
    const int32_t* __restrict__ action;
    double* ver;               // all version vectors
    const double* __restrict__ ver_next; // = ver + voff_next (layer t+1's store), set by the host
    double* ver_cur;                     // = ver + voff (layer t's store)
    const uint64_t* ver_off;   // per layer (H+2)
    const uint64_t* layer_off; // per layer (H+2), flat state index
    double* delta;             // delta[k], k = 1..H+1
    SolveCtrl* ctrl;
    double* values_out;        // extraction: V_{K*} in reference order
    int32_t* act_out;          // extraction: argmax action
    double eps;
    double discount;
    uint64_t row0, n, next_row0; // layer t: first flat state, size; layer t+1 first state
    uint64_t voff, voff_next;    // version offsets of layers t and t+1
    int m;                       // versions of layer t  (H - t)
    int band_lo, band_hi;        // versions [band_lo, band_hi) computed for layer t
    int next_lo;                 // band_lo of layer t+1
    int base, base_next;         // storage slot of version v in layer t (t+1) is v - base;
                                 // the bases keep the consumer's double2 loads 16B-aligned
    int tile;                    // states per block tile
    int stride, stride_next;     // stored version-vector strides of layers t and t+1
    int max_deg;                 // edge slots per state in the tile's shared-memory CSR
    int H;
    int max_sweeps;              // K* cap (H+1, or the caller's max_sweeps)
};

// One block per tile of T consecutive states of layer t:
//   phase 1: the tile's CSR rows (row_ptr, succ, reward, action) -> shared memory, coalesced;
//   phase 2: thread (j, g) of a pass computes versions k = a+2g, a+2g+1 of state j of the pass
//            (the rank's version band [a, b) of this layer; single GPU: [1, m_t+1)): per edge
//            one shared-memory read of (succ, reward) and ONE aligned 16-byte load of the
//            successor's V_{k-1}, V_k (band vectors are stored from version a-1 with an even
//            stride, band starts are odd); the gathers of up to U edges are in flight
//            together; then the strict first maximum per version.  The thread holding k = m_t
//            (the exact value) also records the argmax — that IS the extraction of s whenever
//            K* >= m_t;
//   phase 3: residuals |V_k - V_{k-1}| (a thread's k's are fixed: register running maxima).
//            For k = a the predecessor V_{a-1} is V_0 = 0 when a = 1; otherwise it is the
//            halo column another rank computes, and k_band_low_delta folds it in later.
struct alignas(16) EdgeRec {
    double reward;
    uint32_t succ; // successor index within layer t+1
    int32_t action;
};

// BAND = false: the single-GPU form (lo = 1, storage from V_0), with the shifts compile-time 0.
template <bool DISC, int U, int MINB, bool BAND>
__global__ void __launch_bounds__(kWaveWarps * 32, MINB) k_wave_layer(WaveArgs a) {
    constexpr int P = 2; // versions per thread (one aligned double2 gather per edge)
    // U: edges whose gathers are issued together; MINB: resident blocks per SM (register cap)
    extern __shared__ unsigned long long smem_u64[];
    const int lo = BAND ? a.band_lo : 1;         // first version computed (odd)
    const int nb = a.band_hi - a.band_lo;        // versions computed per state
    const int T = a.tile;
    const int w1 = nb + 1;                       // shared slots per state: V_{lo-1} .. V_{hi-1}
    // the tile's edges first, one 16-byte record each, so every per-edge shared access in the
    // gather loop is an immediate offset from the edge index (no per-edge address arithmetic)
    EdgeRec* sedge = reinterpret_cast<EdgeRec*>(smem_u64);           // [T*max_deg]
    double* sout = reinterpret_cast<double*>(sedge + static_cast<size_t>(T) * a.max_deg); // [T*(nb+1)]
    unsigned long long* sdelta =
        reinterpret_cast<unsigned long long*>(sout + static_cast<size_t>(T) * w1); // [nb]
    uint32_t* srp = reinterpret_cast<uint32_t*>(sdelta + nb);        // [T+1]
    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    for (int j = tid; j < nb; j += nthr) sdelta[j] = 0ull;
    const int G = (nb + P - 1) / P;                // thread groups per state (P versions each)
    const bool wide = G > nthr;                    // groups loop in strides of nthr
    const int spp = wide ? 1 : nthr / G;           // states per pass
    const int my_s = wide ? 0 : tid / G;
    const int my_g0 = wide ? tid : tid - my_s * G;
    const bool active = wide || my_s < spp;
    const uint32_t sn = static_cast<uint32_t>(a.stride_next); // stored stride of layer t+1
    const uint64_t st = static_cast<uint64_t>(a.stride);       // stored stride of layer t
    // successor slot of version (k-1) is k-1-base_next; for k = lo + gP it is even (aligned)
    const uint32_t nshift = BAND ? static_cast<uint32_t>(lo - 1 - a.base_next) : 0u;
    const int oshift = BAND ? lo - a.base : 1; // own storage slot of version lo + j is j + oshift
    const double* vn = a.ver_next; // one 64-bit base: a gather address is one IMAD.WIDE
    const uint32_t nbase = static_cast<uint32_t>(a.next_row0);
    const uint64_t n_tiles = (a.n + T - 1) / T;
    double dmax[P] = {0.0, 0.0}; // narrow case: the thread's k's never change
    // row_ptr of the block's NEXT tile is prefetched into registers while the current tile
    // computes (T+1 <= 513 entries: up to 3 per thread)
    uint32_t rp_next[3];
    auto prefetch_rp = [&](uint64_t tl) {
        if (tl >= n_tiles) return;
        const uint64_t b0 = tl * static_cast<uint64_t>(T);
        const int cnt = static_cast<int>(a.n - b0 < static_cast<uint64_t>(T) ? a.n - b0 : T);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const int j = tid + q * nthr;
            if (j <= cnt) rp_next[q] = __ldg(a.row_ptr + a.row0 + b0 + j);
        }
    };
    prefetch_rp(blockIdx.x);
    for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const uint64_t s0 = tile * static_cast<uint64_t>(T);
        const int nt = static_cast<int>(a.n - s0 < static_cast<uint64_t>(T) ? a.n - s0 : T);
        __syncthreads(); // previous tile's shared-memory readers are done
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const int j = tid + q * nthr;
            if (j <= nt) srp[j] = rp_next[q];
        }
        __syncthreads();
        prefetch_rp(tile + gridDim.x);
        const uint32_t e0 = srp[0];
        const int ne = static_cast<int>(srp[nt] - e0);
        for (int j = tid; j < ne; j += nthr) {
            EdgeRec rec;
            rec.reward = __ldcs(a.reward + e0 + j);
            rec.succ = __ldcs(a.succ + e0 + j) - nbase;
            rec.action = __ldcs(a.action + e0 + j); // the winner's action, without a dependent load
            sedge[j] = rec;
        }
        __syncthreads();
        double* out = a.ver_cur + s0 * st;
        if (active) {
            for (int sl = my_s; sl < nt; sl += spp) {
                const int eb = static_cast<int>(srp[sl] - e0), ee = static_cast<int>(srp[sl + 1] - e0);
                for (int g = my_g0; g < G; g += nthr) {
                    double best[P];
                    int best_e[P];
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        best[p] = -INFINITY;
                        best_e[p] = -1;
                    }
                    const uint32_t nslot = nshift + static_cast<uint32_t>(g * P);
                    // one edge's contribution to both versions: q = r + V_{k-1}(succ), strict
                    // first maximum with its edge (mdp.cpp:254-260)
                    auto relax = [&](int e, const double2& x) {
                        const double r = sedge[e].reward;
                        const double v[P] = {x.x, x.y}; // V_{k-1} of both versions
#pragma unroll
                        for (int p = 0; p < P; ++p) {
                            const double q = DISC ? __dadd_rn(r, __dmul_rn(a.discount, v[p]))
                                                  : __dadd_rn(r, v[p]);
                            if (q > best[p]) { // strict: the first maximal edge wins
                                best[p] = q;
                                best_e[p] = e;
                            }
                        }
                    };
                    int eo = eb;
                    for (; eo + U <= ee; eo += U) { // full rounds: U gathers in flight, no guards
                        double2 x[U];
#pragma unroll
                        for (int u = 0; u < U; ++u)
                            x[u] = __ldg(reinterpret_cast<const double2*>(
                                vn + (sedge[eo + u].succ * sn + nslot)));
#pragma unroll
                        for (int u = 0; u < U; ++u) relax(eo + u, x[u]);
                    }
                    if (eo < ee) { // the last < U edges
                        double2 x[U];
#pragma unroll
                        for (int u = 0; u < U - 1; ++u)
                            if (eo + u < ee)
                                x[u] = __ldg(reinterpret_cast<const double2*>(
                                    vn + (sedge[eo + u].succ * sn + nslot)));
#pragma unroll
                        for (int u = 0; u < U - 1; ++u)
                            if (eo + u < ee) relax(eo + u, x[u]);
                    }
                    double* o = out + sl * st;
                    double* so = sout + sl * w1;
                    if (g == 0 && lo == 1) {
                        o[oshift - 1] = 0.0; // V_0 (the initial iterate), stored for aligned reads
                        so[0] = 0.0;
                    }
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        const int j = g * P + p; // version k = lo + j
                        if (j < nb) {
                            o[j + oshift] = best[p];
                            so[j + 1] = best[p];
                            if (lo + j == a.m) { // exact value: V_{K*}(s) and the policy
                                const uint64_t s = a.row0 + s0 + sl;
                                a.values_out[s] = best[p];
                                a.act_out[s] = best_e[p] >= 0 ? sedge[best_e[p]].action : -1;
                            }
                        }
                    }
                }
            }
        }
        __syncthreads();
        if (active) {
            for (int sl = my_s; sl < nt; sl += spp)
                for (int g = my_g0; g < G; g += nthr) {
                    const double* so = sout + sl * w1;
#pragma unroll
                    for (int p = 0; p < P; ++p) {
                        const int j = g * P + p;
                        if (j < nb && (j > 0 || lo == 1)) {
                            const double d = fabs(so[j + 1] - so[j]);
                            if (!wide) {
                                dmax[p] = dmax[p] < d ? d : dmax[p];
                            } else if (d > 0.0) {
                                atomicMax(&sdelta[j],
                                          static_cast<unsigned long long>(__double_as_longlong(d)));
                            }
                        }
                    }
                }
        }
    }
    if (!wide && active) {
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const int j = my_g0 * P + p;
            if (j < nb && dmax[p] > 0.0)
                atomicMax(&sdelta[j], static_cast<unsigned long long>(__double_as_longlong(dmax[p])));
        }
    }
    __syncthreads();
    for (int j = tid; j < nb; j += nthr)
        if (sdelta[j]) atomicMax(reinterpret_cast<unsigned long long*>(a.delta + lo + j), sdelta[j]);
}

// K* from the residuals, then V_{K*} and the argmax policy for every state.  Warp-cooperative
// like the Jacobi kernel: 32 consecutive rows per warp, the rows' edge range staged with
// coalesced loads (q = r + V_{K*}(succ) into shared memory), then each lane scans its row.
__device__ __forceinline__ int layer_of(const uint64_t* s_layer, int H, uint64_t s) {
    int lo = 0, hi = H; // largest t with layer_off[t] <= s
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_layer[mid] <= s) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

template <bool DISC>
__global__ void __launch_bounds__(kWaveWarps * 32) k_wave_extract(WaveArgs a, int qcap) {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int U = 8;
    __shared__ int s_kstar;
    extern __shared__ uint64_t s_dyn[];
    const int H = a.H;
    uint64_t* s_layer = s_dyn;           // H+2 layer offsets
    uint64_t* s_voff = s_dyn + (H + 2);  // H+2 version offsets
    double* qw = reinterpret_cast<double*>(s_dyn + 2 * (H + 2)) + (threadIdx.x >> 5) * 32 * qcap;
    for (int t = threadIdx.x; t < H + 2; t += blockDim.x) {
        s_layer[t] = a.layer_off[t];
        s_voff[t] = a.ver_off[t];
    }
    if (threadIdx.x == 0) {
        int K = a.max_sweeps;
        for (int k = 1; k <= a.max_sweeps; ++k)
            if (a.delta[k] < a.eps) { // parallel_vi.cpp:66: first sweep whose residual < eps
                K = k;
                break;
            }
        s_kstar = K;
        if (blockIdx.x == 0) {
            a.ctrl->sweeps = K;
            a.ctrl->stop = 1;
        }
    }
    __syncthreads();
    const int K = s_kstar;
    // The layer pass already wrote the exact value and its argmax for every state; they are the
    // extraction against V_{K*} for layers t >= H - K* (min(K*, m_t) = m_t).  Only the prefix
    // of layers t < H - K* (an early stop) is recomputed here; usually it is empty.
    const uint64_t S = H - K > 0 ? s_layer[H - K] : 0;
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t r0 = warp * 32; r0 < S; r0 += n_warps * 32) {
        const uint64_t r = r0 + lane;
        const bool valid = r < S;
        const uint64_t rr = valid ? r : S;
        const uint32_t eb = __ldg(a.row_ptr + rr);
        uint32_t ee = __shfl_down_sync(FULL, eb, 1);
        if (lane == 31) ee = valid ? __ldg(a.row_ptr + r + 1) : eb;
        const uint32_t w0 = __shfl_sync(FULL, eb, 0);
        const uint32_t w1 = __shfl_sync(FULL, ee, 31);
        const int t_r = layer_of(s_layer, H, valid ? r : S - 1);
        // successor layer: t+1 of the source row; when the warp's rows share one layer (the
        // common case) every staged edge has the same successor layer
        const int t_first = __shfl_sync(FULL, t_r, 0);
        const int t_lastv = __shfl_sync(FULL, t_r, 31);
        const bool one_layer = t_first == t_lastv;
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
                if (e < w1) {
                    const int ts = one_layer ? t_first + 1 : layer_of(s_layer, H, sidx[u]);
                    const int ms = H - ts;
                    const int j = K < ms ? K : ms; // V_{K*}(succ) = stored version min(K*, m)
                    v[u] = __ldg(a.ver + s_voff[ts] + (sidx[u] - s_layer[ts]) * wave_stride(ms) + j);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t e = base + u * 32 + lane;
                if (e < w1)
                    qw[e - w0] = DISC ? __dadd_rn(rw[u], __dmul_rn(a.discount, v[u]))
                                      : __dadd_rn(rw[u], v[u]);
            }
        }
        __syncwarp();
        if (valid) {
            const int m_t = H - t_r;
            const int jv = K < m_t ? K : m_t; // V_{K*}(r) = version min(K*, m_t)
            a.values_out[r] = a.ver[s_voff[t_r] + (r - s_layer[t_r]) * wave_stride(m_t) + jv];
            int32_t act = -1;
            double best = -INFINITY;
            uint32_t best_e = 0xffffffffu;
            for (uint32_t e = eb; e < ee; ++e) {
                const double q = qw[e - w0];
                if (q > best) {
                    best = q;
                    best_e = e;
                }
            }
            if (best_e != 0xffffffffu) act = __ldg(a.action + best_e);
            a.act_out[r] = act;
        }
        __syncwarp();
    }
}

// ---- certified pass (VCS_METHOD_CERTIFIED) -----------------------------------------------------
// The reference's observable result is V_{K*}, the argmax against V_{K*} and K* (mdp.hpp:136-175).
// When K* = H+1 (no sweep k <= H has delta_k < eps) every state's output is its EXACT value
// V_{m_t} and the argmax against its successors' exact values: one backward pass.  The same pass
// also carries V_{m_t - 1}(s) (same recursion one version lower, V_0 = 0 for layer H-1), which
// gives for every k the lower bound lb_k = max over layer H-k of |V_k - V_{k-1}| <= delta_k.
// lb_k >= eps for all k <= H proves K* = H+1 (delta_{H+1} = 0 ends the reference's loop): the
// pass is then the whole solve, bit for bit.  Otherwise the full wavefront runs (graph IF node).

// Warp maximum of a non-negative double as its bit pattern (the order of non-negative doubles is
// the order of their bits): two integer reductions instead of five 64-bit shuffle rounds.
__device__ __forceinline__ unsigned long long warp_max_nonneg_bits(double v) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    const uint32_t hi = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(b >> 32));
    const uint32_t lo = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(b >> 32) == hi
                                                           ? static_cast<uint32_t>(b) : 0u);
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}

struct CertArgs {
    const uint32_t* __restrict__ row_ptr;
    const uint32_t* __restrict__ succ;
    const double* __restrict__ reward;
    const int32_t* __restrict__ action;
    const double2* __restrict__ xd_next; // layer t+1: (V_{m-2}, V_{m-1}) relative to layer t
    double2* xd_cur;                     // layer t:   (V_{m-1}, V_m)
    double* values_out;
    int32_t* act_out;
    double* lb;                          // lb[k], k = m_t
    uint64_t row0, n, next_row0;
    int m;
    double discount;
    int write_out; // 0: values/actions are written by another rank
};

// Thread-per-row form of the certified layer: each thread streams its own row's contiguous
// edge range (through L1: a warp's 32 rows are one contiguous span) and keeps U gathers in
// flight; no shared-memory staging.
template <bool DISC, int U, int MINB>
__global__ void __launch_bounds__(256, MINB) k_cert_rows(CertArgs a) {
    constexpr unsigned FULL = 0xffffffffu;
    __shared__ unsigned long long s_lb;
    if (threadIdx.x == 0) s_lb = 0ull;
    __syncthreads();
    double dmax = 0.0;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    // the next row's bounds are loaded while the current row computes (one round trip less)
    uint32_t nb = 0, ne = 0;
    if (r < a.n) {
        nb = __ldg(a.row_ptr + a.row0 + r);
        ne = __ldg(a.row_ptr + a.row0 + r + 1);
    }
    for (; r < a.n; r += stride) {
        const uint32_t eb = nb, ee = ne;
        if (r + stride < a.n) {
            nb = __ldg(a.row_ptr + a.row0 + r + stride);
            ne = __ldg(a.row_ptr + a.row0 + r + stride + 1);
        }
        double hi = -INFINITY, lo = -INFINITY;
        uint32_t best_e = 0xffffffffu;
        for (uint32_t e0 = eb; e0 < ee; e0 += U) {
            uint32_t sidx[U];
            double rw[U];
            double2 x[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (e0 + u < ee) {
                    sidx[u] = __ldcs(a.succ + e0 + u) - static_cast<uint32_t>(a.next_row0);
                    rw[u] = __ldcs(a.reward + e0 + u);
                }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (e0 + u < ee) x[u] = __ldg(a.xd_next + sidx[u]);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (e0 + u < ee) {
                    const double qx = DISC ? __dadd_rn(rw[u], __dmul_rn(a.discount, x[u].x)) : __dadd_rn(rw[u], x[u].x);
                    const double qy = DISC ? __dadd_rn(rw[u], __dmul_rn(a.discount, x[u].y)) : __dadd_rn(rw[u], x[u].y);
                    if (qy > hi) { // strict: the first maximal edge wins (mdp.cpp:254-260)
                        hi = qy;
                        best_e = e0 + u;
                    }
                    if (qx > lo) lo = qx;
                }
        }
        if (a.m == 1) lo = 0.0; // V_0
        a.xd_cur[r] = make_double2(lo, hi);
        if (a.write_out) {
            a.values_out[a.row0 + r] = hi;
            a.act_out[a.row0 + r] = best_e != 0xffffffffu ? __ldg(a.action + best_e) : -1;
        }
        const double d = fabs(hi - lo);
        dmax = dmax < d ? d : dmax;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(FULL, dmax, o);
        dmax = dmax < other ? other : dmax;
    }
    if ((threadIdx.x & 31) == 0 && dmax > 0.0)
        atomicMax(&s_lb, static_cast<unsigned long long>(__double_as_longlong(dmax)));
    __syncthreads();
    if (threadIdx.x == 0 && s_lb)
        atomicMax(reinterpret_cast<unsigned long long*>(a.lb + a.m), s_lb);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); // the next layer may launch
}

// The whole certified pass of a SMALL explicit space (every layer <= kCertSmallStates states and
// <= kCertSmallEdges transitions) in ONE block: the (V_{m-1}, V_m) pairs of two adjacent layers
// stay in shared memory and a layer is a block barrier instead of a kernel launch (the canonical
// instance: 330 layers of <= 614 states).  The CSR slices of layer t-1 (row offsets, successors,
// rewards, actions) are copied into shared memory with cp.async while layer t computes, so a
// layer's critical path is a barrier plus shared-memory reads — no global round trip.  Per state
// exactly k_cert_rows' operations (same edge order, same strict first maximum).
constexpr int kCertSmallStates = 1280;
constexpr int kCertSmallEdges = 3072;
constexpr int kCertSmallMaxH = 2046;
constexpr int kCertSmallThreads = 512;

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))), "l"(src) : "memory");
}

// a space k_cert_small takes: explicit CSR, every layer within the shared-memory stages
inline bool cert_small_ok(const vcs_space* sp) {
    if (sp->implicit || sp->H < 1 || sp->H > kCertSmallMaxH || std::getenv("VCS_NO_SMALL_SOLVE"))
        return false;
    if (sp->max_layer > static_cast<uint64_t>(kCertSmallStates)) return false;
    for (int t = 0; t < sp->H; ++t)
        if (sp->layer_edges[static_cast<size_t>(t)] > static_cast<uint64_t>(kCertSmallEdges)) return false;
    return true;
}

// dynamic shared memory of k_cert_small for a horizon of H
inline size_t cert_small_smem(int H) {
    return static_cast<size_t>(2) * kCertSmallStates * 16 +               // pairs
           static_cast<size_t>(2) * kCertSmallEdges * (8 + 4 + 4) +        // rewards, succ, actions
           static_cast<size_t>(2) * (kCertSmallStates + 1) * 4 +           // row offsets
           static_cast<size_t>(2) * (H + 2) * 4;                           // layer row / edge starts
}

template <bool DISC, int NT>
__global__ void __launch_bounds__(NT, 1)
k_cert_small(CertArgs a, const uint64_t* __restrict__ layer_off, int H) {
    constexpr int KS = kCertSmallStates, NE = kCertSmallEdges;
    extern __shared__ __align__(16) unsigned char cs_raw[];
    double2* xd = reinterpret_cast<double2*>(cs_raw);                 // [2][KS]
    double* srew = reinterpret_cast<double*>(xd + 2 * KS);            // [2][NE]
    uint32_t* ssucc = reinterpret_cast<uint32_t*>(srew + 2 * NE);     // [2][NE]
    int32_t* sact = reinterpret_cast<int32_t*>(ssucc + 2 * NE);       // [2][NE]
    uint32_t* srp = reinterpret_cast<uint32_t*>(sact + 2 * NE);       // [2][KS + 1]
    uint32_t* mrow = srp + 2 * (KS + 1);                              // [H + 2] first state of layer t
    uint32_t* medge = mrow + (H + 2);                                 // [H + 2] first edge of layer t
    __shared__ unsigned long long s_lb[2];
    const int tid = threadIdx.x;
    for (int t = tid; t <= H + 1; t += NT) {
        const uint64_t r = layer_off[t];
        mrow[t] = static_cast<uint32_t>(r);
        medge[t] = __ldg(a.row_ptr + r);
    }
    if (tid < 2) s_lb[tid] = 0ull;
    __syncthreads();
    {
        const uint32_t rH = mrow[H], nH = mrow[H + 1] - rH;
        for (uint32_t i = tid; i < nH; i += NT) xd[(H & 1) * KS + i] = make_double2(0.0, 0.0);
    }
    auto stage = [&](int t) { // layer t's CSR slices -> buffer t & 1 (asynchronously)
        const int b = t & 1;
        const uint32_t r0 = mrow[t], n = mrow[t + 1] - r0, e0 = medge[t], ne = medge[t + 1] - e0;
        for (uint32_t i = tid; i <= n; i += NT) cp_async4(srp + b * (KS + 1) + i, a.row_ptr + r0 + i);
        for (uint32_t e = tid; e < ne; e += NT) {
            cp_async8(srew + b * NE + e, a.reward + e0 + e);
            cp_async4(ssucc + b * NE + e, a.succ + e0 + e);
            cp_async4(sact + b * NE + e, a.action + e0 + e);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (H >= 1) stage(H - 1);
    for (int t = H - 1; t >= 0; --t) {
        const int b = t & 1;
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads(); // layer t's slices landed, layer t+1's pairs and lb are complete
        if (tid == 0 && t + 1 <= H - 1) { // layer t+1's lower bound
            const unsigned long long v = s_lb[(t + 1) & 1];
            if (v) a.lb[H - t - 1] = __longlong_as_double(static_cast<long long>(v));
            s_lb[(t + 1) & 1] = 0ull;
        }
        if (t >= 1) stage(t - 1); // (buffer (t-1)&1 held layer t+1's slices: consumed)
        const uint32_t row0 = mrow[t], n = mrow[t + 1] - row0, next0 = mrow[t + 1], e0 = medge[t];
        const double2* nxt = xd + ((t + 1) & 1) * KS;
        double2* cur = xd + b * KS;
        const uint32_t* rp = srp + b * (KS + 1);
        const double* rw_s = srew + b * NE;
        const uint32_t* sc_s = ssucc + b * NE;
        const int m = H - t;
        double dmax = 0.0;
        for (uint32_t i = tid; i < n; i += NT) {
            const uint32_t eb = rp[i] - e0, ee = rp[i + 1] - e0;
            double hi = -INFINITY, lo = -INFINITY;
            uint32_t best_e = 0xffffffffu;
            // four edges' loads in flight at a time; the maximum runs in edge order
            for (uint32_t e0 = eb; e0 < ee; e0 += 4) {
                double qx[4], qy[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t e = e0 + u < ee ? e0 + u : e0; // (lanes past the row repeat e0)
                    const double rw = rw_s[e];
                    const double2 x = nxt[sc_s[e] - next0];
                    qx[u] = DISC ? __dadd_rn(rw, __dmul_rn(a.discount, x.x)) : __dadd_rn(rw, x.x);
                    qy[u] = DISC ? __dadd_rn(rw, __dmul_rn(a.discount, x.y)) : __dadd_rn(rw, x.y);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (e0 + u >= ee) break;
                    if (qy[u] > hi) { // strict: the first maximal edge wins (mdp.cpp:254-260)
                        hi = qy[u];
                        best_e = e0 + u;
                    }
                    if (qx[u] > lo) lo = qx[u];
                }
            }
            if (m == 1) lo = 0.0; // V_0
            cur[i] = make_double2(lo, hi);
            a.values_out[row0 + i] = hi;
            a.act_out[row0 + i] = best_e != 0xffffffffu ? sact[b * NE + best_e] : -1;
            const double d = fabs(hi - lo);
            dmax = dmax < d ? d : dmax;
        }
        const unsigned long long wm = warp_max_nonneg_bits(dmax);
        if ((tid & 31) == 0 && wm) atomicMax(&s_lb[b], wm);
    }
    __syncthreads();
    if (tid == 0 && H >= 1 && s_lb[0]) a.lb[H] = __longlong_as_double(static_cast<long long>(s_lb[0]));
}

// Certified layer on the implicit-CSR form of a dense space: a state's edges are
// its valid slots (clouds in key order, paid last = the reference's edge order), the successor
// of slot e is rank_t[idx_e], the reward is the layer's kept constant or the retirement formula
// with the builder's rounded operations, the action the slot's cloud.  Per state: an 8-byte key
// in, the (V_{m-1}, V_m) pair, value and action out; no CSR is read.
struct CertImplArgs {
    const uint64_t* __restrict__ keys;   // layer t's packed keys
    const LayerParam* __restrict__ L;    // layer t's parameters (device)
    const uint32_t* __restrict__ rank;   // transition t's rank table
    const double2* __restrict__ xd_next; // layer t+1: (V_{m-2}, V_{m-1})
    double2* xd_cur;                     // layer t:   (V_{m-1}, V_m)
    double* values_out;
    int32_t* act_out;
    double* lb;
    uint64_t row0, n;
    int m;
    double discount;
    // key-space layout of the pairs (DXD): layer t+1's pairs at their successor index, layer t's
    // at its own key-space index (write_own: someone reads them)
    const uint32_t* __restrict__ rank_self; // transition t-1's table: layer t's BFS rank by index
    uint64_t dense_n;                       // layer t's key-space size
    int write_own;
    int write_out;                          // 0: values/actions are written by another rank
    int8_t* act_ks;                         // (VCS_CERT_PERMUTE) winner slot by key-space index
    // key-space order: the indices [d_lo, d_hi) of this launch (the whole key space on one GPU,
    // a rank's contiguous share when the layer is sharded across GPUs)
    uint64_t d_lo, d_hi;
    // (VCS_CERT_TIMELINE) per layer m: globaltimer of the first block's entry, the first block
    // past the PDL wait, and the last block's exit (stored inverted: all three by atomicMin)
    unsigned long long* tl;
};

__device__ __forceinline__ void tl_stamp(unsigned long long* tl, int m, int k) {
    if (!tl || threadIdx.x != 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(tl + 3 * m + k, k == 2 ? ~t : t);
}

// One layer of the implicit certified pass over states first_i, first_i + stride, ... (the
// block has loaded the layer's LayerParam into sL and zeroed s_lb).  DXD: the pairs are stored
// by key-space index (one gather per edge, no rank-table hop); otherwise by BFS index.
template <int WM, bool DISC, bool DXD, bool COHERENT = false>
__device__ __forceinline__ void cert_implicit_layer(const CertImplArgs& a, const LayerParam& L,
                                                    unsigned long long& s_lb, uint64_t first_i,
                                                    uint64_t stride) {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int SL = kDenseSlots;
    const bool retires = L.n_keep != L.n_active;
    const SlotDecoder<WM> dec(L); // the layer's slot constants, in registers
    const int words = L.words;
    const double r_cloud = L.r_cloud_kept, r_paid = L.r_paid_kept;
    double dmax = 0.0;
    uint64_t i = first_i;
    uint64_t kn[WM] = {}; // the next state's key, loaded while the current state computes
    if (i < a.n) load_key<WM>(a.keys + i * static_cast<uint64_t>(words), words, kn);
    tl_stamp(a.tl, a.m, 0);
    // programmatic dependent launch: everything above reads only build outputs; the previous
    // layer's pairs (and this layer's outputs) are touched after the wait
    asm volatile("griddepcontrol.wait;" ::: "memory");
    tl_stamp(a.tl, a.m, 1);
    // the next layer may launch now: its blocks take the slots this grid frees, run their
    // prologue and wait for this grid to complete (griddepcontrol.wait orders the data)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (; i < a.n; i += stride) {
        uint64_t k[WM];
#pragma unroll
        for (int w = 0; w < WM; ++w) k[w] = kn[w];
        if (i + stride < a.n) load_key<WM>(a.keys + (i + stride) * static_cast<uint64_t>(words), words, kn);
        const Slots sl = dec.decode(k);
        double2 x[SL];
        if (DXD) {
#pragma unroll
            for (int e = 0; e < SL; ++e)
                if (sl.valid(e)) // (COHERENT: written earlier in this kernel, read from L2)
                    x[e] = COHERENT ? __ldcg(a.xd_next + dec.idx(sl, e)) : __ldg(a.xd_next + dec.idx(sl, e));
        } else {
            uint32_t rk[SL];
#pragma unroll
            for (int e = 0; e < SL; ++e)
                if (sl.valid(e)) rk[e] = __ldg(a.rank + dec.idx(sl, e));
#pragma unroll
            for (int e = 0; e < SL; ++e)
                if (sl.valid(e)) x[e] = __ldg(a.xd_next + rk[e]);
        }
        double hi = -INFINITY, lo = -INFINITY;
        int best = -1;
#pragma unroll
        for (int e = 0; e < SL; ++e) {
            if (!sl.valid(e)) continue;
            const int pe = e == SL - 1 ? -1 : e;
            const double r = retires ? retiring_reward<WM>(k, pe, L) : (pe < 0 ? r_paid : r_cloud);
            const double qx = DISC ? __dadd_rn(r, __dmul_rn(a.discount, x[e].x)) : __dadd_rn(r, x[e].x);
            const double qy = DISC ? __dadd_rn(r, __dmul_rn(a.discount, x[e].y)) : __dadd_rn(r, x[e].y);
            if (qy > hi) { // strict: the first maximal edge wins (mdp.cpp:254-260)
                hi = qy;
                best = pe;
            }
            if (qx > lo) lo = qx;
        }
        if (a.m == 1) lo = 0.0; // V_0
        if (!DXD) {
            a.xd_cur[i] = make_double2(lo, hi);
        } else if (a.write_own) {
            uint32_t own = 0;
            for (int p = 0; p < L.n_active; ++p)
                own += static_cast<uint32_t>(get_field<WM>(k, L.bit_off[p], L.width[p])) * L.wself[p];
            a.xd_cur[own] = make_double2(lo, hi);
        }
        if (a.write_out) {
            a.values_out[a.row0 + i] = hi;
            a.act_out[a.row0 + i] = best < 0 ? -1 : L.cloud[best];
        }
        const double d = fabs(hi - lo);
        dmax = dmax < d ? d : dmax;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(FULL, dmax, o);
        dmax = dmax < other ? other : dmax;
    }
    if ((threadIdx.x & 31) == 0 && dmax > 0.0)
        atomicMax(&s_lb, static_cast<unsigned long long>(__double_as_longlong(dmax)));
    __syncthreads();
    if (threadIdx.x == 0 && s_lb)
        atomicMax(reinterpret_cast<unsigned long long*>(a.lb + a.m), s_lb);
    tl_stamp(a.tl, a.m, 2);
    // (the next layer was allowed to launch right after the wait above)
}

// One layer in KEY-SPACE order: index d of layer t's key space (d = sum_p f_p * wself[p]) is a
// state iff transition t-1's rank table holds its BFS rank.  The key is decoded from d, the
// successors' pairs are gathered by their key-space index (one hop), the own pair is written at
// d (coalesced) and the value/action at the BFS rank.
template <int WM, bool DISC>
__device__ __forceinline__ void cert_dense_layer(const CertImplArgs& a, const LayerParam& L,
                                                 unsigned long long& s_lb, uint64_t first,
                                                 uint64_t stride) {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int SL = kDenseSlots;
    const bool retires = L.n_keep != L.n_active;
    const SlotDecoder<WM> dec(L);
    const double r_cloud = L.r_cloud_kept, r_paid = L.r_paid_kept;
    constexpr int NF = kDenseSlots - 1; // key-space layers have <= 7 fields
    const int na = L.n_active;
    double dmax = 0.0;
    uint64_t d = a.d_lo + first;
    const uint64_t d_hi = a.d_hi;
    uint32_t rn = d < d_hi ? __ldg(a.rank_self + d) : kEmpty32; // next index's rank
    // mixed-radix digits of d and of the stride, divided out once; the loop steps an odometer
    uint32_t g[NF], sd[NF], rad[NF];
    {
        uint32_t rem = static_cast<uint32_t>(d < d_hi ? d : 0);
        uint32_t srem = static_cast<uint32_t>(stride < a.dense_n ? stride : 0);
#pragma unroll
        for (int p = 0; p < NF; ++p) {
            rad[p] = p < na ? L.radix[p] : 1u;
            g[p] = rem % rad[p];
            rem /= rad[p];
            sd[p] = srem % rad[p];
            srem /= rad[p];
        }
    }
    // clouds retiring at this transition (their free counts are charged by the reward)
    uint32_t retmask = 0;
#pragma unroll
    for (int p = 0; p < NF; ++p)
        if (p < na && L.keep_idx[p] < 0) retmask |= 1u << p;
    const double r_cl = L.r_cloud, r_pd = L.r_paid, gam = L.gamma;
    const int dem = L.demand;
    tl_stamp(a.tl, a.m, 0);
    asm volatile("griddepcontrol.wait;" ::: "memory"); // (PDL) the previous layer's pairs
    tl_stamp(a.tl, a.m, 1);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); // (as in cert_implicit_layer)
    for (; d < d_hi; d += stride) {
        const uint32_t r = rn;
        if (d + stride < d_hi) rn = __ldg(a.rank_self + d + stride);
        // the state's slots straight from its digits (= dec.decode of its packed key), and the
        // retired free VMs (an integer: the reference's fp64 running sum of integers is exact)
        uint32_t base = 0, mask = 0;
        int ret_all = 0;
#pragma unroll
        for (int p = 0; p < NF; ++p) {
            base += g[p] * dec.wn[p];
            if (((dec.sw[p] >> 16) & 1u) && g[p] >= dec.demand) mask |= 1u << p;
            if ((retmask >> p) & 1u) ret_all += static_cast<int>(g[p]);
        }
        { // advance the digits by the stride (the carry out of the top digit ends the loop)
            uint32_t carry = 0;
#pragma unroll
            for (int p = 0; p < NF; ++p) {
                const uint32_t v = g[p] + sd[p] + carry;
                carry = v >= rad[p] ? 1u : 0u;
                g[p] = carry ? v - rad[p] : v;
            }
        }
        if (r == kEmpty32) continue;
        const Slots sl(static_cast<uint64_t>(base) | (static_cast<uint64_t>(mask) << 32));
        // branch-free over the 8 slots: an invalid slot's pair is -inf, which never wins the
        // strict first maximum (and never raises lo)
        double2 x[SL];
#pragma unroll
        for (int e = 0; e < SL; ++e) {
            x[e] = make_double2(-INFINITY, -INFINITY);
            if (sl.valid(e)) x[e] = __ldg(a.xd_next + dec.idx(sl, e));
        }
        double hi = -INFINITY, lo = -INFINITY;
        int best = -1;
#pragma unroll
        for (int e = 0; e < SL; ++e) {
            const int pe = e == SL - 1 ? -1 : e;
            double rw;
            if (retires) { // retiring_reward: beta*n - gamma*retired, two rounded operations
                const int ret = ret_all - ((pe >= 0 && ((retmask >> pe) & 1u)) ? dem : 0);
                rw = __dsub_rn(pe < 0 ? r_pd : r_cl, __dmul_rn(gam, static_cast<double>(ret)));
            } else {
                rw = pe < 0 ? r_paid : r_cloud;
            }
            const double qx = DISC ? __dadd_rn(rw, __dmul_rn(a.discount, x[e].x)) : __dadd_rn(rw, x[e].x);
            const double qy = DISC ? __dadd_rn(rw, __dmul_rn(a.discount, x[e].y)) : __dadd_rn(rw, x[e].y);
            if (qy > hi) { // strict: the first maximal edge wins (mdp.cpp:254-260)
                hi = qy;
                best = pe;
            }
            if (qx > lo) lo = qx;
        }
        if (a.m == 1) lo = 0.0; // V_0
        a.xd_cur[d] = make_double2(lo, hi);
        a.values_out[a.row0 + r] = hi; // (on another GPU: a peer store into the primary's arrays)
        a.act_out[a.row0 + r] = best < 0 ? -1 : L.cloud[best];
        const double dd = fabs(hi - lo);
        dmax = dmax < dd ? dd : dmax;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(FULL, dmax, o);
        dmax = dmax < other ? other : dmax;
    }
    if ((threadIdx.x & 31) == 0 && dmax > 0.0)
        atomicMax(&s_lb, static_cast<unsigned long long>(__double_as_longlong(dmax)));
    __syncthreads();
    if (threadIdx.x == 0 && s_lb)
        atomicMax(reinterpret_cast<unsigned long long*>(a.lb + a.m), s_lb);
    tl_stamp(a.tl, a.m, 2);
    // (the next layer was allowed to launch right after the wait above)
}

// The key-space walk with TWO indices in flight per thread (d and d + stride, both stepped by
// 2*stride): sixteen successor-pair gathers are issued before either evaluation, which hides
// HBM latency on layers whose pair vectors do not fit in L2 (C7: 76 MB per layer).  Arithmetic,
// slot order and the strict first maximum are cert_dense_layer's.
template <int WM, bool DISC>
__device__ __forceinline__ void cert_dense_layer2(const CertImplArgs& a, const LayerParam& L,
                                                  unsigned long long& s_lb, uint64_t first,
                                                  uint64_t stride) {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int SL = kDenseSlots;
    constexpr int NF = kDenseSlots - 1;
    const bool retires = L.n_keep != L.n_active;
    const SlotDecoder<WM> dec(L);
    const double r_cloud = L.r_cloud_kept, r_paid = L.r_paid_kept;
    const int na = L.n_active;
    double dmax = 0.0;
    const uint64_t d_hi = a.d_hi;
    uint64_t d = a.d_lo + first;
    const uint64_t step = 2 * stride;
    uint32_t g0[NF], g1[NF], sd[NF], rad[NF];
    {
        uint32_t r0 = static_cast<uint32_t>(d < d_hi ? d : 0);
        uint32_t r1 = static_cast<uint32_t>(d + stride < d_hi ? d + stride : 0);
        uint32_t srem = static_cast<uint32_t>(step < a.dense_n ? step : 0);
#pragma unroll
        for (int p = 0; p < NF; ++p) {
            rad[p] = p < na ? L.radix[p] : 1u;
            g0[p] = r0 % rad[p];
            r0 /= rad[p];
            g1[p] = r1 % rad[p];
            r1 /= rad[p];
            sd[p] = srem % rad[p];
            srem /= rad[p];
        }
    }
    uint32_t retmask = 0;
#pragma unroll
    for (int p = 0; p < NF; ++p)
        if (p < na && L.keep_idx[p] < 0) retmask |= 1u << p;
    const double r_cl = L.r_cloud, r_pd = L.r_paid, gam = L.gamma;
    const int dem = L.demand;
    uint32_t rk0 = d < d_hi ? __ldg(a.rank_self + d) : kEmpty32;
    uint32_t rk1 = d + stride < d_hi ? __ldg(a.rank_self + d + stride) : kEmpty32;
    asm volatile("griddepcontrol.wait;" ::: "memory"); // (PDL) the previous layer's pairs
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); // (early: see cert_implicit_layer)
    auto slots = [&](const uint32_t (&g)[NF], int& ret_all) {
        uint32_t base = 0, mask = 0;
        ret_all = 0;
#pragma unroll
        for (int p = 0; p < NF; ++p) {
            base += g[p] * dec.wn[p];
            if (((dec.sw[p] >> 16) & 1u) && g[p] >= dec.demand) mask |= 1u << p;
            if ((retmask >> p) & 1u) ret_all += static_cast<int>(g[p]);
        }
        return Slots(static_cast<uint64_t>(base) | (static_cast<uint64_t>(mask) << 32));
    };
    auto advance = [&](uint32_t (&g)[NF]) {
        uint32_t carry = 0;
#pragma unroll
        for (int p = 0; p < NF; ++p) {
            const uint32_t v = g[p] + sd[p] + carry;
            carry = v >= rad[p] ? 1u : 0u;
            g[p] = carry ? v - rad[p] : v;
        }
    };
    auto evaluate = [&](uint64_t dd, uint32_t r, const Slots& sl, int ret_all, const double2 (&x)[SL]) {
        double hi = -INFINITY, lo = -INFINITY;
        int best = -1;
#pragma unroll
        for (int e = 0; e < SL; ++e) {
            const int pe = e == SL - 1 ? -1 : e;
            double rw;
            if (retires) {
                const int ret = ret_all - ((pe >= 0 && ((retmask >> pe) & 1u)) ? dem : 0);
                rw = __dsub_rn(pe < 0 ? r_pd : r_cl, __dmul_rn(gam, static_cast<double>(ret)));
            } else {
                rw = pe < 0 ? r_paid : r_cloud;
            }
            const double qx = DISC ? __dadd_rn(rw, __dmul_rn(a.discount, x[e].x)) : __dadd_rn(rw, x[e].x);
            const double qy = DISC ? __dadd_rn(rw, __dmul_rn(a.discount, x[e].y)) : __dadd_rn(rw, x[e].y);
            if (qy > hi) { // strict: the first maximal edge wins (mdp.cpp:254-260)
                hi = qy;
                best = pe;
            }
            if (qx > lo) lo = qx;
        }
        if (a.m == 1) lo = 0.0; // V_0
        a.xd_cur[dd] = make_double2(lo, hi);
        if (a.write_out) {
            a.values_out[a.row0 + r] = hi;
            a.act_out[a.row0 + r] = best < 0 ? -1 : L.cloud[best];
        }
        const double df = fabs(hi - lo);
        dmax = dmax < df ? df : dmax;
    };
    for (; d < d_hi; d += step) {
        const uint32_t r0 = rk0, r1 = rk1;
        const bool has1 = d + stride < d_hi;
        if (d + step < d_hi) rk0 = __ldg(a.rank_self + d + step);
        if (d + step + stride < d_hi) rk1 = __ldg(a.rank_self + d + step + stride);
        int ra0, ra1;
        const Slots s0 = slots(g0, ra0);
        const Slots s1 = slots(g1, ra1);
        advance(g0);
        advance(g1);
        const bool v0 = r0 != kEmpty32, v1 = has1 && r1 != kEmpty32;
        double2 x0[SL], x1[SL];
#pragma unroll
        for (int e = 0; e < SL; ++e) {
            x0[e] = make_double2(-INFINITY, -INFINITY);
            x1[e] = make_double2(-INFINITY, -INFINITY);
            if (v0 && s0.valid(e)) x0[e] = __ldg(a.xd_next + dec.idx(s0, e));
            if (v1 && s1.valid(e)) x1[e] = __ldg(a.xd_next + dec.idx(s1, e));
        }
        if (v0) evaluate(d, r0, s0, ra0, x0);
        if (v1) evaluate(d + stride, r1, s1, ra1, x1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(FULL, dmax, o);
        dmax = dmax < other ? other : dmax;
    }
    if ((threadIdx.x & 31) == 0 && dmax > 0.0)
        atomicMax(&s_lb, static_cast<unsigned long long>(__double_as_longlong(dmax)));
    __syncthreads();
    if (threadIdx.x == 0 && s_lb)
        atomicMax(reinterpret_cast<unsigned long long*>(a.lb + a.m), s_lb);
    // (the next layer was allowed to launch right after the wait above)
}

__device__ __forceinline__ void load_layer_param(LayerParam& sL, const LayerParam* src,
                                                 unsigned long long& s_lb) {
    __syncthreads(); // the previous layer's readers of sL are done
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(LayerParam) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(&sL)[i] = __ldg(reinterpret_cast<const uint32_t*>(src) + i);
    if (threadIdx.x == 0) s_lb = 0ull;
    __syncthreads();
}

// One launch per layer.  (A single cooperative launch over all layers with a grid sync between
// them measured slower, 0.86 vs 0.66 ms on C4: every sync waits for the slowest block.)
template <int WM, bool DISC, int MINB, bool DXD>
__global__ void __launch_bounds__(256, MINB) k_cert_implicit(CertImplArgs a) {
    __shared__ LayerParam sL;
    __shared__ unsigned long long s_lb;
    load_layer_param(sL, a.L, s_lb);
    cert_implicit_layer<WM, DISC, DXD>(a, sL, s_lb,
                                       static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                                       static_cast<uint64_t>(gridDim.x) * blockDim.x);
}

// The small sparse layers at the bottom of the pass (C4: layers 0-6, 1 to 4,704 states) in ONE
// block: a block barrier per layer instead of a kernel launch.  Per state cert_implicit_layer's
// evaluation (pairs by key-space index, read through L2: the previous layer wrote them in this
// kernel).  `meta`: per layer t <= t_hi its row0 / n / key offset (3 x u64).
constexpr int kTailThreads = 512;
constexpr uint64_t kTailMaxStates = 8192;

template <int WM, bool DISC>
__global__ void __launch_bounds__(kTailThreads, 1) k_cert_tail(CertImplArgs a, const uint64_t* meta,
                                                              const uint64_t* keys,
                                                              const LayerParam* params, double2* xd,
                                                              uint64_t half, int t_hi, int H) {
    __shared__ LayerParam sL;
    __shared__ unsigned long long s_lb;
    for (int t = t_hi; t >= 0; --t) {
        load_layer_param(sL, params + t, s_lb); // (its barriers also order the layers)
        CertImplArgs c = a;
        c.row0 = meta[3 * t];
        c.n = meta[3 * t + 1];
        c.keys = keys + meta[3 * t + 2];
        c.m = H - t;
        c.xd_next = xd + ((t + 1) & 1) * half;
        c.xd_cur = xd + (t & 1) * half;
        c.write_own = t >= 1 ? 1 : 0;
        cert_implicit_layer<WM, DISC, true, true>(c, sL, s_lb, threadIdx.x, blockDim.x);
        __syncthreads(); // this layer's pairs are written before the next layer reads them
    }
}

template <int WM, bool DISC, int MINB>
__global__ void __launch_bounds__(256, MINB) k_cert_dense(CertImplArgs a) {
    __shared__ LayerParam sL;
    __shared__ unsigned long long s_lb;
    load_layer_param(sL, a.L, s_lb);
    cert_dense_layer<WM, DISC>(a, sL, s_lb,
                               static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                               static_cast<uint64_t>(gridDim.x) * blockDim.x);
}

// ---- k_cert_dense_tma: the key-space walk with the successor windows staged by TMA -------------
// On a NON-RETIRING transition (same clouds, same numbering in layers t and t+1) the successor
// of index d through cloud slot p is d - demand*W_p and the paid successor is d itself, so for a
// tile of T consecutive indices [d0, d0+T) the successors of every slot form ONE contiguous
// window of layer t+1's pairs: [d0 - demand*W_p, d0 + T - demand*W_p).  A block owns tiles
// d0 = d_lo + (blockIdx + k*gridDim)*T; its thread 0 streams the windows of the tile NST ahead
// into a shared-memory ring with 1-D bulk copies (cp.async.bulk + mbarrier complete_tx), while
// the 8 warps evaluate the current tile from shared memory.  Windows whose shifts lie within a
// tile of each other are merged into one span (W = 1, 9, 81 overlap the paid window: C4/C7 move
// about half the bytes of eight separate windows).  Arithmetic, slot order and the strict first
// maximum are k_cert_dense's, so the bits are too.
constexpr int kTmaT = 256;  // indices per tile (= consumer threads per block)
constexpr int kTmaNst = 3;  // ring stages
constexpr int kTmaSlots = kDenseSlots; // 7 cloud slots + paid
constexpr int kTmaThreads = kTmaT + 32; // 8 consumer warps + 1 producer warp

struct TmaSpans {
    int n;                          // spans per tile
    int start[kTmaSlots];           // span start relative to d0 (<= 0)
    int len[kTmaSlots];             // span length in pairs (for a full tile)
    int off[kTmaSlots];             // span offset in the stage buffer (pairs)
    int base[kTmaSlots];            // slot e: stage offset of the pair of the tile's index 0
    uint32_t valid_slots;           // bit e: slot e can be valid in this layer
};

struct TmaSmem {
    double2 win[kTmaNst][kTmaSlots * kTmaT];
    uint32_t rank[kTmaNst][kTmaT + 8]; // the tile's BFS ranks (bulk copies need 16-B alignment)
    uint64_t full[kTmaNst];  // the stage's bulk copies landed (1 arrival + tx bytes)
    uint64_t empty[kTmaNst]; // the 8 consumer warps are done with the stage
    LayerParam L;
    TmaSpans sp;
    unsigned long long lb;
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\n"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
                 "r"(parity)
                 : "memory");
}

// Warp-specialised: warp 8 (one elected lane) produces — waits until a stage is free, posts the
// expected bytes and issues the tile's span copies; warps 0-7 consume — each thread evaluates
// one index of the tile from shared memory, then its warp releases the stage.
template <bool DISC>
__global__ void __launch_bounds__(kTmaThreads, 2) k_cert_dense_tma(CertImplArgs a, uint64_t d_next) {
    extern __shared__ __align__(128) unsigned char tma_raw[];
    TmaSmem& sm = *reinterpret_cast<TmaSmem*>(tma_raw);
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int NF = kDenseSlots - 1;
    const int tid = threadIdx.x;
    for (int i = tid; i < static_cast<int>(sizeof(LayerParam) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(&sm.L)[i] = __ldg(reinterpret_cast<const uint32_t*>(a.L) + i);
    if (tid == 0) {
        sm.lb = 0ull;
        for (int k = 0; k < kTmaNst; ++k) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&sm.full[k])) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(&sm.empty[k])),
                         "r"(kTmaT / 32)
                         : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const LayerParam& L = sm.L;
    const int na = L.n_active;
    const int dem = L.demand;
    if (tid == kTmaT) { // the layer's windows, merged into spans (by shift, largest first)
        int shift[kTmaSlots], order[kTmaSlots], ns = 0;
        uint32_t vs = 1u << (kTmaSlots - 1);
        for (int e = 0; e < NF; ++e)
            if (e < na && L.attr[e]) vs |= 1u << e;
        for (int e = 0; e < kTmaSlots; ++e) {
            if (!((vs >> e) & 1u)) continue;
            shift[e] = e == kTmaSlots - 1 ? 0 : dem * static_cast<int>(L.wnext[e]);
            order[ns++] = e;
        }
        for (int i = 1; i < ns; ++i)
            for (int j = i; j > 0 && shift[order[j]] > shift[order[j - 1]]; --j) {
                const int x = order[j];
                order[j] = order[j - 1];
                order[j - 1] = x;
            }
        TmaSpans& P = sm.sp;
        P.n = 0;
        P.valid_slots = vs;
        int off = 0;
        for (int i = 0; i < ns; ++i) {
            const int e = order[i];
            const int st = -shift[e];
            if (P.n > 0 && st <= P.start[P.n - 1] + P.len[P.n - 1]) { // overlaps the open span
                const int end = st + kTmaT;
                const int cur_end = P.start[P.n - 1] + P.len[P.n - 1];
                if (end > cur_end) {
                    P.len[P.n - 1] = end - P.start[P.n - 1];
                    off += end - cur_end;
                }
            } else {
                P.start[P.n] = st;
                P.len[P.n] = kTmaT;
                P.off[P.n] = off;
                off += kTmaT;
                ++P.n;
            }
            P.base[e] = P.off[P.n - 1] + (st - P.start[P.n - 1]);
        }
    }
    __syncthreads();
    const TmaSpans& P = sm.sp;
    const uint64_t d_lo = a.d_lo, d_hi = a.d_hi;
    const uint64_t n_tiles = d_hi > d_lo ? (d_hi - d_lo + kTmaT - 1) / kTmaT : 0;
    const uint64_t G = gridDim.x;
    if (tid >= kTmaT) { // ---- producer warp -------------------------------------------------
        asm volatile("griddepcontrol.wait;" ::: "memory"); // (PDL) the previous layer's pairs
        if (tid == kTmaT) {
            int k = 0;
            for (uint64_t j = blockIdx.x; j < n_tiles; j += G, ++k) {
                const int st = k % kTmaNst;
                if (k >= kTmaNst) mbar_wait(&sm.empty[st], static_cast<uint32_t>(k / kTmaNst - 1) & 1u);
                const int64_t d0 = static_cast<int64_t>(d_lo + j * kTmaT);
                const uint64_t left = d_hi - (d_lo + j * kTmaT);
                const int64_t cut = kTmaT - static_cast<int64_t>(left < kTmaT ? left : kTmaT);
                uint32_t bytes = 0;
                for (int q = 0; q < P.n; ++q) {
                    const int64_t s0 = d0 + P.start[q];
                    const int64_t s1 = s0 + P.len[q] - cut;
                    const int64_t lo = s0 < 0 ? 0 : s0;
                    const int64_t hi = s1 > static_cast<int64_t>(d_next) ? static_cast<int64_t>(d_next) : s1;
                    if (hi > lo) bytes += static_cast<uint32_t>(hi - lo) * 16u;
                }
                // the tile's ranks: from the 16-B aligned address at or below rank_self + d0
                // (the tables of later transitions follow, so rounding up stays in bounds)
                const uint32_t* rsrc = a.rank_self + d0;
                const uint32_t pre = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(rsrc) & 15u) >> 2);
                const uint32_t rcnt = (pre + static_cast<uint32_t>(kTmaT - cut) + 3u) & ~3u;
                bytes += rcnt * 4u;
                const uint32_t bar = smem_addr(&sm.full[st]);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_addr(&sm.rank[st][0])),
                    "l"(rsrc - pre), "r"(rcnt * 4u), "r"(bar)
                    : "memory");
                for (int q = 0; q < P.n; ++q) {
                    const int64_t s0 = d0 + P.start[q];
                    const int64_t s1 = s0 + P.len[q] - cut;
                    const int64_t lo = s0 < 0 ? 0 : s0;
                    const int64_t hi = s1 > static_cast<int64_t>(d_next) ? static_cast<int64_t>(d_next) : s1;
                    if (hi <= lo) continue;
                    const double2* dst = &sm.win[st][P.off[q] + (lo - s0)];
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_addr(dst)),
                        "l"(a.xd_next + lo), "r"(static_cast<uint32_t>(hi - lo) * 16u), "r"(bar)
                        : "memory");
                }
            }
        }
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        return;
    }
    // ---- consumers: a per-thread odometer over d = d_lo + (blockIdx + k*G)*T + tid ------------
    const uint64_t first = d_lo + static_cast<uint64_t>(blockIdx.x) * kTmaT + tid;
    const uint64_t stride = G * kTmaT;
    uint32_t g[NF], sd[NF], rad[NF];
    {
        uint32_t rem = static_cast<uint32_t>(first < d_hi ? first : 0);
        uint32_t srem = static_cast<uint32_t>(stride);
#pragma unroll
        for (int p = 0; p < NF; ++p) {
            rad[p] = p < na ? L.radix[p] : 1u;
            g[p] = rem % rad[p];
            rem /= rad[p];
            sd[p] = srem % rad[p];
            srem /= rad[p];
        }
    }
    int base[kTmaSlots];
#pragma unroll
    for (int e = 0; e < kTmaSlots; ++e) base[e] = P.base[e] + tid;
    const uint32_t vs = P.valid_slots;
    const double r_cloud = L.r_cloud_kept, r_paid = L.r_paid_kept;
    asm volatile("griddepcontrol.wait;" ::: "memory"); // (this layer's outputs after the wait)
    double dmax = 0.0;
    uint64_t d = first;
    int k = 0;
    for (uint64_t j = blockIdx.x; j < n_tiles; j += G, ++k, d += stride) {
        const int st = k % kTmaNst;
        const uint32_t pre = static_cast<uint32_t>(
            (reinterpret_cast<uintptr_t>(a.rank_self + (d - tid)) & 15u) >> 2);
        uint32_t mask = 0;
#pragma unroll
        for (int p = 0; p < NF; ++p)
            if (((vs >> p) & 1u) && g[p] >= static_cast<uint32_t>(dem)) mask |= 1u << p;
        { // advance the digits by the stride
            uint32_t carry = 0;
#pragma unroll
            for (int p = 0; p < NF; ++p) {
                const uint32_t v = g[p] + sd[p] + carry;
                carry = v >= rad[p] ? 1u : 0u;
                g[p] = carry ? v - rad[p] : v;
            }
        }
        mbar_wait(&sm.full[st], static_cast<uint32_t>(k / kTmaNst) & 1u);
        const uint32_t r = d < d_hi ? sm.rank[st][pre + tid] : kEmpty32;
        if (r != kEmpty32) {
            const double2* w = sm.win[st];
            double hi = -INFINITY, lo = -INFINITY;
            int best = -1;
#pragma unroll
            for (int e = 0; e < kTmaSlots; ++e) {
                const bool valid = e == kTmaSlots - 1 || ((mask >> e) & 1u);
                if (!valid) continue;
                const double2 x = w[base[e]];
                const double rw = e == kTmaSlots - 1 ? r_paid : r_cloud;
                const double qx = DISC ? __dadd_rn(rw, __dmul_rn(a.discount, x.x)) : __dadd_rn(rw, x.x);
                const double qy = DISC ? __dadd_rn(rw, __dmul_rn(a.discount, x.y)) : __dadd_rn(rw, x.y);
                if (qy > hi) { // strict: the first maximal edge wins (mdp.cpp:254-260)
                    hi = qy;
                    best = e == kTmaSlots - 1 ? -1 : e;
                }
                if (qx > lo) lo = qx;
            }
            if (a.m == 1) lo = 0.0; // V_0
            a.xd_cur[d] = make_double2(lo, hi);
            if (a.write_out) {
                a.values_out[a.row0 + r] = hi;
                a.act_out[a.row0 + r] = best < 0 ? -1 : L.cloud[best];
            }
            const double dd = fabs(hi - lo);
            dmax = dmax < dd ? dd : dmax;
        }
        __syncwarp();
        if ((tid & 31) == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(&sm.empty[st])) : "memory");
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(FULL, dmax, o);
        dmax = dmax < other ? other : dmax;
    }
    if ((tid & 31) == 0 && dmax > 0.0)
        atomicMax(reinterpret_cast<unsigned long long*>(a.lb + a.m),
                  static_cast<unsigned long long>(__double_as_longlong(dmax)));
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// The key-space walk specialised for NON-RETIRING transitions (every full layer of C3/C4/C7
// but the last): the successor of d through cloud slot p is d - demand*W_p and the paid one is
// d itself, so the successor index needs no digit sum, every cloud edge has the same reward
// (r_cloud_kept) and the paid edge r_paid_kept; the eligible slots and their byte offsets are
// per-layer uniforms.  ~2x fewer instructions per index than the generic walk (390 SASS
// instructions per iteration there); same operations on every edge, same strict first maximum.
template <bool DISC, bool EARLY = false>
__global__ void __launch_bounds__(256, 3) k_cert_dense_nr(CertImplArgs a) {
    __shared__ LayerParam sL;
    __shared__ unsigned long long s_lb;
    load_layer_param(sL, a.L, s_lb);
    const LayerParam& L = sL;
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int NF = kDenseSlots - 1;
    const int na = L.n_active;
    const uint32_t dem = static_cast<uint32_t>(L.demand);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t d_hi = a.d_hi;
    uint64_t d = a.d_lo + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    uint32_t g[NF], sd[NF], rad[NF], off[NF];
    uint32_t elig = 0;
    {
        uint32_t rem = static_cast<uint32_t>(d < d_hi ? d : 0);
        uint32_t srem = static_cast<uint32_t>(stride < a.dense_n ? stride : 0);
#pragma unroll
        for (int p = 0; p < NF; ++p) {
            rad[p] = p < na ? L.radix[p] : 1u;
            g[p] = rem % rad[p];
            rem /= rad[p];
            sd[p] = srem % rad[p];
            srem /= rad[p];
            off[p] = p < na ? dem * L.wnext[p] : 0u;
            if (p < na && L.attr[p]) elig |= 1u << p;
        }
    }
    const double r_cloud = L.r_cloud_kept, r_paid = L.r_paid_kept;
    uint32_t rn = d < d_hi ? __ldg(a.rank_self + d) : kEmpty32;
    double dmax = 0.0;
    asm volatile("griddepcontrol.wait;" ::: "memory"); // (PDL) the previous layer's pairs
    if (EARLY) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (; d < d_hi; d += stride) {
        const uint32_t r = rn;
        if (d + stride < d_hi) rn = __ldg(a.rank_self + d + stride);
        uint32_t mask = 0;
#pragma unroll
        for (int p = 0; p < NF; ++p) mask |= (g[p] >= dem ? 1u : 0u) << p;
        mask &= elig;
        {
            uint32_t carry = 0;
#pragma unroll
            for (int p = 0; p < NF; ++p) {
                const uint32_t v = g[p] + sd[p] + carry;
                carry = v >= rad[p] ? 1u : 0u;
                g[p] = carry ? v - rad[p] : v;
            }
        }
        if (r == kEmpty32) continue;
        const double2* P = a.xd_next + d;
        double2 x[NF];
#pragma unroll
        for (int p = 0; p < NF; ++p)
            if ((mask >> p) & 1u) x[p] = __ldg(P - off[p]);
        const double2 xp = __ldg(P);
        double hi = -INFINITY, lo = -INFINITY;
        int best = -1;
#pragma unroll
        for (int p = 0; p < NF; ++p) {
            if (!((mask >> p) & 1u)) continue;
            const double qx = DISC ? __dadd_rn(r_cloud, __dmul_rn(a.discount, x[p].x)) : __dadd_rn(r_cloud, x[p].x);
            const double qy = DISC ? __dadd_rn(r_cloud, __dmul_rn(a.discount, x[p].y)) : __dadd_rn(r_cloud, x[p].y);
            if (qy > hi) { // strict: the first maximal edge wins (mdp.cpp:254-260)
                hi = qy;
                best = p;
            }
            if (qx > lo) lo = qx;
        }
        {
            const double qx = DISC ? __dadd_rn(r_paid, __dmul_rn(a.discount, xp.x)) : __dadd_rn(r_paid, xp.x);
            const double qy = DISC ? __dadd_rn(r_paid, __dmul_rn(a.discount, xp.y)) : __dadd_rn(r_paid, xp.y);
            if (qy > hi) {
                hi = qy;
                best = -1;
            }
            if (qx > lo) lo = qx;
        }
        if (a.m == 1) lo = 0.0; // V_0
        a.xd_cur[d] = make_double2(lo, hi);
        if (a.act_ks) {
            a.act_ks[d] = static_cast<int8_t>(best); // coalesced; k_cert_permute reorders
        } else if (a.write_out) {
            a.values_out[a.row0 + r] = hi;
            a.act_out[a.row0 + r] = best < 0 ? -1 : L.cloud[best];
        }
        const double dd = fabs(hi - lo);
        dmax = dmax < dd ? dd : dmax;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(FULL, dmax, o);
        dmax = dmax < other ? other : dmax;
    }
    if ((threadIdx.x & 31) == 0 && dmax > 0.0)
        atomicMax(&s_lb, static_cast<unsigned long long>(__double_as_longlong(dmax)));
    __syncthreads();
    if (threadIdx.x == 0 && s_lb)
        atomicMax(reinterpret_cast<unsigned long long*>(a.lb + a.m), s_lb);
    // (with the gather pass the late trigger measured better on C7: 4.91 vs 4.95 ms)
    if (!EARLY) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- k_cert_dense_win: the non-retiring key-space walk with the near successors in shared memory
// The dense layers are bound by L2 (LTS) throughput: ~108 MB of sector traffic per C4 layer of
// 531,441 indices against ~25 MB of algorithmic bytes, two thirds of it the eight shifted pair
// gathers.  On a non-retiring transition the successor of d through cloud slot p is d - c_p
// (c_p = demand * W_p) and the paid one d itself, so for a tile of 256 consecutive indices the
// slots with small shifts (c_p <= kWinShift: W = 1, 9, 81 at radix 9) and the paid slot read ONE
// window [d0 - c_max, d0 + 256) of layer t+1's pairs.  Each block stages its tile's window in
// shared memory with cp.async (double-buffered: the next tile's window streams in while this one
// computes) and gathers only the far slots from global memory.  Same operations, slot order and
// strict first maximum as k_cert_dense_nr, so the same bits.
constexpr int kWinT = 256;
constexpr int kWinShift = 512; // largest shift served from shared memory

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

template <bool DISC>
__global__ void __launch_bounds__(kWinT, 3) k_cert_dense_win(CertImplArgs a) {
    __shared__ LayerParam sL;
    __shared__ unsigned long long s_lb;
    __shared__ __align__(16) double2 win[2][kWinT + kWinShift];
    load_layer_param(sL, a.L, s_lb);
    const LayerParam& L = sL;
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int NF = kDenseSlots - 1;
    const int na = L.n_active;
    const int tid = threadIdx.x;
    const uint32_t dem = static_cast<uint32_t>(L.demand);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kWinT;
    const uint64_t d_hi = a.d_hi;
    uint64_t d0 = a.d_lo + static_cast<uint64_t>(blockIdx.x) * kWinT; // this tile's first index
    uint64_t d = d0 + tid;
    uint32_t g[NF], sd[NF], rad[NF], off[NF];
    uint32_t elig = 0, near = 0, cmax = 0;
    {
        uint32_t rem = static_cast<uint32_t>(d < d_hi ? d : 0);
        uint32_t srem = static_cast<uint32_t>(stride < a.dense_n ? stride : 0);
#pragma unroll
        for (int p = 0; p < NF; ++p) {
            rad[p] = p < na ? L.radix[p] : 1u;
            g[p] = rem % rad[p];
            rem /= rad[p];
            sd[p] = srem % rad[p];
            srem /= rad[p];
            off[p] = p < na ? dem * L.wnext[p] : 0u;
            if (p < na && L.attr[p]) elig |= 1u << p;
            if (p < na && off[p] <= static_cast<uint32_t>(kWinShift)) {
                near |= 1u << p;
                cmax = max(cmax, off[p]);
            }
        }
    }
    const uint32_t wlen = kWinT + cmax; // window [d0 - cmax, d0 + kWinT)
    const double r_cloud = L.r_cloud_kept, r_paid = L.r_paid_kept;
    uint32_t rn = d < d_hi ? __ldg(a.rank_self + d) : kEmpty32;
    double dmax = 0.0;
    // the window of the tile starting at t0 into buffer b (indices outside [0, d_hi) are not read)
    auto stage = [&](uint64_t t0, int b) {
        for (uint32_t i = tid; i < wlen; i += kWinT) {
            const int64_t src = static_cast<int64_t>(t0) - static_cast<int64_t>(cmax) + i;
            if (src >= 0 && static_cast<uint64_t>(src) < d_hi) cp_async16(&win[b][i], a.xd_next + src);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    asm volatile("griddepcontrol.wait;" ::: "memory"); // (PDL) the previous layer's pairs
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); // (early: see cert_implicit_layer)
    if (d0 < d_hi) stage(d0, 0);
    for (int k = 0; d0 < d_hi; ++k, d0 += stride, d += stride) {
        const int b = k & 1;
        if (d0 + stride < d_hi) {
            stage(d0 + stride, b ^ 1);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads(); // this tile's window is complete
        const uint32_t r = rn;
        if (d + stride < d_hi) rn = __ldg(a.rank_self + d + stride);
        uint32_t mask = 0;
#pragma unroll
        for (int p = 0; p < NF; ++p) mask |= (g[p] >= dem ? 1u : 0u) << p;
        mask &= elig;
        {
            uint32_t carry = 0;
#pragma unroll
            for (int p = 0; p < NF; ++p) {
                const uint32_t v = g[p] + sd[p] + carry;
                carry = v >= rad[p] ? 1u : 0u;
                g[p] = carry ? v - rad[p] : v;
            }
        }
        if (d < d_hi && r != kEmpty32) {
            const double2* W = &win[b][tid + cmax]; // the pair of index d
            double2 x[NF];
#pragma unroll
            for (int p = 0; p < NF; ++p)
                if ((mask >> p) & 1u) x[p] = ((near >> p) & 1u) ? W[-static_cast<int>(off[p])]
                                                                 : __ldg(a.xd_next + d - off[p]);
            const double2 xp = W[0];
            double hi = -INFINITY, lo = -INFINITY;
            int best = -1;
#pragma unroll
            for (int p = 0; p < NF; ++p) {
                if (!((mask >> p) & 1u)) continue;
                const double qx = DISC ? __dadd_rn(r_cloud, __dmul_rn(a.discount, x[p].x)) : __dadd_rn(r_cloud, x[p].x);
                const double qy = DISC ? __dadd_rn(r_cloud, __dmul_rn(a.discount, x[p].y)) : __dadd_rn(r_cloud, x[p].y);
                if (qy > hi) { // strict: the first maximal edge wins (mdp.cpp:254-260)
                    hi = qy;
                    best = p;
                }
                if (qx > lo) lo = qx;
            }
            {
                const double qx = DISC ? __dadd_rn(r_paid, __dmul_rn(a.discount, xp.x)) : __dadd_rn(r_paid, xp.x);
                const double qy = DISC ? __dadd_rn(r_paid, __dmul_rn(a.discount, xp.y)) : __dadd_rn(r_paid, xp.y);
                if (qy > hi) {
                    hi = qy;
                    best = -1;
                }
                if (qx > lo) lo = qx;
            }
            if (a.m == 1) lo = 0.0; // V_0
            a.xd_cur[d] = make_double2(lo, hi);
            if (a.write_out) {
                a.values_out[a.row0 + r] = hi;
                a.act_out[a.row0 + r] = best < 0 ? -1 : L.cloud[best];
            }
            const double dd = fabs(hi - lo);
            dmax = dmax < dd ? dd : dmax;
        }
        __syncthreads(); // the window buffer is free for the tile after next
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(FULL, dmax, o);
        dmax = dmax < other ? other : dmax;
    }
    if ((tid & 31) == 0 && dmax > 0.0)
        atomicMax(&s_lb, static_cast<unsigned long long>(__double_as_longlong(dmax)));
    __syncthreads();
    if (tid == 0 && s_lb) atomicMax(reinterpret_cast<unsigned long long*>(a.lb + a.m), s_lb);
}

// (VCS_CERT_PERMUTE experiment) layer t's results in BFS order from the key-space-ordered pairs
// and winner slots: a thread per state decodes its key-space index from its packed key.
template <int WM>
__global__ void __launch_bounds__(256) k_cert_permute(const uint64_t* __restrict__ keys,
                                                      const LayerParam* __restrict__ Lp,
                                                      const double2* __restrict__ xd,
                                                      const int8_t* __restrict__ act_ks, uint64_t n,
                                                      uint64_t row0, double* values_out,
                                                      int32_t* act_out) {
    __shared__ LayerParam L;
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(LayerParam) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(&L)[i] = __ldg(reinterpret_cast<const uint32_t*>(Lp) + i);
    __syncthreads();
    const int words = L.words;
    for (uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
         r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint64_t k[WM];
        load_key<WM>(keys + r * static_cast<uint64_t>(words), words, k);
        uint32_t d = 0;
        for (int p = 0; p < L.n_active; ++p)
            d += static_cast<uint32_t>(get_field<WM>(k, L.bit_off[p], L.width[p])) * L.wself[p];
        const int8_t b = act_ks[d];
        values_out[row0 + r] = xd[d].y;
        act_out[row0 + r] = b < 0 ? -1 : L.cloud[b];
    }
}

template <int WM, bool DISC>
__global__ void __launch_bounds__(256, 2) k_cert_dense2(CertImplArgs a) {
    __shared__ LayerParam sL;
    __shared__ unsigned long long s_lb;
    load_layer_param(sL, a.L, s_lb);
    cert_dense_layer2<WM, DISC>(a, sL, s_lb,
                                static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                                static_cast<uint64_t>(gridDim.x) * blockDim.x);
}

// ---- k_cert_stream: the whole certified pass as ONE persistent kernel --------------------------
// Per-layer launches cost ~3 us each even chained by PDL (measured: 48 near-empty layer launches
// take 0.15 ms of C4's 0.52), and every layer waits for the slowest block of the one before.
// Here blocks pull tiles of T indices from one global counter, in layer order (t = H-1 .. 0, then
// ascending within a layer), and a tile waits only for what it reads:
//   * key-space walk on a non-retiring transition: the successor of d through slot p is
//     d - demand*W_p, so tile k of layer t reads layer t+1's tiles covering
//     [kT - demand*W_p, kT + T - demand*W_p) for its eligible slots and [kT, kT + T) (paid) — at
//     most 16 per-tile flags;
//   * key-space walk on a retiring transition, BFS walk (sparse layers): all of layer t+1.
// Pairs rotate through THREE buffers (layer t in t % 3) and a tile of layer t also waits until
// layer t+2 is complete — the last reader of the buffer it overwrites — so two layers are in
// flight at once.  Deadlock-free without co-residency: a tile is handed out only to a running
// block and waits only for tiles handed out before it.  Producer: stores, block barrier, fence,
// release-store of the tile's flag, count into the layer's done counter.  Consumer: warp 0
// spins (relaxed) on the tile's dependencies, one acquire fence (it invalidates the SM's L1, so
// the pair loads after the block barrier, cached in L1 for the overlapping windows, are fresh).
// Per index the arithmetic is cert_dense_layer's / cert_implicit_layer's, so are the bits.
constexpr int kStreamT = 1024;       // indices (key-space walk) or states (BFS walk) per tile
constexpr int kStreamThreads = 256;
constexpr int kStreamBufs = 4;       // pair buffers in rotation (layer t in buffer t % 4)

struct StreamLayer {
    uint64_t row0, n;        // the layer's BFS rows
    uint64_t dense_n;        // key-space size of the layer
    uint64_t key_off;        // its packed keys (u64 words)
    uint64_t rank_self_off;  // transition t-1's rank table (key-space walk)
    uint32_t tile_start, n_tiles;
    int32_t kind;            // 0: key-space walk, window deps; 1: key-space walk, whole-layer dep;
                             // 2: BFS walk, whole-layer dep
    int32_t m;               // H - t
    uint32_t n_shift;
    uint32_t shift[kDenseSlots]; // kind 0: the eligible slots' demand*W_p, and 0 (paid)
};

struct StreamArgs {
    const StreamLayer* layers; // processing order o = 0..H-1 (t = H-1-o)
    const LayerParam* params;  // by t
    const uint64_t* keys;
    const uint32_t* rank_tables;
    double2* xd;               // 3 buffers of `third` pairs; layer t in buffer t % 3
    uint64_t third;
    double* values_out;
    int32_t* act_out;
    double* lb;
    double discount;
    uint32_t* sync;            // [total_tiles flags | H done counters | work counter]
    uint32_t total_tiles;
    int H;
};

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// spin with relaxed loads (an acquire load per iteration would invalidate L1 every time), then
// one acquire fence once the producer's release-store is seen
__device__ __forceinline__ void wait_ge(const uint32_t* p, uint32_t target) {
    while (ld_relaxed_u32(p) < target) {}
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int WM, bool DISC>
__global__ void __launch_bounds__(kStreamThreads, 2) k_cert_stream(StreamArgs A) {
    // per tile, everything that is latency rather than work is taken off the critical path: the
    // NEXT tile id is fetched while this one computes, its layer's parameters are loaded into
    // the other half of a double buffer behind the computation, and warp 0 checks the tile's
    // (up to 17) dependencies with one lane each, so a satisfied check costs one L2 round trip
    __shared__ LayerParam sLb[2];
    __shared__ uint32_t s_tile[2];
    __shared__ int s_o[2];
    __shared__ unsigned long long s_lb;
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int SL = kDenseSlots;
    constexpr int NF = kDenseSlots - 1;
    constexpr int PW = static_cast<int>(sizeof(LayerParam) / 4);
    constexpr int PPT = (PW + kStreamThreads - 1) / kStreamThreads; // param words per thread
    const int tid = threadIdx.x, lane = tid & 31;
    uint32_t* flags = A.sync;
    uint32_t* done = A.sync + A.total_tiles;
    uint32_t* counter = done + A.H;
    auto layer_of = [&](uint32_t tile, int from) {
        int o = from < 0 ? 0 : from;
        while (tile >= A.layers[o].tile_start + A.layers[o].n_tiles) ++o;
        return o;
    };
    if (tid == 0) {
        s_tile[0] = atomicAdd(counter, 1u);
        s_o[0] = s_tile[0] < A.total_tiles ? layer_of(s_tile[0], 0) : 0;
    }
    __syncthreads();
    if (s_tile[0] < A.total_tiles) // the first tile's parameters, synchronously
        for (int i = tid; i < PW; i += blockDim.x)
            reinterpret_cast<uint32_t*>(&sLb[0])[i] =
                __ldg(reinterpret_cast<const uint32_t*>(A.params + (A.H - 1 - s_o[0])) + i);
    for (int it = 0;; ++it) {
        const int bb = it & 1;
        __syncthreads(); // s_tile[bb], s_o[bb], sLb[bb] are complete
        const uint32_t tile = s_tile[bb];
        if (tile >= A.total_tiles) break;
        const int o = s_o[bb];
        const int t = A.H - 1 - o;
        const StreamLayer* Lp = A.layers + o;
        const uint32_t k = tile - Lp->tile_start;
        const int kind = Lp->kind, m = Lp->m;
        if (tid == 0) {
            s_lb = 0ull;
            const uint32_t nx = atomicAdd(counter, 1u); // the next tile, behind this one
            s_tile[bb ^ 1] = nx;
            s_o[bb ^ 1] = nx < A.total_tiles ? layer_of(nx, o) : o;
        }
        // read-only inputs of the tile (rank entries / packed keys, build outputs) are loaded
        // before the dependency wait, so their latency overlaps it
        constexpr int JT = kStreamT / kStreamThreads;
        constexpr int KP = WM <= 2 ? WM : 1; // keys prefetched for narrow keys only
        uint32_t rr[JT];
        uint64_t kpre[JT][KP];
        if (kind != 2) {
            const uint32_t* rank_self = A.rank_tables + Lp->rank_self_off;
            const uint64_t dense_n = Lp->dense_n;
#pragma unroll
            for (int j = 0; j < JT; ++j) {
                const uint64_t d = static_cast<uint64_t>(k) * kStreamT + j * kStreamThreads + tid;
                rr[j] = d < dense_n ? __ldg(rank_self + d) : kEmpty32;
            }
        } else if (WM <= 2) {
            const int words = sLb[bb].words;
            const uint64_t n = Lp->n;
            const uint64_t* keys = A.keys + Lp->key_off;
#pragma unroll
            for (int j = 0; j < JT; ++j) {
                const uint64_t i = static_cast<uint64_t>(k) * kStreamT + j * kStreamThreads + tid;
#pragma unroll
                for (int w = 0; w < KP; ++w)
                    kpre[j][w] = (i < n && w < words) ? __ldg(keys + i * static_cast<uint64_t>(words) + w) : 0ull;
            }
        }
        if (tid < 32) { // dependencies: one lane per flag / counter
            const uint32_t* wp = nullptr;
            uint32_t want = 0;
            if (lane == 0 && o >= kStreamBufs - 1) { // the last reader of buffer t % B is done
                wp = done + o - (kStreamBufs - 1);
                want = A.layers[o - (kStreamBufs - 1)].n_tiles;
            } else if (lane == 1 && o >= 1 && kind != 0) { // all of layer t+1
                wp = done + o - 1;
                want = A.layers[o - 1].n_tiles;
            } else if (lane >= 2 && o >= 1 && kind == 0) { // layer t+1's tiles under the windows
                const int q = (lane - 2) >> 1, half_sel = (lane - 2) & 1;
                if (q < static_cast<int>(Lp->n_shift)) {
                    const int64_t D = static_cast<int64_t>(Lp->dense_n);
                    const int64_t lo = static_cast<int64_t>(k) * kStreamT - Lp->shift[q];
                    const int64_t a = lo < 0 ? 0 : lo;
                    const int64_t b = (lo + kStreamT) > D ? D : (lo + kStreamT);
                    if (b > a) {
                        const int64_t j = half_sel ? (b - 1) / kStreamT : a / kStreamT;
                        wp = flags + A.layers[o - 1].tile_start + j;
                        want = 1u;
                    }
                }
            }
            if (wp) wait_ge(wp, want);
            __syncwarp();
            if (lane == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncthreads();
        // the next tile's layer parameters: loads issued now, stored after the computation
        const int o_next = s_o[bb ^ 1];
        const bool pf = s_tile[bb ^ 1] < A.total_tiles;
        uint32_t pfw[PPT];
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
            const int i = tid + q * kStreamThreads;
            pfw[q] = (pf && i < PW) ? __ldg(reinterpret_cast<const uint32_t*>(A.params + (A.H - 1 - o_next)) + i) : 0u;
        }
        const LayerParam& L = sLb[bb];
        const double2* xn = A.xd + static_cast<uint64_t>((t + 1) % kStreamBufs) * A.third;
        double2* xc = A.xd + static_cast<uint64_t>(t % kStreamBufs) * A.third;
        const bool retires = L.n_keep != L.n_active;
        const SlotDecoder<WM> dec(L);
        double dmax = 0.0;
        const uint64_t row0 = Lp->row0;
        if (kind != 2) { // ---- key-space walk (cert_dense_layer's evaluation) -------------------
            const int na = L.n_active;
            const uint64_t dense_n = Lp->dense_n;
            const uint32_t* rank_self = A.rank_tables + Lp->rank_self_off;
            uint32_t retmask = 0;
#pragma unroll
            for (int p = 0; p < NF; ++p)
                if (p < na && L.keep_idx[p] < 0) retmask |= 1u << p;
            const double r_cl = L.r_cloud, r_pd = L.r_paid, gam = L.gamma;
            const double r_cloud = L.r_cloud_kept, r_paid = L.r_paid_kept;
            const int dem = L.demand;
            (void)rank_self;
#pragma unroll
            for (int j = 0; j < JT; ++j) {
                const uint64_t d = static_cast<uint64_t>(k) * kStreamT + j * kStreamThreads + tid;
                if (d >= dense_n) break;
                const uint32_t r = rr[j];
                if (r == kEmpty32) continue;
                uint32_t rem = static_cast<uint32_t>(d), base = 0, mask = 0;
                int ret_all = 0;
#pragma unroll
                for (int p = 0; p < NF; ++p) {
                    const uint32_t rad = p < na ? L.radix[p] : 1u;
                    const uint32_t gp = rem % rad;
                    rem /= rad;
                    base += gp * dec.wn[p];
                    if (((dec.sw[p] >> 16) & 1u) && gp >= dec.demand) mask |= 1u << p;
                    if ((retmask >> p) & 1u) ret_all += static_cast<int>(gp);
                }
                const Slots sl(static_cast<uint64_t>(base) | (static_cast<uint64_t>(mask) << 32));
                double2 x[SL];
#pragma unroll
                for (int e = 0; e < SL; ++e) {
                    x[e] = make_double2(-INFINITY, -INFINITY);
                    if (sl.valid(e)) x[e] = __ldca(xn + dec.idx(sl, e));
                }
                double hi = -INFINITY, lo = -INFINITY;
                int best = -1;
#pragma unroll
                for (int e = 0; e < SL; ++e) {
                    const int pe = e == SL - 1 ? -1 : e;
                    double rw;
                    if (retires) {
                        const int ret = ret_all - ((pe >= 0 && ((retmask >> pe) & 1u)) ? dem : 0);
                        rw = __dsub_rn(pe < 0 ? r_pd : r_cl, __dmul_rn(gam, static_cast<double>(ret)));
                    } else {
                        rw = pe < 0 ? r_paid : r_cloud;
                    }
                    const double qx = DISC ? __dadd_rn(rw, __dmul_rn(A.discount, x[e].x)) : __dadd_rn(rw, x[e].x);
                    const double qy = DISC ? __dadd_rn(rw, __dmul_rn(A.discount, x[e].y)) : __dadd_rn(rw, x[e].y);
                    if (qy > hi) { // strict: the first maximal edge wins (mdp.cpp:254-260)
                        hi = qy;
                        best = pe;
                    }
                    if (qx > lo) lo = qx;
                }
                if (m == 1) lo = 0.0; // V_0
                xc[d] = make_double2(lo, hi);
                A.values_out[row0 + r] = hi;
                A.act_out[row0 + r] = best < 0 ? -1 : L.cloud[best];
                const double dd = fabs(hi - lo);
                dmax = dmax < dd ? dd : dmax;
            }
        } else { // ---- BFS walk (cert_implicit_layer's evaluation, pairs by key-space index) -------
            const int words = L.words;
            const double r_cloud = L.r_cloud_kept, r_paid = L.r_paid_kept;
            const uint64_t n = Lp->n;
            const uint64_t* keys = A.keys + Lp->key_off;
#pragma unroll
            for (int j = 0; j < JT; ++j) {
                const uint64_t i = static_cast<uint64_t>(k) * kStreamT + j * kStreamThreads + tid;
                if (i >= n) break;
                uint64_t kk[WM];
                if (WM <= 2) {
#pragma unroll
                    for (int w = 0; w < WM; ++w) kk[w] = kpre[j][w < KP ? w : 0];
                } else {
                    load_key<WM>(keys + i * static_cast<uint64_t>(words), words, kk);
                }
                const Slots sl = dec.decode(kk);
                double2 x[SL];
#pragma unroll
                for (int e = 0; e < SL; ++e)
                    if (sl.valid(e)) x[e] = __ldca(xn + dec.idx(sl, e));
                double hi = -INFINITY, lo = -INFINITY;
                int best = -1;
#pragma unroll
                for (int e = 0; e < SL; ++e) {
                    if (!sl.valid(e)) continue;
                    const int pe = e == SL - 1 ? -1 : e;
                    const double rr = retires ? retiring_reward<WM>(kk, pe, L) : (pe < 0 ? r_paid : r_cloud);
                    const double qx = DISC ? __dadd_rn(rr, __dmul_rn(A.discount, x[e].x)) : __dadd_rn(rr, x[e].x);
                    const double qy = DISC ? __dadd_rn(rr, __dmul_rn(A.discount, x[e].y)) : __dadd_rn(rr, x[e].y);
                    if (qy > hi) {
                        hi = qy;
                        best = pe;
                    }
                    if (qx > lo) lo = qx;
                }
                if (m == 1) lo = 0.0;
                if (t >= 1) {
                    uint32_t own = 0;
                    for (int p = 0; p < L.n_active; ++p)
                        own += static_cast<uint32_t>(get_field<WM>(kk, L.bit_off[p], L.width[p])) * L.wself[p];
                    xc[own] = make_double2(lo, hi);
                }
                A.values_out[row0 + i] = hi;
                A.act_out[row0 + i] = best < 0 ? -1 : L.cloud[best];
                const double dd = fabs(hi - lo);
                dmax = dmax < dd ? dd : dmax;
            }
        }
#pragma unroll
        for (int ofs = 16; ofs > 0; ofs >>= 1) {
            const double other = __shfl_xor_sync(FULL, dmax, ofs);
            dmax = dmax < other ? other : dmax;
        }
        if (lane == 0 && dmax > 0.0)
            atomicMax(&s_lb, static_cast<unsigned long long>(__double_as_longlong(dmax)));
        if (pf) { // (sLb[bb ^ 1] is not read by anyone this iteration)
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
                const int i = tid + q * kStreamThreads;
                if (i < PW) reinterpret_cast<uint32_t*>(&sLb[bb ^ 1])[i] = pfw[q];
            }
        }
        __syncthreads(); // the tile's stores are issued
        if (tid == 0) {
            if (s_lb) atomicMax(reinterpret_cast<unsigned long long*>(A.lb + m), s_lb);
            __threadfence();
            st_release_u32(flags + tile, 1u);
            atomicAdd(done + o, 1u);
        }
    }
}

// K* = H+1 is proven iff lb_k >= eps for k = 1..H (and no sweep cap below H+1).  Sets the graph
// conditional to run the wavefront fallback otherwise.
__global__ void k_cert_check(const double* __restrict__ lb, int H, double eps, int max_sweeps,
                             SolveCtrl* ctrl, cudaGraphConditionalHandle fallback) {
    __shared__ int bad;
    if (threadIdx.x == 0) bad = max_sweeps < H + 1 ? 1 : 0;
    __syncthreads();
    for (int k = 1 + threadIdx.x; k <= H; k += blockDim.x)
        if (!(lb[k] >= eps)) bad = 1; // (NaN-safe: anything but a proven lb_k >= eps)
    __syncthreads();
    if (threadIdx.x == 0) {
        if (!bad) {
            ctrl->sweeps = H + 1;
            ctrl->stop = 1;
            ctrl->certified = 1;
        }
        if (fallback) cudaGraphSetConditional(fallback, bad ? 1u : 0u);
    }
}

// Stored doubles of the version store (V_0..V_{m_t} per state, stride wave_stride(m_t)).
uint64_t wave_versions(const vcs_space* sp, std::vector<uint64_t>* off = nullptr) {
    uint64_t tot = 0;
    if (off) off->assign(static_cast<size_t>(sp->H) + 2, 0);
    for (int t = 0; t <= sp->H; ++t) {
        if (off) (*off)[static_cast<size_t>(t)] = tot;
        tot += (sp->layer_off[t + 1] - sp->layer_off[t]) * static_cast<uint64_t>(wave_stride(sp->H - t));
    }
    if (off) (*off)[static_cast<size_t>(sp->H) + 1] = tot;
    return tot;
}

// Backups the wavefront performs: one per (state, version k = 1..m_t).
uint64_t wave_backups(const vcs_space* sp) {
    uint64_t tot = 0;
    for (int t = 0; t <= sp->H; ++t)
        tot += (sp->layer_off[t + 1] - sp->layer_off[t]) * static_cast<uint64_t>(sp->H - t);
    return tot;
}

// (cudaMemGetInfo is avoided: it can stall for milliseconds; an allocation that still fails
// makes VCS_METHOD_AUTO fall back to Jacobi.)
bool wavefront_fits(const vcs_space* sp) {
    const uint64_t need = wave_versions(sp) * sizeof(double) + (sp->H + 2) * 16;
    return sp->ver.n >= wave_versions(sp) || need < device_bytes(sp->device) / 2;
}

void ensure_wave_buffers(vcs_space* sp, bool sync = true) {
    std::vector<uint64_t> off;
    const uint64_t nv = wave_versions(sp, &off);
    const double t0 = trace_enabled() ? host_ms() : 0.0;
    sp->ver.exact(std::max<uint64_t>(nv, 1), sp->stream);
    if (trace_enabled()) {
        cudaStreamSynchronize(sp->stream);
        std::fprintf(stderr, "[vcs solve] version store %.1f MB alloc %.3f ms\n", nv * 8e-6,
                     host_ms() - t0);
    }
    const double t1 = trace_enabled() ? host_ms() : 0.0;
    sp->ver_off.exact(off.size(), sp->stream);
    sp->layer_off_dev.exact(sp->layer_off.size(), sp->stream);
    const double t2 = trace_enabled() ? host_ms() : 0.0;
    sp->ver_off_host = std::move(off); // lives with the space: the async copies read it
    VCS_CUDA(cudaMemcpyAsync(sp->ver_off.p, sp->ver_off_host.data(), sp->ver_off_host.size() * 8,
                             cudaMemcpyHostToDevice, sp->stream));
    VCS_CUDA(cudaMemcpyAsync(sp->layer_off_dev.p, sp->layer_off.data(), sp->layer_off.size() * 8,
                             cudaMemcpyHostToDevice, sp->stream));
    const double t3 = trace_enabled() ? host_ms() : 0.0;
    if (sync) VCS_CUDA(cudaStreamSynchronize(sp->stream)); // solves may run on a caller's stream
    if (trace_enabled())
        std::fprintf(stderr, "[vcs solve] offsets alloc %.3f copy %.3f sync %.3f ms\n", t2 - t1,
                     t3 - t2, host_ms() - t3);
}

int max_key_words(const vcs_space* sp) {
    int wm = 1;
    for (int w : sp->plan.words) wm = std::max(wm, w);
    return wm;
}

template <class F>
void dispatch_words_solve(int wm, F&& f) {
    if (wm <= 1) f(std::integral_constant<int, 1>{});
    else if (wm <= 2) f(std::integral_constant<int, 2>{});
    else if (wm <= 4) f(std::integral_constant<int, 4>{});
    else f(std::integral_constant<int, 8>{});
}

void record_event(cudaEvent_t ev, cudaStream_t s, bool capturing) {
    if (capturing)
        VCS_CUDA(cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal));
    else
        VCS_CUDA(cudaEventRecord(ev, s));
}

// Enqueue one wavefront solve on `s` (directly, or into a stream capture).
// Raise a kernel's dynamic shared-memory limit on `device` to at least `smem` — only ever
// upwards, and once per (kernel, device, size) (the attribute is per device context).
void raise_smem_limit(const void* fn, int device, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> set;
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = set[{fn, device}];
    if (smem <= cur) return;
    const size_t want = std::max<size_t>(smem, 48 * 1024);
    VCS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(want)));
    cur = want;
}

// Launch k_wave_layer for the band [a.band_lo, a.band_hi) of one layer (a.row0 / n / m /
// strides / bases set by the caller): tile size, shared memory, grid.
void launch_layer(vcs_space* sp, WaveArgs& a, bool disc, cudaStream_t s) {
    // 4 gathers in flight per thread, 4 blocks per SM (64 registers): measured best of
    // (U, blocks) in {(8,3), (4,4), (4,5), (2,6)} on C4
    using LayerFn = void (*)(WaveArgs);
    const bool band = a.band_lo != 1 || a.base != 0 || a.base_next != 0;
    const LayerFn layer_fn = band ? (disc ? k_wave_layer<true, 4, 4, true> : k_wave_layer<false, 4, 4, true>)
                                  : (disc ? k_wave_layer<true, 4, 4, false> : k_wave_layer<false, 4, 4, false>);
    const void* fn = reinterpret_cast<const void*>(layer_fn);
    const int nb = a.band_hi - a.band_lo;
    if (nb <= 0 || a.n == 0) return;
    a.ver_next = a.ver + a.voff_next;
    a.ver_cur = a.ver + a.voff;
    const int qcap = std::max(1, sp->max_degree);
    // tile: whole passes of (states x 2-version groups) threads (the staging of a tile's CSR is
    // amortised over its passes); a small layer gets fewer passes per tile so that its tiles
    // still cover every SM (its passes run in parallel instead)
    const int G = (nb + 1) / 2;
    const int spp = G > kWaveWarps * 32 ? 1 : (kWaveWarps * 32) / G;
    a.max_deg = qcap;
    auto smem_for = [&](int tile) {
        return static_cast<size_t>(nb) * 8 + static_cast<size_t>(tile) * (nb + 1) * 8 +
               static_cast<size_t>(tile) * qcap * 16 + static_cast<size_t>(tile + 1) * 4;
    };
    // 4 passes per tile measured best on C4 (3.96 ms vs 4.49 with 8: the smaller tile's shared
    // memory lets 4 blocks per SM be resident, the register limit); VCS_WAVE_PASSES overrides
    static const int max_passes = [] {
        const char* e = std::getenv("VCS_WAVE_PASSES");
        return e ? std::max(1, std::atoi(e)) : 4;
    }();
    a.tile = G > kWaveWarps * 32 ? 2 : std::min(512, spp * max_passes);
    size_t smem = smem_for(a.tile);
    if (smem > 200 * 1024) raise(VCS_EINVAL, "horizon/out-degree too large for the wavefront tile");
    raise_smem_limit(fn, sp->device, smem);
    int per_sm = 0;
    VCS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kWaveWarps * 32, smem));
    const uint64_t slots = static_cast<uint64_t>(std::max(1, per_sm)) * sp->num_sms;
    if (G <= kWaveWarps * 32 && (a.n + a.tile - 1) / a.tile < slots) {
        const uint64_t per_tile = std::max<uint64_t>(1, (a.n + slots - 1) / slots); // states
        const uint64_t passes = std::min<uint64_t>(max_passes, (per_tile + spp - 1) / spp);
        a.tile = static_cast<int>(std::min<uint64_t>(512, spp * passes));
        smem = smem_for(a.tile);
    }
    const uint64_t tiles = (a.n + a.tile - 1) / a.tile;
    const uint64_t blocks = std::max<uint64_t>(
        1, std::min<uint64_t>(tiles, static_cast<uint64_t>(std::max(1, per_sm)) * sp->num_sms));
    layer_fn<<<static_cast<unsigned>(blocks), kWaveWarps * 32, smem, s>>>(a);
    VCS_LAUNCHED();
}

// `events` = false: no event nodes (the fallback body of a certified graph may not hold any).
void record_wavefront(vcs_space* sp, const GraphKey& key, CachedGraph& g, cudaStream_t s,
                      bool capturing, bool events = true) {
    const bool disc = is_discounted(key.discount);
    WaveArgs a{};
    a.row_ptr = sp->row_ptr.p;
    a.succ = sp->succ.p;
    a.reward = sp->reward.p;
    a.action = sp->action.p;
    a.ver = sp->ver.p;
    a.ver_off = sp->ver_off.p;
    a.layer_off = sp->layer_off_dev.p;
    a.delta = sp->delta.p;
    a.ctrl = sp->ctrl.p;
    a.values_out = sp->v[0].p;
    a.act_out = sp->actions_dev.p;
    a.eps = key.eps;
    a.discount = key.discount;
    a.H = sp->H;
    a.max_sweeps = key.max_sweeps;
    const void* fn_ext = disc ? reinterpret_cast<const void*>(k_wave_extract<true>)
                              : reinterpret_cast<const void*>(k_wave_extract<false>);
    const int qcap = std::max(1, sp->max_degree);
    const size_t smem_ext = static_cast<size_t>(sp->H + 2) * 16 +
                            static_cast<size_t>(kWaveWarps) * 32 * qcap * sizeof(double);
    if (smem_ext > 200 * 1024) raise(VCS_EINVAL, "out-degree too large for the extraction kernel");
    VCS_CUDA(cudaFuncSetAttribute(fn_ext, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(std::max<size_t>(smem_ext, 1024))));
    VCS_CUDA(cudaMemsetAsync(sp->delta.p, 0, (sp->H + 3) * sizeof(double), s));
    VCS_CUDA(cudaMemsetAsync(sp->ctrl.p, 0, sizeof(SolveCtrl), s));
    if (events) record_event(g.ev[0], s, capturing);
    // terminal layer: V = 0.0 (+0), action = kPaidCloud (mdp.cpp:248-251); its stored V_0 = 0
    {
        const uint64_t rH = sp->layer_off[sp->H], nH = sp->S - rH;
        VCS_CUDA(cudaMemsetAsync(sp->v[0].p + rH, 0, nH * sizeof(double), s));
        VCS_CUDA(cudaMemsetAsync(sp->actions_dev.p + rH, 0xff, nH * sizeof(int32_t), s));
        VCS_CUDA(cudaMemsetAsync(sp->ver.p + sp->ver_off_host[sp->H], 0,
                                 nH * wave_stride(0) * sizeof(double), s));
    }
    int launches = 0;
    for (int t = sp->H - 1; t >= 0; --t) {
        a.row0 = sp->layer_off[t];
        a.n = sp->layer_off[t + 1] - sp->layer_off[t];
        a.next_row0 = sp->layer_off[t + 1];
        a.voff = sp->ver_off_host[t];
        a.voff_next = sp->ver_off_host[t + 1];
        a.m = sp->H - t;
        a.band_lo = 1; // single GPU: every version of the layer
        a.band_hi = a.m + 1;
        a.next_lo = 1;
        a.base = 0;
        a.base_next = 0;
        a.stride = wave_stride(a.m);
        a.stride_next = wave_stride(a.m - 1);
        launch_layer(sp, a, disc, s);
        ++launches;
        // layer t's values/actions are final here (unless an early stop needs the fix-up):
        // lets vcs_solve stream them to the host while the remaining layers compute
        if (events && !g.layer_ev.empty() && g.layer_ev[static_cast<size_t>(t)])
            record_event(g.layer_ev[static_cast<size_t>(t)], s, capturing);
    }
    if (events) record_event(g.ev[1], s, capturing);
    int per_sm_ext = 0;
    VCS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_ext, fn_ext, kWaveWarps * 32,
                                                           smem_ext));
    const uint64_t eblocks = std::max<uint64_t>(
        1, std::min<uint64_t>((sp->S + 255) / 256,
                              static_cast<uint64_t>(std::max(1, per_sm_ext)) * sp->num_sms));
    if (disc)
        k_wave_extract<true><<<static_cast<unsigned>(eblocks), kWaveWarps * 32, smem_ext, s>>>(a, qcap);
    else
        k_wave_extract<false><<<static_cast<unsigned>(eblocks), kWaveWarps * 32, smem_ext, s>>>(a, qcap);
    VCS_LAUNCHED();
    if (events) record_event(g.ev[2], s, capturing);
    g.launches = launches + 1;
}

// Enqueue one certified solve: the two-version backward pass, the proof, and the full
// wavefront as the body of a graph IF node that runs only when the proof fails.
//
// Implicit spaces keep the (V_{m-1}, V_m) pairs by key-space index in two halves of the largest
// layer key space (layer t in half t & 1); otherwise (and with VCS_CERT_BFS=1) by BFS index.
bool cert_keyspace(const vcs_space* sp) {
    return sp->implicit && sp->has_plan && !std::getenv("VCS_CERT_BFS");
}
uint64_t cert_half(const vcs_space* sp) {
    uint64_t h = 1;
    for (int t = 1; t <= sp->H; ++t)
        h = std::max<uint64_t>(h, sp->plan.layers[static_cast<size_t>(t - 1)].dense_size);
    return h;
}
bool cert_permute_layer(uint64_t key_space);
// The persistent streaming pass (k_cert_stream, opt-in: VCS_CERT_STREAM=1) applies to key-space
// spaces whose layers stay in L2 (the gather-pass layout of larger ones is per layer).
// Measured on the B200 it is correct and deadlock-free but slower than the PDL-chained layer
// launches: C4 0.75 vs 0.52 ms, C3 0.34 vs 0.18 ms.
bool cert_stream_space(const vcs_space* sp) {
    const char* e = std::getenv("VCS_CERT_STREAM");
    if (!e || std::atoi(e) == 0) return false;
    return cert_keyspace(sp) && !cert_permute_layer(cert_half(sp)) && sp->H >= 1;
}
uint64_t cert_pairs_needed(const vcs_space* sp) {
    // (the streaming pass rotates three buffers, the per-layer launches two)
    return cert_keyspace(sp) ? (cert_stream_space(sp) ? 4 : 2) * cert_half(sp) : sp->S;
}

// Device pointers of the implicit form a certified layer reads (the space's own, or a replica
// of them on another GPU for the multi-GPU pass).
struct CertData {
    const uint64_t* keys;
    const uint32_t* rank_tables;
    const LayerParam* params;
};
CertData cert_data_of(const vcs_space* sp) {
    return CertData{sp->keys.p, sp->rank_tables.p, sp->params_dev.p};
}

// Layer t of the certified pass on the implicit form: which kernel walks it and where its pairs
// live.  Key-space layout (ks): layer t's pairs in half t&1 of `xd` at their key-space index.
struct CertLayer {
    int t = 0;
    uint64_t row0 = 0, n = 0;  // the layer's states (BFS rows)
    uint64_t dense_n = 0;      // the layer's key-space size (0 for the root)
    bool dense_order = false;  // a thread per key-space index (k_cert_dense)
    double2* xd_next = nullptr;
    double2* xd_cur = nullptr;
    uint64_t d_lo = 0, d_hi = 0; // k_cert_dense: the indices of this launch
};
CertLayer cert_layer(const vcs_space* sp, int t, double2* xd, uint64_t half, bool ks) {
    CertLayer L;
    L.t = t;
    L.row0 = sp->layer_off[t];
    L.n = sp->layer_off[t + 1] - sp->layer_off[t];
    if (ks) {
        L.xd_next = xd + ((t + 1) & 1) * half;
        L.xd_cur = xd + (t & 1) * half;
        L.dense_n = t >= 1 ? sp->plan.layers[static_cast<size_t>(t - 1)].dense_size : 0;
        // walk the key space when at least half of it is reached (coalesced pair writes, no
        // key loads); sparse layers walk their states
        L.dense_order = t >= 1 && L.n * 2 >= L.dense_n; // (0.4 / 0.3 / 0.2 measured the same on C4)
    } else {
        L.xd_next = xd + sp->layer_off[t + 1];
        L.xd_cur = xd + L.row0;
    }
    return L;
}

// Layer t's transition keeps every cloud with the same numbering (succ = d - demand*W_p): the
// TMA-staged kernel applies.
// Whether a full layer of this key-space size writes its results in key-space order and lets
// k_cert_permute reorder them (VCS_CERT_PERMUTE=0/1 forces it).  Measured on the B200: the
// scattered value/action stores are 48 % of C7's certified pass (76 MB pair vectors per layer);
// the gather pass brings C7 from 5.36 to 4.91 ms, while on C4 (L2-resident, 8.5 MB) the extra
// launches cost more than the scatter (0.71 vs 0.53 ms).
bool cert_permute_layer(uint64_t key_space) {
    if (const char* e = std::getenv("VCS_CERT_PERMUTE")) return std::atoi(e) != 0;
    return 16 * key_space > (48ull << 20);
}
bool cert_permute_space(const vcs_space* sp) {
    return cert_keyspace(sp) && cert_permute_layer(cert_half(sp));
}

// Layer t's transition keeps every cloud with the same numbering, so succ = d - demand*W_p.
bool cert_nonretiring(const vcs_space* sp, int t) {
    if (t < 1 || t >= sp->H) return false;
    const LayerParam& P = sp->plan.layers[static_cast<size_t>(t)];
    if (P.n_keep != P.n_active || P.dense_size == 0 || P.self_size != P.dense_size) return false;
    for (int p = 0; p < P.n_active; ++p)
        if (P.keep_idx[p] != p || P.wnext[p] != P.wself[p]) return false;
    return P.n_active <= kDenseSlots - 1;
}

// (Opt-in, VCS_CERT_TMA=1: measured on the B200 it does not beat k_cert_dense — C4 0.63 vs
// 0.52 ms, C7 5.6 vs 5.4 ms; its consumers wait on the bulk copies while the scattered
// value/action stores, 27 % of the C7 time, stay.  DESIGN.md section 3.4.)
bool cert_tma_ok(const vcs_space* sp, int t) {
    if (t < 1 || t >= sp->H || !std::getenv("VCS_CERT_TMA")) return false;
    const LayerParam& P = sp->plan.layers[static_cast<size_t>(t)];
    if (P.n_keep != P.n_active || P.dense_size == 0 || P.self_size != P.dense_size) return false;
    for (int p = 0; p < P.n_active; ++p)
        if (P.keep_idx[p] != p || P.wnext[p] != P.wself[p]) return false;
    return P.n_active <= kDenseSlots - 1;
}

// Launch one certified layer on the implicit form (on the current device's stream `s`).
void launch_cert_layer(const vcs_space* sp, const CertData& data, const CertLayer& L,
                       double* values_out, int32_t* act_out, double* lb, double discount,
                       int write_out, bool pdl, cudaStream_t s) {
    const bool disc = is_discounted(discount);
    const int t = L.t;
    const bool ks = cert_keyspace(sp);
    CertImplArgs c{};
    c.values_out = values_out;
    c.act_out = act_out;
    c.lb = lb;
    c.discount = discount;
    c.row0 = L.row0;
    c.n = L.n;
    c.m = sp->H - t;
    c.keys = data.keys + sp->key_off[t];
    c.L = data.params + t;
    c.rank = data.rank_tables + sp->rank_off[t];
    c.xd_next = L.xd_next;
    c.xd_cur = L.xd_cur;
    c.write_out = write_out;
    c.tl = sp->cert_tl.n ? sp->cert_tl.p : nullptr;
    if (ks) {
        c.dense_n = L.dense_n;
        c.rank_self = t >= 1 ? data.rank_tables + sp->rank_off[static_cast<size_t>(t - 1)] : nullptr;
        c.write_own = t >= 1 ? 1 : 0;
        c.d_lo = L.d_lo;
        c.d_hi = L.d_hi;
    }
    const bool dense_order = L.dense_order;
    // the non-retiring walk pays with the gather pass on layers beyond L2 (C7); on L2-resident
    // layers (C4) the generic walk measured as fast or faster (0.517 vs 0.530 ms)
    static const bool win_on = std::getenv("VCS_CERT_WIN") != nullptr;
    if (dense_order && ks && cert_nonretiring(sp, t) && !cert_permute_layer(L.dense_n) && win_on &&
        !std::getenv("VCS_CERT_GENERIC") && !std::getenv("VCS_CERT_TMA") &&
        !std::getenv("VCS_CERT_ILP2")) {
        // the near successors from a shared-memory window per tile (k_cert_dense_win)
        const void* fn = disc ? reinterpret_cast<const void*>(k_cert_dense_win<true>)
                              : reinterpret_cast<const void*>(k_cert_dense_win<false>);
        static thread_local std::map<std::pair<const void*, int>, int> occ_win;
        int dev = 0;
        VCS_CUDA(cudaGetDevice(&dev));
        int& per_sm = occ_win[{fn, dev}];
        if (!per_sm) VCS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kWinT, 0));
        const uint64_t items = L.d_hi > L.d_lo ? L.d_hi - L.d_lo : 0;
        const uint64_t blocks = std::max<uint64_t>(
            1, std::min<uint64_t>((items + kWinT - 1) / kWinT,
                                  static_cast<uint64_t>(std::max(1, per_sm)) * sp->num_sms));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(blocks));
        cfg.blockDim = dim3(kWinT);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        if (disc) VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense_win<true>, c));
        else VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense_win<false>, c));
        VCS_LAUNCHED();
        return;
    }
    static const bool nr_all = std::getenv("VCS_CERT_NR") != nullptr; // (measurement switch)
    if (dense_order && ks && cert_nonretiring(sp, t) && (cert_permute_layer(L.dense_n) || nr_all) &&
        !std::getenv("VCS_CERT_GENERIC") && !std::getenv("VCS_CERT_TMA") &&
        !std::getenv("VCS_CERT_ILP2")) {
        const void* fn = disc ? reinterpret_cast<const void*>(k_cert_dense_nr<true>)
                              : reinterpret_cast<const void*>(k_cert_dense_nr<false>);
        static thread_local std::map<std::pair<const void*, int>, int> occ_nr;
        int dev = 0;
        VCS_CUDA(cudaGetDevice(&dev));
        int& per_sm = occ_nr[{fn, dev}];
        if (!per_sm) VCS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
        const uint64_t items = L.d_hi > L.d_lo ? L.d_hi - L.d_lo : 0;
        const uint64_t blocks = std::max<uint64_t>(
            1, std::min<uint64_t>((items + 255) / 256,
                                  static_cast<uint64_t>(std::max(1, per_sm)) * sp->num_sms));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(blocks));
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        CertImplArgs cx = c;
        // pair vectors beyond L2 (C7): results in key-space order + a gather pass to BFS order
        // (single GPU only: a rank of the multi-GPU pass holds only its range's pairs)
        const bool permute = sp->cert_act_ks.p && c.write_out && L.d_lo == 0 &&
                             L.d_hi == L.dense_n && cert_permute_layer(L.dense_n);
        if (permute) cx.act_ks = sp->cert_act_ks.p;
        if (permute) {
            if (disc) VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense_nr<true, false>, cx));
            else VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense_nr<false, false>, cx));
        } else {
            if (disc) VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense_nr<true, true>, cx));
            else VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense_nr<false, true>, cx));
        }
        if (permute) {
            VCS_LAUNCHED();
            dispatch_words_solve(max_key_words(sp), [&](auto wm) {
                constexpr int WM = decltype(wm)::value;
                const unsigned pb = static_cast<unsigned>(std::min<uint64_t>(
                    (L.n + 255) / 256, static_cast<uint64_t>(sp->num_sms) * 8));
                k_cert_permute<WM><<<std::max(1u, pb), 256, 0, s>>>(
                    data.keys + sp->key_off[t], data.params + t, L.xd_cur, sp->cert_act_ks.p, L.n,
                    L.row0, values_out, act_out);
            });
        }
        VCS_LAUNCHED();
        return;
    }
    if (dense_order && ks && cert_tma_ok(sp, t)) {
        // the successor windows staged in shared memory by bulk copies (k_cert_dense_tma)
        const void* fn = disc ? reinterpret_cast<const void*>(k_cert_dense_tma<true>)
                              : reinterpret_cast<const void*>(k_cert_dense_tma<false>);
        int dev = 0;
        VCS_CUDA(cudaGetDevice(&dev));
        raise_smem_limit(fn, dev, sizeof(TmaSmem));
        const uint64_t tiles = L.d_hi > L.d_lo ? (L.d_hi - L.d_lo + kTmaT - 1) / kTmaT : 0;
        const uint64_t blocks =
            std::max<uint64_t>(1, std::min<uint64_t>(tiles, static_cast<uint64_t>(2) * sp->num_sms));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(blocks));
        cfg.blockDim = dim3(kTmaThreads);
        cfg.dynamicSmemBytes = sizeof(TmaSmem);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        const uint64_t d_next = sp->plan.layers[static_cast<size_t>(t)].dense_size;
        if (disc) VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense_tma<true>, c, d_next));
        else VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense_tma<false>, c, d_next));
        VCS_LAUNCHED();
        return;
    }
    // (opt-in, VCS_CERT_ILP2=1: two indices in flight per thread; measured no faster on the
    // B200 — C7 5.58 vs 5.42 ms, C4 0.55 vs 0.52 ms — the gathers are not latency-per-thread
    // bound)
    const char* ilp_env = std::getenv("VCS_CERT_ILP2");
    const bool ilp2 = dense_order && ks && ilp_env && std::atoi(ilp_env) != 0;
    if (ilp2) {
        dispatch_words_solve(max_key_words(sp), [&](auto wm) {
            constexpr int WM = decltype(wm)::value;
            const void* fn = disc ? reinterpret_cast<const void*>(k_cert_dense2<WM, true>)
                                  : reinterpret_cast<const void*>(k_cert_dense2<WM, false>);
            int dev = 0;
            VCS_CUDA(cudaGetDevice(&dev));
            static thread_local std::map<std::pair<const void*, int>, int> occ2;
            int& per_sm = occ2[{fn, dev}];
            if (!per_sm) VCS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
            const uint64_t items = L.d_hi > L.d_lo ? L.d_hi - L.d_lo : 0;
            const uint64_t blocks = std::max<uint64_t>(
                1, std::min<uint64_t>((items + 511) / 512,
                                      static_cast<uint64_t>(std::max(1, per_sm)) * sp->num_sms));
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(static_cast<unsigned>(blocks));
            cfg.blockDim = dim3(256);
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = pdl ? 1 : 0;
            if (disc) VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense2<WM, true>, c));
            else VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense2<WM, false>, c));
            VCS_LAUNCHED();
        });
        return;
    }
    if (trace_enabled())
        std::fprintf(stderr, "[vcs solve] cert layer %d: n=%llu key space=%llu %s [%llu, %llu)\n", t,
                     static_cast<unsigned long long>(L.n), static_cast<unsigned long long>(L.dense_n),
                     dense_order ? "dense" : "sparse", static_cast<unsigned long long>(L.d_lo),
                     static_cast<unsigned long long>(L.d_hi));
    dispatch_words_solve(max_key_words(sp), [&](auto wm) {
        constexpr int WM = decltype(wm)::value;
        // the key-walking kernel: 3 blocks per SM for keys of <= 2 words (80 registers, no
        // spills); wide keys (4 / 8 words: many-cloud instances) take 2 so they do not spill
        constexpr int IMB = WM <= 2 ? 3 : 2;
        // 3 blocks per SM (80 registers, no spills): C4 0.68 ms vs 0.72 at 4, 0.74 at 2
        static const int cert_minb = [] {
            const char* e = std::getenv("VCS_CERT_MINB"); // (measurements: 2 / 4 blocks per SM)
            const int v = e ? std::atoi(e) : 3;
            return v == 2 || v == 4 ? v : 3;
        }();
        const void* fn =
            dense_order ? (disc ? reinterpret_cast<const void*>(k_cert_dense<WM, true, 3>)
                                : cert_minb == 4 ? reinterpret_cast<const void*>(k_cert_dense<WM, false, 4>)
                                : cert_minb == 2 ? reinterpret_cast<const void*>(k_cert_dense<WM, false, 2>)
                                                 : reinterpret_cast<const void*>(k_cert_dense<WM, false, 3>))
                        : (disc ? reinterpret_cast<const void*>(k_cert_implicit<WM, true, IMB, false>)
                                : reinterpret_cast<const void*>(k_cert_implicit<WM, false, IMB, false>));
        static thread_local std::map<std::pair<const void*, int>, int> occ;
        int dev = 0;
        VCS_CUDA(cudaGetDevice(&dev));
        int& per_sm = occ[{fn, dev}];
        if (!per_sm) VCS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
        const uint64_t items = dense_order ? (L.d_hi > L.d_lo ? L.d_hi - L.d_lo : 0) : L.n;
        const uint64_t blocks = std::max<uint64_t>(
            1, std::min<uint64_t>((items + 255) / 256,
                                  static_cast<uint64_t>(std::max(1, per_sm)) * sp->num_sms));
        // layers after the first launch programmatically (PDL): their blocks load the layer
        // constants and first keys while the previous layer drains.  Not with per-layer events
        // in between (vcs_solve's streamed download) nor across streams.
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(blocks));
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        if (dense_order) {
            if (disc) VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense<WM, true, 3>, c));
            else if (cert_minb == 4) VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense<WM, false, 4>, c));
            else if (cert_minb == 2) VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense<WM, false, 2>, c));
            else VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_dense<WM, false, 3>, c));
        } else if (ks) {
            if (disc) VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_implicit<WM, true, IMB, true>, c));
            else VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_implicit<WM, false, IMB, true>, c));
        } else {
            if (disc) VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_implicit<WM, true, IMB, false>, c));
            else VCS_CUDA(cudaLaunchKernelEx(&cfg, k_cert_implicit<WM, false, IMB, false>, c));
        }
        VCS_LAUNCHED();
    });
}

// The bottom run of small sparse layers that k_cert_tail takes (every layer 0..t_tail walks its
// states, none has more than kTailMaxStates), and their row / key offsets on the device; built
// once per space before any capture.  cert_tail_t = -1: no tail.
void ensure_cert_tail(vcs_space* sp) {
    if (sp->cert_tail_ready) return;
    sp->cert_tail_ready = true;
    sp->cert_tail_t = -1;
    // (opt-in, VCS_CERT_TAIL=1: measured slower on the B200 — C4 0.543 vs 0.518 ms; the
    // PDL-chained launches of those layers overlap better than one block walking them)
    if (!cert_keyspace(sp) || !std::getenv("VCS_CERT_TAIL")) return;
    const uint64_t half = cert_half(sp);
    int t_tail = -1;
    for (int t = 0; t < sp->H; ++t) {
        const CertLayer L = cert_layer(sp, t, nullptr, half, true);
        if (L.dense_order || L.n > kTailMaxStates) break;
        t_tail = t;
    }
    if (t_tail < 1) return; // a single layer gains nothing
    std::vector<uint64_t> meta(3 * (static_cast<size_t>(t_tail) + 1));
    for (int t = 0; t <= t_tail; ++t) {
        meta[3 * t] = sp->layer_off[static_cast<size_t>(t)];
        meta[3 * t + 1] = sp->layer_off[static_cast<size_t>(t) + 1] - sp->layer_off[static_cast<size_t>(t)];
        meta[3 * t + 2] = sp->key_off[static_cast<size_t>(t)];
    }
    sp->cert_tail_meta.exact(meta.size(), sp->stream);
    VCS_CUDA(cudaMemcpyAsync(sp->cert_tail_meta.p, meta.data(), meta.size() * 8, cudaMemcpyHostToDevice,
                             sp->stream));
    VCS_CUDA(cudaStreamSynchronize(sp->stream));
    sp->cert_tail_t = t_tail;
}

// The streaming pass's per-layer table (processing order) and its sync words, built once per
// space before any capture.
void ensure_stream_plan(vcs_space* sp) {
    if (sp->stream_meta.p && sp->stream_tiles) return;
    const int H = sp->H;
    const uint64_t half = cert_half(sp);
    std::vector<StreamLayer> ly(static_cast<size_t>(H));
    uint32_t tiles = 0;
    for (int o = 0; o < H; ++o) {
        const int t = H - 1 - o;
        const CertLayer L = cert_layer(sp, t, nullptr, half, true);
        StreamLayer& Y = ly[static_cast<size_t>(o)];
        Y.row0 = L.row0;
        Y.n = L.n;
        Y.dense_n = L.dense_n;
        Y.key_off = sp->key_off[static_cast<size_t>(t)];
        Y.rank_self_off = t >= 1 ? sp->rank_off[static_cast<size_t>(t - 1)] : 0;
        Y.m = H - t;
        if (L.dense_order) {
            // window deps need layer t+1 walked in the same key space (a key-space-walk layer
            // of the same size) and a non-retiring transition
            bool local = cert_nonretiring(sp, t) && o >= 1;
            if (local) {
                const CertLayer P = cert_layer(sp, t + 1, nullptr, half, true);
                local = P.dense_order && P.dense_n == L.dense_n;
            }
            Y.kind = local ? 0 : 1;
            Y.n_tiles = static_cast<uint32_t>((L.dense_n + kStreamT - 1) / kStreamT);
            if (local) {
                const LayerParam& P = sp->plan.layers[static_cast<size_t>(t)];
                Y.n_shift = 0;
                Y.shift[Y.n_shift++] = 0; // the paid successor: d itself
                for (int p = 0; p < P.n_active && p < kDenseSlots - 1; ++p)
                    if (P.attr[p]) Y.shift[Y.n_shift++] = static_cast<uint32_t>(P.demand) * P.wnext[p];
            }
        } else {
            Y.kind = 2;
            Y.n_tiles = static_cast<uint32_t>((L.n + kStreamT - 1) / kStreamT);
        }
        Y.tile_start = tiles;
        tiles += Y.n_tiles;
    }
    const size_t bytes = ly.size() * sizeof(StreamLayer);
    sp->stream_meta.exact(std::max<size_t>(bytes, 16), sp->stream);
    sp->stream_sync.exact(static_cast<size_t>(tiles) + static_cast<size_t>(H) + 1, sp->stream);
    VCS_CUDA(cudaMemcpyAsync(sp->stream_meta.p, ly.data(), bytes, cudaMemcpyHostToDevice, sp->stream));
    VCS_CUDA(cudaStreamSynchronize(sp->stream));
    sp->stream_tiles = tiles;
}

void record_certified(vcs_space* sp, const GraphKey& key, CachedGraph& g, cudaStream_t s,
                      bool capturing) {
    const bool disc = is_discounted(key.discount);
    const int H = sp->H;
    // (cert_xd / cert_lb are allocated before capture: an allocation inside a capture would
    // become a graph allocation node, and such a graph cannot be relaunched)
    const bool ks = cert_keyspace(sp);
    const uint64_t half = ks ? cert_half(sp) : 0;
    if (sp->cert_xd.n < cert_pairs_needed(sp) || sp->cert_lb.n < static_cast<size_t>(H) + 2)
        raise(VCS_EINVAL, "certified solve buffers were not allocated");
    VCS_CUDA(cudaMemsetAsync(sp->ctrl.p, 0, sizeof(SolveCtrl), s));
    VCS_CUDA(cudaMemsetAsync(sp->cert_lb.p, 0, (H + 2) * sizeof(double), s));
    record_event(g.ev[0], s, capturing);
    {
        const uint64_t rH = sp->layer_off[H], nH = sp->S - rH;
        VCS_CUDA(cudaMemsetAsync(sp->v[0].p + rH, 0, nH * sizeof(double), s));
        VCS_CUDA(cudaMemsetAsync(sp->actions_dev.p + rH, 0xff, nH * sizeof(int32_t), s));
        if (ks) // the terminal layer's single state, key-space index 0 (buffer H % 3 streaming)
            VCS_CUDA(cudaMemsetAsync(sp->cert_xd.p + (key.stream_out == 0 && cert_stream_space(sp)
                                                          ? (H % 4) : (H & 1)) * half,
                                     0, sizeof(double2), s));
        else
            VCS_CUDA(cudaMemsetAsync(sp->cert_xd.p + rH, 0, nH * sizeof(double2), s)); // V_0 = 0
    }
    if (sp->implicit && ks && key.stream_out == 0 && cert_stream_space(sp) && sp->stream_tiles) {
        // the whole pass as one persistent kernel (k_cert_stream)
        VCS_CUDA(cudaMemsetAsync(sp->stream_sync.p, 0,
                                 (static_cast<size_t>(sp->stream_tiles) + H + 1) * sizeof(uint32_t), s));
        StreamArgs A{};
        A.layers = reinterpret_cast<const StreamLayer*>(sp->stream_meta.p);
        A.params = sp->params_dev.p;
        A.keys = sp->keys.p;
        A.rank_tables = sp->rank_tables.p;
        A.xd = sp->cert_xd.p;
        A.third = half;
        A.values_out = sp->v[0].p;
        A.act_out = sp->actions_dev.p;
        A.lb = sp->cert_lb.p;
        A.discount = key.discount;
        A.sync = sp->stream_sync.p;
        A.total_tiles = sp->stream_tiles;
        A.H = H;
        dispatch_words_solve(max_key_words(sp), [&](auto wm) {
            constexpr int WM = decltype(wm)::value;
            const void* fn = disc ? reinterpret_cast<const void*>(k_cert_stream<WM, true>)
                                  : reinterpret_cast<const void*>(k_cert_stream<WM, false>);
            int per_sm = 0;
            VCS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kStreamThreads, 0));
            const unsigned blocks = static_cast<unsigned>(std::max(1, per_sm) * sp->num_sms);
            if (disc) k_cert_stream<WM, true><<<blocks, kStreamThreads, 0, s>>>(A);
            else k_cert_stream<WM, false><<<blocks, kStreamThreads, 0, s>>>(A);
            VCS_LAUNCHED();
        });
        k_cert_check<<<1, 64, 0, s>>>(sp->cert_lb.p, H, key.eps, key.max_sweeps, sp->ctrl.p, 0);
        VCS_LAUNCHED();
        record_event(g.ev[1], s, capturing);
        record_event(g.ev[2], s, capturing);
        g.launches = 2;
        g.implicit = true;
        g.fallback_at_collect = true;
        return;
    }
    if (sp->implicit) { // implicit-CSR form: keys + rank tables; the fallback runs at collect
        const CertData data = cert_data_of(sp);
        int launches = 0;
        // PDL chains the layer launches, except right behind a download event
        const bool pdl = !std::getenv("VCS_NO_PDL");
        // the small sparse layers at the bottom run as one single-block launch (k_cert_tail)
        const int t_tail = ks ? sp->cert_tail_t : -1;
        for (int t = H - 1; t >= 0; --t) {
            if (t == t_tail) {
                CertImplArgs c{};
                c.values_out = sp->v[0].p;
                c.act_out = sp->actions_dev.p;
                c.lb = sp->cert_lb.p;
                c.discount = key.discount;
                c.write_out = 1;
                dispatch_words_solve(max_key_words(sp), [&](auto wm) {
                    constexpr int WM = decltype(wm)::value;
                    if (disc)
                        k_cert_tail<WM, true><<<1, kTailThreads, 0, s>>>(
                            c, sp->cert_tail_meta.p, sp->keys.p, sp->params_dev.p, sp->cert_xd.p, half, t, H);
                    else
                        k_cert_tail<WM, false><<<1, kTailThreads, 0, s>>>(
                            c, sp->cert_tail_meta.p, sp->keys.p, sp->params_dev.p, sp->cert_xd.p, half, t, H);
                    VCS_LAUNCHED();
                });
                ++launches;
                if (!g.layer_ev.empty())
                    for (int u = t; u >= 0; --u)
                        if (g.layer_ev[static_cast<size_t>(u)])
                            record_event(g.layer_ev[static_cast<size_t>(u)], s, capturing);
                break;
            }
            CertLayer L = cert_layer(sp, t, sp->cert_xd.p, half, ks);
            L.d_hi = L.dense_order ? L.dense_n : 0;
            if (L.n) {
                const bool after_event = t + 1 < H && !g.layer_ev.empty() &&
                                         g.layer_ev[static_cast<size_t>(t) + 1] != nullptr;
                launch_cert_layer(sp, data, L, sp->v[0].p, sp->actions_dev.p, sp->cert_lb.p,
                                  key.discount, 1, pdl && t < H - 1 && !after_event, s);
                ++launches;
            }
            if (!g.layer_ev.empty() && g.layer_ev[static_cast<size_t>(t)])
                record_event(g.layer_ev[static_cast<size_t>(t)], s, capturing);
        }
        k_cert_check<<<1, 64, 0, s>>>(sp->cert_lb.p, H, key.eps, key.max_sweeps, sp->ctrl.p, 0);
        VCS_LAUNCHED();
        record_event(g.ev[1], s, capturing);
        record_event(g.ev[2], s, capturing);
        g.launches = launches + 1;
        g.implicit = true;
        g.fallback_at_collect = true;
        return;
    }
    // uncaptured (the first solve of a small explicit space, see enqueue_solve): the pass and
    // its certificate only; a failed certificate runs the fallback at collect
    const bool small = cert_small_ok(sp);
    if (!capturing && !small)
        raise(VCS_EINVAL, "the certified solve is only recorded into a CUDA graph");
    g.fallback_at_collect = !capturing;
    // explicit CSR: k_cert_rows, a thread per row, 4 edges in flight, 4 blocks per SM (C4:
    // 0.75 ms; a warp-cooperative form that staged q pairs in shared memory measured 0.83 ms,
    // more resident warps thrash L1)
    const void* fn = disc ? reinterpret_cast<const void*>(k_cert_rows<true, 4, 4>)
                          : reinterpret_cast<const void*>(k_cert_rows<false, 4, 4>);
    int per_sm = 0;
    VCS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, 0));
    CertArgs a{};
    a.row_ptr = sp->row_ptr.p;
    a.succ = sp->succ.p;
    a.reward = sp->reward.p;
    a.action = sp->action.p;
    a.values_out = sp->v[0].p;
    a.act_out = sp->actions_dev.p;
    a.lb = sp->cert_lb.p;
    a.discount = key.discount;
    a.write_out = 1;
    int launches = 0;
    if (small) {
        // a small space: the whole pass in one block (layer pairs in shared memory)
        if (sp->layer_off_dev.n < static_cast<size_t>(H) + 2) // (ensure_wave_buffers sets it)
            raise(VCS_EINVAL, "layer offsets were not uploaded before the capture");
        const size_t smem = cert_small_smem(H);
        int nt = kCertSmallThreads; // (VCS_CERT_SMALL_THREADS = 256 / 1024: measurements; C1
        // canonical 0.33 ms at 512 against 0.33 at 256 and 0.37 at 1024)
        if (const char* e = std::getenv("VCS_CERT_SMALL_THREADS")) nt = std::atoi(e);
        if (nt != 256 && nt != 1024) nt = 512;
        const void* fn_small =
            nt == 256 ? (disc ? reinterpret_cast<const void*>(k_cert_small<true, 256>)
                              : reinterpret_cast<const void*>(k_cert_small<false, 256>))
            : nt == 512 ? (disc ? reinterpret_cast<const void*>(k_cert_small<true, 512>)
                                : reinterpret_cast<const void*>(k_cert_small<false, 512>))
                        : (disc ? reinterpret_cast<const void*>(k_cert_small<true, 1024>)
                                : reinterpret_cast<const void*>(k_cert_small<false, 1024>));
        raise_smem_limit(fn_small, sp->device, smem);
        const uint64_t* lo_dev = sp->layer_off_dev.p;
        int h_arg = H;
        void* args[] = {&a, const_cast<uint64_t**>(&lo_dev), &h_arg};
        VCS_CUDA(cudaLaunchKernel(fn_small, dim3(1), dim3(nt), args, smem, s));
        VCS_LAUNCHED();
        launches = 1;
        // every layer is final when the one launch is: the download's piece events follow it
        for (cudaEvent_t e : g.layer_ev)
            if (e) record_event(e, s, capturing);
    }
    for (int t = launches ? -1 : H - 1; t >= 0; --t) {
        a.row0 = sp->layer_off[t];
        a.n = sp->layer_off[t + 1] - sp->layer_off[t];
        a.next_row0 = sp->layer_off[t + 1];
        a.m = H - t;
        a.xd_next = sp->cert_xd.p + a.next_row0;
        a.xd_cur = sp->cert_xd.p + a.row0;
        if (a.n) {
            const uint64_t blocks = std::max<uint64_t>(
                1, std::min<uint64_t>((a.n + 255) / 256,
                                      static_cast<uint64_t>(std::max(1, per_sm)) * sp->num_sms));
            if (disc)
                k_cert_rows<true, 4, 4><<<static_cast<unsigned>(blocks), 256, 0, s>>>(a);
            else
                k_cert_rows<false, 4, 4><<<static_cast<unsigned>(blocks), 256, 0, s>>>(a);
            VCS_LAUNCHED();
            ++launches;
        }
        if (!g.layer_ev.empty() && g.layer_ev[static_cast<size_t>(t)])
            record_event(g.layer_ev[static_cast<size_t>(t)], s, capturing);
    }
    // Profiling mode (ncu cannot profile kernels of graphs holding conditional nodes): no
    // fallback node; vcs_solve_collect raises if the proof did not hold.
    static const bool no_fallback = std::getenv("VCS_PROFILE_NO_FALLBACK") != nullptr;
    if (no_fallback || !capturing) {
        k_cert_check<<<1, 64, 0, s>>>(sp->cert_lb.p, H, key.eps, key.max_sweeps, sp->ctrl.p, 0);
        VCS_LAUNCHED();
        record_event(g.ev[1], s, capturing);
        record_event(g.ev[2], s, capturing);
        g.launches = launches + 1;
        return;
    }
    // the proof, then IF (not proven) { the full wavefront } as a conditional graph node
    cudaStreamCaptureStatus cst;
    cudaGraph_t cg = nullptr;
    VCS_CUDA(cudaStreamGetCaptureInfo(s, &cst, nullptr, &cg, nullptr, nullptr));
    if (cst != cudaStreamCaptureStatusActive || !cg) raise(VCS_ECUDA, "stream is not capturing");
    cudaGraphConditionalHandle fallback;
    VCS_CUDA(cudaGraphConditionalHandleCreate(&fallback, cg, 1, cudaGraphCondAssignDefault));
    k_cert_check<<<1, 64, 0, s>>>(sp->cert_lb.p, H, key.eps, key.max_sweeps, sp->ctrl.p, fallback);
    VCS_LAUNCHED();
    ++launches;
    const cudaGraphNode_t* deps = nullptr;
    size_t n_deps = 0;
    VCS_CUDA(cudaStreamGetCaptureInfo(s, &cst, nullptr, &cg, &deps, &n_deps));
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = fallback;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t cond = nullptr;
    VCS_CUDA(cudaGraphAddNode(&cond, cg, deps, n_deps, &cp));
    VCS_CUDA(cudaStreamUpdateCaptureDependencies(s, &cond, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    if (!sp->aux_stream)
        VCS_CUDA(cudaStreamCreateWithFlags(&sp->aux_stream, cudaStreamNonBlocking));
    VCS_CUDA(cudaStreamBeginCaptureToGraph(sp->aux_stream, body, nullptr, nullptr, 0,
                                           cudaStreamCaptureModeThreadLocal));
    const int certified_launches = launches;
    try {
        record_wavefront(sp, key, g, sp->aux_stream, true, /*events=*/false);
    } catch (...) {
        cudaGraph_t dummy = nullptr;
        cudaStreamEndCapture(sp->aux_stream, &dummy);
        throw;
    }
    cudaGraph_t body_out = nullptr;
    VCS_CUDA(cudaStreamEndCapture(sp->aux_stream, &body_out));
    unnote_launch(static_cast<uint64_t>(g.launches)); // the body's kernels were only recorded
    record_event(g.ev[1], s, capturing);
    record_event(g.ev[2], s, capturing);
    g.launches = certified_launches;
}

// Enqueue one Jacobi solve on `s`: zeroing, up to max_sweeps sweep kernels, extraction.
void record_jacobi(vcs_space* sp, const GraphKey& key, CachedGraph& g, cudaStream_t s,
                   bool capturing) {
    const bool disc = is_discounted(key.discount);
    const LaunchShape sw = shape_for(sp, disc, false);
    const LaunchShape ex = shape_for(sp, disc, true);
    SweepArgs a = base_args(sp, sp->v[0].p, sp->v[1].p, sp->delta.p, key.eps, key.discount);
    VCS_CUDA(cudaMemsetAsync(sp->v[0].p, 0, sp->S * sizeof(double), s));
    VCS_CUDA(cudaMemsetAsync(sp->delta.p, 0, (key.max_sweeps + 2) * sizeof(double), s));
    VCS_CUDA(cudaMemsetAsync(sp->ctrl.p, 0, sizeof(SolveCtrl), s));
    record_event(g.ev[0], s, capturing);
    for (int k = 1; k <= key.max_sweeps; ++k) {
        a.k = k;
        a.row_begin = 0;
        a.row_end = static_cast<uint32_t>(sweep_row_end(sp, k, key.skip != 0));
        launch_sweep(sp, a, sw, disc, s);
    }
    record_event(g.ev[1], s, capturing);
    a.k = key.max_sweeps;
    a.row_begin = 0;
    a.row_end = static_cast<uint32_t>(sp->S);
    launch_extract(sp, a, ex, disc, s);
    record_event(g.ev[2], s, capturing);
    g.launches = key.max_sweeps + 1;
}

void record_solve(vcs_space* sp, const GraphKey& key, CachedGraph& g, cudaStream_t s,
                  bool capturing) {
    if (key.method == kMethodWavefront)
        record_wavefront(sp, key, g, s, capturing);
    else if (key.method == kMethodCertified)
        record_certified(sp, key, g, s, capturing);
    else
        record_jacobi(sp, key, g, s, capturing);
}

// Layers whose completion ends a piece of vcs_solve's streamed download (row_bytes per state):
// rows are final layer by layer from the back; a piece closes once it holds >= 16 MB, the last
// one at layer 0.  Only these layers get an event (the others keep their PDL chaining).
std::vector<char> piece_layers(const vcs_space* sp, uint64_t row_bytes) {
    std::vector<char> f(static_cast<size_t>(std::max(0, sp->H)), 0);
    uint64_t chunk_end = sp->S;
    for (int t = sp->H - 1; t >= 0; --t) {
        const uint64_t r0 = sp->layer_off[static_cast<size_t>(t)];
        if ((chunk_end - r0) * row_bytes < (16ull << 20) && t > 0) continue;
        f[static_cast<size_t>(t)] = 1;
        chunk_end = r0;
    }
    return f;
}

// Launch one solve on `s`: the first solve of a (space, options) pair captures the kernel
// sequence into a CUDA graph, every solve replays it with one launch.
CachedGraph& enqueue_solve(vcs_space* sp, const GraphKey& key, cudaStream_t s) {
    auto it = sp->graphs.find(key);
    if (it == sp->graphs.end()) {
        CachedGraph g;
        g.method = key.method;
        g.n_sweeps = key.max_sweeps;
        for (auto& e : g.ev) e = acquire_event(sp->device, true);
        if (key.stream_out && (key.method == kMethodWavefront || key.method == kMethodCertified)) {
            // (stream_out = the download's bytes per state: events at its piece boundaries)
            const std::vector<char> f = piece_layers(sp, static_cast<uint64_t>(key.stream_out));
            g.layer_ev.assign(f.size(), nullptr);
            for (size_t t = 0; t < f.size(); ++t)
                if (f[t]) g.layer_ev[t] = acquire_event(sp->device, false);
        }
        it = sp->graphs.emplace(key, g).first;
    }
    CachedGraph& g = it->second;
    // The first solve of a (space, options) pair on the implicit form launches its kernels
    // directly: a one-shot solve (build -> solve -> free, the e2e path) does not pay the capture
    // and instantiation; the second solve captures the graph every later one replays.
    // (The explicit certified pass needs the graph: its fallback is a conditional node.)
    // With the streamed download too, since the download events sit only at piece boundaries
    // and PDL chains the layers between them (C4 solve + download 4.39 vs 4.48-4.57 ms through
    // the graph, C3 0.67 vs 0.87 ms; with an event after every layer and no PDL, direct
    // launches had idled the GPU).
    // Small explicit spaces (k_cert_small, one launch) too: their graph would carry the whole
    // layer wavefront as the fallback body (canonical: 330 layers, 1.9 ms to capture and
    // instantiate, more than the solve); uncaptured, the fallback runs at collect.
    const bool small_explicit = cert_small_ok(sp);
    const bool direct_ok = (sp->implicit || small_explicit) && key.method == kMethodCertified;
    if ((sp->implicit || small_explicit) && key.method == kMethodCertified &&
        (std::getenv("VCS_NO_GRAPH") || (direct_ok && g.uses == 0 && !g.exec &&
                                                      !std::getenv("VCS_GRAPH_FIRST")))) {
        record_solve(sp, key, g, s, false); // (VCS_NO_GRAPH: always direct; VCS_SYNC_CHECK works)
        ++g.uses;
        return g;
    }
    // (Measured on C4: capture + instantiate + replay of the 49-node solve costs less than
    // enqueueing it directly, whose host work between short layer kernels idles the GPU, so
    // even a one-shot solve goes through the graph.)
    if (!g.exec) {
        const double t0 = trace_enabled() ? host_ms() : 0.0;
        cudaStream_t cs = sp->stream;
        if (cs != s) VCS_CUDA(cudaStreamSynchronize(s)); // no cross-stream work pending
        VCS_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        g_capturing = true;
        try {
            record_solve(sp, key, g, cs, true);
            unnote_launch(static_cast<uint64_t>(g.launches)); // captured, not launched
            g_capturing = false;
        } catch (...) {
            g_capturing = false;
            cudaGraph_t dummy = nullptr;
            cudaStreamEndCapture(cs, &dummy);
            if (dummy) cudaGraphDestroy(dummy);
            throw;
        }
        cudaGraph_t graph = nullptr;
        VCS_CUDA(cudaStreamEndCapture(cs, &graph));
        const double t1 = trace_enabled() ? host_ms() : 0.0;
        const cudaError_t ierr = cudaGraphInstantiate(&g.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (ierr != cudaSuccess)
            raise(VCS_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ierr));
        if (trace_enabled())
            std::fprintf(stderr, "[vcs solve] capture %.3f + instantiate %.3f ms\n", t1 - t0, host_ms() - t1);
    }
    VCS_CUDA(cudaGraphLaunch(g.exec, s));
    note_launch(static_cast<uint64_t>(g.launches));
    ++g.uses;
    return g;
}

void ensure_solve_buffers(vcs_space* sp, int max_sweeps, bool sync = true) {
    const double t0 = trace_enabled() ? host_ms() : 0.0;
    sp->v[0].exact(sp->S, sp->stream);
    sp->v[1].exact(sp->S, sp->stream);
    sp->delta.exact(static_cast<size_t>(max_sweeps) + 2, sp->stream);
    sp->ctrl.exact(1, sp->stream);
    sp->actions_dev.exact(sp->S, sp->stream);
    if (sync) VCS_CUDA(cudaStreamSynchronize(sp->stream)); // pool allocations ready for any stream
    if (trace_enabled()) std::fprintf(stderr, "[vcs solve] solve buffers %.3f ms\n", host_ms() - t0);
}

// ---- version-band sharding of the wavefront (multi-GPU) ---------------------------------------
// Rank r of N owns versions [lo_t, hi_t) = [1 + r*m_t/N, 1 + (r+1)*m_t/N) of every layer t
// (m_t = H - t; floor division: balanced to one version per layer).  Since lo_{t+1} <= lo_t and
// hi_t - 1 <= hi_{t+1}, computing its band of layer t needs only its own band of layer t+1 plus
// ONE column below it (version lo_{t+1} - 1, owned by the rank below): the per-layer exchange is
// a single n_{t+1}-double column.  Storage of layer t holds versions [base_t, hi_t) with
// base_t = lo_t - 1 - pad_t; pad_t = (lo_t - lo_{t-1}) & 1 keeps the consumer's (layer t-1)
// double2 loads 16-byte aligned.

__global__ void k_band_pack(const double* __restrict__ src, uint64_t n, uint32_t stride,
                            uint32_t slot, double* __restrict__ dst) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[i * stride + slot];
}

// Receive the halo column (version lo_t - 1) of layer t, and fold in the residual of the band's
// lowest version, |V_lo - V_{lo-1}|, that the layer kernel could not compute without it.
__global__ void k_band_unpack(double* __restrict__ store, uint64_t n, uint32_t stride,
                              uint32_t slot, const double* __restrict__ src, int has_low,
                              double* __restrict__ delta_lo) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    double d = 0.0;
    if (i < n) {
        const double h = src[i];
        store[i * stride + slot] = h;
        if (has_low) d = fabs(store[i * stride + slot + 1] - h);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double other = __shfl_xor_sync(0xffffffffu, d, o);
        d = d < other ? other : d;
    }
    if ((threadIdx.x & 31) == 0 && d > 0.0)
        atomicMax(reinterpret_cast<unsigned long long*>(delta_lo),
                  static_cast<unsigned long long>(__double_as_longlong(d)));
}

// Early-stop fix-up of layer t (t < H - K): V_K(s) on the rank owning version K of layer t
// (ver_t != nullptr), the argmax against V_K of the successors on the rank owning version K of
// layer t+1 (ver_n != nullptr).
template <bool DISC>
__global__ void k_band_fixup(const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ succ,
                             const double* __restrict__ reward, const int32_t* __restrict__ action,
                             const double* __restrict__ ver_t, uint32_t stride_t, uint32_t slot_t,
                             const double* __restrict__ ver_n, uint32_t stride_n, uint32_t slot_n,
                             uint64_t row0, uint64_t n, uint64_t next_row0, double discount,
                             double* __restrict__ values_out, int32_t* __restrict__ act_out) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t s = row0 + i;
    if (ver_t) values_out[s] = ver_t[i * stride_t + slot_t];
    if (!ver_n) return;
    double best = -INFINITY;
    int32_t act = -1;
    for (uint32_t e = row_ptr[s]; e < row_ptr[s + 1]; ++e) {
        const double v = ver_n[(succ[e] - next_row0) * stride_n + slot_n];
        const double q = DISC ? __dadd_rn(reward[e], __dmul_rn(discount, v)) : __dadd_rn(reward[e], v);
        if (q > best) {
            best = q;
            act = action[e];
        }
    }
    act_out[s] = act;
}

void band_plan(vcs_space* sp, int world, int rank) {
    const int H = sp->H;
    sp->band_lo.assign(static_cast<size_t>(H) + 1, 1);
    sp->band_hi.assign(static_cast<size_t>(H) + 1, 1);
    sp->band_base.assign(static_cast<size_t>(H) + 1, 0);
    sp->band_stride.assign(static_cast<size_t>(H) + 1, 2);
    sp->band_off.assign(static_cast<size_t>(H) + 2, 0);
    for (int t = 0; t <= H; ++t) {
        const long m = H - t;
        sp->band_lo[t] = static_cast<int>(1 + rank * m / world);
        sp->band_hi[t] = static_cast<int>(1 + (rank + 1) * m / world);
    }
    uint64_t off = 0;
    for (int t = 0; t <= H; ++t) {
        const int pad = t == 0 ? 0 : ((sp->band_lo[t] - sp->band_lo[t - 1]) & 1);
        sp->band_base[t] = sp->band_lo[t] - 1 - pad;
        const int width = sp->band_hi[t] - sp->band_base[t];
        sp->band_stride[t] = (width + 2 + 1) & ~1; // consumer pairs may read one version past hi
        sp->band_off[t] = off;
        off += (sp->layer_off[t + 1] - sp->layer_off[t]) * static_cast<uint64_t>(sp->band_stride[t]);
    }
    sp->band_off[static_cast<size_t>(H) + 1] = off;
}

} // namespace

// ---- multi-GPU certified pass (replaces the block-parallel driver of
// parallel_vi.cpp:68-107 for n GPUs of this process) ----------------------------------------------
//
// ONE state space, n ranks (GPUs; a device may repeat, which runs several ranks on one GPU —
// the emulated-rank test mode).  Layer t of the backward pass is split into contiguous ranges of
// its pair index space: the key space (implicit form, dense-order layers) or the BFS rows
// (explicit CSR).  Small and sparse layers are computed whole by every rank (replicated: no
// exchange).  After a split layer t, rank h pulls from each owner q the part of q's range that
// h's layer t-1 reads:
//   * key space, non-retiring transition: a successor index is d - demand*W_p <= d, so rank h
//     with layer-(t-1) range [lo, hi) reads [lo - demand*max_p W_p, hi): a forward halo from
//     the ranks below it;
//   * anything else (retiring transition, explicit CSR, replicated consumer): the whole layer
//     (an all-gather).
// The pulls are peer copies (cudaMemcpyPeerAsync over NVLink) on the puller's stream after the
// owner's layer event; a rank rewrites a pair half two layers later only after every puller's
// copy event (write-after-read).  Values and actions are stored by every rank's kernel straight
// into the primary GPU's result arrays (peer stores).  Each rank's residual lower bounds are
// gathered to the primary, max-reduced and checked there (k_cert_check_multi).  No kernel waits
// on another: all ordering is by stream events, so the same code runs with every rank on one GPU.
// The whole pass is captured into one CUDA graph (one launch per solve).

struct MultiRank {
    int device = 0;
    bool shared = false; // on the primary GPU: reads the space's own buffers
    cudaStream_t stream = nullptr;
    // replicas of the space's read-only data on this rank's GPU (unused when `shared`)
    uint64_t* keys = nullptr;
    uint32_t* rank_tables = nullptr;
    LayerParam* params = nullptr;
    uint32_t* row_ptr = nullptr;
    uint32_t* succ = nullptr;
    double* reward = nullptr;
    int32_t* action = nullptr;
    double2* xd = nullptr; // this rank's pair buffer (key space: two halves; explicit: S pairs)
    double* lb = nullptr;  // H+2 residual lower bounds
    std::vector<cudaEvent_t> ev_layer, ev_copy; // per layer t
    cudaEvent_t ev_done = nullptr;
    std::vector<std::pair<int, void*>> owned; // (device, pointer) allocations
};

struct MultiState {
    std::vector<int> devices;
    int exchange = 0;
    int primary = 0;
    bool keyspace = false;
    uint64_t half = 0;
    std::vector<MultiRank> ranks;
    // plan per layer t (0..H-1): split or replicated, the ranks' ranges and needed windows
    std::vector<char> split;
    std::vector<std::vector<uint64_t>> lo, hi, need_lo, need_hi;
    double* lb_stage = nullptr;
    cudaEvent_t ev_fork = nullptr;
    std::map<GraphKey, CachedGraph> graphs;
    bool no_graph = false;
    double halo_bytes = 0.0;   // pair bytes pulled between ranks per solve
    int split_layers = 0, replicated_layers = 0;
    double max_share = 0.0;    // largest rank share of the split work (1/n = balanced)
};

// One rank of the multi-PROCESS form of the same pass (vcs_cert_shard_*): this process owns one
// rank's GPU; the caller moves the windows between processes (torch.distributed / NCCL).
struct CertShard {
    int world = 1, rank = 0, exchange = 0;
    bool keyspace = false;
    uint64_t half = 0;
    double eps = 1e-6, discount = 1.0;
    int max_sweeps = 0;
    std::vector<char> split;
    std::vector<std::vector<uint64_t>> lo, hi, need_lo, need_hi;
    double halo_bytes = 0.0;
    int split_layers = 0, replicated_layers = 0;
    double max_share = 0.0;
    DevBuf<double2> xd;
    DevBuf<double> lb;
};

namespace {

void* multi_alloc(MultiRank& r, size_t bytes) {
    VCS_CUDA(cudaSetDevice(r.device));
    void* p = nullptr;
    VCS_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    r.owned.emplace_back(r.device, p);
    return p;
}

template <class T>
T* replica(MultiRank& r, const DevBuf<T>& src, size_t n, int src_dev) {
    if (!src.p || n == 0) return nullptr;
    T* p = static_cast<T*>(multi_alloc(r, n * sizeof(T)));
    VCS_CUDA(cudaMemcpyPeer(p, r.device, src.p, src_dev, n * sizeof(T)));
    return p;
}

// The largest successor weight of an eligible cloud of transition t-1 -> t when nothing retires
// and the successor numbering equals the state numbering (then succ = d - demand*W_p); 0 = no
// such bound (the consumer reads the whole layer).
int64_t halo_shift(const vcs_space* sp, int t_consumer) {
    const LayerParam& P = sp->plan.layers[static_cast<size_t>(t_consumer)];
    if (P.n_keep != P.n_active || P.dense_size == 0 || P.self_size != P.dense_size) return -1;
    uint64_t wmax = 0;
    for (int p = 0; p < P.n_active; ++p) {
        if (P.keep_idx[p] != p || P.wnext[p] != P.wself[p]) return -1;
        if (P.attr[p]) wmax = std::max<uint64_t>(wmax, P.wnext[p]);
    }
    return static_cast<int64_t>(static_cast<uint64_t>(P.demand) * wmax);
}

// The split of every layer between n ranks and the windows their next layers read (fills the
// plan fields shared by MultiState and CertShard).
template <class P>
void multi_plan(const vcs_space* sp, int n, P& ms) {
    const int H = sp->H;
    uint64_t min_split = 65536;
    if (const char* e = std::getenv("VCS_MULTI_MIN_SPLIT")) min_split = std::strtoull(e, nullptr, 10);
    ms.split.assign(static_cast<size_t>(H), 0);
    ms.lo.assign(static_cast<size_t>(H), std::vector<uint64_t>(static_cast<size_t>(n), 0));
    ms.hi = ms.need_lo = ms.need_hi = ms.lo;
    std::vector<uint64_t> size(static_cast<size_t>(H), 0);
    ms.split_layers = ms.replicated_layers = 0;
    double split_work = 0.0, max_rank_work = 0.0;
    std::vector<double> rank_work(static_cast<size_t>(n), 0.0);
    for (int t = 0; t < H; ++t) {
        const CertLayer L = cert_layer(sp, t, nullptr, ms.half, ms.keyspace);
        bool split = false;
        uint64_t sz = 0;
        if (ms.keyspace) {
            sz = L.dense_order ? L.dense_n : L.n;
            split = L.dense_order && sz >= min_split && n > 1;
        } else {
            sz = L.n;
            split = sz >= min_split && n > 1;
        }
        size[static_cast<size_t>(t)] = sz;
        ms.split[static_cast<size_t>(t)] = split ? 1 : 0;
        for (int r = 0; r < n; ++r) {
            ms.lo[t][r] = split ? sz * static_cast<uint64_t>(r) / static_cast<uint64_t>(n) : 0;
            ms.hi[t][r] = split ? sz * static_cast<uint64_t>(r + 1) / static_cast<uint64_t>(n) : sz;
            if (split) rank_work[static_cast<size_t>(r)] += static_cast<double>(ms.hi[t][r] - ms.lo[t][r]);
        }
        if (split) {
            ++ms.split_layers;
            split_work += static_cast<double>(sz);
        } else {
            ++ms.replicated_layers;
        }
    }
    for (double w : rank_work) max_rank_work = std::max(max_rank_work, w);
    ms.max_share = split_work > 0 ? max_rank_work / split_work : 1.0;
    // the window of layer t's pairs each rank's layer t-1 reads
    ms.halo_bytes = 0.0;
    for (int t = 1; t < H; ++t) {
        if (!ms.split[static_cast<size_t>(t)]) continue;
        const uint64_t D = size[static_cast<size_t>(t)];
        const bool consumer_split = ms.split[static_cast<size_t>(t - 1)] != 0;
        const int64_t shift = (ms.keyspace && consumer_split && ms.exchange == VCS_EXCHANGE_HALO)
                                  ? halo_shift(sp, t - 1) : -1;
        for (int h = 0; h < n; ++h) {
            uint64_t a = 0, b = D;
            if (shift >= 0) {
                const uint64_t clo = ms.lo[t - 1][h], chi = ms.hi[t - 1][h];
                a = clo > static_cast<uint64_t>(shift) ? clo - static_cast<uint64_t>(shift) : 0;
                b = std::min(D, chi);
                if (chi <= clo) a = b = 0; // no layer t-1 work: nothing needed
            }
            ms.need_lo[t][h] = a;
            ms.need_hi[t][h] = b;
            for (int q = 0; q < n; ++q) {
                if (q == h) continue;
                const uint64_t x = std::max(a, ms.lo[t][q]), y = std::min(b, ms.hi[t][q]);
                if (x < y) ms.halo_bytes += 16.0 * static_cast<double>(y - x);
            }
        }
    }
}

void destroy_rank(MultiRank& r) {
    cudaSetDevice(r.device);
    if (r.stream) cudaStreamSynchronize(r.stream);
    for (auto e : r.ev_layer)
        if (e) cudaEventDestroy(e);
    for (auto e : r.ev_copy)
        if (e) cudaEventDestroy(e);
    if (r.ev_done) cudaEventDestroy(r.ev_done);
    for (auto& [dev, p] : r.owned) {
        cudaSetDevice(dev);
        cudaFree(p);
    }
    r.owned.clear();
    if (r.stream) {
        cudaSetDevice(r.device);
        cudaStreamDestroy(r.stream);
    }
    r.stream = nullptr;
}

// Set up (or reuse) the per-rank state for `devices`.
MultiState& multi_state(vcs_space* sp, const std::vector<int>& devices, int exchange) {
    if (sp->multi && (sp->multi->devices != devices || sp->multi->exchange != exchange)) {
        destroy_multi(sp->multi);
        sp->multi = nullptr;
    }
    if (sp->multi) return *sp->multi;
    auto ms = std::make_unique<MultiState>();
    ms->devices = devices;
    ms->exchange = exchange;
    ms->primary = sp->device;
    ms->keyspace = cert_keyspace(sp);
    if (sp->implicit && !ms->keyspace)
        raise(VCS_EINVAL, "the multi-GPU certified pass needs key-space pairs (unset VCS_CERT_BFS)");
    if (!sp->implicit) ensure_csr(sp);
    ms->half = ms->keyspace ? cert_half(sp) : 0;
    const int H = sp->H;
    const size_t xd_n = ms->keyspace ? 2 * ms->half : sp->S;
    ms->ranks.resize(devices.size());
    try {
        for (size_t i = 0; i < devices.size(); ++i) {
            MultiRank& r = ms->ranks[i];
            r.device = devices[i];
            r.shared = r.device == sp->device;
            VCS_CUDA(cudaSetDevice(r.device));
            VCS_CUDA(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking));
            if (!r.shared) {
                if (sp->implicit) {
                    r.keys = replica(r, sp->keys, sp->key_off.back(), sp->device);
                    r.rank_tables = replica(r, sp->rank_tables, sp->rank_off.back(), sp->device);
                    r.params = replica(r, sp->params_dev, static_cast<size_t>(H), sp->device);
                } else {
                    r.row_ptr = replica(r, sp->row_ptr, sp->S + 1, sp->device);
                    r.succ = replica(r, sp->succ, sp->E, sp->device);
                    r.reward = replica(r, sp->reward, sp->E, sp->device);
                    r.action = replica(r, sp->action, sp->E, sp->device);
                }
            }
            r.xd = static_cast<double2*>(multi_alloc(r, xd_n * sizeof(double2)));
            r.lb = static_cast<double*>(multi_alloc(r, (static_cast<size_t>(H) + 2) * sizeof(double)));
            VCS_CUDA(cudaSetDevice(r.device));
            r.ev_layer.assign(static_cast<size_t>(std::max(H, 1)), nullptr);
            r.ev_copy.assign(static_cast<size_t>(std::max(H, 1)), nullptr);
            for (auto& e : r.ev_layer) VCS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            for (auto& e : r.ev_copy) VCS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            VCS_CUDA(cudaEventCreateWithFlags(&r.ev_done, cudaEventDisableTiming));
        }
        // NVLink peer access between every pair of distinct GPUs (peer stores into the
        // primary's results, halo copies between ranks)
        {
            std::vector<int> uniq(devices.begin(), devices.end());
            uniq.push_back(sp->device);
            std::sort(uniq.begin(), uniq.end());
            uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
            for (int a : uniq)
                for (int b : uniq) {
                    if (a == b) continue;
                    int can = 0;
                    VCS_CUDA(cudaDeviceCanAccessPeer(&can, a, b));
                    if (!can)
                        raise(VCS_ECUDA, "GPU " + std::to_string(a) + " cannot access GPU " +
                                             std::to_string(b) + " (no peer path)");
                    VCS_CUDA(cudaSetDevice(a));
                    const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
                    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                        raise(VCS_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
                    cudaGetLastError();
                }
        }
        { // the ranks' lower bounds, gathered on the primary
            VCS_CUDA(cudaSetDevice(sp->device));
            void* p = nullptr;
            VCS_CUDA(cudaMalloc(&p, devices.size() * (static_cast<size_t>(H) + 2) * sizeof(double)));
            ms->ranks[0].owned.emplace_back(sp->device, p);
            ms->lb_stage = static_cast<double*>(p);
        }
        VCS_CUDA(cudaEventCreateWithFlags(&ms->ev_fork, cudaEventDisableTiming));
        multi_plan(sp, static_cast<int>(ms->ranks.size()), *ms);
    } catch (...) {
        destroy_multi(ms.release());
        VCS_CUDA(cudaSetDevice(sp->device));
        throw;
    }
    sp->multi = ms.release();
    return *sp->multi;
}

// lb[k] = max over ranks, then the certificate test of k_cert_check.
__global__ void k_cert_check_multi(const double* __restrict__ lb_stage, int n_ranks, int H,
                                   double eps, int max_sweeps, double* lb_out, SolveCtrl* ctrl) {
    __shared__ int bad;
    if (threadIdx.x == 0) bad = max_sweeps < H + 1 ? 1 : 0;
    __syncthreads();
    for (int k = 1 + threadIdx.x; k <= H; k += blockDim.x) {
        double m = 0.0;
        for (int r = 0; r < n_ranks; ++r) m = fmax(m, lb_stage[static_cast<size_t>(r) * (H + 2) + k]);
        lb_out[k] = m;
        if (!(m >= eps)) bad = 1;
    }
    __syncthreads();
    if (threadIdx.x == 0 && !bad) {
        ctrl->sweeps = H + 1;
        ctrl->stop = 1;
        ctrl->certified = 1;
    }
}

// Enqueue (or record into a capture on `s`) one multi-GPU certified solve.
void record_multi(vcs_space* sp, MultiState& ms, const GraphKey& key, CachedGraph& g,
                  cudaStream_t s, bool capturing) {
    const int H = sp->H, n = static_cast<int>(ms.ranks.size());
    const bool ks = ms.keyspace;
    int launches = 0;
    VCS_CUDA(cudaSetDevice(sp->device));
    VCS_CUDA(cudaMemsetAsync(sp->ctrl.p, 0, sizeof(SolveCtrl), s));
    const uint64_t rH = sp->layer_off[H], nH = sp->S - rH;
    VCS_CUDA(cudaMemsetAsync(sp->v[0].p + rH, 0, nH * sizeof(double), s));
    VCS_CUDA(cudaMemsetAsync(sp->actions_dev.p + rH, 0xff, nH * sizeof(int32_t), s));
    record_event(g.ev[0], s, capturing);
    VCS_CUDA(cudaEventRecord(ms.ev_fork, s));
    for (auto& r : ms.ranks) {
        VCS_CUDA(cudaSetDevice(r.device));
        VCS_CUDA(cudaStreamWaitEvent(r.stream, ms.ev_fork, 0));
        VCS_CUDA(cudaMemsetAsync(r.lb, 0, (H + 2) * sizeof(double), r.stream));
        if (ks)
            VCS_CUDA(cudaMemsetAsync(r.xd + (H & 1) * ms.half, 0, sizeof(double2), r.stream));
        else
            VCS_CUDA(cudaMemsetAsync(r.xd + rH, 0, nH * sizeof(double2), r.stream));
    }
    // readers[t][q]: ranks that pulled from rank q's layer-t pairs (write-after-read)
    std::vector<std::vector<std::vector<int>>> readers(
        static_cast<size_t>(H) + 2, std::vector<std::vector<int>>(static_cast<size_t>(n)));
    for (int t = H - 1; t >= 0; --t) {
        const bool split = ms.split[static_cast<size_t>(t)] != 0;
        for (int ri = 0; ri < n; ++ri) {
            MultiRank& r = ms.ranks[static_cast<size_t>(ri)];
            VCS_CUDA(cudaSetDevice(r.device));
            // this layer rewrites the pair half of layer t+2: wait for its pullers' copies
            if (t + 2 <= H - 1)
                for (int h : readers[static_cast<size_t>(t + 2)][static_cast<size_t>(ri)])
                    VCS_CUDA(cudaStreamWaitEvent(r.stream, ms.ranks[static_cast<size_t>(h)].ev_copy[static_cast<size_t>(t + 2)], 0));
            CertData data = r.shared ? cert_data_of(sp)
                                     : CertData{r.keys, r.rank_tables, r.params};
            const uint64_t lo = ms.lo[t][ri], hi = ms.hi[t][ri];
            if (ks) {
                CertLayer L = cert_layer(sp, t, r.xd, ms.half, true);
                if (L.dense_order) {
                    L.d_lo = lo;
                    L.d_hi = hi;
                }
                if (L.n && (!L.dense_order || hi > lo)) {
                    launch_cert_layer(sp, data, L, sp->v[0].p, sp->actions_dev.p, r.lb, key.discount,
                                      (split || ri == 0) ? 1 : 0, false, r.stream);
                    ++launches;
                }
            } else if (hi > lo) {
                CertArgs a{};
                a.row_ptr = r.shared ? sp->row_ptr.p : r.row_ptr;
                a.succ = r.shared ? sp->succ.p : r.succ;
                a.reward = r.shared ? sp->reward.p : r.reward;
                a.action = r.shared ? sp->action.p : r.action;
                a.values_out = sp->v[0].p;
                a.act_out = sp->actions_dev.p;
                a.write_out = (split || ri == 0) ? 1 : 0;
                a.lb = r.lb;
                a.discount = key.discount;
                a.row0 = sp->layer_off[t] + lo;
                a.n = hi - lo;
                a.next_row0 = sp->layer_off[t + 1];
                a.m = H - t;
                a.xd_next = r.xd + a.next_row0;
                a.xd_cur = r.xd + a.row0;
                const bool disc = is_discounted(key.discount);
                const unsigned blocks = static_cast<unsigned>(std::max<uint64_t>(
                    1, std::min<uint64_t>((a.n + 255) / 256, static_cast<uint64_t>(4) * sp->num_sms)));
                if (disc) k_cert_rows<true, 4, 4><<<blocks, 256, 0, r.stream>>>(a);
                else k_cert_rows<false, 4, 4><<<blocks, 256, 0, r.stream>>>(a);
                VCS_LAUNCHED();
                ++launches;
            }
            VCS_CUDA(cudaEventRecord(r.ev_layer[static_cast<size_t>(t)], r.stream));
        }
        if (!split || t == 0) continue;
        // pulls: rank h copies from owner q the part of q's range its layer t-1 reads
        const uint64_t base = ks ? (t & 1) * ms.half : sp->layer_off[t];
        for (int h = 0; h < n; ++h) {
            MultiRank& dst = ms.ranks[static_cast<size_t>(h)];
            VCS_CUDA(cudaSetDevice(dst.device));
            for (int q = 0; q < n; ++q) {
                if (q == h) continue;
                const uint64_t x = std::max(ms.need_lo[t][h], ms.lo[t][q]);
                const uint64_t y = std::min(ms.need_hi[t][h], ms.hi[t][q]);
                if (x >= y) continue;
                MultiRank& src = ms.ranks[static_cast<size_t>(q)];
                VCS_CUDA(cudaStreamWaitEvent(dst.stream, src.ev_layer[static_cast<size_t>(t)], 0));
                // (UVA copy: capturable, peer-to-peer over NVLink between the two GPUs)
                VCS_CUDA(cudaMemcpyAsync(dst.xd + base + x, src.xd + base + x,
                                         (y - x) * sizeof(double2), cudaMemcpyDefault, dst.stream));
                readers[static_cast<size_t>(t)][static_cast<size_t>(q)].push_back(h);
            }
            VCS_CUDA(cudaEventRecord(dst.ev_copy[static_cast<size_t>(t)], dst.stream));
        }
    }
    // every rank's lower bounds to the primary; join
    for (int ri = 0; ri < n; ++ri) {
        MultiRank& r = ms.ranks[static_cast<size_t>(ri)];
        VCS_CUDA(cudaSetDevice(r.device));
        VCS_CUDA(cudaMemcpyAsync(ms.lb_stage + static_cast<size_t>(ri) * (H + 2), r.lb,
                                 (H + 2) * sizeof(double), cudaMemcpyDefault, r.stream));
        VCS_CUDA(cudaEventRecord(r.ev_done, r.stream));
    }
    VCS_CUDA(cudaSetDevice(sp->device));
    for (auto& r : ms.ranks) VCS_CUDA(cudaStreamWaitEvent(s, r.ev_done, 0));
    k_cert_check_multi<<<1, 64, 0, s>>>(ms.lb_stage, n, H, key.eps, key.max_sweeps, sp->cert_lb.p,
                                        sp->ctrl.p);
    VCS_LAUNCHED();
    record_event(g.ev[1], s, capturing);
    record_event(g.ev[2], s, capturing);
    g.launches = launches + 1;
}

} // namespace

void destroy_cert_shard(CertShard* cs) {
    if (!cs) return;
    cs->xd.release();
    cs->lb.release();
    delete cs;
}

void destroy_multi(MultiState* ms) {
    if (!ms) return;
    for (auto& r : ms->ranks) destroy_rank(r);
    for (auto& [k, g] : ms->graphs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        for (auto& e : g.ev)
            if (e) cudaEventDestroy(e);
    }
    if (ms->ev_fork) cudaEventDestroy(ms->ev_fork);
    delete ms;
}

namespace {
// Enqueue one multi-GPU certified solve on `s` (the primary's stream): captured into a graph on
// first use, replayed afterwards.
CachedGraph& enqueue_multi(vcs_space* sp, MultiState& ms, const GraphKey& key, cudaStream_t s) {
    auto it = ms.graphs.find(key);
    if (it == ms.graphs.end()) {
        CachedGraph g;
        g.method = kMethodCertified;
        g.n_sweeps = key.max_sweeps;
        for (auto& e : g.ev) VCS_CUDA(cudaEventCreate(&e));
        it = ms.graphs.emplace(key, g).first;
    }
    CachedGraph& g = it->second;
    g.implicit = sp->implicit;
    g.fallback_at_collect = true;
    g.n_ranks = static_cast<int>(ms.ranks.size());
    // the first solve of a space launches directly (a one-shot solve does not pay the capture
    // and instantiation of the multi-device graph); the second captures it
    if (!g.exec && !ms.no_graph && !std::getenv("VCS_NO_GRAPH") &&
        (g.uses > 0 || std::getenv("VCS_GRAPH_FIRST"))) {
        cudaStream_t cs = sp->stream;
        if (cs != s) VCS_CUDA(cudaStreamSynchronize(s));
        VCS_CUDA(cudaSetDevice(sp->device));
        VCS_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        g_capturing = true;
        cudaGraph_t graph = nullptr;
        try {
            record_multi(sp, ms, key, g, cs, true);
            unnote_launch(static_cast<uint64_t>(g.launches));
            g_capturing = false;
            VCS_CUDA(cudaSetDevice(sp->device));
            VCS_CUDA(cudaStreamEndCapture(cs, &graph));
        } catch (const Error& e) {
            g_capturing = false;
            cudaSetDevice(sp->device);
            cudaGraph_t dummy = nullptr;
            cudaStreamEndCapture(cs, &dummy);
            if (dummy) cudaGraphDestroy(dummy);
            cudaGetLastError();
            if (std::getenv("VCS_TRACE")) std::fprintf(stderr, "[vcs multi] capture: %s\n", e.msg.c_str());
            ms.no_graph = true; // this driver / topology cannot capture it: direct launches
        }
        if (graph) {
            const cudaError_t ierr = cudaGraphInstantiate(&g.exec, graph, 0);
            cudaGraphDestroy(graph);
            if (ierr != cudaSuccess) {
                if (std::getenv("VCS_TRACE"))
                    std::fprintf(stderr, "[vcs multi] instantiate: %s\n", cudaGetErrorString(ierr));
                cudaGetLastError();
                g.exec = nullptr;
                ms.no_graph = true;
            }
        }
    }
    VCS_CUDA(cudaSetDevice(sp->device));
    if (g.exec) {
        VCS_CUDA(cudaGraphLaunch(g.exec, s));
        note_launch(static_cast<uint64_t>(g.launches));
    } else {
        record_multi(sp, ms, key, g, s, false);
        VCS_CUDA(cudaSetDevice(sp->device));
    }
    ++g.uses;
    return g;
}
} // namespace

} // namespace vcs

using vcs::guarded;
using vcs::raise;

extern "C" {

namespace {
int enqueue_impl(vcs_space* sp, const vcs_solve_opts* opts, void* stream, int stream_out) {
    return guarded([&] {
        vcs_solve_opts o{1e-6, 1, 0, 1.0, VCS_METHOD_AUTO};
        if (opts) o = *opts;
        if (!(o.epsilon > 0.0))
            raise(VCS_EINVAL, "epsilon must be > 0 (value iteration would never terminate)");
        if (o.method < VCS_METHOD_AUTO || o.method > VCS_METHOD_CERTIFIED)
            raise(VCS_EINVAL, "unknown solve method");
        vcs::bind_device(sp->device);
        int M = sp->H + 1; // delta_{H+1} == 0 on the layered DAG, so this is never binding
        if (o.max_sweeps > 0) M = std::min(M, o.max_sweeps);
        const double t0 = vcs::trace_enabled() ? vcs::host_ms() : 0.0;
        // (no host synchronisation per buffer: the solve's stream is ordered behind the space's
        // stream once, below)
        vcs::ensure_solve_buffers(sp, sp->H + 1, false); // fixed size: cached graphs keep addresses
        int method = o.method;
        if (method == VCS_METHOD_AUTO) // implicit spaces: the fallback's buffers come at collect
            method = sp->implicit || vcs::wavefront_fits(sp) ? VCS_METHOD_CERTIFIED
                                                             : VCS_METHOD_JACOBI;
        // Jacobi and the wavefront read the explicit CSR
        if (method == VCS_METHOD_JACOBI || method == VCS_METHOD_WAVEFRONT) vcs::ensure_csr(sp);
        // (the explicit certified solve keeps the wavefront as its in-graph fallback)
        if ((method == VCS_METHOD_WAVEFRONT || (method == VCS_METHOD_CERTIFIED && !sp->implicit)) &&
            sp->ver_off_host.empty()) {
            try {
                vcs::ensure_wave_buffers(sp, false);
            } catch (const vcs::Error&) {
                if (o.method != VCS_METHOD_AUTO) throw;
                cudaGetLastError();
                method = VCS_METHOD_JACOBI; // the version store does not fit right now
            }
        }
        if (method == VCS_METHOD_CERTIFIED && vcs::cert_permute_space(sp) &&
            sp->cert_act_ks.n < vcs::cert_half(sp)) {
            sp->cert_act_ks.exact(vcs::cert_half(sp), sp->stream);
        }
        if (method == VCS_METHOD_CERTIFIED && sp->cert_xd.n < vcs::cert_pairs_needed(sp)) {
            sp->cert_xd.exact(vcs::cert_pairs_needed(sp), sp->stream);
            sp->cert_lb.exact(static_cast<size_t>(sp->H) + 2, sp->stream);
        }
        if (method == VCS_METHOD_CERTIFIED && sp->implicit && vcs::cert_stream_space(sp))
            vcs::ensure_stream_plan(sp);
        if (method == VCS_METHOD_CERTIFIED && sp->implicit) vcs::ensure_cert_tail(sp);
        if (vcs::trace_enabled())
            std::fprintf(stderr, "[vcs solve] buffers %.3f ms\n", vcs::host_ms() - t0);
        const vcs::GraphKey key{o.epsilon, o.discount,
                                method == VCS_METHOD_JACOBI && o.skip_converged ? 1 : 0, M,
                                method, method != VCS_METHOD_JACOBI ? stream_out : 0};
        static const bool timeline = std::getenv("VCS_CERT_TIMELINE") != nullptr;
        if (timeline && method == VCS_METHOD_CERTIFIED) {
            const size_t n_tl = 3 * (static_cast<size_t>(sp->H) + 2);
            if (sp->cert_tl.n < n_tl) sp->cert_tl.exact(n_tl, sp->stream);
            VCS_CUDA(cudaMemsetAsync(sp->cert_tl.p, 0xff, n_tl * sizeof(unsigned long long), sp->stream));
        }
        const vcs::StreamUse s(sp, stream);
        if (static_cast<cudaStream_t>(s) != sp->stream) { // the buffers above, then the solve
            if (!sp->order_ev) sp->order_ev = vcs::acquire_event(sp->device, false);
            VCS_CUDA(cudaEventRecord(sp->order_ev, sp->stream));
            VCS_CUDA(cudaStreamWaitEvent(s, sp->order_ev, 0));
        }
        auto& g = vcs::enqueue_solve(sp, key, s);
        sp->last_graph = &g;
        sp->last_key_skip = key.skip;
        sp->last_opts = o;
        return VCS_OK;
    });
}
} // namespace

int vcs_solve_enqueue(vcs_space* sp, const vcs_solve_opts* opts, void* stream) {
    std::lock_guard<std::recursive_mutex> space_lock(sp->mu);
    return enqueue_impl(sp, opts, stream, 0);
}

int vcs_solve_multi_enqueue(vcs_space* sp, const vcs_solve_opts* opts, int32_t n_ranks,
                            const int32_t* devices, int32_t exchange, void* stream) {
    std::lock_guard<std::recursive_mutex> space_lock(sp->mu);
    if (n_ranks == 1 && (!devices || devices[0] == sp->device))
        return enqueue_impl(sp, opts, stream, 0);
    return guarded([&] {
        vcs_solve_opts o{1e-6, 1, 0, 1.0, VCS_METHOD_AUTO};
        if (opts) o = *opts;
        if (!(o.epsilon > 0.0))
            raise(VCS_EINVAL, "epsilon must be > 0 (value iteration would never terminate)");
        if (o.method != VCS_METHOD_AUTO && o.method != VCS_METHOD_CERTIFIED)
            raise(VCS_EINVAL, "the multi-GPU solve runs the certified pass (method AUTO or CERTIFIED)");
        if (n_ranks < 1) raise(VCS_EINVAL, "n_gpus must be >= 1");
        if (exchange != VCS_EXCHANGE_HALO && exchange != VCS_EXCHANGE_ALLGATHER)
            raise(VCS_EINVAL, "unknown exchange mode");
        int n_dev = 0;
        VCS_CUDA(cudaGetDeviceCount(&n_dev));
        std::vector<int> devs(static_cast<size_t>(n_ranks));
        for (int r = 0; r < n_ranks; ++r) {
            devs[static_cast<size_t>(r)] = devices ? devices[r] : (sp->device + r) % n_dev;
            if (devs[static_cast<size_t>(r)] < 0 || devs[static_cast<size_t>(r)] >= n_dev)
                raise(VCS_EINVAL, "device index out of range");
        }
        vcs::bind_device(sp->device);
        int M = sp->H + 1;
        if (o.max_sweeps > 0) M = std::min(M, o.max_sweeps);
        vcs::ensure_solve_buffers(sp, sp->H + 1);
        if (sp->cert_lb.n < static_cast<size_t>(sp->H) + 2) {
            sp->cert_lb.exact(static_cast<size_t>(sp->H) + 2, sp->stream);
            VCS_CUDA(cudaStreamSynchronize(sp->stream));
        }
        vcs::MultiState& ms = vcs::multi_state(sp, devs, exchange);
        const vcs::GraphKey key{o.epsilon, o.discount, 0, M, vcs::kMethodCertified, 0};
        const vcs::StreamUse s(sp, stream);
        auto& g = vcs::enqueue_multi(sp, ms, key, s);
        vcs::bind_device(sp->device);
        sp->last_graph = &g;
        sp->last_key_skip = 0;
        sp->last_opts = o;
        sp->last_opts.method = VCS_METHOD_CERTIFIED;
        return VCS_OK;
    });
}

int vcs_solve_multi(vcs_space* sp, const vcs_solve_opts* opts, int32_t n_ranks,
                    const int32_t* devices, int32_t exchange, double* values_out,
                    int32_t* actions_out, vcs_solve_report* report) {
    std::lock_guard<std::recursive_mutex> space_lock(sp->mu);
    const int rc = vcs_solve_multi_enqueue(sp, opts, n_ranks, devices, exchange, nullptr);
    if (rc != VCS_OK) return rc;
    return vcs_solve_collect(sp, values_out, actions_out, report, nullptr);
}

// ---- multi-process form: one rank per process (vcs_cert_shard_*) -------------------------------

int vcs_cert_shard_begin(vcs_space* sp, const vcs_solve_opts* opts, int32_t world, int32_t rank,
                         int32_t exchange, void* stream) {
    std::lock_guard<std::recursive_mutex> space_lock(sp->mu);
    return guarded([&] {
        vcs_solve_opts o{1e-6, 1, 0, 1.0, VCS_METHOD_AUTO};
        if (opts) o = *opts;
        if (!(o.epsilon > 0.0))
            raise(VCS_EINVAL, "epsilon must be > 0 (value iteration would never terminate)");
        if (world < 1 || rank < 0 || rank >= world) raise(VCS_EINVAL, "bad world/rank");
        if (exchange != VCS_EXCHANGE_HALO && exchange != VCS_EXCHANGE_ALLGATHER)
            raise(VCS_EINVAL, "unknown exchange mode");
        vcs::bind_device(sp->device);
        const bool ks = vcs::cert_keyspace(sp);
        if (sp->implicit && !ks)
            raise(VCS_EINVAL, "the sharded certified pass needs key-space pairs (unset VCS_CERT_BFS)");
        if (!sp->implicit) vcs::ensure_csr(sp);
        vcs::ensure_solve_buffers(sp, sp->H + 1);
        if (!sp->cert_shard) sp->cert_shard = new vcs::CertShard;
        vcs::CertShard& cs = *sp->cert_shard;
        cs.world = world;
        cs.rank = rank;
        cs.exchange = exchange;
        cs.keyspace = ks;
        cs.half = ks ? vcs::cert_half(sp) : 0;
        cs.eps = o.epsilon;
        cs.discount = o.discount;
        cs.max_sweeps = o.max_sweeps;
        vcs::multi_plan(sp, world, cs);
        const int H = sp->H;
        cs.xd.exact(ks ? 2 * cs.half : sp->S, sp->stream);
        cs.lb.exact(static_cast<size_t>(H) + 2, sp->stream);
        VCS_CUDA(cudaStreamSynchronize(sp->stream)); // pool allocations ready for any stream
        const vcs::StreamUse s(sp, stream);
        // every output element is written by exactly one rank; the others hold zeros, so a
        // SUM of the ranks' arrays (integer views) assembles the result bit for bit
        VCS_CUDA(cudaMemsetAsync(sp->v[0].p, 0, sp->S * sizeof(double), s));
        VCS_CUDA(cudaMemsetAsync(sp->actions_dev.p, 0, sp->S * sizeof(int32_t), s));
        const uint64_t rH = sp->layer_off[H], nH = sp->S - rH;
        if (rank == 0) VCS_CUDA(cudaMemsetAsync(sp->actions_dev.p + rH, 0xff, nH * sizeof(int32_t), s));
        VCS_CUDA(cudaMemsetAsync(cs.lb.p, 0, (H + 2) * sizeof(double), s));
        if (ks)
            VCS_CUDA(cudaMemsetAsync(cs.xd.p + (H & 1) * cs.half, 0, sizeof(double2), s));
        else
            VCS_CUDA(cudaMemsetAsync(cs.xd.p + rH, 0, nH * sizeof(double2), s));
        return VCS_OK;
    });
}

int vcs_cert_shard_plan(const vcs_space* sp, int32_t t, int32_t q, uint64_t* out) {
    return guarded([&] {
        if (!sp->cert_shard) raise(VCS_EINVAL, "vcs_cert_shard_begin first");
        const vcs::CertShard& cs = *sp->cert_shard;
        if (t < 0 || t >= sp->H || q < 0 || q >= cs.world) raise(VCS_EINVAL, "layer/rank out of range");
        const size_t tt = static_cast<size_t>(t), qq = static_cast<size_t>(q);
        const vcs::CertLayer L = vcs::cert_layer(sp, t, nullptr, cs.half, cs.keyspace);
        out[0] = cs.split[tt] ? 1 : 0;
        out[1] = cs.lo[tt][qq];
        out[2] = cs.hi[tt][qq];
        out[3] = cs.need_lo[tt][qq];
        out[4] = cs.need_hi[tt][qq];
        out[5] = cs.keyspace ? (L.dense_order ? L.dense_n : L.n) : L.n;
        return VCS_OK;
    });
}

int vcs_cert_shard_layer(vcs_space* sp, int32_t t, void* stream) {
    std::lock_guard<std::recursive_mutex> space_lock(sp->mu);
    return guarded([&] {
        if (!sp->cert_shard) raise(VCS_EINVAL, "vcs_cert_shard_begin first");
        vcs::CertShard& cs = *sp->cert_shard;
        if (t < 0 || t >= sp->H) raise(VCS_EINVAL, "layer out of range");
        vcs::bind_device(sp->device);
        const vcs::StreamUse s(sp, stream);
        const size_t tt = static_cast<size_t>(t), rr = static_cast<size_t>(cs.rank);
        const bool split = cs.split[tt] != 0;
        const uint64_t lo = cs.lo[tt][rr], hi = cs.hi[tt][rr];
        const int write_out = (split || cs.rank == 0) ? 1 : 0;
        if (cs.keyspace) {
            vcs::CertLayer L = vcs::cert_layer(sp, t, cs.xd.p, cs.half, true);
            if (L.dense_order) {
                L.d_lo = lo;
                L.d_hi = hi;
            }
            if (L.n && (!L.dense_order || hi > lo))
                vcs::launch_cert_layer(sp, vcs::cert_data_of(sp), L, sp->v[0].p, sp->actions_dev.p,
                                       cs.lb.p, cs.discount, write_out, false, s);
        } else if (hi > lo) {
            vcs::CertArgs a{};
            a.row_ptr = sp->row_ptr.p;
            a.succ = sp->succ.p;
            a.reward = sp->reward.p;
            a.action = sp->action.p;
            a.values_out = sp->v[0].p;
            a.act_out = sp->actions_dev.p;
            a.write_out = write_out;
            a.lb = cs.lb.p;
            a.discount = cs.discount;
            a.row0 = sp->layer_off[tt] + lo;
            a.n = hi - lo;
            a.next_row0 = sp->layer_off[tt + 1];
            a.m = sp->H - t;
            a.xd_next = cs.xd.p + a.next_row0;
            a.xd_cur = cs.xd.p + a.row0;
            const unsigned blocks = static_cast<unsigned>(std::max<uint64_t>(
                1, std::min<uint64_t>((a.n + 255) / 256, static_cast<uint64_t>(4) * sp->num_sms)));
            if (vcs::is_discounted(cs.discount)) vcs::k_cert_rows<true, 4, 4><<<blocks, 256, 0, s>>>(a);
            else vcs::k_cert_rows<false, 4, 4><<<blocks, 256, 0, s>>>(a);
            VCS_LAUNCHED();
        }
        return VCS_OK;
    });
}

int vcs_cert_shard_pairs(const vcs_space* sp, int32_t t, double** pairs) {
    return guarded([&] {
        if (!sp->cert_shard) raise(VCS_EINVAL, "vcs_cert_shard_begin first");
        const vcs::CertShard& cs = *sp->cert_shard;
        if (t < 0 || t > sp->H) raise(VCS_EINVAL, "layer out of range");
        const uint64_t base = cs.keyspace ? (t & 1) * cs.half : sp->layer_off[static_cast<size_t>(t)];
        *pairs = reinterpret_cast<double*>(cs.xd.p + base);
        return VCS_OK;
    });
}

int vcs_cert_shard_buffers(const vcs_space* sp, double** lb, double** values, int32_t** actions) {
    return guarded([&] {
        if (!sp->cert_shard) raise(VCS_EINVAL, "vcs_cert_shard_begin first");
        if (lb) *lb = sp->cert_shard->lb.p;
        if (values) *values = sp->v[0].p;
        if (actions) *actions = sp->actions_dev.p;
        return VCS_OK;
    });
}

int vcs_cert_shard_finish(const vcs_space* sp, const double* lb_max, int32_t* certified) {
    return guarded([&] {
        if (!sp->cert_shard) raise(VCS_EINVAL, "vcs_cert_shard_begin first");
        const vcs::CertShard& cs = *sp->cert_shard;
        const int H = sp->H;
        int M = H + 1;
        if (cs.max_sweeps > 0) M = std::min(M, cs.max_sweeps);
        bool ok = M >= H + 1;
        for (int k = 1; k <= H && ok; ++k) ok = lb_max[k] >= cs.eps; // NaN-safe, as k_cert_check
        *certified = ok ? 1 : 0;
        return VCS_OK;
    });
}

int vcs_multi_info(const vcs_space* sp, vcs_multi_report* out) {
    return guarded([&] {
        if (!sp->multi) raise(VCS_EINVAL, "no multi-GPU solve ran on this space");
        const vcs::MultiState& ms = *sp->multi;
        *out = vcs_multi_report{};
        out->n_ranks = static_cast<int32_t>(ms.ranks.size());
        out->split_layers = ms.split_layers;
        out->replicated_layers = ms.replicated_layers;
        out->exchange = ms.exchange;
        out->halo_bytes = ms.halo_bytes;
        out->max_share = ms.max_share;
        out->graph = ms.no_graph ? 0 : 1;
        return VCS_OK;
    });
}

namespace {
// int32 actions -> int8 (every action of a space with <= 127 clouds fits): the download of the
// action column shrinks 4x and the host widens it back while later chunks are in flight.
__global__ void k_narrow_actions(const int32_t* __restrict__ a, int8_t* __restrict__ b, uint64_t n) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        b[i] = static_cast<int8_t>(a[i]);
}

// Pinned host staging blocks, recycled across spaces (a cudaHostAlloc costs milliseconds).
struct PinnedFreeList {
    std::mutex m;
    std::vector<std::pair<void*, size_t>> blocks;
};
PinnedFreeList& pinned_free_list() {
    static PinnedFreeList* f = new PinnedFreeList; // never destroyed: used until process exit
    return *f;
}
void* pinned_acquire(size_t bytes, size_t* got) {
    auto& f = pinned_free_list();
    {
        std::lock_guard<std::mutex> lk(f.m);
        size_t best = f.blocks.size();
        for (size_t i = 0; i < f.blocks.size(); ++i)
            if (f.blocks[i].second >= bytes &&
                (best == f.blocks.size() || f.blocks[i].second < f.blocks[best].second))
                best = i;
        if (best < f.blocks.size()) {
            auto b = f.blocks[best];
            f.blocks.erase(f.blocks.begin() + static_cast<long>(best));
            *got = b.second;
            return b.first;
        }
    }
    const size_t want = bytes + bytes / 4; // headroom for the next, slightly larger space
    void* p = nullptr;
    VCS_CUDA(cudaHostAlloc(&p, want, cudaHostAllocPortable));
    *got = want;
    return p;
}
void pinned_release(void* p, size_t bytes) {
    auto& f = pinned_free_list();
    std::lock_guard<std::mutex> lk(f.m);
    f.blocks.emplace_back(p, bytes);
    while (f.blocks.size() > 4) { // bounded: free the smallest
        auto it = std::min_element(f.blocks.begin(), f.blocks.end(),
                                   [](const auto& x, const auto& y) { return x.second < y.second; });
        cudaFreeHost(it->first);
        f.blocks.erase(it);
    }
}

// Persistent host workers for the widening (the calling thread works too).
class HostWorkers {
public:
    static HostWorkers& get() {
        static HostWorkers* w = new HostWorkers; // never destroyed: no join at process exit
        return *w;
    }
    // fn(begin, end) over [0, n) in pieces of `grain`; returns when every piece is done
    void parallel_for(size_t n, size_t grain, const std::function<void(size_t, size_t)>& fn) {
        if (n == 0) return;
        // a forked child inherits this object but not the threads: work inline there; so does a
        // caller that finds the pool busy with another thread's job (one job at a time)
        std::unique_lock<std::mutex> job(job_m_, std::try_to_lock);
        if (th_.empty() || n <= grain || getpid() != pid_ || !job.owns_lock()) {
            fn(0, n);
            return;
        }
        std::unique_lock<std::mutex> lk(m_);
        job_ = &fn;
        n_ = n;
        grain_ = grain;
        next_.store(0);
        busy_ = static_cast<int>(th_.size());
        ++gen_;
        cv_.notify_all();
        lk.unlock();
        work();
        lk.lock();
        done_cv_.wait(lk, [&] { return busy_ == 0; });
        job_ = nullptr;
    }

private:
    HostWorkers() : pid_(getpid()) {
        unsigned hw = std::thread::hardware_concurrency();
        // one process per GPU (torchrun): each takes its share of the host's cores
        if (const char* lw = std::getenv("LOCAL_WORLD_SIZE")) {
            const int n = std::atoi(lw);
            if (n > 1) hw /= static_cast<unsigned>(n);
        }
        unsigned cap = 7u; // 7..11 measured equal on the 16-core box; fewer lose, more lose
        if (const char* e = std::getenv("VCS_HOST_WORKERS")) cap = static_cast<unsigned>(std::atoi(e));
        const unsigned n = hw > 2 ? std::min(cap, hw - 1) : 0u;
        for (unsigned i = 0; i < n; ++i) th_.emplace_back([this] { loop(); });
        for (auto& t : th_) t.detach();
    }
    void work() {
        for (;;) {
            const size_t b = next_.fetch_add(grain_);
            if (b >= n_) return;
            (*job_)(b, std::min(n_, b + grain_));
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            std::unique_lock<std::mutex> lk(m_);
            cv_.wait(lk, [&] { return gen_ != seen; });
            seen = gen_;
            lk.unlock();
            work();
            lk.lock();
            if (--busy_ == 0) done_cv_.notify_all();
        }
    }
    const pid_t pid_;
    std::vector<std::thread> th_;
    std::mutex job_m_; // held by the caller whose job the workers run
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(size_t, size_t)>* job_ = nullptr;
    size_t n_ = 0, grain_ = 1;
    std::atomic<size_t> next_{0};
    int busy_ = 0;
    uint64_t gen_ = 0;
};

// int8 -> int32 widening of the action column on the host (plain stores: AVX2 conversion with
// non-temporal stores measured the same on the B200 box, 4.01-4.18 vs 4.02-4.05 ms C4 e2e)
void widen(const int8_t* src, int32_t* dst, size_t n) {
    for (size_t i = 0; i < n; ++i) dst[i] = src[i];
}

bool is_pinned(const void* p) {
    if (!p) return true;
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeHost;
}
} // namespace

namespace {
std::mutex& host_alloc_mu() {
    static std::mutex* m = new std::mutex;
    return *m;
}
std::map<void*, size_t>& host_alloc_sizes() {
    static auto* m = new std::map<void*, size_t>;
    return *m;
}
} // namespace

// Blocks below 1 MB come from malloc (a small result gains nothing from page-locking and would
// tie up a large recycled pinned block); size 0 in the map marks them.
constexpr size_t kPinnedMin = size_t(1) << 20;

void* vcs_host_alloc(uint64_t bytes) {
    try {
        size_t got = 0;
        void* p = nullptr;
        if (bytes < kPinnedMin) {
            p = std::malloc(std::max<size_t>(static_cast<size_t>(bytes), 64));
            if (!p) return nullptr;
        } else {
            p = pinned_acquire(static_cast<size_t>(bytes), &got);
        }
        std::lock_guard<std::mutex> lk(host_alloc_mu());
        host_alloc_sizes()[p] = got;
        return p;
    } catch (...) {
        cudaGetLastError();
        return nullptr;
    }
}

void vcs_host_free(void* p) {
    if (!p) return;
    size_t n = 0;
    {
        std::lock_guard<std::mutex> lk(host_alloc_mu());
        auto it = host_alloc_sizes().find(p);
        if (it == host_alloc_sizes().end()) return;
        n = it->second;
        host_alloc_sizes().erase(it);
    }
    if (n == 0) std::free(p);
    else pinned_release(p, n);
}

uint64_t vcs_space_result_generation(const vcs_space* sp) { return sp->result_gen; }

namespace {
// results of at least this many bytes (12 per state) stream behind the layer pass
uint64_t stream_threshold() { // (read per call: tests force the streamed path on small spaces)
    const char* e = std::getenv("VCS_STREAM_MIN_MB");
    return static_cast<uint64_t>(e ? std::atof(e) * (1 << 20) : 32.0 * (1 << 20));
}
} // namespace

int vcs_solve(vcs_space* sp, const vcs_solve_opts* opts, double* values_out, int32_t* actions_out,
              vcs_solve_report* report) {
    std::lock_guard<std::recursive_mutex> space_lock(sp->mu);
    const double t_start = vcs::trace_enabled() ? vcs::host_ms() : 0.0;
    struct TraceEnd {
        double t0;
        ~TraceEnd() {
            if (vcs::trace_enabled())
                std::fprintf(stderr, "[vcs solve] vcs_solve total %.3f ms\n", vcs::host_ms() - t0);
        }
    } trace_end{t_start};
    const bool pinned_out =
        (values_out || actions_out) && is_pinned(values_out) && is_pinned(actions_out);
    // int8 action column on the wire when every action fits (<= 127 clouds); its device buffer
    // is allocated before the solve is enqueued so the download stream, which waits on the
    // solve's layer events, is ordered after the allocation
    const bool narrow = pinned_out && actions_out && sp->has_plan && sp->plan.n_clouds <= 127 &&
                        sp->S * 12 >= stream_threshold() && !std::getenv("VCS_NO_NARROW");
    if (narrow) {
        const int rca = guarded([&] {
            vcs::bind_device(sp->device);
            sp->act8_dev.exact(sp->S, sp->stream);
            return VCS_OK;
        });
        if (rca != VCS_OK) return rca;
    }
    // streaming the result behind per-layer events pays for large results only: a small one
    // (< 32 MB) goes in one copy after the PDL-chained pass (canonical: 331 layers, 0.8 MB)
    const bool stream_out = pinned_out && sp->S * 12 >= stream_threshold();
    const uint64_t row_bytes = (values_out ? 8 : 0) + (actions_out ? (narrow ? 1 : 4) : 0);
    const int rc = enqueue_impl(sp, opts, nullptr, stream_out ? static_cast<int>(row_bytes) : 0);
    if (rc != VCS_OK) return rc;
    const vcs::CachedGraph& g = *sp->last_graph;
    const bool overlap = g.method != vcs::kMethodJacobi && !g.layer_ev.empty() && pinned_out;
    if (!overlap) return vcs_solve_collect(sp, values_out, actions_out, report, nullptr);
    // Stream each layer's values/actions to the (pinned) host buffers as soon as its layer
    // kernel finished — the 12 B/state download overlaps the rest of the layer pass.
    const int rc2 = guarded([&] {
        if (!sp->d2h_stream) sp->d2h_stream = vcs::acquire_stream(sp->device);
        cudaStream_t d = sp->d2h_stream;
        int8_t* staging = nullptr;
        size_t staging_bytes = 0;
        struct StagingGuard {
            int8_t*& p;
            size_t& n;
            ~StagingGuard() {
                if (p) pinned_release(p, n);
            }
        } staging_guard{staging, staging_bytes};
        if (narrow) staging = static_cast<int8_t*>(pinned_acquire(sp->S, &staging_bytes));
        struct Piece {
            uint64_t r0, r1;
            cudaEvent_t ev;
        };
        std::vector<Piece> pieces;
        auto copy_rows = [&](uint64_t r0, uint64_t r1, cudaStream_t st) {
            if (r1 <= r0) return;
            if (values_out)
                VCS_CUDA(cudaMemcpyAsync(values_out + r0, sp->v[0].p + r0, (r1 - r0) * sizeof(double),
                                         cudaMemcpyDeviceToHost, st));
            if (actions_out)
                VCS_CUDA(cudaMemcpyAsync(actions_out + r0, sp->actions_dev.p + r0,
                                         (r1 - r0) * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        };
        // Rows are final layer by layer, from the back: copy them in chunks of >= 16 MB (fewer,
        // larger DMA transfers), each after the event of its last (lowest) layer.  The terminal
        // layer's rows go with the first chunk: its memsets precede layer H-1's kernel.
        const std::vector<char> piece = vcs::piece_layers(sp, row_bytes);
        uint64_t chunk_end = sp->S;
        for (int t = sp->H - 1; t >= 0; --t) {
            const uint64_t r0 = sp->layer_off[t];
            if (!piece[static_cast<size_t>(t)]) continue;
            VCS_CUDA(cudaStreamWaitEvent(d, g.layer_ev[static_cast<size_t>(t)], 0));
            if (!narrow) {
                copy_rows(r0, chunk_end, d);
            } else {
                const uint64_t n = chunk_end - r0;
                if (values_out)
                    VCS_CUDA(cudaMemcpyAsync(values_out + r0, sp->v[0].p + r0, n * sizeof(double),
                                             cudaMemcpyDeviceToHost, d));
                const unsigned blocks = static_cast<unsigned>(
                    std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(sp->num_sms) * 8));
                k_narrow_actions<<<std::max(1u, blocks), 256, 0, d>>>(sp->actions_dev.p + r0,
                                                                      sp->act8_dev.p + r0, n);
                VCS_LAUNCHED();
                VCS_CUDA(cudaMemcpyAsync(staging + r0, sp->act8_dev.p + r0, n, cudaMemcpyDeviceToHost, d));
                const size_t k = pieces.size();
                if (sp->piece_ev.size() <= k) sp->piece_ev.push_back(vcs::acquire_event(sp->device, false));
                VCS_CUDA(cudaEventRecord(sp->piece_ev[k], d));
                pieces.push_back(Piece{r0, chunk_end, sp->piece_ev[k]});
            }
            chunk_end = r0;
        }
        // widen each int8 piece into the caller's int32 column as soon as it landed (the later
        // pieces are still on the wire, the lower layers still solving): the host widening,
        // not the wire, is the slower of the two on a 16-core host
        const bool tr = vcs::trace_enabled();
        const double tw0 = tr ? vcs::host_ms() : 0.0;
        for (const Piece& pc : pieces) {
            const double ta = tr ? vcs::host_ms() : 0.0;
            VCS_CUDA(cudaEventSynchronize(pc.ev));
            const double tb = tr ? vcs::host_ms() : 0.0;
            const int8_t* src = staging + pc.r0;
            int32_t* dst = actions_out + pc.r0;
            HostWorkers::get().parallel_for(pc.r1 - pc.r0, size_t(1) << 17, [&](size_t b, size_t e) {
                widen(src + b, dst + b, e - b);
            });
            if (tr)
                std::fprintf(stderr, "[vcs solve] piece %llu rows: waited %.3f ms, widened %.3f ms (t=%.3f)\n",
                             static_cast<unsigned long long>(pc.r1 - pc.r0), tb - ta, vcs::host_ms() - tb,
                             vcs::host_ms() - tw0);
        }
        vcs_solve_report local{};
        vcs_solve_report* rep = report ? report : &local;
        const int rc3 = vcs_solve_collect(sp, nullptr, nullptr, rep, nullptr);
        if (rc3 != VCS_OK) vcs::raise(rc3, vcs_last_error());
        // an early stop (K* < H) rewrote the prefix of layers t < H - K* after their events
        // (the pieces above may hold the certified pass's rows there: copied over now)
        const int K = rep->sweeps;
        if (sp->H - K > 0) {
            VCS_CUDA(cudaStreamSynchronize(d));
            copy_rows(0, sp->layer_off[sp->H - K], sp->stream);
            VCS_CUDA(cudaStreamSynchronize(sp->stream));
        }
        VCS_CUDA(cudaStreamSynchronize(d));
        return VCS_OK;
    });
    return rc2;
}

int vcs_solve_collect(vcs_space* sp, double* values_out, int32_t* actions_out,
                      vcs_solve_report* report, void* stream) {
    std::lock_guard<std::recursive_mutex> space_lock(sp->mu);
    return guarded([&] {
        if (!sp->last_graph) raise(VCS_EINVAL, "no solve was enqueued on this space");
        vcs::bind_device(sp->device);
        const vcs::StreamUse s(sp, stream);
        if (sp->cert_tl.n && std::getenv("VCS_CERT_TIMELINE")) { // per-layer timeline, stderr
            std::vector<unsigned long long> tl(sp->cert_tl.n);
            VCS_CUDA(cudaMemcpyAsync(tl.data(), sp->cert_tl.p, tl.size() * 8, cudaMemcpyDeviceToHost, s));
            VCS_CUDA(cudaStreamSynchronize(s));
            unsigned long long t0 = ~0ull;
            for (size_t m = 0; 3 * m + 2 < tl.size(); ++m) t0 = std::min(t0, tl[3 * m]);
            std::fprintf(stderr, "[vcs timeline] layer: entry / past-wait / exit (us from the first entry)\n");
            for (int m = sp->H; m >= 1; --m) {
                const unsigned long long* e = tl.data() + 3 * static_cast<size_t>(m);
                if (e[0] == ~0ull) continue;
                std::fprintf(stderr, "[vcs timeline] t=%d n=%llu: %.2f / %.2f / %.2f\n", sp->H - m,
                             static_cast<unsigned long long>(sp->layer_off[sp->H - m + 1] - sp->layer_off[sp->H - m]),
                             (e[0] - t0) * 1e-3, (e[1] - t0) * 1e-3, (~e[2] - t0) * 1e-3);
            }
        }
        vcs::SolveCtrl ctrl{};
        VCS_CUDA(cudaMemcpyAsync(&ctrl, sp->ctrl.p, sizeof ctrl, cudaMemcpyDeviceToHost, s));
        VCS_CUDA(cudaStreamSynchronize(s));
        const bool deferred = sp->last_graph->fallback_at_collect && !ctrl.certified;
        if (deferred) {
            // the proof failed (an early stop is possible): the layer wavefront on the explicit
            // CSR, materialised now, gives the reference's result
            if (std::getenv("VCS_PROFILE_NO_FALLBACK"))
                raise(VCS_EINVAL, "VCS_PROFILE_NO_FALLBACK: the proof failed, results are invalid");
            vcs_solve_opts fo = sp->last_opts;
            fo.method = VCS_METHOD_WAVEFRONT;
            const int rc = enqueue_impl(sp, &fo, stream, 0);
            if (rc != VCS_OK) vcs::raise(rc, vcs_last_error());
            VCS_CUDA(cudaMemcpyAsync(&ctrl, sp->ctrl.p, sizeof ctrl, cudaMemcpyDeviceToHost, s));
            VCS_CUDA(cudaStreamSynchronize(s));
        }
        auto& g = *sp->last_graph;
        const bool wave = g.method != vcs::kMethodJacobi; // wavefront or certified: V in v[0]
        const int K = ctrl.sweeps;
        if (g.method == vcs::kMethodCertified && !ctrl.certified &&
            std::getenv("VCS_PROFILE_NO_FALLBACK"))
            raise(VCS_EINVAL, "VCS_PROFILE_NO_FALLBACK: the proof failed, results are invalid");
        (void)0;
        // Jacobi leaves V_{K*} in ping-pong buffer K*&1; the wavefront extraction writes it to v[0]
        const double* vsrc = wave ? sp->v[0].p : sp->v[K & 1].p;
        sp->result_values = vsrc;
        sp->result_actions = sp->actions_dev.p;
        ++sp->result_gen;
        if (values_out)
            VCS_CUDA(cudaMemcpyAsync(values_out, vsrc, sp->S * sizeof(double),
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
            const double dbar = sp->S ? static_cast<double>(sp->E) / static_cast<double>(sp->S) : 0.0;
            uint64_t done = 0;
            const bool certified = g.method == vcs::kMethodCertified && ctrl.certified;
            if (certified && g.implicit) {
                // implicit-CSR form: per non-terminal state its key 8 + (V_{m-1}, V_m) pair
                // written 16 and read back 16; per state value 8 + action 4; the rank tables
                // read once (4 B per entry)
                const uint64_t nt = sp->layer_off[sp->H];
                done = 2 * nt;
                if (vcs::cert_keyspace(sp)) {
                    // pairs by key-space index: per layer its own index (full layers: the rank
                    // table entry of every key-space index, 4; sparse layers: the key, 8 per
                    // word), per state value 8 + action 4 + pair written 16, and the
                    // successors' pairs read once (16 per state of layer t+1)
                    double b = 12.0 * static_cast<double>(sp->S - nt); // terminal value/action
                    for (int t = 0; t < sp->H; ++t) {
                        const uint64_t n = sp->layer_off[t + 1] - sp->layer_off[t];
                        const uint64_t n1 = sp->layer_off[t + 2] - sp->layer_off[t + 1];
                        const uint64_t dn = t >= 1 ? sp->plan.layers[static_cast<size_t>(t - 1)].dense_size : 0;
                        const bool dense_order = t >= 1 && n * 2 >= dn;
                        b += dense_order ? 4.0 * static_cast<double>(dn)
                                         : 8.0 * static_cast<double>(n) * sp->plan.words[static_cast<size_t>(t)];
                        b += 28.0 * static_cast<double>(n) + 16.0 * static_cast<double>(n1);
                    }
                    report->model_bytes = b;
                } else {
                    report->model_bytes = 40.0 * nt + 12.0 * sp->S +
                                          4.0 * static_cast<double>(sp->rank_off.empty() ? 0 : sp->rank_off.back());
                }
            } else if (certified) {
                // two versions of every non-terminal state, once; per state: row_ptr 4 +
                // value 8 + action 4 + winning action 4 + its (V_{m-1}, V_m) pair written 16 and
                // read back 16; per edge: succ 4 + reward 8
                const uint64_t nt = sp->layer_off[sp->H];
                done = 2 * nt;
                report->model_bytes = 20.0 * sp->S + 32.0 * nt + 12.0 * sp->E;
            } else if (wave) {
                done = vcs::wave_backups(sp); // every version of every state, once
                // per state: row_ptr 4 + value out 8 + action out 4 + winning action 4; per
                // edge: succ 4 + reward 8; per version: written once + read back once (8 + 8)
                report->model_bytes = 20.0 * sp->S + 12.0 * sp->E + 16.0 * done;
            } else {
                for (int k = 1; k <= K; ++k) done += vcs::sweep_row_end(sp, k, sp->last_key_skip != 0);
                report->model_bytes = (20.0 + 12.0 * dbar) * static_cast<double>(done);
            }
            report->backups_done = done;
            report->sweep_ms = ms_sweep;
            report->extract_ms = ms_ext;
            report->method = g.method == vcs::kMethodCertified && !ctrl.certified
                                 ? vcs::kMethodWavefront // the proof failed: the wavefront ran
                                 : g.method;
            report->fallback_deferred = deferred ? 1 : 0;
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
        vcs::ensure_csr(sp); // the sharded solvers read the explicit CSR
        const vcs::StreamUse s(sp, stream);
        sp->ctrl.exact(1, sp->stream);
        sp->actions_dev.exact(sp->S, sp->stream);
        VCS_CUDA(cudaStreamSynchronize(sp->stream));
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
        vcs_solve_opts o{1e-6, 1, 0, 1.0, VCS_METHOD_JACOBI};
        if (opts) o = *opts;
        const vcs::StreamUse s(sp, stream);
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
        vcs_solve_opts o{1e-6, 1, 0, 1.0, VCS_METHOD_JACOBI};
        if (opts) o = *opts;
        const vcs::StreamUse s(sp, stream);
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

// ---- version-band sharded wavefront --------------------------------------------------------

int vcs_wave_shard_begin(vcs_space* sp, int32_t world, int32_t rank, const vcs_solve_opts* opts,
                         double* delta, void* stream) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world) raise(VCS_EINVAL, "bad world/rank");
        vcs_solve_opts o{1e-6, 1, 0, 1.0, VCS_METHOD_WAVEFRONT};
        if (opts) o = *opts;
        if (!(o.epsilon > 0.0))
            raise(VCS_EINVAL, "epsilon must be > 0 (value iteration would never terminate)");
        vcs::bind_device(sp->device);
        vcs::ensure_csr(sp); // the sharded solvers read the explicit CSR
        const vcs::StreamUse s(sp, stream);
        sp->wave_world = world;
        sp->wave_rank = rank;
        sp->wave_eps = o.epsilon;
        sp->wave_discount = o.discount;
        vcs::band_plan(sp, world, rank);
        const uint64_t total = sp->band_off[static_cast<size_t>(sp->H) + 1];
        if (!delta) raise(VCS_EINVAL, "delta buffer (horizon+3 doubles) required");
        sp->wave_delta = delta;
        sp->band_ver.exact(total + 4, sp->stream); // +4: a consumer pair may read past the end
        sp->v[0].exact(sp->S, sp->stream);
        sp->actions_dev.exact(sp->S, sp->stream);
        VCS_CUDA(cudaStreamSynchronize(sp->stream));
        // zero store: V_0 slots and the constant halo (version 0) of bands starting at 1
        VCS_CUDA(cudaMemsetAsync(sp->band_ver.p, 0, (total + 4) * sizeof(double), s));
        VCS_CUDA(cudaMemsetAsync(delta, 0, (sp->H + 3) * sizeof(double), s));
        const uint64_t rH = sp->layer_off[sp->H], nH = sp->S - rH;
        VCS_CUDA(cudaMemsetAsync(sp->v[0].p + rH, 0, nH * sizeof(double), s));
        VCS_CUDA(cudaMemsetAsync(sp->actions_dev.p + rH, 0xff, nH * sizeof(int32_t), s));
        return VCS_OK;
    });
}

int vcs_wave_shard_band(const vcs_space* sp, int32_t t, int32_t* lo, int32_t* hi) {
    return guarded([&] {
        if (sp->band_lo.empty()) raise(VCS_EINVAL, "vcs_wave_shard_begin was not called");
        if (t < 0 || t > sp->H) raise(VCS_EINVAL, "layer out of range");
        *lo = sp->band_lo[t];
        *hi = sp->band_hi[t];
        return VCS_OK;
    });
}

int vcs_wave_shard_layer(vcs_space* sp, int32_t t, void* stream) {
    return guarded([&] {
        if (sp->band_lo.empty()) raise(VCS_EINVAL, "vcs_wave_shard_begin was not called");
        if (t < 0 || t >= sp->H) raise(VCS_EINVAL, "layer out of range");
        const vcs::StreamUse s(sp, stream);
        const bool disc = vcs::is_discounted(sp->wave_discount);
        vcs::WaveArgs a{};
        a.row_ptr = sp->row_ptr.p;
        a.succ = sp->succ.p;
        a.reward = sp->reward.p;
        a.action = sp->action.p;
        a.ver = sp->band_ver.p;
        a.delta = sp->wave_delta;
        a.values_out = sp->v[0].p;
        a.act_out = sp->actions_dev.p;
        a.eps = sp->wave_eps;
        a.discount = sp->wave_discount;
        a.H = sp->H;
        a.row0 = sp->layer_off[t];
        a.n = sp->layer_off[t + 1] - sp->layer_off[t];
        a.next_row0 = sp->layer_off[t + 1];
        a.voff = sp->band_off[t];
        a.voff_next = sp->band_off[t + 1];
        a.m = sp->H - t;
        a.band_lo = sp->band_lo[t];
        a.band_hi = sp->band_hi[t];
        a.next_lo = sp->band_lo[t + 1];
        a.base = sp->band_base[t];
        a.base_next = sp->band_base[t + 1];
        a.stride = sp->band_stride[t];
        a.stride_next = sp->band_stride[t + 1];
        vcs::launch_layer(sp, a, disc, s);
        return VCS_OK;
    });
}

int vcs_wave_shard_pack(vcs_space* sp, int32_t t, int32_t version, double* dst, void* stream) {
    return guarded([&] {
        if (sp->band_lo.empty()) raise(VCS_EINVAL, "vcs_wave_shard_begin was not called");
        if (t < 0 || t > sp->H || version < sp->band_base[t] || version >= sp->band_hi[t])
            raise(VCS_EINVAL, "version not held by this rank");
        const vcs::StreamUse s(sp, stream);
        const uint64_t n = sp->layer_off[t + 1] - sp->layer_off[t];
        if (!n) return VCS_OK;
        vcs::k_band_pack<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
            sp->band_ver.p + sp->band_off[t], n, static_cast<uint32_t>(sp->band_stride[t]),
            static_cast<uint32_t>(version - sp->band_base[t]), dst);
        VCS_LAUNCHED();
        return VCS_OK;
    });
}

int vcs_wave_shard_unpack(vcs_space* sp, int32_t t, const double* src, void* stream) {
    return guarded([&] {
        if (sp->band_lo.empty()) raise(VCS_EINVAL, "vcs_wave_shard_begin was not called");
        if (t < 0 || t > sp->H) raise(VCS_EINVAL, "layer out of range");
        const vcs::StreamUse s(sp, stream);
        const uint64_t n = sp->layer_off[t + 1] - sp->layer_off[t];
        if (!n) return VCS_OK;
        const int lo = sp->band_lo[t];
        const int has_low = sp->band_hi[t] > lo ? 1 : 0; // residual of version lo needs the halo
        vcs::k_band_unpack<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
            sp->band_ver.p + sp->band_off[t], n, static_cast<uint32_t>(sp->band_stride[t]),
            static_cast<uint32_t>(lo - 1 - sp->band_base[t]), src, has_low,
            sp->wave_delta + lo);
        VCS_LAUNCHED();
        return VCS_OK;
    });
}

int vcs_wave_shard_finish(vcs_space* sp, int32_t K, double* values_out, int32_t* actions_out,
                          void* stream) {
    return guarded([&] {
        if (sp->band_lo.empty()) raise(VCS_EINVAL, "vcs_wave_shard_begin was not called");
        if (K < 1) raise(VCS_EINVAL, "sweep count must be >= 1");
        const vcs::StreamUse s(sp, stream);
        const int H = sp->H;
        const bool disc = vcs::is_discounted(sp->wave_discount);
        auto owns = [&](int t, int k) { return sp->band_lo[t] <= k && k < sp->band_hi[t]; };
        // early-stop fix-up of layers t < H - K: values by the owner of version K of layer t,
        // actions by the owner of version K of layer t+1 (the argmax reads V_K of successors)
        for (int t = 0; t < H - K; ++t) {
            const bool val = owns(t, K), act = owns(t + 1, K);
            if (!val && !act) continue;
            const uint64_t n = sp->layer_off[t + 1] - sp->layer_off[t];
            if (!n) continue;
            const unsigned grid = static_cast<unsigned>((n + 255) / 256);
            auto launch = [&](auto kern) {
                kern<<<grid, 256, 0, s>>>(
                    sp->row_ptr.p, sp->succ.p, sp->reward.p, sp->action.p,
                    val ? sp->band_ver.p + sp->band_off[t] : nullptr,
                    static_cast<uint32_t>(sp->band_stride[t]),
                    static_cast<uint32_t>(val ? K - sp->band_base[t] : 0),
                    act ? sp->band_ver.p + sp->band_off[t + 1] : nullptr,
                    static_cast<uint32_t>(sp->band_stride[t + 1]),
                    static_cast<uint32_t>(act ? K - sp->band_base[t + 1] : 0), sp->layer_off[t], n,
                    sp->layer_off[t + 1], sp->wave_discount, sp->v[0].p, sp->actions_dev.p);
            };
            if (disc) launch(vcs::k_band_fixup<true>);
            else launch(vcs::k_band_fixup<false>);
            VCS_LAUNCHED();
        }
        // every row's value and action reach the host from exactly one rank each: exact rows
        // (t >= H-K, and the terminal layer) from the rank holding version m_t (the last rank),
        // fix-up rows from the owners above
        auto copy = [&](bool values, uint64_t r0, uint64_t r1) {
            if (r1 <= r0) return;
            if (values && values_out)
                VCS_CUDA(cudaMemcpyAsync(values_out + r0, sp->v[0].p + r0, (r1 - r0) * sizeof(double),
                                         cudaMemcpyDeviceToHost, s));
            if (!values && actions_out)
                VCS_CUDA(cudaMemcpyAsync(actions_out + r0, sp->actions_dev.p + r0,
                                         (r1 - r0) * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        };
        const int first_exact = std::max(0, H - K);
        const bool exact_owner = sp->wave_rank == sp->wave_world - 1;
        for (int t = 0; t <= H; ++t) {
            const uint64_t r0 = sp->layer_off[t], r1 = sp->layer_off[t + 1];
            if (t >= first_exact) {
                if (exact_owner) {
                    copy(true, r0, r1);
                    copy(false, r0, r1);
                }
            } else {
                if (owns(t, K)) copy(true, r0, r1);
                if (owns(t + 1, K)) copy(false, r0, r1);
            }
        }
        VCS_CUDA(cudaStreamSynchronize(s));
        return VCS_OK;
    });
}

} // extern "C"
