// vcs_greedy.cu — Alg. 2 first-fit placement on the device (replaces greedy_schedule,
// greedy.cpp:5-30, with feasible() of workload.cpp:22-26).
//
// The scan is sequential through vm_free; the work is split in two:
//   1. k_attr_mask (all SMs): the batched feasibility scoring.  For every (task, cloud) pair the
//      link test `delay <= max_delay && thr >= min_thr` becomes one bit; a warp covers a task,
//      one ballot per 32 clouds, and also writes the task's {demand level, demand} descriptor.
//   2. first fit, one warp per instance:
//      k_first_fit_spec (default, <= 1024 clouds and <= 8 distinct demands): 32 tasks per step,
//        each evaluated against the capacity state at the step start, committed up to the first
//        task whose candidate no longer fits (see the comment at the kernel);
//      k_first_fit_fast (VCS_GREEDY_SERIAL=1): one task per step, AND -> ballot -> ffs;
//      k_first_fit (generic): more clouds or demands, capacity bits from the free counts.
// Placements are bit-exact against the reference (same first feasible cloud, same paid set).
#include "vcs_device.cuh"

#include <algorithm>
#include <cstdio>

namespace vcs {

namespace {

constexpr int kMaxLevels = 16;
constexpr int kPrefetch = 16;

struct GreedyDesc {
    int32_t K, T, W, n_levels; // n_levels == 0: generic capacity test from free counts
    const uint32_t* mask;      // T x W attribute words
    const int2* task;          // T: {level, demand}
    const int32_t* levels;     // n_levels distinct demands (ascending)
    int32_t* free_vms;         // K: in = vm_free, out = remaining free VMs
    int32_t* target;           // T: cloud index or -1
    long long* paid;           // 1
};

// Also writes each task's descriptor {level index, demand} (levels: the n_levels distinct
// demands, ascending; n_levels == 0: level 0).
__global__ void k_attr_mask(int32_t K, int32_t T, int32_t W, const double* __restrict__ c_delay,
                            const double* __restrict__ c_thr, const double* __restrict__ t_delay,
                            const double* __restrict__ t_thr, uint32_t* __restrict__ mask,
                            const int32_t* __restrict__ demand, const int32_t* __restrict__ levels,
                            int32_t n_levels, int2* __restrict__ task) {
    // one warp per task: a ballot per 32 clouds; lane w keeps word w of its group of 32 words
    // and the group is stored coalesced
    const int warp = static_cast<int>((static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    const int n_warps = static_cast<int>((static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5);
    const int lane = threadIdx.x & 31;
    for (int j = warp; j < T; j += n_warps) {
        const double td = __ldg(t_delay + j), tt = __ldg(t_thr + j);
        uint32_t* row = mask + static_cast<size_t>(j) * W;
        for (int w0 = 0; w0 < W; w0 += 32) {
            uint32_t mine = 0;
            const int nw = min(32, W - w0);
            for (int w = 0; w < nw; ++w) {
                const int c = (w0 + w) * 32 + lane;
                const bool ok = c < K && __ldg(c_delay + c) <= td && __ldg(c_thr + c) >= tt;
                const uint32_t bits = __ballot_sync(0xffffffffu, ok);
                if (lane == w) mine = bits;
            }
            if (lane < nw) row[w0 + lane] = mine;
        }
        if (lane == 0) {
            const int32_t d = demand[j];
            int level = 0;
            while (level < n_levels && levels[level] != d) ++level;
            task[j] = make_int2(n_levels ? level : 0, d);
        }
    }
}

__device__ __forceinline__ uint32_t cap_bits_generic(const int32_t* __restrict__ fr, int K, int w,
                                                     int d) {
    uint32_t bits = 0;
    const int c0 = w * 32;
#pragma unroll 8
    for (int b = 0; b < 32; ++b) {
        const int c = c0 + b;
        if (c < K && fr[c] >= d) bits |= 1u << b;
    }
    return bits;
}

// One warp per instance.  Shared memory: free[K] then cap[n_levels][W].
__global__ void __launch_bounds__(32) k_first_fit(const GreedyDesc* __restrict__ descs) {
    extern __shared__ int32_t sm[];
    const GreedyDesc D = descs[blockIdx.x];
    const int lane = threadIdx.x;
    int32_t* fr = sm;
    uint32_t* cap = reinterpret_cast<uint32_t*>(sm + D.K);
    for (int c = lane; c < D.K; c += 32) fr[c] = D.free_vms[c];
    __syncwarp();
    for (int L = 0; L < D.n_levels; ++L)
        for (int w = lane; w < D.W; w += 32) {
            uint32_t bits = 0;
            for (int b = 0; b < 32; ++b) {
                const int c = w * 32 + b;
                if (c < D.K && fr[c] >= D.levels[L]) bits |= 1u << b;
            }
            cap[L * D.W + w] = bits;
        }
    __syncwarp();
    long long paid = 0;
    const bool one_round = D.W <= 32;
    uint32_t cur[kPrefetch], nxt[kPrefetch];
    int2 tcur[kPrefetch], tnxt[kPrefetch];
    auto load_batch = [&](int j0, uint32_t (&m)[kPrefetch], int2 (&tk)[kPrefetch]) {
#pragma unroll
        for (int u = 0; u < kPrefetch; ++u) {
            const int j = j0 + u;
            m[u] = (one_round && j < D.T && lane < D.W) ? __ldg(D.mask + static_cast<size_t>(j) * D.W + lane) : 0u;
            tk[u] = j < D.T ? __ldg(D.task + j) : make_int2(0, 0);
        }
    };
    load_batch(0, cur, tcur);
    for (int j0 = 0; j0 < D.T; j0 += kPrefetch) {
        load_batch(j0 + kPrefetch, nxt, tnxt);
#pragma unroll
        for (int u = 0; u < kPrefetch; ++u) {
            const int j = j0 + u;
            if (j >= D.T) break;
            const int level = tcur[u].x, d = tcur[u].y;
            int winner = -1;
            if (one_round) {
                uint32_t m = cur[u];
                if (m) m &= D.n_levels ? cap[level * D.W + lane] : cap_bits_generic(fr, D.K, lane, d);
                const uint32_t any = __ballot_sync(0xffffffffu, m != 0);
                if (any) {
                    const int src = __ffs(any) - 1;
                    const uint32_t ms = __shfl_sync(0xffffffffu, m, src);
                    winner = src * 32 + __ffs(ms) - 1;
                }
            } else {
                for (int base = 0; base < D.W && winner < 0; base += 32) {
                    const int w = base + lane;
                    uint32_t m = w < D.W ? __ldg(D.mask + static_cast<size_t>(j) * D.W + w) : 0u;
                    if (m) m &= D.n_levels ? cap[level * D.W + w] : cap_bits_generic(fr, D.K, w, d);
                    const uint32_t any = __ballot_sync(0xffffffffu, m != 0);
                    if (any) {
                        const int src = __ffs(any) - 1;
                        const uint32_t ms = __shfl_sync(0xffffffffu, m, src);
                        winner = (base + src) * 32 + __ffs(ms) - 1;
                    }
                }
            }
            if (winner >= 0) {
                if (lane == 0) {
                    const int f = fr[winner] - d;
                    fr[winner] = f;
                    const int w = winner >> 5;
                    const uint32_t bit = 1u << (winner & 31);
                    for (int L = 0; L < D.n_levels; ++L) {
                        uint32_t& word = cap[L * D.W + w];
                        word = f >= D.levels[L] ? (word | bit) : (word & ~bit);
                    }
                    D.target[j] = winner;
                }
            } else {
                paid += d;
                if (lane == 0) D.target[j] = -1;
            }
            __syncwarp();
        }
#pragma unroll
        for (int u = 0; u < kPrefetch; ++u) {
            cur[u] = nxt[u];
            tcur[u] = tnxt[u];
        }
    }
    for (int c = lane; c < D.K; c += 32) D.free_vms[c] = fr[c];
    if (lane == 0) *D.paid = paid;
}

// Fast path: <= 1024 clouds (lane l owns word l: clouds 32l..32l+31) and <= 8 distinct demands.
// The capacity words "free >= level_L" live in REGISTERS of the owning lane; per task the
// critical path is AND -> ballot -> ffs, and only the winning lane updates its free count (in
// shared memory, touched by that lane only) and its capacity bits.  Targets are gathered in
// registers (lane j%32 keeps task j's) and stored 32 at a time, coalesced.
constexpr int kFastLevels = 8;

// NL >= every instance's distinct-demand count (the level loops are unrolled to NL)
template <int NL>
__global__ void __launch_bounds__(32) k_first_fit_fast(const GreedyDesc* __restrict__ descs) {
    extern __shared__ int32_t sm[];
    const GreedyDesc D = descs[blockIdx.x];
    const int lane = threadIdx.x;
    int32_t* fr = sm; // free counts, word-major: cloud c at fr[c]
    for (int c = lane; c < D.K; c += 32) fr[c] = D.free_vms[c];
    __syncwarp();
    int lvl[NL];
    uint32_t capw[NL];
#pragma unroll
    for (int L = 0; L < NL; ++L) {
        lvl[L] = L < D.n_levels ? D.levels[L] : 0x7fffffff;
        uint32_t bits = 0;
        if (L < D.n_levels)
            for (int b = 0; b < 32; ++b) {
                const int c = lane * 32 + b;
                if (c < D.K && fr[c] >= lvl[L]) bits |= 1u << b;
            }
        capw[L] = bits;
    }
    long long paid = 0;
    __shared__ int32_t s_tgt[32];
    uint32_t cur[kPrefetch], nxt[kPrefetch];
    int2 tcur[kPrefetch], tnxt[kPrefetch];
#pragma unroll
    for (int u = 0; u < kPrefetch; ++u) {
        cur[u] = (u < D.T && lane < D.W) ? __ldg(D.mask + static_cast<size_t>(u) * D.W + lane) : 0u;
        tcur[u] = u < D.T ? __ldg(D.task + u) : make_int2(0, 0);
    }
    for (int j0 = 0; j0 < D.T; j0 += kPrefetch) {
#pragma unroll
        for (int u = 0; u < kPrefetch; ++u) { // next batch in flight while this one is scanned
            const int j = j0 + kPrefetch + u;
            nxt[u] = (j < D.T && lane < D.W) ? __ldg(D.mask + static_cast<size_t>(j) * D.W + lane) : 0u;
            tnxt[u] = j < D.T ? __ldg(D.task + j) : make_int2(0, 0);
        }
#pragma unroll
        for (int u = 0; u < kPrefetch; ++u) {
            const int j = j0 + u;
            if (j < D.T) {
                const int level = tcur[u].x, d = tcur[u].y;
                uint32_t c = 0;
#pragma unroll
                for (int L = 0; L < NL; ++L) c = L == level ? capw[L] : c;
                const uint32_t m = cur[u] & c;
                const uint32_t any = __ballot_sync(0xffffffffu, m != 0);
                // the winner is recorded by the owning lane in shared memory (no shuffle on the
                // task chain); the group of 32 targets is written out coalesced
                if (any) {
                    const int src = __ffs(any) - 1;
                    if (lane == src) { // the owning lane updates its free count and bits
                        const int b = __ffs(m) - 1;
                        const int cloud = lane * 32 + b;
                        const int f = fr[cloud] - d;
                        fr[cloud] = f;
                        const uint32_t bit = 1u << b;
#pragma unroll
                        for (int L = 0; L < NL; ++L)
                            capw[L] = f >= lvl[L] ? (capw[L] | bit) : (capw[L] & ~bit);
                        s_tgt[j & 31] = cloud;
                    }
                } else {
                    paid += d;
                    if (lane == 0) s_tgt[j & 31] = -1;
                }
                if ((j & 31) == 31) {
                    __syncwarp();
                    D.target[j - 31 + lane] = s_tgt[lane];
                    __syncwarp();
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kPrefetch; ++u) {
            cur[u] = nxt[u];
            tcur[u] = tnxt[u];
        }
    }
    const int tail = D.T & 31; // the last partial group of 32 targets
    __syncwarp();
    if (tail && lane < tail) D.target[D.T - tail + lane] = s_tgt[lane];
    __syncwarp();
    for (int c = lane; c < D.K; c += 32) D.free_vms[c] = fr[c];
    if (lane == 0) *D.paid = paid;
}

// mbarrier + 1-D bulk copy (TMA) helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile("{\n\t.reg .pred p;\n"
                 "WAIT_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
                 "r"(parity)
                 : "memory");
}

constexpr int kRingBlocks = 4;   // blocks of attribute rows staged in shared memory
// warps of k_first_fit_spec4 (32 / kSpecWarps tasks each): C2 1.83 ms at 8, 1.94 ms at 4
constexpr int kSpecWarps = 8;
constexpr int kBlockRows = 128;  // rows per bulk copy (task arrays are padded to whole blocks)
constexpr int kRingRows = kRingBlocks * kBlockRows;
constexpr int kShadowRows = 32;  // ring rows 0..31 repeated past the end: a chunk never wraps
// dynamic shared memory of k_first_fit_spec: free counts, then the row ring (32 words per row:
// the fast path stores attribute rows at stride 32), then the task ring
__host__ __device__ constexpr size_t spec_free_bytes(size_t K) { return (K * 4 + 127) / 128 * 128; }
__host__ __device__ constexpr size_t spec_smem_bytes(size_t K) {
    return spec_free_bytes(K) + (kRingRows + kShadowRows) * (32 * 4 + 8);
}

// Speculative chunked form of the fast path (the default): 32 tasks per step instead of one.
// Every task of the chunk [j0, j0+32) takes its candidate = first feasible cloud under the
// capacity state S0 at the chunk start (32 independent AND -> ballot -> ffs, pipelined).  Free
// counts only decrease, so under the sequential state S_u of task u the feasible set is a subset
// of S0's: the true answer is >= the candidate and EQUALS it iff the candidate still fits,
// i.e. S0[c] >= inclusive prefix of demands of the chunk's tasks with the same candidate (a
// task without a candidate stays without one: paid).  The chunk commits tasks up to the first
// that fails this test and the next chunk starts there.  A failure leaves its candidate cloud
// with free < that task's demand, clearing a capacity bit for good, so there are at most
// K x n_levels failures: at most T/32 + K*n_levels steps for any input.  Same placements as the
// one-task-per-step scan (greedy.cpp:5-30 order), bit for bit.
// The common case is checked order-free: every placed demand is subtracted atomically from its
// candidate's free count; no count below zero means every prefix fits.  Only an overflowing
// chunk computes the prefixes (match.any groups + popcounts per level).
// Layout: lane l owns capacity word l (clouds 32l..32l+31), in shared memory per level.  The
// attribute rows (stride 32 words) and task descriptors, padded to whole 128-row blocks,
// stream into a 4-block shared-memory ring by 1-D bulk copies (+ 32 shadow rows so a chunk
// never wraps), up to three blocks ahead of the chunk.
template <int NL>
__global__ void __launch_bounds__(32) k_first_fit_spec(const GreedyDesc* __restrict__ descs) {
    extern __shared__ __align__(128) int32_t sm[];
    constexpr int kRing = kRingRows;
    __shared__ __align__(8) uint64_t s_bar[kRingBlocks];
    __shared__ uint32_t s_cap[NL][32]; // word w of level L: bit b = (free[32w+b] >= lvl[L])
    __shared__ __align__(16) uint32_t s_any[32]; // ballot of each task of the chunk
    const GreedyDesc D = descs[blockIdx.x];
    const int lane = threadIdx.x;
    constexpr uint32_t kAll = 0xffffffffu;
    if (D.T == 0) {
        if (lane == 0) *D.paid = 0;
        return;
    }
    constexpr int W = 32; // row stride of the fast path (words past ceil(K/32) are zero)
    const int n_blocks = (D.T + kBlockRows - 1) / kBlockRows;
    uint32_t* s_rows = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(sm) + spec_free_bytes(D.K)); // row j at (j % kRing) * W
    int2* s_task = reinterpret_cast<int2*>(s_rows + static_cast<size_t>(kRing + kShadowRows) * W);
    if (lane == 0) {
        for (int k = 0; k < kRingBlocks; ++k) bar_init(&s_bar[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    int32_t* fr = sm; // free counts, cloud c at fr[c]
    for (int c = lane; c < D.K; c += 32) fr[c] = D.free_vms[c];
    // a chunk near the end reads ring rows past the last block: their (stale) levels must still
    // index s_cap, their ballots belong to tasks past T and are never used
    for (int r = lane; r < kRing + kShadowRows; r += 32) s_task[r] = make_int2(0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    int lvl[NL];
#pragma unroll
    for (int L = 0; L < NL; ++L) {
        lvl[L] = L < D.n_levels ? D.levels[L] : 0x7fffffff;
        uint32_t bits = 0;
        if (L < D.n_levels)
            for (int b = 0; b < 32; ++b) {
                const int c = lane * 32 + b;
                if (c < D.K && fr[c] >= lvl[L]) bits |= 1u << b;
            }
        s_cap[L][lane] = bits;
    }
    const uint32_t le = (2u << lane) - 1u; // lanes <= this one
    int issued = 0, ready = 0;
    auto issue = [&]() { // block `issued` into its ring slot (lane 0)
        const int slot = issued & (kRingBlocks - 1);
        const uint32_t row_bytes = kBlockRows * static_cast<uint32_t>(W) * 4u;
        // (the slot's earlier shared reads were consumed before this point: no proxy fence)
        const uint32_t shadow = slot == 0 ? kShadowRows * (W * 4u + 8u) : 0u;
        bar_expect_tx(&s_bar[slot], row_bytes + kBlockRows * 8u + shadow);
        const uint32_t* src_rows = D.mask + static_cast<size_t>(issued) * kBlockRows * W;
        const int2* src_task = D.task + static_cast<size_t>(issued) * kBlockRows;
        bulk_g2s(&s_rows[static_cast<size_t>(slot) * kBlockRows * W], src_rows, row_bytes, &s_bar[slot]);
        bulk_g2s(&s_task[slot * kBlockRows], src_task, kBlockRows * 8u, &s_bar[slot]);
        if (slot == 0) { // the shadow copy of ring rows 0..31
            bulk_g2s(&s_rows[static_cast<size_t>(kRing) * W], src_rows, kShadowRows * W * 4u, &s_bar[slot]);
            bulk_g2s(&s_task[kRing], src_task, kShadowRows * 8u, &s_bar[slot]);
        }
        ++issued;
    };
    long long paid = 0;
    for (int j0 = 0; j0 < D.T;) {
        const int n = min(32, D.T - j0);
        const int b0 = j0 / kBlockRows;
        // the ring holds blocks b0..b0+3; the chunk needs the blocks of rows j0..j0+31
        if (lane == 0)
            while (issued < b0 + kRingBlocks && issued < n_blocks) issue();
        const int need = min((j0 + 31) / kBlockRows, n_blocks - 1);
        while (ready <= need) {
            bar_wait(&s_bar[ready & (kRingBlocks - 1)], (ready / kRingBlocks) & 1);
            ++ready;
        }
        __syncwarp();
        uint32_t any[32];
        const int r0 = j0 & (kRing - 1); // rows r0..r0+31 are contiguous (shadow rows)
        const uint32_t* rowp = s_rows + r0 * W + lane;
        const int2* taskp = s_task + r0;
#pragma unroll
        for (int u = 0; u < 32; ++u) { // 32 independent evaluations against the chunk-start state
            // branch-free and store-free: a branch region or a shared store per task would
            // serialise the unrolled chains (padding rows: level 0, zero words)
            const uint32_t m = rowp[u * W] & s_cap[taskp[u].x][lane];
            any[u] = __ballot_sync(kAll, m != 0);
        }
        if (lane == 0) {
            uint4* dst = reinterpret_cast<uint4*>(s_any);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                dst[q] = make_uint4(any[4 * q], any[4 * q + 1], any[4 * q + 2], any[4 * q + 3]);
        }
        __syncwarp();
        // lane u resolves task j0+u: the lowest lane with a feasible cloud, its lowest bit
        const int rme = (j0 + lane) & (kRing - 1);
        const int2 tk = s_task[rme];
        const int lvme = lane < n ? tk.x : NL;
        int my_c = -1;
        {
            const uint32_t any = s_any[lane];
            if (lane < n && any) {
                const int src = __ffs(any) - 1;
                const uint32_t m = s_rows[rme * W + src] & s_cap[lvme][src];
                my_c = src * 32 + __ffs(m) - 1;
            }
        }
        const bool placed = my_c >= 0;
        int ncommit = n;
        // common case first: take every placed demand off its candidate's free count.  The totals
        // do not depend on the order, and every inclusive prefix fits iff no count went negative.
        if (placed) atomicAdd(&fr[my_c], -tk.y);
        __syncwarp();
        const int fend = placed ? fr[my_c] : 0;
        if (!__any_sync(kAll, fend < 0)) {
            if (placed) { // clear the capacity bits the cloud lost (idempotent across its group)
                const uint32_t keep = ~(1u << (my_c & 31));
#pragma unroll
                for (int L = 0; L < NL; ++L)
                    if (fend < lvl[L]) atomicAnd(&s_cap[L][my_c >> 5], keep);
            }
        } else {
            if (placed) atomicAdd(&fr[my_c], tk.y); // undo; commit the exact prefix instead
            __syncwarp();
            // same-candidate groups and the inclusive prefix of their demands (levels: popcounts)
            const uint32_t peers = __match_any_sync(kAll, placed ? my_c : -1 - lane);
            int pre = 0;
#pragma unroll
            for (int L = 0; L < NL; ++L)
                if (L < D.n_levels) pre += lvl[L] * __popc(peers & le & __ballot_sync(kAll, lvme == L));
            const int f0 = placed ? fr[my_c] : 0;
            const uint32_t fails = __ballot_sync(kAll, placed && f0 < pre);
            ncommit = __ffs(fails) - 1; // >= 1: the first task fits S0
            const uint32_t cmask = (1u << ncommit) - 1u;
            __syncwarp();
            // the last committed member of each group writes its cloud's new free count and
            // clears the capacity bits the cloud lost
            if (placed && lane < ncommit && !(peers & cmask & ~le)) {
                const int f1 = f0 - pre;
                fr[my_c] = f1;
                const uint32_t keep = ~(1u << (my_c & 31));
#pragma unroll
                for (int L = 0; L < NL; ++L)
                    if (f1 < lvl[L]) atomicAnd(&s_cap[L][my_c >> 5], keep);
            }
        }
        const bool commit = lane < ncommit;
        if (commit) {
            D.target[j0 + lane] = my_c;
            if (!placed) paid += tk.y;
        }
        __syncwarp();
        j0 += ncommit;
    }
    while (ready < issued) { // drain the bulk copies still in flight
        bar_wait(&s_bar[ready & (kRingBlocks - 1)], (ready / kRingBlocks) & 1);
        ++ready;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) paid += __shfl_xor_sync(kAll, paid, o);
    __syncwarp();
    for (int c = lane; c < D.K; c += 32) D.free_vms[c] = fr[c];
    if (lane == 0) *D.paid = paid;
}

// The same first-fit with the 32 candidate evaluations of a chunk split over NW warps (32/NW
// tasks each); warp 0 resolves, validates and commits the chunk between two block barriers.
template <int NL, int NW>
__global__ void __launch_bounds__(NW * 32) k_first_fit_spec4(const GreedyDesc* __restrict__ descs) {
    constexpr int TPW = 32 / NW; // tasks per warp
    extern __shared__ __align__(128) int32_t sm[];
    constexpr int kRing = kRingRows;
    __shared__ __align__(8) uint64_t s_bar[kRingBlocks];
    __shared__ uint32_t s_cap[NL][32]; // word w of level L: bit b = (free[32w+b] >= lvl[L])
    __shared__ __align__(16) uint32_t s_any[32]; // ballot of each task of the chunk
    __shared__ int s_j0;
    const GreedyDesc D = descs[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t kAll = 0xffffffffu;
    if (D.T == 0) {
        if (tid == 0) *D.paid = 0;
        return;
    }
    constexpr int W = 32; // row stride of the fast path (words past ceil(K/32) are zero)
    const int n_blocks = (D.T + kBlockRows - 1) / kBlockRows;
    uint32_t* s_rows = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(sm) + spec_free_bytes(D.K));
    int2* s_task = reinterpret_cast<int2*>(s_rows + static_cast<size_t>(kRing + kShadowRows) * W);
    if (tid == 0) {
        for (int k = 0; k < kRingBlocks; ++k) bar_init(&s_bar[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    int32_t* fr = sm; // free counts, cloud c at fr[c]
    for (int c = tid; c < D.K; c += blockDim.x) fr[c] = D.free_vms[c];
    for (int r = tid; r < kRing + kShadowRows; r += blockDim.x) s_task[r] = make_int2(0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    int lvl[NL];
#pragma unroll
    for (int L = 0; L < NL; ++L) {
        lvl[L] = L < D.n_levels ? D.levels[L] : 0x7fffffff;
        if (warp == 0) {
            uint32_t bits = 0;
            if (L < D.n_levels)
                for (int b = 0; b < 32; ++b) {
                    const int c = lane * 32 + b;
                    if (c < D.K && fr[c] >= lvl[L]) bits |= 1u << b;
                }
            s_cap[L][lane] = bits;
        }
    }
    __syncthreads();
    const uint32_t le = (2u << lane) - 1u; // lanes <= this one
    int issued = 0, ready = 0;
    auto issue = [&]() { // block `issued` into its ring slot (thread 0)
        const int slot = issued & (kRingBlocks - 1);
        const uint32_t row_bytes = kBlockRows * static_cast<uint32_t>(W) * 4u;
        const uint32_t shadow = slot == 0 ? kShadowRows * (W * 4u + 8u) : 0u;
        bar_expect_tx(&s_bar[slot], row_bytes + kBlockRows * 8u + shadow);
        const uint32_t* src_rows = D.mask + static_cast<size_t>(issued) * kBlockRows * W;
        const int2* src_task = D.task + static_cast<size_t>(issued) * kBlockRows;
        bulk_g2s(&s_rows[static_cast<size_t>(slot) * kBlockRows * W], src_rows, row_bytes, &s_bar[slot]);
        bulk_g2s(&s_task[slot * kBlockRows], src_task, kBlockRows * 8u, &s_bar[slot]);
        if (slot == 0) {
            bulk_g2s(&s_rows[static_cast<size_t>(kRing) * W], src_rows, kShadowRows * W * 4u, &s_bar[slot]);
            bulk_g2s(&s_task[kRing], src_task, kShadowRows * 8u, &s_bar[slot]);
        }
        ++issued;
    };
    long long paid = 0;
    for (int j0 = 0; j0 < D.T;) {
        const int n = min(32, D.T - j0);
        const int b0 = j0 / kBlockRows;
        if (tid == 0)
            while (issued < b0 + kRingBlocks && issued < n_blocks) issue();
        const int need = min((j0 + 31) / kBlockRows, n_blocks - 1);
        while (ready <= need) { // every thread waits for the blocks it reads
            bar_wait(&s_bar[ready & (kRingBlocks - 1)], (ready / kRingBlocks) & 1);
            ++ready;
        }
        {   // warp w evaluates tasks TPW*w .. TPW*w + TPW-1 of the chunk
            const int r0 = j0 & (kRing - 1);
            const uint32_t* rowp = s_rows + (r0 + warp * TPW) * W + lane;
            const int2* taskp = s_task + r0 + warp * TPW;
            uint32_t any[TPW];
#pragma unroll
            for (int u = 0; u < TPW; ++u) {
                const uint32_t m = rowp[u * W] & s_cap[taskp[u].x][lane];
                any[u] = __ballot_sync(kAll, m != 0);
            }
            if (lane == 0) {
                uint4* dst = reinterpret_cast<uint4*>(s_any + warp * TPW);
#pragma unroll
                for (int q = 0; q < TPW / 4; ++q)
                    dst[q] = make_uint4(any[4 * q], any[4 * q + 1], any[4 * q + 2], any[4 * q + 3]);
            }
        }
        __syncthreads(); // the chunk's ballots are in; every read of s_cap is done
        if (warp == 0) {
            // lane u resolves task j0+u: the lowest lane with a feasible cloud, its lowest bit
            const int rme = (j0 + lane) & (kRing - 1);
            const int2 tk = s_task[rme];
            const int lvme = lane < n ? tk.x : NL;
            int my_c = -1;
            {
                const uint32_t any = s_any[lane];
                if (lane < n && any) {
                    const int src = __ffs(any) - 1;
                    const uint32_t m = s_rows[rme * W + src] & s_cap[lvme][src];
                    my_c = src * 32 + __ffs(m) - 1;
                }
            }
            const bool placed = my_c >= 0;
            int ncommit = n;
            // common case first: take every placed demand off its candidate's free count.  The totals
            // do not depend on the order, and every inclusive prefix fits iff no count went negative.
            if (placed) atomicAdd(&fr[my_c], -tk.y);
            __syncwarp();
            const int fend = placed ? fr[my_c] : 0;
            if (!__any_sync(kAll, fend < 0)) {
                if (placed) { // clear the capacity bits the cloud lost (idempotent across its group)
                    const uint32_t keep = ~(1u << (my_c & 31));
#pragma unroll
                    for (int L = 0; L < NL; ++L)
                        if (fend < lvl[L]) atomicAnd(&s_cap[L][my_c >> 5], keep);
                }
            } else {
                if (placed) atomicAdd(&fr[my_c], tk.y); // undo; commit the exact prefix instead
                __syncwarp();
                // same-candidate groups and the inclusive prefix of their demands (levels: popcounts)
                const uint32_t peers = __match_any_sync(kAll, placed ? my_c : -1 - lane);
                int pre = 0;
#pragma unroll
                for (int L = 0; L < NL; ++L)
                    if (L < D.n_levels) pre += lvl[L] * __popc(peers & le & __ballot_sync(kAll, lvme == L));
                const int f0 = placed ? fr[my_c] : 0;
                const uint32_t fails = __ballot_sync(kAll, placed && f0 < pre);
                ncommit = __ffs(fails) - 1; // >= 1: the first task fits S0
                const uint32_t cmask = (1u << ncommit) - 1u;
                __syncwarp();
                // the last committed member of each group writes its cloud's new free count and
                // clears the capacity bits the cloud lost
                if (placed && lane < ncommit && !(peers & cmask & ~le)) {
                    const int f1 = f0 - pre;
                    fr[my_c] = f1;
                    const uint32_t keep = ~(1u << (my_c & 31));
#pragma unroll
                    for (int L = 0; L < NL; ++L)
                        if (f1 < lvl[L]) atomicAnd(&s_cap[L][my_c >> 5], keep);
                }
            }
            const bool commit = lane < ncommit;
            if (commit) {
                D.target[j0 + lane] = my_c;
                if (!placed) paid += tk.y;
            }
            __syncwarp();
            if (lane == 0) s_j0 = j0 + ncommit;
        }
        __syncthreads(); // the commit and the next start are visible
        j0 = s_j0;
    }
    while (ready < issued) { // drain the bulk copies still in flight (thread 0)
        bar_wait(&s_bar[ready & (kRingBlocks - 1)], (ready / kRingBlocks) & 1);
        ++ready;
    }
    if (warp == 0) {
#pragma unroll
        for (int o = 16; o; o >>= 1) paid += __shfl_xor_sync(kAll, paid, o);
        __syncwarp();
        for (int c = lane; c < D.K; c += 32) D.free_vms[c] = fr[c];
        if (lane == 0) *D.paid = paid;
    }
}

struct HostGreedy {
    int K, T, W, n_levels;
    std::vector<int32_t> levels;
    size_t smem;
};

HostGreedy plan_greedy(const vcs_instance* in) {
    HostGreedy h{};
    h.K = in->n_clouds;
    h.T = in->n_tasks;
    h.W = std::max(1, (h.K + 31) / 32);
    // distinct demands (at most kMaxLevels, else the generic capacity test).  Branch-free
    // passes: min/max, then a 64-bit presence bitmap when the range allows it (random demands
    // would mispredict a compare-per-task scan); otherwise a short table scan.
    const int32_t* dem = in->task_demand;
    std::vector<int32_t> lv;
    bool small = true;
    if (h.T) {
        int32_t lo = dem[0], hi = dem[0];
        for (int j = 1; j < h.T; ++j) {
            lo = std::min(lo, dem[j]);
            hi = std::max(hi, dem[j]);
        }
        if (static_cast<int64_t>(hi) - lo < 64) {
            uint64_t bits = 0;
            for (int j = 0; j < h.T; ++j) bits |= uint64_t(1) << (dem[j] - lo);
            for (int b = 0; b < 64; ++b)
                if (bits >> b & 1) lv.push_back(lo + b);
            small = static_cast<int>(lv.size()) <= kMaxLevels;
        } else {
            for (int j = 0; j < h.T && small; ++j)
                if (std::find(lv.begin(), lv.end(), dem[j]) == lv.end()) {
                    lv.push_back(dem[j]);
                    small = static_cast<int>(lv.size()) <= kMaxLevels;
                }
            std::sort(lv.begin(), lv.end());
        }
    }
    if (small) {
        h.levels = lv;
        h.n_levels = static_cast<int>(lv.size());
    }
    if (h.W <= 32 && h.n_levels > 0 && h.n_levels <= kFastLevels)
        h.W = 32; // fast path: attribute rows at stride 32 (zero words past ceil(K/32))
    h.smem = static_cast<size_t>(h.K) * 4 + static_cast<size_t>(h.n_levels) * h.W * 4;
    if (h.smem > 200 * 1024)
        raise(VCS_EINVAL, "too many clouds for the device first-fit (shared-memory bound)");
    return h;
}

// Device staging of one instance for the greedy kernels.
struct GreedyDev {
    DevBuf<double> c_delay, c_thr, t_delay, t_thr;
    DevBuf<uint32_t> mask;
    DevBuf<int2> task;
    DevBuf<int32_t> demand, levels, free_vms, target;
    DevBuf<long long> paid;
};

void stage(const vcs_instance* in, const HostGreedy& h, GreedyDev& g, cudaStream_t s) {
    const size_t K = static_cast<size_t>(h.K), T = static_cast<size_t>(h.T);
    g.c_delay.exact(K, s);
    g.c_thr.exact(K, s);
    g.t_delay.exact(T, s);
    g.t_thr.exact(T, s);
    const size_t T_pad = (T + kBlockRows - 1) / kBlockRows * kBlockRows; // whole bulk-copy blocks
    g.mask.exact(std::max<size_t>(T_pad, 1) * static_cast<size_t>(h.W), s);
    g.task.exact(std::max<size_t>(T_pad, 1), s);
    if (T_pad > T) {
        VCS_CUDA(cudaMemsetAsync(g.mask.p + T * h.W, 0, (T_pad - T) * h.W * 4, s));
        VCS_CUDA(cudaMemsetAsync(g.task.p + T, 0, (T_pad - T) * sizeof(int2), s));
    }
    g.demand.exact(std::max<size_t>(T, 1), s);
    g.levels.exact(std::max<size_t>(1, h.levels.size()), s);
    g.free_vms.exact(K, s);
    g.target.exact(T, s);
    g.paid.exact(1, s);
    if (K) {
        VCS_CUDA(cudaMemcpyAsync(g.c_delay.p, in->cloud_delay_ms, K * 8, cudaMemcpyHostToDevice, s));
        VCS_CUDA(cudaMemcpyAsync(g.c_thr.p, in->cloud_thr_kbps, K * 8, cudaMemcpyHostToDevice, s));
        VCS_CUDA(cudaMemcpyAsync(g.free_vms.p, in->cloud_vm_free, K * 4, cudaMemcpyHostToDevice, s));
    }
    if (T) {
        VCS_CUDA(cudaMemcpyAsync(g.t_delay.p, in->task_max_delay_ms, T * 8, cudaMemcpyHostToDevice, s));
        VCS_CUDA(cudaMemcpyAsync(g.t_thr.p, in->task_min_thr_kbps, T * 8, cudaMemcpyHostToDevice, s));
        VCS_CUDA(cudaMemcpyAsync(g.demand.p, in->task_demand, T * 4, cudaMemcpyHostToDevice, s));
    }
    if (!h.levels.empty())
        VCS_CUDA(cudaMemcpyAsync(g.levels.p, h.levels.data(), h.levels.size() * 4,
                                 cudaMemcpyHostToDevice, s));
}

void launch_mask(const HostGreedy& h, GreedyDev& g, int sms, cudaStream_t s) {
    if (!h.T) return;
    const uint64_t blocks = std::min<uint64_t>((static_cast<uint64_t>(h.T) + 7) / 8,
                                               static_cast<uint64_t>(sms) * 16);
    k_attr_mask<<<static_cast<unsigned>(std::max<uint64_t>(1, blocks)), 256, 0, s>>>(
        h.K, h.T, h.W, g.c_delay.p, g.c_thr.p, g.t_delay.p, g.t_thr.p, g.mask.p, g.demand.p,
        g.levels.p, h.n_levels, g.task.p);
    VCS_LAUNCHED();
}

GreedyDesc desc_of(const HostGreedy& h, GreedyDev& g) {
    return GreedyDesc{h.K, h.T, h.W, h.n_levels, g.mask.p, g.task.p, g.levels.p,
                      g.free_vms.p, g.target.p, g.paid.p};
}

bool fast_path(const HostGreedy& h) {
    return h.W <= 32 && h.n_levels > 0 && h.n_levels <= kFastLevels;
}

void launch_first_fit(const GreedyDesc* d_descs, int n, size_t smem, bool fast, size_t max_k,
                      int max_levels, cudaStream_t s) {
    if (fast) {
        static const bool serial = std::getenv("VCS_GREEDY_SERIAL") != nullptr;
        const size_t fs = serial ? std::max<size_t>(max_k * 4, 4) : spec_smem_bytes(max_k);
        auto go = [&](auto kern) {
            VCS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(fs)));
            kern<<<n, 32, fs, s>>>(d_descs);
        };
        auto go4 = [&](auto kern) {
            VCS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(fs)));
            kern<<<n, kSpecWarps * 32, fs, s>>>(d_descs);
        };
        if (serial) {
            if (max_levels <= 1) go(k_first_fit_fast<1>);
            else if (max_levels <= 2) go(k_first_fit_fast<2>);
            else if (max_levels <= 3) go(k_first_fit_fast<3>);
            else if (max_levels <= 4) go(k_first_fit_fast<4>);
            else go(k_first_fit_fast<kFastLevels>);
        } else if (std::getenv("VCS_GREEDY_1WARP")) {
            if (max_levels <= 1) go(k_first_fit_spec<1>);
            else if (max_levels <= 2) go(k_first_fit_spec<2>);
            else if (max_levels <= 3) go(k_first_fit_spec<3>);
            else if (max_levels <= 4) go(k_first_fit_spec<4>);
            else go(k_first_fit_spec<kFastLevels>);
        } else {
            if (max_levels <= 1) go4(k_first_fit_spec4<1, kSpecWarps>);
            else if (max_levels <= 2) go4(k_first_fit_spec4<2, kSpecWarps>);
            else if (max_levels <= 3) go4(k_first_fit_spec4<3, kSpecWarps>);
            else if (max_levels <= 4) go4(k_first_fit_spec4<4, kSpecWarps>);
            else go4(k_first_fit_spec4<kFastLevels, kSpecWarps>);
        }
    } else {
        VCS_CUDA(cudaFuncSetAttribute(k_first_fit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(std::max<size_t>(smem, 1))));
        k_first_fit<<<n, 32, std::max<size_t>(smem, 4), s>>>(d_descs);
    }
    VCS_LAUNCHED();
}

} // namespace
} // namespace vcs

using vcs::guarded;
using vcs::raise;

extern "C" {

int vcs_greedy(const vcs_instance* in, int device, int32_t* target_per_task,
               int64_t* per_cloud_used, int64_t* paid, int64_t* unused) {
    return guarded([&] {
        vcs::bind_device(device);
        const bool tr = vcs::trace_enabled();
        const double t0 = tr ? vcs::host_ms() : 0.0;
        const vcs::HostGreedy h = vcs::plan_greedy(in);
        const double t1 = tr ? vcs::host_ms() : 0.0;
        cudaStream_t s = vcs::acquire_stream(device);
        struct StreamGuard { // (back to the pool once the stream-ordered frees ran)
            cudaStream_t s;
            int device;
            ~StreamGuard() {
                cudaStreamSynchronize(s);
                vcs::release_stream(device, s);
            }
        } guard{s, device};
        vcs::GreedyDev g;
        vcs::stage(in, h, g, s);
        vcs::launch_mask(h, g, vcs::sm_count(device), s);
        vcs::DevBuf<vcs::GreedyDesc> dd;
        dd.exact(1, s);
        const vcs::GreedyDesc desc = vcs::desc_of(h, g);
        VCS_CUDA(cudaMemcpyAsync(dd.p, &desc, sizeof desc, cudaMemcpyHostToDevice, s));
        vcs::launch_first_fit(dd.p, 1, h.smem, vcs::fast_path(h), static_cast<size_t>(h.K),
                              h.n_levels, s);
        const double t2 = tr ? vcs::host_ms() : 0.0;
        std::vector<int32_t> free_out(static_cast<size_t>(h.K));
        long long p = 0;
        if (h.T)
            VCS_CUDA(cudaMemcpyAsync(target_per_task, g.target.p, static_cast<size_t>(h.T) * 4,
                                     cudaMemcpyDeviceToHost, s));
        if (h.K)
            VCS_CUDA(cudaMemcpyAsync(free_out.data(), g.free_vms.p, static_cast<size_t>(h.K) * 4,
                                     cudaMemcpyDeviceToHost, s));
        VCS_CUDA(cudaMemcpyAsync(&p, g.paid.p, sizeof p, cudaMemcpyDeviceToHost, s));
        const double t3 = tr ? vcs::host_ms() : 0.0;
        VCS_CUDA(cudaStreamSynchronize(s));
        const double t4 = tr ? vcs::host_ms() : 0.0;
        if (tr)
            std::fprintf(stderr, "[vcs] greedy T=%d K=%d: plan %.3f ms, stage+enqueue %.3f, d2h enqueue %.3f, sync %.3f\n",
                         h.T, h.K, t1 - t0, t2 - t1, t3 - t2, t4 - t3);
        int64_t placed = 0, capacity = 0;
        for (int c = 0; c < h.K; ++c) {
            const int64_t used = static_cast<int64_t>(in->cloud_vm_free[c]) - free_out[c];
            if (per_cloud_used) per_cloud_used[c] = used;
            placed += used;
            capacity += in->cloud_vm_total[c];
        }
        *paid = h.T ? p : 0;
        *unused = capacity - placed; // greedy.cpp:28: total_capacity - vc_placed
        return VCS_OK;
    });
}

int vcs_greedy_batch(int32_t n, const vcs_instance* insts, int device, int32_t** target_per_task,
                     int64_t* paid, int64_t* unused) {
    return guarded([&] {
        if (n <= 0) return VCS_OK;
        vcs::bind_device(device);
        cudaStream_t s = vcs::acquire_stream(device);
        struct StreamGuard { // (back to the pool once the stream-ordered frees ran)
            cudaStream_t s;
            int device;
            ~StreamGuard() {
                cudaStreamSynchronize(s);
                vcs::release_stream(device, s);
            }
        } guard{s, device};
        std::vector<vcs::HostGreedy> hs;
        std::vector<std::unique_ptr<vcs::GreedyDev>> gs;
        std::vector<vcs::GreedyDesc> descs;
        size_t smem = 4, max_k = 1;
        bool fast = true;
        int max_levels = 1;
        const int sms = vcs::sm_count(device);
        for (int i = 0; i < n; ++i) {
            hs.push_back(vcs::plan_greedy(&insts[i]));
            gs.push_back(std::make_unique<vcs::GreedyDev>());
            vcs::stage(&insts[i], hs.back(), *gs.back(), s);
            vcs::launch_mask(hs.back(), *gs.back(), sms, s);
            descs.push_back(vcs::desc_of(hs.back(), *gs.back()));
            smem = std::max(smem, hs.back().smem);
            max_k = std::max(max_k, static_cast<size_t>(hs.back().K));
            fast = fast && vcs::fast_path(hs.back());
            max_levels = std::max(max_levels, hs.back().n_levels);
        }
        vcs::DevBuf<vcs::GreedyDesc> dd;
        dd.exact(static_cast<size_t>(n), s);
        VCS_CUDA(cudaMemcpyAsync(dd.p, descs.data(), descs.size() * sizeof(vcs::GreedyDesc),
                                 cudaMemcpyHostToDevice, s));
        vcs::launch_first_fit(dd.p, n, smem, fast, max_k, max_levels, s);
        std::vector<std::vector<int32_t>> frees(static_cast<size_t>(n));
        std::vector<long long> ps(static_cast<size_t>(n), 0);
        for (int i = 0; i < n; ++i) {
            const auto& h = hs[static_cast<size_t>(i)];
            frees[i].resize(static_cast<size_t>(h.K));
            if (h.T)
                VCS_CUDA(cudaMemcpyAsync(target_per_task[i], gs[i]->target.p,
                                         static_cast<size_t>(h.T) * 4, cudaMemcpyDeviceToHost, s));
            if (h.K)
                VCS_CUDA(cudaMemcpyAsync(frees[i].data(), gs[i]->free_vms.p,
                                         static_cast<size_t>(h.K) * 4, cudaMemcpyDeviceToHost, s));
            VCS_CUDA(cudaMemcpyAsync(&ps[i], gs[i]->paid.p, sizeof(long long), cudaMemcpyDeviceToHost, s));
        }
        VCS_CUDA(cudaStreamSynchronize(s));
        for (int i = 0; i < n; ++i) {
            const vcs_instance& in = insts[i];
            int64_t placed = 0, capacity = 0;
            for (int c = 0; c < in.n_clouds; ++c) {
                placed += static_cast<int64_t>(in.cloud_vm_free[c]) - frees[i][c];
                capacity += in.cloud_vm_total[c];
            }
            paid[i] = in.n_tasks ? ps[i] : 0;
            unused[i] = capacity - placed;
        }
        return VCS_OK;
    });
}

} // extern "C"
