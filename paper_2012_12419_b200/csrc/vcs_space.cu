// vcs_space.cu — the GPU state-space builder (replaces StateSpace::build, mdp.cpp:81-214),
// the device key index behind locate (mdp.cpp:227-234), and the space handle.
//
// Layered frontier expansion, one layer (decision epoch) at a time:
//   1. scan        out-degree of every frontier state (feasible active clouds + paid, computed
//                  inside the scan's input iterator) -> CSR row offsets (edge order of the
//                  reference: clouds ascending, paid last, mdp.cpp:169-204)
//   2. k_emit      per edge: successor, fp64 reward (separate mul/sub, no FMA, = mdp.cpp:191/202
//                  bits), action.  Each successor gets a table slot that keeps the MINIMUM edge
//                  index carrying it (atomicMin) = its first occurrence in the reference's BFS:
//                  dense path (small key space): slot = the successor's mixed-radix index,
//                  written by k_emit itself into an L2-resident table;
//                  hash path: k_emit writes packed successor keys, k_insert hashes them.
//   3. scan        a successor's layer-local index is the rank of its first edge among all
//                  first edges (flags computed inside the scan's input iterator) -> exactly the
//                  reference's first-insertion order (mdp.cpp:157-165)
//   4. k_finalize  successor indices + next-frontier keys
// Keys are the reference's reduced keys (free counts of still-eligible clouds, mdp.hpp:70-79)
// packed into 64-bit words, ceil(log2(vm_free+1)) bits per cloud.
#include "vcs_device.cuh"
#include "vcs_keys.cuh"

#include <cooperative_groups.h>
#include <math_constants.h>
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

namespace vcs {

namespace {

// Out-degree of frontier state i (the paid edge always exists), 0 past the frontier: the input
// of the row-offset scan.
// (The layer's parameters are read through a pointer: a functor holding the ~1.3 KB struct by
// value would be copied to local memory inside the scan kernel.)
template <int WM>
struct DegreeOp {
    const uint64_t* keys;
    uint32_t n;
    const LayerParam* L;
    __device__ uint32_t operator()(uint32_t i) const {
        if (i >= n) return 0u;
        const int words = L->words, n_active = L->n_active, demand = L->demand;
        uint64_t k[WM];
        load_key<WM>(keys + static_cast<uint64_t>(i) * words, words, k);
        uint32_t d = 1;
        for (int p = 0; p < n_active; ++p)
            if (L->attr[p] && get_field<WM>(k, L->bit_off[p], L->width[p]) >= demand) ++d;
        return d;
    }
};

// flag(j) = 1 iff edge j is the first occurrence of its successor (the table slot holds the
// minimum edge index); 0 past E_t, so a scan over the launch bound gives rank[E_t] = n_{t+1}.
struct FirstEdgeOp {
    const uint32_t* n_edges_dev;
    const uint32_t* table;
    const uint32_t* slot_of;
    __device__ uint32_t operator()(uint32_t j) const {
        return j < *n_edges_dev && table[slot_of[j]] == j ? 1u : 0u;
    }
};

// One edge: successor key in the layer-(t+1) packing, reward, action.  `p` = key position of
// the chosen cloud, or -1 for the paid cloud.
template <int WM>
__device__ __forceinline__ void emit_edge(const uint64_t (&k)[WM], int p, const LayerParam& L,
                                          uint64_t* __restrict__ ekey, double* __restrict__ rw,
                                          int32_t* __restrict__ act) {
    uint64_t nk[WM];
#pragma unroll
    for (int i = 0; i < WM; ++i) nk[i] = 0ull;
    double retired = 0.0; // mdp.cpp:179-185 / :196-197, summed in key-position order
    for (int q = 0; q < L.n_active; ++q) {
        int v = get_field<WM>(k, L.bit_off[q], L.width[q]);
        if (q == p) v -= L.demand;
        if (L.keep_idx[q] >= 0)
            put_field<WM>(nk, L.next_bit_off[q], static_cast<uint64_t>(v));
        else
            retired = __dadd_rn(retired, static_cast<double>(v));
    }
#pragma unroll
    for (int i = 0; i < WM; ++i)
        if (i < L.next_words) ekey[i] = nk[i];
    // beta*n - gamma*retired as two rounded operations (the reference's -O3 x86-64 code has no
    // FMA; nvcc would contract a*b-c*d, so the intrinsics pin the rounding).
    const double base = p < 0 ? L.r_paid : L.r_cloud;
    *rw = __dsub_rn(base, __dmul_rn(L.gamma, retired));
    *act = p < 0 ? -1 : L.cloud[p];
}

// Dense path: the successor of an edge is identified by its mixed-radix index; the first-edge
// table (dense_size entries, L2-resident) is updated right here.  idx(paid successor) =
// sum over kept fields of f_p * W_p; a cloud action subtracts demand * W_p when p is kept.
// (Staging the block's edges in shared memory for coalesced stores measured slower: the
// strided stores merge in L2.)
template <int WM>
__global__ void k_emit_dense(uint32_t n, const uint64_t* __restrict__ keys,
                             const uint32_t* __restrict__ off, const LayerParam L,
                             uint32_t edge_base, uint32_t* __restrict__ row_ptr_layer,
                             uint32_t* __restrict__ eidx, double* __restrict__ reward,
                             int32_t* __restrict__ action, uint32_t* __restrict__ first_edge) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t k[WM];
    load_key<WM>(keys + static_cast<uint64_t>(i) * L.words, L.words, k);
    uint32_t j = off[i];
    row_ptr_layer[i] = edge_base + j;
    uint32_t base = 0;
    for (int p = 0; p < L.n_active; ++p)
        if (L.keep_idx[p] >= 0)
            base += static_cast<uint32_t>(get_field<WM>(k, L.bit_off[p], L.width[p])) * L.wnext[p];
    const bool retires = L.n_keep != L.n_active;
    auto put = [&](uint32_t idx, double r, int32_t a) {
        eidx[j] = idx;
        reward[edge_base + j] = r;
        action[edge_base + j] = a;
        // (the check reads L2: an SM's L1 copy of a hot entry, e.g. the single terminal state's,
        // would stay stale and let every edge through to the serialised atomic)
        if (__ldcg(first_edge + idx) > j) atomicMin(&first_edge[idx], j);
        ++j;
    };
    for (int p = 0; p < L.n_active; ++p) {
        if (!L.attr[p] || get_field<WM>(k, L.bit_off[p], L.width[p]) < L.demand) continue;
        const uint32_t idx =
            L.keep_idx[p] >= 0 ? base - static_cast<uint32_t>(L.demand) * L.wnext[p] : base;
        put(idx, retires ? retiring_reward<WM>(k, p, L) : L.r_cloud_kept, L.cloud[p]);
    }
    put(base, retires ? retiring_reward<WM>(k, -1, L) : L.r_paid_kept, -1);
}

template <int WM>
__global__ void k_emit(uint32_t n, const uint64_t* __restrict__ keys,
                       const uint32_t* __restrict__ off, const LayerParam L, uint32_t edge_base,
                       uint32_t* __restrict__ row_ptr_layer, uint64_t* __restrict__ ekeys,
                       double* __restrict__ reward, int32_t* __restrict__ action) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t k[WM];
    load_key<WM>(keys + static_cast<uint64_t>(i) * L.words, L.words, k);
    uint32_t j = off[i];
    row_ptr_layer[i] = edge_base + j;
    if (L.n_keep == L.n_active) {
        // No cloud retires at this transition (the common case): the next key has the same
        // layout, a cloud action subtracts the demand from its own field, nothing is charged
        // (reward = base - gamma * 0.0, evaluated on the host with the same two IEEE ops).
        for (int p = 0; p < L.n_active; ++p) {
            if (!L.attr[p] || get_field<WM>(k, L.bit_off[p], L.width[p]) < L.demand) continue;
            uint64_t* ek = ekeys + static_cast<uint64_t>(j) * L.next_words;
            const int w = L.bit_off[p] >> 6;
            const uint64_t sub = static_cast<uint64_t>(L.demand) << (L.bit_off[p] & 63);
#pragma unroll
            for (int q = 0; q < WM; ++q)
                if (q < L.next_words) ek[q] = q == w ? k[q] - sub : k[q];
            reward[edge_base + j] = L.r_cloud_kept;
            action[edge_base + j] = L.cloud[p];
            ++j;
        }
        uint64_t* ek = ekeys + static_cast<uint64_t>(j) * L.next_words;
#pragma unroll
        for (int q = 0; q < WM; ++q)
            if (q < L.next_words) ek[q] = k[q];
        reward[edge_base + j] = L.r_paid_kept;
        action[edge_base + j] = -1;
        return;
    }
    for (int p = 0; p < L.n_active; ++p) {
        if (!L.attr[p] || get_field<WM>(k, L.bit_off[p], L.width[p]) < L.demand) continue;
        emit_edge<WM>(k, p, L, ekeys + static_cast<uint64_t>(j) * L.next_words,
                      reward + edge_base + j, action + edge_base + j);
        ++j;
    }
    emit_edge<WM>(k, -1, L, ekeys + static_cast<uint64_t>(j) * L.next_words,
                  reward + edge_base + j, action + edge_base + j);
}

template <int WM>
__global__ void k_insert(const uint32_t* __restrict__ n_edges_dev, const uint64_t* __restrict__ ekeys,
                         int words, uint32_t* __restrict__ table, uint32_t mask,
                         uint32_t* __restrict__ slot_of) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= *n_edges_dev) return;
    uint64_t k[WM];
    load_key<WM>(ekeys + static_cast<uint64_t>(j) * words, words, k);
    uint32_t h = static_cast<uint32_t>(hash_key<WM>(k, words, 0)) & mask;
    for (;;) {
        uint32_t cur = table[h];
        if (cur == kEmpty32) {
            const uint32_t prev = atomicCAS(&table[h], kEmpty32, j);
            if (prev == kEmpty32) {
                slot_of[j] = h;
                return;
            }
            cur = prev;
        }
        if (key_equal<WM>(ekeys + static_cast<uint64_t>(cur) * words, words, k)) {
            // keep the first occurrence (lowest edge index); skip the atomic when a smaller
            // index is already there (heavily shared successors, e.g. the single terminal
            // state, would otherwise serialise on one address)
            if (cur > j) atomicMin(&table[h], j);
            slot_of[j] = h;
            return;
        }
        h = (h + 1) & mask;
    }
}

// Single-word keys narrower than 64 bits (so ~0 is never a key): the table stores the key next
// to the first-edge index, so an insert never re-reads another edge's key.
constexpr uint64_t kEmptyKey = ~0ull;

__global__ void k_insert_kv(const uint32_t* __restrict__ n_edges_dev,
                            const uint64_t* __restrict__ ekeys, unsigned long long* __restrict__ tkey,
                            uint32_t* __restrict__ tidx, uint32_t mask,
                            uint32_t* __restrict__ slot_of) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= *n_edges_dev) return;
    const uint64_t k = ekeys[j];
    uint64_t kk[1] = {k};
    uint32_t h = static_cast<uint32_t>(hash_key<1>(kk, 1, 0)) & mask;
    for (;;) {
        unsigned long long cur = tkey[h];
        if (cur == kEmptyKey) cur = atomicCAS(&tkey[h], kEmptyKey, static_cast<unsigned long long>(k));
        if (cur == kEmptyKey || cur == k) break; // claimed the slot, or the key is already there
        h = (h + 1) & mask;
    }
    if (__ldcg(tidx + h) > j) atomicMin(&tidx[h], j); // the first occurrence (lowest edge index) wins
    slot_of[j] = h;
}

__global__ void k_finalize(const uint32_t* __restrict__ n_edges_dev, const uint32_t* __restrict__ table,
                           const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ rank,
                           const uint64_t* __restrict__ ekeys, int words, uint32_t next_base,
                           uint32_t* __restrict__ succ, uint64_t* __restrict__ next_keys) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= *n_edges_dev) return;
    const uint32_t first = table[slot_of[j]];
    succ[j] = next_base + rank[first];
    if (first == j) {
        const uint64_t* src = ekeys + static_cast<uint64_t>(j) * words;
        uint64_t* dst = next_keys + static_cast<uint64_t>(rank[j]) * words;
        for (int w = 0; w < words; ++w) dst[w] = src[w];
    }
}

// Dense path: successor indices; a first edge also writes its successor's packed key, decoded
// from the mixed-radix index.
template <int WM>
__global__ void k_finalize_dense(const uint32_t* __restrict__ n_edges_dev,
                                 const uint32_t* __restrict__ first_edge,
                                 const uint32_t* __restrict__ eidx, const uint32_t* __restrict__ rank,
                                 const LayerParam L, uint32_t next_base,
                                 uint32_t* __restrict__ succ, uint64_t* __restrict__ next_keys) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= *n_edges_dev) return;
    const uint32_t idx = eidx[j];
    const uint32_t first = first_edge[idx];
    succ[j] = next_base + rank[first];
    if (first != j) return;
    uint64_t nk[WM];
#pragma unroll
    for (int w = 0; w < WM; ++w) nk[w] = 0ull;
    for (int p = 0; p < L.n_active; ++p)
        if (L.keep_idx[p] >= 0)
            put_field<WM>(nk, L.next_bit_off[p], (idx / L.wnext[p]) % L.radix[p]);
    uint64_t* dst = next_keys + static_cast<uint64_t>(rank[j]) * L.next_words;
#pragma unroll
    for (int w = 0; w < WM; ++w)
        if (w < L.next_words) dst[w] = nk[w];
}

__global__ void k_fill_u32(uint32_t* __restrict__ p, uint64_t n, uint32_t v) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

// ---- locate index: one open-addressing table over (layer, key) -> flat state index ----------
template <int WM>
__global__ void k_loc_insert(uint32_t n, const uint64_t* __restrict__ keys, int words, int layer,
                             uint32_t base, uint32_t* __restrict__ table, uint32_t mask) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t k[WM];
    load_key<WM>(keys + static_cast<uint64_t>(i) * words, words, k);
    uint32_t h = static_cast<uint32_t>(hash_key<WM>(k, words, static_cast<uint64_t>(layer) + 1)) &
                 mask;
    while (atomicCAS(&table[h], kEmpty32, base + i) != kEmpty32) h = (h + 1) & mask;
}

struct LocQuery {
    int32_t layer;
    int32_t words;
    int32_t valid;
    int32_t pad;
    uint64_t key[kMaxKeyWords];
};

template <int WM>
__global__ void k_loc_lookup(int64_t n, const LocQuery* __restrict__ q,
                             const uint64_t* __restrict__ keys,
                             const uint64_t* __restrict__ layer_off,
                             const uint64_t* __restrict__ key_off,
                             const uint32_t* __restrict__ table, uint32_t mask,
                             int64_t* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const LocQuery& Q = q[i];
    if (!Q.valid) {
        out[i] = -1;
        return;
    }
    uint64_t k[WM];
#pragma unroll
    for (int w = 0; w < WM; ++w) k[w] = Q.key[w];
    const int t = Q.layer;
    uint32_t h = static_cast<uint32_t>(hash_key<WM>(k, Q.words, static_cast<uint64_t>(t) + 1)) &
                 mask;
    const uint64_t lo = layer_off[t], hi = layer_off[t + 1];
    for (;;) {
        const uint32_t cur = table[h];
        if (cur == kEmpty32) {
            out[i] = -1;
            return;
        }
        if (cur >= lo && cur < hi &&
            key_equal<WM>(keys + key_off[t] + (cur - lo) * static_cast<uint64_t>(Q.words),
                          Q.words, k)) {
            out[i] = cur;
            return;
        }
        h = (h + 1) & mask;
    }
}

// ---- batched policy queries: value_of / action_for over many full states ----
// Per layer t = 0..H: the packed-key layout (active clouds, bit offsets, widths), so keys are
// packed on the device from the callers' free-VM vectors.
struct QueryLayer {
    int32_t n_active;
    int32_t words;
    uint8_t cloud[kMaxActive];
    uint16_t bit_off[kMaxActive];
    uint8_t width[kMaxActive];
};

struct QueryArgs {
    const QueryLayer* layers; // H+1
    const int32_t* last_use;  // per cloud (hidden penalty, mdp.cpp:236-243)
    const uint64_t* layer_off;
    const uint64_t* key_off;
    const uint64_t* keys;
    const uint32_t* table;
    uint32_t mask;
    const double* values;     // V_{K*} of the last solve
    const int32_t* actions;
    const int32_t* free_vms;  // n x n_clouds
    const int32_t* task_index;
    const uint8_t* terminal;
    double* value_out;
    int32_t* action_out;
    int64_t* idx_out;
    int64_t n;
    int32_t n_clouds;
    int32_t H;
    double gamma;
};

template <int WM>
__global__ void k_policy_query(QueryArgs a) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    const int32_t* fv = a.free_vms + i * a.n_clouds;
    const bool term = a.terminal[i] != 0;
    const int t = term ? a.H : a.task_index[i];
    int64_t idx = -1;
    double penalty = 0.0;
    if (t >= 0 && t <= a.H) {
        const QueryLayer& Q = a.layers[t];
        uint64_t k[WM];
#pragma unroll
        for (int w = 0; w < WM; ++w) k[w] = 0ull;
        bool ok = true;
        for (int p = 0; p < Q.n_active; ++p) { // pack_key (vcs_host.cpp)
            const int v = fv[Q.cloud[p]];
            if (v < 0 || v > 0xffff || (Q.width[p] < 31 && v >= (1 << Q.width[p]))) ok = false;
            put_field<WM>(k, Q.bit_off[p], static_cast<uint64_t>(v < 0 ? 0 : v));
        }
        if (ok) {
            uint32_t h = static_cast<uint32_t>(hash_key<WM>(k, Q.words, static_cast<uint64_t>(t) + 1)) &
                         a.mask;
            const uint64_t lo = a.layer_off[t], hi = a.layer_off[t + 1];
            for (;;) {
                const uint32_t cur = a.table[h];
                if (cur == kEmpty32) break;
                if (cur >= lo && cur < hi &&
                    key_equal<WM>(a.keys + a.key_off[t] + (cur - lo) * static_cast<uint64_t>(Q.words),
                                  Q.words, k)) {
                    idx = cur;
                    break;
                }
                h = (h + 1) & a.mask;
            }
        }
        if (a.H > 0) { // (the host's exact operations: no contraction into an FMA)
            double retired = 0.0;
            for (int c = 0; c < a.n_clouds; ++c)
                if (a.last_use[c] < t) retired = __dadd_rn(retired, static_cast<double>(fv[c]));
            penalty = __dmul_rn(a.gamma, retired);
        }
    }
    if (a.idx_out) a.idx_out[i] = idx;
    if (a.value_out) a.value_out[i] = idx >= 0 ? __dsub_rn(a.values[idx], penalty) : CUDART_NAN;
    if (a.action_out)
        a.action_out[i] = (idx >= 0 && !term && t < a.H) ? a.actions[idx] : VCS_NO_ACTION;
}

// rollout (mdp.cpp:305-324) on the device: ONE thread applies the policy from the initial
// state: pack the layer-t key of the current free counts, locate it in the device key index,
// read the last solve's action, apply the transition (free[a] -= demand).  status: 0 ok, 1 a
// visited state is not in the enumerated space (the reference throws std::out_of_range).
template <int WM>
__global__ void k_rollout(QueryArgs a, const int32_t* __restrict__ demand, int32_t* fv,
                          int32_t* targets, int32_t* status) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    for (int c = 0; c < a.n_clouds; ++c) fv[c] = a.free_vms[c];
    for (int t = 0; t < a.H; ++t) {
        const QueryLayer& Q = a.layers[t];
        uint64_t k[WM];
#pragma unroll
        for (int w = 0; w < WM; ++w) k[w] = 0ull;
        for (int p = 0; p < Q.n_active; ++p)
            put_field<WM>(k, Q.bit_off[p], static_cast<uint64_t>(fv[Q.cloud[p]]));
        uint32_t h = static_cast<uint32_t>(hash_key<WM>(k, Q.words, static_cast<uint64_t>(t) + 1)) & a.mask;
        const uint64_t lo = a.layer_off[t], hi = a.layer_off[t + 1];
        int64_t idx = -1;
        for (;;) {
            const uint32_t cur = a.table[h];
            if (cur == kEmpty32) break;
            if (cur >= lo && cur < hi &&
                key_equal<WM>(a.keys + a.key_off[t] + (cur - lo) * static_cast<uint64_t>(Q.words),
                              Q.words, k)) {
                idx = cur;
                break;
            }
            h = (h + 1) & a.mask;
        }
        if (idx < 0) {
            *status = 1;
            return;
        }
        const int32_t act = a.actions[idx];
        targets[t] = act;
        if (act >= 0) fv[act] -= demand[t];
    }
    *status = 0;
}

// The same walk without a key index (no locate table to build): on an explicit CSR the
// successor under action a is the row's edge carrying a (edges are one per action); on the
// implicit form the state's index is the rank table entry of its key-space index
// d = sum_p free[cloud_p] * W_p.
__global__ void k_rollout_csr(const uint32_t* __restrict__ row_ptr, const uint32_t* __restrict__ succ,
                              const int32_t* __restrict__ action, const int32_t* __restrict__ actions,
                              int H, int32_t* targets, int32_t* status) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    uint32_t s = 0; // the initial state is the root (mdp.cpp:81-92)
    for (int t = 0; t < H; ++t) {
        const int32_t a = actions[s];
        targets[t] = a;
        const uint32_t eb = row_ptr[s], ee = row_ptr[s + 1];
        uint32_t nxt = 0xffffffffu;
        for (uint32_t e = eb; e < ee; ++e)
            if (action[e] == a) {
                nxt = succ[e];
                break;
            }
        if (nxt == 0xffffffffu) {
            *status = 1;
            return;
        }
        s = nxt;
    }
    *status = 0;
}

__global__ void k_rollout_rank(const LayerParam* __restrict__ params, const uint32_t* __restrict__ rank_tables,
                               const uint64_t* __restrict__ rank_off, const uint64_t* __restrict__ layer_off,
                               const int32_t* __restrict__ actions, const int32_t* __restrict__ demand,
                               int32_t* fv, int H, int32_t* targets, int32_t* status) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    uint64_t idx = 0; // the root
    for (int t = 0; t < H; ++t) {
        if (t > 0) {
            const LayerParam& L = params[t]; // layer t's own numbering (wself)
            uint64_t d = 0;
            for (int p = 0; p < L.n_active; ++p)
                d += static_cast<uint64_t>(fv[L.cloud[p]]) * L.wself[p];
            const uint32_t r = rank_tables[rank_off[t - 1] + d];
            if (r == kEmpty32) {
                *status = 1;
                return;
            }
            idx = layer_off[t] + r;
        }
        const int32_t a = actions[idx];
        targets[t] = a;
        if (a >= 0) fv[a] -= demand[t];
    }
    *status = 0;
}

uint32_t blocks_for(uint64_t n, uint32_t threads) {
    return static_cast<uint32_t>((n + threads - 1) / threads);
}

uint64_t pow2_at_least(uint64_t n) {
    uint64_t c = 1024;
    while (c < n) c <<= 1;
    return c;
}

// Device-side layer counters written by k_counters into mapped pinned host memory, so a layer
// needs exactly one host synchronisation (to size the next layer's launches and buffers).
struct LayerCounters {
    uint32_t n_edges; // E_t
    uint32_t n_next;  // n_{t+1}
};

__global__ void k_counters(const uint32_t* __restrict__ off_end, const uint32_t* __restrict__ rank,
                           LayerCounters* __restrict__ out) {
    const uint32_t e = *off_end;
    out->n_edges = e;
    out->n_next = rank[e];
}

// Mapped pinned counter blocks are recycled across builds (a cudaHostAlloc costs far more than
// a whole small layer).
std::mutex g_counters_mu;
std::vector<LayerCounters*> g_counters_free;

struct Scratch {
    DevBuf<uint32_t> off, slot, rank, table, eidx;
    DevBuf<unsigned long long> edge_count; // (pull form) E_t
    DevBuf<uint64_t> ekeys, tkey;
    DevBuf<LayerParam> params; // every layer's LayerParam (read by the degree scan)
    DevBuf<uint8_t> cub_tmp;
    LayerCounters* counters = nullptr;     // mapped pinned host memory
    LayerCounters* counters_dev = nullptr; // its device alias
    Scratch() {
        {
            std::lock_guard<std::mutex> lock(g_counters_mu);
            if (!g_counters_free.empty()) {
                counters = g_counters_free.back();
                g_counters_free.pop_back();
            }
        }
        if (!counters)
            VCS_CUDA(cudaHostAlloc(&counters, sizeof(LayerCounters),
                                   cudaHostAllocMapped | cudaHostAllocPortable));
        VCS_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&counters_dev), counters, 0));
    }
    ~Scratch() {
        std::lock_guard<std::mutex> lock(g_counters_mu);
        g_counters_free.push_back(counters);
    }
};

template <class InputIt>
void exclusive_scan(Scratch& sc, InputIt in, uint32_t* out, uint64_t n, cudaStream_t s) {
    size_t bytes = 0;
    VCS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, static_cast<int64_t>(n), s));
    sc.cub_tmp.exact(bytes, s);
    VCS_CUDA(cub::DeviceScan::ExclusiveSum(sc.cub_tmp.p, bytes, in, out, static_cast<int64_t>(n), s));
    note_launch();
}

// ---- pull form of the layered implicit builder (non-retiring transitions, see k_build_dense) --
// k_pull_first: per successor index d' of layer t+1, the first edge min((BFS index << 3) | slot)
// over its predecessors (the paid edge of d' itself, slot p of d' + demand*W_p), read from layer
// t's own rank table; clears the first edge's bit in the edge-key bitmap (all ones before) and
// sums the in-degrees (= E_t).  k_pull_rank: the BFS rank of every reached d' from the word
// prefixes of the bitmap; rank table (coalesced) and next-layer keys (digits of d').
__global__ void k_pull_first(const uint32_t* __restrict__ rank_self, const LayerParam* __restrict__ Lp,
                             uint32_t Dn, uint32_t* __restrict__ first, uint32_t* bm,
                             unsigned long long* edges) {
    __shared__ LayerParam L;
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(LayerParam) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(&L)[i] = __ldg(reinterpret_cast<const uint32_t*>(Lp) + i);
    __syncthreads();
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t deg = 0;
    if (d < Dn) {
        const uint32_t dem = static_cast<uint32_t>(L.demand);
        uint32_t rk[kDenseSlots];
        uint32_t rem = d;
#pragma unroll
        for (int p = 0; p < kDenseSlots - 1; ++p) {
            rk[p] = kEmpty32;
            if (p >= L.n_active) continue;
            const uint32_t rad = L.radix[p];
            const uint32_t g = rem % rad;
            rem /= rad;
            if (L.attr[p] && g + dem < rad) rk[p] = __ldg(rank_self + d + dem * L.wnext[p]);
        }
        rk[kDenseSlots - 1] = __ldg(rank_self + d); // the paid predecessor: d itself
        uint32_t best = kEmpty32;
#pragma unroll
        for (int p = 0; p < kDenseSlots; ++p)
            if (rk[p] != kEmpty32) {
                best = min(best, (rk[p] << 3) | static_cast<uint32_t>(p));
                ++deg;
            }
        first[d] = best;
        if (best != kEmpty32) atomicAnd(bm + (best >> 5), ~(1u << (best & 31u)));
    }
    deg = __reduce_add_sync(0xffffffffu, deg);
    if ((threadIdx.x & 31) == 0 && deg) atomicAdd(edges, static_cast<unsigned long long>(deg));
}

struct FirstBitsOp { // first edges in bitmap word w (the bitmap holds them as cleared bits)
    const uint32_t* bm;
    uint32_t nw;
    __device__ uint32_t operator()(uint32_t w) const {
        return w < nw ? static_cast<uint32_t>(__popc(~bm[w])) : 0u;
    }
};

template <int WM>
__global__ void k_pull_rank(const uint32_t* __restrict__ first, const uint32_t* __restrict__ bm,
                            const uint32_t* __restrict__ wpre, const LayerParam* __restrict__ Lp,
                            uint32_t Dn, uint32_t* __restrict__ rank_table,
                            uint64_t* __restrict__ keys_next) {
    __shared__ LayerParam L;
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(LayerParam) / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(&L)[i] = __ldg(reinterpret_cast<const uint32_t*>(Lp) + i);
    __syncthreads();
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= Dn) return;
    const uint32_t f = first[d];
    if (f == kEmpty32) {
        rank_table[d] = kEmpty32;
        return;
    }
    const uint32_t w = f >> 5;
    const uint32_t rank = wpre[w] + static_cast<uint32_t>(__popc(~bm[w] & ((1u << (f & 31u)) - 1u)));
    rank_table[d] = rank;
    uint64_t nk[WM];
#pragma unroll
    for (int i = 0; i < WM; ++i) nk[i] = 0ull;
    uint32_t rem = d;
    for (int p = 0; p < L.n_active; ++p) {
        const uint32_t rad = L.radix[p];
        put_field<WM>(nk, L.next_bit_off[p], static_cast<uint64_t>(rem % rad));
        rem /= rad;
    }
    const int nw = L.next_words;
#pragma unroll
    for (int i = 0; i < WM; ++i)
        if (i < nw) keys_next[static_cast<uint64_t>(rank) * nw + i] = nk[i];
}

// A transition into a one-state layer (the terminal layer when every cloud retires): every edge
// reaches index 0, whose first edge is the root-most state's first edge — rank 0; E_t = the
// degree sum.
__global__ void k_single_successor(const uint32_t* __restrict__ off_end, uint32_t* rank_table,
                                   uint64_t* key_next, int next_words, LayerCounters* out) {
    rank_table[0] = 0;
    for (int w = 0; w < next_words; ++w) key_next[w] = 0ull;
    out->n_edges = *off_end;
    out->n_next = 1;
}

__global__ void k_pull_counters(const unsigned long long* __restrict__ edges,
                                const uint32_t* __restrict__ wpre, uint32_t nw,
                                LayerCounters* __restrict__ out) {
    out->n_edges = static_cast<uint32_t>(*edges);
    out->n_next = wpre[nw];
}

// ---- persistent dense builder ----------------------------------------------------------------
// When every layer's successor key space is dense (mixed-radix index, see LayerParam) and the
// CSR fits at its a-priori bound, the whole build is ONE cooperative kernel: per layer
//   phase 1  degrees of the block's state chunk -> block sums                      | grid sync
//   phase 2  each block scans the block sums itself; emit edges (reward bits as k_emit_dense),
//            row offsets, atomicMin of the edge into the first-edge table        | grid sync
//   phase 3  first-occurrence flags of the block's edge chunk -> block sums          | grid sync
//   phase 4  ranks of first edges = successor indices in BFS order; first edges write the next
//            frontier's keys and rank_of[idx]; the state cap is checked           | grid sync
//   phase 5  (with the next layer's phase 1) successor ids of every edge; clear the table
// No host round trip per layer (the multi-kernel path needs one to size the next layer).
namespace cg = cooperative_groups;

struct DenseBuild {
    const LayerParam* __restrict__ params; // H
    uint64_t* keys;
    uint32_t* row_ptr;
    uint32_t* succ;
    double* reward;
    int32_t* action;
    uint32_t* table0;    // first-edge tables, alternating per layer (dense_max entries each)
    uint32_t* table1;
    uint32_t* rank_tables; // per transition t (at sum of dense_size of t' < t): successor
                           // mixed-radix index -> its layer-local state index (kept: the
                           // implicit-CSR solver reads them)
    uint32_t* bsum;      // per (round, block)
    uint64_t* desc;      // per state of the current layer: Slots::pack()
    uint32_t* jfirst;    // per state of the current layer: its first edge (layer-local)
    uint64_t* stamps;    // VCS_TRACE: globaltimer at each phase boundary, 6 per layer (or null)
    uint64_t* info;      // n_t for t = 0..H at [t], E_t for t = 0..H-1 at [H+1+t]
    int32_t* status;     // 0 ok, 1 state cap exceeded, 2 more than 2^32-1 states
    uint64_t state_cap;
    uint32_t dense_max;
    int max_rounds;      // bsum holds max_rounds x gridDim.x entries
    int H;
    int pull;            // the pull form may run on layers marked LayerParam::pull
};

constexpr int kDenseThreads = 256;
constexpr int kPullMaxBlocks = 1024; // (round, block) prefixes of the pull form in shared memory

// Successor key of the edge choosing key position p (-1 = paid), in layer t+1's packing.
template <int WM>
__device__ __forceinline__ void next_key(const uint64_t (&k)[WM], int p, const LayerParam& L,
                                         uint64_t (&nk)[WM]) {
#pragma unroll
    for (int w = 0; w < WM; ++w) nk[w] = 0ull;
    if (L.n_keep == L.n_active) { // same layout: subtract the demand from the chosen field
#pragma unroll
        for (int w = 0; w < WM; ++w) nk[w] = k[w];
        if (p >= 0) {
            const int off = L.bit_off[p];
#pragma unroll
            for (int w = 0; w < WM; ++w)
                if (w == (off >> 6)) nk[w] -= static_cast<uint64_t>(L.demand) << (off & 63);
        }
        return;
    }
    for (int q = 0; q < L.n_active; ++q) {
        if (L.keep_idx[q] < 0) continue;
        int v = get_field<WM>(k, L.bit_off[q], L.width[q]);
        if (q == p) v -= L.demand;
        put_field<WM>(nk, L.next_bit_off[q], static_cast<uint64_t>(v));
    }
}

// Prefixes of (round r, block b) for every round r over the per-(round, block) sums in
// round-major order, into s_before[r]; returns the grand total.  Warp r sums round r (coalesced,
// all loads in flight), then one thread combines the <= 8 rounds.
__device__ __forceinline__ uint32_t round_prefixes(const uint32_t* __restrict__ bsum, int R, int G,
                                                   int b, uint32_t* s_before) {
    __shared__ uint32_t s_part[8], s_tot[8], s_total;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w < R) {
        uint32_t part = 0, tot = 0;
        // eight loads in flight per lane (G <= 256 blocks: one batch)
        for (int i0 = lane; i0 < G; i0 += 8 * 32) {
            uint32_t v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = i0 + 32 * k;
                v[k] = i < G ? __ldcg(bsum + w * G + i) : 0u;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                tot += v[k];
                if (i0 + 32 * k < b) part += v[k];
            }
        }
        part = __reduce_add_sync(0xffffffffu, part);
        tot = __reduce_add_sync(0xffffffffu, tot);
        if (lane == 0) {
            s_part[w] = part;
            s_tot[w] = tot;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int r = 0; r < R; ++r) {
            s_before[r] = acc + s_part[r];
            acc += s_tot[r];
        }
        s_total = acc;
    }
    __syncthreads();
    return s_total;
}

// Per-round block sums without a block barrier per round: warp sums, shared atomics.
__device__ __forceinline__ void round_add(uint32_t* s_round, int r, uint32_t v) {
    const uint32_t w = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(s_round + r, w);
}

__device__ __forceinline__ void stamp(uint64_t* stamps, int slot) {
    if (stamps && blockIdx.x == 0 && threadIdx.x == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        stamps[slot] = t;
    }
}

// EXPLICIT: also write the CSR (row_ptr, succ, reward, action).  Without it the build keeps
// only keys, layer sizes and the rank tables: the implicit-CSR form.
template <int WM, int MINB, bool EXPLICIT>
__global__ void __launch_bounds__(kDenseThreads, MINB) k_build_dense(DenseBuild A) {
    using Scan = cub::BlockScan<uint32_t, kDenseThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ LayerParam sL;
    __shared__ uint32_t s_round[8];  // per-round block sums
    __shared__ uint32_t s_before[8]; // per-round prefixes of this block
    // a round's edges of this block are one contiguous range: staged here, written coalesced
    __shared__ double s_rew[kDenseThreads * kDenseSlots];
    __shared__ int32_t s_act[kDenseThreads * kDenseSlots];
    cg::grid_group grid = cg::this_grid();
    const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
    const uint32_t T = static_cast<uint32_t>(G) * blockDim.x; // states per round
    const uint32_t q = static_cast<uint32_t>(b) * blockDim.x + tid;
    uint64_t S_t = 0;   // first state of layer t
    uint64_t E = 0;     // edges of layers < t
    uint64_t key_t = 0; // first key word of layer t
    uint64_t rank_t = 0; // first entry of transition t's rank table
    uint64_t rank_prev = 0; // transition t-1's (layer t's own index -> BFS index)
    uint32_t n_t = 1;
    if (b == 0 && tid == 0) A.info[0] = 1;
    auto publish_rounds = [&](int R) { // s_round -> bsum[r * G + b]
        __syncthreads();
        if (tid < R) A.bsum[tid * G + b] = s_round[tid];
    };
    constexpr int SL = kDenseSlots;
    for (int t = 0; t < A.H; ++t) {
        __syncthreads();
        for (int i = tid; i < static_cast<int>(sizeof(LayerParam) / 4); i += blockDim.x)
            reinterpret_cast<uint32_t*>(&sL)[i] = reinterpret_cast<const uint32_t*>(A.params + t)[i];
        if (tid < 8) s_round[tid] = 0;
        __syncthreads();
        const LayerParam& L = sL;
        const SlotDecoder<WM> dec(L); // the layer's slot constants, in registers
        uint32_t* table = (t & 1) ? A.table1 : A.table0;
        const uint64_t S_next = S_t + n_t;
        const uint64_t key_next = key_t + static_cast<uint64_t>(n_t) * L.words;
        const int R = static_cast<int>((n_t + T - 1) / T); // rounds: state r*T + q
        const bool retires = L.n_keep != L.n_active;
        auto key_of = [&](uint32_t i, uint64_t (&k)[WM]) {
            load_key<WM>(A.keys + key_t + static_cast<uint64_t>(i) * L.words, L.words, k);
        };
        stamp(A.stamps, 6 * t + 0);
        if (!EXPLICIT && WM == 1 && A.pull && L.pull && t >= 1 &&
            (L.dense_size + T - 1) / T <= 8 && (static_cast<uint64_t>(n_t) + 4 * T - 1) / (4 * T) <= 2) {
            // Pull form (a non-retiring transition numbered alike on both sides): successor d'
            // has the paid predecessor d' and, per eligible cloud p, the predecessor
            // d' + demand*W_p (when that free count fits the cloud); the predecessors' BFS
            // indices come from layer t's own rank table (transition t-1), read as shifted
            // streams.  Its first edge is the minimum of (index << 3 | slot) over them — what the
            // push form's atomicMin finds — without an atomic per edge.  The BFS numbering of
            // layer t+1 is the order of those first edges: a bitmap over the edge keys (bit
            // cleared = a first edge; the table starts all ones), popcount prefixes, and every
            // reached d' looks up its rank.
            constexpr int RB = 8;
            constexpr int NF = kDenseSlots - 1;
            const uint32_t Dn = L.dense_size;
            const int R1 = static_cast<int>((Dn + T - 1) / T);
            const uint32_t* __restrict__ rs = A.rank_tables + rank_prev; // layer t: index -> BFS index
            uint32_t* bm = table;
            const uint32_t dem = static_cast<uint32_t>(L.demand);
            uint32_t g[NF], sd[NF], rad[NF], wp[NF], nbo[NF], elig = 0;
            {
                uint32_t rem = q < Dn ? q : 0u, srem = T < Dn ? static_cast<uint32_t>(T) : 0u;
#pragma unroll
                for (int p = 0; p < NF; ++p) {
                    const bool on = p < L.n_active;
                    rad[p] = on ? L.radix[p] : 1u;
                    wp[p] = on ? L.wnext[p] : 0u;
                    nbo[p] = on ? L.next_bit_off[p] : 0u;
                    if (on && L.attr[p]) elig |= 1u << p;
                    g[p] = rem % rad[p];
                    rem /= rad[p];
                    sd[p] = srem % rad[p];
                    srem /= rad[p];
                }
            }
            stamp(A.stamps, 6 * t + 1);
            uint32_t fr[RB];
            uint64_t kr[RB];
            uint32_t dsum = 0;
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                const uint32_t d = static_cast<uint32_t>(r) * T + q;
                fr[r] = kEmpty32;
                kr[r] = 0ull;
                if (r >= R1 || d >= Dn) continue;
                uint32_t rk[NF + 1];
                rk[NF] = __ldcg(rs + d); // the paid predecessor: d itself
#pragma unroll
                for (int p = 0; p < NF; ++p)
                    rk[p] = ((elig >> p) & 1u) && g[p] + dem < rad[p] ? __ldcg(rs + d + dem * wp[p]) : kEmpty32;
                uint32_t best = kEmpty32;
                uint64_t key = 0ull;
#pragma unroll
                for (int p = 0; p < NF; ++p) {
                    key |= static_cast<uint64_t>(g[p]) << nbo[p];
                    if (rk[p] != kEmpty32) {
                        best = min(best, (rk[p] << 3) | static_cast<uint32_t>(p));
                        ++dsum;
                    }
                }
                if (rk[NF] != kEmpty32) {
                    best = min(best, (rk[NF] << 3) | static_cast<uint32_t>(NF));
                    ++dsum;
                }
                fr[r] = best;
                kr[r] = key;
                if (best != kEmpty32) atomicAnd(bm + (best >> 5), ~(1u << (best & 31u)));
                // the next round's digits: d + T
                uint32_t carry = 0;
#pragma unroll
                for (int p = 0; p < NF; ++p) {
                    const uint32_t v = g[p] + sd[p] + carry;
                    carry = v >= rad[p] ? 1u : 0u;
                    g[p] = carry ? v - rad[p] : v;
                }
            }
            dsum = __reduce_add_sync(0xffffffffu, dsum);
            if ((tid & 31) == 0 && dsum)
                atomicAdd(reinterpret_cast<unsigned long long*>(A.info + A.H + 1 + t),
                          static_cast<unsigned long long>(dsum));
            grid.sync();
            stamp(A.stamps, 6 * t + 2);
            // first edges per bitmap word; block-local exclusive prefixes of the words
            uint32_t* wpre = reinterpret_cast<uint32_t*>(A.desc);
            const uint32_t NW = (n_t + 3u) / 4u; // 8 * n_t edge keys
            const int R2 = static_cast<int>((NW + T - 1) / T);
            {
                __shared__ uint32_t s_ws2[2][kDenseThreads / 32];
                const int lane = tid & 31, warp = tid >> 5;
                uint32_t c[2], wex[2];
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const uint32_t w = static_cast<uint32_t>(r) * T + q;
                    c[r] = (r < R2 && w < NW) ? static_cast<uint32_t>(__popc(~__ldcg(bm + w))) : 0u;
                    uint32_t incl = c[r];
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += y;
                    }
                    wex[r] = incl - c[r];
                    if (lane == 31) s_ws2[r][warp] = incl;
                }
                __syncthreads();
#pragma unroll
                for (int r = 0; r < 2; ++r) {
                    const uint32_t w = static_cast<uint32_t>(r) * T + q;
                    uint32_t before = wex[r], tot = 0;
                    for (int k = 0; k < kDenseThreads / 32; ++k) {
                        before += k < warp ? s_ws2[r][k] : 0u;
                        tot += s_ws2[r][k];
                    }
                    if (r < R2 && w < NW) wpre[w] = before;
                    if (tid == 0 && r < R2) s_round[r] = tot;
                }
            }
            publish_rounds(R2);
            grid.sync();
            stamp(A.stamps, 6 * t + 3);
            // global prefixes of every (round, block) of the words, in shared memory
            __shared__ uint32_t s_gpre[2 * kPullMaxBlocks];
            uint32_t n_next = 0;
            {
                // (every thread's <= 8 sums loaded at once: M = R2 * G <= 2 * kPullMaxBlocks)
                constexpr int PER = 2 * kPullMaxBlocks / kDenseThreads;
                const int M = R2 * G;
                const int per = (M + kDenseThreads - 1) / kDenseThreads;
                uint32_t v[PER], loc = 0;
#pragma unroll
                for (int k = 0; k < PER; ++k) {
                    const int i = tid * per + k;
                    v[k] = (k < per && i < M) ? __ldcg(A.bsum + i) : 0u;
                    loc += v[k];
                }
                uint32_t ex;
                Scan(scan_tmp).ExclusiveSum(loc, ex, n_next);
#pragma unroll
                for (int k = 0; k < PER; ++k) {
                    const int i = tid * per + k;
                    if (k < per && i < M) s_gpre[i] = ex;
                    ex += v[k];
                }
                __syncthreads();
            }
            if (S_next + n_next > A.state_cap || S_next + n_next >= 0xffffffffull) {
                if (b == 0 && tid == 0) {
                    *A.status = S_next + n_next > A.state_cap ? 1 : 2;
                    A.info[t + 1] = n_next;
                }
                return; // every block takes the same decision
            }
            // ranks: the rank table of transition t (coalesced, by d') and the next layer's keys
            // (every round's two gathers first, then the stores)
            uint32_t bmw[RB], wpv[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                const uint32_t f = fr[r];
                bmw[r] = f != kEmpty32 ? __ldcg(bm + (f >> 5)) : 0u;
                wpv[r] = f != kEmpty32 ? __ldcg(wpre + (f >> 5)) : 0u;
            }
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                const uint32_t d = static_cast<uint32_t>(r) * T + q;
                if (r >= R1 || d >= Dn) continue;
                const uint32_t f = fr[r];
                uint32_t rank = kEmpty32;
                if (f != kEmpty32) {
                    const uint32_t w = f >> 5;
                    const uint32_t rw = w >= T ? 1u : 0u;
                    const uint32_t bw = (w - rw * static_cast<uint32_t>(T)) / kDenseThreads;
                    rank = s_gpre[rw * G + bw] + wpv[r] +
                           static_cast<uint32_t>(__popc(~bmw[r] & ((1u << (f & 31u)) - 1u)));
                    A.keys[key_next + rank] = kr[r];
                }
                A.rank_tables[rank_t + d] = rank;
            }
            if (b == 0 && tid == 0) A.info[t + 1] = n_next;
            if (tid < 8) s_round[tid] = 0;
            grid.sync();
            stamp(A.stamps, 6 * t + 4);
            for (uint32_t i = q; i < A.dense_max; i += T) table[i] = kEmpty32;
            S_t = S_next;
            key_t = key_next;
            rank_prev = rank_t;
            rank_t += L.dense_size;
            n_t = n_next;
            continue;
        }
        if (!EXPLICIT && WM == 1) {
            // Implicit form, single-word keys, all of a thread's rounds at once: keys,
            // descriptors and first-edge masks stay in registers across the grid syncs, the
            // table loads of four rounds are in flight together, and ranks come from warp scans
            // with one block barrier (instead of a block scan per round).
            constexpr int RB = 8; // rounds (the host guarantees R <= 8)
            uint64_t kr[RB], dr[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                const uint32_t i = static_cast<uint32_t>(r) * T + q;
                kr[r] = (r < R && i < n_t) ? A.keys[key_t + i] : 0ull;
            }
            stamp(A.stamps, 6 * t + 1);
            uint32_t dsum = 0;
            const bool red = L.dense_size > 4096;
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                const uint32_t i = static_cast<uint32_t>(r) * T + q;
                dr[r] = 0ull;
                if (r >= R || i >= n_t) continue;
                const uint64_t k1[1] = {kr[r]};
                const Slots sl = reinterpret_cast<const SlotDecoder<1>&>(dec).decode(k1);
                dr[r] = sl.pack();
                dsum += sl.deg();
#pragma unroll
                for (int e = 0; e < SL; ++e) {
                    if (!sl.valid(e)) continue;
                    const uint32_t key = (i << 3) | static_cast<uint32_t>(e);
                    uint32_t* slot = &table[dec.idx(sl, e)];
                    if (red || __ldcg(slot) > key) atomicMin(slot, key);
                }
            }
            dsum = __reduce_add_sync(0xffffffffu, dsum);
            if ((tid & 31) == 0 && dsum)
                atomicAdd(reinterpret_cast<unsigned long long*>(A.info + A.H + 1 + t),
                          static_cast<unsigned long long>(dsum));
            grid.sync();
            stamp(A.stamps, 6 * t + 2);
            // first-occurrence masks (kept for the rank phase), counts per (round, block)
            uint32_t fm[RB];
#pragma unroll
            for (int h = 0; h < RB; h += 4) {
                uint32_t cur[4][SL];
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) {
                    const int r = h + rr;
                    // (a live state may have descriptor 0: only the paid edge, to index 0)
                    const bool live = r < R && static_cast<uint32_t>(r) * T + q < n_t;
                    const Slots sl(dr[r]);
#pragma unroll
                    for (int e = 0; e < SL; ++e)
                        if (live && sl.valid(e)) cur[rr][e] = __ldcg(table + dec.idx(sl, e));
                }
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) {
                    const int r = h + rr;
                    const uint32_t i = static_cast<uint32_t>(r) * T + q;
                    const bool live = r < R && i < n_t;
                    const Slots sl(dr[r]);
                    uint32_t f = 0;
#pragma unroll
                    for (int e = 0; e < SL; ++e)
                        if (live && sl.valid(e) && cur[rr][e] == ((i << 3) | static_cast<uint32_t>(e)))
                            f |= 1u << e;
                    fm[r] = f;
                    if (r < R) round_add(s_round, r, static_cast<uint32_t>(__popc(f)));
                }
            }
            publish_rounds(R);
            grid.sync();
            stamp(A.stamps, 6 * t + 3);
            const uint32_t n_next = round_prefixes(A.bsum, R, G, b, s_before);
            if (S_next + n_next > A.state_cap || S_next + n_next >= 0xffffffffull) {
                if (b == 0 && tid == 0) {
                    *A.status = S_next + n_next > A.state_cap ? 1 : 2;
                    A.info[t + 1] = n_next;
                }
                return; // every block takes the same decision
            }
            // ranks: warp exclusive scans of every round, one barrier for the warps' offsets
            __shared__ uint32_t s_wsum[RB][kDenseThreads / 32];
            const int lane = tid & 31, warp = tid >> 5;
            uint32_t wex[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                const uint32_t f = static_cast<uint32_t>(__popc(fm[r]));
                uint32_t incl = f;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                wex[r] = incl - f;
                if (lane == 31) s_wsum[r][warp] = incl;
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                if (!fm[r]) continue;
                uint32_t rank = s_before[r] + wex[r];
                for (int w = 0; w < warp; ++w) rank += s_wsum[r][w];
                const uint64_t k1[1] = {kr[r]};
                const Slots sl(dr[r]);
                // over the set bits, not unrolled: 8 x 8 inlined next_key bodies made the kernel
                // large enough to miss in the instruction cache (shared-memory slot constants)
#pragma unroll 1
                for (uint32_t m = fm[r]; m; m &= m - 1) {
                    const int e = __ffs(m) - 1;
                    A.rank_tables[rank_t + sl.idx(e, L)] = rank;
                    uint64_t nk[1];
                    next_key<1>(k1, e == SL - 1 ? -1 : e, L, nk);
                    A.keys[key_next + rank] = nk[0];
                    ++rank;
                }
            }
            if (b == 0 && tid == 0) A.info[t + 1] = n_next;
            if (tid < 8) s_round[tid] = 0;
            grid.sync();
            stamp(A.stamps, 6 * t + 4);
            for (uint32_t i = q; i < A.dense_max; i += T) table[i] = kEmpty32;
            S_t = S_next;
            key_t = key_next;
            rank_prev = rank_t;
            rank_t += L.dense_size;
            n_t = n_next;
            continue;
        }
        if (!EXPLICIT) {
            // Implicit form: no edge offsets are needed.  Edges are ordered by (state, slot), so
            // the first edge into a successor is the minimum of (i << 3 | slot) over its edges.
            // phase 1: descriptors, degree sum (E_t), first-edge atomicMin
            stamp(A.stamps, 6 * t + 1);
            uint32_t dsum = 0;
            for (int r = 0; r < R; ++r) {
                const uint32_t i = static_cast<uint32_t>(r) * T + q;
                if (i >= n_t) continue;
                uint64_t k[WM];
                key_of(i, k);
                const Slots sl = dec.decode(k);
                A.desc[i] = sl.pack();
                dsum += sl.deg();
                if (L.dense_size > 4096) {
                    // a large successor space spreads the edges: plain reductions, no result
                    // and no check load (nothing on the thread's latency chain)
#pragma unroll
                    for (int e = 0; e < SL; ++e)
                        if (sl.valid(e))
                            atomicMin(&table[dec.idx(sl, e)], (i << 3) | static_cast<uint32_t>(e));
                } else {
                    // few successors (e.g. the single terminal state): read first, so that
                    // heavily shared entries are not serialised by atomics
                    uint32_t cur[SL];
#pragma unroll
                    for (int e = 0; e < SL; ++e)
                        if (sl.valid(e)) cur[e] = __ldcg(table + dec.idx(sl, e));
#pragma unroll
                    for (int e = 0; e < SL; ++e) {
                        const uint32_t key = (i << 3) | static_cast<uint32_t>(e);
                        if (sl.valid(e) && cur[e] > key) atomicMin(&table[dec.idx(sl, e)], key);
                    }
                }
            }
            dsum = __reduce_add_sync(0xffffffffu, dsum);
            if ((tid & 31) == 0 && dsum)
                atomicAdd(reinterpret_cast<unsigned long long*>(A.info + A.H + 1 + t),
                          static_cast<unsigned long long>(dsum));
            grid.sync();
            stamp(A.stamps, 6 * t + 2);
            // phase 2: first-occurrence counts per (round, block)
            for (int r = 0; r < R; ++r) {
                const uint32_t i = static_cast<uint32_t>(r) * T + q;
                uint32_t f = 0;
                if (i < n_t) {
                    const Slots sl(__ldcg(A.desc + i));
                    uint32_t cur[SL];
#pragma unroll
                    for (int e = 0; e < SL; ++e)
                        if (sl.valid(e)) cur[e] = __ldcg(table + dec.idx(sl, e));
#pragma unroll
                    for (int e = 0; e < SL; ++e)
                        if (sl.valid(e) && cur[e] == ((i << 3) | static_cast<uint32_t>(e))) ++f;
                }
                round_add(s_round, r, f);
            }
            publish_rounds(R);
            grid.sync();
            stamp(A.stamps, 6 * t + 3);
            // phase 3: ranks, next keys, cap check
            const uint32_t n_next = round_prefixes(A.bsum, R, G, b, s_before);
            if (S_next + n_next > A.state_cap || S_next + n_next >= 0xffffffffull) {
                if (b == 0 && tid == 0) {
                    *A.status = S_next + n_next > A.state_cap ? 1 : 2;
                    A.info[t + 1] = n_next;
                }
                return; // every block takes the same decision
            }
            for (int r = 0; r < R; ++r) {
                const uint32_t i = static_cast<uint32_t>(r) * T + q;
                const Slots sl(i < n_t ? __ldcg(A.desc + i) : 0ull);
                uint32_t first = 0;
                if (i < n_t) {
                    uint32_t cur[SL];
#pragma unroll
                    for (int e = 0; e < SL; ++e)
                        if (sl.valid(e)) cur[e] = __ldcg(table + dec.idx(sl, e));
#pragma unroll
                    for (int e = 0; e < SL; ++e)
                        if (sl.valid(e) && cur[e] == ((i << 3) | static_cast<uint32_t>(e)))
                            first |= 1u << e;
                }
                uint32_t rank;
                Scan(scan_tmp).ExclusiveSum(static_cast<uint32_t>(__popc(first)), rank);
                __syncthreads();
                rank += s_before[r];
                if (first) {
                    uint64_t k[WM];
                    key_of(i, k);
#pragma unroll
                    for (int e = 0; e < SL; ++e) {
                        if (!((first >> e) & 1u)) continue;
                        A.rank_tables[rank_t + dec.idx(sl, e)] = rank;
                        uint64_t nk[WM];
                        next_key<WM>(k, e == SL - 1 ? -1 : e, L, nk);
                        uint64_t* dst = A.keys + key_next + static_cast<uint64_t>(rank) * L.next_words;
#pragma unroll
                        for (int w = 0; w < WM; ++w)
                            if (w < L.next_words) dst[w] = nk[w];
                        ++rank;
                    }
                }
            }
            if (b == 0 && tid == 0) A.info[t + 1] = n_next;
            if (tid < 8) s_round[tid] = 0;
            grid.sync();
            stamp(A.stamps, 6 * t + 4);
            for (uint32_t i = q; i < A.dense_max; i += T) table[i] = kEmpty32;
            S_t = S_next;
            key_t = key_next;
            rank_prev = rank_t;
            rank_t += L.dense_size;
            n_t = n_next;
            continue;
        }
        // phase 1: degrees per (round, block); each state's slot descriptor
        for (int r = 0; r < R; ++r) {
            const uint32_t i = static_cast<uint32_t>(r) * T + q;
            uint32_t d = 0;
            if (i < n_t) {
                uint64_t k[WM];
                key_of(i, k);
                const Slots sl = dec.decode(k);
                d = sl.deg();
                A.desc[i] = sl.pack();
            }
            round_add(s_round, r, d);
        }
        publish_rounds(R);
        grid.sync();
        stamp(A.stamps, 6 * t + 1);
        // phase 2: row offsets, rewards, actions, first-edge atomicMin
        const uint32_t E_t = round_prefixes(A.bsum, R, G, b, s_before);
        for (int r = 0; r < R; ++r) {
            const uint32_t i = static_cast<uint32_t>(r) * T + q;
            const Slots sl(i < n_t ? __ldcg(A.desc + i) : 0ull);
            const uint32_t deg = i < n_t ? sl.deg() : 0u;
            uint32_t excl, cnt;
            Scan(scan_tmp).ExclusiveSum(deg, excl, cnt);
            __syncthreads();
            const uint32_t j0 = s_before[r]; // the block's first edge in this round
            if (i < n_t) {
                const uint32_t j = j0 + excl;
                A.jfirst[i] = j;
                if (EXPLICIT) A.row_ptr[S_t + i] = static_cast<uint32_t>(E + j);
                uint32_t cur[SL];
#pragma unroll
                for (int e = 0; e < SL; ++e)
                    if (sl.valid(e)) cur[e] = __ldcg(table + dec.idx(sl, e)); // the state's checks in flight
                uint64_t k[WM];
                if (EXPLICIT && retires) key_of(i, k);
#pragma unroll
                for (int e = 0; e < SL; ++e) {
                    if (!sl.valid(e)) continue;
                    const int pe = e == SL - 1 ? -1 : e;
                    const uint32_t o = excl + (e == SL - 1 ? sl.deg() - 1u : sl.off(e));
                    if (EXPLICIT) {
                        s_rew[o] = retires ? retiring_reward<WM>(k, pe, L)
                                           : (pe < 0 ? L.r_paid_kept : L.r_cloud_kept);
                        s_act[o] = pe < 0 ? -1 : L.cloud[pe];
                    }
                    if (cur[e] > j0 + o) atomicMin(&table[dec.idx(sl, e)], j0 + o); // first edge wins
                }
            }
            if (EXPLICIT) {
                __syncthreads();
                for (uint32_t o = tid; o < cnt; o += blockDim.x) {
                    A.reward[E + j0 + o] = s_rew[o];
                    A.action[E + j0 + o] = s_act[o];
                }
            }
        }
        if (tid < 8) s_round[tid] = 0;
        grid.sync();
        stamp(A.stamps, 6 * t + 2);
        // phase 3: first-occurrence flags per (round, block)
        for (int r = 0; r < R; ++r) {
            const uint32_t i = static_cast<uint32_t>(r) * T + q;
            uint32_t f = 0;
            if (i < n_t) {
                const Slots sl(__ldcg(A.desc + i));
                const uint32_t j = __ldcg(A.jfirst + i);
                uint32_t cur[SL];
#pragma unroll
                for (int e = 0; e < SL; ++e)
                    if (sl.valid(e)) cur[e] = __ldcg(table + dec.idx(sl, e));
#pragma unroll
                for (int e = 0; e < SL; ++e)
                    if (sl.valid(e))
                        f += cur[e] == j + (e == SL - 1 ? sl.deg() - 1u : sl.off(e)) ? 1u : 0u;
            }
            round_add(s_round, r, f);
        }
        publish_rounds(R);
        grid.sync();
        stamp(A.stamps, 6 * t + 3);
        // phase 4: ranks of first edges = successor indices; next frontier keys; cap check
        const uint32_t n_next = round_prefixes(A.bsum, R, G, b, s_before);
        if (S_next + n_next > A.state_cap || S_next + n_next >= 0xffffffffull) {
            if (b == 0 && tid == 0) {
                *A.status = S_next + n_next > A.state_cap ? 1 : 2;
                A.info[t + 1] = n_next;
            }
            return; // every block takes the same decision
        }
        for (int r = 0; r < R; ++r) {
            const uint32_t i = static_cast<uint32_t>(r) * T + q;
            const Slots sl(i < n_t ? __ldcg(A.desc + i) : 0ull);
            const uint32_t j = i < n_t ? __ldcg(A.jfirst + i) : 0u;
            uint32_t first = 0; // bit e: slot e is its successor's first edge
            if (i < n_t) {
                uint32_t cur[SL];
#pragma unroll
                for (int e = 0; e < SL; ++e)
                    if (sl.valid(e)) cur[e] = __ldcg(table + dec.idx(sl, e));
#pragma unroll
                for (int e = 0; e < SL; ++e)
                    if (sl.valid(e) && cur[e] == j + (e == SL - 1 ? sl.deg() - 1u : sl.off(e)))
                        first |= 1u << e;
            }
            uint32_t rank;
            Scan(scan_tmp).ExclusiveSum(static_cast<uint32_t>(__popc(first)), rank);
            __syncthreads();
            rank += s_before[r];
            if (first) {
                uint64_t k[WM];
                key_of(i, k); // the parent key: next keys are derived from it
#pragma unroll
                for (int e = 0; e < SL; ++e) {
                    if (!((first >> e) & 1u)) continue;
                    A.rank_tables[rank_t + dec.idx(sl, e)] = rank;
                    uint64_t nk[WM];
                    next_key<WM>(k, e == SL - 1 ? -1 : e, L, nk);
                    uint64_t* dst = A.keys + key_next + static_cast<uint64_t>(rank) * L.next_words;
#pragma unroll
                    for (int w = 0; w < WM; ++w)
                        if (w < L.next_words) dst[w] = nk[w];
                    ++rank;
                }
            }
        }
        if (b == 0 && tid == 0) {
            A.info[t + 1] = n_next;
            A.info[A.H + 1 + t] = E_t;
        }
        grid.sync();
        stamp(A.stamps, 6 * t + 4);
        // phase 5: successor ids (explicit form); clear this layer's first-edge table for layer
        // t+2 (layer t+1 uses the other one)
        uint32_t* s_succ = reinterpret_cast<uint32_t*>(s_act); // (phase 2 is done with it)
        __shared__ uint32_t s_j0, s_j1;
        for (int r = 0; EXPLICIT && r < R; ++r) {
            const uint32_t i = static_cast<uint32_t>(r) * T + q;
            const uint32_t blk0 = static_cast<uint32_t>(r) * T + static_cast<uint32_t>(b) * blockDim.x;
            __syncthreads();
            if (tid == 0) { // this block's edge range in round r: first and last valid state
                const uint32_t last = min(n_t, blk0 + blockDim.x);
                if (blk0 < n_t) {
                    s_j0 = __ldcg(A.jfirst + blk0);
                    s_j1 = __ldcg(A.jfirst + last - 1) + Slots(__ldcg(A.desc + last - 1)).deg();
                } else {
                    s_j0 = s_j1 = 0;
                }
            }
            __syncthreads();
            const uint32_t j0 = s_j0, cnt = s_j1 - s_j0;
            if (i < n_t) {
                const Slots sl(__ldcg(A.desc + i));
                const uint32_t o0 = __ldcg(A.jfirst + i) - j0;
                uint32_t rk[SL];
#pragma unroll
                for (int e = 0; e < SL; ++e)
                    if (sl.valid(e)) rk[e] = __ldcg(A.rank_tables + rank_t + dec.idx(sl, e));
#pragma unroll
                for (int e = 0; e < SL; ++e)
                    if (sl.valid(e))
                        s_succ[o0 + (e == SL - 1 ? sl.deg() - 1u : sl.off(e))] =
                            static_cast<uint32_t>(S_next) + rk[e];
            }
            __syncthreads();
            for (uint32_t o = tid; o < cnt; o += blockDim.x) A.succ[E + j0 + o] = s_succ[o];
        }
        for (uint32_t i = q; i < A.dense_max; i += T) table[i] = kEmpty32;
        S_t = S_next;
        E += E_t;
        key_t = key_next;
        rank_prev = rank_t;
        rank_t += L.dense_size;
        n_t = n_next;
    }
    // the terminal layer's rows have no edges (mdp.cpp:207-209)
    if (EXPLICIT)
        for (uint32_t i = q; i <= n_t; i += T) A.row_ptr[S_t + i] = static_cast<uint32_t>(E);
}

// Host side of the persistent dense builder.  Returns false (nothing done) when it does not
// apply: some layer's key space is not dense, the a-priori CSR bound is not affordable, or the
// device cannot launch cooperative kernels.  VCS_BUILD_LAYERED forces the multi-kernel path.
template <int WM, bool EXPLICIT>
bool build_dense(vcs_space* sp, uint64_t state_cap) {
    // (read per build: tests.  VCS_BUILD_NO_PERSISTENT takes the layered implicit path.)
    const bool layered = std::getenv("VCS_BUILD_LAYERED") != nullptr ||
                         (!EXPLICIT && std::getenv("VCS_BUILD_NO_PERSISTENT") != nullptr);
    const LayerPlan& pl = sp->plan;
    const int H = pl.horizon;
    if (layered || H < 1) return false;
    uint64_t s_bound = 1, e_bound = 0, k_bound = static_cast<uint64_t>(pl.words[0]);
    uint64_t e_layer_max = 1, dense_max = 1, nb = 1;
    for (int t = 0; t < H; ++t) {
        const LayerParam& L = pl.layers[static_cast<size_t>(t)];
        if (!L.dense_size || L.n_active > kDenseSlots - 1) return false;
        int maxdeg = 1;
        for (int p = 0; p < L.n_active; ++p) maxdeg += L.attr[p] ? 1 : 0;
        const uint64_t e_ub = nb * static_cast<uint64_t>(maxdeg);
        e_bound += e_ub;
        e_layer_max = std::max(e_layer_max, e_ub);
        dense_max = std::max<uint64_t>(dense_max, L.dense_size);
        nb = std::min<uint64_t>({nb * static_cast<uint64_t>(maxdeg), state_cap, L.dense_size});
        s_bound += nb;
        k_bound += nb * static_cast<uint64_t>(L.next_words);
        if (e_bound >= 0xffffffffull || s_bound >= 0xffffffffull) return false;
    }
    uint64_t rank_total = 0;
    for (int t = 0; t < H; ++t) rank_total += pl.layers[static_cast<size_t>(t)].dense_size;
    const uint64_t bytes = (EXPLICIT ? e_bound * 16 + s_bound * 4 : 0) + k_bound * 8 +
                           e_layer_max * 4 + dense_max * 8 + rank_total * 4;
    if (bytes > device_bytes(sp->device) / 8) return false;
    int coop = 0;
    VCS_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, sp->device));
    if (!coop) return false;
    // (2 blocks per SM; forcing 3 or 4 by register caps measured slower)
    const void* fn = reinterpret_cast<const void*>(k_build_dense<WM, 2, EXPLICIT>);
    int per_sm = 0;
    VCS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kDenseThreads, 0));
    if (per_sm < 1) return false;
    const int G = per_sm * sp->num_sms;
    // rounds of G*256 states per layer (the kernel keeps <= 8 per-round offsets in registers)
    uint64_t n_max = 1;
    {
        uint64_t nb2 = 1;
        for (int t = 0; t < H; ++t) {
            const LayerParam& L = pl.layers[static_cast<size_t>(t)];
            int maxdeg = 1;
            for (int p = 0; p < L.n_active; ++p) maxdeg += L.attr[p] ? 1 : 0;
            nb2 = std::min<uint64_t>({nb2 * static_cast<uint64_t>(maxdeg), state_cap, L.dense_size});
            n_max = std::max(n_max, nb2);
        }
    }
    const uint64_t T = static_cast<uint64_t>(G) * kDenseThreads;
    const int max_rounds = static_cast<int>((n_max + T - 1) / T);
    if (max_rounds > 8) return false;

    const double t_setup = trace_enabled() ? host_ms() : 0.0;
    cudaStream_t s = sp->stream;
    sp->keys.reserve(k_bound, 0, s);
    if (EXPLICIT) {
        sp->row_ptr.reserve(s_bound + 1, 0, s);
        sp->succ.reserve(e_bound, 0, s);
        sp->reward.reserve(e_bound, 0, s);
        sp->action.reserve(e_bound, 0, s);
    }
    sp->rank_tables.exact(rank_total, s);
    // unreached successor indices read as kEmpty32 (the certified pass walks layers in key-space
    // order and skips them).  The pull form writes every entry of its transitions' tables: only
    // the push transitions' runs are cleared (C4: 6 of 48).
    {
        // (the kernel's own condition for the pull form, A.pull included)
        const bool pull_on = !EXPLICIT && WM == 1 && G <= kPullMaxBlocks && !std::getenv("VCS_BUILD_NO_PULL");
        uint64_t off = 0, run0 = 0, run = 0;
        for (int t = 0; t < H; ++t) {
            const LayerParam& L = pl.layers[static_cast<size_t>(t)];
            const bool pulled = pull_on && L.pull && t >= 1 && L.dense_size <= 8 * T;
            if (!pulled) {
                if (!run) run0 = off;
                run += L.dense_size;
            }
            if ((pulled || t + 1 == H) && run) {
                VCS_CUDA(cudaMemsetAsync(sp->rank_tables.p + run0, 0xff, run * sizeof(uint32_t), s));
                run = 0;
            }
            off += L.dense_size;
        }
    }
    DevBuf<uint32_t> tables, bsum;
    DevBuf<uint64_t> desc;
    DevBuf<uint32_t> jfirst;
    DevBuf<uint64_t> stamps;
    DevBuf<uint64_t> info;
    DevBuf<int32_t> status;
    tables.exact(2 * dense_max, s);
    bsum.exact(static_cast<size_t>(G) * max_rounds, s);
    desc.exact(n_max, s);
    jfirst.exact(n_max, s);
    info.exact(2 * static_cast<size_t>(H) + 2, s);
    status.exact(1, s);
    sp->params_dev.exact(static_cast<size_t>(H), s); // kept: the implicit-CSR solver reads it
    VCS_CUDA(cudaMemcpyAsync(sp->params_dev.p, pl.layers.data(), H * sizeof(LayerParam),
                             cudaMemcpyHostToDevice, s));
    VCS_CUDA(cudaMemcpyAsync(sp->keys.p, pl.init_key.data(), pl.words[0] * sizeof(uint64_t),
                             cudaMemcpyHostToDevice, s));
    VCS_CUDA(cudaMemsetAsync(tables.p, 0xff, 2 * dense_max * sizeof(uint32_t), s));
    VCS_CUDA(cudaMemsetAsync(status.p, 0, sizeof(int32_t), s));
    VCS_CUDA(cudaMemsetAsync(info.p, 0, (2 * static_cast<size_t>(H) + 2) * sizeof(uint64_t), s));
    DenseBuild A{};
    A.params = sp->params_dev.p;
    A.keys = sp->keys.p;
    A.row_ptr = sp->row_ptr.p;
    A.succ = sp->succ.p;
    A.reward = sp->reward.p;
    A.action = sp->action.p;
    A.table0 = tables.p;
    A.table1 = tables.p + dense_max;
    A.rank_tables = sp->rank_tables.p;
    A.bsum = bsum.p;
    A.desc = desc.p;
    A.jfirst = jfirst.p;
    if (trace_enabled()) {
        stamps.exact(6 * static_cast<size_t>(H) + 6, s);
        A.stamps = stamps.p;
    }
    A.info = info.p;
    A.status = status.p;
    A.state_cap = state_cap;
    A.dense_max = static_cast<uint32_t>(dense_max);
    A.max_rounds = max_rounds;
    A.H = H;
    A.pull = (G <= kPullMaxBlocks && !std::getenv("VCS_BUILD_NO_PULL")) ? 1 : 0; // (as above)
    void* args[] = {&A};
    const double t_launch = trace_enabled() ? host_ms() : 0.0;
    VCS_CUDA(cudaLaunchCooperativeKernel(fn, G, kDenseThreads, args, 0, s));
    VCS_LAUNCHED();
    std::vector<uint64_t> hinfo(2 * static_cast<size_t>(H) + 2);
    int32_t hstatus = 0;
    VCS_CUDA(cudaMemcpyAsync(hinfo.data(), info.p, hinfo.size() * sizeof(uint64_t),
                             cudaMemcpyDeviceToHost, s));
    VCS_CUDA(cudaMemcpyAsync(&hstatus, status.p, sizeof hstatus, cudaMemcpyDeviceToHost, s));
    VCS_CUDA(cudaStreamSynchronize(s));
    if (trace_enabled())
        std::fprintf(stderr, "[vcs build] persistent dense builder: %d blocks, setup %.3f ms, "
                             "kernel %.3f ms\n", G, t_launch - t_setup, host_ms() - t_launch);
    if (trace_enabled() && stamps.p) {
        std::vector<uint64_t> st(6 * static_cast<size_t>(H));
        VCS_CUDA(cudaMemcpy(st.data(), stamps.p, st.size() * 8, cudaMemcpyDeviceToHost));
        double ph[5] = {};
        for (int t = 0; t < H; ++t) {
            const uint64_t end = t + 1 < H ? st[6 * (t + 1)] : st[6 * t + 4];
            for (int k = 0; k < 5; ++k) {
                const uint64_t a = st[6 * t + k], b = k < 4 ? st[6 * t + k + 1] : end;
                if (b > a) ph[k] += (b - a) * 1e-6;
            }
        }
        std::fprintf(stderr, "[vcs build] phase ms: degrees %.3f emit %.3f flags %.3f ranks %.3f "
                             "succ+next-layer-start %.3f\n", ph[0], ph[1], ph[2], ph[3], ph[4]);
    }
    if (hstatus == 1)
        raise(VCS_ECAP, "reachable state space exceeds cap of " + std::to_string(state_cap) +
                            " states");
    if (hstatus == 2) raise(VCS_EINVAL, "more than 2^32-1 states are not supported");
    sp->layer_off.assign(static_cast<size_t>(H) + 2, 0);
    sp->layer_edges.assign(static_cast<size_t>(H) + 1, 0);
    sp->key_off.assign(static_cast<size_t>(H) + 2, 0);
    sp->max_layer = 0;
    uint64_t S = 0, E = 0;
    for (int t = 0; t <= H; ++t) {
        const uint64_t n = hinfo[static_cast<size_t>(t)];
        sp->layer_off[static_cast<size_t>(t)] = S;
        sp->key_off[static_cast<size_t>(t) + 1] =
            sp->key_off[static_cast<size_t>(t)] + n * static_cast<uint64_t>(pl.words[static_cast<size_t>(t)]);
        S += n;
        sp->max_layer = std::max(sp->max_layer, n);
        if (t < H) {
            sp->layer_edges[static_cast<size_t>(t)] = hinfo[static_cast<size_t>(H) + 1 + t];
            E += sp->layer_edges[static_cast<size_t>(t)];
        }
    }
    sp->layer_off[static_cast<size_t>(H) + 1] = S;
    sp->S = S;
    sp->E = E;
    sp->rank_off.assign(static_cast<size_t>(H) + 1, 0);
    for (int t = 0; t < H; ++t)
        sp->rank_off[static_cast<size_t>(t) + 1] =
            sp->rank_off[static_cast<size_t>(t)] + pl.layers[static_cast<size_t>(t)].dense_size;
    sp->implicit = true;     // keys + rank tables + params_dev
    sp->csr_ready = EXPLICIT; // (ensure_csr re-runs the build with EXPLICIT to materialise)
    return true;
}

// ---- single-CTA builder for small spaces (every layer <= kSmallStates / WM states) ---------------
// The whole layered BFS of mdp.cpp:81-214 in ONE block and ONE launch: the frontier keys, the
// layer's successor keys and the first-occurrence hash table live in shared memory, so a layer
// costs a handful of block barriers instead of a host round trip (the canonical instance: 330
// layers of at most 614 states).  Same edge order (clouds by key position, paid last), same
// first-insertion numbering (the lowest edge index of a successor ranks it), same reward
// operations — the CSR it writes is bit-identical to the layered builder's.  A layer larger than
// the shared-memory tables aborts with status 3 and the host takes the layered path.
constexpr int kSmallStates = 1024; // per layer, divided by the key words
constexpr int kSmallEdges = 4096;  // per layer, divided by the key words
constexpr int kSmallThreadsDefault = 512;

struct SmallBuild {
    const LayerParam* params; // H
    uint64_t* keys;           // all layers' packed keys (the layer-0 key is preset)
    uint32_t* row_ptr;
    uint32_t* succ;
    double* reward;
    int32_t* action;
    uint64_t* info;           // out: n_t for t = 0..H, then E_t for t = 0..H-1
    int32_t* status;          // out: 0 ok, 1 state cap, 2 > 2^32-1, 3 a layer overflowed
    uint64_t state_cap;
    uint64_t edge_cap;        // room in succ / reward / action
    uint64_t state_room;      // room in row_ptr / keys (states)
    int H;
    long long* cycles;        // VCS_TRACE: clock64 at the six phase boundaries of every layer
};

// Exclusive scan of v over the block with ONE barrier: warp scans, the warp totals in `ws`
// (NT / 32 entries; alternate two arrays between consecutive scans so that no trailing barrier
// is needed), then every thread sums the totals of the warps before its own.
template <int NT>
__device__ __forceinline__ uint32_t block_exscan1(uint32_t v, uint32_t* ws, uint32_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    static_assert(NT % 128 == 0, "warp totals are read four at a time");
    uint32_t before = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < NT / 32; k += 4) {
        const uint4 s = *reinterpret_cast<const uint4*>(ws + k);
        before += (k < w ? s.x : 0u) + (k + 1 < w ? s.y : 0u) + (k + 2 < w ? s.z : 0u) +
                  (k + 3 < w ? s.w : 0u);
        tot += s.x + s.y + s.z + s.w;
    }
    *total = tot;
    return before + x - v;
}

// A thread owns a contiguous run of the layer's states (spt = ceil(n / NT) of them) while it
// emits their edges (one scan numbers them), then a contiguous run of ceil(E_t / NT) edges while
// they are hashed and ranked (one scan orders the first occurrences): five block barriers per
// layer, and no thread hashes a high-degree state's edges alone.  The successor key of every edge is derived from the state's paid successor (one pass over the key's fields
// per state): a kept cloud subtracts demand from its field, a retiring one from the retired sum
// (small integers: the double sums are exact, the reward's two rounded operations are the
// reference's).
template <int WM, int NT>
__global__ void __launch_bounds__(NT, 1) k_build_small(SmallBuild A) {
    constexpr int NS = kSmallStates / WM;
    constexpr int NE = kSmallEdges / WM;
    constexpr int TC = 2 * NE; // table slots (power of two)
    constexpr int RS = (NS + NT - 1) / NT; // states per thread at most
    extern __shared__ __align__(16) unsigned char small_raw[];
    uint64_t* front = reinterpret_cast<uint64_t*>(small_raw);            // NS * WM
    uint64_t* ekey = front + static_cast<size_t>(NS) * WM;               // NE * WM
    uint32_t* table = reinterpret_cast<uint32_t*>(ekey + static_cast<size_t>(NE) * WM); // TC
    uint32_t* trank = table + TC;                                        // TC
    uint32_t* slot_of = trank + TC;                                      // NE
    __shared__ __align__(16) uint32_t ws[2][NT / 32];
    __shared__ __align__(16) LayerParam Lbuf[2]; // layer t's parameters, and t+1's behind it
    static_assert(offsetof(LayerParam, fdesc) % 16 == 0 && sizeof(LayerParam) % 16 == 0,
                  "field descriptors are read as uint4");
    const int tid = threadIdx.x;
    constexpr int PW = static_cast<int>(sizeof(LayerParam) / 4);
    constexpr int PWT = (PW + NT - 1) / NT; // parameter words per thread
    const uint32_t* pw = reinterpret_cast<const uint32_t*>(A.params);
    for (int i = tid; i < PW; i += NT) reinterpret_cast<uint32_t*>(&Lbuf[0])[i] = pw[i];
    uint32_t pf[PWT]; // the parameters of layer t + 1, loaded one layer ahead
#pragma unroll
    for (int k = 0; k < PWT; ++k) {
        const int i = tid + k * NT;
        pf[k] = (A.H > 1 && i < PW) ? __ldg(pw + PW + i) : 0u;
    }
    for (int i = tid; i < TC; i += NT) table[i] = kEmpty32;
    for (int w = tid; w < WM; w += NT) front[w] = A.keys[w];
    uint64_t S = 1, E = 0, key_base = 0; // states through the current layer / edges before it
    uint32_t n = 1;
    if (tid == 0) A.info[0] = 1;
    __syncthreads();
    for (int t = 0; t < A.H; ++t) {
        const LayerParam& L = Lbuf[t & 1];
        // layer t+1's parameters into the other buffer (last read during layer t-1, whose
        // phases ended at its third barrier), then fetch layer t+2's
        if (t + 1 < A.H) {
#pragma unroll
            for (int k = 0; k < PWT; ++k) {
                const int i = tid + k * NT;
                if (i < PW) reinterpret_cast<uint32_t*>(&Lbuf[(t + 1) & 1])[i] = pf[k];
            }
            if (t + 2 < A.H) {
#pragma unroll
                for (int k = 0; k < PWT; ++k) {
                    const int i = tid + k * NT;
                    if (i < PW) pf[k] = __ldg(pw + static_cast<size_t>(t + 2) * PW + i);
                }
            }
        }
        const int words = L.words, nw = L.next_words, na = L.n_active, dem = L.demand;
        auto tick = [&](int k) {
            if (A.cycles && tid == 0) A.cycles[6 * t + k] = clock64();
        };
        tick(0);
        const uint32_t spt = (n + NT - 1) / NT;
        const uint32_t i0 = static_cast<uint32_t>(tid) * spt;
        // A. per state: valid-cloud mask, paid successor key, retired VMs (four fields per
        //    step: the shared-memory loads of a step are independent)
        uint64_t mask[RS], nk0[RS][WM];
        int ret0[RS];
        uint32_t deg = 0;
#pragma unroll
        for (int r = 0; r < RS; ++r) {
            const uint32_t i = i0 + r;
            mask[r] = 0;
            ret0[r] = 0;
#pragma unroll
            for (int w = 0; w < WM; ++w) nk0[r][w] = 0ull;
            if (static_cast<uint32_t>(r) >= spt || i >= n) continue;
            uint64_t k[WM];
            load_key<WM>(front + static_cast<size_t>(i) * WM, words, k);
            // (the descriptors past n_active are 0: zero-width retired fields, adding nothing)
            for (int q0 = 0; q0 < na; q0 += 4) {
                const uint4 f4 = *reinterpret_cast<const uint4*>(L.fdesc + q0);
                const uint32_t fd[4] = {f4.x, f4.y, f4.z, f4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t f = fd[u];
                    const int v = get_field<WM>(k, f & 511u, (f >> 9) & 63u);
                    if (((f >> 15) & 1u) && v >= dem) mask[r] |= 1ull << (q0 + u);
                    if ((f >> 16) & 1u)
                        put_field<WM>(nk0[r], (f >> 17) & 511u, static_cast<uint64_t>(v));
                    else
                        ret0[r] += v;
                }
            }
            deg += static_cast<uint32_t>(__popcll(mask[r])) + 1u;
        }
        uint32_t E_t = 0;
        const uint32_t e0 = block_exscan1<NT>(deg, ws[0], &E_t); // barrier 1
        tick(1);
        if (E_t > static_cast<uint32_t>(NE) || E + E_t > A.edge_cap) {
            if (tid == 0) *A.status = 3;
            return;
        }
        // B. emit: successor keys to shared memory, rewards / actions / row offsets to HBM
        {
            const double r_paid = L.r_paid, r_cloud = L.r_cloud, gam = L.gamma;
            uint32_t j = e0;
#pragma unroll
            for (int r = 0; r < RS; ++r) {
                const uint32_t i = i0 + r;
                if (static_cast<uint32_t>(r) >= spt || i >= n) continue;
                A.row_ptr[S - n + i] = static_cast<uint32_t>(E + j);
                for (uint64_t m = mask[r];; m &= m - 1) {
                    const int p = m ? __ffsll(static_cast<long long>(m)) - 1 : -1;
                    uint64_t* dst = ekey + static_cast<size_t>(j) * WM;
                    int ret = ret0[r];
                    uint64_t nk[WM];
#pragma unroll
                    for (int w = 0; w < WM; ++w) nk[w] = nk0[r][w];
                    int act = -1;
                    if (p >= 0) {
                        const uint32_t f = L.fdesc[p];
                        act = L.cloud[p];
                        if ((f >> 16) & 1u) {
                            const int off = static_cast<int>((f >> 17) & 511u);
#pragma unroll
                            for (int w = 0; w < WM; ++w)
                                if (w == (off >> 6)) nk[w] -= static_cast<uint64_t>(dem) << (off & 63);
                        } else {
                            ret -= dem;
                        }
                    }
#pragma unroll
                    for (int w = 0; w < WM; ++w) dst[w] = nk[w];
                    A.reward[E + j] = __dsub_rn(p < 0 ? r_paid : r_cloud, __dmul_rn(gam, static_cast<double>(ret)));
                    A.action[E + j] = act;
                    ++j;
                    if (p < 0) break;
                }
            }
        }
        __syncthreads(); // barrier 2
        tick(2);
        // first-occurrence table: the lowest edge number of every successor key.  From here on
        // a thread owns a contiguous run of ept edges (balanced, whatever the states' degrees)
        const uint32_t ept = (E_t + NT - 1) / NT;
        const uint32_t j0 = min(static_cast<uint32_t>(tid) * ept, E_t);
        const uint32_t j1 = min(j0 + ept, E_t);
        for (uint32_t j = j0; j < j1; ++j) {
            uint64_t k[WM];
            load_key<WM>(ekey + static_cast<size_t>(j) * WM, nw, k);
            // (single-word keys: one multiply-shift — the slot is table-internal, the numbering
            // depends only on the minimum edge of each key)
            uint32_t h = WM == 1 ? static_cast<uint32_t>((k[0] * 0x9e3779b97f4a7c15ull) >> 40) & (TC - 1)
                                 : static_cast<uint32_t>(hash_key<WM>(k, nw, 0)) & (TC - 1);
            for (;;) {
                uint32_t cur = table[h];
                if (cur == kEmpty32) {
                    const uint32_t prev = atomicCAS(&table[h], kEmpty32, j);
                    if (prev == kEmpty32) break;
                    cur = prev;
                }
                if (key_equal<WM>(ekey + static_cast<size_t>(cur) * WM, nw, k)) {
                    if (cur > j) atomicMin(&table[h], j);
                    break;
                }
                h = (h + 1) & (TC - 1);
            }
            slot_of[j] = h;
        }
        __syncthreads(); // barrier 3
        tick(3);
        // C. ranks of the first occurrences in edge order = the reference's insertion order
        uint32_t firsts = 0;
        for (uint32_t j = j0; j < j1; ++j) firsts += table[slot_of[j]] == j ? 1u : 0u;
        uint32_t n_next = 0;
        uint32_t rk = block_exscan1<NT>(firsts, ws[1], &n_next); // barrier 4
        tick(4);
        if (S + n_next > A.state_cap || S + n_next > A.state_room || n_next > static_cast<uint32_t>(NS)) {
            if (tid == 0) *A.status = S + n_next > A.state_cap ? 1 : 3;
            return;
        }
        const uint64_t next_key_base = key_base + static_cast<uint64_t>(n) * words;
        for (uint32_t j = j0; j < j1; ++j) {
            const uint32_t h = slot_of[j];
            if (table[h] != j) continue;
            trank[h] = rk;
#pragma unroll
            for (int w = 0; w < WM; ++w) {
                const uint64_t x = w < nw ? ekey[static_cast<size_t>(j) * WM + w] : 0ull;
                front[static_cast<size_t>(rk) * WM + w] = x;
                if (w < nw) A.keys[next_key_base + static_cast<uint64_t>(rk) * nw + w] = x;
            }
            ++rk;
        }
        __syncthreads(); // barrier 5
        tick(5);
        // D. successor ids; the first occurrences clear their table slots
        for (uint32_t j = j0; j < j1; ++j) {
            const uint32_t h = slot_of[j];
            A.succ[E + j] = static_cast<uint32_t>(S + trank[h]);
            if (table[h] == j) table[h] = kEmpty32;
        }
        if (tid == 0) {
            A.info[t + 1] = n_next;
            A.info[A.H + 1 + t] = E_t;
        }
        E += E_t;
        S += n_next;
        key_base = next_key_base;
        n = n_next;
    }
    // the terminal layer's rows have no edges (mdp.cpp:207-209)
    for (uint32_t i = tid; i <= n; i += NT) A.row_ptr[S - n + i] = static_cast<uint32_t>(E);
    if (tid == 0) *A.status = 0;
}

// Rank table of transition t (the implicit form): key-space index of layer t+1 -> layer-local
// BFS index (the rank of the successor's first edge), empty where no state was reached.
__global__ void k_rank_table(const uint32_t* __restrict__ first_edge,
                             const uint32_t* __restrict__ rank, uint32_t n,
                             uint32_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t f = first_edge[i];
    out[i] = f == kEmpty32 ? kEmpty32 : rank[f];
}

void raise_smem_limit_space(const void* fn, int device, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, size_t> set;
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = set[{fn, device}];
    if (smem <= cur) return;
    VCS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    cur = smem;
}

// Every layer of a dense plan fits k_build_small's tables by its key-space bound (n_{t+1} <=
// dense_size_t, E_t <= n_t * out-degree bound).
template <int WM>
bool small_dense_fits(const LayerPlan& pl) {
    constexpr uint64_t NS = kSmallStates / WM, NE = kSmallEdges / WM;
    uint64_t n = 1;
    for (const LayerParam& L : pl.layers) {
        if (!L.dense_size || L.dense_size > NS) return false;
        int maxdeg = 1;
        for (int p = 0; p < L.n_active; ++p) maxdeg += L.attr[p] ? 1 : 0;
        if (n * static_cast<uint64_t>(maxdeg) > NE) return false;
        n = L.dense_size;
    }
    return !pl.layers.empty();
}

// Host side of k_build_small: returns false (nothing kept) when the space is not small.
template <int WM>
bool build_small(vcs_space* sp, uint64_t state_cap) {
    const LayerPlan& pl = sp->plan;
    const int H = pl.horizon;
    if (H < 1 || H > 4096 || std::getenv("VCS_BUILD_LAYERED") || std::getenv("VCS_NO_SMALL_BUILD"))
        return false;
    const double t_setup = trace_enabled() ? host_ms() : 0.0;
    constexpr int NS = kSmallStates / WM, NE = kSmallEdges / WM, TC = 2 * NE;
    const size_t smem = static_cast<size_t>(NS) * WM * 8 + static_cast<size_t>(NE) * WM * 8 +
                        static_cast<size_t>(TC) * 8 + static_cast<size_t>(NE) * 4;
    const uint64_t state_room = std::min<uint64_t>(static_cast<uint64_t>(H) * NS + 1, state_cap + NS);
    const uint64_t edge_room = static_cast<uint64_t>(H) * NE;
    if (edge_room >= 0xffffffffull || state_room >= 0xffffffffull) return false;
    cudaStream_t s = sp->stream;
    // block size: 512 threads (VCS_SMALL_THREADS = 128 / 256 / 1024 for measurements; C1
    // canonical: 1.10 ms at 512 against 1.24 at 256 and 1.54 at 1024)
    int nt = kSmallThreadsDefault;
    if (const char* e = std::getenv("VCS_SMALL_THREADS")) nt = std::atoi(e);
    if (nt != 1024 && nt != 256 && nt != 128) nt = 512;
    const void* fn = nt == 1024 ? reinterpret_cast<const void*>(k_build_small<WM, 1024>)
                     : nt == 256 ? reinterpret_cast<const void*>(k_build_small<WM, 256>)
                     : nt == 128 ? reinterpret_cast<const void*>(k_build_small<WM, 128>)
                                 : reinterpret_cast<const void*>(k_build_small<WM, 512>);
    raise_smem_limit_space(fn, sp->device, smem);
    sp->keys.reserve(state_room * WM, 0, s);
    sp->row_ptr.reserve(state_room + 1, 0, s);
    sp->succ.reserve(edge_room, 0, s);
    sp->reward.reserve(edge_room, 0, s);
    sp->action.reserve(edge_room, 0, s);
    DevBuf<LayerParam> params;
    DevBuf<uint64_t> info;
    DevBuf<int32_t> status;
    params.exact(static_cast<size_t>(H), s);
    info.exact(2 * static_cast<size_t>(H) + 2, s);
    status.exact(1, s);
    VCS_CUDA(cudaMemcpyAsync(params.p, pl.layers.data(), H * sizeof(LayerParam),
                             cudaMemcpyHostToDevice, s));
    VCS_CUDA(cudaMemcpyAsync(sp->keys.p, pl.init_key.data(), pl.words[0] * sizeof(uint64_t),
                             cudaMemcpyHostToDevice, s));
    VCS_CUDA(cudaMemsetAsync(status.p, 0xff, sizeof(int32_t), s));
    SmallBuild A{};
    A.params = params.p;
    A.keys = sp->keys.p;
    A.row_ptr = sp->row_ptr.p;
    A.succ = sp->succ.p;
    A.reward = sp->reward.p;
    A.action = sp->action.p;
    A.info = info.p;
    A.status = status.p;
    A.state_cap = state_cap;
    A.edge_cap = edge_room;
    A.state_room = state_room;
    A.H = H;
    DevBuf<long long> cycles;
    if (trace_enabled()) {
        cycles.exact(6 * static_cast<size_t>(H) + 6, s);
        A.cycles = cycles.p;
    }
    void* args[] = {&A};
    const double t_launch = trace_enabled() ? host_ms() : 0.0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (trace_enabled()) {
        cudaEventCreate(&ev0);
        cudaEventCreate(&ev1);
        cudaEventRecord(ev0, s);
    }
    VCS_CUDA(cudaLaunchKernel(fn, dim3(1), dim3(nt), args, smem, s));
    VCS_LAUNCHED();
    if (trace_enabled()) cudaEventRecord(ev1, s);
    std::vector<uint64_t> hinfo(2 * static_cast<size_t>(H) + 2);
    int32_t hstatus = -1;
    VCS_CUDA(cudaMemcpyAsync(hinfo.data(), info.p, hinfo.size() * sizeof(uint64_t),
                             cudaMemcpyDeviceToHost, s));
    VCS_CUDA(cudaMemcpyAsync(&hstatus, status.p, sizeof hstatus, cudaMemcpyDeviceToHost, s));
    VCS_CUDA(cudaStreamSynchronize(s));
    if (trace_enabled()) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev0, ev1);
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
        std::fprintf(stderr, "[vcs build] small builder (%d threads): setup %.3f ms, kernel %.3f ms, "
                     "launch to results %.3f ms, status %d\n", nt, t_launch - t_setup, ms,
                     host_ms() - t_launch, hstatus);
        if (hstatus == 0) {
            std::vector<long long> c(6 * static_cast<size_t>(H));
            VCS_CUDA(cudaMemcpy(c.data(), cycles.p, c.size() * 8, cudaMemcpyDeviceToHost));
            double ph[6] = {};
            for (int t = 0; t + 1 < H; ++t)
                for (int k = 0; k < 6; ++k)
                    ph[k] += static_cast<double>((k < 5 ? c[6 * t + k + 1] : c[6 * (t + 1)]) - c[6 * t + k]);
            std::fprintf(stderr, "[vcs build] small builder kcycles: fields+scan %.0f emit %.0f hash %.0f "
                         "firsts+scan %.0f ranks %.0f succ %.0f (layers 0..%d)\n", ph[0] * 1e-3,
                         ph[1] * 1e-3, ph[2] * 1e-3, ph[3] * 1e-3, ph[4] * 1e-3, ph[5] * 1e-3, H - 2);
        }
    }
    if (hstatus == 1)
        raise(VCS_ECAP, "reachable state space exceeds cap of " + std::to_string(state_cap) +
                            " states");
    if (hstatus != 0) return false; // a layer outgrew the shared-memory tables
    sp->layer_off.assign(static_cast<size_t>(H) + 2, 0);
    sp->layer_edges.assign(static_cast<size_t>(H) + 1, 0);
    sp->key_off.assign(static_cast<size_t>(H) + 2, 0);
    sp->max_layer = 0;
    uint64_t S = 0, E = 0;
    for (int t = 0; t <= H; ++t) {
        const uint64_t n = hinfo[static_cast<size_t>(t)];
        sp->layer_off[static_cast<size_t>(t)] = S;
        sp->key_off[static_cast<size_t>(t) + 1] =
            sp->key_off[static_cast<size_t>(t)] + n * static_cast<uint64_t>(pl.words[static_cast<size_t>(t)]);
        S += n;
        sp->max_layer = std::max(sp->max_layer, n);
        if (t < H) {
            sp->layer_edges[static_cast<size_t>(t)] = hinfo[static_cast<size_t>(H) + 1 + t];
            E += sp->layer_edges[static_cast<size_t>(t)];
        }
    }
    sp->layer_off[static_cast<size_t>(H) + 1] = S;
    sp->S = S;
    sp->E = E;
    sp->implicit = false;
    sp->csr_ready = true;
    return true;
}

// The layered build can produce the implicit form too (IMPLICIT: every layer dense, <= 7 active
// clouds): a layer's CSR lives in scratch only long enough to rank its successors, then the
// rank table is extracted; only keys + rank tables + params stay resident.  This is the path
// for spaces the persistent builder declines (more than 8 rounds of states per layer, e.g. C7's
// 4.8 M-state layers).
bool implicit_layered_ok(const LayerPlan& pl) {
    if (pl.horizon < 1) return false;
    for (const auto& L : pl.layers)
        if (!L.dense_size || L.n_active > kDenseSlots - 1) return false;
    return true;
}

// Per layer: count -> scan -> emit -> insert -> mark -> scan -> finalize -> counters, with the
// edge-side launches sized by the host-known bound E_t <= n_t * max_degree_t (the kernels read
// the exact E_t from device memory), and ONE stream synchronisation at the end of the layer.
template <int WM, bool IMPLICIT = false>
void build_layers(vcs_space* sp, uint64_t state_cap) {
    const double t_setup = trace_enabled() ? host_ms() : 0.0;
    const LayerPlan& pl = sp->plan;
    const int H = pl.horizon;
    cudaStream_t s = sp->stream;
    Scratch sc;

    if (H > 0) {
        sc.params.exact(static_cast<size_t>(H), s);
        VCS_CUDA(cudaMemcpyAsync(sc.params.p, pl.layers.data(), H * sizeof(LayerParam),
                                 cudaMemcpyHostToDevice, s));
    }
    sp->layer_off.assign(static_cast<size_t>(H) + 2, 0);
    sp->layer_edges.assign(static_cast<size_t>(H) + 1, 0);
    sp->key_off.assign(static_cast<size_t>(H) + 2, 0);
    // Upper bounds of the space: n_{t+1} <= min(dense key-space size, n_t * maxdeg_t, cap).
    // When they are affordable the CSR arrays are allocated once at the bound (the same few
    // pool requests on every build, no growth copies); otherwise they grow geometrically.
    uint64_t s_bound = 1, e_bound = 0, k_bound = static_cast<uint64_t>(pl.words[0]);
    {
        uint64_t nb = 1;
        for (int t = 0; t < H && e_bound < (1ull << 40); ++t) {
            const LayerParam& L = pl.layers[static_cast<size_t>(t)];
            int maxdeg = 1;
            for (int p = 0; p < L.n_active; ++p) maxdeg += L.attr[p] ? 1 : 0;
            e_bound += nb * static_cast<uint64_t>(maxdeg);
            nb = std::min<uint64_t>(nb * static_cast<uint64_t>(maxdeg), state_cap);
            if (L.dense_size) nb = std::min<uint64_t>(nb, L.dense_size);
            s_bound += nb;
            k_bound += nb * static_cast<uint64_t>(L.next_words);
        }
    }
    const bool presize = !std::getenv("VCS_BUILD_NO_PRESIZE") && // (tests: the growth path)
                         e_bound < 0xffffffffull && s_bound < 0xffffffffull &&
                         (IMPLICIT ? 0 : e_bound * 16 + s_bound * 4) + k_bound * 8 <=
                             device_bytes(sp->device) / 8;
    sp->keys.reserve(presize ? k_bound : 1u << 20, 0, s);
    VCS_CUDA(cudaMemcpyAsync(sp->keys.p, pl.init_key.data(), pl.words[0] * sizeof(uint64_t),
                             cudaMemcpyHostToDevice, s));
    // IMPLICIT: one layer's CSR in scratch (rank_off: per transition, dense_size entries)
    DevBuf<uint32_t> lay_row_ptr, lay_succ;
    DevBuf<double> lay_reward;
    DevBuf<int32_t> lay_action;
    if (IMPLICIT) {
        sp->rank_off.assign(static_cast<size_t>(H) + 1, 0);
        for (int t = 0; t < H; ++t)
            sp->rank_off[static_cast<size_t>(t) + 1] =
                sp->rank_off[static_cast<size_t>(t)] + pl.layers[static_cast<size_t>(t)].dense_size;
        sp->rank_tables.exact(std::max<uint64_t>(sp->rank_off.back(), 1), s);
    } else {
        sp->row_ptr.reserve(presize ? s_bound + 1 : 1u << 20, 0, s);
        sp->succ.reserve(presize ? e_bound : 1u << 20, 0, s);
        sp->reward.reserve(presize ? e_bound : 1u << 20, 0, s);
        sp->action.reserve(presize ? e_bound : 1u << 20, 0, s);
    }

    uint64_t S = 1, E = 0, n_t = 1;
    sp->max_layer = 1;
    constexpr uint32_t T = 256;
    const bool pull = !std::getenv("VCS_BUILD_NO_PULL");
    double t_last = host_ms();
    if (trace_enabled())
        std::fprintf(stderr, "[vcs build] setup %.3f ms (presize %d: S<=%llu E<=%llu)\n",
                     t_last - t_setup, presize ? 1 : 0, static_cast<unsigned long long>(s_bound),
                     static_cast<unsigned long long>(e_bound));
    for (int t = 0; t < H; ++t) {
        const LayerParam& L = pl.layers[static_cast<size_t>(t)];
        sp->layer_off[static_cast<size_t>(t) + 1] = S;
        const uint64_t key_t = sp->key_off[static_cast<size_t>(t)];
        sp->key_off[static_cast<size_t>(t) + 1] = key_t + n_t * static_cast<uint64_t>(L.words);
        int maxdeg = 1;
        for (int p = 0; p < L.n_active; ++p) maxdeg += L.attr[p] ? 1 : 0;
        const uint64_t e_ub = n_t * static_cast<uint64_t>(maxdeg); // E_t <= e_ub
        if (E + e_ub >= 0xffffffffull)
            raise(VCS_EINVAL, "more than 2^32-1 transitions are not supported");

        if (IMPLICIT && pull && L.pull && t >= 1) {
            // pull form: no per-layer CSR scratch, no atomic per edge (see k_pull_first)
            const uint32_t Dn = L.dense_size;
            const uint64_t nw = (n_t * 8 + 31) / 32;
            const uint64_t key_next = sp->key_off[static_cast<size_t>(t) + 1];
            sp->keys.reserve(key_next + static_cast<uint64_t>(Dn) * L.next_words, key_next, s);
            sc.table.exact(Dn, s); // first edge per successor index
            sc.eidx.exact(nw, s);  // edge-key bitmap (a cleared bit = a first edge)
            sc.rank.exact(nw + 1, s);
            sc.edge_count.exact(1, s);
            VCS_CUDA(cudaMemsetAsync(sc.eidx.p, 0xff, nw * sizeof(uint32_t), s));
            VCS_CUDA(cudaMemsetAsync(sc.edge_count.p, 0, sizeof(unsigned long long), s));
            k_pull_first<<<blocks_for(Dn, T), T, 0, s>>>(
                sp->rank_tables.p + sp->rank_off[static_cast<size_t>(t) - 1], sc.params.p + t, Dn,
                sc.table.p, sc.eidx.p, sc.edge_count.p);
            VCS_LAUNCHED();
            exclusive_scan(sc,
                           thrust::make_transform_iterator(thrust::counting_iterator<uint32_t>(0),
                                                           FirstBitsOp{sc.eidx.p, static_cast<uint32_t>(nw)}),
                           sc.rank.p, nw + 1, s); // rank[nw] = n_{t+1}
            k_pull_rank<WM><<<blocks_for(Dn, T), T, 0, s>>>(
                sc.table.p, sc.eidx.p, sc.rank.p, sc.params.p + t, Dn,
                sp->rank_tables.p + sp->rank_off[static_cast<size_t>(t)], sp->keys.p + key_next);
            VCS_LAUNCHED();
            k_pull_counters<<<1, 1, 0, s>>>(sc.edge_count.p, sc.rank.p, static_cast<uint32_t>(nw),
                                            sc.counters_dev);
            VCS_LAUNCHED();
            VCS_CUDA(cudaStreamSynchronize(s)); // the layer's single host round trip
        } else if (IMPLICIT && L.dense_size == 1 && pl.words[static_cast<size_t>(t) + 1] == 1 &&
                   pl.key_bits[static_cast<size_t>(t) + 1] == 0) {
            // into a single state (no field left): only the degree sum is needed
            sc.off.exact(n_t + 1, s);
            exclusive_scan(sc,
                           thrust::make_transform_iterator(
                               thrust::counting_iterator<uint32_t>(0),
                               DegreeOp<WM>{sp->keys.p + key_t, static_cast<uint32_t>(n_t),
                                            sc.params.p + t}),
                           sc.off.p, n_t + 1, s);
            const uint64_t key_next = sp->key_off[static_cast<size_t>(t) + 1];
            sp->keys.reserve(key_next + 1, key_next, s);
            k_single_successor<<<1, 1, 0, s>>>(sc.off.p + n_t,
                                               sp->rank_tables.p + sp->rank_off[static_cast<size_t>(t)],
                                               sp->keys.p + key_next, L.next_words, sc.counters_dev);
            VCS_LAUNCHED();
            VCS_CUDA(cudaStreamSynchronize(s));
        } else {
        sc.off.exact(n_t + 1, s);
        exclusive_scan(sc,
                       thrust::make_transform_iterator(
                           thrust::counting_iterator<uint32_t>(0),
                           DegreeOp<WM>{sp->keys.p + key_t, static_cast<uint32_t>(n_t),
                                        sc.params.p + t}),
                       sc.off.p, n_t + 1, s);
        const uint32_t* e_dev = sc.off.p + n_t; // exact E_t on the device

        const uint64_t row0 = sp->layer_off[static_cast<size_t>(t)];
        // where this layer's CSR goes: the resident arrays, or (IMPLICIT) the layer scratch
        uint32_t* rp_out;
        uint32_t* succ_out;
        double* rw_out;
        int32_t* act_out;
        uint32_t ebase;
        if (IMPLICIT) {
            lay_row_ptr.exact(n_t + 1, s);
            lay_succ.exact(e_ub, s);
            lay_reward.exact(e_ub, s);
            lay_action.exact(e_ub, s);
            rp_out = lay_row_ptr.p;
            succ_out = lay_succ.p;
            rw_out = lay_reward.p;
            act_out = lay_action.p;
            ebase = 0;
        } else {
            sp->row_ptr.reserve(row0 + n_t + 1, row0, s);
            sp->succ.reserve(E + e_ub, E, s);
            sp->reward.reserve(E + e_ub, E, s);
            sp->action.reserve(E + e_ub, E, s);
            rp_out = sp->row_ptr.p + row0;
            succ_out = sp->succ.p + E;
            rw_out = sp->reward.p;
            act_out = sp->action.p;
            ebase = static_cast<uint32_t>(E);
        }
        const uint64_t key_next = sp->key_off[static_cast<size_t>(t) + 1];
        sp->keys.reserve(key_next + e_ub * static_cast<uint64_t>(L.next_words), key_next, s);
        const uint64_t cap = pow2_at_least(2 * e_ub);
        // dense successor indices when the next key space is small: a first-edge table of
        // dense_size words instead of a hash table of 2*E_t slots
        const bool dense = IMPLICIT || (L.dense_size != 0 &&
                                        static_cast<uint64_t>(L.dense_size) * 4 <=
                                            std::max<uint64_t>(16ull << 20, cap * 12));
        if (dense) {
            sc.table.exact(L.dense_size, s);
            sc.eidx.exact(e_ub, s);
            VCS_CUDA(cudaMemsetAsync(sc.table.p, 0xff, L.dense_size * sizeof(uint32_t), s));
            k_emit_dense<WM><<<blocks_for(n_t, T), T, 0, s>>>(
                static_cast<uint32_t>(n_t), sp->keys.p + key_t, sc.off.p, L, ebase, rp_out,
                sc.eidx.p, rw_out, act_out, sc.table.p);
            VCS_LAUNCHED();
            sc.rank.exact(e_ub + 1, s);
            exclusive_scan(sc,
                           thrust::make_transform_iterator(
                               thrust::counting_iterator<uint32_t>(0),
                               FirstEdgeOp{e_dev, sc.table.p, sc.eidx.p}),
                           sc.rank.p, e_ub + 1, s); // rank[E_t] = n_{t+1}
            k_finalize_dense<WM><<<blocks_for(e_ub, T), T, 0, s>>>(
                e_dev, sc.table.p, sc.eidx.p, sc.rank.p, L, static_cast<uint32_t>(S), succ_out,
                sp->keys.p + key_next);
            VCS_LAUNCHED();
            if (IMPLICIT) {
                k_rank_table<<<blocks_for(L.dense_size, T), T, 0, s>>>(
                    sc.table.p, sc.rank.p, L.dense_size,
                    sp->rank_tables.p + sp->rank_off[static_cast<size_t>(t)]);
                VCS_LAUNCHED();
            }
        } else {
            sc.ekeys.exact(e_ub * static_cast<uint64_t>(L.next_words), s);
            k_emit<WM><<<blocks_for(n_t, T), T, 0, s>>>(
                static_cast<uint32_t>(n_t), sp->keys.p + key_t, sc.off.p, L,
                static_cast<uint32_t>(E), sp->row_ptr.p + row0, sc.ekeys.p, sp->reward.p,
                sp->action.p);
            VCS_LAUNCHED();
            sc.table.exact(cap, s);
            sc.slot.exact(e_ub, s);
            VCS_CUDA(cudaMemsetAsync(sc.table.p, 0xff, cap * sizeof(uint32_t), s));
            if (L.next_words == 1 && pl.key_bits[static_cast<size_t>(t) + 1] < 64) {
                sc.tkey.exact(cap, s);
                VCS_CUDA(cudaMemsetAsync(sc.tkey.p, 0xff, cap * sizeof(uint64_t), s));
                k_insert_kv<<<blocks_for(e_ub, T), T, 0, s>>>(
                    e_dev, sc.ekeys.p, reinterpret_cast<unsigned long long*>(sc.tkey.p),
                    sc.table.p, static_cast<uint32_t>(cap - 1), sc.slot.p);
            } else {
                k_insert<WM><<<blocks_for(e_ub, T), T, 0, s>>>(
                    e_dev, sc.ekeys.p, L.next_words, sc.table.p, static_cast<uint32_t>(cap - 1),
                    sc.slot.p);
            }
            VCS_LAUNCHED();
            sc.rank.exact(e_ub + 1, s);
            exclusive_scan(sc,
                           thrust::make_transform_iterator(
                               thrust::counting_iterator<uint32_t>(0),
                               FirstEdgeOp{e_dev, sc.table.p, sc.slot.p}),
                           sc.rank.p, e_ub + 1, s); // rank[E_t] = n_{t+1}
            k_finalize<<<blocks_for(e_ub, T), T, 0, s>>>(
                e_dev, sc.table.p, sc.slot.p, sc.rank.p, sc.ekeys.p, L.next_words,
                static_cast<uint32_t>(S), sp->succ.p + E, sp->keys.p + key_next);
            VCS_LAUNCHED();
        }
        k_counters<<<1, 1, 0, s>>>(e_dev, sc.rank.p, sc.counters_dev);
        VCS_LAUNCHED();
        VCS_CUDA(cudaStreamSynchronize(s)); // the layer's single host round trip
        }
        const uint64_t E_t = sc.counters->n_edges;
        const uint64_t n_next = sc.counters->n_next;
        if (S + n_next > state_cap)
            raise(VCS_ECAP, "reachable state space exceeds cap of " + std::to_string(state_cap) +
                                " states");
        if (S + n_next >= 0xffffffffull)
            raise(VCS_EINVAL, "more than 2^32-1 states are not supported");

        sp->layer_edges[static_cast<size_t>(t)] = E_t;
        E += E_t;
        S += n_next;
        n_t = n_next;
        sp->max_layer = std::max<uint64_t>(sp->max_layer, n_t);
        if (trace_enabled()) {
            const double now = host_ms();
            std::fprintf(stderr, "[vcs build] layer %d: n=%llu E_t=%llu  %.3f ms\n", t,
                         static_cast<unsigned long long>(n_t),
                         static_cast<unsigned long long>(E_t), now - t_last);
            t_last = now;
        }
    }
    sp->layer_off[static_cast<size_t>(H) + 1] = S;
    sp->key_off[static_cast<size_t>(H) + 1] =
        sp->key_off[static_cast<size_t>(H)] + n_t * static_cast<uint64_t>(pl.words[H]);
    if (IMPLICIT) {
        sp->params_dev.exact(static_cast<size_t>(H), s); // the implicit-CSR solver reads it
        VCS_CUDA(cudaMemcpyAsync(sp->params_dev.p, pl.layers.data(), H * sizeof(LayerParam),
                                 cudaMemcpyHostToDevice, s));
        VCS_CUDA(cudaStreamSynchronize(s));
        sp->S = S;
        sp->E = E;
        sp->implicit = true;
        sp->csr_ready = false;
        if (trace_enabled()) std::fprintf(stderr, "[vcs build] final (implicit) %.3f ms\n", host_ms() - t_last);
        return;
    }
    // Terminal layer: no outgoing edges (mdp.cpp:207-209).
    const uint64_t rowH = sp->layer_off[static_cast<size_t>(H)];
    sp->row_ptr.reserve(S + 1, rowH, s);
    k_fill_u32<<<blocks_for(S + 1 - rowH, T), T, 0, s>>>(sp->row_ptr.p + rowH, S + 1 - rowH,
                                                         static_cast<uint32_t>(E));
    VCS_LAUNCHED();
    VCS_CUDA(cudaStreamSynchronize(s));
    sp->S = S;
    sp->E = E;
    if (trace_enabled()) std::fprintf(stderr, "[vcs build] final %.3f ms\n", host_ms() - t_last);
}

int words_template(int w) {
    if (w <= 1) return 1;
    if (w <= 2) return 2;
    if (w <= 4) return 4;
    return 8;
}

template <class F>
void dispatch_words(int wm, F&& f) {
    switch (words_template(wm)) {
    case 1: f(std::integral_constant<int, 1>{}); break;
    case 2: f(std::integral_constant<int, 2>{}); break;
    case 4: f(std::integral_constant<int, 4>{}); break;
    default: f(std::integral_constant<int, 8>{}); break;
    }
}

int max_words(const vcs_space* sp) {
    int wm = 1;
    for (int w : sp->plan.words) wm = std::max(wm, w);
    return wm;
}

void ensure_locate_index(vcs_space* sp) {
    if (sp->loc_cap) return;
    const uint64_t cap = pow2_at_least(2 * sp->S);
    if (cap > 0xffffffffull) raise(VCS_EINVAL, "state space too large for the locate index");
    sp->loc_table.exact(cap, sp->stream);
    cudaStream_t s = sp->stream;
    VCS_CUDA(cudaMemsetAsync(sp->loc_table.p, 0xff, cap * sizeof(uint32_t), s));
    dispatch_words(max_words(sp), [&](auto wm) {
        constexpr int WM = decltype(wm)::value;
        for (int t = 0; t <= sp->H; ++t) {
            const uint64_t n = sp->layer_off[t + 1] - sp->layer_off[t];
            if (!n) continue;
            k_loc_insert<WM><<<blocks_for(n, 256), 256, 0, s>>>(
                static_cast<uint32_t>(n), sp->keys.p + sp->key_off[t], sp->plan.words[t], t,
                static_cast<uint32_t>(sp->layer_off[t]), sp->loc_table.p,
                static_cast<uint32_t>(cap - 1));
            VCS_LAUNCHED();
        }
    });
    VCS_CUDA(cudaStreamSynchronize(s));
    sp->loc_cap = cap;
}

} // namespace

thread_local bool g_capturing = false;

void debug_sync_check(const char* file, int line) {
    static const bool on = std::getenv("VCS_SYNC_CHECK") != nullptr;
    if (!on || g_capturing) return; // inside a stream capture nothing has run yet
    const cudaError_t e = cudaDeviceSynchronize();
    if (std::getenv("VCS_SYNC_CHECK_VERBOSE"))
        std::fprintf(stderr, "[vcs sync-check] %s:%d %s\n", file, line, cudaGetErrorString(e));
    if (e != cudaSuccess) {
        std::fprintf(stderr, "[vcs sync-check] fault after the launch at %s:%d: %s\n", file, line,
                     cudaGetErrorString(e));
        raise(VCS_ECUDA, std::string("fault after launch at ") + file + ":" + std::to_string(line));
    }
}

bool trace_enabled() {
    static const bool on = std::getenv("VCS_TRACE") != nullptr;
    return on;
}

double host_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

// Materialise the explicit CSR of a space built in the implicit form: the dense builder runs
// again with EXPLICIT (same keys and layer order, bit for bit); the layered builder if the CSR
// bound is not affordable.
void ensure_csr(vcs_space* sp) {
    if (sp->csr_ready) return;
    bind_device(sp->device);
    const double t0 = trace_enabled() ? host_ms() : 0.0;
    dispatch_words(max_words(sp), [&](auto wm) {
        constexpr int WM = decltype(wm)::value;
        if (!build_dense<WM, true>(sp, sp->state_cap)) build_layers<WM>(sp, sp->state_cap);
    });
    sp->csr_ready = true;
    if (trace_enabled()) std::fprintf(stderr, "[vcs build] explicit CSR materialised in %.3f ms\n",
                                      host_ms() - t0);
}

void bind_device(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        raise(VCS_ECUDA, "no CUDA device available (the solver has no CPU fallback)");
    if (device < 0 || device >= n) raise(VCS_EINVAL, "device ordinal out of range");
    VCS_CUDA(cudaSetDevice(device));
    init_pool(device);
}

void init_pool(int device) {
    static std::once_flag once[64];
    if (device < 0 || device >= 64) return;
    std::call_once(once[device], [device] {
        cudaMemPool_t pool = nullptr;
        if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return;
        uint64_t keep = ~0ull; // keep freed blocks cached in the pool (no trim at sync points)
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    });
}

namespace {
struct BigBlock {
    void* p;
    size_t bytes;
    uint64_t stamp;
};
struct BigCache {
    std::mutex mu;
    std::vector<BigBlock> blocks[64];
    size_t bytes[64] = {};
    uint64_t clock = 0;
};
BigCache& big_cache() {
    static BigCache* c = new BigCache; // never destroyed: blocks die with the context
    return *c;
}
} // namespace

size_t device_bytes(int device) {
    static std::mutex mu;
    static size_t total[64] = {};
    if (device < 0 || device >= 64) return 0;
    std::lock_guard<std::mutex> lock(mu);
    if (!total[device]) {
        cudaDeviceProp prop{};
        if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) total[device] = prop.totalGlobalMem;
    }
    return total[device];
}

namespace {
int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}
} // namespace

void* dev_alloc(size_t bytes, cudaStream_t s, size_t* got) {
    if (bytes == 0) bytes = 1;
    const int dev = current_device();
    if (bytes >= kBigBlock && dev >= 0 && dev < 64) {
        BigCache& c = big_cache();
        std::lock_guard<std::mutex> lock(c.mu);
        auto& v = c.blocks[dev];
        size_t best = v.size();
        for (size_t i = 0; i < v.size(); ++i)
            if (v[i].bytes >= bytes && v[i].bytes <= bytes + bytes / 4 &&
                (best == v.size() || v[i].bytes < v[best].bytes))
                best = i;
        if (best != v.size()) {
            void* p = v[best].p;
            *got = v[best].bytes;
            c.bytes[dev] -= v[best].bytes;
            v.erase(v.begin() + static_cast<std::ptrdiff_t>(best));
            return p;
        }
    }
    void* p = nullptr;
    cudaError_t err = cudaMallocAsync(&p, bytes, s);
    if (err == cudaErrorMemoryAllocation && dev >= 0 && dev < 64) {
        cudaGetLastError();
        BigCache& c = big_cache(); // out of memory: drop the cache and retry once
        {
            std::lock_guard<std::mutex> lock(c.mu);
            for (auto& b : c.blocks[dev]) cudaFreeAsync(b.p, s);
            c.blocks[dev].clear();
            c.bytes[dev] = 0;
        }
        err = cudaMallocAsync(&p, bytes, s);
    }
    if (err != cudaSuccess)
        raise(VCS_ECUDA, std::string("cudaMallocAsync: ") + cudaGetErrorString(err));
    *got = bytes;
    return p;
}

void dev_release_idle(void* p, size_t bytes, cudaStream_t s) {
    const int dev = current_device();
    if (bytes < kBigBlock || dev < 0 || dev >= 64) {
        cudaFreeAsync(p, s);
        return;
    }
    const size_t limit = device_bytes(dev) / 4; // at most a quarter of the device stays cached
    BigCache& c = big_cache();
    std::lock_guard<std::mutex> lock(c.mu);
    auto& v = c.blocks[dev];
    v.push_back({p, bytes, ++c.clock});
    c.bytes[dev] += bytes;
    while (c.bytes[dev] > limit && !v.empty()) {
        size_t oldest = 0;
        for (size_t i = 1; i < v.size(); ++i)
            if (v[i].stamp < v[oldest].stamp) oldest = i;
        cudaFreeAsync(v[oldest].p, s);
        c.bytes[dev] -= v[oldest].bytes;
        v.erase(v.begin() + static_cast<std::ptrdiff_t>(oldest));
    }
}

int sm_count(int device) {
    int v = 0;
    VCS_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
    return v;
}

namespace {
struct HandlePool {
    std::mutex mu;
    std::vector<std::pair<int, cudaStream_t>> streams;
    std::vector<std::pair<int, cudaEvent_t>> events[2]; // [timing]
};
HandlePool& handle_pool() {
    static HandlePool* p = new HandlePool; // never destroyed: handles die with the context
    return *p;
}
constexpr size_t kPoolStreams = 32, kPoolEvents = 1024;
} // namespace

cudaStream_t acquire_stream(int device) {
    {
        HandlePool& P = handle_pool();
        std::lock_guard<std::mutex> lock(P.mu);
        for (size_t i = P.streams.size(); i-- > 0;)
            if (P.streams[i].first == device) {
                cudaStream_t s = P.streams[i].second;
                P.streams.erase(P.streams.begin() + static_cast<std::ptrdiff_t>(i));
                return s;
            }
    }
    cudaStream_t s = nullptr;
    VCS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    return s;
}

void release_stream(int device, cudaStream_t s) {
    if (!s) return;
    {
        HandlePool& P = handle_pool();
        std::lock_guard<std::mutex> lock(P.mu);
        if (P.streams.size() < kPoolStreams) {
            P.streams.emplace_back(device, s);
            return;
        }
    }
    cudaStreamDestroy(s);
}

cudaEvent_t acquire_event(int device, bool timing) {
    {
        HandlePool& P = handle_pool();
        std::lock_guard<std::mutex> lock(P.mu);
        auto& v = P.events[timing ? 1 : 0];
        for (size_t i = v.size(); i-- > 0;)
            if (v[i].first == device) {
                cudaEvent_t e = v[i].second;
                v.erase(v.begin() + static_cast<std::ptrdiff_t>(i));
                return e;
            }
    }
    cudaEvent_t e = nullptr;
    VCS_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
    return e;
}

void release_event(int device, cudaEvent_t e, bool timing) {
    if (!e) return;
    {
        HandlePool& P = handle_pool();
        std::lock_guard<std::mutex> lock(P.mu);
        auto& v = P.events[timing ? 1 : 0];
        if (v.size() < kPoolEvents) {
            v.emplace_back(device, e);
            return;
        }
    }
    cudaEventDestroy(e);
}

} // namespace vcs

vcs_space::~vcs_space() {
    vcs::destroy_multi(multi);
    vcs::destroy_cert_shard(cert_shard);
    cudaSetDevice(device);
    for (auto& [st, ev] : use_ev) {
        if (!ev) continue;
        cudaEventSynchronize(ev);
        cudaEventDestroy(ev);
    }
    if (stream) cudaStreamSynchronize(stream);
    if (d2h_stream) cudaStreamSynchronize(d2h_stream);
    for (auto& [k, g] : graphs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        for (auto& e : g.ev) vcs::release_event(device, e, true);
        for (auto& e : g.layer_ev) vcs::release_event(device, e, false);
    }
    for (auto e : piece_ev) vcs::release_event(device, e, false);
    vcs::release_event(device, order_ev, false);
    vcs::release_stream(device, d2h_stream);
    if (aux_stream) cudaStreamDestroy(aux_stream);
    // the stream is idle: big blocks go to the per-device cache for the next space, the rest
    // back to the pool (stream-ordered frees are issued while the stream is alive)
    row_ptr.release_idle();
    succ.release_idle();
    reward.release_idle();
    action.release_idle();
    keys.release_idle();
    v[0].release_idle();
    v[1].release_idle();
    delta.release_idle();
    ctrl.release_idle();
    actions_dev.release_idle();
    act8_dev.release_idle();
    ver.release_idle();
    cert_xd.release_idle();
    cert_act_ks.release_idle();
    stream_meta.release_idle();
    stream_sync.release_idle();
    cert_tail_meta.release_idle();
    cert_lb.release_idle();
    cert_tl.release_idle();
    band_ver.release_idle();
    ver_off.release_idle();
    layer_off_dev.release_idle();
    loc_table.release_idle();
    query_meta.release_idle();
    rank_tables.release_idle();
    params_dev.release_idle();
    // (every DevBuf member must be released above: their destructors would free on the
    // destroyed stream below)
    if (stream) {
        cudaStreamSynchronize(stream);
        vcs::release_stream(device, stream);
    }
}

using vcs::guarded;
using vcs::raise;

namespace {
std::unique_ptr<vcs_space> new_space(int device) {
    vcs::bind_device(device);
    auto sp = std::make_unique<vcs_space>();
    sp->device = device;
    sp->num_sms = vcs::sm_count(device);
    sp->stream = vcs::acquire_stream(device);
    return sp;
}
} // namespace

extern "C" {

int vcs_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int vcs_space_build(const vcs_instance* inst, uint64_t state_cap, int device, vcs_space** out) {
    return guarded([&] {
        if (!inst || !out) raise(VCS_EINVAL, "null argument");
        for (int j = 0; j < inst->n_tasks; ++j)
            if (inst->task_demand[j] < 0)
                raise(VCS_EINVAL, "negative vm_demand is not supported by the device builder");
        const double tp = vcs::trace_enabled() ? vcs::host_ms() : 0.0;
        vcs::LayerPlan plan = vcs::make_layer_plan(inst); // throws the 65535 error first
        auto sp = new_space(device);
        if (vcs::trace_enabled())
            std::fprintf(stderr, "[vcs build] plan + space %.3f ms\n", vcs::host_ms() - tp);
        sp->plan = std::move(plan);
        sp->has_plan = true;
        sp->H = sp->plan.horizon;
        int maxdeg = 1;
        for (const auto& L : sp->plan.layers) {
            int d = 1;
            for (int p = 0; p < L.n_active; ++p) d += L.attr[p] ? 1 : 0;
            maxdeg = std::max(maxdeg, d);
        }
        sp->max_degree = maxdeg;
        const auto t0 = std::chrono::steady_clock::now();
        sp->state_cap = state_cap;
        // dense spaces: the implicit-CSR form (keys + rank tables), the explicit CSR is
        // materialised on first use (vcs::ensure_csr); VCS_BUILD_EXPLICIT builds it right away
        const bool explicit_now = std::getenv("VCS_BUILD_EXPLICIT") != nullptr;
        vcs::dispatch_words(vcs::max_words(sp.get()), [&](auto wm) {
            constexpr int WM = decltype(wm)::value;
            // a tiny dense space (every layer's key space within the single-CTA tables, e.g. the
            // small C5 points) is built in one block: the cooperative grid's barriers cost more
            // than its layers
            if (vcs::small_dense_fits<WM>(sp->plan) && vcs::build_small<WM>(sp.get(), state_cap))
                return;
            const bool dense = explicit_now ? vcs::build_dense<WM, true>(sp.get(), state_cap)
                                            : vcs::build_dense<WM, false>(sp.get(), state_cap);
            if (dense) return;
            if (vcs::build_small<WM>(sp.get(), state_cap)) return;
            if (!explicit_now && !std::getenv("VCS_BUILD_LAYERED") &&
                vcs::implicit_layered_ok(sp->plan))
                vcs::build_layers<WM, true>(sp.get(), state_cap);
            else
                vcs::build_layers<WM>(sp.get(), state_cap);
        });
        const auto t1 = std::chrono::steady_clock::now();
        sp->build_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        *out = sp.release();
        return VCS_OK;
    });
}

int vcs_space_from_csr(uint64_t n_states, uint64_t n_edges, int32_t horizon,
                       const uint64_t* layer_offset, const uint64_t* row_ptr, const uint32_t* succ,
                       const double* reward, const int32_t* action, int device, vcs_space** out) {
    return guarded([&] {
        if (n_edges >= 0xffffffffull || n_states >= 0xffffffffull)
            raise(VCS_EINVAL, "more than 2^32-1 states or transitions are not supported");
        if (n_states < 1 || horizon < 0) raise(VCS_EINVAL, "empty state space");
        auto sp = new_space(device);
        sp->S = n_states;
        sp->E = n_edges;
        sp->H = horizon;
        sp->layer_off.assign(layer_offset, layer_offset + horizon + 2);
        sp->layer_edges.assign(static_cast<size_t>(horizon) + 1, 0);
        std::vector<uint32_t> rp32(n_states + 1);
        int maxdeg = 1;
        for (uint64_t i = 0; i <= n_states; ++i) {
            rp32[i] = static_cast<uint32_t>(row_ptr[i]);
            if (i < n_states)
                maxdeg = std::max<int>(maxdeg, static_cast<int>(row_ptr[i + 1] - row_ptr[i]));
        }
        for (int t = 0; t <= horizon; ++t) {
            sp->layer_edges[t] = row_ptr[sp->layer_off[t + 1]] - row_ptr[sp->layer_off[t]];
            sp->max_layer = std::max(sp->max_layer, sp->layer_off[t + 1] - sp->layer_off[t]);
        }
        sp->max_degree = maxdeg;

        cudaStream_t s = sp->stream;
        sp->row_ptr.exact(n_states + 1, sp->stream);
        sp->succ.exact(n_edges, sp->stream);
        sp->reward.exact(n_edges, sp->stream);
        sp->action.exact(n_edges, sp->stream);
        VCS_CUDA(cudaMemcpyAsync(sp->row_ptr.p, rp32.data(), rp32.size() * 4, cudaMemcpyHostToDevice, s));
        if (n_edges) {
            VCS_CUDA(cudaMemcpyAsync(sp->succ.p, succ, n_edges * 4, cudaMemcpyHostToDevice, s));
            VCS_CUDA(cudaMemcpyAsync(sp->reward.p, reward, n_edges * 8, cudaMemcpyHostToDevice, s));
            VCS_CUDA(cudaMemcpyAsync(sp->action.p, action, n_edges * 4, cudaMemcpyHostToDevice, s));
        }
        VCS_CUDA(cudaStreamSynchronize(s));
        *out = sp.release();
        return VCS_OK;
    });
}

int vcs_space_info_get(const vcs_space* sp, vcs_space_info* info) {
    return guarded([&] {
        info->n_states = sp->S;
        info->n_edges = sp->E;
        info->horizon = sp->H;
        int wm = 0;
        for (int w : sp->plan.words) wm = std::max(wm, w);
        info->key_words = wm;
        info->max_layer = sp->max_layer;
        info->max_degree = sp->max_degree;
        info->device = sp->device;
        info->build_ms = sp->build_ms;
        info->device_bytes = (sp->S + 1) * 4 + sp->E * (4 + 8 + 4) + sp->S * 16;
        return VCS_OK;
    });
}

int vcs_space_layer_offsets(const vcs_space* sp, uint64_t* layer_offset) {
    return guarded([&] {
        std::copy(sp->layer_off.begin(), sp->layer_off.end(), layer_offset);
        return VCS_OK;
    });
}

int vcs_space_layer_edges(const vcs_space* sp, uint64_t* layer_edges) {
    return guarded([&] {
        std::copy(sp->layer_edges.begin(), sp->layer_edges.end(), layer_edges);
        return VCS_OK;
    });
}

int vcs_space_csr(const vcs_space* sp, uint64_t* row_ptr, uint32_t* succ, double* reward,
                  int32_t* action) {
    return guarded([&] {
        vcs::ensure_csr(const_cast<vcs_space*>(sp));
        vcs::bind_device(sp->device);
        cudaStream_t s = sp->stream;
        if (row_ptr) {
            std::vector<uint32_t> rp(sp->S + 1);
            VCS_CUDA(cudaMemcpyAsync(rp.data(), sp->row_ptr.p, rp.size() * 4, cudaMemcpyDeviceToHost, s));
            VCS_CUDA(cudaStreamSynchronize(s));
            for (size_t i = 0; i < rp.size(); ++i) row_ptr[i] = rp[i];
        }
        if (sp->E) {
            if (succ) VCS_CUDA(cudaMemcpyAsync(succ, sp->succ.p, sp->E * 4, cudaMemcpyDeviceToHost, s));
            if (reward) VCS_CUDA(cudaMemcpyAsync(reward, sp->reward.p, sp->E * 8, cudaMemcpyDeviceToHost, s));
            if (action) VCS_CUDA(cudaMemcpyAsync(action, sp->action.p, sp->E * 4, cudaMemcpyDeviceToHost, s));
        }
        VCS_CUDA(cudaStreamSynchronize(s));
        return VCS_OK;
    });
}

int vcs_space_locate(vcs_space* sp, int64_t n, const int32_t* free_vms, const int32_t* task_index,
                     const uint8_t* terminal, int64_t* idx_out) {
    std::lock_guard<std::recursive_mutex> space_lock(sp->mu);
    return guarded([&] {
        if (!sp->has_plan) raise(VCS_EINVAL, "space was not built from an instance");
        if (n <= 0) return VCS_OK;
        vcs::bind_device(sp->device);
        const int K = sp->plan.n_clouds;
        std::vector<vcs::LocQuery> q(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            const int t = terminal[i] ? sp->H : task_index[i];
            if (t < 0 || t > sp->H) raise(VCS_EINVAL, "task index outside horizon");
            auto& Q = q[static_cast<size_t>(i)];
            std::memset(&Q, 0, sizeof Q);
            Q.layer = t;
            Q.words = sp->plan.words[t];
            Q.valid = vcs::pack_key(sp->plan, t, free_vms + i * K, Q.key) ? 1 : 0;
        }
        vcs::ensure_locate_index(sp);
        cudaStream_t s = sp->stream;
        vcs::DevBuf<vcs::LocQuery> dq;
        vcs::DevBuf<int64_t> dout;
        vcs::DevBuf<uint64_t> dmeta;
        dq.exact(static_cast<size_t>(n), sp->stream);
        dout.exact(static_cast<size_t>(n), sp->stream);
        dmeta.exact(2 * (static_cast<size_t>(sp->H) + 2), sp->stream);
        VCS_CUDA(cudaMemcpyAsync(dq.p, q.data(), q.size() * sizeof(vcs::LocQuery), cudaMemcpyHostToDevice, s));
        VCS_CUDA(cudaMemcpyAsync(dmeta.p, sp->layer_off.data(), (sp->H + 2) * 8, cudaMemcpyHostToDevice, s));
        VCS_CUDA(cudaMemcpyAsync(dmeta.p + sp->H + 2, sp->key_off.data(), (sp->H + 2) * 8, cudaMemcpyHostToDevice, s));
        vcs::dispatch_words(vcs::max_words(sp), [&](auto wm) {
            constexpr int WM = decltype(wm)::value;
            vcs::k_loc_lookup<WM><<<vcs::blocks_for(static_cast<uint64_t>(n), 128), 128, 0, s>>>(
                n, dq.p, sp->keys.p, dmeta.p, dmeta.p + sp->H + 2, sp->loc_table.p,
                static_cast<uint32_t>(sp->loc_cap - 1), dout.p);
            VCS_LAUNCHED();
        });
        VCS_CUDA(cudaMemcpyAsync(idx_out, dout.p, n * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        VCS_CUDA(cudaStreamSynchronize(s));
        return VCS_OK;
    });
}

int vcs_space_hidden_penalty(const vcs_space* sp, int64_t n, const int32_t* free_vms,
                             const int32_t* task_index, const uint8_t* terminal, double* out) {
    return guarded([&] {
        if (!sp->has_plan) raise(VCS_EINVAL, "space was not built from an instance");
        const int K = sp->plan.n_clouds;
        for (int64_t i = 0; i < n; ++i) {
            if (sp->H == 0) { // mdp.cpp:237: nothing was ever schedulable
                out[i] = 0.0;
                continue;
            }
            const int t = terminal[i] ? sp->H : task_index[i];
            double retired = 0.0;
            for (int c = 0; c < K; ++c)
                if (sp->plan.last_use[c] < t) retired += free_vms[i * K + c];
            out[i] = sp->plan.layers.empty() ? 0.0 : sp->plan.layers[0].gamma * retired;
        }
        return VCS_OK;
    });
}

namespace {
bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}
} // namespace

namespace {
// Device key layouts, last_use, layer and key offsets for the query / rollout kernels (once per
// space); returns the QueryArgs fields that point into them.
void ensure_query_meta(vcs_space* sp, vcs::QueryArgs& a) {
    const int K = sp->plan.n_clouds, H = sp->H;
    const size_t ql = sizeof(vcs::QueryLayer) * (static_cast<size_t>(H) + 1);
    const size_t lu = ((sizeof(int32_t) * std::max(K, 1) + 7) / 8) * 8;
    const size_t lo = sizeof(uint64_t) * (static_cast<size_t>(H) + 2);
    if (!sp->query_meta.p) {
            std::vector<unsigned char> blob(ql + lu + 2 * lo, 0);
            auto* layers = reinterpret_cast<vcs::QueryLayer*>(blob.data());
            for (int t = 0; t <= H; ++t) {
                auto& Q = layers[t];
                Q.n_active = static_cast<int32_t>(sp->plan.active[t].size());
                Q.words = sp->plan.words[t];
                for (int p = 0; p < Q.n_active; ++p) {
                    const int c = sp->plan.active[t][p];
                    Q.cloud[p] = static_cast<uint8_t>(c);
                    Q.bit_off[p] = sp->plan.bit_off[t][p];
                    Q.width[p] = static_cast<uint8_t>(sp->plan.width_of_cloud[c]);
                }
            }
            std::memcpy(blob.data() + ql, sp->plan.last_use.data(), sizeof(int32_t) * K);
            std::memcpy(blob.data() + ql + lu, sp->layer_off.data(), lo);
            std::memcpy(blob.data() + ql + lu + lo, sp->key_off.data(), lo);
            sp->query_meta.exact(blob.size(), sp->stream);
            VCS_CUDA(cudaMemcpyAsync(sp->query_meta.p, blob.data(), blob.size(),
                                     cudaMemcpyHostToDevice, sp->stream));
            VCS_CUDA(cudaStreamSynchronize(sp->stream));
    }
    a.layers = reinterpret_cast<const vcs::QueryLayer*>(sp->query_meta.p);
    a.last_use = reinterpret_cast<const int32_t*>(sp->query_meta.p + ql);
    a.layer_off = reinterpret_cast<const uint64_t*>(sp->query_meta.p + ql + lu);
    a.key_off = reinterpret_cast<const uint64_t*>(sp->query_meta.p + ql + lu + lo);
    a.keys = sp->keys.p;
    a.table = sp->loc_table.p;
    a.mask = static_cast<uint32_t>(sp->loc_cap - 1);
    a.values = sp->result_values;
    a.actions = sp->result_actions;
    a.n_clouds = K;
    a.H = H;
    a.gamma = sp->plan.layers.empty() ? 0.0 : sp->plan.layers[0].gamma;
}
} // namespace

int vcs_policy_query(vcs_space* sp, int64_t n, const int32_t* free_vms, const int32_t* task_index,
                     const uint8_t* terminal, double* value_out, int32_t* action_out,
                     int64_t* idx_out, void* stream) {
    std::lock_guard<std::recursive_mutex> space_lock(sp->mu);
    return guarded([&] {
        if (!sp->has_plan) raise(VCS_EINVAL, "space was not built from an instance");
        if (!sp->result_values)
            raise(VCS_EINVAL, "no solve results on this space (vcs_solve / vcs_solve_collect first)");
        if (n <= 0) return VCS_OK;
        if (!free_vms || !task_index || !terminal) raise(VCS_EINVAL, "null argument");
        vcs::bind_device(sp->device);
        const vcs::StreamUse s(sp, stream);
        vcs::ensure_locate_index(sp);
        const int K = sp->plan.n_clouds;
        vcs::QueryArgs a{};
        ensure_query_meta(sp, a);
        // host or device buffers: device ones are used in place, host ones staged
        vcs::DevBuf<int32_t> dfv, dti, dact;
        vcs::DevBuf<uint8_t> dte;
        vcs::DevBuf<double> dval;
        vcs::DevBuf<int64_t> didx;
        auto stage_in = [&](const auto* src, auto& buf, size_t count) {
            using T = std::remove_cv_t<std::remove_pointer_t<decltype(src)>>;
            if (is_device_ptr(src)) return src;
            buf.exact(count, s);
            VCS_CUDA(cudaMemcpyAsync(buf.p, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
            return static_cast<const T*>(buf.p);
        };
        auto stage_out = [&](auto* dst, auto& buf, size_t count) {
            if (!dst || is_device_ptr(dst)) return dst;
            buf.exact(count, s);
            return buf.p;
        };
        const size_t nn = static_cast<size_t>(n);
        a.free_vms = stage_in(free_vms, dfv, nn * static_cast<size_t>(K));
        a.task_index = stage_in(task_index, dti, nn);
        a.terminal = stage_in(terminal, dte, nn);
        a.value_out = stage_out(value_out, dval, nn);
        a.action_out = stage_out(action_out, dact, nn);
        a.idx_out = stage_out(idx_out, didx, nn);
        a.n = n;
        vcs::dispatch_words(vcs::max_words(sp), [&](auto wm) {
            constexpr int WM = decltype(wm)::value;
            vcs::k_policy_query<WM><<<vcs::blocks_for(static_cast<uint64_t>(n), 256), 256, 0, s>>>(a);
            VCS_LAUNCHED();
        });
        bool host_out = false;
        auto copy_out = [&](auto* dst, auto* staged, size_t count) {
            if (dst && staged != dst) {
                VCS_CUDA(cudaMemcpyAsync(dst, staged, count * sizeof(*dst), cudaMemcpyDeviceToHost, s));
                host_out = true;
            }
        };
        copy_out(value_out, a.value_out, nn);
        copy_out(action_out, a.action_out, nn);
        copy_out(idx_out, a.idx_out, nn);
        // staged buffers are freed in stream order; host outputs are complete on return
        if (host_out || dfv.p || dti.p || dte.p) VCS_CUDA(cudaStreamSynchronize(s));
        return VCS_OK;
    });
}

int vcs_rollout(vcs_space* sp, const vcs_instance* inst, int32_t* target_per_task, void* stream) {
    std::lock_guard<std::recursive_mutex> space_lock(sp->mu);
    return guarded([&] {
        if (!sp->has_plan) raise(VCS_EINVAL, "space was not built from an instance");
        if (!sp->result_actions)
            raise(VCS_EINVAL, "no solve results on this space (vcs_solve / vcs_solve_collect first)");
        if (!inst || !target_per_task) raise(VCS_EINVAL, "null argument");
        const int K = sp->plan.n_clouds, H = sp->H;
        if (inst->n_clouds != K || inst->n_tasks != H)
            raise(VCS_EINVAL, "instance does not match the space");
        if (H == 0) return VCS_OK;
        vcs::bind_device(sp->device);
        const vcs::StreamUse s(sp, stream);
        // one staging block: initial free counts, demands, scratch free counts, targets, status,
        // then (implicit form) the layer and rank-table offsets
        const size_t nk = static_cast<size_t>(std::max(K, 1)), nh = static_cast<size_t>(H);
        const size_t n32 = (2 * nk + 2 * nh + 1 + 1) & ~size_t(1); // (u64 offsets stay aligned)
        const bool rank_walk = sp->implicit && !sp->rank_off.empty() && !sp->csr_ready;
        std::vector<int32_t> host(n32 + (rank_walk ? 2 * (nh + 2) * 2 : 0), 0);
        std::memcpy(host.data(), inst->cloud_vm_free, sizeof(int32_t) * static_cast<size_t>(K));
        std::memcpy(host.data() + nk, inst->task_demand, sizeof(int32_t) * nh);
        if (rank_walk) {
            std::memcpy(host.data() + n32, sp->layer_off.data(), sizeof(uint64_t) * (nh + 2));
            std::memcpy(host.data() + n32 + 2 * (nh + 2), sp->rank_off.data(), sizeof(uint64_t) * (nh + 1));
        }
        vcs::DevBuf<int32_t> buf;
        buf.exact(host.size(), s);
        VCS_CUDA(cudaMemcpyAsync(buf.p, host.data(), sizeof(int32_t) * host.size(),
                                 cudaMemcpyHostToDevice, s));
        int32_t* fv = buf.p + nk + nh;
        int32_t* tg = fv + nk;
        int32_t* st = tg + nh;
        VCS_CUDA(cudaMemcpyAsync(fv, buf.p, sizeof(int32_t) * nk, cudaMemcpyDeviceToDevice, s));
        if (rank_walk) {
            const uint64_t* lo = reinterpret_cast<const uint64_t*>(buf.p + n32);
            vcs::k_rollout_rank<<<1, 32, 0, s>>>(sp->params_dev.p, sp->rank_tables.p,
                                                 lo + (nh + 2), lo, sp->result_actions, buf.p + nk,
                                                 fv, H, tg, st);
            VCS_LAUNCHED();
        } else if (sp->csr_ready) {
            vcs::k_rollout_csr<<<1, 32, 0, s>>>(sp->row_ptr.p, sp->succ.p, sp->action.p,
                                                sp->result_actions, H, tg, st);
            VCS_LAUNCHED();
        } else {
            vcs::ensure_locate_index(sp);
            vcs::QueryArgs a{};
            ensure_query_meta(sp, a);
            a.free_vms = buf.p;
            vcs::dispatch_words(vcs::max_words(sp), [&](auto wm) {
                constexpr int WM = decltype(wm)::value;
                vcs::k_rollout<WM><<<1, 32, 0, s>>>(a, buf.p + nk, fv, tg, st);
                VCS_LAUNCHED();
            });
        }
        VCS_CUDA(cudaMemcpyAsync(host.data() + 2 * nk + nh, tg, sizeof(int32_t) * (nh + 1),
                                 cudaMemcpyDeviceToHost, s));
        VCS_CUDA(cudaStreamSynchronize(s));
        if (host[2 * nk + 2 * nh] != 0)
            raise(VCS_ERANGE, "state not reachable in enumerated space");
        std::memcpy(target_per_task, host.data() + 2 * nk + nh, sizeof(int32_t) * nh);
        return VCS_OK;
    });
}

void vcs_space_free(vcs_space* sp) { delete sp; }

} // extern "C"
