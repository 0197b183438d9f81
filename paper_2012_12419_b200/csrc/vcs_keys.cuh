// vcs_keys.cuh — device helpers on packed reduced keys shared by the builder and the solver:
// field access, hashing, the retirement reward and the static edge slots of a dense state.
#pragma once

#include "vcs_internal.h"

#include <cstdint>

namespace vcs {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

template <int WM>
__device__ __forceinline__ uint64_t hash_key(const uint64_t (&k)[WM], int words, uint64_t salt) {
    uint64_t h = mix64(salt * 0x9e3779b97f4a7c15ull + 0x632be59bd9b4e019ull);
#pragma unroll
    for (int i = 0; i < WM; ++i)
        if (i < words) h = mix64(h ^ k[i]);
    return h;
}

template <int WM>
__device__ __forceinline__ void load_key(const uint64_t* __restrict__ p, int words,
                                         uint64_t (&k)[WM]) {
#pragma unroll
    for (int i = 0; i < WM; ++i) k[i] = i < words ? p[i] : 0ull;
}

template <int WM>
__device__ __forceinline__ bool key_equal(const uint64_t* __restrict__ p, int words,
                                          const uint64_t (&k)[WM]) {
    bool eq = true;
#pragma unroll
    for (int i = 0; i < WM; ++i)
        if (i < words) eq &= (p[i] == k[i]);
    return eq;
}

template <int WM>
__device__ __forceinline__ int get_field(const uint64_t (&k)[WM], int off, int width) {
    const int w = off >> 6;
    uint64_t word = k[0];
#pragma unroll
    for (int i = 1; i < WM; ++i)
        if (i == w) word = k[i];
    return static_cast<int>((word >> (off & 63)) & ((1ull << width) - 1ull));
}

template <int WM>
__device__ __forceinline__ void put_field(uint64_t (&k)[WM], int off, uint64_t v) {
    const int w = off >> 6;
#pragma unroll
    for (int i = 0; i < WM; ++i)
        if (i == w) k[i] |= v << (off & 63);
}

// Reward of one edge when clouds retire at this transition (mdp.cpp:179-185 / :196-197):
// beta*n - gamma*retired, retired summed in key-position order.  p = -1: the paid cloud.
template <int WM>
__device__ __forceinline__ double retiring_reward(const uint64_t (&k)[WM], int p,
                                                  const LayerParam& L) {
    double retired = 0.0;
    for (int q = 0; q < L.n_active; ++q) {
        if (L.keep_idx[q] >= 0) continue;
        int v = get_field<WM>(k, L.bit_off[q], L.width[q]);
        if (q == p) v -= L.demand;
        retired = __dadd_rn(retired, static_cast<double>(v));
    }
    const double base = p < 0 ? L.r_paid : L.r_cloud;
    return __dsub_rn(base, __dmul_rn(L.gamma, retired));
}

constexpr int kDenseSlots = 8; // edge slots of a state: clouds 0..6 by key position, 7 = paid

// A state's edges as 8 static slots: slot p < 7 is the edge choosing the cloud at key position p
// (valid if eligible with enough free VMs), slot 7 the paid edge (always valid).  The state is
// described by two words — the paid successor's mixed-radix index and the valid-cloud mask —
// from which every slot's row offset (the reference's order: clouds ascending, paid last) and
// successor index follow with a few integer operations (slot indices are compile-time).
struct Slots {
    uint32_t base; // successor index of the paid edge (nothing subtracted)
    uint32_t mask; // bit p: the cloud at key position p is a valid action
    __device__ __forceinline__ Slots(uint64_t desc)
        : base(static_cast<uint32_t>(desc)), mask(static_cast<uint32_t>(desc >> 32)) {}
    template <int WM>
    __device__ __forceinline__ Slots(const uint64_t (&k)[WM], const LayerParam& L) : base(0), mask(0) {
#pragma unroll
        for (int p = 0; p < kDenseSlots - 1; ++p) {
            if (p >= L.n_active) continue;
            const uint32_t f = static_cast<uint32_t>(get_field<WM>(k, L.bit_off[p], L.width[p]));
            if (L.keep_idx[p] >= 0) base += f * L.wnext[p];
            if (L.attr[p] && f >= static_cast<uint32_t>(L.demand)) mask |= 1u << p;
        }
    }
    __device__ __forceinline__ uint64_t pack() const {
        return static_cast<uint64_t>(base) | (static_cast<uint64_t>(mask) << 32);
    }
    __device__ __forceinline__ bool valid(int e) const {
        return e == kDenseSlots - 1 || ((mask >> e) & 1u);
    }
    __device__ __forceinline__ uint32_t off(int e) const {
        return static_cast<uint32_t>(__popc(mask & ((1u << e) - 1u)));
    }
    __device__ __forceinline__ uint32_t deg() const { return static_cast<uint32_t>(__popc(mask)) + 1u; }
    __device__ __forceinline__ uint32_t idx(int e, const LayerParam& L) const {
        return (e < kDenseSlots - 1 && e < L.n_active && L.keep_idx[e] >= 0)
                   ? base - static_cast<uint32_t>(L.demand) * L.wnext[e]
                   : base;
    }
};

// The slot constants of one layer held in registers (a thread decodes many states per layer):
// per cloud slot p the key word, shift, field mask (0 = slot unused), the successor weight
// W_p (0 when the cloud retires: its successor index does not move), and the eligibility mask.
template <int WM>
struct SlotDecoder {
    uint32_t sw[kDenseSlots - 1]; // bits 0-5 shift, 8-15 width, 16 eligible, 17 used, 24+ key word
    uint32_t wn[kDenseSlots - 1];
    uint32_t demand;
    __device__ __forceinline__ explicit SlotDecoder(const LayerParam& L) {
        demand = static_cast<uint32_t>(L.demand);
#pragma unroll
        for (int p = 0; p < kDenseSlots - 1; ++p) {
            const bool on = p < L.n_active;
            const uint32_t off = on ? L.bit_off[p] : 0u;
            sw[p] = (off & 63u) | ((on ? static_cast<uint32_t>(L.width[p]) : 0u) << 8) |
                    ((on && L.attr[p]) ? 1u << 16 : 0u) | (on ? 1u << 17 : 0u) | ((off >> 6) << 24);
            wn[p] = (on && L.keep_idx[p] >= 0) ? L.wnext[p] : 0u;
        }
    }
    __device__ __forceinline__ uint32_t field(const uint64_t (&k)[WM], int p) const {
        uint64_t w = k[0];
#pragma unroll
        for (int i = 1; i < WM; ++i)
            if (static_cast<uint32_t>(i) == (sw[p] >> 24)) w = k[i];
        const uint32_t width = (sw[p] >> 8) & 0xffu;
        return static_cast<uint32_t>(w >> (sw[p] & 63u)) & ((1u << width) - 1u);
    }
    // the state's Slots (same result as Slots(k, L))
    __device__ __forceinline__ Slots decode(const uint64_t (&k)[WM]) const {
        uint32_t base = 0, mask = 0;
#pragma unroll
        for (int p = 0; p < kDenseSlots - 1; ++p) {
            const uint32_t f = field(k, p);
            base += f * wn[p];
            if (((sw[p] >> 16) & 1u) && f >= demand) mask |= 1u << p;
        }
        return Slots(static_cast<uint64_t>(base) | (static_cast<uint64_t>(mask) << 32));
    }
    __device__ __forceinline__ uint32_t idx(const Slots& sl, int e) const {
        return e < kDenseSlots - 1 ? sl.base - demand * wn[e] : sl.base;
    }
};

} // namespace
} // namespace vcs
