// lp_common.cuh -- shared device definitions of the label-propagation engine.
//
// Vocabulary:
//   position  p   index of a vertex in the visit order (order[p] = vertex id);
//                 every per-vertex device array is indexed by position.
//   slot      s   index in the *storage* order: active vertices grouped by
//                 degree bin, ascending position inside a bin.  Rows of the
//                 storage CSR are laid out in slot order so each bin streams
//                 contiguous memory.
//   label         a vertex id (the reference's label values, rak.py:168).
//   L0 / x        labels at sweep start (read-only during a sweep) / the
//                 working labels being solved for this sweep.
//   batch         positions [b*bs, (b+1)*bs); a vertex reads x for
//                 neighbours in earlier batches and L0 for the rest.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lp {

constexpr int32_t kEmpty = -1;

enum WeightMode : int { kUnit = 0, kFixed = 1, kFloat = 2 };
enum TieRule : int { kScanFirst = 0, kRandom = 1, kMinLabel = 2 };

template <int WM> struct Acc;
template <> struct Acc<kUnit> { using T = uint32_t; };
template <> struct Acc<kFixed> { using T = unsigned long long; };
// kFloat: weights that are not float32-exact fixed point (stored as float32)
// are summed in float64 -- exact for any row whose weights span less than
// 2^(29 - log2(degree)) in magnitude, so the sums (and ties) do not depend
// on the atomics' order: deterministic, like the reference's float64 tally
// (rak.py:105)
template <> struct Acc<kFloat> { using T = double; };

__host__ __device__ __forceinline__ uint32_t fmix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x85EBCA6Bu;
    x ^= x >> 13;
    x *= 0xC2B2AE35u;
    x ^= x >> 16;
    return x;
}

// Counter RNG for non-strict ties; same definition as the oracle's
// or_tie_hash (oracle/lp_oracle.c) -- keyed by (seed, sweep, vertex, label).
__host__ __device__ __forceinline__ uint32_t tie_hash(uint32_t seed, uint32_t sweep, uint32_t vertex,
                                                      uint32_t label) {
    uint32_t h = fmix32(seed ^ (sweep * 0x9E3779B9u + 0x7F4A7C15u));
    h = fmix32(h ^ (vertex * 0x85EBCA6Bu + 0x68E31DA4u));
    h = fmix32(h ^ (label * 0xC2B2AE35u + 0xB5297A4Du));
    return h;
}

// Counter RNG for SLPA's speaker draw: listener `listener` hears its k-th
// speaking (non-self) neighbour in round t; same definition as the oracle's
// or_speak_hash (oracle/lp_oracle.c).
__host__ __device__ __forceinline__ uint32_t speak_hash(uint32_t seed, uint32_t t, uint32_t listener, uint32_t k) {
    return tie_hash(seed ^ 0x53504B52u, t, listener, k);
}

// Candidate label for the argmax.  Ordering: larger weight, then larger
// `sec`, then larger `ter`.  (sec, ter) encode the tie rule so that the
// maximum is unique per distinct label:
//   scan-first  sec = ~first_pos            (earliest first occurrence)
//   min-label   sec = ~label
//   random      sec = tie_hash(...), ter = ~first_pos
template <typename A> struct Cand {
    A w;
    uint32_t sec;
    uint32_t ter;
    int32_t lab;
};

template <typename A> __device__ __forceinline__ bool better(const Cand<A>& a, const Cand<A>& b) {
    if (a.w != b.w) return a.w > b.w;
    if (a.sec != b.sec) return a.sec > b.sec;
    return a.ter > b.ter;
}

template <typename A> __device__ __forceinline__ Cand<A> none_cand() {
    Cand<A> c;
    c.w = A(0);
    c.sec = 0;
    c.ter = 0;
    c.lab = -1;
    return c;
}

template <int TIE, typename A>
__device__ __forceinline__ Cand<A> make_cand(A w, int32_t lab, uint32_t first, uint32_t seed, uint32_t sweep,
                                             uint32_t vertex) {
    Cand<A> c;
    c.w = w;
    c.lab = lab;
    if (TIE == kScanFirst) {
        c.sec = ~first;
        c.ter = 0;
    } else if (TIE == kMinLabel) {
        c.sec = ~(uint32_t)lab;
        c.ter = 0;
    } else {
        c.sec = tie_hash(seed, sweep, vertex, (uint32_t)lab);
        c.ter = ~first;
    }
    return c;
}

__device__ __forceinline__ unsigned long long shfl_u64(unsigned long long v, int src) {
    uint32_t lo = (uint32_t)v, hi = (uint32_t)(v >> 32);
    lo = __shfl_xor_sync(0xffffffffu, lo, src);
    hi = __shfl_xor_sync(0xffffffffu, hi, src);
    return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ uint32_t shfl_idx_any(uint32_t v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ float shfl_idx_any(float v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ double shfl_idx_any(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ unsigned long long shfl_idx_any(unsigned long long v, int src) {
    return __shfl_sync(0xffffffffu, v, src);
}
__device__ __forceinline__ uint32_t shfl_xor_any(uint32_t v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ float shfl_xor_any(float v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ double shfl_xor_any(double v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ unsigned long long shfl_xor_any(unsigned long long v, int m) { return shfl_u64(v, m); }

template <typename A> __device__ __forceinline__ Cand<A> warp_best(Cand<A> c) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        Cand<A> o;
        o.w = shfl_xor_any(c.w, m);
        o.sec = __shfl_xor_sync(0xffffffffu, c.sec, m);
        o.ter = __shfl_xor_sync(0xffffffffu, c.ter, m);
        o.lab = __shfl_xor_sync(0xffffffffu, c.lab, m);
        if (better(o, c)) c = o;
    }
    return c;
}

// Hash-table slot of a label (multiplicative hashing into 2^bits slots).
__device__ __forceinline__ uint32_t slot_hash(int32_t lab, uint32_t bits) {
    return ((uint32_t)lab * 0x9E3779B1u) >> (32 - bits);
}
// Partition of a label for multi-pass hub evaluation.
// (A multiplicative hash independent of slot_hash's multiplier; nested:
// part_of(l, 4P) / 4 == part_of(l, P), which the 4-way re-split relies on.)
__device__ __forceinline__ uint32_t part_of(int32_t lab, uint32_t parts) {
    return __umulhi((uint32_t)lab * 0x2C1B3C6Du + 0x297A2D39u, parts);
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

}  // namespace lp
