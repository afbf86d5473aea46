// lp_slpa_kernels.cuh -- SLPA (speaker-listener) kernels around the RAK tally.
//
// Reference: slpa.py.  One speaking round t (slpa.py:96-110) is a RAK sweep
// whose phase-1 gather draws each speaker's spoken label from its memory
// (k_gather_pieces<kGatherSlpa>, lp_rak_kernels.cuh) instead of reading its
// current label; the tally, argmax and tie rules are the RAK kernels'
// (slpa.py:85 calls rak._pick_from_tally).  Memories live in an int32
// [n x T] array; the slot a round appends is solved in the working label
// array x and copied into the memory by k_slpa_commit when the round ends.
#pragma once
#include "lp_rak_kernels.cuh"

namespace lp {

// slpa.py:51-66 -- most frequent label of a memory, frequency ties to the
// smallest id.  O(filled^2) like the reference; memories are short.
__device__ __forceinline__ int32_t modal_label(const int32_t* __restrict__ row, int filled) {
    int32_t best = -1;
    int best_c = 0;
    for (int i = 0; i < filled; ++i) {
        const int32_t lab = row[i];
        int c = 0;
        for (int j = 0; j < filled; ++j) c += row[j] == lab;
        if (c > best_c || (c == best_c && lab < best)) {
            best = lab;
            best_c = c;
        }
    }
    return best;
}

// slpa.py:186-189: slot 0 = own id
__global__ void k_slpa_init(int32_t* __restrict__ slots, int32_t* __restrict__ guess, int64_t n, int T) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        slots[v * T] = (int32_t)v;
        guess[v] = (int32_t)v;
    }
}

// Listeners without speakers (idle slots of the INDEX plan) append their own
// modal label (slpa.py:82-84).  Nobody hears them (no arcs), so they can be
// solved outside the rounds.
__global__ void k_slpa_idle(const int32_t* __restrict__ svid, int64_t s_beg, int64_t s_end,
                            const int32_t* __restrict__ slots, int T, int t, int32_t* __restrict__ x) {
    for (int64_t s = s_beg + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < s_end;
         s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = svid[s];
        x[v] = modal_label(slots + (size_t)v * T, t);
    }
}

// End of round t: append x to the memories (slpa.py:104-105) and count the
// listeners that repeated their previous append (slpa.py:106-108).
__global__ void k_slpa_commit(const int32_t* __restrict__ x, const int32_t* __restrict__ prev,
                              int32_t* __restrict__ slots, int64_t n, int T, int t, int count_repeats,
                              unsigned long long* repeats) {
    unsigned long long r = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t lab = x[v];
        slots[(size_t)v * T + t] = lab;
        r += count_repeats && lab == prev[v];
    }
    for (int m = 16; m >= 1; m >>= 1) r += __shfl_xor_sync(0xffffffffu, r, m);
    if ((threadIdx.x & 31) == 0 && r) atomicAdd(repeats, r);
}

// slpa.py:147-150: the disjoint projection
__global__ void k_slpa_project(const int32_t* __restrict__ slots, int64_t n, int T, int filled,
                               int64_t* __restrict__ out) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        out[v] = modal_label(slots + (size_t)v * T, filled);
}

__global__ void k_slots_to64(const int32_t* __restrict__ slots, int64_t* __restrict__ out, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = slots[i];
}

}  // namespace lp
