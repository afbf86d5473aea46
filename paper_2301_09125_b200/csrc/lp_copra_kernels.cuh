// lp_copra_kernels.cuh -- COPRA (bounded label sets with belonging
// coefficients) on the INDEX plan.
//
// Reference: copra.py.  _copra_seq (:124-176) visits v = 0..n-1 in place;
// per vertex it accumulates acc[lab] += bels[u,j] * w over the non-self
// neighbours' label sets in scan order (:135-146), then _select_labels
// (:53-108) keeps the first <= k labels in first-touch order whose share
// reaches 1/k (tally*k >= total), renormalises them, sorts them by label,
// and _best_of_row (:111-121) caches the best label.
//
// Exactness.  Belongings are float64 as in the reference and every
// floating-point operation is the reference's, in the reference's order:
// products are rounded (__dmul_rn, no FMA contraction), each label's sum is
// accumulated in scan order (a warp processes 32 contributions at a time;
// the lowest lane of each equal-label group adds the group's values one by
// one in lane order), `total` and `kept` are summed serially in first-touch
// order (the touched list is built in scan order: new labels are appended
// per 32-contribution chunk in lane order).  So label sets, belongings and
// best labels are bit-identical to the oracle's restatement (and, for the
// in-place schedule with unit or float32-exact weights, to the reference) --
// except the fallback draw among tied maxima, which uses the counter hash
// instead of the sequential xorshift stream.
//
// Schedule: as RAK's (lp_engine.cu): B batches over the index order; a
// vertex reads the working (X) state of earlier-batch neighbours and the
// sweep-start (L0) state of the others; the sweep is solved as the fixed
// point of that triangular system with the mark queue.
#pragma once
#include "lp_rak_kernels.cuh"

namespace lp {

constexpr int kCopraMaxLabels = 32;  // label-set bound on the GPU (one lane per kept label)
constexpr int kCopraWarps = 8;       // warps per block, warp kernel
constexpr int kCopraBits = 9;        // per-warp smem table: 512 slots
constexpr int kCopraLimit = 384;     // distinct labels a per-warp table takes before spilling

struct CopraArgs {
    const uint32_t* __restrict__ soff;
    const uint32_t* __restrict__ snbr;  // neighbour id << 2 | kEarlier | kLater
    const uint32_t* __restrict__ sw;    // weights (fixed-point or float bits), null = unit
    int wmode;
    int shift;                          // fixed-point scale
    const int32_t* __restrict__ svid;
    const int32_t* __restrict__ slot_of;
    int K;                              // max_labels
    // sweep-start state (read-only in a sweep) and the working state
    const int32_t* __restrict__ labs0;  // [n x K]
    const double* __restrict__ bels0;   // [n x K]
    const int32_t* __restrict__ size0;  // [n]
    int32_t* labsX;
    double* belsX;
    int32_t* sizeX;
    int32_t* bestX;
    int32_t* ndist;                     // per-slot distinct count of the last evaluation
    // frontier
    int32_t* mark;
    int32_t* mq_out;
    int32_t* mq_len;
    // work: dense slot range or a vertex queue; spill list for big tables
    const int32_t* __restrict__ queue;  // null: dense over slots [0, S)
    const int32_t* __restrict__ queue_len;
    int32_t S;
    int32_t* cursor;                    // work cursor (reset per launch)
    int32_t* big;                       // slots whose tables exceed the warp table
    int32_t* big_len;
    int32_t* big_cursor;
    // big-table scratch (per block of the big kernel)
    int32_t* gkeys;
    double* gvals;
    int32_t* gtl;
    uint32_t gbits;
    unsigned long long* counters;
    uint32_t seed;
    uint32_t sweep;
};

__device__ __forceinline__ double copra_weight(const CopraArgs& a, uint32_t e) {
    if (!a.sw) return 1.0;
    const uint32_t raw = __ldg(a.sw + e);
    if (a.wmode == kFixed) return ldexp((double)raw, -a.shift);  // exact: the original float32 value
    return (double)__uint_as_float(raw);
}

__device__ __forceinline__ double shfl_f64(double x, int src) {
    const long long b = __double_as_longlong(x);
    const int lo = __shfl_sync(0xffffffffu, (int)(b & 0xffffffff), src);
    const int hi = __shfl_sync(0xffffffffu, (int)(b >> 32), src);
    return __longlong_as_double(((long long)hi << 32) | (unsigned int)lo);
}

// Per-warp evaluation scratch (shared memory for the warp kernel).
struct CopraWarpSmem {
    double stage[32];
    int32_t outl[kCopraMaxLabels];
    double outb[kCopraMaxLabels];
};

// Evaluate one vertex (slot s) with the whole warp into a table of 2^bits
// slots (keys kEmpty, vals 0 on entry; restored on exit).  Returns false if
// the distinct labels exceeded `limit` (nothing written).
__device__ bool copra_eval(const CopraArgs& a, int32_t s, int32_t* keys, double* vals, int32_t* tl, uint32_t bits,
                           int limit, CopraWarpSmem& sm) {
    const int lane = threadIdx.x & 31;
    const uint32_t mask = (1u << bits) - 1u;
    const int32_t v = __ldg(a.svid + s);
    const uint32_t beg = __ldg(a.soff + s);
    const int d = (int)(__ldg(a.soff + s + 1) - beg);
    const int K = a.K;
    int cnt = 0;
    bool overflow = false;
    // ---- tally (copra.py:135-146) ----
    for (int k0 = 0; k0 < d && !overflow; k0 += 32) {
        const int k = k0 + lane;
        uint32_t nb = 0;
        int su = 0;
        double w = 0.0;
        if (k < d) {
            nb = __ldg(a.snbr + beg + k);
            const int32_t u = (int32_t)(nb >> 2);
            su = (nb & kEarlier) ? *((volatile int32_t*)a.sizeX + u) : __ldg(a.size0 + u);
            su = min(max(su, 0), K);
            w = copra_weight(a, beg + k);
        }
        int incl = su;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        const int excl = incl - su;
        for (int c0 = 0; c0 < tot; c0 += 32) {
            const int c = c0 + lane;
            int r = 0;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1) {
                const int ex = __shfl_sync(0xffffffffu, excl, r + step);
                if (r + step < 32 && ex <= c) r += step;
            }
            const uint32_t nbr_r = __shfl_sync(0xffffffffu, nb, r);
            const int j = c - __shfl_sync(0xffffffffu, excl, r);
            const double wr = shfl_f64(w, r);
            int32_t lab = kEmpty;
            double val = 0.0;
            if (c < tot) {
                const int32_t u = (int32_t)(nbr_r >> 2);
                const size_t at = (size_t)u * K + j;
                double bel;
                if (nbr_r & kEarlier) {
                    lab = *((volatile int32_t*)a.labsX + at);
                    bel = *((volatile double*)a.belsX + at);
                } else {
                    lab = __ldg(a.labs0 + at);
                    bel = __ldg(a.bels0 + at);
                }
                val = __dmul_rn(bel, wr);  // bels[u, j] * w, rounded (copra.py:146)
            }
            sm.stage[lane] = val;
            const uint32_t grp = __match_any_sync(0xffffffffu, lab);
            const bool leader = lab != kEmpty && (__ffs(grp) - 1) == lane;
            int slot = -1;
            bool isnew = false;
            if (leader) {
                uint32_t h = slot_hash(lab, bits);
                while (true) {
                    const int32_t key = keys[h];
                    if (key == lab) {
                        slot = (int)h;
                        break;
                    }
                    if (key == kEmpty) {
                        const int32_t prev = atomicCAS(keys + h, kEmpty, lab);
                        if (prev == kEmpty) {
                            slot = (int)h;
                            isnew = true;
                            break;
                        }
                        if (prev == lab) {
                            slot = (int)h;
                            break;
                        }
                    }
                    h = (h + 1) & mask;
                }
            }
            const uint32_t nbal = __ballot_sync(0xffffffffu, isnew);
            if (isnew) tl[cnt + __popc(nbal & lanemask_lt())] = slot;
            cnt += __popc(nbal);
            __syncwarp();
            if (leader) {
                double acc = vals[slot];
                for (uint32_t m = grp; m; m &= m - 1) acc = __dadd_rn(acc, sm.stage[__ffs(m) - 1]);
                vals[slot] = acc;
            }
            __syncwarp();
            if (cnt > limit) {
                overflow = true;
                break;
            }
        }
    }
    if (overflow) {
        for (int i = lane; i < cnt; i += 32) {
            const int sl = tl[i];
            keys[sl] = kEmpty;
            vals[sl] = 0.0;
        }
        __syncwarp();
        return false;
    }
    // ---- _select_labels (copra.py:53-108) ----
    double total = 0.0;  // serial, touched order (:59-61)
    if (lane == 0) {
#pragma unroll 4
        for (int i = 0; i < cnt; ++i) total = __dadd_rn(total, vals[tl[i]]);
    }
    total = shfl_f64(total, 0);
    int kk = 0;  // kept so far (:64-71): first <= K labels with tally*K >= total, touched order
    for (int i0 = 0; i0 < cnt && kk < K; i0 += 32) {
        const int i = i0 + lane;
        bool q = false;
        int32_t lab = 0;
        double w = 0.0;
        if (i < cnt) {
            const int sl = tl[i];
            w = vals[sl];
            lab = keys[sl];
            q = __dmul_rn(w, (double)K) >= total;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, q);
        if (q) {
            const int rank = kk + __popc(bal & lanemask_lt());
            if (rank < K) {
                sm.outl[rank] = lab;
                sm.outb[rank] = w;
            }
        }
        kk = min(K, kk + __popc(bal));
    }
    __syncwarp();
    int32_t mylab = 0;
    double myb = 0.0;
    if (kk > 0) {
        double kept = 0.0;
        if (lane == 0)
            for (int i = 0; i < kk; ++i) kept = __dadd_rn(kept, sm.outb[i]);
        kept = shfl_f64(kept, 0);
        const double inv = __ddiv_rn(1.0, kept);  // (:94-96)
        if (lane < kk) {
            mylab = sm.outl[lane];
            myb = __dmul_rn(sm.outb[lane], inv);
        }
    } else {
        // nothing qualifies: one maximum-weight label, belonging 1 (:72-93); among
        // tied maxima the largest counter hash wins (first in touched order on equal hashes)
        double bw = -1.0;
        for (int i = lane; i < cnt; i += 32) bw = fmax(bw, vals[tl[i]]);
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) bw = fmax(bw, __shfl_xor_sync(0xffffffffu, bw, m));
        uint32_t bh = 0, bpos = 0xffffffffu;
        int32_t blab = kEmpty;
        for (int i = lane; i < cnt; i += 32) {
            const int sl = tl[i];
            if (vals[sl] != bw) continue;
            const uint32_t h = tie_hash(a.seed, a.sweep, (uint32_t)v, (uint32_t)keys[sl]);
            if (blab == kEmpty || h > bh || (h == bh && (uint32_t)i < bpos)) {
                bh = h;
                bpos = (uint32_t)i;
                blab = keys[sl];
            }
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) {
            const uint32_t oh = __shfl_xor_sync(0xffffffffu, bh, m);
            const uint32_t op = __shfl_xor_sync(0xffffffffu, bpos, m);
            const int32_t ol = __shfl_xor_sync(0xffffffffu, blab, m);
            if (ol != kEmpty && (blab == kEmpty || oh > bh || (oh == bh && op < bpos))) {
                bh = oh;
                bpos = op;
                blab = ol;
            }
        }
        kk = 1;
        if (lane == 0) {
            mylab = blab;
            myb = 1.0;
        }
    }
    // restore the table
    for (int i = lane; i < cnt; i += 32) {
        const int sl = tl[i];
        keys[sl] = kEmpty;
        vals[sl] = 0.0;
    }
    // sort the kept labels by id (:97-107): rank = number of smaller labels
    int rank = 0;
    for (int j = 0; j < kk; ++j) {
        const int32_t o = __shfl_sync(0xffffffffu, mylab, j);
        rank += (lane < kk) && o < mylab;
    }
    // _best_of_row (:111-121): maximum belonging, smallest id among ties
    double bb = lane < kk ? myb : -1.0;
    int32_t bl = lane < kk ? mylab : 0x7fffffff;
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, bb, m);
        const int32_t ol = __shfl_xor_sync(0xffffffffu, bl, m);
        if (ob > bb || (ob == bb && ol < bl)) {
            bb = ob;
            bl = ol;
        }
    }
    // ---- commit: compare with the working state; write and mark on change ----
    const size_t row = (size_t)v * K;
    bool diff = *((volatile int32_t*)a.sizeX + v) != kk;
    if (lane < kk) {
        diff |= *((volatile int32_t*)a.labsX + row + rank) != mylab;
        diff |= __double_as_longlong(*((volatile double*)a.belsX + row + rank)) != __double_as_longlong(myb);
    }
    diff = __any_sync(0xffffffffu, diff);
    if (diff) {
        if (lane < kk) {
            a.labsX[row + rank] = mylab;
            a.belsX[row + rank] = myb;
        }
        if (lane == 0) {
            a.sizeX[v] = kk;
            a.bestX[v] = bl;
        }
        __threadfence();
        if (a.mark) mark_row(a, beg, d, lane, 32);
    }
    if (lane == 0) a.ndist[s] = cnt;
    return true;
}

// Warp per vertex over the dense slot range or the queue; tables in smem.
__global__ void __launch_bounds__(kCopraWarps * 32, 3) k_copra_warp(CopraArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int slots = 1 << kCopraBits;
    double* vals = (double*)smem_raw + warp * slots;
    int32_t* keys = (int32_t*)((double*)smem_raw + kCopraWarps * slots) + warp * slots;
    int32_t* tl = (int32_t*)((double*)smem_raw + kCopraWarps * slots) + kCopraWarps * slots + warp * slots;
    CopraWarpSmem* sms = (CopraWarpSmem*)((int32_t*)((double*)smem_raw + kCopraWarps * slots) + 2 * kCopraWarps * slots);
    CopraWarpSmem& sm = sms[warp];
    for (int i = lane; i < slots; i += 32) {
        keys[i] = kEmpty;
        vals[i] = 0.0;
    }
    __syncwarp();
    const int cnt = a.queue ? *a.queue_len : a.S;
    while (true) {
        int idx = 0;
        if (lane == 0) idx = atomicAdd(a.cursor, 1);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx >= cnt) break;
        const int32_t s = a.queue ? __ldg(a.slot_of + __ldg(a.queue + idx)) : idx;
        if (s < 0) continue;
        const int est = nd_count(__ldg(a.ndist + s));
        bool done = false;
        if (est + (est >> 2) <= kCopraLimit) done = copra_eval(a, s, keys, vals, tl, kCopraBits, kCopraLimit, sm);
        if (!done && lane == 0) a.big[atomicAdd(a.big_len, 1)] = s;
    }
}

// Block (one warp) per big vertex; tables in per-block global scratch.
__global__ void __launch_bounds__(32) k_copra_big(CopraArgs a) {
    __shared__ CopraWarpSmem sm;
    const int lane = threadIdx.x & 31;
    const size_t slots = (size_t)1 << a.gbits;
    int32_t* keys = a.gkeys + blockIdx.x * slots;
    double* vals = a.gvals + blockIdx.x * slots;
    int32_t* tl = a.gtl + blockIdx.x * slots;
    const int cnt = *a.big_len;
    while (true) {
        int idx = 0;
        if (lane == 0) idx = atomicAdd(a.big_cursor, 1);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx >= cnt) break;
        copra_eval(a, a.big[idx], keys, vals, tl, a.gbits, (int)(slots >> 1) + (int)(slots >> 2), sm);
    }
}

__global__ void k_copra_gtab_init(int32_t* keys, double* vals, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = kEmpty;
        vals[i] = 0.0;
    }
}

// copra.py:254-258: labs[:, 0] = v, bels[:, 0] = 1, sizes = 1, best = v
__global__ void k_copra_init(int32_t* __restrict__ labs, double* __restrict__ bels, int32_t* __restrict__ size,
                             int32_t* __restrict__ best, int64_t n, int K) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        for (int j = 0; j < K; ++j) {
            labs[v * K + j] = j == 0 ? (int32_t)v : 0;
            bels[v * K + j] = j == 0 ? 1.0 : 0.0;
        }
        size[v] = 1;
        best[v] = (int32_t)v;
    }
}

// frontier: clear the marks of the queued vertices before the round evaluates any
__global__ void k_clear_marks(const int32_t* __restrict__ q, const int32_t* __restrict__ qlen, int32_t* mark) {
    const int cnt = *qlen;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) mark[q[i]] = 0;
}

// copra.py:171-173: vertices whose best label changed this sweep
__global__ void k_count_changed(const int32_t* __restrict__ a, const int32_t* __restrict__ b, int64_t n,
                                unsigned long long* out) {
    unsigned long long c = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        c += a[v] != b[v];
    for (int m = 16; m >= 1; m >>= 1) c += __shfl_xor_sync(0xffffffffu, c, m);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void k_copra_download(const int32_t* __restrict__ labs, const double* __restrict__ bels,
                                 const int32_t* __restrict__ size, const int32_t* __restrict__ best,
                                 int64_t* __restrict__ labs64, double* __restrict__ bels64,
                                 int64_t* __restrict__ size64, int64_t* __restrict__ best64, int64_t n, int K,
                                 int Kout) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int sz = size[v];
        if (labs64)
            for (int j = 0; j < Kout; ++j) {
                labs64[v * Kout + j] = j < sz ? labs[v * K + j] : 0;
                bels64[v * Kout + j] = j < sz ? bels[v * K + j] : 0.0;
            }
        if (size64) size64[v] = sz;
        best64[v] = best[v];
    }
}

}  // namespace lp
