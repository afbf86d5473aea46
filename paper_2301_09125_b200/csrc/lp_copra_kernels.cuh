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

#ifdef LP_DEBUG_BOUNDS
#define LP_CHECK(cond, what)                                                                         \
    do {                                                                                            \
        if (!(cond)) {                                                                              \
            printf("LP_CHECK failed: %s (block %d thread %d)\n", what, blockIdx.x, threadIdx.x);    \
            __trap();                                                                               \
        }                                                                                           \
    } while (0)
#else
#define LP_CHECK(cond, what) \
    do {                     \
    } while (0)
#endif

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
    unsigned long long* mark;
    int32_t* mq_out;
    int32_t* mq_len;
    uint32_t* mbits;                    // marked-vertex bitmap: marks are fire-and-forget bit sets and
                                        // k_bits_to_queue builds the next queue after the round (an append
                                        // per 32 arcs of every changed row all landed on mq_len); null:
                                        // queue on the mark's 0 -> nonzero transition (mark_row)
    // work: dense slot range or a vertex queue; spill list for big tables
    const int32_t* __restrict__ queue;  // null: dense over slots [0, S)
    const int32_t* __restrict__ queue_len;
    int32_t pre_routed;                 // the rows certain to need the team (copra_team_row) were listed
                                        // by k_copra_route and run beside the warp tiers: those skip them
    int32_t* route_mark;                // per slot: route_id of the round that listed it (the decision is
    int32_t route_id;                   // taken once: the estimate it reads moves while the round runs)
    int32_t long_row;                   // rows with more contributions (degree x K) skip the warp tiers:
                                        // one warp walking a hub's 100K contributions is the tail of
                                        // every round (0 = off)
    int32_t S;
    int32_t* cursor;                    // work cursor (reset per launch)
    int32_t* big;                       // slots whose tables exceed the warp table
    int32_t* big_len;
    int32_t* big_cursor;
    // team scratch (per block of the team kernel): entries, first-touch order, contribution map
    int32_t* gelab;
    double* geval;
    int32_t* gefirst;
    int32_t* grlab;
    double* grval;
    int32_t* gfmap;     // [gcap_contrib] per block, -1 between uses
    int32_t* gblab;     // [gcap_contrib] per block: bucketed contributions
    double* gbval;
    int32_t* gbc;
    int32_t* gslab;     // [gcap_contrib] per block: staged contributions (label, value)
    double* gsval;
    int32_t* gwc;       // [W x kCopraMaxParts] per block: partition counts / offsets
    int32_t* gqs;       // [kCopraMaxParts + 1] per block: bucket starts
    size_t gcap_entries;
    size_t gcap_contrib;
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

// Per-warp evaluation scratch.
struct CopraWarpSmem {
    double stage[32];
    int32_t outl[kCopraMaxLabels];
    double outb[kCopraMaxLabels];
};

// Walk the contributions (label, bels[u,j] * w) of arcs [k_lo, k_hi) of row
// s in scan order (copra.py:135-146), 32 at a time; fn(lab, val, c, valid)
// is called by the whole warp per chunk, c = contribution index from k_lo.
template <class Fn>
__device__ __forceinline__ void for_each_contribution(const CopraArgs& a, int32_t s, int k_lo, int k_hi, Fn fn) {
    const int lane = threadIdx.x & 31;
    const uint32_t beg = __ldg(a.soff + s);
    const int K = a.K;
    int cbase = 0;
    for (int k0 = k_lo; k0 < k_hi; k0 += 32) {
        const int k = k0 + lane;
        uint32_t nb = 0;
        int su = 0;
        double w = 0.0;
        if (k < k_hi) {
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
            fn(lab, val, cbase + c, c < tot);
        }
        cbase += tot;
    }
}

// Add one chunk of up to 32 contributions (lab kEmpty = none) to a warp's
// table of 2^bits slots, in lane order: each label's lowest lane inserts
// it (new labels join the touched list tl in lane order) and adds the
// group's values one by one.  cnt (warp-uniform) = distinct labels so far.
__device__ __forceinline__ void tally_chunk(int32_t lab, double val, int c, int32_t* keys, double* vals,
                                            int32_t* firsts, int32_t* tl, uint32_t bits, int& cnt, double* stage) {
    const int lane = threadIdx.x & 31;
    const uint32_t mask = (1u << bits) - 1u;
    stage[lane] = val;
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
    if (isnew) {
        tl[cnt + __popc(nbal & lanemask_lt())] = slot;
        if (firsts) firsts[slot] = c;
    }
    cnt += __popc(nbal);
    __syncwarp();
    if (leader) {
        double acc = vals[slot];
        for (uint32_t m = grp; m; m &= m - 1) acc = __dadd_rn(acc, stage[__ffs(m) - 1]);
        vals[slot] = acc;
    }
    __syncwarp();
}

__device__ __forceinline__ void table_restore(int32_t* keys, double* vals, const int32_t* tl, int cnt) {
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < cnt; i += 32) {
        const int sl = tl[i];
        keys[sl] = kEmpty;
        vals[sl] = 0.0;
    }
    __syncwarp();
}

// The end of an evaluation (one warp): lanes < kk hold the kept labels and
// their normalised belongings; sort by label (copra.py:97-107), best label
// (_best_of_row, :111-121), compare with the working state, write and mark
// the later-batch neighbours on change.
__device__ void copra_commit(const CopraArgs& a, int32_t s, int cnt, int kk, int32_t mylab, double myb) {
    const int lane = threadIdx.x & 31;
    const int32_t v = __ldg(a.svid + s);
    const uint32_t beg = __ldg(a.soff + s);
    const int d = (int)(__ldg(a.soff + s + 1) - beg);
    const int K = a.K;
    // sort the kept labels by id: rank = number of smaller labels
    int rank = 0;
    for (int j = 0; j < kk; ++j) {
        const int32_t o = __shfl_sync(0xffffffffu, mylab, j);
        rank += (lane < kk) && o < mylab;
    }
    // maximum belonging, smallest id among ties
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
        if (a.mark && a.mbits) {
            for (int k = lane; k < d; k += 32) {
                const uint32_t nb = __ldg(a.snbr + beg + k);
                if (nb & kLater) {
                    const int32_t u = (int32_t)(nb >> 2);
                    atomicOr(a.mbits + (u >> 5), 1u << (u & 31));
                }
            }
        } else if (a.mark) {
            mark_row(a, beg, d, lane, 32);
        }
    }
    if (lane == 0) a.ndist[s] = cnt;
}

// Phase 2 (one warp): _select_labels + _best_of_row over the distinct
// labels in first-touch order (get(i) -> label, tally), then compare with
// the working state; write and mark later-batch neighbours on change.
template <class Get>
__device__ void copra_finish(const CopraArgs& a, int32_t s, int cnt, Get get, CopraWarpSmem& sm) {
    const int lane = threadIdx.x & 31;
    const int32_t v = __ldg(a.svid + s);
    const uint32_t beg = __ldg(a.soff + s);
    const int d = (int)(__ldg(a.soff + s + 1) - beg);
    const int K = a.K;
    // total (copra.py:59-61) is the serial float64 sum in touched order, and it
    // is used only by the test tally * K >= total (:64-71).  A parallel sum of
    // the same positive values is within E = (cnt + 32) * 2^-52 * sum of it, so
    // the test is decided by the parallel sum unless tally * K falls inside
    // that band -- or exactly, when every tally is an integer (the parallel
    // sum is then exact too).  Only an undecided vertex pays the serial sum.
    double tpar = 0.0;
    bool allint = true;
    for (int i = lane; i < cnt; i += 32) {
        int32_t l;
        double w;
        get(i, l, w);
        tpar += w;
        allint &= w == floor(w);
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) tpar += __shfl_xor_sync(0xffffffffu, tpar, m);
    allint = __all_sync(0xffffffffu, allint) && tpar < 9007199254740992.0;
    const double band = allint ? 0.0 : tpar * (double)(cnt + 32) * 2.220446049250313e-16;
    double total = tpar;
    bool exact_total = allint;
    int kk = 0;  // (:64-71): first <= K labels with tally * K >= total, touched order
    for (int pass = 0; pass < 2; ++pass) {
        kk = 0;
        bool undecided = false;
        for (int i0 = 0; i0 < cnt && kk < K; i0 += 32) {
            const int i = i0 + lane;
            bool qual = false;
            int32_t lab = 0;
            double w = 0.0;
            if (i < cnt) {
                get(i, lab, w);
                const double p = __dmul_rn(w, (double)K);
                if (exact_total) {
                    qual = p >= total;
                } else if (p >= total + band) {
                    qual = true;
                } else if (!(p < total - band)) {
                    undecided = true;
                }
            }
            if (__any_sync(0xffffffffu, undecided)) break;
            const uint32_t bal = __ballot_sync(0xffffffffu, qual);
            if (qual) {
                const int rank = kk + __popc(bal & lanemask_lt());
                if (rank < K) {
                    sm.outl[rank] = lab;
                    sm.outb[rank] = w;
                }
            }
            kk = min(K, kk + __popc(bal));
        }
        if (!__any_sync(0xffffffffu, undecided)) break;
        // undecided: the reference's serial total, touched order (the warp loads
        // 32 tallies at a time and every lane runs the same serial sum)
        total = 0.0;
        for (int i0 = 0; i0 < cnt; i0 += 32) {
            double w = 0.0;
            if (i0 + lane < cnt) {
                int32_t l;
                get(i0 + lane, l, w);
            }
            const int m = min(32, cnt - i0);
            for (int j = 0; j < m; ++j) total = __dadd_rn(total, shfl_f64(w, j));
        }
        exact_total = true;
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
        for (int i = lane; i < cnt; i += 32) {
            int32_t l;
            double w;
            get(i, l, w);
            bw = fmax(bw, w);
        }
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) bw = fmax(bw, __shfl_xor_sync(0xffffffffu, bw, m));
        uint32_t bh = 0, bpos = 0xffffffffu;
        int32_t blab = kEmpty;
        for (int i = lane; i < cnt; i += 32) {
            int32_t l;
            double w;
            get(i, l, w);
            if (w != bw) continue;
            const uint32_t h = tie_hash(a.seed, a.sweep, (uint32_t)v, (uint32_t)l);
            if (blab == kEmpty || h > bh || (h == bh && (uint32_t)i < bpos)) {
                bh = h;
                bpos = (uint32_t)i;
                blab = l;
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
    copra_commit(a, s, cnt, kk, mylab, myb);
}

// A row that the warp tiers would only pass on: more contributions than one warp should walk, or
// an estimate beyond the larger warp table (2048 slots, 3/4 full).
__device__ __forceinline__ bool copra_team_row(const CopraArgs& a, int32_t s) {
    const int est = nd_count(__ldg(a.ndist + s));
    const int d = (int)(__ldg(a.soff + s + 1) - __ldg(a.soff + s));
    return (a.long_row > 0 && (long long)d * a.K > a.long_row) || est + (est >> 2) > (1 << 11) / 4 * 3;
}

// The round's team rows, listed up front so that the team kernel starts beside the warp tiers
// (its largest hub, alone in one block for ~2 ms, is the round's tail) instead of after them.
__global__ void k_copra_route(CopraArgs a, int32_t* __restrict__ out, int32_t* out_len) {
    const int items = a.queue ? *a.queue_len : a.S;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < items; idx += gridDim.x * blockDim.x) {
        const int32_t s = a.queue ? __ldg(a.slot_of + __ldg(a.queue + idx)) : idx;
        if (s >= 0 && copra_team_row(a, s)) {
            a.route_mark[s] = a.route_id;
            out[atomicAdd(out_len, 1)] = s;
        }
    }
}

// Warp per vertex, table of 2^BITS slots in smem.  Input: `in` (slots)
// when given, else the dense slot range / the vertex queue of the round.
// Rows whose distinct labels may exceed 3/4 of the table go to `out`.
template <int BITS, int NW>
__host__ __device__ constexpr size_t copra_warp_smem_bytes() {
    return (size_t)NW * (1 << BITS) * (sizeof(double) + 2 * sizeof(int32_t)) + NW * sizeof(CopraWarpSmem);
}

template <int BITS, int NW, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
    k_copra_warp(CopraArgs a, const int32_t* __restrict__ in, const int32_t* __restrict__ in_len, int32_t* cursor,
                 int32_t* out, int32_t* out_len) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int slots = 1 << BITS;
    constexpr int limit = slots / 4 * 3;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* vals = (double*)smem_raw + warp * slots;
    int32_t* keys = (int32_t*)((double*)smem_raw + NW * slots) + warp * slots;
    int32_t* tl = (int32_t*)((double*)smem_raw + NW * slots) + NW * slots + warp * slots;
    CopraWarpSmem* sms = (CopraWarpSmem*)((int32_t*)((double*)smem_raw + NW * slots) + 2 * NW * slots);
    CopraWarpSmem& sm = sms[warp];
    for (int i = lane; i < slots; i += 32) {
        keys[i] = kEmpty;
        vals[i] = 0.0;
    }
    __syncwarp();
    const int items = in ? *in_len : (a.queue ? *a.queue_len : a.S);
    while (true) {
        int idx = 0;
        if (lane == 0) idx = atomicAdd(cursor, 1);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx >= items) break;
        const int32_t s = in ? __ldg(in + idx) : (a.queue ? __ldg(a.slot_of + __ldg(a.queue + idx)) : idx);
        if (s < 0) continue;
        if (a.pre_routed && a.route_mark[s] == a.route_id) continue;  // (on the team's list already)
        const int est = nd_count(__ldg(a.ndist + s));
        int dist = -1;
        const int d = (int)(__ldg(a.soff + s + 1) - __ldg(a.soff + s));
        const bool long_row = a.long_row > 0 && (long long)d * a.K > a.long_row;
        if (!long_row && est + (est >> 2) <= limit) {
            int seen = 0;
            bool over = false;
            for_each_contribution(a, s, 0, d, [&](int32_t lab, double val, int c, bool) {
                if (over) return;
                tally_chunk(lab, val, c, keys, vals, nullptr, tl, BITS, seen, sm.stage);
                if (seen > limit) {
                    table_restore(keys, vals, tl, seen);
                    over = true;
                }
            });
            dist = over ? -1 : seen;
        }
        if (dist < 0) {
            if (lane == 0) out[atomicAdd(out_len, 1)] = s;
            continue;
        }
        copra_finish(a, s, dist, [&](int i, int32_t& l, double& w) {
            const int sl = tl[i];
            l = keys[sl];
            w = vals[sl];
        }, sm);
        table_restore(keys, vals, tl, dist);
    }
}

// Team path for big rows: a block of kCopraTeamWarps warps per vertex.
// Labels are split into P hash partitions.  (1) each warp counts, for its
// contiguous range of the row's arcs, the contributions of every partition;
// (2) a stable scatter puts every contribution into its partition's bucket in
// scan order (bucket q = warp ranges in order, each in scan order); (3) warp
// w tallies buckets w, w + W, ... with its smem table -- per-label order is
// the scan order because a label lives in one bucket; (4) the entries
// (label, tally, first contribution) are put back into first-touch order via
// a contribution-indexed map and one warp finishes the vertex.  A bucket
// with more distinct labels than a warp table holds restarts the vertex with
// twice the partitions.
constexpr int kCopraTeamWarps = 16;
constexpr int kCopraTeamBits = 8;      // per-warp table, 256 slots
constexpr int kCopraTeamLimit = 192;
constexpr int kCopraMaxParts = 4096;

__host__ __device__ constexpr size_t copra_team_smem_bytes() {
    return (size_t)kCopraTeamWarps * (1 << kCopraTeamBits) * (sizeof(double) + 3 * sizeof(int32_t)) +
           (size_t)kCopraTeamWarps * sizeof(CopraWarpSmem) + 256;
}

constexpr int kQualMax = 64;  // qualifiers the unordered finish handles

__global__ void __launch_bounds__(kCopraTeamWarps * 32, 2) k_copra_team(CopraArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double s_red[kCopraTeamWarps];
    __shared__ int s_ai[kCopraTeamWarps];
    __shared__ int s_nq, s_und;
    __shared__ int32_t s_qfirst[kQualMax], s_qlab[kQualMax];
    __shared__ double s_qw[kQualMax];
    constexpr int slots = 1 << kCopraTeamBits;
    constexpr int W = kCopraTeamWarps;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    double* vals = (double*)smem_raw + warp * slots;
    int32_t* ibase = (int32_t*)((double*)smem_raw + W * slots);
    int32_t* keys = ibase + warp * slots;
    int32_t* firsts = ibase + W * slots + warp * slots;
    int32_t* tl = ibase + 2 * W * slots + warp * slots;
    CopraWarpSmem* sms = (CopraWarpSmem*)(ibase + 3 * W * slots);
    CopraWarpSmem& sm = sms[warp];
    int32_t* ctl = (int32_t*)(sms + W);  // [0] item [1] entries [2] overflow [3] contributions [16..16+W) warp bases
    // per-block global scratch
    const size_t D = a.gcap_entries, Cc = a.gcap_contrib;
    int32_t* Elab = a.gelab + blockIdx.x * D;
    double* Eval = a.geval + blockIdx.x * D;
    int32_t* Efirst = a.gefirst + blockIdx.x * D;
    int32_t* Rlab = a.grlab + blockIdx.x * D;
    double* Rval = a.grval + blockIdx.x * D;
    int32_t* F = a.gfmap + blockIdx.x * Cc;
    int32_t* Blab = a.gblab + blockIdx.x * Cc;
    double* Bval = a.gbval + blockIdx.x * Cc;
    int32_t* Bc = a.gbc + blockIdx.x * Cc;
    int32_t* Slab = a.gslab + blockIdx.x * Cc;
    double* Sval = a.gsval + blockIdx.x * Cc;
    int32_t* Wc = a.gwc + blockIdx.x * (size_t)(W * kCopraMaxParts);  // [W][P] counts -> offsets
    int32_t* Qs = a.gqs + blockIdx.x * (size_t)(kCopraMaxParts + 1);  // bucket starts
    for (int i = lane; i < slots; i += 32) {
        keys[i] = kEmpty;
        vals[i] = 0.0;
    }
    const int nitems = *a.big_len;
    while (true) {
        __syncthreads();
        if (tid == 0) ctl[0] = atomicAdd(a.big_cursor, 1);
        __syncthreads();
        const int idx = ctl[0];
        if (idx >= nitems) break;
        const int32_t s = a.big[idx];
        const int d = (int)(__ldg(a.soff + s + 1) - __ldg(a.soff + s));
        const int k_lo = (int)((long long)d * warp / W), k_hi = (int)((long long)d * (warp + 1) / W);
        const int est = nd_count(__ldg(a.ndist + s));
        int P = W;
        while (P < kCopraMaxParts && P * kCopraTeamLimit < est + (est >> 2)) P *= 2;
        // (0) stage the warp's contributions once: earlier-batch label sets may
        // change under a running round, and every later pass must see the same
        // data (the region of arcs [k_lo, k_hi) holds at most (k_hi - k_lo) * K)
        const int sbase = k_lo * a.K;
        int mine = 0;
        for_each_contribution(a, s, k_lo, k_hi, [&](int32_t lab, double val, int c, bool valid) {
            if (valid) {
                LP_CHECK((size_t)(sbase + c) < Cc, "stage index");
                Slab[sbase + c] = lab;
                Sval[sbase + c] = val;
            }
            mine += __popc(__ballot_sync(0xffffffffu, valid));
        });
        __syncwarp();
        while (true) {  // retry with more partitions on a table overflow
            // (1) per-warp partition counts
            for (int q = lane; q < P; q += 32) Wc[warp * P + q] = 0;
            __syncwarp();
            for (int i0 = 0; i0 < mine; i0 += 32) {
                const bool valid = i0 + lane < mine;
                const uint32_t q = valid ? part_of(Slab[sbase + i0 + lane], (uint32_t)P) : 0xffffffffu;
                const uint32_t grp = __match_any_sync(0xffffffffu, q);
                if (valid && (__ffs(grp) - 1) == lane) Wc[warp * P + q] += __popc(grp);
                __syncwarp();
            }
            if (lane == 0) ctl[16 + warp] = mine;
            if (tid == 0) {
                ctl[1] = 0;
                ctl[2] = 0;
            }
            __syncthreads();
            // bucket starts (serial over P by warp 0: P <= 4096) and per-warp offsets
            if (warp == 0) {
                int run = 0;
                for (int q0 = 0; q0 < P; q0 += 32) {
                    const int q = q0 + lane;
                    int tot = 0;
                    if (q < P)
                        for (int w = 0; w < W; ++w) tot += Wc[w * P + q];
                    int incl = tot;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int t = __shfl_up_sync(0xffffffffu, incl, o);
                        if (lane >= o) incl += t;
                    }
                    if (q < P) {
                        int off = run + incl - tot;
                        Qs[q] = off;
                        for (int w = 0; w < W; ++w) {
                            const int cnum = Wc[w * P + q];
                            Wc[w * P + q] = off;
                            off += cnum;
                        }
                    }
                    run += __shfl_sync(0xffffffffu, incl, 31);
                }
                if (lane == 0) {
                    Qs[P] = run;
                    int cb = 0;
                    for (int w = 0; w < W; ++w) {
                        const int m = ctl[16 + w];
                        ctl[16 + w] = cb;
                        cb += m;
                    }
                    ctl[3] = cb;
                }
            }
            __syncthreads();
            // (2) stable scatter into buckets
            const int cb = ctl[16 + warp];
            for (int i0 = 0; i0 < mine; i0 += 32) {
                const int c = i0 + lane;
                const bool valid = c < mine;
                int32_t lab = kEmpty;
                double val = 0.0;
                if (valid) {
                    lab = Slab[sbase + c];
                    val = Sval[sbase + c];
                }
                const uint32_t q = valid ? part_of(lab, (uint32_t)P) : 0xffffffffu;
                const uint32_t grp = __match_any_sync(0xffffffffu, q);
                int pos = 0;
                if (valid) pos = Wc[warp * P + q] + __popc(grp & lanemask_lt());
                __syncwarp();
                if (valid && (__ffs(grp) - 1) == lane) Wc[warp * P + q] += __popc(grp);
                if (valid) {
                    LP_CHECK(pos >= 0 && (size_t)pos < Cc, "bucket position");
                    Blab[pos] = lab;
                    Bval[pos] = val;
                    Bc[pos] = cb + c;
                }
                __syncwarp();
            }
            __syncthreads();
            // (3) tally the buckets
            for (int q = warp; q < P; q += W) {
                const int qb = Qs[q], qe = Qs[q + 1];
                int cnt = 0;
                bool over = false;
                for (int i0 = qb; i0 < qe; i0 += 32) {
                    const int i = i0 + lane;
                    const bool valid = i < qe;
                    tally_chunk(valid ? Blab[i] : kEmpty, valid ? Bval[i] : 0.0, valid ? Bc[i] : 0, keys, vals, firsts,
                                tl, kCopraTeamBits, cnt, sm.stage);
                    if (cnt > kCopraTeamLimit) {
                        over = true;
                        break;
                    }
                }
                if (over) {
                    table_restore(keys, vals, tl, cnt);
                    if (lane == 0) ctl[2] = 1;
                    break;
                }
                int base = 0;
                if (lane == 0) base = atomicAdd(ctl + 1, cnt);
                base = __shfl_sync(0xffffffffu, base, 0);
                for (int i = lane; i < cnt; i += 32) {
                    const int sl = tl[i];
                    LP_CHECK((size_t)(base + i) < D, "entry index");
                    Elab[base + i] = keys[sl];
                    Eval[base + i] = vals[sl];
                    Efirst[base + i] = firsts[sl];
                    keys[sl] = kEmpty;
                    vals[sl] = 0.0;
                }
                __syncwarp();
            }
            __syncthreads();
            if (ctl[2] == 0) break;
            if (P >= kCopraMaxParts) {  // cannot happen for n <= 1.5M; reported, never silent
                if (tid == 0) atomicAdd(a.counters + kCtrCount + 1, 1ull);
                break;
            }
            P *= 2;
        }
        // (4) finish without the first-touch order when possible: the parallel
        // total decides every qualification test (see copra_finish), the
        // qualifiers (few) are ordered by their first contribution, and the
        // fallback tie-break uses the first contribution too.  An undecided
        // test or too many qualifiers take the ordered path below.
        const int nent = ctl[1], C = ctl[3];
        {
            double tp = 0.0;
            bool ai = true;
            for (int e = tid; e < nent; e += blockDim.x) {
                const double w = Eval[e];
                tp += w;
                ai &= w == floor(w);
            }
#pragma unroll
            for (int m = 16; m >= 1; m >>= 1) tp += __shfl_xor_sync(0xffffffffu, tp, m);
            ai = __all_sync(0xffffffffu, ai);
            if (lane == 0) {
                s_red[warp] = tp;
                s_ai[warp] = ai ? 1 : 0;
            }
            if (tid == 0) {
                s_nq = 0;
                s_und = 0;
            }
            __syncthreads();
            double T = 0.0;
            bool AI = true;
            for (int w2 = 0; w2 < W; ++w2) {
                T += s_red[w2];
                AI = AI && s_ai[w2];
            }
            AI = AI && T < 9007199254740992.0;
            const double band = AI ? 0.0 : T * (double)(nent + 32) * 2.220446049250313e-16;
            for (int e = tid; e < nent; e += blockDim.x) {
                const double p = __dmul_rn(Eval[e], (double)a.K);
                if (AI ? p >= T : p >= T + band) {
                    const int qi = atomicAdd(&s_nq, 1);
                    if (qi < kQualMax) {
                        s_qfirst[qi] = Efirst[e];
                        s_qlab[qi] = Elab[e];
                        s_qw[qi] = Eval[e];
                    }
                } else if (!AI && !(p < T - band)) {
                    s_und = 1;
                }
            }
            __syncthreads();
            if (!s_und && s_nq <= kQualMax) {
                if (warp == 0) {
                    const int nq = s_nq, K = a.K;
                    int kk = 0;
                    int32_t mylab = 0;
                    double myb = 0.0;
                    if (nq > 0) {
                        // the first <= K qualifiers in touched order
                        for (int qi = lane; qi < nq; qi += 32) {
                            int rank = 0;
                            for (int j = 0; j < nq; ++j) rank += s_qfirst[j] < s_qfirst[qi];
                            if (rank < K) {
                                sm.outl[rank] = s_qlab[qi];
                                sm.outb[rank] = s_qw[qi];
                            }
                        }
                        __syncwarp();
                        kk = min(nq, K);
                        double kept = 0.0;
                        for (int i = 0; i < kk; ++i) kept = __dadd_rn(kept, sm.outb[i]);  // (every lane)
                        const double inv = __ddiv_rn(1.0, kept);
                        if (lane < kk) {
                            mylab = sm.outl[lane];
                            myb = __dmul_rn(sm.outb[lane], inv);
                        }
                    } else {
                        // fallback (copra.py:72-93): maximum tally; the largest counter
                        // hash among tied maxima, the earliest first touch on equal hashes
                        double bw = -1.0;
                        for (int e = lane; e < nent; e += 32) bw = fmax(bw, Eval[e]);
#pragma unroll
                        for (int m = 16; m >= 1; m >>= 1) bw = fmax(bw, __shfl_xor_sync(0xffffffffu, bw, m));
                        const uint32_t vv = (uint32_t)__ldg(a.svid + s);
                        uint32_t bh = 0, bf = 0xffffffffu;
                        int32_t bl = kEmpty;
                        for (int e = lane; e < nent; e += 32) {
                            if (Eval[e] != bw) continue;
                            const uint32_t h = tie_hash(a.seed, a.sweep, vv, (uint32_t)Elab[e]);
                            const uint32_t f = (uint32_t)Efirst[e];
                            if (bl == kEmpty || h > bh || (h == bh && f < bf)) {
                                bh = h;
                                bf = f;
                                bl = Elab[e];
                            }
                        }
#pragma unroll
                        for (int m = 16; m >= 1; m >>= 1) {
                            const uint32_t oh = __shfl_xor_sync(0xffffffffu, bh, m);
                            const uint32_t of = __shfl_xor_sync(0xffffffffu, bf, m);
                            const int32_t ol = __shfl_xor_sync(0xffffffffu, bl, m);
                            if (ol != kEmpty && (bl == kEmpty || oh > bh || (oh == bh && of < bf))) {
                                bh = oh;
                                bf = of;
                                bl = ol;
                            }
                        }
                        kk = 1;
                        if (lane == 0) {
                            mylab = bl;
                            myb = 1.0;
                        }
                    }
                    copra_commit(a, s, nent, kk, mylab, myb);
                }
                continue;
            }
        }
        // ordered path: F[first] = entry, then an ordered compaction of F
        LP_CHECK((size_t)C <= Cc, "contributions");
        for (int e = tid; e < nent; e += blockDim.x) {
            LP_CHECK(Efirst[e] >= 0 && Efirst[e] < C, "first index");
            F[Efirst[e]] = e;
        }
        __syncthreads();
        int run = 0;  // entries placed so far (block-uniform)
        for (int c0 = 0; c0 < C; c0 += blockDim.x) {
            const int c = c0 + tid;
            const int e = c < C ? F[c] : -1;
            const bool has = e >= 0;
            const uint32_t bal = __ballot_sync(0xffffffffu, has);
            if (lane == 0) sm.outl[0] = __popc(bal);  // per-warp count (outl reused as scratch)
            __syncthreads();
            int before = run;
            for (int w = 0; w < warp; ++w) before += sms[w].outl[0];
            if (has) {
                const int r = before + __popc(bal & lanemask_lt());
                LP_CHECK((size_t)r < D && e < nent, "rank");
                Rlab[r] = Elab[e];
                Rval[r] = Eval[e];
                F[c] = -1;
            }
            for (int w = 0; w < W; ++w) run += sms[w].outl[0];
            __syncthreads();
        }
        if (warp == 0)
            copra_finish(a, s, nent, [&](int i, int32_t& l, double& w) {
                l = Rlab[i];
                w = Rval[i];
            }, sm);
    }
}

__global__ void k_fill_i32(int32_t* p, int32_t v, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
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
__global__ void k_clear_marks(const int32_t* __restrict__ q, const int32_t* __restrict__ qlen,
                              unsigned long long* mark) {
    const int cnt = *qlen;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) mark[q[i]] = 0ull;
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
