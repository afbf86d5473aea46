// lp_rak_kernels.cuh -- the RAK sweep kernels (the hot path).
//
// Replaces the body of the reference's sweep, rak.py:97-113 (_rak_seq) /
// :138-154 (_rak_par): for each vertex, accumulate the weights of its
// neighbours' labels, take the argmax under the tie rule, write the label
// and count the change.
//
// Every round has two phases.  Phase 1 (k_gather_*) streams the neighbour
// index of every arc of the rows to evaluate and gathers that neighbour's
// label into an arc-aligned buffer `lbuf` -- a flat, coalesced pass with
// eight loads in flight per thread, which is what the memory system needs
// (a warp walking one row at a time keeps too few loads in flight).
// Phase 2 (the kernels below) tallies each row from `lbuf`, contiguously.
//
// Work is routed per round by the degree d and an estimate `est` of the
// vertex's distinct neighbour labels (the count seen at its previous
// evaluation, plus margin): label diversity collapses after the first sweep,
// so the table a vertex needs shrinks with it.
//
//   k_small  thread per vertex (d <= 16): register tally, O(d^2) compares
//   k_warp   warp per vertex (est <= 256, d <= 2048): 512-slot shared hash;
//            __match_any_sync folds equal labels of a 32-arc chunk so one
//            leader lane updates the table per distinct label; the argmax is
//            a __shfl_xor_sync reduction over the touched list; 128 arcs of
//            gathers in flight per warp.  Overflow spills the vertex to k_team.
//   k_team   block per work item: 8 warps / 4096-slot table for mid rows,
//            16 warps / 8192-slot table for hubs.  A hub item is
//              (vertex, label partition q of P): labels split by hash so each
//                partition's distinct labels fit one table; partitions run on
//                different blocks, the last to finish merges P candidates;
//              (vertex, arc slice r of R): a huge row with few distinct labels
//                is cut into R slices; slice blocks tally in shared memory and
//                fold their tables into a small per-vertex global table
//                (L2-resident); the last slice takes the argmax.
//            A shared table that overflows is split 4-way again (work stack),
//            so every item completes in the round it was routed to.
//
// The changed-vertex count (rak.py:111-113) is fused: per-thread deltas,
// one atomic per warp.
#pragma once
#include <type_traits>

#include "lp_common.cuh"

namespace lp {

struct HubCand {
    unsigned long long w;  // weight bits (u32 / u64 / float bits)
    unsigned long long w2; // runner-up weight bits (margin test)
    uint32_t sec;
    uint32_t ter;
    int32_t lab;
    int32_t nd;
    int32_t single;  // kSingle labels absent from this partition's table
};

// A k_team work item.
struct Item {
    int32_t s;   // slot
    int32_t q;   // partition index
    int32_t P;   // partitions
    int32_t r;   // slice index
    int32_t R;   // slices
    int32_t cb;  // merge state base (cand[cb..cb+P), cand_done[cb]); -1 when P = R = 1
    int32_t gt;  // global slice-table base (entries), R > 1
    int32_t gbits;  // global slice table of 2^gbits slots, R > 1
};

// route-list lengths / cursors (device ints)
enum {
    kLenS4 = 0,   // small rows, d <= 4
    kLenS8 = 1,   // d <= 8
    kLenS16 = 2,  // d <= 16
    kLenWarp = 3,     // warp per vertex, 512-slot table
    kLenTeam = 4,
    kLenHub = 5,
    kLenWarpBig = 6,  // warp per vertex, 2048-slot table
    kCandCursor = 7,
    kTeamCursor = 8,
    kHubCursor = 9,
    kGtabCursor = 10,
    kWarpCursor = 11,  // + warp class (0 / 1)
    kLenGather = 13,   // phase-1 pieces (row, arc range) of frontier rounds
    kGatherCursor = 14,
    kLenChg = 15,      // pieces of the rows whose label changed this round (deferred marks)
    kChgCursor = 16,
    kLenTeam2 = 17,    // 16-warp team, 8192-slot table (est <= kTeam2Est, d <= kTeamMaxDeg)
    kTeam2Cursor = 18,
    kLenMid = 19,      // thread per row, kSmallMax < d <= kMidMax (k_mid)
    kLenRouted = 20,   // pieces of every routed row, fused or not (the round-size decisions)
    kLenCount = 21
};

struct Routes {
    int32_t* small[3];  // slot lists by small degree class (4, 8, 16)
    int32_t* mid;       // thread-per-row rows of kSmallMax < d <= kMidMax
    int32_t* warp[2];   // slot lists of the two warp classes
    Item* team;
    Item* team2;
    Item* hub;
    int32_t* len;  // kLen*
    HubCand* cand;
    int32_t* cand_done;
    int64_t gcap;    // slots in the global slice-table pool
    int32_t* gtl;    // per slice table: slots of its entries in insertion order (same indexing)
    int32_t* gkeys;  // global slice tables (SoA)
    uint32_t* gfirst;
    unsigned long long* gacc;
    int32_t* gcount;  // distinct count per slice table (indexed by cb)
    int32_t* gslot;   // frontier rounds: phase-1 pieces: slot ...
    int32_t* gk0;     // ... and first arc of the piece within the row (<= kPieceArcs arcs)
    int32_t* cslot;   // changed rows as pieces: slot ...
    int32_t* ck0;     // ... and first arc
};

struct EvalArgs {
    const uint32_t* __restrict__ soff;  // storage row offsets [S+1]
    const uint32_t* __restrict__ snbr;  // neighbour vertex id << 2 | kEarlier | kLater
    const uint32_t* __restrict__ sw;    // arc weights (fixed-point u32 or float bits); null = unit
    const unsigned long long* __restrict__ swsum;  // per-slot total weight (fixed mode), null otherwise
    const int32_t* __restrict__ svid;   // slot -> vertex id
    const int32_t* __restrict__ L0;     // labels at sweep start, by vertex id (read-only in a sweep)
    int32_t* x;                         // working labels, by vertex id
    int32_t* lbuf;                      // phase 1 output: label of every arc's neighbour
    unsigned long long* mark;           // next-round marks by vertex id: weight of the changed earlier
                                        // neighbours since the last routing (0 = unmarked); null = no
                                        // cross-batch deps
    unsigned long long* gap;            // per slot: lower bound of (winner - runner-up) weight at the
                                        // last evaluation (0 = unknown); null = no margin skipping
    const int32_t* __restrict__ pos;    // vertex -> visit position (wave horizon test)
    int32_t mark_all;                   // 0: mark later-batch neighbours (inside a sweep); 2: the sweep
                                        // boundary, every neighbour that reads this row's sweep-start
                                        // label (not the later-batch ones); 1: every neighbour
    int32_t horizon;                    // dense waves: only positions < horizon have been evaluated
                                        // this sweep and need marks; INT32_MAX = all
    int32_t* mq_out;                    // queue of newly marked vertices (this round's writes)
    int32_t* mq_len;                    // its length
    uint32_t* mbits;                    // marked-vertex bitmap: the pass kernels set bits with fire-and-
                                        // forget atomics, k_bits_to_queue compacts them into mq_out
    int32_t* ndist;                     // per-slot distinct-label count of the last evaluation
    unsigned long long* counters;       // see kCtr* below
    Routes r;
    int32_t bin;  // counter slot of this launch
    uint32_t seed;
    uint32_t sweep;                     // RAK: sweep number; SLPA: speaking round t
    const int32_t* __restrict__ slots;  // SLPA memories [n x T] (slot t lives in x until the round ends)
    int32_t T;
    int32_t cap_route;  // route a row to the smallest table that holds d entries even when its
                        // estimate is larger (such a row can never overflow that table)
    int32_t id_single;  // first sweep from labels = ids, duplicate-free rows: see kSingle
    int32_t two_team;   // ... and unit weights: the team / hub kernels take the two passes too
    int32_t warp_maxd[2];  // longest row routed to warp class 0 / 1 (longer rows go to the teams)
    int32_t reg_est;       // rows estimated to hold more labels skip the warp register table
    int32_t mid_max;       // rows of kSmallMax < d <= mid_max go to k_mid (0 = off)
    int32_t first_est_min, first_est_div;  // first round of a singleton sweep: rows longer than
                                           // first_est_min estimate d / first_est_div labels
    // hub rows split into P > 1 label partitions: k_hub_bucket reorders each
    // row's labels (and arc positions) by partition, so a partition block reads
    // its own bucket instead of the whole row (null = off)
    int32_t* hb_lab;
    uint32_t* hb_pos;
    int2* hb_off;  // per partition item (cb + q): (bucket start, length); length -1 = not bucketed
    // fused gather (RAK): the tally kernels read each arc's neighbour index and
    // gather its label themselves (arc_label) instead of a phase-1 pass through
    // lbuf -- 8 bytes per arc less DRAM traffic and no separate gather launch
    int32_t fused = 0;
    int32_t fuse_maxd = 0;  // rows of degree <= fuse_maxd are fused: routing adds no phase-1 pieces for them
};

// First sweep from labels = vertex ids (rak.py:168): a neighbour that has not
// been evaluated yet this sweep still carries its own id, so (rows being
// duplicate-free) its label occurs once in the row unless an evaluated
// neighbour's label equals it.  Phase 1 then stores the id with kSingle set
// (no label load), and the hash tallies run two passes: evaluated labels are
// inserted, flagged ones are only looked up (bumped when present, else counted
// as singletons of weight 1).  With unit weights a singleton cannot win unless
// every label has weight 1 -- then the winner is picked over all arcs.  The
// tables hold a few percent of the row instead of half of it.
constexpr int32_t kSingle = 1 << 30;
__device__ __forceinline__ int32_t lb_strip(const EvalArgs& a, int32_t v) { return a.id_single ? (v & ~kSingle) : v; }  // (v >= 0)


// phase-1 variants: what an arc's neighbour contributes to the tally
enum GatherAlg : int { kGatherRak = 0, kGatherSlpa = 1 };

// neighbour flags (low bits of snbr): the neighbour is in an earlier batch
// (read its current-sweep label) / in a later batch (mark it when this
// row's label changes).  Neither: same batch -> sweep-start label.
constexpr uint32_t kEarlier = 1u, kLater = 2u;

// counters: [0] changed delta (reset per sweep), [1] label writes (reset per
// round), [4+k] arcs scanned and [8+k] vertices evaluated by kernel k
// (k = 0 hub team, 1 8-warp team, 2 warp, 3 small; accumulated over a run)
// [14] kernel-side failures (a team table split stack exhausted): the run fails
enum { kCtrChanged = 0, kCtrWrites = 1, kCtrGathered = 2, kCtrArcs = 4, kCtrVerts = 8, kCtrError = 14, kCtrCount = 15 };

// ndist[s]: low 30 bits = distinct labels seen at the last evaluation;
// kMajBit = that evaluation's winner held a strict majority of the row's
// weight.  A vertex flagged so first tries the majority check: count the
// weight of its current label; if it exceeds half the row it is the unique
// argmax (no tie is possible) and the tally is skipped entirely.
constexpr int32_t kMajBit = 1 << 30;
__host__ __device__ __forceinline__ int32_t nd_count(int32_t v) { return v & (kMajBit - 1); }

#ifdef LP_PATH_STATS
#define LP_STAT(a, k) atomicAdd((a).counters + 20 + (k), 1ull)  // (past COPRA's kCtrCount + 1)
#else
#define LP_STAT(a, k) \
    do {              \
    } while (0)
#endif

#ifndef LP_TEAM_U
#define LP_TEAM_U 2
#endif
#ifndef LP_TEAM_J2
#define LP_TEAM_J2 4  // label loads in flight per lane in the team kernels' flagged-label lookups
#endif
constexpr int kSmallMax = 16;     // thread-per-vertex bound (degree)
#ifndef LP_WARP_REG_EST
#define LP_WARP_REG_EST 8  // rows estimated to hold more labels skip the warp register table (LP_REG_EST;
                           // 8 measured 4% faster than 32 on R-MAT-22: the register table costs a
                           // ballot per entry per chunk)
#endif
// warp classes: 0 = 512-slot table (est <= 256, d <= 2048, 8 warps/block),
// 1 = 1024-slot table (est <= 512, d <= 8192, 4 warps/block)
template <int WC> struct WarpClass;
template <> struct WarpClass<0> {
    static constexpr int kBits = 9, kEst = 256, kMaxDeg = 2048, kWarps = 8, kList = 3;
};
template <> struct WarpClass<1> {
    static constexpr int kBits = 10, kEst = 512, kMaxDeg = 8192, kWarps = 4, kList = 6;  // (4: +25% resident warps)
};
constexpr int kWarpEst = WarpClass<0>::kEst;
constexpr int kTeamEst = 2048;    // 8-warp team: 4096-slot table
constexpr int kTeamMaxDeg = 16384;
constexpr int kTeamBits = 12, kTeamThreads = 256;
constexpr int kTeam2Bits = 13, kTeam2Threads = 512;  // 16-warp team: 8192 slots
constexpr int kTeam2Est = 6144;
constexpr int kHubBits = 14, kHubThreads = 1024;  // 32-warp team: 16384 slots
constexpr int kHubPlan = 8192;     // distinct labels planned per hub partition
constexpr int kSliceArcs = 8192;   // arcs per slice
constexpr int kSliceEst = 1024;    // slicing only when distinct labels are few
constexpr int kGlobalBits = 11;    // per-vertex global slice table: 2048 slots
constexpr int kGlobalCap = 1536;

template <int WM> __device__ __forceinline__ typename Acc<WM>::T arc_weight(const EvalArgs& a, uint32_t e) {
    if constexpr (WM == kUnit) {
        return 1u;
    } else if constexpr (WM == kFixed) {
        return (unsigned long long)__ldg(a.sw + e);
    } else {
        return (double)__uint_as_float(__ldg(a.sw + e));
    }
}

// Label of a neighbour under the batched schedule (phase 1).
__device__ __forceinline__ int32_t gather_label(const EvalArgs& a, uint32_t nb) {
    const int32_t u = (int32_t)(nb >> 2);
    if (nb & kEarlier) return a.x[u];
    return a.id_single ? (u | kSingle) : __ldg(a.L0 + u);  // (first sweep: L0[u] == u)
}

// Label of arc e as the tally sees it: fused rounds gather it here (a read of x
// may race with another row's write this round; the writer marks this row, so
// the next round repeats the evaluation -- the fixed point is unchanged, and
// the synchronous schedule reads only the immutable L0); two-phase rounds read
// the phase-1 buffer.
__device__ __forceinline__ int32_t arc_label(const EvalArgs& a, uint32_t e) {
    if (a.fused) return gather_label(a, __ldg(a.snbr + e));
    return a.lbuf[e];
}

__device__ __forceinline__ void flush_counters(const EvalArgs& a, long long dchg, long long arcs, long long writes,
                                               long long verts) {
    // one atomic per warp per counter (all lanes of the warp reach this point)
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        dchg += __shfl_xor_sync(0xffffffffu, dchg, m);
        arcs += __shfl_xor_sync(0xffffffffu, arcs, m);
        writes += __shfl_xor_sync(0xffffffffu, writes, m);
        verts += __shfl_xor_sync(0xffffffffu, verts, m);
    }
    if ((threadIdx.x & 31) == 0) {
        if (dchg) atomicAdd(a.counters + kCtrChanged, (unsigned long long)dchg);
        if (arcs) atomicAdd(a.counters + kCtrArcs + a.bin, (unsigned long long)arcs);
        if (writes) atomicAdd(a.counters + kCtrWrites, (unsigned long long)writes);
        if (verts) atomicAdd(a.counters + kCtrVerts + a.bin, (unsigned long long)verts);
    }
}

// Record the winner's margin over the rest of the row (lower bound
// 2 * winner - total, useful when the winner holds a strict majority).
template <typename A> __device__ __forceinline__ void store_gap(const EvalArgs& a, int32_t s, A win, A total) {
    if (a.gap) {
        if constexpr (std::is_floating_point<A>::value) {
            a.gap[s] = 0ull;
        } else {
            a.gap[s] = (win + win > total) ? (unsigned long long)(win + win - total) : 0ull;
        }
    }
}

// Record the exact lead of the winner (largest label weight w1) over the
// runner-up (w2).
template <typename A> __device__ __forceinline__ void store_lead(const EvalArgs& a, int32_t s, A w1, A w2) {
    if (a.gap) {
        if constexpr (std::is_floating_point<A>::value)
            a.gap[s] = 0ull;
        else
            a.gap[s] = (unsigned long long)(w1 - w2);
    }
}

// Write a vertex's new label (one thread).  Returns true when it changed.
__device__ __forceinline__ bool commit_label(const EvalArgs& a, int32_t v, int32_t lab, long long& dchg,
                                             long long& writes) {
    const int32_t old = a.x[v];
    if (lab == old || lab < 0) return false;
    a.x[v] = lab;
    const int32_t l0 = __ldg(a.L0 + v);
    dchg += (long long)(lab != l0) - (long long)(old != l0);
    ++writes;
    return true;
}

// Same, with the vertex's current and sweep-start labels already loaded.
__device__ __forceinline__ bool commit_label_known(const EvalArgs& a, int32_t v, int32_t lab, int32_t old, int32_t l0,
                                                   long long& dchg, long long& writes) {
    if (lab == old || lab < 0) return false;
    a.x[v] = lab;
    dchg += (long long)(lab != l0) - (long long)(old != l0);
    ++writes;
    return true;
}

// Mark the later-batch neighbours of a vertex whose label changed; a vertex
// marked for the first time this round joins the mark queue (warp-aggregated
// append), so the next round routes only the queue instead of scanning n.
// A later-batch neighbour needs a mark only if it may already have read this
// vertex's label this sweep: during the dense waves, only positions below the
// horizon have been evaluated (a later wave reads the new label anyway).
__device__ __forceinline__ bool needs_mark(const EvalArgs& a, int32_t u) {
    return a.horizon == INT32_MAX || __ldg(a.pos + u) < a.horizon;
}
template <typename Args> __device__ __forceinline__ bool needs_mark(const Args&, int32_t) { return true; }

// weight a change adds to a neighbour's mark (margin units: counts, or the
// fixed-point weights; 1 when margins are not tracked)
__device__ __forceinline__ unsigned long long mark_weight(const EvalArgs& a, uint32_t e) {
    return (a.gap && a.sw) ? (unsigned long long)__ldg(a.sw + e) : 1ull;
}
template <typename Args> __device__ __forceinline__ unsigned long long mark_weight(const Args&, uint32_t) {
    return 1ull;
}

template <typename Args>
__device__ __forceinline__ void mark_row(const Args& a, uint32_t beg, int d, int from, int step) {
    const int lane = threadIdx.x & 31;
    for (int k = from; k < d; k += step) {
        const uint32_t nb = __ldg(a.snbr + beg + k);
        const int32_t u = (int32_t)(nb >> 2);
        const bool win =
            (nb & kLater) && needs_mark(a, u) && atomicAdd(a.mark + u, mark_weight(a, beg + k)) == 0ull;
        const uint32_t act = __activemask();
        const uint32_t bal = __ballot_sync(act, win);
        if (bal) {
            const int leader = __ffs(bal) - 1;
            int b0 = 0;
            if (lane == leader) b0 = atomicAdd(a.mq_len, __popc(bal));
            b0 = __shfl_sync(act, b0, leader);
            if (win) a.mq_out[b0 + __popc(bal & lanemask_lt())] = u;
        }
    }
}

// ---------------------------------------------------------------------------
// phase 1: label gather
// ---------------------------------------------------------------------------
// Dense round: every arc of the active slots, flat and coalesced.
__global__ void __launch_bounds__(256) k_gather_dense(EvalArgs a, int64_t m) {
    constexpr int J = 8;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < m; base += stride * J) {
        uint32_t nb[J];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int64_t e = base + j * stride;
            nb[j] = e < m ? __ldg(a.snbr + e) : 0u;
        }
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const int64_t e = base + j * stride;
            if (e < m) a.lbuf[e] = gather_label(a, nb[j]);
        }
    }
}

// Frontier round: the routed rows, as pieces of at most kPieceArcs arcs.  A
// warp takes 32 pieces at a time (lane j loads piece j), scans their lengths
// in registers and streams the flattened arcs eight loads deep; each lane
// finds its piece by a 5-step search over the warp's prefix (shuffles only).
constexpr int kPieceArcs = 256;

// Pieces a warp takes at a time: 32 (one per lane) when there are plenty, fewer
// when a short list -- often a few hub rows of a late frontier round -- would
// otherwise leave most of the grid idle behind a handful of warps.
__device__ __forceinline__ int pieces_per_warp(int cnt) {
    const int warps = (int)(gridDim.x * blockDim.x / 32);
    return max(1, min(32, cnt / max(warps, 1)));
}

template <int ALG>
__global__ void __launch_bounds__(256) k_gather_pieces(EvalArgs a, const int32_t* __restrict__ gslot,
                                                       const int32_t* __restrict__ gk0,
                                                       const int32_t* __restrict__ count, int32_t* cursor) {
    constexpr int J = 8;
    const int lane = threadIdx.x & 31;
    const int cnt = *count;
    const int per = pieces_per_warp(cnt);
    while (true) {
        int b0 = 0;
        if (lane == 0) b0 = atomicAdd(cursor, per);
        b0 = __shfl_sync(0xffffffffu, b0, 0);
        if (b0 >= cnt) break;
        uint32_t pbeg = 0, plen = 0, pk0 = 0;
        int32_t pv = 0;
        if (lane < per && b0 + lane < cnt) {
            const int32_t s = gslot[b0 + lane];
            pk0 = (uint32_t)gk0[b0 + lane];
            const uint32_t rb = __ldg(a.soff + s), re = __ldg(a.soff + s + 1);
            pbeg = rb + pk0;
            plen = min((uint32_t)kPieceArcs, re - pbeg);
            if (ALG == kGatherSlpa) pv = __ldg(a.svid + s);
        }
        // inclusive prefix of piece lengths
        uint32_t incl = plen;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - plen;
        if (lane == 0) atomicAdd(a.counters + kCtrGathered, (unsigned long long)total);
        for (uint32_t base = 0; base < total; base += 32 * J) {
            uint32_t e[J];
            uint32_t nb[J];
            uint32_t key[J];
            int32_t lv[J];
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const uint32_t i = base + j * 32 + lane;
                // piece r: largest r with excl[r] <= i
                int r = 0;
#pragma unroll
                for (int step = 16; step >= 1; step >>= 1) {
                    const uint32_t ex = __shfl_sync(0xffffffffu, excl, r + step);
                    if (r + step < 32 && ex <= i) r += step;
                }
                const uint32_t pb = __shfl_sync(0xffffffffu, pbeg, r);
                const uint32_t pe = __shfl_sync(0xffffffffu, excl, r);
                if (ALG == kGatherSlpa) {
                    key[j] = __shfl_sync(0xffffffffu, pk0, r) + (i - pe);  // arc index within the row
                    lv[j] = __shfl_sync(0xffffffffu, pv, r);
                }
                e[j] = i < total ? pb + (i - pe) : 0xffffffffu;
                nb[j] = i < total ? __ldg(a.snbr + e[j]) : 0u;
            }
#pragma unroll
            for (int j = 0; j < J; ++j) {
                if (e[j] == 0xffffffffu) continue;
                if (ALG == kGatherRak) {
                    a.lbuf[e[j]] = gather_label(a, nb[j]);
                } else {
                    // slpa.py:76-77: the speaker u says slots[u, draw(filled[u])]; u has
                    // t + 1 filled slots if it is in an earlier batch (it already
                    // listened and appended this round), else t.
                    const int32_t u = (int32_t)(nb[j] >> 2);
                    const uint32_t t = a.sweep;
                    const uint32_t filled = t + ((nb[j] & kEarlier) ? 1u : 0u);
                    const uint32_t q = speak_hash(a.seed, t, (uint32_t)lv[j], key[j]) % filled;
                    a.lbuf[e[j]] = q == t ? a.x[u] : __ldg(a.slots + (size_t)u * a.T + q);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// deferred marks
// ---------------------------------------------------------------------------
// A vertex whose label changed does not walk its row inline (a dependent
// row load plus one returning atomic per 32 arcs, fully exposed in the tally
// kernels); it appends its row, as pieces, to the changed list, and
// k_mark_pieces walks all changed rows after the round's tally kernels with
// eight loads in flight per lane.

// one thread: push row s (d arcs)
__device__ __forceinline__ void push_changed(const EvalArgs& a, int32_t s, int d) {
    const int np = (d + kPieceArcs - 1) / kPieceArcs;
    const int b0 = atomicAdd(a.r.len + kLenChg, np);
    for (int q = 0; q < np; ++q) {
        a.r.cslot[b0 + q] = s;
        a.r.ck0[b0 + q] = q * kPieceArcs;
    }
}

// active lanes of a warp, rows of <= kPieceArcs arcs: one atomic per warp
__device__ __forceinline__ void push_changed_small(const EvalArgs& a, bool ch, int32_t s) {
    const uint32_t act = __activemask();
    const uint32_t bal = __ballot_sync(act, ch);
    if (!bal) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(bal) - 1;
    int b0 = 0;
    if (lane == leader) b0 = atomicAdd(a.r.len + kLenChg, __popc(bal));
    b0 = __shfl_sync(act, b0, leader);
    if (ch) {
        const int idx = b0 + __popc(bal & lanemask_lt());
        a.r.cslot[idx] = s;
        a.r.ck0[idx] = 0;
    }
}

// every thread of a <= 1024-thread block, rows of <= kPieceArcs arcs: one atomic per block (the
// changed list's length is one counter for the whole grid; a dense round of small rows appended
// to it once per warp, ~100K times in ~100 us).  sw: 2 x 34 shared words, `par` alternates.
__device__ __forceinline__ void push_changed_block(const EvalArgs& a, bool ch, int32_t s, int32_t (*sw)[34], int par) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    const uint32_t bal = __ballot_sync(0xffffffffu, ch);
    int32_t* w = sw[par & 1];
    if (lane == 0) w[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
        const int c = lane < nw ? w[lane] : 0;
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        int b0 = 0;
        if (lane == 0 && tot) b0 = atomicAdd(a.r.len + kLenChg, tot);
        b0 = __shfl_sync(0xffffffffu, b0, 0);
        if (lane < nw) w[lane] = b0 + incl - c;
    }
    __syncthreads();
    if (ch) {
        const int idx = w[warp] + __popc(bal & lanemask_lt());
        a.r.cslot[idx] = s;
        a.r.ck0[idx] = 0;
    }
}

// ... the same for rows of any length (np pieces each; every thread of the block calls)
__device__ __forceinline__ void push_changed_rows_block(const EvalArgs& a, bool ch, int32_t s, int d, int32_t (*sw)[34],
                                                        int par) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    const int np = ch ? (d + kPieceArcs - 1) / kPieceArcs : 0;
    int wi = np;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
    }
    int32_t* w = sw[par & 1];
    if (lane == 31) w[warp] = wi;
    __syncthreads();
    if (warp == 0) {
        const int c = lane < nw ? w[lane] : 0;
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        int b0 = 0;
        if (lane == 0 && tot) b0 = atomicAdd(a.r.len + kLenChg, tot);
        b0 = __shfl_sync(0xffffffffu, b0, 0);
        if (lane < nw) w[lane] = b0 + incl - c;
    }
    __syncthreads();
    const int at = w[warp] + wi - np;
    for (int q = 0; q < np; ++q) {
        a.r.cslot[at + q] = s;
        a.r.ck0[at + q] = q * kPieceArcs;
    }
}

// whole warp: lane v pushes row (s, d) when bit v of `chm` is set
__device__ __forceinline__ void push_changed_batch(const EvalArgs& a, uint32_t chm, int32_t s, int d) {
    const int lane = threadIdx.x & 31;
    const int np = ((chm >> lane) & 1u) ? (d + kPieceArcs - 1) / kPieceArcs : 0;
    int incl = np;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    const int tot = __shfl_sync(0xffffffffu, incl, 31);
    int b0 = 0;
    if (lane == 31 && tot) b0 = atomicAdd(a.r.len + kLenChg, tot);
    b0 = __shfl_sync(0xffffffffu, b0, 31);
    for (int q = 0; q < np; ++q) {
        a.r.cslot[b0 + incl - np + q] = s;
        a.r.ck0[b0 + incl - np + q] = q * kPieceArcs;
    }
}

// Sweep boundary: the rows whose label differs between two label arrays
// (this sweep's result vs the previous one) join the changed list, so that
// k_mark_pieces (mark_all) can queue every neighbour for the next sweep.
__global__ void k_sweep_changes(EvalArgs a, const int32_t* __restrict__ lnew, const int32_t* __restrict__ lold,
                                int32_t S) {
    __shared__ int32_t s_push[2][34];
    int par = 0;
    for (int32_t base = blockIdx.x * blockDim.x; base < S; base += gridDim.x * blockDim.x, ++par) {
        const int32_t s = base + threadIdx.x;
        bool ch = false;
        int d = 0;
        if (s < S) {
            const int32_t v = __ldg(a.svid + s);
            ch = lnew[v] != lold[v];
            d = (int)(__ldg(a.soff + s + 1) - __ldg(a.soff + s));
        }
        push_changed_rows_block(a, ch, s, d, s_push, par);
    }
}

// changed flags of the rows on the changed list (first pieces)
// Changed-vertex flags are a bitmap (bit v of word v / 32): the pull pass
// gathers one flag per arc, and 512 KB for R-MAT-22 stays cache-resident
// where a byte array (4 MB) thrashes L1.
__device__ __forceinline__ bool chg_bit(const uint32_t* __restrict__ chg, int32_t v) {
    return (__ldg(chg + (v >> 5)) >> (v & 31)) & 1u;
}

__global__ void k_flags_from_changed(EvalArgs a, uint32_t* __restrict__ chg) {
    const int cnt = a.r.len[kLenChg];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x)
        if (a.r.ck0[i] == 0) {
            const int32_t v = __ldg(a.svid + a.r.cslot[i]);
            atomicOr(chg + (v >> 5), 1u << (v & 31));
        }
}

// (whole warps: 32 consecutive vertices -> one bitmap word)
// Random ties (non-strict): the winner among tied labels is drawn from a hash
// keyed by the sweep, so a vertex whose last evaluation ended in a tie (lead 0)
// may move although no neighbour changed.  At a sweep boundary those vertices
// join the frontier next to the neighbours of the changed ones (a lead > 0
// with an unchanged neighbourhood keeps its label: the draw is not consulted).
__global__ void k_mark_ties(EvalArgs a, int32_t S) {
    for (int32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
        if (a.gap[s] != 0ull) continue;
        const int32_t v = __ldg(a.svid + s);
        atomicOr(a.mark + v, 1ull);  // (nonzero: queued by either compaction; +1 only widens the margin test)
        if (a.mbits) atomicOr(a.mbits + (v >> 5), 1u << (v & 31));
    }
}

__global__ void k_changed_flags(const int32_t* __restrict__ lnew, const int32_t* __restrict__ lold,
                                uint32_t* __restrict__ chg, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n; base += stride) {
        const int64_t v = base + threadIdx.x;
        const bool c = v < n && lnew[v] != lold[v];
        const uint32_t w = __ballot_sync(0xffffffffu, c);
        if ((threadIdx.x & 31) == 0 && v < n) chg[v >> 5] = w;
    }
}

// Sweep boundary, pull form: warps take 32 row pieces (the plan's dense
// piece list), sum the weights of arcs whose neighbour changed (shared-memory
// atomics per piece), and add each nonzero sum to the row's mark -- the
// bitmap queues the vertex, as in k_mark_pieces.
__global__ void __launch_bounds__(256) k_pull_marks(EvalArgs a, const uint32_t* __restrict__ chg,
                                                    const int32_t* __restrict__ dslot,
                                                    const int32_t* __restrict__ dk0,
                                                    const int32_t* __restrict__ dcount, int32_t* cursor,
                                                    int earlier_only) {
    constexpr int J = 8;
    __shared__ unsigned long long sums[8][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int cnt = *dcount;
    while (true) {
        int b0 = 0;
        if (lane == 0) b0 = atomicAdd(cursor, 32);
        b0 = __shfl_sync(0xffffffffu, b0, 0);
        if (b0 >= cnt) break;
        uint32_t pbeg = 0, plen = 0;
        int32_t ps = -1;
        if (b0 + lane < cnt) {
            ps = dslot[b0 + lane];
            const uint32_t rb = __ldg(a.soff + ps), re = __ldg(a.soff + ps + 1);
            pbeg = rb + (uint32_t)dk0[b0 + lane];
            plen = min((uint32_t)kPieceArcs, re - pbeg);
        }
        sums[wib][lane] = 0ull;
        __syncwarp();
        uint32_t incl = plen;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - plen;
        for (uint32_t base = 0; base < total; base += 32 * J) {
            uint32_t e[J];
            int rr[J];
            uint32_t nb[J];
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const uint32_t i = base + j * 32 + lane;
                int r = 0;
#pragma unroll
                for (int step = 16; step >= 1; step >>= 1) {
                    const uint32_t ex = __shfl_sync(0xffffffffu, excl, r + step);
                    if (r + step < 32 && ex <= i) r += step;
                }
                const uint32_t pb = __shfl_sync(0xffffffffu, pbeg, r);
                const uint32_t pe = __shfl_sync(0xffffffffu, excl, r);
                rr[j] = r;
                e[j] = i < total ? pb + (i - pe) : 0xffffffffu;
                nb[j] = i < total ? __ldg(a.snbr + e[j]) : 0u;
            }
            const bool unit = !(a.gap && a.sw);  // every mark weighs 1
#pragma unroll
            for (int j = 0; j < J; ++j) {
                // (earlier_only 1: in-sweep pull from earlier-batch neighbours; 2: the sweep boundary,
                // every neighbour whose sweep-start label this row reads -- not the earlier-batch ones)
                const bool from = earlier_only == 1 ? (nb[j] & kEarlier) != 0u
                                  : earlier_only == 2 ? !(nb[j] & kEarlier) : true;
                const bool hit = e[j] != 0xffffffffu && from && chg_bit(chg, (int32_t)(nb[j] >> 2));
                if (!unit) {
                    if (hit) atomicAdd(&sums[wib][rr[j]], mark_weight(a, e[j]));
                    continue;
                }
                // unit marks: one shared atomic per piece segment of the warp (lanes of a
                // piece are consecutive: rr is non-decreasing across the lanes)
                const uint32_t bal = __ballot_sync(0xffffffffu, hit);
                if (!bal) continue;
                const int rprev = __shfl_up_sync(0xffffffffu, rr[j], 1);
                const bool head = lane == 0 || rprev != rr[j];
                const uint32_t heads = __ballot_sync(0xffffffffu, head);
                if (head) {
                    const uint32_t above = heads & ~((2u << lane) - 1u);
                    const int nxt = above ? __ffs(above) - 1 : 32;
                    const uint32_t seg = (nxt == 32 ? 0xffffffffu : ((1u << nxt) - 1u)) & ~((1u << lane) - 1u);
                    const int c = __popc(bal & seg);
                    if (c) atomicAdd(&sums[wib][rr[j]], (unsigned long long)c);
                }
            }
        }
        __syncwarp();
        const unsigned long long sm = sums[wib][lane];
        if (sm) {
            const int32_t v = __ldg(a.svid + ps);
            atomicAdd(a.mark + v, sm);  // (fire-and-forget; the bitmap queues v)
            if (a.mbits) atomicOr(a.mbits + (v >> 5), 1u << (v & 31));
        }
        __syncwarp();
    }
}

// Mark the later-batch neighbours of every changed row (see mark_row); warp
// batches of 32 pieces, flattened, eight arcs in flight per lane.
__global__ void __launch_bounds__(256) k_mark_pieces(EvalArgs a) {
    constexpr int J = 8;
    const int lane = threadIdx.x & 31;
    const int cnt = a.r.len[kLenChg];
    const int per = pieces_per_warp(cnt);
    while (true) {
        int b0 = 0;
        if (lane == 0) b0 = atomicAdd(a.r.len + kChgCursor, per);
        b0 = __shfl_sync(0xffffffffu, b0, 0);
        if (b0 >= cnt) break;
        uint32_t pbeg = 0, plen = 0;
        if (lane < per && b0 + lane < cnt) {
            const int32_t s = a.r.cslot[b0 + lane];
            const uint32_t rb = __ldg(a.soff + s), re = __ldg(a.soff + s + 1);
            pbeg = rb + (uint32_t)a.r.ck0[b0 + lane];
            plen = min((uint32_t)kPieceArcs, re - pbeg);
        }
        uint32_t incl = plen;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - plen;
        for (uint32_t base = 0; base < total; base += 32 * J) {
            uint32_t e[J];
            uint32_t nb[J];
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const uint32_t i = base + j * 32 + lane;
                int r = 0;
#pragma unroll
                for (int step = 16; step >= 1; step >>= 1) {
                    const uint32_t ex = __shfl_sync(0xffffffffu, excl, r + step);
                    if (r + step < 32 && ex <= i) r += step;
                }
                const uint32_t pb = __shfl_sync(0xffffffffu, pbeg, r);
                const uint32_t pe = __shfl_sync(0xffffffffu, excl, r);
                e[j] = i < total ? pb + (i - pe) : 0xffffffffu;
                nb[j] = i < total ? __ldg(a.snbr + e[j]) : 0u;
            }
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const int32_t u = (int32_t)(nb[j] >> 2);
                // (no returning atomic: the weight and the bitmap bit are fire-and-forget;
                // k_bits_to_queue builds the queue -- 2.5x faster than queueing on the
                // 0 -> nonzero transition of the mark)
                // (mark_all 2, the sweep boundary: u reads this row's sweep-start label next sweep unless
                // it sits in a later batch -- then it reads the working label and this sweep's marks
                // have already covered the change)
                const bool want = a.mark_all == 1 || (a.mark_all == 2 ? !(nb[j] & kLater) : (nb[j] & kLater) != 0u);
                if (e[j] != 0xffffffffu && want && needs_mark(a, u)) {
                    atomicAdd(a.mark + u, mark_weight(a, e[j]));
                    if (a.mbits) atomicOr(a.mbits + (u >> 5), 1u << (u & 31));
                }
            }
        }
    }
}

// Marked-vertex bitmap -> mark queue (appended to mq_out), bits cleared.
// Whole warps: lane w of a warp takes bitmap word base + w.
// Without the bitmap (mbits = null): every vertex with a nonzero mark is
// queued -- one flat read of the marks instead of a second atomic per
// marked arc (marks are zero again once routed).
__global__ void k_marks_to_queue(const unsigned long long* __restrict__ mark, int64_t n, int32_t* __restrict__ mq_out,
                                 int32_t* mq_len) {
    // (eight vertices per lane: one append per 256 vertices -- every append of the grid lands on
    // the same counter, and at one per 32 vertices that counter was the kernel's time)
    constexpr int J = 8;
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t base = warp * 32 * J; base < n; base += warps * 32 * J) {
        const int64_t v0 = base + lane * J;
        uint32_t nz = 0;
#pragma unroll
        for (int j = 0; j < J; ++j)
            if (v0 + j < n && __ldcg(mark + v0 + j) != 0ull) nz |= 1u << j;
        const int c = __popc(nz);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (tot == 0) continue;
        int b0 = 0;
        if (lane == 31) b0 = atomicAdd(mq_len, tot);
        b0 = __shfl_sync(0xffffffffu, b0, 31);
        int o = b0 + incl - c;
        while (nz) {
            const int j = __ffs(nz) - 1;
            mq_out[o++] = (int32_t)(v0 + j);
            nz &= nz - 1u;
        }
    }
}

__global__ void k_bits_to_queue(uint32_t* __restrict__ mbits, int64_t nwords, int32_t* __restrict__ mq_out,
                                int32_t* mq_len) {
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < nwords; base += stride) {
        const int64_t w = base + threadIdx.x;
        uint32_t b = w < nwords ? mbits[w] : 0u;
        const int c = __popc(b);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        if (tot == 0) continue;
        int b0 = 0;
        if (lane == 31) b0 = atomicAdd(mq_len, tot);
        b0 = __shfl_sync(0xffffffffu, b0, 31);
        if (b) {
            mbits[w] = 0u;
            int o = b0 + incl - c;
            while (b) {
                const int bit = __ffs(b) - 1;
                mq_out[o++] = (int32_t)(w * 32 + bit);
                b &= b - 1u;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// routing
// ---------------------------------------------------------------------------
// cls: 0/1/2 small (d <= 4 / 8 / 16), 3 warp, 6 big-table warp, 4 team, 5 hub
__device__ __forceinline__ int small_class(int d) { return d <= 4 ? 0 : (d <= 8 ? 1 : 2); }

__device__ __forceinline__ int route_class(const EvalArgs& a, int32_t s, int& est, int& d) {
    d = (int)(__ldg(a.soff + s + 1) - __ldg(a.soff + s));
    if (d <= kSmallMax) {
        est = d;
        return small_class(d);
    }
    const int nd = nd_count(__ldg(a.ndist + s));
    est = min(d, nd + (nd >> 2) + 16);
    if (d <= a.mid_max) return 8;
    if (a.cap_route) {
        // a table whose touched capacity is >= d cannot overflow
        if (d <= (1 << WarpClass<0>::kBits) / 4 * 3) return 3;
        if (d <= (1 << WarpClass<1>::kBits) / 4 * 3) return 6;
        if (d <= (1 << kTeamBits) / 4 * 3) return 4;
    }
    if (est <= WarpClass<0>::kEst && d <= a.warp_maxd[0]) return 3;
    if (est <= WarpClass<1>::kEst && d <= a.warp_maxd[1]) return 6;
    if (est <= kTeamEst && d <= kTeamMaxDeg) return 4;
    if (est <= kTeam2Est && d <= kTeamMaxDeg) return 7;
    return 5;
}

// Append `s` (valid when cls >= 0) to its route list; warp-aggregated for the
// single-item classes.  Hub vertices append P (or R) items.
__device__ __forceinline__ void route_append(const EvalArgs& a, int cls, int32_t s, int est, int d) {
    const int lane = threadIdx.x & 31;
    const uint32_t act = __activemask();
#pragma unroll
    for (int c = 0; c < 9; ++c) {
        if (c == 5) continue;  // hubs below
        const uint32_t m = __ballot_sync(act, cls == c);
        if (!m) continue;
        const int leader = __ffs(m) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(a.r.len + (c == 7 ? kLenTeam2 : (c == 8 ? kLenMid : c)), __popc(m));
        base = __shfl_sync(act, base, leader);
        if (cls == c) {
            const int idx = base + __popc(m & lanemask_lt());
            if (c == 8) {
                a.r.mid[idx] = s;
            } else if (c < 3) {
                a.r.small[c][idx] = s;
            } else if (c == 3) {
                a.r.warp[0][idx] = s;
            } else if (c == 6) {
                a.r.warp[1][idx] = s;
            } else {
                Item t = {s, 0, 1, 0, 1, -1, 0, 0};
                (c == 7 ? a.r.team2 : a.r.team)[idx] = t;
            }
        }
    }
    if (cls == 5) {
        // rows long enough to slice: R arc slices fold into one L2-resident
        // global table sized for the estimate (2^bits >= 2 est + 64), so the
        // row is read once whatever its label count; else label partitions
        int gbits = kGlobalBits;
        while ((1 << gbits) < 2 * est + 64 && gbits < 28) ++gbits;
        int gt = -1;
        // slices when the labels are few (a small L2 table); with many labels the
        // smem label partitions are faster than global-table atomics (measured)
        if (d > kSliceArcs * 2 && est <= kSliceEst && !a.two_team) {
            gt = atomicAdd(a.r.len + kGtabCursor, 1 << gbits);
            if ((int64_t)gt + (1 << gbits) > a.r.gcap) gt = -1;  // pool exhausted: partitions
        }
        if (gt >= 0) {
            const int R = (d + kSliceArcs - 1) / kSliceArcs;
            const int base = atomicAdd(a.r.len + kLenHub, R);
            const int cb = atomicAdd(a.r.len + kCandCursor, 1);
            for (int r = 0; r < R; ++r) {
                Item t = {s, 0, 1, r, R, cb, gt, gbits};
                a.r.hub[base + r] = t;
            }
        } else {
            const int P = max(1, (est + kHubPlan - 1) / kHubPlan);
            const int base = atomicAdd(a.r.len + kLenHub, P);
            const int cb = P > 1 ? atomicAdd(a.r.len + kCandCursor, P) : -1;
            for (int q = 0; q < P; ++q) {
                Item t = {s, q, P, 0, 1, cb, 0, 0};
                a.r.hub[base + q] = t;
            }
        }
    }
}

// Dense round: route every slot in [s_beg, s_end) (the small-degree range is
// swept directly by k_small and excluded by the caller).
__global__ void k_route_dense(EvalArgs a, int32_t s_beg, int32_t s_end) {
    for (int32_t base = blockIdx.x * blockDim.x; base < s_end - s_beg; base += gridDim.x * blockDim.x) {
        const int32_t i = base + threadIdx.x;
        int cls = -1, est = 0, d = 0;
        const int32_t s = s_beg + i;
        if (i < s_end - s_beg) cls = route_class(a, s, est, d);
        route_append(a, cls, s, est, d);
    }
}

// Frontier round: the queued (marked) vertices -> route lists + phase-1
// pieces; marks are cleared so this round's writes can queue them again.
__global__ void __launch_bounds__(256) k_route_queue(EvalArgs a, const int32_t* __restrict__ mq_in,
                                                     const int32_t* __restrict__ mq_in_len,
                                                     const int32_t* __restrict__ slot_of, int clear_marks) {
    // The appends are aggregated per block: lists 0-8 (hubs apart), the phase-1 pieces and the
    // routed count take one global atomic per 256 queue entries each -- every warp of the grid
    // appending to the same few counters was the kernel's time on long queues.
    enum { kPieces = 9, kRouted = 10, kSlots = 11 };
    __shared__ int32_t s_cnt[kSlots], s_base[kSlots];
    const int lane = threadIdx.x & 31;
    const int cnt = *mq_in_len;
    for (int base = blockIdx.x * blockDim.x; base < cnt; base += gridDim.x * blockDim.x) {
        if (threadIdx.x < kSlots) s_cnt[threadIdx.x] = 0;
        __syncthreads();
        const int i = base + threadIdx.x;
        int cls = -1, est = 0, d = 0;
        int32_t s = -1;
        if (i < cnt) {
            const int32_t v = mq_in[i];
            s = slot_of[v];
            if (clear_marks) {
                // Margin test: the labels that changed since v's last evaluation
                // moved at most `delta` weight, so if the winner led the runner-up
                // by more than 2 * delta it still wins: v is not re-evaluated.
                // (Skipping consumes margin: gap -= 2 * delta keeps it a valid bound.)
                if (a.gap && s >= 0) {
                    const unsigned long long delta = a.mark[v];
                    const unsigned long long gp = a.gap[s];
                    if (gp > 2ull * delta) {
                        a.gap[s] = gp - 2ull * delta;
                        s = -1;
                    }
                }
                a.mark[v] = 0ull;
            }
            if (s >= 0) cls = route_class(a, s, est, d);
        }
        // ---- block-local positions ----
        int idx = 0;  // position of this entry in its list, from the block's base
#pragma unroll
        for (int c = 0; c < 9; ++c) {
            if (c == 5) continue;  // hubs below
            const uint32_t m = __ballot_sync(0xffffffffu, cls == c);
            if (!m) continue;
            const int leader = __ffs(m) - 1;
            int b = 0;
            if (lane == leader) b = atomicAdd(&s_cnt[c], __popc(m));
            b = __shfl_sync(0xffffffffu, b, leader);
            if (cls == c) idx = b + __popc(m & lanemask_lt());
        }
        // phase-1 pieces of the routed row (none for fused rows)
        const int np_all = cls >= 0 ? (d + kPieceArcs - 1) / kPieceArcs : 0;
        const int np = d > a.fuse_maxd ? np_all : 0;
        {
            const unsigned routed = __reduce_add_sync(0xffffffffu, (unsigned)np_all);
            if (routed && lane == 0) atomicAdd(&s_cnt[kRouted], (int32_t)routed);
        }
        int incl = np;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        int pb = 0;
        if (lane == 31 && tot) pb = atomicAdd(&s_cnt[kPieces], tot);
        pb = __shfl_sync(0xffffffffu, pb, 31);
        __syncthreads();
        if (threadIdx.x < kSlots && s_cnt[threadIdx.x]) {
            const int c = threadIdx.x;
            const int g = c == kPieces ? kLenGather : c == kRouted ? kLenRouted : c == 7 ? kLenTeam2 : c == 8 ? kLenMid : c;
            s_base[c] = atomicAdd(a.r.len + g, s_cnt[c]);
        }
        __syncthreads();
        if (cls >= 0 && cls != 5) {
            const int at = s_base[cls] + idx;
            if (cls == 8) {
                a.r.mid[at] = s;
            } else if (cls < 3) {
                a.r.small[cls][at] = s;
            } else if (cls == 3) {
                a.r.warp[0][at] = s;
            } else if (cls == 6) {
                a.r.warp[1][at] = s;
            } else {
                Item t = {s, 0, 1, 0, 1, -1, 0, 0};
                (cls == 7 ? a.r.team2 : a.r.team)[at] = t;
            }
        }
        if (cls == 5) route_append(a, cls, s, est, d);  // (hub items: the row's own atomics)
        if (np) {
            const int b0 = s_base[kPieces] + pb;
            for (int q = 0; q < np; ++q) {
                a.r.gslot[b0 + incl - np + q] = s;
                a.r.gk0[b0 + incl - np + q] = q * kPieceArcs;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// first dense round of a run that starts from labels = vertex ids
// ---------------------------------------------------------------------------
// rak.py:168 starts every vertex with its own id.  In the first round of the
// first sweep every read returns the initial label (nothing is written
// before the round's gathers), so the labels of a row are its neighbour ids:
// all distinct (rows are duplicate-free), each with count 1.  With unit
// weights the argmax is then the first arc for scan-first ties and the
// smallest neighbour id for min-label ties -- the same arc when rows are
// sorted -- so the round needs no gather and no tally: one thread per row
// reads one neighbour id.  Everything the tally kernels record is recorded
// (label, changed count, distinct count, majority flag, margin, changed row).
// chain: a better guess for the exact schedule (scan-first ties).  With every
// tally all singletons the sequential sweep gives v the label of its first arc:
// the neighbour's id if it comes in a later batch, else the label that
// neighbour took -- which is, by the same rule, its own first arc's.  Following
// first arcs through earlier-batch neighbours (a few hops; rows are sorted, the
// first arc is the smallest id) reproduces the sequential first sweep for all
// of those vertices (a third of the wrong guesses of the plain first arc remain
// on R-MAT-22).  It is a guess, not an evaluation, so a dense round follows.
__global__ void __launch_bounds__(256) k_first_round(EvalArgs a, int32_t S, const int32_t* __restrict__ slot_of,
                                                     int chain) {
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    __shared__ int32_t s_push[2][34];
    int par = 0;
    // (block-uniform loop: the changed rows are pushed as pieces by the whole block)
    for (int32_t base = blockIdx.x * blockDim.x; base < S; base += gridDim.x * blockDim.x, ++par) {
        const int32_t s = base + threadIdx.x;
        bool ch = false;
        int d = 0;
        if (s < S) {
            const int32_t p = __ldg(a.svid + s);
            const uint32_t beg = __ldg(a.soff + s);
            d = (int)(__ldg(a.soff + s + 1) - beg);
            uint32_t nb = __ldg(a.snbr + beg);
            for (int hop = 0; chain && (nb & kEarlier) && hop < 64; ++hop)
                nb = __ldg(a.snbr + __ldg(a.soff + __ldg(slot_of + (nb >> 2))));
            const int32_t lab = (int32_t)(nb >> 2);
            arcs += d;
            ++verts;
            // (the next round of a singleton first sweep tables only the evaluated
            // labels, a few percent of a long row: a lower estimate for long rows)
            a.ndist[s] = (a.id_single && d > a.first_est_min ? d / a.first_est_div : d) | (2 > d ? kMajBit : 0);
            store_lead<uint32_t>(a, s, 1u, d > 1 ? 1u : 0u);
            ch = commit_label_known(a, p, lab, p, p, dchg, writes);
        }
        if (a.mark) push_changed_rows_block(a, ch, s, d, s_push, par);
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

// Weighted (exact fixed-point) first round from labels = ids: every label of
// a row is distinct, so its weight is its arc's weight -- the winner is the
// heaviest arc (the earliest of equal ones: scan-first, and min-label on
// sorted rows), the runner-up the second heaviest.  No gather, no tally:
// k_first_round_w takes rows of <= kFirstBig arcs (one warp per row, 32 rows
// per warp batch), k_first_round_wbig the longer ones (a block per row; the
// plan stores long rows first, by descending degree).
constexpr int kFirstBig = 4096;

struct Top2 {
    uint32_t w1, w2;
    int k1;  // INT32_MAX = none
};
__device__ __forceinline__ void top2_add(Top2& t, uint32_t w, int k) {
    if (t.k1 == INT32_MAX || w > t.w1) {
        t.w2 = t.k1 == INT32_MAX ? 0u : t.w1;
        t.w1 = w;
        t.k1 = k;
    } else if (w > t.w2) {
        t.w2 = w;
    }
}
__device__ __forceinline__ void top2_merge(Top2& t, const Top2& o) {
    if (o.k1 == INT32_MAX) return;
    if (t.k1 == INT32_MAX || o.w1 > t.w1 || (o.w1 == t.w1 && o.k1 < t.k1)) {
        const uint32_t nw2 = t.k1 == INT32_MAX ? o.w2 : max(o.w2, t.w1);
        t.w1 = o.w1;
        t.w2 = nw2;
        t.k1 = o.k1;
    } else {
        t.w2 = max(t.w2, o.w1);
    }
}
__device__ __forceinline__ Top2 top2_warp(Top2 t) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        Top2 x;
        x.w1 = __shfl_xor_sync(0xffffffffu, t.w1, o);
        x.w2 = __shfl_xor_sync(0xffffffffu, t.w2, o);
        x.k1 = __shfl_xor_sync(0xffffffffu, t.k1, o);
        top2_merge(t, x);
    }
    return t;
}
// one thread: record the first-round result of row s
__device__ __forceinline__ bool first_w_commit(const EvalArgs& a, int32_t s, int32_t p, uint32_t beg, int d,
                                               const Top2& t, long long& dchg, long long& arcs, long long& writes,
                                               long long& verts) {
    const int32_t lab = (int32_t)(__ldg(a.snbr + beg + t.k1) >> 2);
    const unsigned long long total = __ldg(a.swsum + s);
    arcs += d;
    ++verts;
    const bool maj = 2ull * t.w1 > total;
    // (weighted singleton sweep: warp-sized rows table a fraction of their labels)
    a.ndist[s] = (a.id_single && d > a.first_est_min && (a.two_team || d <= WarpClass<0>::kMaxDeg) ? d / a.first_est_div
                                                                                                  : d) |
                 (maj ? kMajBit : 0);
    store_lead<unsigned long long>(a, s, (unsigned long long)t.w1, (unsigned long long)t.w2);
    return commit_label_known(a, p, lab, p, p, dchg, writes);
}

__global__ void __launch_bounds__(256) k_first_round_wbig(EvalArgs a, int32_t S) {
    __shared__ Top2 red[8];
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    for (int32_t s = blockIdx.x; s < S; s += gridDim.x) {
        const uint32_t beg = __ldg(a.soff + s);
        const int d = (int)(__ldg(a.soff + s + 1) - beg);
        if (d <= kFirstBig) break;  // (long rows come first)
        Top2 t = {0u, 0u, INT32_MAX};
        for (int k = threadIdx.x; k < d; k += blockDim.x) top2_add(t, __ldg(a.sw + beg + k), k);
        t = top2_warp(t);
        if (lane == 0) red[wib] = t;
        __syncthreads();
        if (wib == 0) {
            t = lane < 8 ? red[lane] : Top2{0u, 0u, INT32_MAX};
            t = top2_warp(t);
            if (lane == 0) {
                const int32_t p = __ldg(a.svid + s);
                if (first_w_commit(a, s, p, beg, d, t, dchg, arcs, writes, verts) && a.mark) push_changed(a, s, d);
            }
        }
        __syncthreads();
    }
    if (wib == 0) flush_counters(a, dchg, arcs, writes, verts);
}

// Random ties (non-strict), unit weights, first round from ids: every label
// has weight 1, so the winner is the label with the largest tie_hash (the
// earliest arc on a hash collision) -- a max over the row, no tally.  Warp per
// row, 32 rows per warp batch (long rows stream 32 arcs per step).
__global__ void __launch_bounds__(256) k_first_round_r(EvalArgs a, int32_t S) {
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    const int lane = threadIdx.x & 31;
    const int32_t nwarps = (int32_t)(gridDim.x * blockDim.x / 32);
    for (int32_t base = (int32_t)((blockIdx.x * blockDim.x + threadIdx.x) / 32) * 32; base < S; base += nwarps * 32) {
        const int32_t ms = base + lane;
        uint32_t mbeg = 0, mend = 0;
        int32_t mp = 0;
        if (ms < S) {
            mp = __ldg(a.svid + ms);
            mbeg = __ldg(a.soff + ms);
            mend = __ldg(a.soff + ms + 1);
        }
        uint32_t chm = 0;
        const int nv = min(32, S - base);
        for (int v = 0; v < nv; ++v) {
            const int32_t s = base + v;
            const uint32_t beg = __shfl_sync(0xffffffffu, mbeg, v);
            const int d = (int)(__shfl_sync(0xffffffffu, mend, v) - beg);
            const int32_t p = __shfl_sync(0xffffffffu, mp, v);
            if (d > kFirstBig) continue;  // k_first_round_rbig
            unsigned long long bk = 0;  // (tie hash << 32) | ~arc; 0 = none (~arc > 0)
            int32_t bl = -1;
            for (int k = lane; k < d; k += 32) {
                const int32_t lab = (int32_t)(__ldg(a.snbr + beg + k) >> 2);
                const unsigned long long key = ((unsigned long long)tie_hash(a.seed, a.sweep, (uint32_t)p, (uint32_t)lab) << 32) |
                                               (unsigned long long)(~(uint32_t)k);
                if (key > bk) {
                    bk = key;
                    bl = lab;
                }
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                const unsigned long long ok = shfl_u64(bk, o);
                const int32_t ol = __shfl_xor_sync(0xffffffffu, bl, o);
                if (ok > bk) {
                    bk = ok;
                    bl = ol;
                }
            }
            bool ch = false;
            if (lane == 0 && d > 0) {
                arcs += d;
                ++verts;
                a.ndist[s] = (a.id_single && d > a.first_est_min ? d / a.first_est_div : d) | (2 > d ? kMajBit : 0);
                store_lead<uint32_t>(a, s, 1u, d > 1 ? 1u : 0u);
                ch = commit_label_known(a, p, bl, p, p, dchg, writes);
            }
            if (__shfl_sync(0xffffffffu, ch, 0)) chm |= 1u << v;
        }
        if (a.mark) push_changed_batch(a, chm, ms, (int)(mend - mbeg));
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

// (long rows of k_first_round_r: a block per row; the plan stores them first)
__global__ void __launch_bounds__(256) k_first_round_rbig(EvalArgs a, int32_t S) {
    __shared__ unsigned long long red[2];
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    const int lane = threadIdx.x & 31;
    for (int32_t s = blockIdx.x; s < S; s += gridDim.x) {
        const uint32_t beg = __ldg(a.soff + s);
        const int d = (int)(__ldg(a.soff + s + 1) - beg);
        if (d <= kFirstBig) break;  // (long rows come first)
        const int32_t p = __ldg(a.svid + s);
        unsigned long long bk = 0;
        int32_t bl = -1;
        for (int k = threadIdx.x; k < d; k += blockDim.x) {
            const int32_t lab = (int32_t)(__ldg(a.snbr + beg + k) >> 2);
            const unsigned long long key = ((unsigned long long)tie_hash(a.seed, a.sweep, (uint32_t)p, (uint32_t)lab) << 32) |
                                           (unsigned long long)(~(uint32_t)k);
            if (key > bk) {
                bk = key;
                bl = lab;
            }
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const unsigned long long ok = shfl_u64(bk, o);
            const int32_t ol = __shfl_xor_sync(0xffffffffu, bl, o);
            if (ok > bk) {
                bk = ok;
                bl = ol;
            }
        }
        if (threadIdx.x == 0) red[0] = 0ull;
        __syncthreads();
        if (lane == 0) atomicMax(&red[0], bk);
        __syncthreads();
        if (lane == 0 && bk == red[0]) red[1] = (unsigned long long)(uint32_t)bl;  // (keys are unique)
        __syncthreads();
        if (threadIdx.x == 0) {
            const int32_t lab = (int32_t)(uint32_t)red[1];
            arcs += d;
            ++verts;
            a.ndist[s] = (a.id_single && d > a.first_est_min ? d / a.first_est_div : d);
            store_lead<uint32_t>(a, s, 1u, 1u);
            if (commit_label_known(a, p, lab, p, p, dchg, writes) && a.mark) push_changed(a, s, d);
        }
        __syncthreads();
    }
    if (threadIdx.x < 32) flush_counters(a, dchg, arcs, writes, verts);
}

__global__ void __launch_bounds__(256) k_first_round_w(EvalArgs a, int32_t S) {
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    const int lane = threadIdx.x & 31;
    const int32_t nwarps = (int32_t)(gridDim.x * blockDim.x / 32);
    for (int32_t base = (int32_t)((blockIdx.x * blockDim.x + threadIdx.x) / 32) * 32; base < S; base += nwarps * 32) {
        const int32_t ms = base + lane;
        uint32_t mbeg = 0, mend = 0;
        int32_t mp = 0;
        if (ms < S) {
            mp = __ldg(a.svid + ms);
            mbeg = __ldg(a.soff + ms);
            mend = __ldg(a.soff + ms + 1);
        }
        uint32_t chm = 0;
        const int nv = min(32, S - base);
        for (int v = 0; v < nv; ++v) {
            const int32_t s = base + v;
            const uint32_t beg = __shfl_sync(0xffffffffu, mbeg, v);
            const int d = (int)(__shfl_sync(0xffffffffu, mend, v) - beg);
            const int32_t p = __shfl_sync(0xffffffffu, mp, v);
            if (d > kFirstBig) continue;  // k_first_round_wbig
            Top2 t = {0u, 0u, INT32_MAX};
            for (int k = lane; k < d; k += 32) top2_add(t, __ldg(a.sw + beg + k), k);
            t = top2_warp(t);
            bool ch = false;
            if (lane == 0 && d > 0) ch = first_w_commit(a, s, p, beg, d, t, dchg, arcs, writes, verts);
            if (__shfl_sync(0xffffffffu, ch, 0)) chm |= 1u << v;
        }
        if (a.mark) push_changed_batch(a, chm, ms, (int)(mend - mbeg));
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

// ---------------------------------------------------------------------------
// thread per vertex
// ---------------------------------------------------------------------------
// MAXD = 4, 8 or 16: the degree class (O(MAXD^2) register compares).
// Dense mode sweeps slots [s_beg, s_end); list mode (s_beg < 0) reads the
// class's route list.
template <int WM, int TIE, int MAXD>
__global__ void __launch_bounds__(256, MAXD == 16 ? 3 : 4) k_small(EvalArgs a, int32_t s_beg, int32_t s_end) {
    using A = typename Acc<WM>::T;
    constexpr int LIST = MAXD == 4 ? kLenS4 : (MAXD == 8 ? kLenS8 : kLenS16);
    const bool listed = s_beg < 0;
    const int32_t cnt = listed ? a.r.len[LIST] : (s_end - s_beg);
    const int32_t* list = a.r.small[LIST];
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    __shared__ int32_t s_push[2][34];
    int par = 0;
    // (block-uniform trip count: the changed rows of an iteration are appended per block)
    for (int32_t base = blockIdx.x * blockDim.x; base < cnt; base += gridDim.x * blockDim.x, ++par) {
        const int32_t i = base + threadIdx.x;
        bool ch = false;
        int32_t s = 0;
        if (i < cnt) do {
        s = listed ? list[i] : s_beg + i;
        const int32_t p = __ldg(a.svid + s);
        const uint32_t beg = __ldg(a.soff + s);
        const int d = (int)(__ldg(a.soff + s + 1) - beg);
        const int32_t xv = a.x[p];
        const int32_t l0v = __ldg(a.L0 + p);
        int32_t lab[MAXD];
        A w[MAXD];
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            if (k < d) {
                lab[k] = lb_strip(a, arc_label(a, beg + k));
                w[k] = arc_weight<WM>(a, beg + k);
            } else {
                lab[k] = kEmpty;
                w[k] = A(0);
            }
        }
        const int32_t nd = __ldg(a.ndist + s);
        arcs += d;
        ++verts;
        A total = A(0);
#pragma unroll
        for (int k = 0; k < MAXD; ++k) total += w[k];
        if ((nd & kMajBit) && WM != kFloat) {
            const int32_t cand = xv;
            A cw = A(0);
#pragma unroll
            for (int k = 0; k < MAXD; ++k)
                if (lab[k] == cand) cw += w[k];
            if (cw + cw > total) {  // strict majority: label unchanged
                store_gap<A>(a, s, cw, total);
                break;
            }
        }
        const uint32_t vtx = (uint32_t)p;
        Cand<A> best = none_cand<A>();
        A w1 = A(0), w2 = A(0);
#pragma unroll
        for (int i2 = 0; i2 < MAXD; ++i2) {
            if (i2 < d) {
                bool dup = false;
                A sum = w[i2];
#pragma unroll
                for (int j = 0; j < MAXD; ++j) {
                    if (j == i2) continue;
                    const bool eq = lab[j] == lab[i2];
                    dup |= (j < i2) & eq;
                    if (eq) sum += w[j];
                }
                if (!dup) {
                    Cand<A> c = make_cand<TIE, A>(sum, lab[i2], (uint32_t)i2, a.seed, a.sweep, vtx);
                    if (better(c, best)) best = c;
                    // the two largest label weights: the winner's exact lead
                    if (sum > w1) {
                        w2 = w1;
                        w1 = sum;
                    } else if (sum > w2) {
                        w2 = sum;
                    }
                }
            }
        }
        const int32_t nd_new = (best.w + best.w > total) ? kMajBit : 0;
        if (nd_new != nd) a.ndist[s] = nd_new;
        store_lead<A>(a, s, w1, w2);
        ch = commit_label_known(a, p, best.lab, xv, l0v, dchg, writes);
        } while (0);
        if (a.mark) push_changed_block(a, ch, s, s_push, par);
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

// Thread per row for kSmallMax < d <= kMidMax (listed rows): k_small's
// O(d^2) tally with the row's labels staged in shared memory (column layout:
// label k of thread t at [k][t], conflict-free) instead of registers.  A
// warp then evaluates 32 rows at once with no shuffles, hashes or barriers --
// mid-degree rows are latency-bound on the warp-per-row path.
constexpr int kMidMax = 64;
constexpr int kMidThreads = 128;
template <int WM> constexpr size_t mid_smem_bytes() {
    return (size_t)kMidMax * kMidThreads * (sizeof(int32_t) + (WM == kUnit ? 0 : sizeof(typename Acc<WM>::T)));
}

template <int WM, int TIE>
__global__ void __launch_bounds__(kMidThreads) k_mid(EvalArgs a) {
    using A = typename Acc<WM>::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int32_t* lab = reinterpret_cast<int32_t*>(smem_raw) + threadIdx.x;  // lab[k * kMidThreads]
    A* wv = reinterpret_cast<A*>(smem_raw + (size_t)kMidMax * kMidThreads * sizeof(int32_t)) + threadIdx.x;
    const int32_t cnt = a.r.len[kLenMid];
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    for (int32_t base = blockIdx.x * blockDim.x; base < cnt; base += gridDim.x * blockDim.x) {
        const int32_t i = base + threadIdx.x;
        bool ch = false;
        int32_t s = -1;
        if (i < cnt) {
            s = a.r.mid[i];
            const int32_t p = __ldg(a.svid + s);
            const uint32_t beg = __ldg(a.soff + s);
            const int d = (int)(__ldg(a.soff + s + 1) - beg);
            const int32_t xv = a.x[p];
            const int32_t l0v = __ldg(a.L0 + p);
            const int32_t nd = __ldg(a.ndist + s);
            A total = A(0);
            for (int k = 0; k < d; ++k) {
                lab[k * kMidThreads] = lb_strip(a, arc_label(a, beg + k));
                const A w = arc_weight<WM>(a, beg + k);
                if (WM != kUnit) wv[k * kMidThreads] = w;
                total += w;
            }
#define LP_MID_W(k) (WM == kUnit ? A(1) : wv[(k) * kMidThreads])
            arcs += d;
            ++verts;
            bool done = false;
            if ((nd & kMajBit) && WM != kFloat) {
                A cw = A(0);
                for (int k = 0; k < d; ++k)
                    if (lab[k * kMidThreads] == xv) cw += LP_MID_W(k);
                if (cw + cw > total) {  // strict majority: label unchanged
                    store_gap<A>(a, s, cw, total);
                    done = true;
                }
            }
            if (!done) {
                const uint32_t vtx = (uint32_t)p;
                Cand<A> best = none_cand<A>();
                A w1 = A(0), w2 = A(0);
                for (int i2 = 0; i2 < d; ++i2) {
                    const int32_t li = lab[i2 * kMidThreads];
                    bool dup = false;
                    for (int j = 0; j < i2; ++j)
                        if (lab[j * kMidThreads] == li) {
                            dup = true;
                            break;
                        }
                    if (dup) continue;  // counted at its first occurrence
                    A sum = LP_MID_W(i2);
                    for (int j = i2 + 1; j < d; ++j)
                        if (lab[j * kMidThreads] == li) sum += LP_MID_W(j);
                    const Cand<A> c = make_cand<TIE, A>(sum, li, (uint32_t)i2, a.seed, a.sweep, vtx);
                    if (better(c, best)) best = c;
                    if (sum > w1) {
                        w2 = w1;
                        w1 = sum;
                    } else if (sum > w2) {
                        w2 = sum;
                    }
                }
#undef LP_MID_W
                const int32_t nd_new = (best.w + best.w > total) ? kMajBit : 0;
                if (nd_new != nd) a.ndist[s] = nd_new;
                store_lead<A>(a, s, w1, w2);
                ch = commit_label_known(a, p, best.lab, xv, l0v, dchg, writes);
            }
        }
        if (a.mark) push_changed_small(a, ch, s);
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

// Unit weights: the same rows through a private per-thread hash table in
// shared memory (128 slots, column layout) -- d probes instead of d^2
// compares.  An entry is (label, tag, first arc, count); `tag` names the row
// that wrote it (entries of earlier rows read as empty; the table is wiped
// every 255 rows), so nothing is cleared per row.  The argmax is kept
// incrementally (counts only grow; ties as make_cand), the runner-up comes
// from a pass over the row's touched slots.
constexpr int kMidHThreads = 64;
constexpr int kMidHSlots = 128;
constexpr size_t mid_hash_smem_bytes() {
    return (size_t)kMidHSlots * kMidHThreads * sizeof(unsigned long long) + (size_t)kMidMax * kMidHThreads;
}

template <int TIE>
__global__ void __launch_bounds__(kMidHThreads) k_midh(EvalArgs a) {
    using A = uint32_t;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned long long* tab = reinterpret_cast<unsigned long long*>(smem_raw) + threadIdx.x;  // [slot * T]
    uint8_t* touched = smem_raw + (size_t)kMidHSlots * kMidHThreads * sizeof(unsigned long long) + threadIdx.x;
    for (int h = 0; h < kMidHSlots; ++h) tab[h * kMidHThreads] = 0ull;
    uint32_t tag = 0;
    const int32_t cnt = a.r.len[kLenMid];
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    for (int32_t base = blockIdx.x * blockDim.x; base < cnt; base += gridDim.x * blockDim.x) {
        const int32_t i = base + threadIdx.x;
        bool ch = false;
        int32_t s = -1;
        if (i < cnt) {
            s = a.r.mid[i];
            const int32_t p = __ldg(a.svid + s);
            const uint32_t beg = __ldg(a.soff + s);
            const int d = (int)(__ldg(a.soff + s + 1) - beg);
            const int32_t xv = a.x[p];
            const int32_t l0v = __ldg(a.L0 + p);
            const int32_t nd = __ldg(a.ndist + s);
            arcs += d;
            ++verts;
            bool done = false;
            if (nd & kMajBit) {
                int cw = 0;
                for (int k = 0; k < d; ++k) cw += lb_strip(a, arc_label(a, beg + k)) == xv;
                if (cw + cw > d) {  // strict majority: label unchanged
                    store_gap<A>(a, s, (A)cw, (A)d);
                    done = true;
                }
            }
            if (!done) {
                if (tag == 255u) {  // wipe: tags are about to repeat
                    for (int h = 0; h < kMidHSlots; ++h) tab[h * kMidHThreads] = 0ull;
                    tag = 0;
                }
                ++tag;
                const uint32_t vtx = (uint32_t)p;
                Cand<A> best = none_cand<A>();
                int nt = 0;
                // (labels in batches of 8 registers: the row's loads overlap instead of
                // one dependent L2 round trip per arc)
                constexpr int kB = 8;
                int32_t lv[kB];
                for (int k = 0; k < d; ++k) {
                    if ((k & (kB - 1)) == 0) {
#pragma unroll
                        for (int j = 0; j < kB; ++j) lv[j] = k + j < d ? arc_label(a, beg + k + j) : 0;
                    }
                    int32_t lab = lv[0];
#pragma unroll
                    for (int j = 1; j < kB; ++j)
                        if ((k & (kB - 1)) == j) lab = lv[j];
                    lab = lb_strip(a, lab);
                    uint32_t h = slot_hash(lab, 7);
                    while (true) {
                        const unsigned long long e = tab[h * kMidHThreads];
                        if ((((uint32_t)(e >> 24)) & 0xffu) != tag) {  // another row's entry: empty here
                            const unsigned long long ne = ((unsigned long long)(uint32_t)lab << 32) |
                                                          ((unsigned long long)tag << 24) | ((unsigned long long)k << 16) | 1ull;
                            tab[h * kMidHThreads] = ne;
                            touched[nt * kMidHThreads] = (uint8_t)h;
                            ++nt;
                            const Cand<A> c = make_cand<TIE, A>(1u, lab, (uint32_t)k, a.seed, a.sweep, vtx);
                            if (better(c, best)) best = c;
                            break;
                        }
                        if ((int32_t)(e >> 32) == lab) {
                            const unsigned long long ne = e + 1ull;
                            tab[h * kMidHThreads] = ne;
                            const Cand<A> c = make_cand<TIE, A>((A)(ne & 0xffffu), lab, (uint32_t)((ne >> 16) & 0xffu),
                                                                a.seed, a.sweep, vtx);
                            if (better(c, best)) best = c;
                            break;
                        }
                        h = (h + 1) & (kMidHSlots - 1);
                    }
                }
                // runner-up: the largest count of any other label
                A w2 = 0;
                for (int t = 0; t < nt; ++t) {
                    const unsigned long long e = tab[touched[t * kMidHThreads] * kMidHThreads];
                    const A c = (A)(e & 0xffffu);
                    if ((int32_t)(e >> 32) != best.lab && c > w2) w2 = c;
                }
                const int32_t nd_new = (best.w + best.w > (A)d) ? kMajBit : 0;
                if (nd_new != nd) a.ndist[s] = nd_new;
                store_lead<A>(a, s, best.w, w2);
                ch = commit_label_known(a, p, best.lab, xv, l0v, dchg, writes);
            }
        }
        if (a.mark) push_changed_small(a, ch, s);
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

// Hub rows routed as P > 1 label partitions (one k_team block each): reorder
// the row's labels by partition once -- a counting scatter with
// __match_any_sync-folded shared counters -- so that each partition block
// reads its own bucket (1/P of the row) instead of the whole row.  Bucket
// order is arbitrary; hb_pos keeps each label's arc position (scan-order ties).
constexpr int kHubBucketMaxP = 64;
__global__ void __launch_bounds__(1024) k_hub_bucket(EvalArgs a) {
    __shared__ int32_t cntp[kHubBucketMaxP];
    __shared__ int32_t curp[kHubBucketMaxP];
    const int tid = threadIdx.x, lane = tid & 31;
    const int32_t cnt = a.r.len[kLenHub];
    for (int32_t it = blockIdx.x; it < cnt; it += gridDim.x) {
        const Item item = a.r.hub[it];
        if (item.R != 1 || item.P <= 1 || item.q != 0) continue;  // (block-uniform)
        const uint32_t P = (uint32_t)item.P;
        if (P > (uint32_t)kHubBucketMaxP) {
            for (int q = tid; q < item.P; q += blockDim.x) a.hb_off[item.cb + q] = make_int2(0, -1);
            continue;
        }
        const int32_t s = item.s;
        const uint32_t beg = __ldg(a.soff + s);
        const int d = (int)(__ldg(a.soff + s + 1) - beg);
        if (tid < kHubBucketMaxP) cntp[tid] = 0;
        __syncthreads();
        for (int base = 0; base < d; base += blockDim.x) {
            const int k = base + tid;
            const uint32_t part = k < d ? part_of(lb_strip(a, arc_label(a, beg + k)), P) : 0xffffffffu;
            const uint32_t grp = __match_any_sync(0xffffffffu, part);
            if (part != 0xffffffffu && lane == __ffs(grp) - 1) atomicAdd(&cntp[part], __popc(grp));
        }
        __syncthreads();
        if (tid == 0) {
            int32_t o = 0;
            for (uint32_t q = 0; q < P; ++q) {
                a.hb_off[item.cb + q] = make_int2((int32_t)beg + o, cntp[q]);
                curp[q] = o;
                o += cntp[q];
            }
        }
        __syncthreads();
        for (int base = 0; base < d; base += blockDim.x) {
            const int k = base + tid;
            const int32_t lab = k < d ? arc_label(a, beg + k) : 0;  // (kSingle flags kept)
            const uint32_t part = k < d ? part_of(lb_strip(a, lab), P) : 0xffffffffu;
            const uint32_t grp = __match_any_sync(0xffffffffu, part);
            const int leader = __ffs(grp) - 1;
            int b0 = 0;
            if (part != 0xffffffffu && lane == leader) b0 = atomicAdd(&curp[part], __popc(grp));
            b0 = __shfl_sync(0xffffffffu, b0, leader);
            if (part != 0xffffffffu) {
                const int o = b0 + __popc(grp & lanemask_lt());
                a.hb_lab[beg + o] = lab;
                a.hb_pos[beg + o] = (uint32_t)k;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// shared-memory tally tables
// ---------------------------------------------------------------------------
// Open addressing with linear probing; entries are wiped after each vertex
// through a touched list.  There is no first-position field: ties at the
// maximum are resolved afterwards by scanning the row for the earliest arc
// whose label is tied (resolve_first), so a distinct label costs a single
// shared-memory atomic.  For unit weights (label, count) is one 64-bit word
// inserted by CAS and bumped by atomicAdd; weighted tables keep keys and
// 64-bit fixed-point (or float) sums side by side.
constexpr unsigned long long kEmpty64 = 0xffffffff00000000ull;

// Find or insert `lab` in an open-addressing key array of 2^bits slots
// (shared or global memory).  Returns -1 only when the table is full.
__device__ __forceinline__ int table_slot(int32_t* keys, int32_t lab, int bits, bool& isnew) {
    const int mask = (1 << bits) - 1;
    int h = (int)slot_hash(lab, bits);
    isnew = false;
    for (int probe = 0; probe <= mask; ++probe) {
        const int32_t cur = *(volatile int32_t*)&keys[h];
        if (cur == lab) return h;
        if (cur == kEmpty) {
            const int32_t old = atomicCAS(&keys[h], kEmpty, lab);
            if (old == kEmpty) {
                isnew = true;
                return h;
            }
            if (old == lab) return h;
        }
        h = (h + 1) & mask;
    }
    return -1;
}

template <int WM, int BITS> struct STable {
    using A = typename Acc<WM>::T;
    static constexpr int HB = 1 << BITS;
    int32_t keys[HB];
    A acc[HB];
    __device__ __forceinline__ void init(int h) {
        keys[h] = kEmpty;
        acc[h] = A(0);
    }
    __device__ __forceinline__ int32_t key(int h) const { return keys[h]; }
    __device__ __forceinline__ A weight(int h) const { return acc[h]; }
    __device__ __forceinline__ int add(int32_t lab, A w, bool& isnew) {
        const int h = table_slot(keys, lab, BITS, isnew);
        if (h >= 0) atomicAdd(&acc[h], w);
        return h;
    }
    __device__ __forceinline__ void add_at(int h, A w) { atomicAdd(&acc[h], w); }
    __device__ __forceinline__ int find(int32_t lab) const {
        int h = (int)slot_hash(lab, BITS);
        for (int probe = 0; probe < HB; ++probe) {
            const int32_t cur = keys[h];
            if (cur == lab) return h;
            if (cur == kEmpty) return -1;
            h = (h + 1) & (HB - 1);
        }
        return -1;
    }
};

template <int BITS> struct STable<kUnit, BITS> {
    using A = uint32_t;
    static constexpr int HB = 1 << BITS;
    unsigned long long ent[HB];
    __device__ __forceinline__ void init(int h) { ent[h] = kEmpty64; }
    __device__ __forceinline__ int32_t key(int h) const { return (int32_t)(ent[h] >> 32); }
    __device__ __forceinline__ A weight(int h) const { return (uint32_t)ent[h]; }
    __device__ __forceinline__ void add_at(int h, uint32_t c) { atomicAdd(&ent[h], (unsigned long long)c); }
    __device__ __forceinline__ int add(int32_t lab, uint32_t c, bool& isnew) {
        int h = (int)slot_hash(lab, BITS);
        isnew = false;
        const unsigned long long mine = ((unsigned long long)(uint32_t)lab << 32) | c;
        for (int probe = 0; probe < HB; ++probe) {
            const unsigned long long e = *(volatile unsigned long long*)&ent[h];
            const int32_t k = (int32_t)(e >> 32);
            if (k == lab) {
                atomicAdd(&ent[h], (unsigned long long)c);
                return h;
            }
            if (k == kEmpty) {
                const unsigned long long old = atomicCAS(&ent[h], kEmpty64, mine);
                if (old == kEmpty64) {
                    isnew = true;
                    return h;
                }
                if ((int32_t)(old >> 32) == lab) {
                    atomicAdd(&ent[h], (unsigned long long)c);
                    return h;
                }
            }
            h = (h + 1) & (HB - 1);
        }
        return -1;
    }
    __device__ __forceinline__ int find(int32_t lab) const {
        int h = (int)slot_hash(lab, BITS);
        for (int probe = 0; probe < HB; ++probe) {
            const int32_t k = (int32_t)(ent[h] >> 32);
            if (k == lab) return h;
            if (k == kEmpty) return -1;
            h = (h + 1) & (HB - 1);
        }
        return -1;
    }
};

// Argmax candidate with the number of distinct labels sharing its
// (weight, sec) key -- `mult` > 1 means the first-position scan decides.
template <typename A> struct Best {
    A w;
    A w2;          // largest weight of any other label (== w on a tie at the maximum)
    uint32_t sec;
    uint32_t ter;  // ~first position once resolved, else 0
    int32_t lab;
    int32_t mult;
};

template <typename A> __device__ __forceinline__ A from_bits_any(unsigned long long b) {
    if constexpr (std::is_same<A, double>::value)
        return __longlong_as_double((long long)b);
    else if constexpr (std::is_same<A, float>::value)
        return __uint_as_float((uint32_t)b);
    else
        return (A)b;
}

template <typename A> __device__ __forceinline__ Best<A> none_best() {
    Best<A> b;
    b.w = A(0);
    b.w2 = A(0);
    b.sec = 0;
    b.ter = 0;
    b.lab = -1;
    b.mult = 0;
    return b;
}

template <int TIE>
__device__ __forceinline__ uint32_t sec_of(int32_t lab, uint32_t seed, uint32_t sweep, uint32_t vtx) {
    if (TIE == kScanFirst) return 0u;
    if (TIE == kMinLabel) return ~(uint32_t)lab;
    return tie_hash(seed, sweep, vtx, (uint32_t)lab);
}

// merge y into x (x keeps the larger key; equal keys add multiplicities)
// (w2 follows: the runner-up of the merge is the loser's weight or the
// winner's own runner-up, whichever is larger)
template <typename A> __device__ __forceinline__ void merge_best(Best<A>& x, const Best<A>& y) {
    if (y.mult == 0) return;
    if (x.mult == 0) {
        x = y;
    } else if (y.w > x.w || (y.w == x.w && (y.sec > x.sec || (y.sec == x.sec && y.ter > x.ter)))) {
        const A xw = x.w;
        x = y;
        x.w2 = x.w2 > xw ? x.w2 : xw;
    } else if (y.w == x.w && y.sec == x.sec && y.ter == x.ter) {
        x.mult += y.mult;
        x.lab = min(x.lab, y.lab);
        x.w2 = x.w;
    } else {
        x.w2 = x.w2 > y.w ? x.w2 : y.w;
    }
}

template <typename A> __device__ __forceinline__ Best<A> warp_merge(Best<A> b) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
        Best<A> o;
        o.w = shfl_xor_any(b.w, m);
        o.w2 = shfl_xor_any(b.w2, m);
        o.sec = __shfl_xor_sync(0xffffffffu, b.sec, m);
        o.ter = __shfl_xor_sync(0xffffffffu, b.ter, m);
        o.lab = __shfl_xor_sync(0xffffffffu, b.lab, m);
        o.mult = __shfl_xor_sync(0xffffffffu, b.mult, m);
        merge_best(b, o);
    }
    return b;
}

// Order-preserving 64-bit image of a (non-negative) weight, for max-reductions.
template <typename A> __device__ __forceinline__ unsigned long long wbits(A w) {
    if constexpr (std::is_same<A, double>::value)
        return (unsigned long long)__double_as_longlong(w);  // (non-negative: order-preserving)
    else if constexpr (std::is_same<A, float>::value)
        return (unsigned long long)__float_as_uint(w);
    else
        return (unsigned long long)w;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const unsigned long long u = shfl_u64(v, o);
        v = u > v ? u : v;
    }
    return v;
}

// Winner of the `nt` touched entries of a table, reduced over the calling
// group (one warp: GROUP_NW = 1, else a block of GROUP_NW warps using the
// shared scratch `red`).  Three cheap passes instead of a struct reduction:
// max weight, max tie key among the maxima, then how many entries share both
// (mult > 1 -> the caller resolves by scan order).
struct ArgmaxScratch {
    unsigned long long w;
    unsigned long long w2;  // largest weight below the maximum
    uint32_t sec;
    int32_t cnt;
    int32_t lab;
    int32_t cntw;           // entries at the maximum weight
};

template <int WM, int TIE, int BITS, int GROUP_NW>
__device__ __forceinline__ Best<typename Acc<WM>::T> table_argmax(const STable<WM, BITS>& t, const uint16_t* touched,
                                                                  int nt, int tid, uint32_t seed, uint32_t sweep,
                                                                  uint32_t vtx, ArgmaxScratch* red) {
    using A = typename Acc<WM>::T;
    constexpr int NT = GROUP_NW * 32;
    const int lane = threadIdx.x & 31;
    // 1. max weight
    unsigned long long mw = 0;
    for (int i = tid; i < nt; i += NT) {
        const unsigned long long b = wbits<A>(t.weight(touched[i]));
        mw = b > mw ? b : mw;
    }
    mw = warp_max_u64(mw);
    if (GROUP_NW > 1) {
        if (tid == 0) {
            red->w = 0;
            red->w2 = 0;
            red->sec = 0;
            red->cnt = 0;
            red->lab = -1;
            red->cntw = 0;
        }
        __syncthreads();
        if (lane == 0) atomicMax(&red->w, mw);
        __syncthreads();
        mw = red->w;
    }
    // 2. max tie key among the maxima (scan-first: none)
    uint32_t ms = 0;
    if (TIE != kScanFirst) {
        for (int i = tid; i < nt; i += NT) {
            const int h = touched[i];
            if (wbits<A>(t.weight(h)) == mw) {
                const uint32_t sc = sec_of<TIE>(t.key(h), seed, sweep, vtx);
                ms = sc > ms ? sc : ms;
            }
        }
        ms = __reduce_max_sync(0xffffffffu, ms);
        if (GROUP_NW > 1) {
            if (lane == 0) atomicMax(&red->sec, ms);
            __syncthreads();
            ms = red->sec;
        }
    }
    // 3. multiplicity and one label; entries at the maximum weight and the
    //    largest weight below it (the winner's lead, for the margin test)
    int c = 0, cw = 0;
    unsigned long long m2 = 0;
    int32_t lab = -1;
    for (int i = tid; i < nt; i += NT) {
        const int h = touched[i];
        const unsigned long long b = wbits<A>(t.weight(h));
        if (b == mw) {
            ++cw;
            if (TIE == kScanFirst || sec_of<TIE>(t.key(h), seed, sweep, vtx) == ms) {
                ++c;
                lab = t.key(h);
            }
        } else {
            m2 = b > m2 ? b : m2;
        }
    }
    Best<A> r;
    r.w = from_bits_any<A>(mw);
    r.sec = ms;
    r.ter = 0;
    const int wc = (int)__reduce_add_sync(0xffffffffu, (unsigned)c);
    const int wcw = (int)__reduce_add_sync(0xffffffffu, (unsigned)cw);
    m2 = warp_max_u64(m2);
    const unsigned hasb = __ballot_sync(0xffffffffu, lab >= 0);
    const int32_t wl = hasb ? __shfl_sync(0xffffffffu, lab, __ffs(hasb) - 1) : -1;
    int tcw = wcw;
    if (GROUP_NW > 1) {
        if (lane == 0) {
            if (wc) {
                atomicAdd(&red->cnt, wc);
                red->lab = wl;
            }
            if (wcw) atomicAdd(&red->cntw, wcw);
            if (m2) atomicMax(&red->w2, m2);
        }
        __syncthreads();
        r.mult = red->cnt;
        r.lab = red->lab;
        tcw = red->cntw;
        m2 = red->w2;
        __syncthreads();
    } else {
        r.mult = wc;
        r.lab = wl;
    }
    r.w2 = tcw > 1 ? r.w : from_bits_any<A>(m2);
    return r;
}

// Sum of `w` over the lanes in `m` (all lanes call; result in every lane).
template <typename A> __device__ __forceinline__ A masked_sum(uint32_t m, A w) {
    A v = ((m >> (threadIdx.x & 31)) & 1u) ? w : A(0);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += shfl_xor_any(v, o);
    return v;
}

// Winner of a row whose labels all have weight 1 (first sweep, kSingle): the
// tie rule over every arc -- largest tie key, then the earliest arc (what the
// table path's scan-order resolution gives).  One warp (red = null) or a
// block of NT threads (red = 2 shared words).
template <int TIE>
__device__ __forceinline__ int32_t all_singles_winner(const EvalArgs& a, uint32_t beg, int d, uint32_t vtx, int tid,
                                                      int NT, unsigned long long* red) {
    unsigned long long bk = 0;
    int32_t bl = -1;
    for (int k = tid; k < d; k += NT) {
        const int32_t lab = lb_strip(a, arc_label(a, beg + k));
        const unsigned long long key =
            ((unsigned long long)sec_of<TIE>(lab, a.seed, a.sweep, vtx) << 32) | (unsigned long long)(~(uint32_t)k);
        if (bl < 0 || key > bk) {
            bk = key;
            bl = lab;
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const unsigned long long ok = shfl_u64(bk, o);
        const int32_t ol = __shfl_xor_sync(0xffffffffu, bl, o);
        if (ol >= 0 && (bl < 0 || ok > bk)) {
            bk = ok;
            bl = ol;
        }
    }
    if (red == nullptr) return bl;
    if (tid == 0) red[0] = 0ull;
    __syncthreads();
    if ((tid & 31) == 0 && bl >= 0) atomicMax(&red[0], bk);
    __syncthreads();
    if ((tid & 31) == 0 && bl >= 0 && bk == red[0]) red[1] = (unsigned long long)(uint32_t)bl;
    __syncthreads();
    const int32_t r = (int32_t)(uint32_t)red[1];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------
// warp per vertex
// ---------------------------------------------------------------------------
template <int WM, int WC> struct WarpTable {
    static constexpr int kCap = (1 << WarpClass<WC>::kBits) / 4 * 3;  // touched entries before a spill
    STable<WM, WarpClass<WC>::kBits> t;
    uint16_t touched[kCap + 32];
    uint32_t sig[32];  // key signature (kSingle two-pass lookups); zero between rows
};

// 10-bit signature hash of a label (independent of slot_hash)
__device__ __forceinline__ uint32_t sig_hash(int32_t lab) { return ((uint32_t)lab * 0x85EBCA77u) >> 22; }

// Insert one 32-arc chunk into a shared table.  agg: fold equal labels with
// __match_any_sync first (rows with few distinct labels); otherwise every lane
// inserts its own label (rows whose labels are mostly distinct).
// Returns this lane's slot when it created a new entry, else -1.
// GSUM: fixed-point weights of a match group summed (two redux.sync) before one
// table atomic -- measured faster in the team kernels (long rows, hot labels),
// slower in the warp kernel
template <int WM, int BITS, bool GSUM = false>
__device__ __forceinline__ int insert_chunk(STable<WM, BITS>& t, int32_t lab, typename Acc<WM>::T w, bool agg,
                                            bool& full) {
    using A = typename Acc<WM>::T;
    const int lane = threadIdx.x & 31;
    bool isnew = false;
    int h = -1;
    if (agg) {
        const uint32_t grp = __match_any_sync(0xffffffffu, lab);
        const int leader = __ffs(grp) - 1;
        if constexpr (WM == kUnit) {
            if (lab != kEmpty && lane == leader) h = t.add(lab, (A)__popc(grp), isnew);
        } else if constexpr (WM == kFixed && GSUM) {
            const uint32_t wu = (uint32_t)w;
            const unsigned long long gs = ((unsigned long long)__reduce_add_sync(grp, wu >> 16) << 16) +
                                          (unsigned long long)__reduce_add_sync(grp, wu & 0xffffu);
            if (lab != kEmpty && lane == leader) h = t.add(lab, (A)gs, isnew);
        } else {
            if (lab != kEmpty && lane == leader) h = t.add(lab, A(0), isnew);
            const int hb = __shfl_sync(0xffffffffu, h, leader);
            if (lab != kEmpty && hb >= 0) atomicAdd(&t.acc[hb], w);
        }
        if (lab != kEmpty && lane == leader && h < 0) full = true;
    } else if (lab != kEmpty) {
        if constexpr (WM == kUnit)
            h = t.add(lab, 1u, isnew);
        else
            h = t.add(lab, w, isnew);
        if (h < 0) full = true;
    }
    return isnew ? h : -1;
}

// Warp per vertex.  Tally first in a warp-wide register table (entry t lives
// in lane t: key, weight, first position; up to 32 distinct labels) -- after
// the first sweep most rows hold a handful of labels and this path needs no
// shared memory and no atomics.  Rows estimated to hold more labels, or that
// outgrow the register table, use the warp's shared-memory hash.
// TWO: the kSingle two-pass tally (first sweep from ids; a separate
// instantiation keeps the other sweeps' code and registers unchanged)
template <int WM, int TIE, int WC, bool TWO>
__global__ void __launch_bounds__(WarpClass<WC>::kWarps * 32, WC == 0 && WM == kUnit ? 4 : 3) k_warp(EvalArgs a) {
    using A = typename Acc<WM>::T;
    using WT = WarpTable<WM, WC>;
    constexpr int kWarpBits = WarpClass<WC>::kBits;
    constexpr int kWarpCap = WT::kCap;
    constexpr int kWarpsPerBlock = WarpClass<WC>::kWarps;
    constexpr int HB = 1 << kWarpBits;
    // 32-arc chunks gathered per step (the two-pass first-sweep instantiation keeps fewer in flight:
    // measured 2.7% faster per exact R-MAT-22 detection at 2 than at 4, 1 and 3 in between)
    constexpr int U = TWO ? 2 : 4;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WT* tab = reinterpret_cast<WT*>(smem_raw) + wib;
    for (int h = lane; h < HB; h += 32) tab->t.init(h);
    tab->sig[lane] = 0u;
    __syncwarp();

    const int32_t cnt = a.r.len[WarpClass<WC>::kList];
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    const int32_t* list = a.r.warp[WC];
    const int cursor = kWarpCursor + WC;
    // batch size: 32 when the list is long, down to 1 so that short
    // (frontier) lists still spread over every warp
    const int bcap = max(1, min(32, cnt / (int)(gridDim.x * kWarpsPerBlock)));
    // ... and adapted to the arcs a batch held: the routed lists put long rows
    // first, and 32 of them in one warp's batch is a tail of the whole kernel
    int bsz = min(bcap, 2);
    while (true) {
        int32_t b0 = 0;
        if (lane == 0) b0 = atomicAdd(a.r.len + cursor, bsz);
        b0 = __shfl_sync(0xffffffffu, b0, 0);
        if (b0 >= cnt) break;
        const int nv = min(bsz, cnt - b0);
        int32_t ms = -1, mp = 0, mnd = 0, mx = 0, ml0 = 0;
        uint32_t mbeg = 0, mend = 0;
        if (lane < nv) {
            ms = list[b0 + lane];
            mp = __ldg(a.svid + ms);
            mbeg = __ldg(a.soff + ms);
            mend = __ldg(a.soff + ms + 1);
            mnd = __ldg(a.ndist + ms);
            // a vertex's label is written only by its own evaluation, once per
            // round: safe to load it with the batch
            mx = a.x[mp];
            ml0 = __ldg(a.L0 + mp);
        }
        // prefetched first label block of the current vertex
        int32_t nbr_next[U];
        {
            const uint32_t beg0 = __shfl_sync(0xffffffffu, mbeg, 0);
            const int d0 = (int)(__shfl_sync(0xffffffffu, mend, 0) - beg0);
#pragma unroll
            for (int c = 0; c < U; ++c) {
                const int k = c * 32 + lane;
                nbr_next[c] = (k < d0) ? arc_label(a, beg0 + k) : kEmpty;
            }
        }
        uint32_t chm = 0;  // batch vertices whose label changed (deferred marks)
        for (int v = 0; v < nv; ++v) {
            const int32_t s = __shfl_sync(0xffffffffu, ms, v);
            const int32_t p = __shfl_sync(0xffffffffu, mp, v);
            const uint32_t beg = __shfl_sync(0xffffffffu, mbeg, v);
            const int d = (int)(__shfl_sync(0xffffffffu, mend, v) - beg);
            const int32_t nd = __shfl_sync(0xffffffffu, mnd, v);
            const uint32_t vtx = (uint32_t)p;
            // prefetch the next block: of this row, else the next vertex's first one
#define LP_WARP_PREFETCH(base_done, wrap)                                                       \
    do {                                                                                        \
        uint32_t nb_beg = beg;                                                                  \
        int nb_base = (base_done) + 32 * U, nb_d = d;                                           \
        if (nb_base >= d && (wrap)) {                                                           \
            nb_base = 0;                                                                        \
        } else if (nb_base >= d) {                                                              \
            const int vn = v + 1 < nv ? v + 1 : v;                                              \
            nb_beg = __shfl_sync(0xffffffffu, mbeg, vn);                                        \
            nb_d = v + 1 < nv ? (int)(__shfl_sync(0xffffffffu, mend, vn) - nb_beg) : 0;         \
            nb_base = 0;                                                                        \
        }                                                                                       \
        _Pragma("unroll") for (int c_ = 0; c_ < U; ++c_) {                                      \
            const int k_ = nb_base + c_ * 32 + lane;                                            \
            nbr_next[c_] = (k_ < nb_d) ? arc_label(a, nb_beg + k_) : kEmpty;                   \
        }                                                                                       \
    } while (0)
            A total;
            if constexpr (WM == kUnit)
                total = (A)d;
            else if constexpr (WM == kFixed)
                total = (A)__ldg(a.swsum + s);
            else
                total = A(0);
            // ---- majority check (vertices whose last winner held > half the row) ----
            const int32_t xv = __shfl_sync(0xffffffffu, mx, v);
            const int32_t l0v = __shfl_sync(0xffffffffu, ml0, v);
            if (WM != kFloat && (nd & kMajBit)) {
                const int32_t cand = xv;
                A cw = A(0);
                for (int base = 0; base < d; base += 32 * U) {
                    int32_t labv[U];
#pragma unroll
                    for (int c = 0; c < U; ++c) {
                        const int k = base + c * 32 + lane;
                        labv[c] = (k < d) ? nbr_next[c] : kEmpty;
                    }
                    LP_WARP_PREFETCH(base, false);
#pragma unroll
                    for (int c = 0; c < U; ++c) {
                        const int k = base + c * 32 + lane;
                        if (k < d && (TWO ? lb_strip(a, labv[c]) : labv[c]) == cand) cw += arc_weight<WM>(a, beg + k);
                    }
                }
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) cw += shfl_xor_any(cw, o);
                if (cw + cw > total) {  // strict majority: the label stays
                    if (lane == 0) {
                        arcs += d;
                        ++verts;
                        store_gap<A>(a, s, cw, total);
                        LP_STAT(a, 0);
                    }
                    continue;
                }
                if (lane == 0) LP_STAT(a, 5);
                // no majority any more: full tally from the first block
#pragma unroll
                for (int c = 0; c < U; ++c) {
                    const int k = c * 32 + lane;
                    nbr_next[c] = (k < d) ? arc_label(a, beg + k) : kEmpty;
                }
            }
            const int est = min(d, nd_count(nd) + (nd_count(nd) >> 2) + 16);
            // fold equal labels (__match_any_sync) before inserting (per-lane inserts of
            // diverse rows measured 2x slower: hot labels serialise on one address)
            const bool agg = true;
            // register table (rows estimated to hold few labels)
            int32_t tkey = kEmpty;
            A tacc = A(0);
            uint32_t tfirst = 0;
            int K = 0;                  // register entries in use (warp-uniform)
            bool hashed = est > a.reg_est;  // use the shared hash
            int ntouched = 0;
            bool overflow = false;
            int singles = 0;  // (two passes) flagged labels absent from the table, this lane
            // (weighted two passes: the best absent flagged label of this lane, and the two
            // largest absent weights -- a singleton's weight is its arc's)
            Cand<A> sbest = none_cand<A>();
            A s1w = A(0), s2w = A(0);
            constexpr int npass = TWO ? 2 : 1;
            uint32_t mysig = 0;  // (two passes, hashed) lane's word of the table keys' 1024-bit signature
            for (int pass = 0; pass < npass && !overflow; ++pass) {
            if (TWO && pass == 1 && hashed) {
                // a flagged label whose signature bit is clear is absent: no probe
                for (int t = lane; t < ntouched; t += 32) {
                    const uint32_t h2 = sig_hash(tab->t.key(tab->touched[t]));
                    atomicOr(&tab->sig[h2 >> 5], 1u << (h2 & 31u));
                }
                __syncwarp();
                mysig = tab->sig[lane];
                tab->sig[lane] = 0u;
            }
            for (int base = 0; base < d && !overflow; base += 32 * U) {
                int32_t labv[U];
                A wv[U];
#pragma unroll
                for (int c = 0; c < U; ++c) {
                    const int k = base + c * 32 + lane;
                    labv[c] = (k < d) ? nbr_next[c] : kEmpty;
                    wv[c] = (k < d) ? arc_weight<WM>(a, beg + k) : A(0);
                }
                LP_WARP_PREFETCH(base, pass + 1 < npass);
#pragma unroll
                for (int c = 0; c < U; ++c) {
                    if (base + c * 32 >= d) break;  // warp-uniform
                    const int k0 = base + c * 32;
                    int32_t lab = labv[c];
                    const bool flag = TWO && lab >= 0 && (lab & kSingle);
                    if (TWO && lab >= 0) lab = lb_strip(a, lab);
                    if (TWO && pass == 1) {
                        // flagged labels: look up only
                        if (!__any_sync(0xffffffffu, flag)) continue;
                        bool hit = false;
                        if (!hashed) {
                            for (int t = 0; t < K; ++t) {
                                const int32_t key = __shfl_sync(0xffffffffu, tkey, t);
                                const uint32_t m = __ballot_sync(0xffffffffu, flag && lab == key);
                                if (m) {
                                    A add;
                                    if constexpr (WM == kUnit)
                                        add = (A)__popc(m);
                                    else
                                        add = masked_sum<A>(m, wv[c]);
                                    if (lane == t) {
                                        tacc += add;
                                        // (scan-first: a flagged arc may precede the entry's first one)
                                        tfirst = min(tfirst, (uint32_t)(k0 + __ffs(m) - 1));
                                    }
                                    hit |= flag && lab == key;
                                }
                            }
                        } else {
                            const uint32_t h2 = sig_hash(lab);
                            const uint32_t word = __shfl_sync(0xffffffffu, mysig, (int)(h2 >> 5));
                            if (flag && ((word >> (h2 & 31u)) & 1u)) {
                                const int h = tab->t.find(lab);
                                if (h >= 0) {
                                    tab->t.add_at(h, WM == kUnit ? A(1) : wv[c]);
                                    hit = true;
                                }
                            }
                        }
                        singles += (flag && !hit) ? 1 : 0;
                        if (WM != kUnit && flag && !hit) {
                            const A w = wv[c];
                            const Cand<A> sc = make_cand<TIE, A>(w, lab, (uint32_t)(k0 + lane), a.seed, a.sweep, vtx);
                            if (better(sc, sbest)) sbest = sc;
                            if (w > s1w) {
                                s2w = s1w;
                                s1w = w;
                            } else if (w > s2w) {
                                s2w = w;
                            }
                        }
                        continue;
                    }
                    if (flag) lab = kEmpty;  // pass 0 of two: evaluated labels only
                    if (TWO && !__any_sync(0xffffffffu, lab != kEmpty)) continue;  // (all flagged)
                    if (!hashed) {
                        uint32_t pending = __ballot_sync(0xffffffffu, lab != kEmpty);
                        for (int t = 0; t < K && pending; ++t) {
                            const int32_t key = __shfl_sync(0xffffffffu, tkey, t);
                            const uint32_t m = __ballot_sync(0xffffffffu, lab == key) & pending;
                            if (m) {
                                pending &= ~m;
                                A add;
                                if constexpr (WM == kUnit)
                                    add = (A)__popc(m);
                                else
                                    add = masked_sum<A>(m, wv[c]);
                                if (lane == t) tacc += add;
                            }
                        }
                        while (pending && K < 32) {
                            const int leader = __ffs(pending) - 1;
                            const int32_t key = __shfl_sync(0xffffffffu, lab, leader);
                            const uint32_t m = __ballot_sync(0xffffffffu, lab == key) & pending;
                            pending &= ~m;
                            A add;
                            if constexpr (WM == kUnit)
                                add = (A)__popc(m);
                            else
                                add = masked_sum<A>(m, wv[c]);
                            if (lane == K) {
                                tkey = key;
                                tacc = add;
                                tfirst = (uint32_t)(k0 + leader);
                            }
                            ++K;
                        }
                        if (!pending) continue;
                        // more than 32 distinct labels: move the register table
                        // to the shared hash, insert the rest of the chunk there
                        bool isnew = false;
                        int h = -1;
                        if (lane < K) h = tab->t.add(tkey, tacc, isnew);
                        const uint32_t nb = __ballot_sync(0xffffffffu, isnew);
                        if (isnew) tab->touched[__popc(nb & lanemask_lt())] = (uint16_t)h;
                        ntouched = __popc(nb);
                        __syncwarp();
                        hashed = true;
                        if (!((pending >> lane) & 1u)) lab = kEmpty;
                    }
                    bool full = false;
                    const int h = insert_chunk<WM, kWarpBits>(tab->t, lab, wv[c], agg, full);
                    const uint32_t nb = __ballot_sync(0xffffffffu, h >= 0);
                    if (h >= 0) {
                        const int idx = ntouched + __popc(nb & lanemask_lt());
                        if (idx < kWarpCap + 32) tab->touched[idx] = (uint16_t)h;
                    }
                    ntouched += __popc(nb);
                    __syncwarp();
                    if (ntouched > kWarpCap || __any_sync(0xffffffffu, full)) {
                        overflow = true;
                        break;
                    }
                }
            }
            }
            if (overflow) {
                if (lane == 0) LP_STAT(a, 4);
                // too many distinct labels for this table: wipe it and hand the
                // vertex to the team kernel (launched after this one); the
                // prefetched block may be this row's, refetch the next vertex's
                for (int h = lane; h < HB; h += 32) tab->t.init(h);
                if (lane == 0) {
                    if (WC == 0 && d <= WarpClass<1>::kMaxDeg) {
                        // next class up: the big-table warp kernel runs after this one
                        const int idx = atomicAdd(a.r.len + kLenWarpBig, 1);
                        a.r.warp[1][idx] = s;
                    } else {
                        const int idx = atomicAdd(a.r.len + kLenTeam, 1);
                        Item t = {s, 0, 1, 0, 1, -1, 0, 0};
                        a.r.team[idx] = t;
                    }
                    a.ndist[s] = max(nd_count(nd), 2 * WarpClass<WC>::kEst);
                }
                __syncwarp();
                LP_WARP_PREFETCH(d, false);
                continue;
            }
            int32_t winner;
            A wbest;
            A wsecond = A(0);
            if (!hashed) {
                Cand<A> best = none_cand<A>();
                if (lane < K) best = make_cand<TIE, A>(tacc, tkey, tfirst, a.seed, a.sweep, vtx);
                // only the first K lanes hold entries: reduce over the smallest power of two >= K
                for (int m = 16; m >= 1; m >>= 1) {
                    if (m >= K) continue;  // warp-uniform
                    Cand<A> o;
                    o.w = shfl_xor_any(best.w, m);
                    o.sec = __shfl_xor_sync(0xffffffffu, best.sec, m);
                    o.ter = __shfl_xor_sync(0xffffffffu, best.ter, m);
                    o.lab = __shfl_xor_sync(0xffffffffu, best.lab, m);
                    if (better(o, best)) best = o;
                }
                winner = __shfl_sync(0xffffffffu, best.lab, 0);
                wbest = best.w;  // valid in lane 0
                if (lane == 0) LP_STAT(a, 1);
                // runner-up weight (exact lead for the margin test)
                A w2 = (lane < K && tkey != winner) ? tacc : A(0);
#pragma unroll
                for (int m = 16; m >= 1; m >>= 1) {
                    const A o = shfl_xor_any(w2, m);
                    w2 = o > w2 ? o : w2;
                }
                wsecond = w2;
            } else {
                const Best<A> b = table_argmax<WM, TIE, kWarpBits, 1>(tab->t, tab->touched, ntouched, lane, a.seed,
                                                                     a.sweep, vtx, nullptr);
                winner = b.lab;
                wbest = b.w;
                wsecond = b.w2;
                if (lane == 0) LP_STAT(a, b.mult > 1 ? 3 : 2);
                if (b.mult > 1) {
                    // several labels tie at the maximum: the earliest in scan order wins
                    winner = -1;
                    for (int base = 0; base < d && winner < 0; base += 32) {
                        const int k = base + lane;
                        bool ok = false;
                        int32_t lab = kEmpty;
                        if (k < d) {
                            lab = arc_label(a, beg + k);
                            if (TWO) lab = lb_strip(a, lab);
                            const int h = tab->t.find(lab);
                            ok = h >= 0 && tab->t.weight(h) == b.w && sec_of<TIE>(lab, a.seed, a.sweep, vtx) == b.sec;
                        }
                        const uint32_t hit = __ballot_sync(0xffffffffu, ok);
                        if (hit) winner = __shfl_sync(0xffffffffu, lab, __ffs(hit) - 1);
                    }
                }
                __syncwarp();
                for (int t = lane; t < ntouched; t += 32) tab->t.init(tab->touched[t]);
                __syncwarp();
            }
            if (TWO && WM != kUnit) {
                const int nsingle = (int)__reduce_add_sync(0xffffffffu, (unsigned)singles);
                wbest = shfl_idx_any(wbest, 0);
                if (nsingle > 0) {
                    // the best absent flagged label against the table's winner
                    const Cand<A> sb = warp_best(sbest);
#pragma unroll
                    for (int o = 16; o >= 1; o >>= 1) {
                        const A o1 = shfl_xor_any(s1w, o), o2 = shfl_xor_any(s2w, o);
                        const A lo = s1w < o1 ? s1w : o1;
                        s1w = s1w > o1 ? s1w : o1;
                        const A m2 = s2w > o2 ? s2w : o2;
                        s2w = lo > m2 ? lo : m2;
                    }
                    const bool table = (hashed ? ntouched : K) > 0;
                    if (!table || sb.w > wbest) {
                        wsecond = table ? (wbest > s2w ? wbest : s2w) : s2w;
                        winner = sb.lab;
                        wbest = sb.w;
                    } else if (sb.w < wbest) {
                        wsecond = wsecond > s1w ? wsecond : s1w;
                    } else {
                        // equal weights: the tie rule decides (the table winner's first arc)
                        int first = -1;
                        for (int base = 0; base < d && first < 0; base += 32) {
                            const int k = base + lane;
                            const bool hitw = k < d && lb_strip(a, arc_label(a, beg + k)) == winner;
                            const uint32_t hm = __ballot_sync(0xffffffffu, hitw);
                            if (hm) first = base + __ffs(hm) - 1;
                        }
                        const Cand<A> tc = make_cand<TIE, A>(wbest, winner, (uint32_t)first, a.seed, a.sweep, vtx);
                        if (better(sb, tc)) winner = sb.lab;
                        wsecond = wbest;
                    }
                }
            }
            if (TWO && WM == kUnit) {
                const int nsingle = (int)__reduce_add_sync(0xffffffffu, (unsigned)singles);
                wbest = __shfl_sync(0xffffffffu, wbest, 0);
                if (nsingle > 0) {
                    if (wbest < A(2)) {
                        // every label has weight 1: the tie rule over all arcs
                        winner = all_singles_winner<TIE>(a, beg, d, vtx, lane, 32, nullptr);
                        wbest = A(1);
                        wsecond = d > 1 ? A(1) : A(0);
                    } else if (wsecond < A(1)) {
                        wsecond = A(1);
                    }
                }
            }
            bool changed = false;
            if (lane == 0) {
                arcs += d;
                ++verts;
                const bool maj = WM != kFloat && wbest + wbest > total;
                a.ndist[s] = (hashed ? ntouched : K) | (maj ? kMajBit : 0);
                store_lead<A>(a, s, wbest, wsecond);
                changed = commit_label_known(a, p, winner, xv, l0v, dchg, writes);
            }
            changed = __shfl_sync(0xffffffffu, changed, 0);
            if (changed) chm |= 1u << v;
        }
        if (a.mark) push_changed_batch(a, chm, ms, (int)(mend - mbeg));
        {
            constexpr int kBatchArcs = 1024;
            const int tot = (int)__reduce_add_sync(0xffffffffu, lane < nv ? (unsigned)(mend - mbeg) : 0u);
            bsz = max(1, min(bcap, (int)((long long)nv * kBatchArcs / max(tot, 1))));
        }
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

// ---------------------------------------------------------------------------
// block (team) per work item
// ---------------------------------------------------------------------------
template <int WM, int TBITS> struct TeamTable {
    static constexpr int HB = 1 << TBITS;
    static constexpr int CAP = HB / 4 * 3;  // touched capacity; beyond it = overflow
    STable<WM, TBITS> t;
    uint16_t touched[CAP];
};

template <typename A> __device__ __forceinline__ unsigned long long to_bits(A w) {
    if constexpr (std::is_same<A, double>::value)
        return (unsigned long long)__double_as_longlong(w);  // (non-negative: order-preserving)
    else if constexpr (std::is_same<A, float>::value)
        return (unsigned long long)__float_as_uint(w);
    else
        return (unsigned long long)w;
}
template <typename A> __device__ __forceinline__ A from_bits(unsigned long long b) {
    if constexpr (std::is_same<A, double>::value)
        return __longlong_as_double((long long)b);
    else if constexpr (std::is_same<A, float>::value)
        return __uint_as_float((uint32_t)b);
    else
        return (A)b;
}

template <typename A> __device__ __forceinline__ void gacc_add(unsigned long long* acc, A w) {
    if constexpr (std::is_same<A, double>::value)
        atomicAdd(reinterpret_cast<double*>(acc), w);
    else if constexpr (std::is_same<A, float>::value)
        atomicAdd(reinterpret_cast<float*>(acc), w);
    else
        atomicAdd(acc, (unsigned long long)w);
}
template <typename A> __device__ __forceinline__ A gacc_read(const unsigned long long* acc) {
    if constexpr (std::is_same<A, double>::value)
        return __ldcg(reinterpret_cast<const double*>(acc));
    else if constexpr (std::is_same<A, float>::value)
        return __ldcg(reinterpret_cast<const float*>(acc));
    else
        return (A)__ldcg(acc);
}

template <int WM, int TIE, int NT, int TBITS, bool DYNAMIC>
__global__ void __launch_bounds__(NT, NT >= 1024 ? 1 : (NT == 512 ? 2 : 3)) k_team(EvalArgs a, int which) {
    using A = typename Acc<WM>::T;
    using Tab = TeamTable<WM, TBITS>;
    constexpr int HB = Tab::HB;
    constexpr int CAP = Tab::CAP;
    constexpr int NW = NT / 32;
    constexpr int U = LP_TEAM_U;  // 32-arc chunks in flight per warp
    constexpr int STACK = 40;
    constexpr int GHB = 1 << kGlobalBits;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Tab* tab = reinterpret_cast<Tab*>(smem_raw);
    __shared__ int32_t s_nt;
    __shared__ int32_t s_item;
    __shared__ int32_t s_flag;
    __shared__ int32_t s_last;
    __shared__ int32_t s_gnew;
    __shared__ int32_t s_full;
    __shared__ int32_t s_sp;
    __shared__ int32_t s_single;  // kSingle labels absent from the tables (this item)
    __shared__ int32_t s_fb;      // every label has weight 1: pick over all arcs
    __shared__ unsigned long long s_fbred[2];
    __shared__ unsigned long long s_first;  // (position << 32) | label of the earliest tied arc
    __shared__ uint32_t s_stack[STACK][2];  // (parts, want)
    __shared__ Best<A> s_red[NW];
    __shared__ A s_cw[NW];
    __shared__ ArgmaxScratch s_arg;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    // kSingle two-pass tally (first sweep from ids; hub rows are then routed as
    // label partitions, never as slices: a slice cannot look labels up after
    // the other slices' inserts)
    const bool two = a.two_team;
    for (int h = tid; h < HB; h += NT) tab->t.init(h);
    const Item* items = which == kLenHub ? a.r.hub : (which == kLenTeam2 ? a.r.team2 : a.r.team);
    const int cursor = which == kLenHub ? kHubCursor : (which == kLenTeam2 ? kTeam2Cursor : kTeamCursor);
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    int32_t it = blockIdx.x;
    __syncthreads();
    const int32_t cnt = a.r.len[which];

    auto block_merge = [&](Best<A> b) -> Best<A> {
        b = warp_merge(b);
        if (lane == 0) s_red[warp] = b;
        __syncthreads();
        Best<A> r = lane < NW ? s_red[lane] : none_best<A>();
        r = warp_merge(r);
        __syncthreads();
        return r;
    };

    // Best label of row arcs [0, d) restricted to label partitions taken from
    // the work stack (preloaded by the caller).  Sub-splits on overflow.
    // `single`: one whole-row pass (no first position needed unless tied).
    auto row_best = [&](const uint32_t beg, const int d, const uint32_t vtx, bool single,
                        bool agg, int& distinct, int2 bk = make_int2(0, -1), uint32_t topP = 1) -> Best<A> {
        Best<A> overall = none_best<A>();
        distinct = 0;
        // bucketed: the arcs are the partition's bucket hb_lab/hb_pos[bk.x, bk.x + bk.y)
        const bool bucketed = bk.y >= 0;
        const int dd = bucketed ? bk.y : d;
        while (true) {
            const int sp = s_sp;
            if (sp == 0) break;
            const uint32_t parts = s_stack[sp - 1][0], want = s_stack[sp - 1][1];
            __syncthreads();
            if (tid == 0) {
                s_sp = sp - 1;
                s_nt = 0;
                s_full = 0;
            }
            __syncthreads();
            // raw labels (and bucket arc positions) of the warp's next U chunks,
            // loaded one step ahead: the loads of step i+1 are in flight while
            // step i inserts (the tally was stalled on these loads)
            int32_t pre_lab[U];
            uint32_t pre_pos[U];
            auto fetch = [&](int base) {
#pragma unroll
                for (int c = 0; c < U; ++c) {
                    const int k = base + c * 32 + lane;
                    pre_lab[c] = kEmpty;
                    pre_pos[c] = 0;
                    if (k < dd) {
                        if (bucketed) {
                            pre_lab[c] = a.hb_lab[bk.x + k];
                            if (WM != kUnit) pre_pos[c] = a.hb_pos[bk.x + k];
                        } else {
                            pre_lab[c] = arc_label(a, beg + k);
                        }
                    }
                }
            };
            fetch(warp * 32 * U);
            for (int base = warp * 32 * U; base < dd; base += NT * U) {
                int32_t labv[U];
                A wv[U];
                int32_t raw[U];
                uint32_t rpos[U];
#pragma unroll
                for (int c = 0; c < U; ++c) {
                    raw[c] = pre_lab[c];
                    rpos[c] = pre_pos[c];
                }
                if (base + NT * U < dd) fetch(base + NT * U);
#pragma unroll
                for (int c = 0; c < U; ++c) {
                    const int k = base + c * 32 + lane;
                    int32_t lab = kEmpty;
                    A w = A(0);
                    if (bucketed) {
                        if (k < dd) {
                            lab = raw[c];
                            w = WM == kUnit ? A(1) : arc_weight<WM>(a, beg + rpos[c]);
                            if (two && (lab & kSingle)) lab = kEmpty;  // (looked up below)
                            else {
                                lab = lb_strip(a, lab);
                                if (parts > topP && part_of(lab, parts) != want) lab = kEmpty;
                            }
                        }
                    } else if (k < d) {
                        lab = raw[c];
                        w = arc_weight<WM>(a, beg + k);
                        if (two && (lab & kSingle)) lab = kEmpty;  // (two passes: looked up below)
                        else if (parts > 1 && part_of(lb_strip(a, lab), parts) != want) lab = kEmpty;
                        else lab = lb_strip(a, lab);
                    }
                    labv[c] = lab;
                    wv[c] = w;
                }
#pragma unroll
                for (int c = 0; c < U; ++c) {
                    bool full = false;
                    const int h = insert_chunk<WM, TBITS, true>(tab->t, labv[c], wv[c], agg, full);
                    const uint32_t nb = __ballot_sync(0xffffffffu, h >= 0);
                    if (nb) {
                        int b0 = 0;
                        if (lane == 0) b0 = atomicAdd(&s_nt, __popc(nb));
                        b0 = __shfl_sync(0xffffffffu, b0, 0);
                        const int idx = b0 + __popc(nb & lanemask_lt());
                        if (h >= 0 && idx < CAP) tab->touched[idx] = (uint16_t)h;
                    }
                    if (__any_sync(0xffffffffu, full) && lane == 0) s_full = 1;
                }
                if (__shfl_sync(0xffffffffu, *(volatile int32_t*)&s_nt, 0) > CAP ||
                    __shfl_sync(0xffffffffu, *(volatile int32_t*)&s_full, 0))
                    break;  // overflowing
            }
            __syncthreads();
            const int nt = s_nt;
            const bool overflow = nt > CAP || s_full;
            if (overflow) {
                for (int h = tid; h < HB; h += NT) tab->t.init(h);
                __syncthreads();
                if (tid == 0) {
                    if (s_sp + 4 > STACK || parts >= (1u << 28)) {
                        // no room for another 4-way split: fail the run loudly
                        // (the engine checks kCtrError after every sweep)
                        atomicAdd(a.counters + kCtrError, 1ull);
                    } else {
                        for (int j = 3; j >= 0; --j) {
                            s_stack[s_sp][0] = parts * 4;
                            s_stack[s_sp][1] = want * 4 + j;
                            ++s_sp;
                        }
                    }
                }
                single = false;
                __syncthreads();
                continue;
            }
            Best<A> sb = none_best<A>();  // (weighted) best absent flagged label of this partition
            if (two) {
                // pass 2: flagged labels of this partition are looked up only
                int sg = 0;
                for (int k = tid; k < dd && bucketed; k += NT) {
                    int32_t lab = a.hb_lab[bk.x + k];
                    if (lab & kSingle) {
                        lab = lb_strip(a, lab);
                        if (parts <= topP || part_of(lab, parts) == want) {
                            const int h = tab->t.find(lab);
                            if (h >= 0)
                                tab->t.add_at(h, A(1));
                            else
                                ++sg;
                        }
                    }
                }
                // (four label loads in flight per lane: one block walks the whole row, and a
                // hub's 100K arcs at one dependent load per step were the round's tail)
                constexpr int J2 = LP_TEAM_J2;
                for (int base0 = warp * 32; base0 < d && !bucketed; base0 += NT * J2) {
                    int32_t pl[J2];
#pragma unroll
                    for (int j = 0; j < J2; ++j) {
                        const int k = base0 + j * NT + lane;
                        pl[j] = k < d ? arc_label(a, beg + k) : 0;
                    }
#pragma unroll
                    for (int j = 0; j < J2; ++j) {
                    const int k = base0 + j * NT + lane;
                    if (k < d) {
                        int32_t lab = pl[j];
                        if (lab & kSingle) {
                            lab = lb_strip(a, lab);
                            if (parts <= 1 || part_of(lab, parts) == want) {
                                const A w = WM == kUnit ? A(1) : arc_weight<WM>(a, beg + k);
                                const int h = tab->t.find(lab);
                                if (h >= 0) {
                                    tab->t.add_at(h, w);
                                } else {
                                    ++sg;
                                    if constexpr (WM != kUnit) {
                                        // a weighted singleton competes with its arc's weight
                                        Best<A> c;
                                        c.w = w;
                                        c.w2 = A(0);
                                        c.sec = sec_of<TIE>(lab, a.seed, a.sweep, vtx);
                                        c.ter = ~(uint32_t)k;
                                        c.lab = lab;
                                        c.mult = 1;
                                        merge_best(sb, c);
                                    }
                                }
                            }
                        }
                    }
                    }
                }
                sg = (int)__reduce_add_sync(0xffffffffu, (unsigned)sg);
                if (lane == 0 && sg) atomicAdd(&s_single, sg);
                __syncthreads();
                if constexpr (WM != kUnit) sb = block_merge(sb);
            }
            Best<A> b = table_argmax<WM, TIE, TBITS, NW>(tab->t, tab->touched, nt, tid, a.seed, a.sweep, vtx, &s_arg);
            const bool last_pass = single && s_sp == 0;
            // (weighted singletons: a tie in weight with the table's winner needs its
            // first arc -- resolve it)
            const bool wsing = WM != kUnit && two && sb.mult > 0;
            const bool force = wsing && nt > 0 && sb.w == b.w;
            if (b.mult > 1 || !last_pass || force) {
                // earliest arc (scan order) whose label carries the pass maximum
                if (tid == 0) s_first = ~0ull;
                __syncthreads();
                if (bucketed) {
                    // (bucket order is not scan order: every hit proposes its position)
                    for (int k = tid; k < dd; k += NT) {
                        const int32_t lab = lb_strip(a, a.hb_lab[bk.x + k]);
                        if (parts <= topP || part_of(lab, parts) == want) {
                            const int h = tab->t.find(lab);
                            if (h >= 0 && tab->t.weight(h) == b.w && sec_of<TIE>(lab, a.seed, a.sweep, vtx) == b.sec)
                                atomicMin(&s_first, ((unsigned long long)a.hb_pos[bk.x + k] << 32) | (uint32_t)lab);
                        }
                    }
                }
                for (int base = warp * 32; base < d && !bucketed; base += NT) {
                    const unsigned long long seen = __shfl_sync(0xffffffffu, *(volatile unsigned long long*)&s_first, 0);
                    if ((unsigned long long)base > (seen >> 32)) break;  // an earlier hit exists
                    const int k = base + lane;
                    bool ok = false;
                    int32_t lab = kEmpty;
                    if (k < d) {
                        lab = lb_strip(a, arc_label(a, beg + k));
                        if (parts <= 1 || part_of(lab, parts) == want) {
                            const int h = tab->t.find(lab);
                            ok = h >= 0 && tab->t.weight(h) == b.w &&
                                 sec_of<TIE>(lab, a.seed, a.sweep, vtx) == b.sec;
                        }
                    }
                    const uint32_t hit = __ballot_sync(0xffffffffu, ok);
                    if (hit) {
                        const int j = __ffs(hit) - 1;
                        if (lane == j) atomicMin(&s_first, ((unsigned long long)k << 32) | (uint32_t)lab);
                        break;
                    }
                }
                __syncthreads();
                const unsigned long long f = s_first;
                b.lab = (int32_t)(uint32_t)f;
                b.ter = ~(uint32_t)(f >> 32);
                b.mult = 1;
            }
            if (wsing) {
                if (nt == 0)
                    b = sb;
                else
                    merge_best(b, sb);
            }
            merge_best(overall, b);
            distinct += nt;
            for (int t = tid; t < nt; t += NT) tab->t.init(tab->touched[t]);
            __syncthreads();
        }
        return overall;
    };

    while (true) {
        if (DYNAMIC) {
            if (tid == 0) s_item = atomicAdd(a.r.len + cursor, 1);
            __syncthreads();
            it = s_item;
        }
        if (it >= cnt) break;
        const Item item = items[it];
        const int32_t s = item.s;
        const int32_t p = __ldg(a.svid + s);
        const uint32_t beg = __ldg(a.soff + s);
        const int d = (int)(__ldg(a.soff + s + 1) - beg);
        const uint32_t vtx = (uint32_t)p;
        const int32_t nd = __ldg(a.ndist + s);
        A total;
        if constexpr (WM == kUnit)
            total = (A)d;
        else if constexpr (WM == kFixed)
            total = (A)__ldg(a.swsum + s);
        else
            total = A(0);
        // ---- majority check for whole-row items of flagged vertices ----
        if (WM != kFloat && item.P == 1 && item.R == 1 && (nd & kMajBit)) {
            const int32_t cand = a.x[p];
            A cw = A(0);
            for (int base = warp * 32 * U; base < d; base += NT * U) {
                int32_t labv[U];
#pragma unroll
                for (int c = 0; c < U; ++c) {
                    const int k = base + c * 32 + lane;
                    labv[c] = (k < d) ? lb_strip(a, arc_label(a, beg + k)) : kEmpty;
                }
#pragma unroll
                for (int c = 0; c < U; ++c) {
                    const int k = base + c * 32 + lane;
                    if (k < d && labv[c] == cand) cw += arc_weight<WM>(a, beg + k);
                }
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) cw += shfl_xor_any(cw, o);
            if (lane == 0) s_cw[warp] = cw;
            __syncthreads();
            A tot_cw = A(0);
#pragma unroll
            for (int w2 = 0; w2 < NW; ++w2) tot_cw += s_cw[w2];
            __syncthreads();
            if (tot_cw + tot_cw > total) {  // strict majority: the label stays
                if (tid == 0) {
                    arcs += d;
                    ++verts;
                    store_gap<A>(a, s, tot_cw, total);
                }
                if (!DYNAMIC) it += gridDim.x;
                continue;
            }
        }
        const int est = min(d, nd_count(nd) + (nd_count(nd) >> 2) + 16);
        const bool agg = true;
        Best<A> best = none_best<A>();
        int distinct = 0;
        bool last = true;
        if (item.R == 1) {
            if (tid == 0) {
                s_sp = 1;
                s_stack[0][0] = (uint32_t)item.P;
                s_stack[0][1] = (uint32_t)item.q;
                s_single = 0;
                s_fb = 0;
            }
            __syncthreads();
            int2 bk = make_int2(0, -1);
            if (item.P > 1 && a.hb_off) bk = a.hb_off[item.cb + item.q];
            best = row_best(beg, d, vtx, item.P == 1, agg, distinct, bk, (uint32_t)item.P);
            if (WM == kUnit && item.P == 1 && two && tid == 0 && s_single > 0) {
                if (best.w < A(2))
                    s_fb = 1;
                else if (best.w2 < A(1))
                    best.w2 = A(1);
            }
            if (item.P > 1) {
                // the last partition block merges the P candidates
                if (tid == 0) {
                    HubCand hc;
                    hc.w = to_bits<A>(best.w);
                    hc.w2 = to_bits<A>(best.w2);
                    hc.sec = best.sec;
                    hc.ter = best.ter;
                    hc.lab = best.lab;
                    hc.nd = distinct;
                    hc.single = s_single;
                    a.r.cand[item.cb + item.q] = hc;
                    __threadfence();
                    s_last = atomicAdd(a.r.cand_done + item.cb, 1) == item.P - 1;
                    if (s_last) {
                        __threadfence();
                        distinct = 0;
                        int msingle = 0;
                        best = none_best<A>();
                        for (int j = 0; j < item.P; ++j) {
                            const HubCand* src = a.r.cand + item.cb + j;
                            Best<A> o;
                            o.w = from_bits<A>(__ldcg(&src->w));
                            o.w2 = from_bits<A>(__ldcg(&src->w2));
                            o.sec = __ldcg(&src->sec);
                            o.ter = __ldcg(&src->ter);
                            o.lab = __ldcg(&src->lab);
                            o.mult = 1;
                            distinct += __ldcg(&src->nd);
                            msingle += __ldcg(&src->single);
                            merge_best(best, o);
                        }
                        if (WM == kUnit && two && msingle > 0) {
                            if (best.w < A(2))
                                s_fb = 1;
                            else if (best.w2 < A(1))
                                best.w2 = A(1);
                        }
                        a.r.cand_done[item.cb] = 0;
                    }
                }
                __syncthreads();
                last = s_last;
            }
            __syncthreads();
            if (s_fb) {  // (block-uniform; set only where this block commits)
                const int32_t wl = all_singles_winner<TIE>(a, beg, d, vtx, tid, NT, s_fbred);
                if (tid == 0) {
                    best.lab = wl;
                    best.w = A(1);
                    best.w2 = d > 1 ? A(1) : A(0);
                }
            }
        } else {
            // ---- arc slice: fold this slice into the per-vertex global table ----
            const int k_lo = (int)((long long)d * item.r / item.R);
            const int k_hi = (int)((long long)d * (item.r + 1) / item.R);
            int32_t* gkeys = a.r.gkeys + item.gt;
            uint32_t* gfirst = a.r.gfirst + item.gt;
            unsigned long long* gacc = a.r.gacc + item.gt;
            int32_t* gtl = a.r.gtl + item.gt;
            const int gbits = item.gbits;
            const int gcapv = (1 << gbits) / 4 * 3;
            if (tid == 0) s_gnew = 0;
            __syncthreads();
            for (int base = k_lo + warp * 32; base < k_hi; base += NT) {
                const int k = base + lane;
                int32_t lab = kEmpty;
                A w = A(0);
                if (k < k_hi) {
                    lab = lb_strip(a, arc_label(a, beg + k));
                    w = arc_weight<WM>(a, beg + k);
                }
                const uint32_t grp = __match_any_sync(0xffffffffu, lab);
                const int leader = __ffs(grp) - 1;
                int g = -1;
                bool isnew = false;
                if (lab != kEmpty && lane == leader) {
                    g = table_slot(gkeys, lab, gbits, isnew);
                    if (g >= 0) {
                        atomicMin(gfirst + g, (uint32_t)k);
                        if constexpr (WM == kUnit) gacc_add<A>(gacc + g, (A)__popc(grp));
                    } else {
                        atomicAdd(&s_gnew, 1);  // table full
                    }
                }
                // new entries join the table's list: one counter atomic per warp chunk
                const uint32_t nbal = __ballot_sync(0xffffffffu, isnew);
                if (nbal) {
                    int t0 = 0;
                    if (lane == __ffs(nbal) - 1) t0 = atomicAdd(a.r.gcount + item.cb, __popc(nbal));
                    t0 = __shfl_sync(0xffffffffu, t0, __ffs(nbal) - 1);
                    const int ti = t0 + __popc(nbal & lanemask_lt());
                    if (isnew && ti < gcapv) gtl[ti] = g;
                }
                if constexpr (WM != kUnit) {
                    const int gb = __shfl_sync(0xffffffffu, g, leader);
                    if (lab != kEmpty && gb >= 0) gacc_add<A>(gacc + gb, w);
                }
            }
            __syncthreads();
            if (tid == 0) {
                if (s_gnew) atomicAdd(a.r.gcount + item.cb, 1 << 28);  // table full: slow path
                __threadfence();
                s_last = atomicAdd(a.r.cand_done + item.cb, 1) == item.R - 1;
                if (s_last) __threadfence();
            }
            __syncthreads();
            last = s_last;
            if (last) {
                const int gcount = __ldcg(a.r.gcount + item.cb);
                const bool ok = gcount <= gcapv;
                Best<A> b = none_best<A>();
                if (ok) {
                    for (int i = tid; i < gcount; i += NT) {
                        const int g = __ldcg(gtl + i);
                        const int32_t key = __ldcg(gkeys + g);
                        Best<A> c;
                        c.w = gacc_read<A>(gacc + g);
                        c.w2 = A(0);
                        c.lab = key;
                        c.sec = sec_of<TIE>(key, a.seed, a.sweep, vtx);
                        c.ter = ~__ldcg(gfirst + g);
                        c.mult = 1;
                        merge_best(b, c);
                    }
                    for (int i = tid; i < gcount; i += NT) {
                        const int g = __ldcg(gtl + i);
                        gkeys[g] = kEmpty;
                        gfirst[g] = 0xffffffffu;
                        gacc[g] = 0ull;
                    }
                } else {
                    for (int g = tid; g < (1 << gbits); g += NT) {
                        gkeys[g] = kEmpty;
                        gfirst[g] = 0xffffffffu;
                        gacc[g] = 0ull;
                    }
                }
                best = block_merge(b);
                distinct = gcount;
                if (tid == 0) {
                    a.r.cand_done[item.cb] = 0;
                    a.r.gcount[item.cb] = 0;
                }
                if (!ok) {
                    // rare slow path: labels were underestimated; this block
                    // redoes the whole row in four label partitions (or more)
                    if (tid == 0) {
                        for (int j = 0; j < 4; ++j) {
                            s_stack[j][0] = 4;
                            s_stack[j][1] = (uint32_t)j;
                        }
                        s_sp = 4;
                    }
                    __syncthreads();
                    best = row_best(beg, d, vtx, false, false, distinct);
                }
            }
        }
        if (tid == 0) {
            s_flag = 0;
            if (last) {
                arcs += d;
                ++verts;
                const bool maj = WM != kFloat && best.w + best.w > total;
                a.ndist[s] = distinct | (maj ? kMajBit : 0);
                store_lead<A>(a, s, best.w, best.w2);
                s_flag = commit_label(a, p, best.lab, dchg, writes) ? 1 : 0;
            }
        }
        if (tid == 0 && s_flag && a.mark) push_changed(a, s, d);
        __syncthreads();
        if (!DYNAMIC) it += gridDim.x;
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

template <int WM, int WC> constexpr size_t warp_smem_bytes() {
    return sizeof(WarpTable<WM, WC>) * WarpClass<WC>::kWarps;
}
template <int WM, int TBITS> constexpr size_t team_smem_bytes() { return sizeof(TeamTable<WM, TBITS>); }

}  // namespace lp
