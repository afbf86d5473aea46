// lp_rak_kernels.cuh -- the RAK sweep kernels (the hot path).
//
// Replaces the body of the reference's sweep, rak.py:97-113 (_rak_seq) /
// :138-154 (_rak_par): for each vertex, accumulate the weights of its
// neighbours' labels, take the argmax under the tie rule, write the label
// and count the change.
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
    uint32_t sec;
    uint32_t ter;
    int32_t lab;
    int32_t nd;
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
    int32_t pad;
};

// route-list lengths / cursors (device ints)
enum {
    kLenS4 = 0,   // small rows, d <= 4
    kLenS8 = 1,   // d <= 8
    kLenS16 = 2,  // d <= 16
    kLenWarp = 3,
    kLenTeam = 4,
    kLenHub = 5,
    kCandCursor = 6,
    kTeamCursor = 7,
    kHubCursor = 8,
    kGtabCursor = 9,
    kLenCount = 12
};

struct Routes {
    int32_t* small[3];  // slot lists by small degree class (4, 8, 16)
    int32_t* warp;
    Item* team;
    Item* hub;
    int32_t* len;  // kLen*
    HubCand* cand;
    int32_t* cand_done;
    int32_t* gkeys;  // global slice tables (SoA)
    uint32_t* gfirst;
    unsigned long long* gacc;
    int32_t* gcount;  // distinct count per slice table (indexed by cb)
};

struct EvalArgs {
    const uint32_t* __restrict__ soff;  // storage row offsets [S+1]
    const int32_t* __restrict__ snbr;   // neighbour positions
    const uint32_t* __restrict__ sw;    // arc weights (fixed-point u32 or float bits); null = unit
    const int32_t* __restrict__ spos;   // slot -> position
    const int32_t* __restrict__ vid;    // position -> vertex id
    const int32_t* __restrict__ L0;     // labels at sweep start (read-only in a sweep)
    int32_t* x;                         // working labels (read + written in place)
    uint8_t* mark;                      // next-round marks by position, null = no cross-batch deps
    int32_t* ndist;                     // per-slot distinct-label count of the last evaluation
    unsigned long long* counters;       // see kCtr* below
    Routes r;
    int32_t bs;   // batch size in positions
    int32_t bin;  // counter slot of this launch
    uint32_t seed;
    uint32_t sweep;
};

// counters: [0] changed delta (reset per sweep), [1] label writes (reset per
// round), [4+k] arcs scanned and [8+k] vertices evaluated by kernel k
// (k = 0 hub team, 1 8-warp team, 2 warp, 3 small; accumulated over a run)
enum { kCtrChanged = 0, kCtrWrites = 1, kCtrArcs = 4, kCtrVerts = 8, kCtrCount = 12 };

constexpr int kSmallMax = 16;     // thread-per-vertex bound (degree)
constexpr int kWarpEst = 256;     // warp path: estimated distinct labels
constexpr int kWarpMaxDeg = 2048;
constexpr int kWarpBits = 9;      // 512-slot warp table
constexpr int kWarpCap = 384;     // touched entries before a warp spills
constexpr int kWarpsPerBlock = 8;
constexpr int kTeamEst = 2048;    // 8-warp team: 4096-slot table
constexpr int kTeamMaxDeg = 16384;
constexpr int kTeamBits = 12, kTeamThreads = 256;
constexpr int kHubBits = 13, kHubThreads = 512;  // 16-warp team: 8192 slots
constexpr int kHubPlan = 4096;     // distinct labels planned per hub partition
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
        return __uint_as_float(__ldg(a.sw + e));
    }
}

// Neighbour label under the batched schedule: neighbours in an earlier batch
// have already been solved this sweep (x), the rest still hold L0.
__device__ __forceinline__ int32_t read_label(const EvalArgs& a, int32_t u, int32_t thr) {
    return (u < thr) ? a.x[u] : __ldg(a.L0 + u);
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

// Write a vertex's new label (one thread).  Returns true when it changed.
__device__ __forceinline__ bool commit_label(const EvalArgs& a, int32_t p, int32_t lab, long long& dchg,
                                             long long& writes) {
    const int32_t old = a.x[p];
    if (lab == old || lab < 0) return false;
    a.x[p] = lab;
    const int32_t l0 = __ldg(a.L0 + p);
    dchg += (long long)(lab != l0) - (long long)(old != l0);
    ++writes;
    return true;
}

// Mark the later-batch neighbours of a vertex whose label changed.
__device__ __forceinline__ void mark_row(const EvalArgs& a, uint32_t beg, int d, int32_t thr, int from, int step) {
    const int32_t nb = thr + a.bs;
    for (int k = from; k < d; k += step) {
        const int32_t u = __ldg(a.snbr + beg + k);
        if (u >= nb) a.mark[u] = 1;
    }
}

// ---------------------------------------------------------------------------
// routing
// ---------------------------------------------------------------------------
// cls: 0/1/2 small (d <= 4 / 8 / 16), 3 warp, 4 team, 5 hub
__device__ __forceinline__ int small_class(int d) { return d <= 4 ? 0 : (d <= 8 ? 1 : 2); }

__device__ __forceinline__ int route_class(const EvalArgs& a, int32_t s, int& est, int& d) {
    d = (int)(__ldg(a.soff + s + 1) - __ldg(a.soff + s));
    if (d <= kSmallMax) {
        est = d;
        return small_class(d);
    }
    const int nd = __ldg(a.ndist + s);
    est = min(d, nd + (nd >> 2) + 16);
    if (est <= kWarpEst && d <= kWarpMaxDeg) return 3;
    if (est <= kTeamEst && d <= kTeamMaxDeg) return 4;
    return 5;
}

// Append `s` (valid when cls >= 0) to its route list; warp-aggregated for the
// single-item classes.  Hub vertices append P (or R) items.
__device__ __forceinline__ void route_append(const EvalArgs& a, int cls, int32_t s, int est, int d) {
    const int lane = threadIdx.x & 31;
    const uint32_t act = __activemask();
#pragma unroll
    for (int c = 0; c < 5; ++c) {
        const uint32_t m = __ballot_sync(act, cls == c);
        if (!m) continue;
        const int leader = __ffs(m) - 1;
        int base = 0;
        if (lane == leader) base = atomicAdd(a.r.len + c, __popc(m));
        base = __shfl_sync(act, base, leader);
        if (cls == c) {
            const int idx = base + __popc(m & lanemask_lt());
            if (c < 3) {
                a.r.small[c][idx] = s;
            } else if (c == 3) {
                a.r.warp[idx] = s;
            } else {
                Item t = {s, 0, 1, 0, 1, -1, 0, 0};
                a.r.team[idx] = t;
            }
        }
    }
    if (cls == 5) {
        if (d > kSliceArcs * 2 && est <= kSliceEst) {
            const int R = (d + kSliceArcs - 1) / kSliceArcs;
            const int base = atomicAdd(a.r.len + kLenHub, R);
            const int cb = atomicAdd(a.r.len + kCandCursor, 1);
            const int gt = atomicAdd(a.r.len + kGtabCursor, 1 << kGlobalBits);
            for (int r = 0; r < R; ++r) {
                Item t = {s, 0, 1, r, R, cb, gt, 0};
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

// Frontier round: marked positions -> route lists (marks cleared).
__global__ void k_route_marked(EvalArgs a, uint8_t* __restrict__ mark, const int32_t* __restrict__ slot_of_pos,
                               int64_t n) {
    for (int64_t base = (blockIdx.x * (int64_t)blockDim.x) * 4; base < n; base += (int64_t)gridDim.x * blockDim.x * 4) {
        const int64_t p0 = base + (int64_t)threadIdx.x * 4;
        uint32_t word = 0;
        if (p0 + 4 <= n) {
            word = *reinterpret_cast<const uint32_t*>(mark + p0);
            if (word) *reinterpret_cast<uint32_t*>(mark + p0) = 0u;
        } else {
            for (int j = 0; j < 4 && p0 + j < n; ++j) {
                word |= (uint32_t)mark[p0 + j] << (8 * j);
                mark[p0 + j] = 0;
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int cls = -1, est = 0, d = 0;
            int32_t s = -1;
            if ((word >> (8 * j)) & 0xffu) {
                s = slot_of_pos[p0 + j];
                if (s >= 0) cls = route_class(a, s, est, d);
            }
            route_append(a, cls, s, est, d);
        }
    }
}

// ---------------------------------------------------------------------------
// thread per vertex
// ---------------------------------------------------------------------------
// MAXD = 4, 8 or 16: the degree class (O(MAXD^2) register compares).
// Dense mode sweeps slots [s_beg, s_end); list mode (s_beg < 0) reads the
// class's route list.
template <int WM, int TIE, int MAXD>
__global__ void __launch_bounds__(256) k_small(EvalArgs a, int32_t s_beg, int32_t s_end) {
    using A = typename Acc<WM>::T;
    constexpr int LIST = MAXD == 4 ? kLenS4 : (MAXD == 8 ? kLenS8 : kLenS16);
    const bool listed = s_beg < 0;
    const int32_t cnt = listed ? a.r.len[LIST] : (s_end - s_beg);
    const int32_t* list = a.r.small[LIST];
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        const int32_t s = listed ? list[i] : s_beg + i;
        const int32_t p = __ldg(a.spos + s);
        const uint32_t beg = __ldg(a.soff + s);
        const int d = (int)(__ldg(a.soff + s + 1) - beg);
        const int32_t thr = (p / a.bs) * a.bs;
        int32_t nbr[MAXD];
#pragma unroll
        for (int k = 0; k < MAXD; ++k) nbr[k] = (k < d) ? __ldg(a.snbr + beg + k) : 0;
        int32_t lab[MAXD];
        A w[MAXD];
#pragma unroll
        for (int k = 0; k < MAXD; ++k) {
            if (k < d) {
                lab[k] = read_label(a, nbr[k], thr);
                w[k] = arc_weight<WM>(a, beg + k);
            } else {
                lab[k] = kEmpty;
                w[k] = A(0);
            }
        }
        const uint32_t vtx = (TIE == kRandom) ? (uint32_t)__ldg(a.vid + p) : 0u;
        Cand<A> best = none_cand<A>();
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
                }
            }
        }
        arcs += d;
        ++verts;
        if (commit_label(a, p, best.lab, dchg, writes) && a.mark) {
            const int32_t nb = thr + a.bs;
#pragma unroll
            for (int k = 0; k < MAXD; ++k)
                if (k < d && nbr[k] >= nb) a.mark[nbr[k]] = 1;
        }
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

// ---------------------------------------------------------------------------
// warp per vertex
// ---------------------------------------------------------------------------
template <typename A> struct WarpTable {
    int32_t keys[1 << kWarpBits];
    A acc[1 << kWarpBits];
    uint16_t first[1 << kWarpBits];
    uint16_t touched[kWarpCap + 32];
};

// Sum of `w` over the lanes in `m` (all lanes call; result in every lane).
template <typename A> __device__ __forceinline__ A masked_sum(uint32_t m, A w) {
    A v = ((m >> (threadIdx.x & 31)) & 1u) ? w : A(0);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += shfl_xor_any(v, o);
    return v;
}

// Warp per vertex.  Tally first in a warp-wide register table (entry t lives
// in lane t: key, weight, first position; up to 32 distinct labels) -- after
// the first sweep most rows hold a handful of labels and this path needs no
// shared memory and no atomics.  A row with more distinct labels spills the
// register table into the warp's shared-memory hash and continues there.
template <int WM, int TIE>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_warp(EvalArgs a) {
    using A = typename Acc<WM>::T;
    constexpr int HB = 1 << kWarpBits;
    constexpr int U = 4;  // 32-arc chunks gathered per step
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpTable<A>* tab = reinterpret_cast<WarpTable<A>*>(smem_raw) + wib;
    for (int h = lane; h < HB; h += 32) tab->keys[h] = kEmpty;
    __syncwarp();

    const int32_t cnt = a.r.len[kLenWarp];
    const int32_t nwarps = gridDim.x * kWarpsPerBlock;
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;

    // insert one chunk's labels into the shared hash (leaders of equal-label groups)
    auto hash_chunk = [&](int32_t lab, A w, int k, int& ntouched) {
        const uint32_t grp = __match_any_sync(0xffffffffu, lab);
        const int leader = __ffs(grp) - 1;
        int h = -1;
        bool isnew = false;
        if (lab != kEmpty && lane == leader) {
            h = (int)slot_hash(lab, kWarpBits);
            while (true) {
                const int32_t cur = tab->keys[h];
                if (cur == lab) break;
                if (cur == kEmpty) {
                    const int32_t old = atomicCAS(&tab->keys[h], kEmpty, lab);
                    if (old == kEmpty) {
                        isnew = true;
                        tab->first[h] = (uint16_t)k;
                        tab->acc[h] = A(0);
                        break;
                    }
                    if (old == lab) break;
                }
                h = (h + 1) & (HB - 1);
            }
            // leaders hold distinct labels -> distinct slots: plain update
            if constexpr (WM == kUnit) tab->acc[h] += (A)__popc(grp);
        }
        if constexpr (WM != kUnit) {
            __syncwarp();
            const int hb = __shfl_sync(0xffffffffu, h, leader);
            if (lab != kEmpty) atomicAdd(&tab->acc[hb], w);
        }
        const uint32_t nb = __ballot_sync(0xffffffffu, isnew);
        if (isnew) {
            const int idx = ntouched + __popc(nb & lanemask_lt());
            if (idx < kWarpCap + 32) tab->touched[idx] = (uint16_t)h;
        }
        ntouched += __popc(nb);
        __syncwarp();
    };

    for (int32_t i = blockIdx.x * kWarpsPerBlock + wib; i < cnt; i += nwarps) {
        const int32_t s = a.r.warp[i];
        const int32_t p = __ldg(a.spos + s);
        const uint32_t beg = __ldg(a.soff + s);
        const int d = (int)(__ldg(a.soff + s + 1) - beg);
        const int32_t thr = (p / a.bs) * a.bs;
        // register table
        int32_t tkey = kEmpty;
        A tacc = A(0);
        uint32_t tfirst = 0;
        int K = 0;               // register entries in use (warp-uniform)
        bool hashed = false;     // spilled to the shared hash
        int ntouched = 0;
        bool overflow = false;
        for (int base = 0; base < d && !overflow; base += 32 * U) {
            int32_t nbr[U];
#pragma unroll
            for (int c = 0; c < U; ++c) {
                const int k = base + c * 32 + lane;
                nbr[c] = (k < d) ? __ldg(a.snbr + beg + k) : -1;
            }
            int32_t labv[U];
            A wv[U];
#pragma unroll
            for (int c = 0; c < U; ++c) {
                const int k = base + c * 32 + lane;
                labv[c] = (k < d) ? read_label(a, nbr[c], thr) : kEmpty;
                wv[c] = (k < d) ? arc_weight<WM>(a, beg + k) : A(0);
            }
#pragma unroll
            for (int c = 0; c < U; ++c) {
                if (base + c * 32 >= d) break;  // warp-uniform
                const int k0 = base + c * 32;
                int32_t lab = labv[c];
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
                    // more than 32 distinct labels: move the register table to
                    // the shared hash, then insert the rest of this chunk there
                    bool isnew = false;
                    int h = -1;
                    if (lane < K) {
                        h = (int)slot_hash(tkey, kWarpBits);
                        while (true) {
                            const int32_t old = atomicCAS(&tab->keys[h], kEmpty, tkey);
                            if (old == kEmpty) break;
                            h = (h + 1) & (HB - 1);
                        }
                        isnew = true;
                        tab->acc[h] = tacc;
                        tab->first[h] = (uint16_t)tfirst;
                    }
                    const uint32_t nb = __ballot_sync(0xffffffffu, isnew);
                    if (isnew) tab->touched[__popc(nb & lanemask_lt())] = (uint16_t)h;
                    ntouched = __popc(nb);
                    __syncwarp();
                    hashed = true;
                    if (!((pending >> lane) & 1u)) lab = kEmpty;
                }
                hash_chunk(lab, wv[c], k0 + lane, ntouched);
                if (ntouched > kWarpCap) {
                    overflow = true;
                    break;
                }
            }
        }
        if (overflow) {
            // too many distinct labels for this table: wipe it and hand the
            // vertex to the team kernel (launched after this one)
            for (int h = lane; h < HB; h += 32) tab->keys[h] = kEmpty;
            if (lane == 0) {
                const int idx = atomicAdd(a.r.len + kLenTeam, 1);
                Item t = {s, 0, 1, 0, 1, -1, 0, 0};
                a.r.team[idx] = t;
                a.ndist[s] = max(__ldg(a.ndist + s), 2 * kWarpEst);
            }
            __syncwarp();
            continue;
        }
        const uint32_t vtx = (TIE == kRandom) ? (uint32_t)__ldg(a.vid + p) : 0u;
        Cand<A> best = none_cand<A>();
        if (!hashed) {
            if (lane < K) best = make_cand<TIE, A>(tacc, tkey, tfirst, a.seed, a.sweep, vtx);
        } else {
            for (int t = lane; t < ntouched; t += 32) {
                const int h = tab->touched[t];
                Cand<A> c = make_cand<TIE, A>(tab->acc[h], tab->keys[h], tab->first[h], a.seed, a.sweep, vtx);
                if (better(c, best)) best = c;
            }
        }
        best = warp_best(best);
        if (hashed) {
            __syncwarp();
            for (int t = lane; t < ntouched; t += 32) tab->keys[tab->touched[t]] = kEmpty;
            __syncwarp();
        }
        bool changed = false;
        if (lane == 0) {
            arcs += d;
            ++verts;
            a.ndist[s] = hashed ? ntouched : K;
            changed = commit_label(a, p, best.lab, dchg, writes);
        }
        changed = __shfl_sync(0xffffffffu, changed, 0);
        if (changed && a.mark) mark_row(a, beg, d, thr, lane, 32);
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

// ---------------------------------------------------------------------------
// block (team) per work item
// ---------------------------------------------------------------------------
template <typename A, int TBITS> struct TeamTable {
    static constexpr int HB = 1 << TBITS;
    static constexpr int CAP = HB / 4 * 3;  // touched capacity; beyond it = overflow
    int32_t keys[HB];
    A acc[HB];
    uint32_t first[HB];
    uint16_t touched[CAP];
};

template <typename A> __device__ __forceinline__ unsigned long long to_bits(A w) {
    if constexpr (std::is_same<A, float>::value)
        return (unsigned long long)__float_as_uint(w);
    else
        return (unsigned long long)w;
}
template <typename A> __device__ __forceinline__ A from_bits(unsigned long long b) {
    if constexpr (std::is_same<A, float>::value)
        return __uint_as_float((uint32_t)b);
    else
        return (A)b;
}

// Find or insert `lab` in an open-addressing table of 2^bits keys (shared or
// global memory).  Returns -1 only when the table is full.
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

template <typename A> __device__ __forceinline__ void gacc_add(unsigned long long* acc, A w) {
    if constexpr (std::is_same<A, float>::value)
        atomicAdd(reinterpret_cast<float*>(acc), w);
    else
        atomicAdd(acc, (unsigned long long)w);
}
template <typename A> __device__ __forceinline__ A gacc_read(const unsigned long long* acc) {
    if constexpr (std::is_same<A, float>::value)
        return __ldcg(reinterpret_cast<const float*>(acc));
    else
        return (A)__ldcg(acc);
}

template <int WM, int TIE, int NT, int TBITS, bool DYNAMIC>
__global__ void __launch_bounds__(NT) k_team(EvalArgs a, int which) {
    using A = typename Acc<WM>::T;
    using Tab = TeamTable<A, TBITS>;
    constexpr int HB = Tab::HB;
    constexpr int CAP = Tab::CAP;
    constexpr int NW = NT / 32;
    constexpr int U = 2;
    constexpr int STACK = 40;
    constexpr int GHB = 1 << kGlobalBits;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Tab* tab = reinterpret_cast<Tab*>(smem_raw);
    __shared__ int32_t s_nt;
    __shared__ int32_t s_item;
    __shared__ int32_t s_flag;
    __shared__ int32_t s_last;
    __shared__ int32_t s_gnew;
    __shared__ int32_t s_sp;
    __shared__ uint32_t s_stack[STACK][2];  // (parts, want)
    __shared__ Cand<A> s_red[NW];

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    for (int h = tid; h < HB; h += NT) {
        tab->keys[h] = kEmpty;
        tab->acc[h] = A(0);
        tab->first[h] = 0xffffffffu;
    }
    const Item* items = which == kLenHub ? a.r.hub : a.r.team;
    const int cursor = which == kLenHub ? kHubCursor : kTeamCursor;
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    int32_t it = blockIdx.x;
    __syncthreads();
    const int32_t cnt = a.r.len[which];

    while (true) {
        if (DYNAMIC) {
            if (tid == 0) s_item = atomicAdd(a.r.len + cursor, 1);
            __syncthreads();
            it = s_item;
        }
        if (it >= cnt) break;
        const Item item = items[it];
        const int32_t s = item.s;
        const int32_t p = __ldg(a.spos + s);
        const uint32_t beg = __ldg(a.soff + s);
        const int d = (int)(__ldg(a.soff + s + 1) - beg);
        const int32_t thr = (p / a.bs) * a.bs;
        const uint32_t vtx = (TIE == kRandom) ? (uint32_t)__ldg(a.vid + p) : 0u;
        const int k_lo = (int)((long long)d * item.r / item.R);
        const int k_hi = (int)((long long)d * (item.r + 1) / item.R);
        const bool sliced = item.R > 1;
        int32_t* gkeys = sliced ? a.r.gkeys + item.gt : nullptr;
        uint32_t* gfirst = sliced ? a.r.gfirst + item.gt : nullptr;
        unsigned long long* gacc = sliced ? a.r.gacc + item.gt : nullptr;
        Cand<A> best = none_cand<A>();
        int distinct = 0;
        if (tid == 0) {
            s_sp = 1;
            s_stack[0][0] = (uint32_t)item.P;
            s_stack[0][1] = (uint32_t)item.q;
            s_gnew = 0;
        }
        __syncthreads();

        // ---- tally this item's arcs; the work stack splits overflowing passes ----
        while (true) {
            const int sp = s_sp;
            if (sp == 0) break;
            const uint32_t parts = s_stack[sp - 1][0], want = s_stack[sp - 1][1];
            __syncthreads();
            if (tid == 0) {
                s_sp = sp - 1;
                s_nt = 0;
            }
            __syncthreads();
            for (int base = k_lo + warp * 32 * U; base < k_hi; base += NT * U) {
                int32_t labv[U];
                A wv[U];
#pragma unroll
                for (int c = 0; c < U; ++c) {
                    const int k = base + c * 32 + lane;
                    int32_t lab = kEmpty;
                    A w = A(0);
                    if (k < k_hi) {
                        lab = read_label(a, __ldg(a.snbr + beg + k), thr);
                        w = arc_weight<WM>(a, beg + k);
                        if (parts > 1 && part_of(lab, parts) != want) lab = kEmpty;
                    }
                    labv[c] = lab;
                    wv[c] = w;
                }
#pragma unroll
                for (int c = 0; c < U; ++c) {
                    const int k = base + c * 32 + lane;
                    const int32_t lab = labv[c];
                    const uint32_t grp = __match_any_sync(0xffffffffu, lab);
                    const int leader = __ffs(grp) - 1;
                    int h = -1;
                    bool isnew = false;
                    if (lab != kEmpty && lane == leader) {
                        h = table_slot(tab->keys, lab, TBITS, isnew);
                        if (h >= 0) {
                            atomicMin(&tab->first[h], (uint32_t)k);
                            if constexpr (WM == kUnit) atomicAdd(&tab->acc[h], (A)__popc(grp));
                        }
                    }
                    if constexpr (WM != kUnit) {
                        const int hb = __shfl_sync(0xffffffffu, h, leader);
                        if (lab != kEmpty && hb >= 0) atomicAdd(&tab->acc[hb], wv[c]);
                    }
                    const uint32_t nb = __ballot_sync(0xffffffffu, isnew);
                    if (nb) {
                        int b0 = 0;
                        if (lane == 0) b0 = atomicAdd(&s_nt, __popc(nb));
                        b0 = __shfl_sync(0xffffffffu, b0, 0);
                        const int idx = b0 + __popc(nb & lanemask_lt());
                        if (isnew && idx < CAP) tab->touched[idx] = (uint16_t)h;
                    }
                }
                if (__shfl_sync(0xffffffffu, *(volatile int32_t*)&s_nt, 0) > CAP) break;  // overflowing
            }
            __syncthreads();
            const int nt = s_nt;
            const bool overflow = nt > CAP;
            if (!overflow) {
                // fold the touched entries into the candidate or the global slice table; wipe them
                for (int t = tid; t < nt; t += NT) {
                    const int h = tab->touched[t];
                    const int32_t key = tab->keys[h];
                    if (sliced) {
                        bool isnew = false;
                        const int g = table_slot(gkeys, key, kGlobalBits, isnew);
                        if (g >= 0) {
                            atomicMin(gfirst + g, tab->first[h]);
                            gacc_add<A>(gacc + g, tab->acc[h]);
                        }
                        if (isnew || g < 0) atomicAdd(&s_gnew, g < 0 ? (1 << 20) : 1);
                    } else {
                        Cand<A> c = make_cand<TIE, A>(tab->acc[h], key, tab->first[h], a.seed, a.sweep, vtx);
                        if (better(c, best)) best = c;
                    }
                    tab->keys[h] = kEmpty;
                    tab->acc[h] = A(0);
                    tab->first[h] = 0xffffffffu;
                }
                distinct += nt;
            } else {
                for (int h = tid; h < HB; h += NT) {
                    tab->keys[h] = kEmpty;
                    tab->acc[h] = A(0);
                    tab->first[h] = 0xffffffffu;
                }
            }
            __syncthreads();
            if (overflow && tid == 0) {
                for (int j = 3; j >= 0; --j) {
                    s_stack[s_sp][0] = parts * 4;
                    s_stack[s_sp][1] = want * 4 + j;
                    ++s_sp;
                }
            }
            __syncthreads();
        }

        // ---- merge ----
        // block reduce of this item's candidate (all threads get it)
        best = warp_best(best);
        if (lane == 0) s_red[warp] = best;
        __syncthreads();
        best = warp_best(lane < NW ? s_red[lane] : none_cand<A>());
        if (tid == 0) {
            s_flag = 0;
            s_last = 1;
            if (sliced) {
                if (s_gnew) atomicAdd(a.r.gcount + item.cb, s_gnew);
                __threadfence();
                s_last = atomicAdd(a.r.cand_done + item.cb, 1) == item.R - 1;
                if (s_last) __threadfence();
            } else if (item.P > 1) {
                HubCand hc;
                hc.w = to_bits<A>(best.w);
                hc.sec = best.sec;
                hc.ter = best.ter;
                hc.lab = best.lab;
                hc.nd = distinct;
                a.r.cand[item.cb + item.q] = hc;
                __threadfence();
                s_last = atomicAdd(a.r.cand_done + item.cb, 1) == item.P - 1;
                if (s_last) {
                    __threadfence();
                    distinct = 0;
                    best = none_cand<A>();
                    for (int j = 0; j < item.P; ++j) {
                        const HubCand* src = a.r.cand + item.cb + j;
                        Cand<A> o;
                        o.w = from_bits<A>(__ldcg(&src->w));
                        o.sec = __ldcg(&src->sec);
                        o.ter = __ldcg(&src->ter);
                        o.lab = __ldcg(&src->lab);
                        distinct += __ldcg(&src->nd);
                        if (better(o, best)) best = o;
                    }
                    a.r.cand_done[item.cb] = 0;
                }
            }
        }
        __syncthreads();
        if (sliced && s_last) {
            // last slice: argmax over the per-vertex global table, then wipe it
            const int gcount = __ldcg(a.r.gcount + item.cb);
            best = none_cand<A>();
            if (gcount <= kGlobalCap) {
                for (int g = tid; g < GHB; g += NT) {
                    const int32_t key = __ldcg(gkeys + g);
                    if (key == kEmpty) continue;
                    Cand<A> c = make_cand<TIE, A>(gacc_read<A>(gacc + g), key, __ldcg(gfirst + g), a.seed, a.sweep, vtx);
                    if (better(c, best)) best = c;
                }
            }
            for (int g = tid; g < GHB; g += NT) {
                gkeys[g] = kEmpty;
                gfirst[g] = 0xffffffffu;
                gacc[g] = 0ull;
            }
            best = warp_best(best);
            __syncthreads();
            if (lane == 0) s_red[warp] = best;
            __syncthreads();
            best = warp_best(lane < NW ? s_red[lane] : none_cand<A>());
            if (tid == 0) {
                distinct = gcount;
                a.r.cand_done[item.cb] = 0;
                a.r.gcount[item.cb] = 0;
                if (gcount > kGlobalCap) s_last = 2;  // global table overflowed: redo whole row below
            }
            __syncthreads();
            if (s_last == 2) {
                // rare slow path: this block recomputes the whole row with the
                // splitting stack (labels were underestimated)
                if (tid == 0) {
                    s_sp = 1;
                    s_stack[0][0] = 4;
                    s_stack[0][1] = 0;
                    s_stack[1][0] = 4;
                    s_stack[1][1] = 1;
                    s_stack[2][0] = 4;
                    s_stack[2][1] = 2;
                    s_stack[3][0] = 4;
                    s_stack[3][1] = 3;
                    s_sp = 4;
                }
                __syncthreads();
                best = none_cand<A>();
                distinct = 0;
                while (true) {
                    const int sp = s_sp;
                    if (sp == 0) break;
                    const uint32_t parts = s_stack[sp - 1][0], want = s_stack[sp - 1][1];
                    __syncthreads();
                    if (tid == 0) {
                        s_sp = sp - 1;
                        s_nt = 0;
                    }
                    __syncthreads();
                    for (int base = warp * 32; base < d; base += NT) {
                        const int k = base + lane;
                        int32_t lab = kEmpty;
                        A w = A(0);
                        if (k < d) {
                            lab = read_label(a, __ldg(a.snbr + beg + k), thr);
                            w = arc_weight<WM>(a, beg + k);
                            if (part_of(lab, parts) != want) lab = kEmpty;
                        }
                        bool isnew = false;
                        int h = -1;
                        if (lab != kEmpty) {
                            h = table_slot(tab->keys, lab, TBITS, isnew);
                            if (h >= 0) {
                                atomicMin(&tab->first[h], (uint32_t)k);
                                atomicAdd(&tab->acc[h], w);
                            }
                            if (isnew) atomicAdd(&s_nt, 1);
                        }
                        if (__shfl_sync(0xffffffffu, *(volatile int32_t*)&s_nt, 0) > CAP) break;
                    }
                    __syncthreads();
                    const bool overflow = s_nt > CAP;
                    // (slow path: full-table scan instead of a touched list)
                    for (int h = tid; h < HB; h += NT) {
                        const int32_t key = tab->keys[h];
                        if (key == kEmpty) continue;
                        if (!overflow) {
                            Cand<A> c = make_cand<TIE, A>(tab->acc[h], key, tab->first[h], a.seed, a.sweep, vtx);
                            if (better(c, best)) best = c;
                        }
                        tab->keys[h] = kEmpty;
                        tab->acc[h] = A(0);
                        tab->first[h] = 0xffffffffu;
                    }
                    if (!overflow) distinct += s_nt;
                    __syncthreads();
                    if (overflow && tid == 0) {
                        for (int j = 3; j >= 0; --j) {
                            s_stack[s_sp][0] = parts * 4;
                            s_stack[s_sp][1] = want * 4 + j;
                            ++s_sp;
                        }
                    }
                    __syncthreads();
                }
                best = warp_best(best);
                if (lane == 0) s_red[warp] = best;
                __syncthreads();
                best = warp_best(lane < NW ? s_red[lane] : none_cand<A>());
            }
        }
        if (tid == 0 && s_last) {
            arcs += d;
            ++verts;
            a.ndist[s] = distinct;
            s_flag = commit_label(a, p, best.lab, dchg, writes) ? 1 : 0;
        }
        __syncthreads();
        if (s_flag && a.mark) mark_row(a, beg, d, thr, tid, NT);
        if (!DYNAMIC) it += gridDim.x;
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

template <typename A> constexpr size_t warp_smem_bytes() { return sizeof(WarpTable<A>) * kWarpsPerBlock; }
template <typename A, int TBITS> constexpr size_t team_smem_bytes() { return sizeof(TeamTable<A, TBITS>); }

}  // namespace lp
