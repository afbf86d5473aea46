// lp_rak_kernels.cuh -- the RAK sweep kernels (the hot path).
//
// Replaces the body of the reference's sweep, rak.py:97-113 (_rak_seq) /
// :138-154 (_rak_par): for each vertex, accumulate the weights of its
// neighbours' labels, take the argmax under the tie rule, write the label
// and count the change.  Three degree bins, one kernel family each:
//
//   k_small  thread per vertex (2 <= deg <= 16): register tally, O(d^2)
//   k_warp   warp per vertex  (17..256): shared-memory open-addressing
//            hash, __match_any_sync groups equal labels in a 32-arc chunk so
//            one leader lane inserts per distinct label, argmax reduced with
//            __shfl_xor_sync
//   k_block  block per vertex (> 256): block-wide shared hash; hubs whose
//            distinct-label count exceeds the table are done in label-hash
//            partitions (multi-pass), overflow detected and retried
//
// Every kernel runs either densely over a slot range (round 1 of a sweep)
// or over a compacted frontier list (later rounds).  The changed-vertex
// count (rak.py:111-113) is fused: per-thread deltas, one atomic per warp.
#pragma once
#include "lp_common.cuh"

namespace lp {

struct EvalArgs {
    const uint32_t* __restrict__ soff;  // storage row offsets [S+1]
    const int32_t* __restrict__ snbr;   // neighbour positions
    const uint32_t* __restrict__ sw;    // arc weights (fixed-point u32 or float bits); null = unit
    const int32_t* __restrict__ spos;   // slot -> position
    const int32_t* __restrict__ vid;    // position -> vertex id
    const int32_t* __restrict__ L0;     // labels at sweep start (read-only in a sweep)
    int32_t* x;                         // working labels (read + written in place)
    uint8_t* mark;                      // next-round marks by position, null = no cross-batch deps
    int32_t* ndist;                     // per-slot distinct-label estimate (block bin)
    unsigned long long* counters;       // see kCtr* below
    int32_t bs;                         // batch size in positions
    int32_t bin;                        // degree bin of this launch (per-bin counters)
    uint32_t seed;
    uint32_t sweep;
};

// counters: [0] changed delta (reset per sweep), [1] label writes and [2] hub
// work cursor (reset per round), [4+bin] arcs scanned and [8+bin] vertices
// evaluated (accumulated over a run)
enum { kCtrChanged = 0, kCtrWrites = 1, kCtrCursor = 2, kCtrArcs = 4, kCtrVerts = 8, kCtrCount = 12 };

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
    // one atomic per warp per counter (all lanes reach this point)
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

// -------------------------------------------------------------------------
// thread per vertex
// -------------------------------------------------------------------------
constexpr int kSmallMax = 16;

template <int WM, int TIE>
__global__ void __launch_bounds__(256) k_small(EvalArgs a, const int32_t* __restrict__ list,
                                               const int32_t* __restrict__ list_len, int32_t s_beg,
                                               int32_t s_end) {
    using A = typename Acc<WM>::T;
    const int32_t cnt = list ? *list_len : (s_end - s_beg);
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += gridDim.x * blockDim.x) {
        const int32_t s = list ? list[i] : s_beg + i;
        const int32_t p = __ldg(a.spos + s);
        const uint32_t beg = __ldg(a.soff + s);
        const int d = (int)(__ldg(a.soff + s + 1) - beg);
        const int32_t thr = (p / a.bs) * a.bs;
        int32_t lab[kSmallMax];
        A w[kSmallMax];
#pragma unroll
        for (int k = 0; k < kSmallMax; ++k) {
            if (k < d) {
                lab[k] = read_label(a, __ldg(a.snbr + beg + k), thr);
                w[k] = arc_weight<WM>(a, beg + k);
            } else {
                lab[k] = kEmpty;
                w[k] = A(0);
            }
        }
        const uint32_t vtx = (TIE == kRandom) ? (uint32_t)__ldg(a.vid + p) : 0u;
        Cand<A> best = none_cand<A>();
#pragma unroll
        for (int i = 0; i < kSmallMax; ++i) {
            if (i < d) {
                bool dup = false;
                A sum = A(0);
#pragma unroll
                for (int j = 0; j < kSmallMax; ++j) {
                    const bool eq = lab[j] == lab[i];
                    dup |= (j < i) & eq;
                    if (eq) sum += w[j];
                }
                if (!dup) {
                    Cand<A> c = make_cand<TIE, A>(sum, lab[i], (uint32_t)i, a.seed, a.sweep, vtx);
                    if (better(c, best)) best = c;
                }
            }
        }
        arcs += d;
        ++verts;
        const int32_t old = a.x[p];
        if (best.lab != old) {
            a.x[p] = best.lab;
            const int32_t l0 = __ldg(a.L0 + p);
            dchg += (long long)(best.lab != l0) - (long long)(old != l0);
            ++writes;
            if (a.mark) {
                const int32_t nb = thr + a.bs;
                for (int k = 0; k < d; ++k) {
                    const int32_t u = __ldg(a.snbr + beg + k);
                    if (u >= nb) a.mark[u] = 1;
                }
            }
        }
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

// -------------------------------------------------------------------------
// warp per vertex
// -------------------------------------------------------------------------
constexpr int kWarpMax = 256;      // max degree handled by a warp
constexpr int kWarpHashBits = 9;   // 512-slot table: load factor <= 0.5
constexpr int kWarpsPerBlock = 4;

template <typename A> struct WarpTable {
    int32_t keys[1 << kWarpHashBits];
    A acc[1 << kWarpHashBits];
    uint32_t first[1 << kWarpHashBits];
    int16_t touched[kWarpMax];
};

template <int WM, int TIE>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_warp(EvalArgs a, const int32_t* __restrict__ list,
                                                              const int32_t* __restrict__ list_len, int32_t s_beg,
                                                              int32_t s_end) {
    using A = typename Acc<WM>::T;
    constexpr int HB = 1 << kWarpHashBits;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpTable<A>* tab = reinterpret_cast<WarpTable<A>*>(smem_raw) + wib;
    for (int h = lane; h < HB; h += 32) tab->keys[h] = kEmpty;
    __syncwarp();

    const int32_t cnt = list ? *list_len : (s_end - s_beg);
    const int32_t nwarps = gridDim.x * kWarpsPerBlock;
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    for (int32_t i = blockIdx.x * kWarpsPerBlock + wib; i < cnt; i += nwarps) {
        const int32_t s = list ? list[i] : s_beg + i;
        const int32_t p = __ldg(a.spos + s);
        const uint32_t beg = __ldg(a.soff + s);
        const int d = (int)(__ldg(a.soff + s + 1) - beg);
        const int32_t thr = (p / a.bs) * a.bs;
        int ntouched = 0;
        // gather 64 arcs per step (two loads in flight per lane), insert per 32
        for (int base = 0; base < d; base += 64) {
            int32_t labv[2];
            A wv[2];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int k = base + c * 32 + lane;
                if (k < d) {
                    labv[c] = read_label(a, __ldg(a.snbr + beg + k), thr);
                    wv[c] = arc_weight<WM>(a, beg + k);
                } else {
                    labv[c] = kEmpty;
                    wv[c] = A(0);
                }
            }
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int k = base + c * 32 + lane;
                const int32_t lab = labv[c];
                const uint32_t grp = __match_any_sync(0xffffffffu, lab);
                const int leader = __ffs(grp) - 1;
                int h = -1;
                bool isnew = false;
                if (lab != kEmpty && lane == leader) {
                    h = (int)slot_hash(lab, kWarpHashBits);
                    while (true) {
                        const int32_t old = atomicCAS(&tab->keys[h], kEmpty, lab);
                        if (old == kEmpty) {
                            isnew = true;
                            tab->first[h] = (uint32_t)k;
                            tab->acc[h] = A(0);
                            break;
                        }
                        if (old == lab) break;
                        h = (h + 1) & (HB - 1);
                    }
                    if constexpr (WM == kUnit) tab->acc[h] += (A)__popc(grp);
                }
                if constexpr (WM != kUnit) {
                    __syncwarp();
                    const int hb = __shfl_sync(0xffffffffu, h, leader);
                    if (lab != kEmpty) atomicAdd(&tab->acc[hb], wv[c]);
                }
                const uint32_t nb = __ballot_sync(0xffffffffu, isnew);
                if (isnew) tab->touched[ntouched + __popc(nb & lanemask_lt())] = (int16_t)h;
                ntouched += __popc(nb);
                __syncwarp();  // table updates of this chunk visible to the next one
            }
        }
        __syncwarp();
        const uint32_t vtx = (TIE == kRandom) ? (uint32_t)__ldg(a.vid + p) : 0u;
        Cand<A> best = none_cand<A>();
        for (int t = lane; t < ntouched; t += 32) {
            const int h = tab->touched[t];
            Cand<A> c = make_cand<TIE, A>(tab->acc[h], tab->keys[h], tab->first[h], a.seed, a.sweep, vtx);
            if (better(c, best)) best = c;
        }
        best = warp_best(best);
        __syncwarp();
        for (int t = lane; t < ntouched; t += 32) tab->keys[tab->touched[t]] = kEmpty;
        __syncwarp();
        if (lane == 0) {
            arcs += d;
            ++verts;
        }
        const int32_t old = a.x[p];
        if (best.lab != old) {  // warp-uniform
            if (lane == 0) {
                a.x[p] = best.lab;
                const int32_t l0 = __ldg(a.L0 + p);
                dchg += (long long)(best.lab != l0) - (long long)(old != l0);
                ++writes;
            }
            if (a.mark) {
                const int32_t nb = thr + a.bs;
                for (int k = lane; k < d; k += 32) {
                    const int32_t u = __ldg(a.snbr + beg + k);
                    if (u >= nb) a.mark[u] = 1;
                }
            }
        }
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

// -------------------------------------------------------------------------
// block per vertex
// -------------------------------------------------------------------------
template <typename A, int HBITS> struct BlockTable {
    static constexpr int HB = 1 << HBITS;
    static constexpr int CAP = HB / 4 * 3;  // touched-list capacity; beyond it = overflow
    int32_t keys[HB];
    A acc[HB];
    uint32_t first[HB];
    int32_t touched[CAP];
};

template <int WM, int TIE, int HBITS, int NT, bool DYNAMIC>
__global__ void __launch_bounds__(NT) k_block(EvalArgs a, const int32_t* __restrict__ list,
                                              const int32_t* __restrict__ list_len, int32_t s_beg,
                                              int32_t s_end) {
    using A = typename Acc<WM>::T;
    using Tab = BlockTable<A, HBITS>;
    constexpr int HB = Tab::HB;
    constexpr int CAP = Tab::CAP;
    constexpr int NW = NT / 32;
    constexpr int USABLE = HB / 2;  // distinct labels planned per pass
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Tab* tab = reinterpret_cast<Tab*>(smem_raw);
    __shared__ int32_t s_nt;
    __shared__ int32_t s_ovf;
    __shared__ int32_t s_item;
    __shared__ int32_t s_flag;
    __shared__ Cand<A> s_red[NW];

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    for (int h = tid; h < HB; h += NT) {
        tab->keys[h] = kEmpty;
        tab->acc[h] = A(0);
        tab->first[h] = 0xffffffffu;
    }
    const int32_t cnt = list ? *list_len : (s_end - s_beg);
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    int32_t it = blockIdx.x;
    while (true) {
        if (DYNAMIC) {
            if (tid == 0) s_item = (int32_t)atomicAdd(a.counters + kCtrCursor, 1ull);
            __syncthreads();
            it = s_item;
        } else {
            __syncthreads();
        }
        if (it >= cnt) break;
        const int32_t s = list ? list[it] : s_beg + it;
        const int32_t p = __ldg(a.spos + s);
        const uint32_t beg = __ldg(a.soff + s);
        const int d = (int)(__ldg(a.soff + s + 1) - beg);
        const int32_t thr = (p / a.bs) * a.bs;
        const uint32_t vtx = (TIE == kRandom) ? (uint32_t)__ldg(a.vid + p) : 0u;
        int est = d;
        if (a.ndist) est = min(d, max(1, __ldg(a.ndist + s) + (__ldg(a.ndist + s) >> 2)));
        uint32_t parts = (uint32_t)max(1, (est + USABLE - 1) / USABLE);
        Cand<A> best;
        int distinct;
        while (true) {  // retried with more partitions on overflow
            best = none_cand<A>();
            distinct = 0;
            bool overflow = false;
            for (uint32_t q = 0; q < parts; ++q) {
                if (tid == 0) {
                    s_nt = 0;
                    s_ovf = 0;
                }
                __syncthreads();
                for (int base = warp * 64; base < d; base += NT * 2) {
                    int32_t labv[2];
                    A wv[2];
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int k = base + c * 32 + lane;
                        int32_t lab = kEmpty;
                        A w = A(0);
                        if (k < d) {
                            lab = read_label(a, __ldg(a.snbr + beg + k), thr);
                            w = arc_weight<WM>(a, beg + k);
                            if (parts > 1 && part_of(lab, parts) != q) lab = kEmpty;
                        }
                        labv[c] = lab;
                        wv[c] = w;
                    }
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const int k = base + c * 32 + lane;
                        const int32_t lab = labv[c];
                        const uint32_t grp = __match_any_sync(0xffffffffu, lab);
                        const int leader = __ffs(grp) - 1;
                        int h = -1;
                        bool isnew = false;
                        if (lab != kEmpty && lane == leader && !*(volatile int32_t*)&s_ovf) {
                            h = (int)slot_hash(lab, HBITS);
                            for (int probe = 0; probe < HB; ++probe) {
                                const int32_t old = atomicCAS(&tab->keys[h], kEmpty, lab);
                                if (old == kEmpty) {
                                    isnew = true;
                                    break;
                                }
                                if (old == lab) break;
                                h = (h + 1) & (HB - 1);
                            }
                            atomicMin(&tab->first[h], (uint32_t)k);
                            if constexpr (WM == kUnit) atomicAdd(&tab->acc[h], (A)__popc(grp));
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
                            if (isnew) {
                                const int idx = b0 + __popc(nb & lanemask_lt());
                                if (idx < CAP)
                                    tab->touched[idx] = h;
                                else
                                    s_ovf = 1;
                            }
                        }
                    }
                }
                __syncthreads();
                const int nt = s_nt;
                if (s_ovf || nt > CAP) {
                    overflow = true;
                    // entries past CAP are not in the touched list: wipe everything
                    for (int h = tid; h < HB; h += NT) {
                        tab->keys[h] = kEmpty;
                        tab->acc[h] = A(0);
                        tab->first[h] = 0xffffffffu;
                    }
                    __syncthreads();
                    break;
                }
                for (int t = tid; t < nt; t += NT) {
                    const int h = tab->touched[t];
                    Cand<A> c = make_cand<TIE, A>(tab->acc[h], tab->keys[h], tab->first[h], a.seed, a.sweep, vtx);
                    if (better(c, best)) best = c;
                }
                distinct += nt;
                __syncthreads();
                for (int t = tid; t < nt; t += NT) {
                    const int h = tab->touched[t];
                    tab->keys[h] = kEmpty;
                    tab->acc[h] = A(0);
                    tab->first[h] = 0xffffffffu;
                }
            }
            if (!overflow) break;
            parts *= 4;
        }
        best = warp_best(best);
        if (lane == 0) s_red[warp] = best;
        __syncthreads();
        if (warp == 0) {
            Cand<A> c = lane < NW ? s_red[lane] : none_cand<A>();
            c = warp_best(c);
            if (lane == 0) {
                const int32_t old = a.x[p];
                s_flag = 0;
                if (c.lab != old) {
                    a.x[p] = c.lab;
                    const int32_t l0 = __ldg(a.L0 + p);
                    dchg += (long long)(c.lab != l0) - (long long)(old != l0);
                    ++writes;
                    s_flag = 1;
                }
                arcs += d;  // algorithmic arcs (multi-pass re-reads not counted)
                ++verts;
                if (a.ndist) a.ndist[s] = distinct;
            }
        }
        __syncthreads();
        if (s_flag && a.mark) {
            const int32_t nb = thr + a.bs;
            for (int k = tid; k < d; k += NT) {
                const int32_t u = __ldg(a.snbr + beg + k);
                if (u >= nb) a.mark[u] = 1;
            }
        }
        if (!DYNAMIC) it += gridDim.x;
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

template <typename A> constexpr size_t warp_smem_bytes() { return sizeof(WarpTable<A>) * kWarpsPerBlock; }
template <typename A, int HBITS> constexpr size_t block_smem_bytes() { return sizeof(BlockTable<A, HBITS>); }

}  // namespace lp
