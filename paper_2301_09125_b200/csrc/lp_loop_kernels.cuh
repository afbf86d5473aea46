// lp_loop_kernels.cuh -- the frontier loop: many rounds of the sweep's
// fixed-point iteration in ONE cooperative launch.
//
// The exact schedules end every sweep with a tail of frontier
// rounds that each re-evaluate a few hundred rows, and on small graphs
// (BASELINE config 0: planted n = 100k) every round is that small: the cost
// is launch latency and the host round trip, not work.  k_frontier_loop keeps
// the round loop on the device: a resident grid (cudaLaunchCooperativeKernel)
// walks the mark queue with one warp per row -- margin test, fused label
// gather, tally in the warp's shared-memory table, argmax under the tie rule,
// commit, marks on the later-batch neighbours with the queue append on a
// mark's 0 -> nonzero transition -- then meets at a grid barrier and starts on
// the queue the round just built.  It returns when a round queues nothing
// (the sweep's fixed point), or hands the queue back to the class kernels
// when it holds rows this kernel does not take (longer than the warp table's
// capacity) or grows past the caller's bound.
//
// SLPA's speaking rounds run through the same loop (the spoken label is drawn from the
// speaker's memory, loop_label).
// Same evaluation as the class kernels (reference: _rak_seq's tally and
// _pick_from_tally, rak.py:57-116): every label of the row is tallied
// (first-sweep singleton flags are not used: a neighbour in a later batch
// contributes its sweep-start label), ties at the maximum go to the earliest
// arc / the smallest label / the largest tie hash, the exact lead over the
// runner-up is recorded for the margin test.
#pragma once
#include "lp_rak_kernels.cuh"

namespace lp {

constexpr int kLoopBits = 9;                               // 512-slot table per warp
constexpr int kLoopMaxDeg = (1 << kLoopBits) / 4 * 3;      // rows up to 384 arcs can never overflow it
constexpr int kLoopLongDeg = 2048;                         // frontier rounds also try rows up to this long: a
                                                           // late sweep's rows hold few distinct labels
constexpr int kLoopWarps = 8;

struct LoopCtl {
    unsigned int bar;   // grid barrier arrivals (monotonic)
    int32_t len[3];     // rotating queue lengths: round r reads len[r % 3], appends to len[(r + 1) % 3]
    int32_t out_buf;    // which of the two queues holds the unfinished queue (0 / 1)
    int32_t out_len;    // its length; 0 = the round queued nothing (fixed point)
    int32_t rounds;     // rounds run
    int32_t leftover[2];  // rows handed back unevaluated (longer than kLoopMaxDeg), by round parity
};

// Label that arc k of listener v's row contributes (read through L2: other SMs write x inside the
// launch).  RAK: the neighbour's working label if it is in an earlier batch, else its sweep-start
// label (gather_label).  SLPA (a.slots): the speaker's draw from its memory (k_gather_pieces,
// slpa.py:76-77) -- slot t, the one this round appends, lives in x.
__device__ __forceinline__ int32_t loop_label(const EvalArgs& a, uint32_t nb, int32_t v, int k) {
    const int32_t u = (int32_t)(nb >> 2);
    if (a.slots) {
        const uint32_t t = a.sweep;
        const uint32_t filled = t + ((nb & kEarlier) ? 1u : 0u);
        const uint32_t q = speak_hash(a.seed, t, (uint32_t)v, (uint32_t)k) % filled;
        return q == t ? __ldcg(a.x + u) : __ldg(a.slots + (size_t)u * a.T + q);
    }
    return (nb & kEarlier) ? __ldcg(a.x + u) : __ldg(a.L0 + u);
}

template <int WM> struct LoopTable {
    STable<WM, kLoopBits> t;
    uint16_t touched[kLoopMaxDeg + 32];
};
template <int WM> constexpr size_t loop_smem_bytes() { return sizeof(LoopTable<WM>) * kLoopWarps; }

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// every block of the (co-resident) grid arrives; epoch counts the barriers passed
__device__ __forceinline__ void loop_barrier(unsigned int* bar, unsigned int& epoch) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        const unsigned int target = (epoch + 1u) * gridDim.x;
        while (ld_acquire_u32(bar) < target) __nanosleep(32);
        __threadfence();
    }
    __syncthreads();
    ++epoch;
}

// list0 / list0_len (or list0_cnt when null): the first round's queue (the mark queue the class kernels left, or -- dense --
// every vertex in visit order); q[0] / q[1]: the two queues the rounds alternate between, q[first_dst]
// the first round's output (!= list0).
// dense: the first round evaluates unmarked rows (no margin test, marks untouched).
template <int WM, int TIE>
__global__ void __launch_bounds__(kLoopWarps * 32) k_frontier_loop(EvalArgs a, const int32_t* __restrict__ list0,
                                                                   const int32_t* list0_len, int list0_cnt, int32_t* q0,
                                                                   int32_t* q1,
                                                                   int first_dst, const int32_t* __restrict__ slot_of,
                                                                   LoopCtl* ctl, int32_t* mq_len, int dense,
                                                                   int max_queue, int max_rounds) {
    using A = typename Acc<WM>::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    LoopTable<WM>* tab = reinterpret_cast<LoopTable<WM>*>(smem_raw) + wib;
    for (int h = lane; h < (1 << kLoopBits); h += 32) tab->t.init(h);
    __syncwarp();
    const int gw = blockIdx.x * kLoopWarps + wib;
    const int nw = gridDim.x * kLoopWarps;
    long long dchg = 0, arcs = 0, writes = 0, verts = 0;
    unsigned int epoch = 0;
    int cnt = list0_len ? *list0_len : list0_cnt;
    const int32_t* src = list0;
    int dst_i = first_dst;
    int r = 0;
    while (true) {
        int32_t* dst = dst_i ? q1 : q0;
        int32_t* dst_len = ctl->len + (r + 1) % 3;
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->len[(r + 2) % 3] = 0;  // (idle this round: next round's output)
        const bool first_dense = dense && r == 0;
        for (int i = gw; i < cnt; i += nw) {
            const int32_t v = __ldcg(src + i);
            const int32_t s = __ldg(slot_of + v);
            if (s < 0) continue;  // (an isolated vertex of the dense list)
            const uint32_t beg = __ldg(a.soff + s);
            const int d = (int)(__ldg(a.soff + s + 1) - beg);
            const bool ours = d <= (first_dense ? kLoopMaxDeg : kLoopLongDeg);
            if (first_dense && !ours) {
                // not this kernel's row, unmarked: mark it so that the class kernels route it
                // (unless a neighbour's mark has queued it already)
                if (lane == 0) {
                    if (atomicAdd(a.mark + v, 1ull) == 0ull) dst[atomicAdd(dst_len, 1)] = v;
                    atomicAdd(&ctl->leftover[r & 1], 1);
                }
                continue;
            }
            unsigned long long delta0 = 0ull;  // (the mark taken from v, should the row go back)
            if (!first_dense) {
                // margin test on the weight that changed since v's last evaluation (k_route_queue);
                // fetch-and-clear: a concurrent mark either lands before (counted in delta, its label
                // write is visible below) or after (0 -> nonzero: the marker queues v again)
                unsigned long long delta = 0ull;
                if (lane == 0) delta = atomicExch(a.mark + v, 0ull);
                delta = __shfl_sync(0xffffffffu, delta, 0);
                delta0 = delta;
                __threadfence();
                if (a.gap) {
                    const unsigned long long gp = __ldcg(a.gap + s);
                    if (gp > 2ull * delta) {
                        if (lane == 0) a.gap[s] = gp - 2ull * delta;
                        continue;
                    }
                }
                if (!ours) {
                    // a long row that needs its evaluation: the mark goes back and the row into the
                    // next queue for the class kernels (a marker that found the mark cleared has
                    // queued it already)
                    if (lane == 0) {
                        if (atomicAdd(a.mark + v, delta ? delta : 1ull) == 0ull) dst[atomicAdd(dst_len, 1)] = v;
                        atomicAdd(&ctl->leftover[r & 1], 1);
                    }
                    continue;
                }
            }
            // ---- tally ----
            int ntouched = 0;
            bool overflow = false;
            for (int base = 0; base < d; base += 32) {
                const int k = base + lane;
                int32_t lab = kEmpty;
                A w = A(0);
                if (k < d) {
                    lab = loop_label(a, __ldg(a.snbr + beg + k), v, k);
                    w = arc_weight<WM>(a, beg + k);
                }
                bool full = false;
                const int h = insert_chunk<WM, kLoopBits>(tab->t, lab, w, true, full);
                const uint32_t nb = __ballot_sync(0xffffffffu, h >= 0);
                if (h >= 0) {
                    const int idx = ntouched + __popc(nb & lanemask_lt());
                    if (idx < kLoopMaxDeg + 32) tab->touched[idx] = (uint16_t)h;
                }
                ntouched += __popc(nb);
                __syncwarp();
                if (ntouched > kLoopMaxDeg || __any_sync(0xffffffffu, full)) {
                    overflow = true;
                    break;
                }
            }
            if (overflow) {
                // more distinct labels than the warp table takes: wipe it, the class kernels
                // evaluate the row (mark restored as for a row that is not ours)
                for (int h = lane; h < (1 << kLoopBits); h += 32) tab->t.init(h);
                __syncwarp();
                if (lane == 0) {
                    if (atomicAdd(a.mark + v, delta0 ? delta0 : 1ull) == 0ull) dst[atomicAdd(dst_len, 1)] = v;
                    atomicAdd(&ctl->leftover[r & 1], 1);
                }
                continue;
            }
            const uint32_t vtx = (uint32_t)v;
            const Best<A> b = table_argmax<WM, TIE, kLoopBits, 1>(tab->t, tab->touched, ntouched, lane, a.seed, a.sweep,
                                                                   vtx, nullptr);
            int32_t winner = b.lab;
            if (b.mult > 1) {
                // several labels tie at the maximum: the earliest in scan order wins (a label that
                // moved since the tally finds no entry; its writer marks this row again)
                winner = -1;
                for (int base = 0; base < d && winner < 0; base += 32) {
                    const int k = base + lane;
                    bool ok = false;
                    int32_t lab = kEmpty;
                    if (k < d) {
                        lab = loop_label(a, __ldg(a.snbr + beg + k), v, k);
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
            bool changed = false;
            if (lane == 0) {
                arcs += d;
                ++verts;
                A total;
                if constexpr (WM == kUnit)
                    total = (A)d;
                else if constexpr (WM == kFixed)
                    total = (A)__ldg(a.swsum + s);
                else
                    total = A(0);
                const bool maj = WM != kFloat && b.w + b.w > total;
                a.ndist[s] = ntouched | (maj ? kMajBit : 0);
                store_lead<A>(a, s, b.w, b.w2);
                changed = commit_label_known(a, v, winner, __ldcg(a.x + v), __ldg(a.L0 + v), dchg, writes);
                if (changed) __threadfence();  // the label before its marks
            }
            changed = __shfl_sync(0xffffffffu, changed, 0);
            if (changed && a.mark) {
                for (int base = 0; base < d; base += 32) {
                    const int k = base + lane;
                    bool win = false;
                    int32_t u = 0;
                    if (k < d) {
                        const uint32_t nb = __ldg(a.snbr + beg + k);
                        u = (int32_t)(nb >> 2);
                        win = (nb & kLater) && atomicAdd(a.mark + u, mark_weight(a, beg + k)) == 0ull;
                    }
                    const uint32_t bal = __ballot_sync(0xffffffffu, win);
                    if (bal) {
                        int b0 = 0;
                        if (lane == 0) b0 = atomicAdd(dst_len, __popc(bal));
                        b0 = __shfl_sync(0xffffffffu, b0, 0);
                        if (win) dst[b0 + __popc(bal & lanemask_lt())] = u;
                    }
                }
            }
        }
        loop_barrier(&ctl->bar, epoch);
        const int next_cnt = __ldcg(dst_len);
        // (by parity: a block already in the next round counts into the other word)
        const int left = __ldcg(&ctl->leftover[r & 1]);
        ++r;
        if (next_cnt == 0 || left > 0 || next_cnt > max_queue || r >= max_rounds) {
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                ctl->out_buf = dst_i;
                ctl->out_len = next_cnt;
                ctl->rounds = r;
                mq_len[dst_i] = next_cnt;
                mq_len[dst_i ^ 1] = 0;
            }
            break;
        }
        src = dst;
        cnt = next_cnt;
        dst_i ^= 1;
    }
    flush_counters(a, dchg, arcs, writes, verts);
}

}  // namespace lp
