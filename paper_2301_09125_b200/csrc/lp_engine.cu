// lp_engine.cu -- graph handle, plan builder, sweep driver and C-ABI.
//
// Reference mapping:
//   lp_graph_create  <- the Graph arrays handed to the numba kernels
//                       (graph.py:44-50; rak.py:177-192)
//   lp_rak_run       <- rak_detect's timed region (rak.py:172-193): the
//                       sweep loop of _rak_seq / _rak_par with the
//                       tolerance test `changed <= tolerance * n`
//                       (rak.py:114-115) and the iteration count semantics
//                       (rak.py:94-95)
//
// Schedule.  The visit order is cut into B batches of
// bs = ceil(n/B) positions.  A vertex reads the current-sweep label of
// neighbours in earlier batches and the sweep-start label of the others.
// B = n is the reference's in-place asynchronous sweep; B = 1 is a Jacobi
// sweep.  For B > 1 the sweep is solved as the unique fixed point of that
// triangular system: round 1 evaluates every vertex in place, and a vertex
// whose label changes marks its later-batch neighbours for re-evaluation in
// the next round, until a round marks nothing.  Whatever a vertex read in a
// round, it is re-evaluated if any earlier-batch neighbour changed after its
// read, so the final labels are exactly those of the sequential batched
// sweep -- for B = n, bit-identical to rak._rak_seq.
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/labelprop_cuda.h"
#include "lp_common.cuh"
#include "lp_host.h"
#include "lp_rak_kernels.cuh"

using namespace lp;

// ---------------------------------------------------------------------------
// bins
// ---------------------------------------------------------------------------
enum Bin : int { kBinHub = 0, kBinLarge = 1, kBinMid = 2, kBinSmall = 3, kBinIdle = 4, kNumBins = 4 };
constexpr int kHubMin = 2048;   // deg > kHubMin: hub kernel (8K table, multi-pass)
constexpr int kLargeMin = kWarpMax;  // deg > 256: block kernel (4K table)
constexpr int kHubBits = 13, kHubThreads = 512;
constexpr int kLargeBits = 12, kLargeThreads = 256;

#define LP_CK(call)                                                                         \
    do {                                                                                    \
        cudaError_t _e = (call);                                                            \
        if (_e != cudaSuccess) {                                                            \
            lp_set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__, __LINE__, \
                         cudaGetErrorString(_e));                                           \
            return LP_ERR_CUDA;                                                             \
        }                                                                                   \
    } while (0)

template <typename T> static cudaError_t dalloc(T** p, size_t count, int64_t* bytes) {
    *bytes += (int64_t)(count * sizeof(T));
    return cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
}

struct Plan {
    bool valid = false;
    bool custom_order = false;
    uint32_t seed = 0;
    uint64_t order_hash = 0;
    int32_t* vid = nullptr;          // position -> vertex
    int32_t* pos = nullptr;          // vertex -> position
    int32_t* spos = nullptr;         // slot -> position (n entries; first S active)
    int32_t* slot_of_pos = nullptr;  // position -> slot or -1
    uint32_t* soff = nullptr;        // [S+1]
    int32_t* snbr = nullptr;         // [m_active]
    uint32_t* sw = nullptr;          // [m_active] or null
    int32_t* ndist = nullptr;        // [S]
    int64_t S = 0;
    int64_t m_active = 0;
    int32_t bin_beg[kNumBins + 1] = {0, 0, 0, 0, 0};
};

struct lp_graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int64_t n = 0, m = 0;
    int64_t max_degree = 0;
    int wmode = kUnit;
    int fixed_shift = 0;
    int64_t bytes = 0;
    // original CSR (device, int32)
    uint32_t* off = nullptr;
    int32_t* nbr = nullptr;
    uint32_t* w = nullptr;  // converted weights (fixed-point or float bits)
    Plan plan;
    // run state
    int32_t* labA = nullptr;
    int32_t* labB = nullptr;
    int32_t* cur = nullptr;  // the buffer holding the latest labels
    uint8_t* mark = nullptr;
    int32_t* lists = nullptr;  // kNumBins frontier lists of n entries
    int32_t* list_len = nullptr;  // kNumBins
    unsigned long long* counters = nullptr;
    int64_t* out64 = nullptr;
    int32_t* h_list_len = nullptr;          // pinned
    unsigned long long* h_counters = nullptr;  // pinned
    void* cub_tmp = nullptr;
    size_t cub_tmp_bytes = 0;
    int num_sms = 148;
    bool labels_valid = false;
    std::vector<cudaEvent_t> event_pool;
};

// ---------------------------------------------------------------------------
// setup kernels
// ---------------------------------------------------------------------------
__global__ void k_i64_to_u32(const int64_t* __restrict__ in, uint32_t* __restrict__ out, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)in[i];
}

// neighbours -> int32 with range check; bad[0] counts out-of-range ids
__global__ void k_nbr_convert(const int64_t* __restrict__ in, int32_t* __restrict__ out, int64_t count, int64_t n,
                              unsigned long long* bad) {
    unsigned long long nbad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = in[i];
        nbad += (v < 0 || v >= n);
        out[i] = (int32_t)v;
    }
    if (nbad) atomicAdd(bad, nbad);
}

// weight analysis: [0] #(w != 1), [1] #(not float32-exact or not positive finite),
// [2] min frexp exponent (biased +2048), [3] max frexp exponent (biased)
__global__ void k_weight_scan(const double* __restrict__ w, int64_t count, unsigned long long* stat) {
    unsigned long long not_one = 0, bad = 0;
    int emin = 1 << 20, emax = -(1 << 20);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = w[i];
        not_one += (x != 1.0);
        const float f = (float)x;
        if (!(x > 0.0) || !isfinite(x) || (double)f != x) {
            ++bad;
        } else {
            int e;
            frexp(x, &e);
            emin = min(emin, e);
            emax = max(emax, e);
        }
    }
    if (not_one) atomicAdd(stat + 0, not_one);
    if (bad) atomicAdd(stat + 1, bad);
    if (emin != (1 << 20)) {
        atomicMin(stat + 2, (unsigned long long)(emin + 2048));
        atomicMax(stat + 3, (unsigned long long)(emax + 2048));
    }
}

__global__ void k_weight_convert(const double* __restrict__ w, uint32_t* __restrict__ out, int64_t count, int mode,
                                 int shift) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = w[i];
        out[i] = (mode == kFixed) ? (uint32_t)ldexp(x, shift) : __float_as_uint((float)x);
    }
}

__global__ void k_degree_max(const uint32_t* __restrict__ off, int64_t n, unsigned long long* out) {
    unsigned long long mx = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        mx = max(mx, (unsigned long long)(off[v + 1] - off[v]));
    atomicMax(out, mx);
}

__global__ void k_plan_pos(const int64_t* __restrict__ order, int32_t* __restrict__ vid, int32_t* __restrict__ pos,
                           int64_t n, unsigned long long* bad) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = order[p];
        if (v < 0 || v >= n) {
            atomicAdd(bad, 1ull);
            continue;
        }
        vid[p] = (int32_t)v;
        pos[v] = (int32_t)p;
    }
}

// every vertex must own exactly one position: pos[] was preset to -1
__global__ void k_plan_check_perm(const int32_t* __restrict__ vid, const int32_t* __restrict__ pos, int64_t n,
                                  unsigned long long* bad) {
    unsigned long long b = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = pos[v];
        b += (p < 0 || vid[p] != (int32_t)v);
    }
    if (b) atomicAdd(bad, b);
}

__device__ __forceinline__ int degree_bin(uint32_t d, bool self_only) {
    if (d == 0 || (d == 1 && self_only)) return kBinIdle;  // label provably cannot move
    if (d > (uint32_t)kHubMin) return kBinHub;
    if (d > (uint32_t)kLargeMin) return kBinLarge;
    if (d > (uint32_t)kSmallMax) return kBinMid;
    return kBinSmall;
}

__global__ void k_plan_bins(const int32_t* __restrict__ vid, const uint32_t* __restrict__ off,
                            const int32_t* __restrict__ nbr, uint8_t* __restrict__ bin, int64_t n,
                            unsigned long long* counts) {
    __shared__ unsigned long long sc[kBinIdle + 1];
    if (threadIdx.x <= kBinIdle) sc[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = vid[p];
        const uint32_t d = off[v + 1] - off[v];
        const int b = degree_bin(d, d == 1 && nbr[off[v]] == v);
        bin[p] = (uint8_t)b;
        atomicAdd(&sc[b], 1ull);
    }
    __syncthreads();
    if (threadIdx.x <= kBinIdle && sc[threadIdx.x]) atomicAdd(counts + threadIdx.x, sc[threadIdx.x]);
}

__global__ void k_iota(int32_t* a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int32_t)i;
}

__global__ void k_plan_slots(const int32_t* __restrict__ spos, const int32_t* __restrict__ vid,
                             const uint32_t* __restrict__ off, int32_t* __restrict__ slot_of_pos,
                             uint32_t* __restrict__ sdeg, int32_t* __restrict__ ndist, int64_t n, int64_t S) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = spos[s];
        if (s < S) {
            const int32_t v = vid[p];
            const uint32_t d = off[v + 1] - off[v];
            slot_of_pos[p] = (int32_t)s;
            sdeg[s] = d;
            ndist[s] = (int32_t)d;
        } else {
            slot_of_pos[p] = -1;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) sdeg[S] = 0;
}

// one warp per slot: copy the row, translating neighbour ids to positions
__global__ void k_plan_rows(const int32_t* __restrict__ spos, const int32_t* __restrict__ vid,
                            const int32_t* __restrict__ pos, const uint32_t* __restrict__ off,
                            const int32_t* __restrict__ nbr, const uint32_t* __restrict__ w,
                            const uint32_t* __restrict__ soff, int32_t* __restrict__ snbr, uint32_t* __restrict__ sw,
                            int64_t S) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
    for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; s < S; s += warps) {
        const int32_t v = vid[spos[s]];
        const uint32_t src = off[v], d = off[v + 1] - src, dst = soff[s];
        for (uint32_t k = lane; k < d; k += 32) {
            snbr[dst + k] = pos[nbr[src + k]];
            if (w) sw[dst + k] = w[src + k];
        }
    }
}

__global__ void k_init_labels(const int32_t* __restrict__ vid, const int64_t* __restrict__ init, int32_t* __restrict__ lab,
                              int64_t n) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        lab[p] = init ? (int32_t)init[vid[p]] : vid[p];
}

__global__ void k_check_labels(const int64_t* __restrict__ init, int64_t n, unsigned long long* bad) {
    unsigned long long b = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b += (init[i] < 0 || init[i] >= n);
    if (b) atomicAdd(bad, b);
}

__global__ void k_scatter_labels(const int32_t* __restrict__ vid, const int32_t* __restrict__ lab, int64_t* __restrict__ out,
                                 int64_t n) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        out[vid[p]] = lab[p];
}

// frontier compaction: marked positions -> per-bin slot lists (marks cleared)
struct BinBounds {
    int32_t beg[kNumBins + 1];
};

__global__ void k_compact(uint8_t* __restrict__ mark, const int32_t* __restrict__ slot_of_pos, int64_t n,
                          BinBounds bins, int32_t* __restrict__ lists, int32_t* __restrict__ list_len, int64_t cap) {
    const int lane = threadIdx.x & 31;
    for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 4; base < n;
         base += (int64_t)gridDim.x * blockDim.x * 4) {
        uint32_t word = 0;
        if (base + 4 <= n) {
            word = *reinterpret_cast<const uint32_t*>(mark + base);
            if (word) *reinterpret_cast<uint32_t*>(mark + base) = 0u;
        } else {
            for (int j = 0; j < 4 && base + j < n; ++j) {
                word |= (uint32_t)mark[base + j] << (8 * j);
                mark[base + j] = 0;
            }
        }
        for (int j = 0; j < 4; ++j) {
            int b = -1;
            int32_t s = -1;
            if ((word >> (8 * j)) & 0xff) {
                s = slot_of_pos[base + j];
                if (s >= 0) {
                    b = 0;
                    while (b < kNumBins - 1 && s >= bins.beg[b + 1]) ++b;
                }
            }
            // warp-aggregated append per bin
            for (int bb = 0; bb < kNumBins; ++bb) {
                const uint32_t msk = __ballot_sync(__activemask(), b == bb);
                if (!msk) continue;
                int32_t base_idx = 0;
                const int leader = __ffs(msk) - 1;
                if (lane == leader) base_idx = atomicAdd(list_len + bb, __popc(msk));
                base_idx = __shfl_sync(__activemask(), base_idx, leader);
                if (b == bb) lists[bb * cap + base_idx + __popc(msk & lanemask_lt())] = s;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------
static int grid_for(int64_t work, int per_block, int cap_blocks) {
    int64_t g = (work + per_block - 1) / per_block;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, cap_blocks));
}

// Launch accounting: counts every sweep-kernel launch; with LP_RAK_PROFILE
// also brackets each one with a CUDA event pair on the handle's stream.
struct Prof {
    bool on = false;
    int launches = 0;
    int64_t bin_launches[kNumBins] = {0, 0, 0, 0};
    std::vector<cudaEvent_t>* pool = nullptr;
    std::vector<int> tags;  // bin per pair, -1 = auxiliary
    size_t used = 0;
    cudaEvent_t next() {
        if (used == pool->size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            pool->push_back(e);
        }
        return (*pool)[used++];
    }
    void begin(cudaStream_t st, int tag) {
        if (tag >= 0) {
            ++launches;
            ++bin_launches[tag];
        }
        if (!on) return;
        tags.push_back(tag);
        cudaEventRecord(next(), st);
    }
    void end(cudaStream_t st, int) {
        if (on) cudaEventRecord(next(), st);
    }
};

template <int WM, int TIE> struct Launcher {
    static cudaError_t setup() {
        cudaError_t e;
        e = cudaFuncSetAttribute(k_warp<WM, TIE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)warp_smem_bytes<typename Acc<WM>::T>());
        if (e) return e;
        e = cudaFuncSetAttribute(k_block<WM, TIE, kLargeBits, kLargeThreads, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)block_smem_bytes<typename Acc<WM>::T, kLargeBits>());
        if (e) return e;
        e = cudaFuncSetAttribute(k_block<WM, TIE, kHubBits, kHubThreads, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)block_smem_bytes<typename Acc<WM>::T, kHubBits>());
        return e;
    }
    // dense: lists == nullptr, slot ranges from the plan; frontier: per-bin lists
    static void round(lp_graph* g, EvalArgs a, bool dense, int64_t* h_counts, Prof* prof) {
        using A = typename Acc<WM>::T;
        const Plan& P = g->plan;
        const int sms = g->num_sms;
        for (int b = 0; b < kNumBins; ++b) {
            const int64_t cnt = dense ? (P.bin_beg[b + 1] - P.bin_beg[b]) : h_counts[b];
            if (cnt <= 0) continue;
            const int32_t* list = dense ? nullptr : g->lists + (int64_t)b * g->n;
            const int32_t* len = dense ? nullptr : g->list_len + b;
            const int32_t sb = P.bin_beg[b], se = P.bin_beg[b + 1];
            a.bin = b;
            prof->begin(g->stream, b);
            switch (b) {
                case kBinHub:
                    k_block<WM, TIE, kHubBits, kHubThreads, true>
                        <<<grid_for(cnt, 1, sms), kHubThreads, block_smem_bytes<A, kHubBits>(), g->stream>>>(a, list, len,
                                                                                                       sb, se);
                    break;
                case kBinLarge:
                    k_block<WM, TIE, kLargeBits, kLargeThreads, false>
                        <<<grid_for(cnt, 1, sms * 3), kLargeThreads, block_smem_bytes<A, kLargeBits>(), g->stream>>>(
                            a, list, len, sb, se);
                    break;
                case kBinMid:
                    k_warp<WM, TIE><<<grid_for(cnt, kWarpsPerBlock, sms * 8), kWarpsPerBlock * 32,
                                      warp_smem_bytes<A>(), g->stream>>>(a, list, len, sb, se);
                    break;
                default:
                    k_small<WM, TIE><<<grid_for(cnt, 256, sms * 8), 256, 0, g->stream>>>(a, list, len, sb, se);
                    break;
            }
            prof->end(g->stream, b);
        }
    }
};

typedef void (*round_fn)(lp_graph*, EvalArgs, bool, int64_t*, Prof*);
typedef cudaError_t (*setup_fn)();

template <int WM> static void pick_fns(int tie, round_fn* r, setup_fn* s) {
    switch (tie) {
        case kRandom:
            *r = Launcher<WM, kRandom>::round;
            *s = Launcher<WM, kRandom>::setup;
            break;
        case kMinLabel:
            *r = Launcher<WM, kMinLabel>::round;
            *s = Launcher<WM, kMinLabel>::setup;
            break;
        default:
            *r = Launcher<WM, kScanFirst>::round;
            *s = Launcher<WM, kScanFirst>::setup;
    }
}

// ---------------------------------------------------------------------------
// graph handle
// ---------------------------------------------------------------------------
static void free_plan(Plan& P) {
    cudaFree(P.vid);
    cudaFree(P.pos);
    cudaFree(P.spos);
    cudaFree(P.slot_of_pos);
    cudaFree(P.soff);
    cudaFree(P.snbr);
    cudaFree(P.sw);
    cudaFree(P.ndist);
    P = Plan();
}

static void destroy_graph(lp_graph* g) {
    if (!g) return;
    free_plan(g->plan);
    cudaFree(g->off);
    cudaFree(g->nbr);
    cudaFree(g->w);
    cudaFree(g->labA);
    cudaFree(g->labB);
    cudaFree(g->mark);
    cudaFree(g->lists);
    cudaFree(g->list_len);
    cudaFree(g->counters);
    cudaFree(g->out64);
    cudaFree(g->cub_tmp);
    if (g->h_list_len) cudaFreeHost(g->h_list_len);
    if (g->h_counters) cudaFreeHost(g->h_counters);
    for (cudaEvent_t e : g->event_pool) cudaEventDestroy(e);
    if (g->ev0) cudaEventDestroy(g->ev0);
    if (g->ev1) cudaEventDestroy(g->ev1);
    if (g->stream) cudaStreamDestroy(g->stream);
    delete g;
}

static int ensure_cub_tmp(lp_graph* g, size_t bytes) {
    if (bytes <= g->cub_tmp_bytes) return LP_OK;
    cudaFree(g->cub_tmp);
    g->cub_tmp = nullptr;
    g->cub_tmp_bytes = 0;
    LP_CK(cudaMalloc(&g->cub_tmp, bytes));
    g->cub_tmp_bytes = bytes;
    return LP_OK;
}

static uint64_t hash_order(const int64_t* order, int64_t n) {
    uint64_t h = 1469598103934665603ull;
    for (int64_t i = 0; i < n; ++i) {
        h ^= (uint64_t)order[i];
        h *= 1099511628211ull;
    }
    return h;
}

// Build (or reuse) the position / storage plan for a visit order.
static int build_plan(lp_graph* g, const int64_t* order_host, uint32_t seed, float* plan_ms) {
    const int64_t n = g->n;
    bool custom = order_host != nullptr;
    uint64_t oh = custom ? hash_order(order_host, n) : 0;
    Plan& P = g->plan;
    *plan_ms = 0.f;
    if (P.valid && P.custom_order == custom && (custom ? P.order_hash == oh : P.seed == seed)) return LP_OK;
    free_plan(P);
    std::vector<int64_t> own;
    if (!custom) {
        own.resize((size_t)n);
        lp_host_shuffled_indices(n, seed, own.data());
        order_host = own.data();
    }
    cudaStream_t st = g->stream;
    LP_CK(cudaEventRecord(g->ev0, st));
    int64_t bytes = 0;
    LP_CK(dalloc(&P.vid, n, &bytes));
    LP_CK(dalloc(&P.pos, n, &bytes));
    LP_CK(dalloc(&P.spos, n, &bytes));
    LP_CK(dalloc(&P.slot_of_pos, n, &bytes));
    LP_CK(dalloc(&P.ndist, n, &bytes));
    int64_t* d_order = nullptr;
    uint8_t* d_bin = nullptr;
    uint8_t* d_bin_sorted = nullptr;
    int32_t* d_iota = nullptr;
    uint32_t* d_sdeg = nullptr;
    int64_t tmpb = 0;
    LP_CK(dalloc(&d_order, n, &tmpb));
    LP_CK(dalloc(&d_bin, n, &tmpb));
    LP_CK(dalloc(&d_bin_sorted, n, &tmpb));
    LP_CK(dalloc(&d_iota, n, &tmpb));
    LP_CK(dalloc(&d_sdeg, n + 1, &tmpb));
    LP_CK(cudaMemcpyAsync(d_order, order_host, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    LP_CK(cudaMemsetAsync(g->counters, 0, 8 * sizeof(unsigned long long), st));
    const int G = g->num_sms * 8;
    LP_CK(cudaMemsetAsync(P.pos, 0xff, n * sizeof(int32_t), st));
    k_plan_pos<<<G, 256, 0, st>>>(d_order, P.vid, P.pos, n, g->counters);
    k_plan_check_perm<<<G, 256, 0, st>>>(P.vid, P.pos, n, g->counters);
    LP_CK(cudaMemcpyAsync(g->h_counters, g->counters, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    LP_CK(cudaStreamSynchronize(st));
    if (g->h_counters[0]) {  // checked before any kernel dereferences vid[]
        cudaFree(d_order);
        cudaFree(d_bin);
        cudaFree(d_bin_sorted);
        cudaFree(d_iota);
        cudaFree(d_sdeg);
        free_plan(P);
        lp_set_error("order is not a permutation of range(n)");
        return LP_ERR_INVALID;
    }
    k_plan_bins<<<G, 256, 0, st>>>(P.vid, g->off, g->nbr, d_bin, n, g->counters + 1);
    k_iota<<<G, 256, 0, st>>>(d_iota, n);
    size_t need = 0;
    LP_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, d_bin, d_bin_sorted, d_iota, P.spos, (int)n, 0, 3, st));
    size_t need2 = 0;
    LP_CK(cub::DeviceScan::ExclusiveSum(nullptr, need2, d_sdeg, d_sdeg, (int)(n + 1), st));
    if (int rc = ensure_cub_tmp(g, std::max(need, need2))) return rc;
    LP_CK(cub::DeviceRadixSort::SortPairs(g->cub_tmp, need, d_bin, d_bin_sorted, d_iota, P.spos, (int)n, 0, 3, st));
    LP_CK(cudaMemcpyAsync(g->h_counters, g->counters, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    LP_CK(cudaStreamSynchronize(st));
    int64_t acc = 0;
    for (int b = 0; b < kNumBins; ++b) {
        P.bin_beg[b] = (int32_t)acc;
        acc += (int64_t)g->h_counters[1 + b];
    }
    P.bin_beg[kNumBins] = (int32_t)acc;
    P.S = acc;
    k_plan_slots<<<G, 256, 0, st>>>(P.spos, P.vid, g->off, P.slot_of_pos, d_sdeg, P.ndist, n, P.S);
    LP_CK(dalloc(&P.soff, P.S + 1, &bytes));
    LP_CK(cub::DeviceScan::ExclusiveSum(g->cub_tmp, need2, d_sdeg, P.soff, (int)(P.S + 1), st));
    uint32_t m_active = 0;
    LP_CK(cudaMemcpyAsync(&m_active, P.soff + P.S, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    LP_CK(cudaStreamSynchronize(st));
    P.m_active = m_active;
    LP_CK(dalloc(&P.snbr, P.m_active, &bytes));
    if (g->w) LP_CK(dalloc(&P.sw, P.m_active, &bytes));
    k_plan_rows<<<g->num_sms * 16, 256, 0, st>>>(P.spos, P.vid, P.pos, g->off, g->nbr, g->w, P.soff, P.snbr, P.sw,
                                                 P.S);
    LP_CK(cudaGetLastError());
    LP_CK(cudaEventRecord(g->ev1, st));
    LP_CK(cudaEventSynchronize(g->ev1));
    LP_CK(cudaEventElapsedTime(plan_ms, g->ev0, g->ev1));
    cudaFree(d_order);
    cudaFree(d_bin);
    cudaFree(d_bin_sorted);
    cudaFree(d_iota);
    cudaFree(d_sdeg);
    P.valid = true;
    P.custom_order = custom;
    P.seed = seed;
    P.order_hash = oh;
    g->bytes += bytes;
    return LP_OK;
}

extern "C" int lp_graph_create(int64_t n, int64_t m, const int64_t* offsets, const int64_t* neighbors,
                               const double* weights, int32_t device, lp_graph** out) {
    if (!out) return lp_fail(LP_ERR_INVALID, "out is NULL");
    *out = nullptr;
    if (n < 0 || m < 0) return lp_fail(LP_ERR_INVALID, "negative vertex or edge count");
    if (n >= (int64_t)INT32_MAX) return lp_fail(LP_ERR_UNSUPPORTED, "vertex count must be < 2^31-1");
    if (m >= (int64_t)UINT32_MAX) return lp_fail(LP_ERR_UNSUPPORTED, "edge count must be < 2^32-1");
    if (n > 0 && !offsets) return lp_fail(LP_ERR_INVALID, "offsets is NULL");
    if (m > 0 && !neighbors) return lp_fail(LP_ERR_INVALID, "neighbors is NULL");
    if (n > 0 && (offsets[0] != 0 || offsets[n] != m))
        return lp_fail(LP_ERR_INVALID, "offsets must start at 0 and end at edge_count");
    for (int64_t v = 0; v < n; ++v)
        if (offsets[v + 1] < offsets[v]) return lp_fail(LP_ERR_INVALID, "offsets must be non-decreasing");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return lp_fail(LP_ERR_CUDA, "no CUDA device available (liblabelprop_cuda needs a B200)");
    if (device >= 0) LP_CK(cudaSetDevice(device));
    lp_graph* g = new lp_graph();
    int rc = LP_OK;
    auto fail = [&](int code) {
        destroy_graph(g);
        return code;
    };
    if (cudaGetDevice(&g->device) != cudaSuccess) return fail(lp_fail(LP_ERR_CUDA, "cudaGetDevice failed"));
    cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->device);
    g->n = n;
    g->m = m;
#define G_CK(call)                                                                                      \
    do {                                                                                                \
        cudaError_t _e = (call);                                                                        \
        if (_e != cudaSuccess)                                                                          \
            return fail(lp_fail(_e == cudaErrorMemoryAllocation ? LP_ERR_NOMEM : LP_ERR_CUDA,           \
                                "CUDA error %s at %s:%d", cudaGetErrorName(_e), __FILE__, __LINE__)); \
    } while (0)
    G_CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    G_CK(cudaEventCreate(&g->ev0));
    G_CK(cudaEventCreate(&g->ev1));
    cudaStream_t st = g->stream;
    G_CK(dalloc(&g->off, n + 1, &g->bytes));
    G_CK(dalloc(&g->nbr, m, &g->bytes));
    G_CK(dalloc(&g->labA, n, &g->bytes));
    G_CK(dalloc(&g->labB, n, &g->bytes));
    G_CK(dalloc(&g->mark, n + 4, &g->bytes));
    G_CK(dalloc(&g->lists, (size_t)kNumBins * std::max<int64_t>(n, 1), &g->bytes));
    G_CK(dalloc(&g->list_len, kNumBins, &g->bytes));
    G_CK(dalloc(&g->counters, 32, &g->bytes));
    G_CK(dalloc(&g->out64, n, &g->bytes));
    G_CK(cudaMallocHost((void**)&g->h_list_len, kNumBins * sizeof(int32_t)));
    G_CK(cudaMallocHost((void**)&g->h_counters, 32 * sizeof(unsigned long long)));
    G_CK(cudaMemsetAsync(g->mark, 0, n + 4, st));
    G_CK(cudaMemsetAsync(g->counters, 0, 32 * sizeof(unsigned long long), st));
    {
        int64_t* tmp = nullptr;
        int64_t tb = 0;
        G_CK(dalloc(&tmp, std::max(n + 1, m), &tb));
        G_CK(cudaMemcpyAsync(tmp, offsets, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        k_i64_to_u32<<<g->num_sms * 8, 256, 0, st>>>(tmp, g->off, n + 1);
        if (m > 0) {
            G_CK(cudaMemcpyAsync(tmp, neighbors, m * sizeof(int64_t), cudaMemcpyHostToDevice, st));
            k_nbr_convert<<<g->num_sms * 8, 256, 0, st>>>(tmp, g->nbr, m, n, g->counters);
        }
        if (weights && m > 0) {
            G_CK(cudaMemcpyAsync(tmp, weights, m * sizeof(double), cudaMemcpyHostToDevice, st));
            unsigned long long init[4] = {0, 0, ~0ull, 0};
            G_CK(cudaMemcpyAsync(g->counters + 4, init, sizeof(init), cudaMemcpyHostToDevice, st));
            k_weight_scan<<<g->num_sms * 8, 256, 0, st>>>((const double*)tmp, m, g->counters + 4);
        }
        k_degree_max<<<g->num_sms * 8, 256, 0, st>>>(g->off, n, g->counters + 8);
        G_CK(cudaMemcpyAsync(g->h_counters, g->counters, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        G_CK(cudaStreamSynchronize(st));
        if (g->h_counters[0]) {
            cudaFree(tmp);
            return fail(lp_fail(LP_ERR_INVALID, "neighbor ids must lie in [0, vertex_count)"));
        }
        g->max_degree = (int64_t)g->h_counters[8];
        g->wmode = kUnit;
        if (weights && m > 0 && g->h_counters[4 + 0] != 0) {
            const unsigned long long bad = g->h_counters[4 + 1];
            const int emin = (int)g->h_counters[4 + 2] - 2048, emax = (int)g->h_counters[4 + 3] - 2048;
            // fixed point: w * 2^shift is an integer < 2^32 for every float32 weight when
            // shift = 24 - emin and (emax - emin + 24) <= 32; row sums stay < 2^64
            const int span = emax - emin + 24;
            const double deg_bits = std::log2((double)std::max<int64_t>(2, g->max_degree));
            if (bad == 0 && span <= 32 && span + deg_bits < 63.0) {
                g->wmode = kFixed;
                g->fixed_shift = 24 - emin;
            } else {
                g->wmode = kFloat;
            }
            G_CK(dalloc(&g->w, m, &g->bytes));
            k_weight_convert<<<g->num_sms * 8, 256, 0, st>>>((const double*)tmp, g->w, m, g->wmode, g->fixed_shift);
        }
        G_CK(cudaStreamSynchronize(st));
        cudaFree(tmp);
    }
    G_CK(cudaGetLastError());
    *out = g;
    (void)rc;
    return LP_OK;
#undef G_CK
}

extern "C" int lp_graph_destroy(lp_graph* g) {
    if (!g) return LP_OK;
    cudaSetDevice(g->device);
    destroy_graph(g);
    return LP_OK;
}

extern "C" int lp_graph_get_info(const lp_graph* g, lp_graph_info* info) {
    if (!g || !info) return lp_fail(LP_ERR_INVALID, "NULL argument");
    memset(info, 0, sizeof(*info));
    info->vertex_count = g->n;
    info->edge_count = g->m;
    info->weight_mode = g->wmode;
    info->fixed_shift = g->fixed_shift;
    info->max_degree = g->max_degree;
    info->device_bytes = g->bytes;
    info->device = g->device;
    return LP_OK;
}

extern "C" void* lp_graph_stream(lp_graph* g) { return g ? (void*)g->stream : nullptr; }

// ---------------------------------------------------------------------------
// RAK driver
// ---------------------------------------------------------------------------
static int rak_core(lp_graph* g, const lp_rak_opts* o, const int64_t* order, const int64_t* labels_init,
                    int64_t* changed_per_iter, lp_run_stats* stats) {
    if (!g || !o) return lp_fail(LP_ERR_INVALID, "NULL argument");
    if (!(o->tolerance > 0.0 && o->tolerance <= 1.0)) return lp_fail(LP_ERR_INVALID, "tolerance must be in (0, 1]");
    if (o->max_iterations < 1) return lp_fail(LP_ERR_INVALID, "max_iterations must be >= 1");
    if (o->tie < 0 || o->tie > 2) return lp_fail(LP_ERR_INVALID, "unknown tie rule");
    if (o->batches < 0) return lp_fail(LP_ERR_INVALID, "batches must be >= 0");
    LP_CK(cudaSetDevice(g->device));
    lp_run_stats st_local;
    lp_run_stats* S = stats ? stats : &st_local;
    memset(S, 0, sizeof(*S));
    const int64_t n = g->n;
    g->labels_valid = false;
    if (n == 0) {
        g->labels_valid = true;
        return LP_OK;
    }
    float plan_ms = 0.f;
    if (int rc = build_plan(g, order, o->seed, &plan_ms)) return rc;
    S->plan_ms = plan_ms;
    Plan& P = g->plan;
    cudaStream_t st = g->stream;
    round_fn run_round = nullptr;
    setup_fn setup = nullptr;
    if (g->wmode == kFixed)
        pick_fns<kFixed>(o->tie, &run_round, &setup);
    else if (g->wmode == kFloat)
        pick_fns<kFloat>(o->tie, &run_round, &setup);
    else
        pick_fns<kUnit>(o->tie, &run_round, &setup);
    LP_CK(setup());

    const int64_t B = (o->batches == 0 || o->batches > n) ? n : o->batches;
    const int64_t bs = (n + B - 1) / B;
    const bool cross = bs < n;  // some vertex depends on an earlier batch
    if (labels_init) {
        int64_t* tmp = g->out64;
        LP_CK(cudaMemcpyAsync(tmp, labels_init, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        LP_CK(cudaMemsetAsync(g->counters, 0, sizeof(unsigned long long), st));
        k_check_labels<<<g->num_sms * 4, 256, 0, st>>>(tmp, n, g->counters);
        unsigned long long bad = 0;
        LP_CK(cudaMemcpyAsync(&bad, g->counters, sizeof(bad), cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
        if (bad) return lp_fail(LP_ERR_INVALID, "initial labels must lie in [0, vertex_count)");
        k_init_labels<<<g->num_sms * 8, 256, 0, st>>>(P.vid, tmp, g->labA, n);
    } else {
        k_init_labels<<<g->num_sms * 8, 256, 0, st>>>(P.vid, nullptr, g->labA, n);
    }
    LP_CK(cudaGetLastError());

    int32_t* L0 = g->labA;
    int32_t* X = g->labB;
    EvalArgs a;
    a.soff = P.soff;
    a.snbr = P.snbr;
    a.sw = P.sw;
    a.spos = P.spos;
    a.vid = P.vid;
    a.mark = cross ? g->mark : nullptr;
    a.ndist = P.ndist;
    a.counters = g->counters;
    a.bs = (int32_t)bs;
    a.seed = o->seed;
    BinBounds bins_only;
    memcpy(bins_only.beg, P.bin_beg, sizeof(P.bin_beg));

    LP_CK(cudaMemsetAsync(g->counters, 0, kCtrCount * sizeof(unsigned long long), st));
    Prof prof;
    prof.on = (o->flags & LP_RAK_PROFILE) != 0;
    prof.pool = &g->event_pool;
    LP_CK(cudaEventRecord(g->ev0, st));
    int it = 0;
    int rounds = 0;
    int64_t h_counts[kNumBins];
    while (it < o->max_iterations) {
        ++it;
        a.sweep = (uint32_t)it;
        a.L0 = L0;
        a.x = X;
        LP_CK(cudaMemcpyAsync(X, L0, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        LP_CK(cudaMemsetAsync(g->counters + kCtrChanged, 0, 3 * sizeof(unsigned long long), st));
        run_round(g, a, true, h_counts, &prof);
        ++rounds;
        while (cross) {
            LP_CK(cudaMemsetAsync(g->list_len, 0, kNumBins * sizeof(int32_t), st));
            prof.begin(st, -1);
            k_compact<<<g->num_sms * 8, 256, 0, st>>>(g->mark, P.slot_of_pos, n, bins_only, g->lists, g->list_len, n);
            prof.end(st, -1);
            LP_CK(cudaMemcpyAsync(g->h_list_len, g->list_len, kNumBins * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
            LP_CK(cudaStreamSynchronize(st));
            int64_t total = 0;
            for (int b = 0; b < kNumBins; ++b) total += (h_counts[b] = g->h_list_len[b]);
            if (total == 0) break;
            LP_CK(cudaMemsetAsync(g->counters + kCtrWrites, 0, 2 * sizeof(unsigned long long), st));
            run_round(g, a, false, h_counts, &prof);
            ++rounds;
        }
        LP_CK(cudaMemcpyAsync(g->h_counters, g->counters, kCtrCount * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                              st));
        LP_CK(cudaStreamSynchronize(st));
        LP_CK(cudaGetLastError());
        const int64_t changed = (int64_t)g->h_counters[kCtrChanged];
        if (changed_per_iter) changed_per_iter[it - 1] = changed;
        std::swap(L0, X);  // L0 now holds this sweep's labels
        if ((double)changed <= o->tolerance * (double)n) break;  // rak.py:114-115
    }
    LP_CK(cudaEventRecord(g->ev1, st));
    LP_CK(cudaEventSynchronize(g->ev1));
    float ms = 0.f;
    LP_CK(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
    g->cur = L0;
    g->labels_valid = true;
    S->iterations = it;
    S->rounds = rounds;
    S->kernel_ms = ms;
    S->arcs_dense = g->m * it;
    S->launches = prof.launches;
    for (int b = 0; b < kNumBins; ++b) {
        S->bin_arcs[b] = (int64_t)g->h_counters[kCtrArcs + b];
        S->bin_vertices[b] = (int64_t)g->h_counters[kCtrVerts + b];
        S->bin_launches[b] = prof.bin_launches[b];
        S->arcs_scanned += S->bin_arcs[b];
    }
    for (size_t i = 0; i < prof.tags.size(); ++i) {
        float e = 0.f;
        LP_CK(cudaEventElapsedTime(&e, g->event_pool[2 * i], g->event_pool[2 * i + 1]));
        if (prof.tags[i] >= 0)
            S->bin_ms[prof.tags[i]] += e;
        else
            S->aux_ms += e;
    }
    return LP_OK;
}

extern "C" int lp_rak_run_resident(lp_graph* g, const lp_rak_opts* opts, const int64_t* order, lp_run_stats* stats) {
    return rak_core(g, opts, order, nullptr, nullptr, stats);
}

extern "C" int lp_labels_download(lp_graph* g, int64_t* labels_out) {
    if (!g || !labels_out) return lp_fail(LP_ERR_INVALID, "NULL argument");
    if (!g->labels_valid) return lp_fail(LP_ERR_INVALID, "no labels: run a detection first");
    if (g->n == 0) return LP_OK;
    LP_CK(cudaSetDevice(g->device));
    k_scatter_labels<<<g->num_sms * 8, 256, 0, g->stream>>>(g->plan.vid, g->cur, g->out64, g->n);
    LP_CK(cudaMemcpyAsync(labels_out, g->out64, g->n * sizeof(int64_t), cudaMemcpyDeviceToHost, g->stream));
    LP_CK(cudaStreamSynchronize(g->stream));
    return LP_OK;
}

extern "C" int lp_rak_run(lp_graph* g, const lp_rak_opts* opts, const int64_t* order, const int64_t* labels_init,
                          int64_t* labels_out, int64_t* changed_per_iter, lp_run_stats* stats) {
    if (!labels_out) return lp_fail(LP_ERR_INVALID, "labels_out is NULL");
    if (int rc = rak_core(g, opts, order, labels_init, changed_per_iter, stats)) return rc;
    return lp_labels_download(g, labels_out);
}

extern "C" int lp_device_count(int32_t* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (count) *count = (e == cudaSuccess) ? c : 0;
    return LP_OK;
}

extern "C" int lp_host_register(void* ptr, int64_t bytes) {
    if (!ptr || bytes <= 0) return lp_fail(LP_ERR_INVALID, "bad host range");
    LP_CK(cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault));
    return LP_OK;
}

extern "C" int lp_host_unregister(void* ptr) {
    if (!ptr) return lp_fail(LP_ERR_INVALID, "NULL pointer");
    LP_CK(cudaHostUnregister(ptr));
    return LP_OK;
}
