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
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <vector>

#include "../../include/labelprop_cuda.h"
#include "lp_common.cuh"
#include "lp_host.h"
#include "lp_rak_kernels.cuh"
#include "lp_loop_kernels.cuh"
#include "lp_slpa_kernels.cuh"
#include "lp_copra_kernels.cuh"

using namespace lp;

// Storage bins: rows with d > kSmallMax (sorted by degree, descending, so the
// dense route hands out the largest hubs first), then the small rows by degree
// class 9..16, 5..8, 2..4 (visit order inside a class), then idle vertices (no
// arc but a self-loop: label fixed).
enum Bin : int { kBinBig = 0, kBinS16 = 1, kBinS8 = 2, kBinS4 = 3, kBinIdle = 4, kNumBins = 5 };
// per-kernel accounting slots (lp_run_stats.bin_*)
enum KernelSlot : int { kKHub = 0, kKTeam = 1, kKWarp = 2, kKSmall = 3, kKSlots = 4, kKGather = 4 };

#define LP_CK(call)                                                                                  \
    do {                                                                                             \
        cudaError_t _e = (call);                                                                     \
        if (_e != cudaSuccess) {                                                                     \
            lp_set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__, __LINE__,     \
                         cudaGetErrorString(_e));                                                    \
            return LP_ERR_CUDA;                                                                      \
        }                                                                                            \
    } while (0)

// Device memory comes from the device's stream-ordered pool (cudaMallocAsync
// on the handle's stream, release threshold raised once): a fresh handle or
// plan reuses the memory of earlier ones instead of paying cudaMalloc /
// cudaFree (tens of ms for the GB-sized CSR buffers).  tl_stream is the
// stream of the handle the calling API function works on.
static thread_local cudaStream_t tl_stream = nullptr;

struct StreamScope {
    cudaStream_t saved;
    explicit StreamScope(cudaStream_t s) : saved(tl_stream) { tl_stream = s; }
    ~StreamScope() { tl_stream = saved; }
};

static cudaError_t pool_alloc(void** p, size_t bytes) {
    return cudaMallocAsync(p, std::max<size_t>(bytes, 1), tl_stream);
}
template <typename T> static cudaError_t pool_alloc(T** p, size_t bytes) { return pool_alloc((void**)p, bytes); }

static void dfree(void* p) {
    if (p) cudaFreeAsync(p, tl_stream);
}

template <typename T> static cudaError_t dalloc(T** p, size_t count, int64_t* bytes) {
    *bytes += (int64_t)(count * sizeof(T));
    return pool_alloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
}

// keep freed pool memory for reuse instead of returning it to the driver
static void pool_keep(int device) {
    static int done = -1;
    if (done == device) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done = device;
}

// Plan kinds: RAK (seeded/custom visit order, self-loop arcs kept: the
// reference tally counts them, rak.py:99-105) and INDEX (identity order,
// self arcs dropped: COPRA and SLPA skip them, copra.py:137-139,
// slpa.py:75).
enum PlanKind : int { kPlanRak = 0, kPlanIndex = 1, kNumPlanKinds = 2 };

struct Plan {
    bool valid = false;
    bool custom_order = false;
    int kind = kPlanRak;
    uint32_t seed = 0;
    uint64_t order_hash = 0;
    int32_t* pos = nullptr;          // vertex -> visit position
    int32_t* svid = nullptr;         // slot -> vertex (n entries; first S active)
    int32_t* slot_of = nullptr;      // vertex -> slot or -1
    uint32_t* soff = nullptr;        // [S+1]
    uint32_t* snbr = nullptr;        // [m_active] neighbour id << 2 | batch flags
    uint32_t* sw = nullptr;          // [m_active] or null
    unsigned long long* swsum = nullptr;  // [S] row weight totals (fixed-point mode)
    int32_t* ndist = nullptr;        // [S]
    int32_t* lbuf = nullptr;         // [m_active] phase-1 gathered labels
    int32_t* hb_lab = nullptr;       // [m_active] hub rows' labels bucketed by partition (k_hub_bucket)
    uint32_t* hb_pos = nullptr;      // [m_active] ... and their arc positions
    int64_t S = 0;
    int64_t m_active = 0;
    int64_t flags_bs = -1;           // batch size the snbr flags were computed for
    int32_t bin_beg[kNumBins + 1] = {0, 0, 0, 0, 0, 0};  // slot range of each bin (idle: [.., n))
    int32_t big_end = 0;             // slots [0, big_end) are big rows, [big_end, S) small
    // arcs of the rows longer than 16 / than mid_max: big rows come first in
    // storage order, by descending degree, so each is a prefix of the arcs
    int64_t arcs_gt16 = 0, arcs_gt_mid = 0;
    // visit order (position -> vertex) and the dense-wave lengths
    int32_t* vorder = nullptr;
    int32_t* wave_len = nullptr;     // [kMaxWaves] device
    int waves = 0;                   // waves wave_len was built for
    // every active row as phase-1 pieces (INDEX plans: SLPA's dense rounds)
    int32_t* dslot = nullptr;
    int32_t* dk0 = nullptr;
    int32_t* dcount = nullptr;       // device copy of the piece count
    int64_t npieces = 0;
    int64_t bytes = 0;
};

struct lp_graph {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaStream_t aux[2] = {nullptr, nullptr};  // concurrent tally kernels of a round
    cudaEvent_t ev_fork = nullptr, ev_join[2] = {nullptr, nullptr};
    cudaEvent_t ev_route = nullptr, ev_gather = nullptr;  // dense route / phase-1 gather done (round())
    int64_t n = 0, m = 0;
    int64_t max_degree = 0;
    int64_t sliceable = 0;  // rows long enough to be cut into slices
    int64_t slice_slots = 0;  // their largest global tables, summed
    int wmode = kUnit;
    int fixed_shift = 0;
    int64_t bytes = 0;
    // original CSR (device, int32)
    uint32_t* off = nullptr;
    int32_t* nbr = nullptr;
    uint32_t* w = nullptr;  // converted weights (fixed-point or float bits)
    Plan plans[kNumPlanKinds];
    int pk = kPlanRak;  // the plan the current run uses
    Plan& plan() { return plans[pk]; }
    // run state
    bool l2_persist = true;  // persisting L2 window over the label arrays (set_l2_window)
    bool fuse_forced = false;  // LP_FUSE_MAXD given: no per-run choice
    int run_fuse = 16;         // the current run's fuse_maxd (rak_core: every row when the sweep cascades)
    int fuse_maxd = 16;      // RAK rows of degree <= this gather their labels in the tally kernel
                             // (EvalArgs::fused); >= 2^30: every row (LP_FUSE_MAXD, -1 = all)
    int32_t* labA = nullptr;
    int32_t* labB = nullptr;
    int32_t* cur = nullptr;  // the buffer holding the latest labels
    unsigned long long* mark = nullptr;  // frontier marks by vertex id (changed weight since routing)
    unsigned long long* gap = nullptr;   // per slot: winner margin lower bound at the last evaluation
    uint32_t* chg = nullptr;             // sweep boundary: label changed in the last sweep (bitmap)
    int32_t* mq[2] = {nullptr, nullptr};  // mark queues (alternate per round)
    int32_t* mq_len = nullptr;  // their lengths [2]
    uint32_t* mbits = nullptr;  // marked-vertex bitmap (all zero between passes)
    int2* hb_off = nullptr;     // hub partition buckets (per item cb + q)
    bool mark_bitmap = true;    // LP_MARK_BITMAP=0: always queue marked vertices by scanning the marks
    int mark_scan_div = 16;     // ... scan when more than n / mark_scan_div rows changed (LP_MARK_SCAN_DIV)
    bool hub_bucket = false;    // LP_HUB_BUCKET=1: bucket hub partitions (measured: no gain once hubs
                                // use the singleton two-pass tally)
    int first_est_min = 256, first_est_div = 4;  // LP_FIRST_EST_MIN / LP_FIRST_EST_DIV (tuned on R-MAT-22)
    int32_t* slots = nullptr;   // SLPA memories [n x T]
    size_t slots_cap = 0;
    // COPRA label sets (sweep-start and working), [n x K] rows
    int32_t* clabs[2] = {nullptr, nullptr};
    double* cbels[2] = {nullptr, nullptr};
    int32_t* csize[2] = {nullptr, nullptr};
    int32_t* cbest[2] = {nullptr, nullptr};
    size_t ccap = 0;            // cells (n * K) the label-set buffers hold
    int32_t* ccur = nullptr;    // work cursors [4]
    int32_t* cbig = nullptr;    // team list [n]
    int32_t* cmid = nullptr;    // tier-1 list [n]
    // COPRA team scratch, per team block: entries [gent], contribution map [gcon]
    int32_t* gelab = nullptr;
    double* geval = nullptr;
    int32_t* gefirst = nullptr;
    int32_t* grlab = nullptr;
    double* grval = nullptr;
    int32_t* gfmap = nullptr;
    int32_t* gblab = nullptr;
    double* gbval = nullptr;
    int32_t* gbc = nullptr;
    int32_t* gwc = nullptr;
    int32_t* gqs = nullptr;
    int32_t* gslab = nullptr;
    double* gsval = nullptr;
    size_t gent = 0, gcon = 0;
    int gblocks = 0;
    Routes routes;
    int64_t cap_items = 0;
    unsigned long long* counters = nullptr;
    int64_t* out64 = nullptr;
    int32_t* h_len = nullptr;                  // pinned route lengths
    unsigned long long* h_counters = nullptr;  // pinned
    void* cub_tmp = nullptr;
    size_t cub_tmp_bytes = 0;
    int num_sms = 148;
    int waves = 1;  // dense waves of the cross-batch schedules (LP_WAVES overrides)
    bool copra_bitmap = true;   // LP_COPRA_BITMAP=0: COPRA marks queue on the mark's transition (mark_row)
    bool copra_overlap = true;  // LP_COPRA_OVERLAP=0: the team rows after the warp tiers, on one stream
    int32_t* croute = nullptr;  // COPRA: the round's pre-routed team rows [n]
    int32_t* croute_mark = nullptr;  // ... and per slot the id of the round that listed it [n]
    int32_t copra_rid = 0;           // round ids (never reused by a handle)
    int copra_long = 32768;  // COPRA rows with more contributions (degree x K) go to the 16-warp team
                             // (LP_COPRA_LONG, 0 = off; R-MAT-20 k = 8 in place 122 -> 85 ms)
    // frontier loop (lp_loop_kernels.cuh): rounds that evaluate at most loop_rows rows continue on the
    // device in one cooperative launch (LP_LOOP_ROWS, 0 = off); graphs whose rows all fit the loop's
    // warp table, hold at most loop_dense_arcs arcs and average >= 12 arcs a row run their dense rounds
    // there too (LP_LOOP_DENSE_ARCS; SLPA planted-1M 21 -> 14 ms)
    int64_t loop_rows = 8192;
    int64_t loop_dense_arcs = 64 << 20;
    int loop_max_queue = 1 << 16;
    int loop_blocks_per_sm = 0;  // 0 = the kernel's occupancy (LP_LOOP_BLOCKS)
    LoopCtl* loop_ctl = nullptr;  // device
    LoopCtl* h_loop = nullptr;    // pinned
    cudaError_t (*loop_run)(lp_graph*, const EvalArgs&, const int32_t*, const int32_t*, int, int, int, int) = nullptr;
    bool margin_skip = true;  // frontier margin test (LP_MARGIN=0 disables)
    bool debug_rounds = false;  // LP_DEBUG_ROUNDS=1: per-round route sizes on stderr
    bool rows_sorted = false;  // every row strictly increasing (duplicate-free), checked at upload
    bool first_round_shortcut = true;  // LP_FIRST_ROUND=0 disables k_first_round
    bool first_chain = true;           // LP_FIRST_CHAIN=0: plain first-arc guess in exact schedules
    bool sweep_frontier = true;        // active frontier across sweeps (LP_SWEEP_FRONTIER=0 disables)
    double carry_frac = 0.5;           // ... after sweeps that changed <= this share of the rows (LP_CARRY_FRAC)
    bool pull_rounds = false;  // LP_PULL_ROUNDS=1: pulled marks instead of full rounds after big rounds (measured: no gain)
    double pull_max_frac = 0.8;  // ... but a full round after rounds that changed more (LP_PULL_MAX)
    double dense_frac = 0.35;   // a round that changed >= this share of the active rows is followed by a
                                // full round instead of marks + frontier (LP_DENSE_FRAC; >= 1 disables)
    int cap_route = 0;      // LP_CAP_ROUTE=1: route rows by table capacity >= degree (measured: no gain)
    bool id_single = true;  // LP_ID_SINGLE=0: no singleton labels in the first sweep (see kSingle)
    int push_div = 3;
    bool id_single_random = true;  // LP_ID_SINGLE_RANDOM=0: no singleton labels with random ties
    bool id_single_w = true;       // LP_ID_SINGLE_W=0: no singleton labels with fixed-point weights
    bool two_team_w = true;        // LP_TWO_TEAM_W=0: weighted team / hub rows insert every label
    int reg_est = LP_WARP_REG_EST;  // LP_REG_EST
    int mid_max = kMidMax;          // LP_MID_MAX: thread-per-row k_mid up to this degree (0 = off)
    bool mid_hash = true;           // LP_MID_HASH=0: unit-weight mid rows by O(d^2) compares (k_mid)      // sweep boundary: push marks from the changed rows when <= 1/push_div of the
                            // rows changed, else pull (LP_PUSH_DIV)
    int warp_maxd[2] = {WarpClass<0>::kMaxDeg, WarpClass<1>::kMaxDeg};  // LP_WARP0_MAXD / LP_WARP1_MAXD
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

// flat form: row-start flags, then every arc that is not a row start must be
// strictly above its predecessor
__global__ void k_row_starts(const uint32_t* __restrict__ off, int64_t n, int64_t m, uint8_t* __restrict__ start) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        if ((int64_t)off[v] < m) start[off[v]] = 1;
}
__global__ void k_rows_sorted_flat(const int32_t* __restrict__ nbr, const uint8_t* __restrict__ start, int64_t m,
                                   unsigned long long* bad) {
    unsigned long long b = 0;
    for (int64_t e = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
        b += !start[e] && nbr[e] <= nbr[e - 1];
    for (int o = 16; o >= 1; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(bad, b);
}

// bad[0] counts arcs not strictly above their predecessor in the row
__global__ void k_rows_sorted(const uint32_t* __restrict__ off, const int32_t* __restrict__ nbr, int64_t n,
                              unsigned long long* bad) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
    unsigned long long b = 0;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; v < n; v += warps)
        for (uint32_t e = off[v] + 1 + lane; e < off[v + 1]; e += 32) b += nbr[e] <= nbr[e - 1];
    if (b) atomicAdd(bad, b);
}

// bad[0] counts decreasing offsets
__global__ void k_offsets_check(const int64_t* __restrict__ off, int64_t n, unsigned long long* bad) {
    unsigned long long b = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        b += off[v + 1] < off[v];
    if (b) atomicAdd(bad, b);
}

// neighbours -> int32 with range check; bad[0] counts out-of-range ids
// neighbours [lo, hi) -> int32 with the range check (bad[0]) and the
// strictly-increasing-rows check (sorted_bad[0]: arcs that are not a row start
// and not above their predecessor; the arc before lo is already converted)
__global__ void k_nbr_convert_check(const int64_t* __restrict__ in, int32_t* __restrict__ out,
                                    const uint8_t* __restrict__ start, int64_t lo, int64_t hi, int64_t n,
                                    unsigned long long* bad, unsigned long long* sorted_bad) {
    unsigned long long nbad = 0, nuns = 0;
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = in[i];
        nbad += (v < 0 || v >= n);
        out[i] = (int32_t)v;
        if (i > 0 && !start[i]) {
            const int64_t prev = i > lo ? in[i - 1] : (int64_t)out[i - 1];
            nuns += v <= prev;
        }
    }
    for (int o = 16; o >= 1; o >>= 1) {
        nbad += __shfl_xor_sync(0xffffffffu, nbad, o);
        nuns += __shfl_xor_sync(0xffffffffu, nuns, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (nbad) atomicAdd(bad, nbad);
        if (nuns) atomicAdd(sorted_bad, nuns);
    }
}

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

// [0] max degree, [1] rows longer than two slices, [2] their largest
// global slice tables (slots), summed
__global__ void k_degree_stats(const uint32_t* __restrict__ off, int64_t n, unsigned long long* out) {
    unsigned long long mx = 0, sl = 0, slots = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long d = off[v + 1] - off[v];
        mx = max(mx, d);
        if (d > 2ull * kSliceArcs) {
            ++sl;
            unsigned long long t = 1ull << kGlobalBits;
            while (t < 2 * d + 64) t <<= 1;
            slots += t;
        }
    }
    atomicMax(out, mx);
    if (sl) atomicAdd(out + 1, sl);
    if (slots) atomicAdd(out + 2, slots);
}

__global__ void k_plan_pos(const int64_t* __restrict__ order, int32_t* __restrict__ pos, int64_t n,
                           unsigned long long* bad) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = order[p];
        if (v < 0 || v >= n) {
            atomicAdd(bad, 1ull);
            continue;
        }
        pos[v] = (int32_t)p;
    }
}

// every vertex must own exactly one position: pos[] was preset to -1
__global__ void k_plan_check_perm(const int64_t* __restrict__ order, const int32_t* __restrict__ pos, int64_t n,
                                  unsigned long long* bad) {
    unsigned long long b = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = pos[v];
        b += (p < 0 || order[p] != v);
    }
    if (b) atomicAdd(bad, b);
}

// storage sort key per vertex: bin in bits 32..34; big rows by descending
// degree (the dense route then hands out the largest hubs first); inside a
// small class vertex-id order (neighbouring rows share neighbours: locality
// for the label gathers)
// arcs of row v that are not its self-loop (INDEX plans)
__device__ __forceinline__ uint32_t row_degree(const uint32_t* __restrict__ off, const int32_t* __restrict__ nbr,
                                               int64_t v, int noself) {
    const uint32_t b = off[v], e = off[v + 1];
    if (!noself) return e - b;
    uint32_t selfs = 0;
    for (uint32_t i = b; i < e; ++i) selfs += nbr[i] == (int32_t)v;
    return e - b - selfs;
}

__global__ void k_plan_keys(const uint32_t* __restrict__ off, const int32_t* __restrict__ nbr,
                            unsigned long long* __restrict__ key, int64_t n, unsigned long long* counts,
                            uint32_t* __restrict__ deg, int noself) {
    __shared__ unsigned long long sc[kNumBins];
    if (threadIdx.x < kNumBins) sc[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t d = row_degree(off, nbr, v, noself);
        deg[v] = d;
        int b;
        if (d == 0 || (!noself && d == 1 && nbr[off[v]] == (int32_t)v))
            b = kBinIdle;  // RAK: label provably cannot move; INDEX: no speaker / contributor
        else if (d > (uint32_t)kSmallMax)
            b = kBinBig;
        else
            b = d > 8 ? kBinS16 : (d > 4 ? kBinS8 : kBinS4);
        key[v] = ((unsigned long long)b << 32) | (b == kBinBig ? (0xffffffffull - d) : 0ull);
        atomicAdd(&sc[b], 1ull);
    }
    __syncthreads();
    if (threadIdx.x < kNumBins && sc[threadIdx.x]) atomicAdd(counts + threadIdx.x, sc[threadIdx.x]);
}

// first slot of [0, big_end) (rows by descending degree) whose degree is <= maxd
__global__ void k_first_short(const uint32_t* __restrict__ soff, int32_t big_end, int maxd, int32_t* first) {
    for (int32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < big_end; s += gridDim.x * blockDim.x) {
        const bool shortrow = (int)(soff[s + 1] - soff[s]) <= maxd;
        const bool prev_long = s == 0 || (int)(soff[s] - soff[s - 1]) > maxd;
        if (shortrow && prev_long) atomicMin(first, s);
    }
}

__global__ void k_plan_vorder(const int32_t* __restrict__ pos, int32_t* __restrict__ vorder, int64_t n) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        vorder[pos[v]] = (int32_t)v;
}

__global__ void k_iota64(int64_t* a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = i;
}

__global__ void k_iota(int32_t* a, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a[i] = (int32_t)i;
}

__global__ void k_plan_slots(const int32_t* __restrict__ svid, const uint32_t* __restrict__ deg,
                             int32_t* __restrict__ slot_of, uint32_t* __restrict__ sdeg, int64_t n, int64_t S) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = svid[s];
        if (s < S) {
            slot_of[v] = (int32_t)s;
            sdeg[s] = deg[v];
        } else {
            slot_of[v] = -1;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) sdeg[S] = 0;
}

// distinct-label estimates restart from the degree at every run
__global__ void k_reset_ndist(const uint32_t* __restrict__ soff, int32_t* __restrict__ ndist, int64_t S) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S; s += (int64_t)gridDim.x * blockDim.x)
        ndist[s] = (int32_t)(soff[s + 1] - soff[s]);
}

// one warp per slot: copy the row (neighbour ids, flags cleared) and weights;
// INDEX plans drop the self-loop arcs (order of the others kept)
__global__ void k_plan_rows(const int32_t* __restrict__ svid, const uint32_t* __restrict__ off,
                            const int32_t* __restrict__ nbr, const uint32_t* __restrict__ w,
                            const uint32_t* __restrict__ soff, uint32_t* __restrict__ snbr, uint32_t* __restrict__ sw,
                            int64_t S, int noself) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
    for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; s < S; s += warps) {
        const int32_t v = svid[s];
        const uint32_t src = off[v], d = off[v + 1] - src;
        uint32_t dst = soff[s];
        for (uint32_t k0 = 0; k0 < d; k0 += 32) {
            const uint32_t k = k0 + lane;
            const int32_t u = k < d ? nbr[src + k] : -1;
            const bool keep = k < d && !(noself && u == v);
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const uint32_t o = dst + __popc(bal & lanemask_lt());
                snbr[o] = (uint32_t)u << 2;
                if (w) sw[o] = w[src + k];
            }
            dst += __popc(bal);
        }
    }
}

// RAK plans: copy the rows into the storage CSR as flat pieces (warps take 32
// pieces, eight arcs in flight per lane) and set the batch flags on the way.
__global__ void __launch_bounds__(256)
    k_plan_rows_pieces(const int32_t* __restrict__ svid, const uint32_t* __restrict__ off,
                       const int32_t* __restrict__ nbr, const uint32_t* __restrict__ w,
                       const uint32_t* __restrict__ soff, uint32_t* __restrict__ snbr, uint32_t* __restrict__ sw,
                       const int32_t* __restrict__ dslot, const int32_t* __restrict__ dk0,
                       const int32_t* __restrict__ dcount, int32_t* cursor, const int32_t* __restrict__ pos,
                       int64_t bs, int flags_on) {
    constexpr int J = 8;
    const int lane = threadIdx.x & 31;
    const int cnt = *dcount;
    while (true) {
        int b0 = 0;
        if (lane == 0) b0 = atomicAdd(cursor, 32);
        b0 = __shfl_sync(0xffffffffu, b0, 0);
        if (b0 >= cnt) break;
        uint32_t src = 0, dst = 0, plen = 0;
        int64_t bv = 0;
        if (b0 + lane < cnt) {
            const int32_t s = dslot[b0 + lane];
            const int32_t v = svid[s];
            const uint32_t k0 = (uint32_t)dk0[b0 + lane];
            src = off[v] + k0;
            dst = soff[s] + k0;
            plen = min((uint32_t)kPieceArcs, soff[s + 1] - dst);
            if (flags_on) bv = (int64_t)pos[v] / bs;
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
            uint32_t se[J], de[J];
            int32_t u[J];
            long long bvj[J];
#pragma unroll
            for (int j = 0; j < J; ++j) {
                const uint32_t i = base + j * 32 + lane;
                int r = 0;
#pragma unroll
                for (int step = 16; step >= 1; step >>= 1) {
                    const uint32_t ex = __shfl_sync(0xffffffffu, excl, r + step);
                    if (r + step < 32 && ex <= i) r += step;
                }
                const uint32_t pe = __shfl_sync(0xffffffffu, excl, r);
                se[j] = __shfl_sync(0xffffffffu, src, r) + (i - pe);
                de[j] = __shfl_sync(0xffffffffu, dst, r) + (i - pe);
                bvj[j] = __shfl_sync(0xffffffffu, bv, r);
                u[j] = i < total ? nbr[se[j]] : -1;
            }
#pragma unroll
            for (int j = 0; j < J; ++j) {
                if (u[j] < 0) continue;
                uint32_t f = 0;
                if (flags_on) {
                    const int64_t bu = (int64_t)pos[u[j]] / bs;
                    f = (bu < bvj[j] ? kEarlier : 0u) | (bu > bvj[j] ? kLater : 0u);
                }
                snbr[de[j]] = ((uint32_t)u[j] << 2) | f;
                if (w) sw[de[j]] = w[se[j]];
            }
        }
    }
}

// INDEX plans: pieces (slot, first arc) of every active row, for phase-1
// gathers that need the row of each arc
__global__ void k_plan_piece_counts(const uint32_t* __restrict__ soff, uint32_t* __restrict__ cnt, int64_t S) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s <= S; s += (int64_t)gridDim.x * blockDim.x)
        cnt[s] = s < S ? (soff[s + 1] - soff[s] + kPieceArcs - 1) / kPieceArcs : 0u;
}
__global__ void k_plan_pieces(const uint32_t* __restrict__ soff, const uint32_t* __restrict__ pbeg,
                              int32_t* __restrict__ dslot, int32_t* __restrict__ dk0, int64_t S) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S; s += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t np = pbeg[s + 1] - pbeg[s];
        for (uint32_t q = 0; q < np; ++q) {
            dslot[pbeg[s] + q] = (int32_t)s;
            dk0[pbeg[s] + q] = (int32_t)(q * kPieceArcs);
        }
    }
}

// batch flags of every arc for batch size bs: kEarlier when the neighbour's
// batch precedes the row vertex's, kLater when it follows (bs >= n: none)
__global__ void k_set_flags(const int32_t* __restrict__ svid, const int32_t* __restrict__ pos,
                            const uint32_t* __restrict__ soff, uint32_t* __restrict__ snbr, int64_t S, int64_t bs,
                            int clear_only) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
    for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; s < S; s += warps) {
        const int64_t bv = clear_only ? 0 : (int64_t)pos[svid[s]] / bs;
        for (uint32_t e = soff[s] + lane; e < soff[s + 1]; e += 32) {
            const uint32_t nb = snbr[e] & ~3u;
            uint32_t f = 0;
            if (!clear_only) {
                const int64_t bu = (int64_t)pos[nb >> 2] / bs;
                f = (bu < bv ? kEarlier : 0u) | (bu > bv ? kLater : 0u);
            }
            snbr[e] = nb | f;
        }
    }
}

// per-slot total of the fixed-point row weights (majority test)
__global__ void k_plan_wsum(const uint32_t* __restrict__ soff, const uint32_t* __restrict__ sw,
                            unsigned long long* __restrict__ swsum, int64_t S) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
    for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; s < S; s += warps) {
        unsigned long long acc = 0;
        for (uint32_t e = soff[s] + lane; e < soff[s + 1]; e += 32) acc += sw[e];
        for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) swsum[s] = acc;
    }
}

__global__ void k_init_labels(const int64_t* __restrict__ init, int32_t* __restrict__ lab, int64_t n) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        lab[v] = init ? (int32_t)init[v] : (int32_t)v;
}

__global__ void k_check_labels(const int64_t* __restrict__ init, int64_t n, unsigned long long* bad) {
    unsigned long long b = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        b += (init[i] < 0 || init[i] >= n);
    if (b) atomicAdd(bad, b);
}

__global__ void k_labels_to64(const int32_t* __restrict__ lab, int64_t* __restrict__ out, int64_t n) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        out[v] = lab[v];
}

__global__ void k_gtab_init(int32_t* keys, uint32_t* first, unsigned long long* acc, int64_t count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = kEmpty;
        first[i] = 0xffffffffu;
        acc[i] = 0ull;
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
    int64_t slot_launches[kKSlots + 1] = {0, 0, 0, 0, 0};
    std::vector<cudaEvent_t>* pool = nullptr;
    std::vector<int> tags;  // kernel slot per pair, -1 = routing
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
        ++launches;
        if (tag >= 0) ++slot_launches[tag];
        if (!on) return;
        tags.push_back(tag);
        cudaEventRecord(next(), st);
    }
    void end(cudaStream_t st) {
        if (on) cudaEventRecord(next(), st);
    }
};

template <int WM, int TIE> struct Launcher {
    using A = typename Acc<WM>::T;
    static int occ_warp[2], occ_team, occ_team2, occ_hub, occ_mid, occ_midh, occ_loop, done_device;
    template <int WC> static cudaError_t setup_warp() {
        cudaError_t e;
        if constexpr (WM == kUnit || WM == kFixed) {
            e = cudaFuncSetAttribute(k_warp<WM, TIE, WC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)warp_smem_bytes<WM, WC>());
            if (e) return e;
        }
        e = cudaFuncSetAttribute(k_warp<WM, TIE, WC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)warp_smem_bytes<WM, WC>());
        if (e) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_warp[WC], k_warp<WM, TIE, WC, false>,
                                                          WarpClass<WC>::kWarps * 32, warp_smem_bytes<WM, WC>());
        occ_warp[WC] = std::max(occ_warp[WC], 1);
        return e;
    }
    static cudaError_t setup(int device) {
        if (done_device == device) return cudaSuccess;
        cudaError_t e;
        if ((e = setup_warp<0>())) return e;
        if ((e = setup_warp<1>())) return e;
        e = cudaFuncSetAttribute(k_team<WM, TIE, kTeamThreads, kTeamBits, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)team_smem_bytes<WM, kTeamBits>());
        if (e) return e;
        e = cudaFuncSetAttribute(k_mid<WM, TIE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mid_smem_bytes<WM>());
        if (e) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_mid, k_mid<WM, TIE>, kMidThreads, mid_smem_bytes<WM>());
        if (e) return e;
        occ_mid = std::max(occ_mid, 1);
        if constexpr (WM == kUnit) {
            e = cudaFuncSetAttribute(k_midh<TIE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mid_hash_smem_bytes());
            if (e) return e;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_midh, k_midh<TIE>, kMidHThreads, mid_hash_smem_bytes());
            if (e) return e;
            occ_midh = std::max(occ_midh, 1);
        }
        e = cudaFuncSetAttribute(k_team<WM, TIE, kTeam2Threads, kTeam2Bits, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)team_smem_bytes<WM, kTeam2Bits>());
        if (e) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_team2, k_team<WM, TIE, kTeam2Threads, kTeam2Bits, true>,
                                                          kTeam2Threads, team_smem_bytes<WM, kTeam2Bits>());
        if (e) return e;
        occ_team2 = std::max(occ_team2, 1);
        e = cudaFuncSetAttribute(k_team<WM, TIE, kHubThreads, kHubBits, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)team_smem_bytes<WM, kHubBits>());
        if (e) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_team, k_team<WM, TIE, kTeamThreads, kTeamBits, false>,
                                                          kTeamThreads, team_smem_bytes<WM, kTeamBits>());
        if (e) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_hub, k_team<WM, TIE, kHubThreads, kHubBits, true>,
                                                          kHubThreads, team_smem_bytes<WM, kHubBits>());
        if (e) return e;
        occ_team = std::max(occ_team, 1);
        occ_hub = std::max(occ_hub, 1);
        e = cudaFuncSetAttribute(k_frontier_loop<WM, TIE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)loop_smem_bytes<WM>());
        if (e) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_loop, k_frontier_loop<WM, TIE>, kLoopWarps * 32,
                                                          loop_smem_bytes<WM>());
        if (e) return e;
        occ_loop = std::max(occ_loop, 1);
        done_device = device;
        return cudaSuccess;
    }
    template <int WC>
    static void launch_warp(lp_graph* g, EvalArgs a, int64_t cnt, bool dense, Prof* prof, cudaStream_t s) {
        const int sms = g->num_sms;
        a.bin = kKWarp;
        prof->begin(s, kKWarp);
        // (frontier rounds: a warp per listed row up to the resident grid -- a late
        // round's few long rows each get their own warp instead of queueing
        // 32 deep behind one block's eight warps)
        const int per_block = WarpClass<WC>::kWarps;
        const int grid = dense ? sms * occ_warp[WC] : grid_for(cnt, per_block, sms * occ_warp[WC]);
        if constexpr (WM == kUnit || WM == kFixed) {
            if (a.id_single) {
                k_warp<WM, TIE, WC, true><<<grid, WarpClass<WC>::kWarps * 32, warp_smem_bytes<WM, WC>(), s>>>(a);
                prof->end(s);
                return;
            }
        }
        k_warp<WM, TIE, WC, false><<<grid, WarpClass<WC>::kWarps * 32, warp_smem_bytes<WM, WC>(), s>>>(a);
        prof->end(s);
    }
    // The frontier loop (lp_loop_kernels.cuh): rounds on the device until a round queues
    // nothing or the queue goes back to the class kernels; the caller reads g->loop_ctl.
    static cudaError_t loop(lp_graph* g, const EvalArgs& a, const int32_t* list0, const int32_t* list0_len,
                            int list0_cnt, int first_dst, int dense, int max_queue) {
        const Plan& P = g->plan();
        EvalArgs b = a;
        b.bin = kKWarp;
        int32_t* q0 = g->mq[0];
        int32_t* q1 = g->mq[1];
        const int32_t* slot_of = P.slot_of;
        LoopCtl* ctl = g->loop_ctl;
        int32_t* mq_len = g->mq_len;
        int max_rounds = 1 << 20;
        void* args[] = {&b, &list0, &list0_len, &list0_cnt, &q0, &q1, &first_dst, &slot_of, &ctl, &mq_len, &dense, &max_queue,
                        &max_rounds};
#ifdef LP_LOOP_TEST_FAIL
        return cudaErrorCooperativeLaunchTooLarge;  // (test build: the caller's fallback path)
#endif
        const int per_sm = g->loop_blocks_per_sm > 0 ? std::min(g->loop_blocks_per_sm, occ_loop) : occ_loop;
        return cudaLaunchCooperativeKernel((const void*)k_frontier_loop<WM, TIE>, dim3(g->num_sms * per_sm),
                                           dim3(kLoopWarps * 32), args, loop_smem_bytes<WM>(), g->stream);
    }
    // One round.  dense: k_small sweeps the small slot range and the other
    // slots are routed; frontier: everything comes from the marked route.
    static void round(lp_graph* g, EvalArgs a, bool dense, const int32_t* h_len, Prof* prof, int alg) {
        const Plan& P = g->plan();
        const int sms = g->num_sms;
        cudaStream_t st = g->stream;
        // Fused gathers (RAK): rows of degree <= fuse_maxd gather their
        // neighbour labels inside the tally kernel (arc_label); the phase-1 pass
        // covers only the longer rows, which come first in storage order.
        const bool rak = alg == kGatherRak;
        const bool fuse_all = rak && g->run_fuse >= (1 << 30);
        const bool fuse_small = rak && g->run_fuse >= kSmallMax;
        const bool fuse_mid = rak && a.mid_max > 0 && g->run_fuse >= a.mid_max;
        const int64_t gather_arcs = fuse_all ? 0 : fuse_mid ? P.arcs_gt_mid : fuse_small ? P.arcs_gt16 : P.m_active;
        EvalArgs af = a, ag = a;  // fused / two-phase launches
        af.fused = 1;
        ag.fused = fuse_all ? 1 : 0;
        // The tally kernels of a round are independent except for the spill chain
        // warp<0> -> warp<1> -> team (overflowing rows move up a class), so they
        // run on three streams: the chain on the handle's stream, the small and
        // mid rows and team2 on aux[0], the hubs on aux[1]; their tails overlap.
        // Fused small rows start at once, beside the phase-1 gather.
        // (Running the routed lists of the chain concurrently and the spills
        // afterwards, on a fourth stream, measured slower: the kernels share the
        // SMs' shared memory, the round is throughput-bound.)
        cudaStream_t sB = g->aux[0], sC = g->aux[1];
        cudaEventRecord(g->ev_fork, st);
        cudaStreamWaitEvent(sB, g->ev_fork, 0);
        cudaStreamWaitEvent(sC, g->ev_fork, 0);
        auto small_rows = [&](const EvalArgs& sa) {
            // small rows, one launch per degree class (MAXD 16, 8, 4)
            for (int c = 0; c < 3; ++c) {
                const int bin = kBinS16 + c;
                const int list = kLenS16 - c;
                const int64_t cnt = dense ? (P.bin_beg[bin + 1] - P.bin_beg[bin]) : h_len[list];
                if (cnt <= 0) continue;
                const int32_t sb = dense ? P.bin_beg[bin] : -1, se = dense ? P.bin_beg[bin + 1] : -1;
                EvalArgs b = sa;
                b.bin = kKSmall;
                prof->begin(sB, kKSmall);
                const int grid = grid_for(cnt, 256, sms * 8);
                if (c == 0)
                    k_small<WM, TIE, 16><<<grid, 256, 0, sB>>>(b, sb, se);
                else if (c == 1)
                    k_small<WM, TIE, 8><<<grid, 256, 0, sB>>>(b, sb, se);
                else
                    k_small<WM, TIE, 4><<<grid, 256, 0, sB>>>(b, sb, se);
                prof->end(sB);
            }
        };
        auto join = [&]() {
            cudaEventRecord(g->ev_join[0], sB);
            cudaEventRecord(g->ev_join[1], sC);
            cudaStreamWaitEvent(st, g->ev_join[0], 0);
            cudaStreamWaitEvent(st, g->ev_join[1], 0);
        };
        if (fuse_small) small_rows(af);
        // ---- route the big rows (dense rounds) ----
        if (dense && P.big_end > 0) {
            prof->begin(st, -1);
            k_route_dense<<<grid_for(P.big_end, 256, sms * 8), 256, 0, st>>>(a, 0, P.big_end);
            prof->end(st);
        }
        cudaEventRecord(g->ev_route, st);
        // ---- phase 1: gather the neighbour labels of the two-phase rows ----
        if (alg == kGatherSlpa) {
            prof->begin(st, kKGather);
            if (dense)
                k_gather_pieces<kGatherSlpa><<<grid_for(P.npieces, 32 * 8, sms * 16), 256, 0, st>>>(
                    a, P.dslot, P.dk0, P.dcount, a.r.len + kGatherCursor);
            else
                k_gather_pieces<kGatherSlpa><<<grid_for(h_len[kLenGather], 4 * 8, sms * 16), 256, 0, st>>>(
                    a, a.r.gslot, a.r.gk0, a.r.len + kLenGather, a.r.len + kGatherCursor);
            prof->end(st);
        } else if (fuse_all) {
        } else if (dense) {
            if (gather_arcs > 0) {
                prof->begin(st, kKGather);
                k_gather_dense<<<grid_for(gather_arcs, 256 * 8, sms * 16), 256, 0, st>>>(a, gather_arcs);
                prof->end(st);
            }
        } else if (h_len[kLenGather] > 0) {
            prof->begin(st, kKGather);
            k_gather_pieces<kGatherRak><<<grid_for(h_len[kLenGather], 4 * 8, sms * 16), 256, 0, st>>>(
                a, a.r.gslot, a.r.gk0, a.r.len + kLenGather, a.r.len + kGatherCursor);
            prof->end(st);
        }
        cudaEventRecord(g->ev_gather, st);
        const bool big = dense && P.big_end > 0;
        auto hub_rows = [&]() {
            if (!(big || h_len[kLenHub] > 0)) return;
            cudaStreamWaitEvent(sC, g->ev_gather, 0);
            EvalArgs b = ag;
            b.bin = kKHub;
            prof->begin(sC, kKHub);
            if (b.hb_off) k_hub_bucket<<<sms * 2, 1024, 0, sC>>>(b);
            const int grid = dense ? sms * occ_hub : grid_for(h_len[kLenHub], 1, sms * occ_hub);
            k_team<WM, TIE, kHubThreads, kHubBits, true>
                <<<grid, kHubThreads, team_smem_bytes<WM, kHubBits>(), sC>>>(b, kLenHub);
            prof->end(sC);
        };
        // ---- phase 2: tally ----
        if (!fuse_small) {
            cudaStreamWaitEvent(sB, g->ev_gather, 0);
            small_rows(ag);
        }
        if (a.mid_max > 0 && (big || h_len[kLenMid] > 0)) {
            cudaStreamWaitEvent(sB, fuse_mid ? g->ev_route : g->ev_gather, 0);
            EvalArgs b = fuse_mid ? af : ag;
            b.bin = kKSmall;
            prof->begin(sB, kKSmall);
            bool hashed = false;
            if constexpr (WM == kUnit) {
                if (g->mid_hash) {
                    const int grid = dense ? sms * occ_midh : grid_for(h_len[kLenMid], kMidHThreads, sms * occ_midh);
                    k_midh<TIE><<<grid, kMidHThreads, mid_hash_smem_bytes(), sB>>>(b);
                    hashed = true;
                }
            }
            if (!hashed) {
                const int grid = dense ? sms * occ_mid : grid_for(h_len[kLenMid], kMidThreads, sms * occ_mid);
                k_mid<WM, TIE><<<grid, kMidThreads, mid_smem_bytes<WM>(), sB>>>(b);
            }
            prof->end(sB);
        }
        if (big || h_len[kLenWarp] > 0) launch_warp<0>(g, ag, h_len[kLenWarp], dense, prof, st);
        // each class may spill into the next one: launch on any upstream work
        if (big || h_len[kLenWarp] + h_len[kLenWarpBig] > 0)
            launch_warp<1>(g, ag, h_len[kLenWarp] + h_len[kLenWarpBig], dense, prof, st);
        if (big || (h_len[kLenWarp] + h_len[kLenWarpBig] + h_len[kLenTeam]) > 0) {
            EvalArgs b = ag;
            b.bin = kKTeam;
            prof->begin(st, kKTeam);
            k_team<WM, TIE, kTeamThreads, kTeamBits, false>
                <<<sms * occ_team, kTeamThreads, team_smem_bytes<WM, kTeamBits>(), st>>>(b, kLenTeam);
            prof->end(st);
        }
        if (big || h_len[kLenTeam2] > 0) {
            cudaStreamWaitEvent(sB, g->ev_gather, 0);
            EvalArgs b = ag;
            b.bin = kKTeam;
            prof->begin(sB, kKTeam);
            const int grid = dense ? sms * occ_team2 : grid_for(h_len[kLenTeam2], 1, sms * occ_team2);
            k_team<WM, TIE, kTeam2Threads, kTeam2Bits, true>
                <<<grid, kTeam2Threads, team_smem_bytes<WM, kTeam2Bits>(), sB>>>(b, kLenTeam2);
            prof->end(sB);
        }
        hub_rows();
        join();
        // (the deferred marks of the rows that changed this round are launched
        // by the sweep driver: mark_pass)
    }
};
template <int WM, int TIE> int Launcher<WM, TIE>::occ_warp[2] = {1, 1};
template <int WM, int TIE> int Launcher<WM, TIE>::occ_team = 1;
template <int WM, int TIE> int Launcher<WM, TIE>::occ_team2 = 1;
template <int WM, int TIE> int Launcher<WM, TIE>::occ_hub = 1;
template <int WM, int TIE> int Launcher<WM, TIE>::occ_mid = 1;
template <int WM, int TIE> int Launcher<WM, TIE>::occ_midh = 1;
template <int WM, int TIE> int Launcher<WM, TIE>::occ_loop = 1;
template <int WM, int TIE> int Launcher<WM, TIE>::done_device = -1;

typedef void (*round_fn)(lp_graph*, EvalArgs, bool, const int32_t*, Prof*, int);
typedef cudaError_t (*setup_fn)(int);

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

typedef cudaError_t (*loop_fn)(lp_graph*, const EvalArgs&, const int32_t*, const int32_t*, int, int, int, int);
template <int WM> static loop_fn pick_loop(int tie) {
    switch (tie) {
        case kRandom: return Launcher<WM, kRandom>::loop;
        case kMinLabel: return Launcher<WM, kMinLabel>::loop;
        default: return Launcher<WM, kScanFirst>::loop;
    }
}

// ---------------------------------------------------------------------------
// graph handle
// ---------------------------------------------------------------------------
static void free_plan(Plan& P) {
    dfree(P.pos);
    dfree(P.svid);
    dfree(P.slot_of);
    dfree(P.soff);
    dfree(P.snbr);
    dfree(P.sw);
    dfree(P.swsum);
    dfree(P.ndist);
    dfree(P.lbuf);
    dfree(P.hb_lab);
    dfree(P.hb_pos);
    dfree(P.vorder);
    dfree(P.wave_len);
    dfree(P.dslot);
    dfree(P.dk0);
    dfree(P.dcount);
    P = Plan();
}

static void free_routes(Routes& r) {
    for (int c = 0; c < 3; ++c) dfree(r.small[c]);
    dfree(r.warp[0]);
    dfree(r.warp[1]);
    dfree(r.team);
    dfree(r.team2);
    dfree(r.mid);
    dfree(r.hub);
    dfree(r.len);
    dfree(r.cand);
    dfree(r.cand_done);
    dfree(r.gkeys);
    dfree(r.gtl);
    dfree(r.gfirst);
    dfree(r.gacc);
    dfree(r.gcount);
    dfree(r.gslot);
    dfree(r.gk0);
    dfree(r.cslot);
    dfree(r.ck0);
    r = Routes();
}

static void destroy_graph(lp_graph* g) {
    if (!g) return;
    StreamScope ss(g->stream);
    for (Plan& P : g->plans) free_plan(P);
    free_routes(g->routes);
    dfree(g->mq[0]);
    dfree(g->mq[1]);
    dfree(g->mq_len);
    dfree(g->mbits);
    dfree(g->hb_off);
    dfree(g->slots);
    for (int i = 0; i < 2; ++i) {
        dfree(g->clabs[i]);
        dfree(g->cbels[i]);
        dfree(g->csize[i]);
        dfree(g->cbest[i]);
    }
    dfree(g->ccur);
    dfree(g->cbig);
    dfree(g->cmid);
    dfree(g->croute);
    dfree(g->croute_mark);
    dfree(g->gelab);
    dfree(g->geval);
    dfree(g->gefirst);
    dfree(g->grlab);
    dfree(g->grval);
    dfree(g->gfmap);
    dfree(g->gblab);
    dfree(g->gbval);
    dfree(g->gbc);
    dfree(g->gwc);
    dfree(g->gqs);
    dfree(g->gslab);
    dfree(g->gsval);
    dfree(g->off);
    dfree(g->nbr);
    dfree(g->w);
    dfree(g->labA);  // (labB lives in the same allocation)
    dfree(g->mark);
    dfree(g->gap);
    dfree(g->chg);
    dfree(g->counters);
    dfree(g->out64);
    dfree(g->cub_tmp);
    if (g->h_len) cudaFreeHost(g->h_len);
    dfree(g->loop_ctl);
    if (g->h_counters) cudaFreeHost(g->h_counters);
    for (cudaEvent_t e : g->event_pool) cudaEventDestroy(e);
    if (g->ev0) cudaEventDestroy(g->ev0);
    if (g->ev1) cudaEventDestroy(g->ev1);
    if (g->stream) {
        cudaStreamSynchronize(g->stream);  // the pool frees above are ordered on it
        cudaStreamDestroy(g->stream);
    }
    for (int i = 0; i < 2; ++i) {
        if (g->aux[i]) cudaStreamSynchronize(g->aux[i]);  // (shared streams: not destroyed)
        if (g->ev_join[i]) cudaEventDestroy(g->ev_join[i]);
    }
    if (g->ev_fork) cudaEventDestroy(g->ev_fork);
    if (g->ev_route) cudaEventDestroy(g->ev_route);
    if (g->ev_gather) cudaEventDestroy(g->ev_gather);
    delete g;
}

static int ensure_cub_tmp(lp_graph* g, size_t bytes) {
    if (bytes <= g->cub_tmp_bytes) return LP_OK;
    dfree(g->cub_tmp);
    g->cub_tmp = nullptr;
    g->cub_tmp_bytes = 0;
    LP_CK(pool_alloc(&g->cub_tmp, bytes));
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

struct TmpBufs {
    int64_t* order = nullptr;
    unsigned long long* key = nullptr;
    unsigned long long* key_sorted = nullptr;
    int32_t* iota = nullptr;
    uint32_t* sdeg = nullptr;
    uint32_t* deg = nullptr;
    ~TmpBufs() {
        dfree(deg);
        dfree(order);
        dfree(key);
        dfree(key_sorted);
        dfree(iota);
        dfree(sdeg);
    }
};

// shuffled_indices(n, seed) is a sequential Fisher-Yates pass (~17 ms for
// n = 2^22); the last (n, seed) result is kept process-wide, so fresh graph
// handles of the same size and seed (e.g. a re-uploaded graph) skip it.
static void cached_shuffle(int64_t n, uint32_t seed, int64_t* out) {
    static std::mutex mu;
    static int64_t c_n = -1;
    static uint32_t c_seed = 0;
    static std::vector<int64_t> c_order;
    std::lock_guard<std::mutex> lock(mu);
    if (c_n != n || c_seed != seed) {
        c_order.resize((size_t)n);
        lp_host_shuffled_indices(n, seed, c_order.data());
        c_n = n;
        c_seed = seed;
    }
    std::memcpy(out, c_order.data(), (size_t)n * sizeof(int64_t));
}

// Device copy of the last shuffled order per device (kept for the process),
// copied into `dst` on the handle's stream and completed while the lock is
// held (another thread may replace the shared copy right after).
static int device_shuffle(lp_graph* g, int64_t n, uint32_t seed, int64_t* dst) {
    struct Entry {
        int64_t n = -1;
        uint32_t seed = 0;
        int64_t* d = nullptr;
        size_t cap = 0;
    };
    static std::mutex mu;
    static Entry cache[64];
    std::lock_guard<std::mutex> lock(mu);
    Entry& e = cache[g->device & 63];
    if (e.n != n || e.seed != seed) {
        std::vector<int64_t> h((size_t)n);
        cached_shuffle(n, seed, h.data());
        if ((size_t)n > e.cap) {
            if (e.d) cudaFree(e.d);
            e.d = nullptr;
            e.cap = 0;
            LP_CK(cudaMalloc((void**)&e.d, std::max<size_t>((size_t)n, 1) * sizeof(int64_t)));
            e.cap = (size_t)n;
        }
        // (ordered on the handle's stream and completed before return: a pageable
        // cudaMemcpy may return before its DMA lands, and the handle's
        // non-blocking stream would then copy a stale order -- seen as a rare
        // "order is not a permutation" when consecutive runs change the order)
        LP_CK(cudaMemcpyAsync(e.d, h.data(), (size_t)n * sizeof(int64_t), cudaMemcpyHostToDevice, g->stream));
        LP_CK(cudaStreamSynchronize(g->stream));
        e.n = n;
        e.seed = seed;
    }
    LP_CK(cudaMemcpyAsync(dst, e.d, (size_t)n * sizeof(int64_t), cudaMemcpyDeviceToDevice, g->stream));
    LP_CK(cudaStreamSynchronize(g->stream));
    return LP_OK;
}

// Build (or reuse) the plan of a kind and visit order: positions, the
// degree-binned storage CSR (neighbour ids), the phase-1 label buffer.
// RAK plans follow `order_host` (NULL: shuffled_indices(n, seed)); INDEX
// plans use the identity order and ignore both.
static int build_plan(lp_graph* g, int kind, const int64_t* order_host, uint32_t seed, float* plan_ms,
                      int64_t bs_hint = -1) {
    const int64_t n = g->n;
    g->pk = kind;
    const bool index = kind == kPlanIndex;
    if (index) order_host = nullptr;
    const bool custom = order_host != nullptr;
    const uint64_t oh = custom ? hash_order(order_host, n) : 0;
    Plan& P = g->plan();
    *plan_ms = 0.f;
    if (P.valid && (index || (P.custom_order == custom && (custom ? P.order_hash == oh : P.seed == seed))))
        return LP_OK;
    g->bytes -= P.bytes;
    free_plan(P);
    // the visit order on the device: identity (INDEX), the caller's, or
    // shuffled_indices(n, seed) from the process-wide device cache
    cudaStream_t st = g->stream;
    LP_CK(cudaEventRecord(g->ev0, st));
    int64_t bytes = 0;
    LP_CK(dalloc(&P.pos, n, &bytes));
    LP_CK(dalloc(&P.svid, n, &bytes));
    LP_CK(dalloc(&P.slot_of, n, &bytes));
    LP_CK(dalloc(&P.ndist, n, &bytes));
    TmpBufs t;
    int64_t tmpb = 0;
    LP_CK(dalloc(&t.order, n, &tmpb));
    LP_CK(dalloc(&t.key, n, &tmpb));
    LP_CK(dalloc(&t.key_sorted, n, &tmpb));
    LP_CK(dalloc(&t.iota, n, &tmpb));
    LP_CK(dalloc(&t.sdeg, n + 1, &tmpb));
    LP_CK(dalloc(&t.deg, n, &tmpb));
    if (custom) {
        LP_CK(cudaMemcpyAsync(t.order, order_host, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    } else if (!index) {
        if (int rc = device_shuffle(g, n, seed, t.order)) return rc;
    } else {
        k_iota64<<<g->num_sms * 8, 256, 0, st>>>(t.order, n);
    }
    LP_CK(cudaMemsetAsync(g->counters, 0, 8 * sizeof(unsigned long long), st));
    LP_CK(cudaMemsetAsync(P.pos, 0xff, n * sizeof(int32_t), st));
    const int G = g->num_sms * 8;
    k_plan_pos<<<G, 256, 0, st>>>(t.order, P.pos, n, g->counters);
    k_plan_check_perm<<<G, 256, 0, st>>>(t.order, P.pos, n, g->counters);
    LP_CK(cudaMemcpyAsync(g->h_counters, g->counters, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    LP_CK(cudaStreamSynchronize(st));
    if (g->h_counters[0]) {
        free_plan(P);
        return lp_fail(LP_ERR_INVALID, "order is not a permutation of range(n)");
    }
    LP_CK(dalloc(&P.vorder, n, &bytes));
    k_plan_vorder<<<G, 256, 0, st>>>(P.pos, P.vorder, n);
    k_plan_keys<<<G, 256, 0, st>>>(g->off, g->nbr, t.key, n, g->counters + 1, t.deg, index ? 1 : 0);
    k_iota<<<G, 256, 0, st>>>(t.iota, n);
    size_t need = 0, need2 = 0;
    LP_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, t.key, t.key_sorted, t.iota, P.svid, (int)n, 0, 35, st));
    LP_CK(cub::DeviceScan::ExclusiveSum(nullptr, need2, t.sdeg, t.sdeg, (int)(n + 1), st));
    if (int rc = ensure_cub_tmp(g, std::max(need, need2))) return rc;
    LP_CK(cub::DeviceRadixSort::SortPairs(g->cub_tmp, need, t.key, t.key_sorted, t.iota, P.svid, (int)n, 0, 35, st));
    LP_CK(cudaMemcpyAsync(g->h_counters, g->counters, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    LP_CK(cudaStreamSynchronize(st));
    {
        int64_t acc = 0;
        for (int b = 0; b < kNumBins; ++b) {
            P.bin_beg[b] = (int32_t)acc;
            acc += (int64_t)g->h_counters[1 + b];
        }
        P.bin_beg[kNumBins] = (int32_t)acc;
    }
    P.big_end = P.bin_beg[kBinS16];
    P.S = P.bin_beg[kBinIdle];
    k_plan_slots<<<G, 256, 0, st>>>(P.svid, t.deg, P.slot_of, t.sdeg, n, P.S);
    LP_CK(dalloc(&P.soff, P.S + 1, &bytes));
    LP_CK(cub::DeviceScan::ExclusiveSum(g->cub_tmp, need2, t.sdeg, P.soff, (int)(P.S + 1), st));
    uint32_t m_active = 0;
    LP_CK(cudaMemcpyAsync(&m_active, P.soff + P.S, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    {
        // arcs of the rows longer than 16 / than mid_max (prefixes of the storage order)
        int32_t* first = reinterpret_cast<int32_t*>(g->counters + 8);
        const int32_t init = P.big_end;
        LP_CK(cudaMemcpyAsync(first, &init, sizeof(int32_t), cudaMemcpyHostToDevice, st));
        k_first_short<<<grid_for(P.big_end, 256, g->num_sms * 8), 256, 0, st>>>(P.soff, P.big_end,
                                                                                 std::max(g->mid_max, kSmallMax), first);
        uint32_t off2[2] = {0, 0};
        int32_t fs = 0;
        LP_CK(cudaMemcpyAsync(&fs, first, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        LP_CK(cudaMemcpyAsync(&off2[0], P.soff + P.big_end, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
        LP_CK(cudaMemcpyAsync(&off2[1], P.soff + fs, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
        P.arcs_gt16 = off2[0];
        P.arcs_gt_mid = off2[1];
    }
    P.m_active = m_active;
    LP_CK(dalloc(&P.snbr, P.m_active, &bytes));
    LP_CK(dalloc(&P.lbuf, P.m_active, &bytes));
    LP_CK(dalloc(&P.hb_lab, P.m_active, &bytes));
    LP_CK(dalloc(&P.hb_pos, P.m_active, &bytes));
    if (g->w) LP_CK(dalloc(&P.sw, P.m_active, &bytes));
    if (index)
        k_plan_rows<<<g->num_sms * 16, 256, 0, st>>>(P.svid, g->off, g->nbr, g->w, P.soff, P.snbr, P.sw, P.S, 1);
    {
        // dense piece list (reuses t.sdeg as the per-slot piece counts / offsets):
        // SLPA's dense gathers, the pull marks at sweep boundaries, the RAK row copy
        k_plan_piece_counts<<<G, 256, 0, st>>>(P.soff, t.sdeg, P.S);
        LP_CK(cub::DeviceScan::ExclusiveSum(g->cub_tmp, need2, t.sdeg, t.sdeg, (int)(P.S + 1), st));
        uint32_t np = 0;
        LP_CK(cudaMemcpyAsync(&np, t.sdeg + P.S, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
        P.npieces = np;
        LP_CK(dalloc(&P.dslot, np, &bytes));
        LP_CK(dalloc(&P.dk0, np, &bytes));
        LP_CK(dalloc(&P.dcount, 1, &bytes));
        const int32_t npi = (int32_t)np;
        LP_CK(cudaMemcpyAsync(P.dcount, &npi, sizeof(int32_t), cudaMemcpyHostToDevice, st));
        k_plan_pieces<<<G, 256, 0, st>>>(P.soff, t.sdeg, P.dslot, P.dk0, P.S);
    }
    int64_t flags_key = -1;
    if (!index) {
        // RAK rows: flat piece copy with the batch flags of this run's batch size
        const bool none = bs_hint <= 0 || bs_hint >= n;
        flags_key = none ? n : bs_hint;
        LP_CK(cudaMemsetAsync(g->routes.len + kGatherCursor, 0, sizeof(int32_t), st));
        k_plan_rows_pieces<<<g->num_sms * 16, 256, 0, st>>>(P.svid, g->off, g->nbr, g->w, P.soff, P.snbr, P.sw,
                                                          P.dslot, P.dk0, P.dcount, g->routes.len + kGatherCursor,
                                                          P.pos, none ? 1 : bs_hint, none ? 0 : 1);
    }
    if (g->wmode == kFixed && P.S > 0) {
        LP_CK(dalloc(&P.swsum, P.S, &bytes));
        k_plan_wsum<<<g->num_sms * 16, 256, 0, st>>>(P.soff, P.sw, P.swsum, P.S);
    }
    LP_CK(cudaGetLastError());
    LP_CK(cudaEventRecord(g->ev1, st));
    LP_CK(cudaEventSynchronize(g->ev1));
    LP_CK(cudaEventElapsedTime(plan_ms, g->ev0, g->ev1));
    P.valid = true;
    P.kind = kind;
    P.custom_order = custom;
    P.seed = seed;
    P.order_hash = oh;
    P.flags_bs = flags_key;
    P.bytes = bytes;
    g->bytes += bytes;
    return LP_OK;
}

// (Re)compute the batch flags of the storage CSR for batch size bs.
static int ensure_flags(lp_graph* g, int64_t bs, float* ms) {
    Plan& P = g->plan();
    const bool none = bs >= g->n;  // one batch: no cross-batch reads or marks
    const int64_t key = none ? g->n : bs;
    if (P.flags_bs == key) return LP_OK;
    if (P.S > 0) {
        LP_CK(cudaEventRecord(g->ev0, g->stream));
        k_set_flags<<<g->num_sms * 16, 256, 0, g->stream>>>(P.svid, P.pos, P.soff, P.snbr, P.S, none ? 1 : bs,
                                                           none ? 1 : 0);
        LP_CK(cudaGetLastError());
        LP_CK(cudaEventRecord(g->ev1, g->stream));
        LP_CK(cudaEventSynchronize(g->ev1));
        float e = 0.f;
        LP_CK(cudaEventElapsedTime(&e, g->ev0, g->ev1));
        *ms += e;
    }
    P.flags_bs = key;
    return LP_OK;
}

static cudaError_t alloc_routes(lp_graph* g) {
    Routes& r = g->routes;
    const int64_t n = std::max<int64_t>(g->n, 1);
    // hub items: one per partition (<= est / kHubPlan + 1) or per slice
    g->cap_items = n + g->m / (kHubPlan / 2) + g->m / kSliceArcs + 1024;
    // slice-table pool: every sliceable row at its largest table (2^bits >= 2 d + 64)
    const int64_t gpool = std::max<int64_t>(g->slice_slots, (int64_t)1 << kGlobalBits);
    r.gcap = gpool;
    cudaError_t e;
    for (int c = 0; c < 3; ++c)
        if ((e = dalloc(&r.small[c], n, &g->bytes))) return e;
    if ((e = dalloc(&r.warp[0], n, &g->bytes))) return e;
    if ((e = dalloc(&r.warp[1], n, &g->bytes))) return e;
    if ((e = dalloc(&r.team, 2 * n, &g->bytes))) return e;
    if ((e = dalloc(&r.team2, n, &g->bytes))) return e;
    if ((e = dalloc(&r.mid, n, &g->bytes))) return e;
    if ((e = dalloc(&r.hub, g->cap_items, &g->bytes))) return e;
    if ((e = dalloc(&r.len, kLenCount, &g->bytes))) return e;
    if ((e = dalloc(&r.cand, g->cap_items, &g->bytes))) return e;
    if ((e = dalloc(&g->hb_off, g->cap_items, &g->bytes))) return e;
    if ((e = dalloc(&r.cand_done, g->cap_items, &g->bytes))) return e;
    if ((e = dalloc(&r.gcount, g->cap_items, &g->bytes))) return e;
    if ((e = dalloc(&r.gkeys, gpool, &g->bytes))) return e;
    if ((e = dalloc(&r.gtl, gpool, &g->bytes))) return e;
    if ((e = dalloc(&r.gfirst, gpool, &g->bytes))) return e;
    if ((e = dalloc(&r.gacc, gpool, &g->bytes))) return e;
    // phase-1 pieces: one per row plus one per extra kPieceArcs arcs
    const int64_t pieces = n + g->m / kPieceArcs + 1;
    if ((e = dalloc(&r.gslot, pieces, &g->bytes))) return e;
    if ((e = dalloc(&r.gk0, pieces, &g->bytes))) return e;
    if ((e = dalloc(&r.cslot, pieces, &g->bytes))) return e;
    if ((e = dalloc(&r.ck0, pieces, &g->bytes))) return e;
    if ((e = cudaMemsetAsync(r.cand_done, 0, g->cap_items * sizeof(int32_t), g->stream))) return e;
    if ((e = cudaMemsetAsync(r.gcount, 0, g->cap_items * sizeof(int32_t), g->stream))) return e;
    k_gtab_init<<<g->num_sms * 4, 256, 0, g->stream>>>(r.gkeys, r.gfirst, r.gacc, gpool);
    return cudaGetLastError();
}

extern "C" int lp_graph_create(int64_t n, int64_t m, const int64_t* offsets, const int64_t* neighbors,
                               const double* weights, int32_t device, lp_graph** out) {
    if (!out) return lp_fail(LP_ERR_INVALID, "out is NULL");
    *out = nullptr;
    if (n < 0 || m < 0) return lp_fail(LP_ERR_INVALID, "negative vertex or edge count");
    if (n >= ((int64_t)1 << 30)) return lp_fail(LP_ERR_UNSUPPORTED, "vertex count must be < 2^30");
    if (m >= (int64_t)INT32_MAX) return lp_fail(LP_ERR_UNSUPPORTED, "edge count must be < 2^31-1");
    if (n > 0 && !offsets) return lp_fail(LP_ERR_INVALID, "offsets is NULL");
    if (m > 0 && !neighbors) return lp_fail(LP_ERR_INVALID, "neighbors is NULL");
    if (n > 0 && (offsets[0] != 0 || offsets[n] != m))
        return lp_fail(LP_ERR_INVALID, "offsets must start at 0 and end at edge_count");
    // (monotonicity of offsets is checked on the device after the upload)
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return lp_fail(LP_ERR_CUDA, "no CUDA device available (liblabelprop_cuda needs a B200)");
    if (device >= 0) LP_CK(cudaSetDevice(device));
    lp_graph* g = new lp_graph();
    auto fail = [&](int code) {
        destroy_graph(g);
        return code;
    };
    if (cudaGetDevice(&g->device) != cudaSuccess) return fail(lp_fail(LP_ERR_CUDA, "cudaGetDevice failed"));
    cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->device);
    if (const char* ev = getenv("LP_L2_PERSIST")) g->l2_persist = atoi(ev) != 0;
    if (const char* ev = getenv("LP_FUSE_MAXD")) {
        g->fuse_maxd = atoi(ev) < 0 ? (1 << 30) : atoi(ev);
        g->fuse_forced = true;
    }
    if (const char* ev = getenv("LP_COPRA_BITMAP")) g->copra_bitmap = atoi(ev) != 0;
    if (const char* ev = getenv("LP_COPRA_OVERLAP")) g->copra_overlap = atoi(ev) != 0;
    if (const char* ev = getenv("LP_COPRA_LONG")) g->copra_long = std::max(0, atoi(ev));
    if (const char* ev = getenv("LP_WAVES")) g->waves = std::max(1, std::min(1024, atoi(ev)));
    if (const char* ev = getenv("LP_LOOP_ROWS")) g->loop_rows = std::max(0, atoi(ev));
    if (const char* ev = getenv("LP_LOOP_DENSE_ARCS")) g->loop_dense_arcs = std::max(0, atoi(ev));
    if (const char* ev = getenv("LP_LOOP_MAX_QUEUE")) g->loop_max_queue = std::max(1, atoi(ev));
    if (const char* ev = getenv("LP_LOOP_BLOCKS")) g->loop_blocks_per_sm = std::max(0, atoi(ev));
    if (const char* ev = getenv("LP_MARGIN")) g->margin_skip = atoi(ev) != 0;
    if (const char* ev = getenv("LP_DEBUG_ROUNDS")) g->debug_rounds = atoi(ev) != 0;
    if (const char* ev = getenv("LP_DENSE_FRAC")) g->dense_frac = atof(ev);
    if (const char* ev = getenv("LP_PULL_ROUNDS")) g->pull_rounds = atoi(ev) != 0;
    if (const char* ev = getenv("LP_PULL_MAX")) g->pull_max_frac = atof(ev);
    if (const char* ev = getenv("LP_FIRST_ROUND")) g->first_round_shortcut = atoi(ev) != 0;
    if (const char* ev = getenv("LP_FIRST_CHAIN")) g->first_chain = atoi(ev) != 0;
    if (const char* ev = getenv("LP_SWEEP_FRONTIER")) g->sweep_frontier = atoi(ev) != 0;
    if (const char* ev = getenv("LP_CARRY_FRAC")) g->carry_frac = atof(ev);
    if (const char* ev = getenv("LP_CAP_ROUTE")) g->cap_route = atoi(ev) != 0;
    if (const char* ev = getenv("LP_ID_SINGLE")) g->id_single = atoi(ev) != 0;
    if (const char* ev = getenv("LP_PUSH_DIV")) g->push_div = std::max(1, atoi(ev));
    if (const char* ev = getenv("LP_ID_SINGLE_RANDOM")) g->id_single_random = atoi(ev) != 0;
    if (const char* ev = getenv("LP_ID_SINGLE_W")) g->id_single_w = atoi(ev) != 0;
    if (const char* ev = getenv("LP_TWO_TEAM_W")) g->two_team_w = atoi(ev) != 0;
    if (const char* ev = getenv("LP_REG_EST")) g->reg_est = std::max(0, std::min(32, atoi(ev)));
    if (const char* ev = getenv("LP_MID_MAX")) g->mid_max = std::max(0, std::min(kMidMax, atoi(ev)));
    if (const char* ev = getenv("LP_MID_HASH")) g->mid_hash = atoi(ev) != 0;
    if (const char* ev = getenv("LP_HUB_BUCKET")) g->hub_bucket = atoi(ev) != 0;
    if (const char* ev = getenv("LP_MARK_BITMAP")) g->mark_bitmap = atoi(ev) != 0;
    if (const char* ev = getenv("LP_MARK_SCAN_DIV")) g->mark_scan_div = std::max(1, atoi(ev));
    if (const char* ev = getenv("LP_FIRST_EST_MIN")) g->first_est_min = std::max(16, atoi(ev));
    if (const char* ev = getenv("LP_FIRST_EST_DIV")) g->first_est_div = std::max(1, atoi(ev));
    if (const char* ev = getenv("LP_WARP0_MAXD")) g->warp_maxd[0] = std::max(17, std::min(WarpClass<0>::kMaxDeg, atoi(ev)));
    if (const char* ev = getenv("LP_WARP1_MAXD")) g->warp_maxd[1] = std::max(17, std::min(WarpClass<1>::kMaxDeg, atoi(ev)));
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
    {
        // the auxiliary tally streams are per device and live for the process
        // (creating / destroying streams per handle costs milliseconds)
        static std::mutex mu;
        static cudaStream_t pool[64][2];
        static bool made[64] = {};
        std::lock_guard<std::mutex> lock(mu);
        const int dv = g->device & 63;
        if (!made[dv]) {
            for (int i = 0; i < 2; ++i) G_CK(cudaStreamCreateWithFlags(&pool[dv][i], cudaStreamNonBlocking));
            made[dv] = true;
        }
        for (int i = 0; i < 2; ++i) {
            g->aux[i] = pool[dv][i];
            G_CK(cudaEventCreateWithFlags(&g->ev_join[i], cudaEventDisableTiming));
        }
    }
    G_CK(cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming));
    G_CK(cudaEventCreateWithFlags(&g->ev_route, cudaEventDisableTiming));
    G_CK(cudaEventCreateWithFlags(&g->ev_gather, cudaEventDisableTiming));
    StreamScope ss(g->stream);
    pool_keep(g->device);
    G_CK(cudaEventCreate(&g->ev0));
    G_CK(cudaEventCreate(&g->ev1));
    cudaStream_t st = g->stream;
    G_CK(dalloc(&g->off, n + 1, &g->bytes));
    G_CK(dalloc(&g->nbr, m, &g->bytes));
    // L0 / x side by side: one persisting L2 window covers both (set_l2_window)
    G_CK(dalloc(&g->labA, 2 * n + 32, &g->bytes));
    g->labB = g->labA + ((n + 31) & ~(int64_t)31);
    G_CK(dalloc(&g->mark, n + 4, &g->bytes));
    G_CK(dalloc(&g->gap, n + 4, &g->bytes));
    G_CK(dalloc(&g->chg, n / 32 + 2, &g->bytes));
    G_CK(dalloc(&g->mq[0], n + 4, &g->bytes));
    G_CK(dalloc(&g->mq[1], n + 4, &g->bytes));
    G_CK(dalloc(&g->mq_len, 4, &g->bytes));
    G_CK(dalloc(&g->mbits, n / 32 + 2, &g->bytes));
    G_CK(cudaMemsetAsync(g->mbits, 0, (n / 32 + 2) * sizeof(uint32_t), g->stream));
    G_CK(dalloc(&g->counters, 32, &g->bytes));
    G_CK(dalloc(&g->out64, n, &g->bytes));
    G_CK(cudaMallocHost((void**)&g->h_len, kLenCount * sizeof(int32_t)));
    G_CK(pool_alloc(&g->loop_ctl, sizeof(LoopCtl)));
    // (pinned: 32 counter words, then the frontier loop's control block)
    G_CK(cudaMallocHost((void**)&g->h_counters, 32 * sizeof(unsigned long long) + sizeof(LoopCtl)));
    g->h_loop = reinterpret_cast<LoopCtl*>(g->h_counters + 32);
    G_CK(cudaMemsetAsync(g->mark, 0, (n + 4) * sizeof(unsigned long long), st));
    G_CK(cudaMemsetAsync(g->gap, 0, (n + 4) * sizeof(unsigned long long), st));
    G_CK(cudaMemsetAsync(g->counters, 0, 32 * sizeof(unsigned long long), st));
    {
        // Upload pipeline: the host arrays go over PCIe on a copy stream (aux[1])
        // in chunks; the handle's stream converts and checks each chunk as it
        // lands (int64 -> int32, range, rows strictly increasing), so only the
        // last chunk's work trails the transfer.  Offsets first: the row-start
        // flags, degree statistics and route buffers are ready before the
        // neighbours finish arriving.
        int64_t* tmp = nullptr;
        int64_t tb = 0;
        G_CK(dalloc(&tmp, std::max(n + 1, m), &tb));
        cudaStream_t cs = g->aux[1];
        cudaEvent_t ev_copy = nullptr;
        G_CK(cudaEventCreateWithFlags(&ev_copy, cudaEventDisableTiming));
        struct EvGuard {
            cudaEvent_t e;
            ~EvGuard() { cudaEventDestroy(e); }
        } ev_guard{ev_copy};
        G_CK(cudaEventRecord(ev_copy, st));  // (the memsets above precede the copies)
        G_CK(cudaStreamWaitEvent(cs, ev_copy, 0));
        G_CK(cudaMemcpyAsync(tmp, offsets, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, cs));
        G_CK(cudaEventRecord(ev_copy, cs));
        G_CK(cudaStreamWaitEvent(st, ev_copy, 0));
        k_i64_to_u32<<<g->num_sms * 8, 256, 0, st>>>(tmp, g->off, n + 1);
        k_offsets_check<<<g->num_sms * 8, 256, 0, st>>>(tmp, n, g->counters + 11);
        k_degree_stats<<<g->num_sms * 8, 256, 0, st>>>(g->off, n, g->counters + 8);
        uint8_t* rs = nullptr;
        int64_t rb = 0;
        if (m > 0) {
            G_CK(dalloc(&rs, m, &rb));
            G_CK(cudaMemsetAsync(rs, 0, m, st));
            k_row_starts<<<g->num_sms * 8, 256, 0, st>>>(g->off, n, m, rs);
        }
        // (the neighbours may overwrite tmp once the offsets are converted)
        G_CK(cudaEventRecord(ev_copy, st));
        G_CK(cudaStreamWaitEvent(cs, ev_copy, 0));
        constexpr int64_t kChunk = (int64_t)1 << 25;  // 32M arcs = 256 MB per transfer
        std::vector<cudaEvent_t> evs;
        struct EvsGuard {
            std::vector<cudaEvent_t>& v;
            ~EvsGuard() {
                for (cudaEvent_t e : v) cudaEventDestroy(e);
            }
        } evs_guard{evs};
        for (int64_t lo = 0; lo < m; lo += kChunk) {
            const int64_t len = std::min(kChunk, m - lo);
            cudaEvent_t e = nullptr;
            G_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            evs.push_back(e);
            G_CK(cudaMemcpyAsync(tmp + lo, neighbors + lo, len * sizeof(int64_t), cudaMemcpyHostToDevice, cs));
            G_CK(cudaEventRecord(e, cs));
            G_CK(cudaStreamWaitEvent(st, e, 0));
            k_nbr_convert_check<<<g->num_sms * 8, 256, 0, st>>>(tmp, g->nbr, rs, lo, lo + len, n, g->counters,
                                                                 g->counters + 12);
        }
        if (weights && m > 0) {
            // (after the neighbours' conversions: the weights reuse tmp)
            G_CK(cudaEventRecord(ev_copy, st));
            G_CK(cudaStreamWaitEvent(cs, ev_copy, 0));
            unsigned long long init[4] = {0, 0, ~0ull, 0};
            G_CK(cudaMemcpyAsync(g->counters + 4, init, sizeof(init), cudaMemcpyHostToDevice, st));
            for (int64_t lo = 0; lo < m; lo += kChunk) {
                const int64_t len = std::min(kChunk, m - lo);
                cudaEvent_t e = nullptr;
                G_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                evs.push_back(e);
                G_CK(cudaMemcpyAsync(tmp + lo, weights + lo, len * sizeof(double), cudaMemcpyHostToDevice, cs));
                G_CK(cudaEventRecord(e, cs));
                G_CK(cudaStreamWaitEvent(st, e, 0));
                k_weight_scan<<<g->num_sms * 8, 256, 0, st>>>((const double*)tmp + lo, len, g->counters + 4);
            }
        }
        G_CK(cudaMemcpyAsync(g->h_counters, g->counters, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        G_CK(cudaStreamSynchronize(st));
        dfree(rs);
        if (g->h_counters[11]) {
            dfree(tmp);
            return fail(lp_fail(LP_ERR_INVALID, "offsets must be non-decreasing"));
        }
        if (g->h_counters[0]) {
            dfree(tmp);
            return fail(lp_fail(LP_ERR_INVALID, "neighbor ids must lie in [0, vertex_count)"));
        }
        g->max_degree = (int64_t)g->h_counters[8];
        g->rows_sorted = g->h_counters[12] == 0;
        g->sliceable = (int64_t)g->h_counters[9];
        g->slice_slots = (int64_t)g->h_counters[10];
        g->wmode = kUnit;
        if (weights && m > 0 && g->h_counters[4 + 0] != 0) {
            const unsigned long long bad = g->h_counters[4 + 1];
            const int emin = (int)g->h_counters[4 + 2] - 2048, emax = (int)g->h_counters[4 + 3] - 2048;
            // fixed point: w * 2^shift is an integer < 2^32 for every float32 weight when
            // shift = 24 - emin and (emax - emin + 24) <= 32.  The integer row sums equal
            // the reference's float64 sums (rak.py:105) only while those are exact, i.e.
            // every partial sum fits the 53-bit significand: span + ceil(log2(degree)) <= 53
            const int span = emax - emin + 24;
            const int deg_bits = (int)std::ceil(std::log2((double)std::max<int64_t>(2, g->max_degree)));
            if (bad == 0 && span <= 32 && span + deg_bits <= 53) {
                g->wmode = kFixed;
                g->fixed_shift = 24 - emin;
            } else {
                g->wmode = kFloat;
            }
            G_CK(dalloc(&g->w, m, &g->bytes));
            k_weight_convert<<<g->num_sms * 8, 256, 0, st>>>((const double*)tmp, g->w, m, g->wmode, g->fixed_shift);
        }
        G_CK(cudaStreamSynchronize(st));
        dfree(tmp);
    }
    G_CK(alloc_routes(g));
    G_CK(cudaStreamSynchronize(st));
    G_CK(cudaGetLastError());
    *out = g;
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

// Device lengths of the W dense waves (positions [w*ws, (w+1)*ws) of the order).
static int ensure_waves(lp_graph* g, int W) {
    Plan& P = g->plan();
    if (P.waves == W && P.wave_len) return LP_OK;
    dfree(P.wave_len);
    P.wave_len = nullptr;
    LP_CK(pool_alloc(&P.wave_len, W * sizeof(int32_t)));
    std::vector<int32_t> h((size_t)W);
    const int64_t ws = (g->n + W - 1) / W;
    for (int w = 0; w < W; ++w) h[(size_t)w] = (int32_t)std::max<int64_t>(0, std::min<int64_t>(ws, g->n - w * ws));
    LP_CK(cudaMemcpyAsync(P.wave_len, h.data(), W * sizeof(int32_t), cudaMemcpyHostToDevice, g->stream));
    LP_CK(cudaStreamSynchronize(g->stream));
    P.waves = W;
    return LP_OK;
}

// One sweep (RAK) or speaking round (SLPA): the dense round over every
// active row, then frontier rounds over the mark queue until a round marks
// nothing.  One host sync per frontier round (route sizes).
// the vertices a marking pass flagged in the bitmap -> a.mq_out (bits cleared)
// Marking mode of a pass: the bitmap (a second, cheap atomic per marked arc;
// compaction reads n/32 words) for passes over few changed rows, the flat scan
// of the marks (compaction reads 8 B per vertex) for big ones.
static EvalArgs marks_mode(lp_graph* g, const EvalArgs& a, int64_t changed_rows) {
    EvalArgs b = a;
    b.mbits = (g->mark_bitmap && changed_rows * g->mark_scan_div <= g->n) ? g->mbits : nullptr;
    return b;
}

static void bits_to_queue(lp_graph* g, const EvalArgs& a) {
    if (!a.mbits) {
        k_marks_to_queue<<<grid_for(g->n, 256 * 8, g->num_sms * 8), 256, 0, g->stream>>>(g->mark, g->n, a.mq_out, a.mq_len);
        return;
    }
    const int64_t nwords = g->n / 32 + 1;
    k_bits_to_queue<<<grid_for(nwords, 256, g->num_sms * 8), 256, 0, g->stream>>>(g->mbits, nwords, a.mq_out, a.mq_len);
}

static int solve_sweep(lp_graph* g, EvalArgs& a, bool cross, round_fn run_round, int alg, Prof* prof, int* rounds,
                       int64_t* gathered, bool first_ids = false, bool carry = false, bool first_random = false,
                       bool first_chain = false) {
    const Plan& P = g->plan();
    cudaStream_t st = g->stream;
    LP_CK(cudaMemsetAsync(g->routes.len, 0, kLenCount * sizeof(int32_t), st));
    int q = 0;  // the queue routed next / this round's writes queue into mq[q]
    a.mq_out = g->mq[q];
    a.mq_len = g->mq_len + q;
    a.horizon = INT32_MAX;
    a.mark_all = 0;
    // carry: mq[0] already holds the vertices whose inputs changed since their
    // last evaluation (built at the sweep boundary); keep it
    LP_CK(cudaMemsetAsync(g->mq_len + (carry ? 1 : 0), 0, (carry ? 1 : 2) * sizeof(int32_t), st));
    // (grid sized by the changed rows when known: every warp of the grid takes
    // one atomic on the shared piece cursor, ~10 us for a full grid)
    // (compact: the bitmap becomes the queue; the dense waves compact once after
    // the last wave, so that a vertex marked by two waves is queued once)
    auto mark_pass = [&](int64_t changed_rows, bool compact = true) {
        const int64_t pieces = changed_rows + changed_rows / 8 + 32;
        const EvalArgs b = marks_mode(g, a, changed_rows);
        prof->begin(st, -1);
        k_mark_pieces<<<grid_for(pieces, 4 * 8, g->num_sms * 16), 256, 0, st>>>(b);
        if (compact) bits_to_queue(g, b);
        prof->end(st);
    };
    // the tally kernels' arguments: without cross-batch reads (synchronous schedule) one round is
    // the sweep and nobody walks the round's changed rows -- no list (the sweep boundary rebuilds
    // it from the labels); one append per warp on the list's counter is measurable
    auto targs = [&]() {
        EvalArgs t = a;
        if (!cross) t.mark = nullptr;
        return t;
    };
    // writes of the round just run (label changes); one sync
    auto round_writes = [&](int64_t* w) -> int {
        LP_CK(cudaMemcpyAsync(g->h_counters + kCtrWrites, g->counters + kCtrWrites, sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
        *w = (int64_t)g->h_counters[kCtrWrites];
        return LP_OK;
    };
    const int64_t dense_at = (int64_t)(g->dense_frac * (double)P.S);
    enum { kNextDense, kNextFirst, kNextQueue };
    int next = first_ids ? kNextFirst : kNextDense;
    // The frontier loop: the rounds from here on run in one cooperative launch (lp_loop_kernels.cuh)
    // until a round queues nothing (*done) or the queue comes back (rows longer than the loop's
    // table, or more than loop_max_queue of them): then the class kernels route mq[q] as usual.
    bool loop_ok = g->loop_run && cross && a.mark && g->loop_rows > 0;  // (RAK and SLPA: a.slots)
    // (warp per row: not for graphs of very short rows -- the grid's 4-arc rows stay thread per row)
    bool loop_dense = loop_ok && g->max_degree <= kLoopMaxDeg && P.m_active <= g->loop_dense_arcs &&
                            P.m_active >= 12 * P.S;
    auto run_loop = [&](const int32_t* list0, const int32_t* list0_len, int list0_cnt, int first_dst, bool dense,
                        bool* done) -> int {
        LP_CK(cudaMemsetAsync(g->loop_ctl, 0, sizeof(LoopCtl), st));
        prof->begin(st, kKWarp);
        const cudaError_t e = g->loop_run(g, a, list0, list0_len, list0_cnt, first_dst, dense ? 1 : 0,
                                          loop_dense ? INT32_MAX : g->loop_max_queue);  // (every row is the loop's)
        prof->end(st);
        if (e != cudaSuccess) {
            // no cooperative launch here (the grid must be co-resident: a device shared through MPS,
            // a debugger ...): nothing ran; this handle keeps to the class kernels from now on
            cudaGetLastError();
            g->loop_rows = 0;
            loop_ok = loop_dense = false;
            *done = false;
            return LP_OK;
        }
        LP_CK(cudaMemcpyAsync(g->h_loop, g->loop_ctl, sizeof(LoopCtl), cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
        *rounds += g->h_loop->rounds;
        if (g->debug_rounds)
            fprintf(stderr, "[lp] frontier loop: %d rounds, queue left %d (%d rows handed back)\n", g->h_loop->rounds,
                    g->h_loop->out_len, g->h_loop->leftover[0] + g->h_loop->leftover[1]);
        *done = g->h_loop->out_len == 0;
        q = g->h_loop->out_buf;  // (the queue to route next, its length in mq_len[q])
        a.mq_out = g->mq[q];
        a.mq_len = g->mq_len + q;
        next = kNextQueue;
        return LP_OK;
    };
    if (carry) {
        int32_t ql = 0;
        LP_CK(cudaMemcpyAsync(g->h_len, g->mq_len, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
        ql = g->h_len[0];
        if (g->debug_rounds) fprintf(stderr, "[lp] sweep start: carried queue %d (dense at %lld)\n", ql, (long long)dense_at);
        if (ql == 0) return LP_OK;  // no vertex saw a neighbour change: the sweep changes nothing
        next = kNextQueue;  // (the margin test filters the queue; see the switch below)
        if (loop_ok && (loop_dense || (ql <= g->loop_max_queue && ql <= 4 * g->loop_rows))) {
            bool done = false;
            if (int rc = run_loop(g->mq[0], g->mq_len, 0, 1, false, &done)) return rc;
            if (done) return LP_OK;
        }
    }
    // Dense waves: the visit order in W consecutive position ranges, each
    // routed and evaluated after the previous one, so a wave reads the
    // current-sweep labels of all earlier waves; a changed label marks only
    // the later neighbours in positions already evaluated (its own wave).
    auto dense_waves = [&](int W) -> int {
        if (int rc = ensure_waves(g, W)) return rc;
        const int64_t ws = (g->n + W - 1) / W;
        for (int w = 0; w < W; ++w) {
            LP_CK(cudaMemsetAsync(g->routes.len, 0, kLenCount * sizeof(int32_t), st));
            prof->begin(st, -1);
            k_route_queue<<<g->num_sms * 4, 256, 0, st>>>(a, P.vorder + w * ws, P.wave_len + w, P.slot_of, 0);
            prof->end(st);
            LP_CK(cudaMemcpyAsync(g->h_len, g->routes.len, kLenCount * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
            LP_CK(cudaStreamSynchronize(st));
            a.horizon = (int32_t)std::min<int64_t>(g->n, (w + 1) * ws);
            if (g->h_len[kLenRouted] > 0) {
                run_round(g, targs(), false, g->h_len, prof, alg);
                if (a.mark) mark_pass(g->n, false);
            }
            ++*rounds;
        }
        a.horizon = INT32_MAX;
        if (a.mark) bits_to_queue(g, marks_mode(g, a, g->n));  // (the waves' mode)
        next = kNextQueue;
        return LP_OK;
    };
    const int W = (cross && !carry && !first_ids) ? g->waves : 1;
    if (W > 1)
        if (int rc = dense_waves(W)) return rc;
    cudaEvent_t dbg0 = nullptr, dbg1 = nullptr;
    if (g->debug_rounds) {
        cudaEventCreate(&dbg0);
        cudaEventCreate(&dbg1);
    }
    bool small_round = false;
    int64_t last_routed = 0;
    while (true) {
        if (dbg0) cudaEventRecord(dbg0, st);
        if (next == kNextDense && loop_dense) {
            // every row fits the loop's warp table: the dense round (visit order) and all the
            // frontier rounds after it in one launch
            LP_CK(cudaMemsetAsync(g->mq_len, 0, 2 * sizeof(int32_t), st));
            bool done = false;
            if (int rc = run_loop(P.vorder, nullptr, (int)g->n, 0, true, &done)) return rc;
            *gathered += P.m_active;
            if (done) break;
            continue;
        }
        if (next == kNextQueue) {
            // route the queue (margin test); this round's writes queue into the other one
            LP_CK(cudaMemsetAsync(g->routes.len, 0, kLenCount * sizeof(int32_t), st));
            LP_CK(cudaMemsetAsync(g->mq_len + (q ^ 1), 0, sizeof(int32_t), st));
            prof->begin(st, -1);
            k_route_queue<<<g->num_sms * 4, 256, 0, st>>>(a, g->mq[q], g->mq_len + q, P.slot_of, 1);
            prof->end(st);
            LP_CK(cudaMemcpyAsync(g->h_len, g->routes.len, kLenCount * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
            LP_CK(cudaStreamSynchronize(st));
            if (g->debug_rounds) {
                int32_t ql = 0;
                cudaMemcpy(&ql, g->mq_len + q, sizeof(int32_t), cudaMemcpyDeviceToHost);
                fprintf(stderr, "[lp] round %d: queue %d small %d/%d/%d warp %d warpbig %d team %d team2 %d hub-items %d pieces %d\n",
                        *rounds, ql, g->h_len[kLenS16], g->h_len[kLenS16 - 1], g->h_len[kLenS16 - 2],
                        g->h_len[kLenWarp], g->h_len[kLenWarpBig], g->h_len[kLenTeam], g->h_len[kLenTeam2],
                        g->h_len[kLenHub], g->h_len[kLenGather]);
            }
            if (g->h_len[kLenRouted] == 0) break;  // everything queued passed the margin test
            q ^= 1;
            a.mq_out = g->mq[q];
            a.mq_len = g->mq_len + q;
            LP_CK(cudaMemsetAsync(g->counters + kCtrWrites, 0, sizeof(unsigned long long), st));
            if ((double)g->h_len[kLenRouted] >= g->dense_frac * (double)P.npieces) {
                // most rows survived the margin test: a full round is cheaper than the
                // routed frontier (the routes are dropped; every margin is refreshed)
                LP_CK(cudaMemsetAsync(g->routes.len, 0, kLenCount * sizeof(int32_t), st));
                LP_CK(cudaMemsetAsync(g->mq_len + q, 0, sizeof(int32_t), st));
                run_round(g, targs(), true, g->h_len, prof, alg);
                if (alg == kGatherRak) *gathered += P.m_active;
            } else {
                run_round(g, targs(), false, g->h_len, prof, alg);
                // a routed frontier smaller than the full-round threshold cannot write
                // that many labels: no need to read the write count (one sync less)
                int64_t routed = 0;
                for (int c = 0; c <= kLenWarpBig; ++c) routed += g->h_len[c];
                routed += g->h_len[kLenTeam2] + g->h_len[kLenMid];
                small_round = routed < dense_at && !dbg0;
                last_routed = routed;
            }
        } else {
            // every active row (dense), or the trivial first round from labels = ids
            LP_CK(cudaMemsetAsync(g->routes.len, 0, kLenCount * sizeof(int32_t), st));
            LP_CK(cudaMemsetAsync(g->counters + kCtrWrites, 0, sizeof(unsigned long long), st));
            a.mq_out = g->mq[q];
            a.mq_len = g->mq_len + q;
            LP_CK(cudaMemsetAsync(g->mq_len + q, 0, sizeof(int32_t), st));
            if (next == kNextFirst) {
                a.bin = kKSmall;
                prof->begin(st, kKSmall);
                if (g->wmode == kFixed) {
                    k_first_round_wbig<<<g->num_sms * 4, 256, 0, st>>>(targs(), (int32_t)P.S);
                    k_first_round_w<<<grid_for(P.S, 256, g->num_sms * 16), 256, 0, st>>>(targs(), (int32_t)P.S);
                }
                else if (first_random) {
                    k_first_round_rbig<<<g->num_sms * 4, 256, 0, st>>>(targs(), (int32_t)P.S);
                    k_first_round_r<<<grid_for(P.S, 256, g->num_sms * 16), 256, 0, st>>>(targs(), (int32_t)P.S);
                }
                else {
                    // (a full round always follows the chained guess: its changed rows need no list --
                    // one append per warp on the list's single counter was a third of this kernel)
                    EvalArgs af = targs();
                    if (first_chain) af.mark = nullptr;
                    k_first_round<<<grid_for(P.S, 256, g->num_sms * 16), 256, 0, st>>>(af, (int32_t)P.S, P.slot_of,
                                                                                      first_chain ? 1 : 0);
                }
                prof->end(st);
            } else {
                run_round(g, targs(), true, g->h_len, prof, alg);  // (refreshes every margin)
                if (alg == kGatherRak) *gathered += P.m_active;  // (piece gathers count themselves)
            }
        }
        ++*rounds;
        if (!cross) break;  // no cross-batch reads: one round solves the sweep
        if (small_round) {
            small_round = false;
            mark_pass(last_routed);  // (an empty change list marks nothing; the next route ends the loop)
            next = kNextQueue;
            if (loop_ok && last_routed <= g->loop_rows) {
                bool done = false;
                if (int rc = run_loop(g->mq[q], g->mq_len + q, 0, q ^ 1, false, &done)) return rc;
                if (done) break;
            }
            continue;
        }
        int64_t w = 0;
        if (int rc = round_writes(&w)) return rc;
        if (dbg0) {
            cudaEventRecord(dbg1, st);
            cudaEventSynchronize(dbg1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, dbg0, dbg1);
            fprintf(stderr, "[lp]   round %d (%s): %.3f ms, %lld label writes\n", *rounds,
                    next == kNextQueue ? "frontier" : (next == kNextFirst ? "first" : "dense"), ms, (long long)w);
        }
        if (w == 0 && !(first_chain && next == kNextFirst)) break;  // nothing changed: every read is final
        if (first_chain && next == kNextFirst) {
            // the chained first round is a guess, not an evaluation: verify every row
            // (in position-ordered waves instead: measured 1.3-7x slower)
            next = kNextDense;
        } else if (w >= dense_at) {
            if (g->pull_rounds && P.npieces > 0 && (double)w < g->pull_max_frac * (double)P.S) {
                // most labels moved: every row pulls the changed flags of its
                // earlier-batch neighbours (one flat pass instead of an atomic per
                // later-batch arc of every changed row); the margin test then
                // filters the queue, and a still-large frontier runs as a full round
                LP_CK(cudaMemsetAsync(g->chg, 0, (g->n / 32 + 1) * sizeof(uint32_t), st));
                k_flags_from_changed<<<g->num_sms * 8, 256, 0, st>>>(a, g->chg);
                LP_CK(cudaMemsetAsync(g->routes.len + kGatherCursor, 0, sizeof(int32_t), st));
                prof->begin(st, -1);
                const EvalArgs b = marks_mode(g, a, w);
                k_pull_marks<<<g->num_sms * 16, 256, 0, st>>>(b, g->chg, P.dslot, P.dk0, P.dcount,
                                                             g->routes.len + kGatherCursor, 1);
                bits_to_queue(g, b);
                prof->end(st);
                next = kNextQueue;
            } else {
                // a full round costs less than marking and routing nearly every row
                next = kNextDense;
            }
        } else {
            mark_pass(w);
            next = kNextQueue;
            if (loop_ok && w <= g->loop_rows) {
                bool done = false;
                if (int rc = run_loop(g->mq[q], g->mq_len + q, 0, q ^ 1, false, &done)) return rc;
                if (done) break;
            }
        }
    }
    if (dbg0) {
        cudaEventDestroy(dbg0);
        cudaEventDestroy(dbg1);
    }
    return LP_OK;
}

// Per-run statistics from the counters (already downloaded to h_counters)
// and the profiling events.
static int finish_stats(lp_graph* g, const Prof& prof, lp_run_stats* S, int it, int rounds, int64_t gathered,
                        float ms) {
    S->iterations = it;
    S->rounds = rounds;
    S->kernel_ms = ms;
    S->arcs_dense = g->plan().m_active * it;
    S->launches = prof.launches;
    S->arcs_gathered = gathered + (int64_t)g->h_counters[kCtrGathered];
    S->gather_launches = prof.slot_launches[kKGather];
    for (int b = 0; b < kKSlots; ++b) {
        S->bin_arcs[b] = (int64_t)g->h_counters[kCtrArcs + b];
        S->bin_vertices[b] = (int64_t)g->h_counters[kCtrVerts + b];
        S->bin_launches[b] = prof.slot_launches[b];
        S->arcs_scanned += S->bin_arcs[b];
    }
    for (size_t i = 0; i < prof.tags.size(); ++i) {
        float e = 0.f;
        LP_CK(cudaEventElapsedTime(&e, g->event_pool[2 * i], g->event_pool[2 * i + 1]));
        if (prof.tags[i] == kKGather)
            S->gather_ms += e;
        else if (prof.tags[i] >= 0)
            S->bin_ms[prof.tags[i]] += e;
        else
            S->aux_ms += e;
    }
    return LP_OK;
}

// Keep the two label arrays (L0 and x, 8 bytes per vertex: 33.6 MB for
// R-MAT-22) resident in L2 while the round's index stream and label buffer
// (1 GB per dense round) stream past them: a persisting access-policy window
// on every stream the round's kernels run on, with the device's persisting
// carve-out sized to the window.  The random neighbour-label gathers then hit
// L2 instead of HBM.
static void set_l2_window(lp_graph* g) {
    if (!g->l2_persist || g->n == 0) return;
    static std::mutex mu;
    static int64_t limit_set[64] = {};
    int max_window = 0, max_persist = 0;
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, g->device);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, g->device);
    if (max_window <= 0 || max_persist <= 0) return;
    const size_t want = (size_t)(g->labB - g->labA + g->n) * sizeof(int32_t);
    const size_t bytes = std::min(want, (size_t)max_window);
    const size_t carve = std::min(bytes, (size_t)max_persist);
    {
        std::lock_guard<std::mutex> lock(mu);
        if (limit_set[g->device & 63] < (int64_t)carve) {
            if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve) != cudaSuccess) {
                cudaGetLastError();
                return;
            }
            limit_set[g->device & 63] = (int64_t)carve;
        }
    }
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow.base_ptr = g->labA;
    v.accessPolicyWindow.num_bytes = bytes;
    v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)carve / (double)bytes);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStream_t sts[3] = {g->stream, g->aux[0], g->aux[1]};
    for (cudaStream_t s : sts)
        if (s && cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) cudaGetLastError();
}

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
    StreamScope ss(g->stream);
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
    const int64_t B = (o->batches == 0 || o->batches > n) ? n : o->batches;
    const int64_t bs = (n + B - 1) / B;
    if (int rc = build_plan(g, kPlanRak, order, o->seed, &plan_ms, bs)) return rc;
    const bool cross = bs < n;  // some vertex depends on an earlier batch
    if (int rc = ensure_flags(g, bs, &plan_ms)) return rc;
    S->plan_ms = plan_ms;
    set_l2_window(g);
    Plan& P = g->plan();
    cudaStream_t st = g->stream;
    round_fn run_round = nullptr;
    setup_fn setup = nullptr;
    if (g->wmode == kFixed)
        pick_fns<kFixed>(o->tie, &run_round, &setup);
    else if (g->wmode == kFloat)
        pick_fns<kFloat>(o->tie, &run_round, &setup);
    else
        pick_fns<kUnit>(o->tie, &run_round, &setup);
    LP_CK(setup(g->device));
    g->loop_run = g->wmode == kFixed   ? pick_loop<kFixed>(o->tie)
                  : g->wmode == kFloat ? pick_loop<kFloat>(o->tie)
                                       : pick_loop<kUnit>(o->tie);

    if (labels_init) {
        int64_t* tmp = g->out64;
        LP_CK(cudaMemcpyAsync(tmp, labels_init, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        LP_CK(cudaMemsetAsync(g->counters, 0, sizeof(unsigned long long), st));
        k_check_labels<<<g->num_sms * 4, 256, 0, st>>>(tmp, n, g->counters);
        unsigned long long bad = 0;
        LP_CK(cudaMemcpyAsync(&bad, g->counters, sizeof(bad), cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
        if (bad) return lp_fail(LP_ERR_INVALID, "initial labels must lie in [0, vertex_count)");
        k_init_labels<<<g->num_sms * 8, 256, 0, st>>>(tmp, g->labA, n);
    } else {
        k_init_labels<<<g->num_sms * 8, 256, 0, st>>>(nullptr, g->labA, n);
    }
    if (P.S > 0) k_reset_ndist<<<g->num_sms * 8, 256, 0, st>>>(P.soff, P.ndist, P.S);
    LP_CK(cudaGetLastError());

    int32_t* L0 = g->labA;
    int32_t* X = g->labB;
    EvalArgs a;
    a.soff = P.soff;
    a.snbr = P.snbr;
    a.sw = P.sw;
    a.swsum = P.swsum;
    a.svid = P.svid;
    a.lbuf = P.lbuf;
    // marks: cross-batch dependencies inside a sweep, and (track) the active
    // frontier across sweeps: a sweep re-evaluates only vertices with a
    // neighbour that changed since their last evaluation
    // (not with random ties: tie_hash is keyed by the sweep, so an unchanged
    // neighbourhood can still produce a different winner)
    // (random ties: tie_hash is keyed by the sweep, so a vertex whose last
    // evaluation tied may move with an unchanged neighbourhood; the margin
    // array tells which ones tied, k_mark_ties queues them at the boundary)
    const bool gap_ok = g->wmode != kFloat && g->margin_skip;
    const bool track = g->sweep_frontier && (o->tie != kRandom || gap_ok);
    a.mark = (cross || track) ? g->mark : nullptr;
    a.gap = ((cross || track) && g->wmode != kFloat && g->margin_skip) ? g->gap : nullptr;
    a.mark_all = 0;
    a.pos = P.pos;
    a.slots = nullptr;  // (SLPA's memories: lp_slpa_run)
    a.T = 0;
    a.horizon = INT32_MAX;
    a.mq_out = nullptr;
    a.mq_len = nullptr;
    a.ndist = P.ndist;
    a.counters = g->counters;
    a.r = g->routes;
    a.bin = 0;
    a.seed = o->seed;
    a.cap_route = g->cap_route;
    a.id_single = 0;
    a.two_team = 0;
    a.mbits = g->mbits;  // (per marking pass: marks_mode)
    a.first_est_min = g->first_est_min;
    a.first_est_div = g->first_est_div;
    // (unit weights only: with weights the bucketed arcs' weight loads are
    // indirect, measured slower on R-MAT-22 float32 weights)
    const bool buckets = g->hub_bucket && g->wmode == kUnit;
    a.hb_lab = buckets ? P.hb_lab : nullptr;
    a.hb_pos = buckets ? P.hb_pos : nullptr;
    a.hb_off = buckets ? g->hb_off : nullptr;
    a.warp_maxd[0] = g->warp_maxd[0];
    a.warp_maxd[1] = g->warp_maxd[1];
    a.reg_est = g->reg_est;
    a.mid_max = g->mid_max > kSmallMax ? g->mid_max : 0;
    a.fused = 0;  // (per launch: Launcher::round)
    // fused row classes: k_small rows (d <= 16), k_mid rows (d <= mid_max), or all
    // Exact schedules whose first sweep cascades -- weights or random ties: the all-singleton
    // tallies of a sweep from ids have leads near zero, so nearly every changed neighbour passes
    // the margin test -- fuse every row: a tally that reads the working labels in place sees what
    // the round has already written (Gauss-Seidel inside the round), where the phase-1 snapshot
    // repeats the whole cascade level by level (R-MAT-22 float32 weights 57 -> 32 ms on average --
    // 23 to 41: how the round's streams interleave decides how many full rounds the first sweep
    // takes -- random ties 31 -> 25 ms; unit weights with scan-first ties: two-phase long rows
    // stay 7% faster, 5.87 vs 6.27 ms).
    g->run_fuse = g->fuse_forced ? g->fuse_maxd
                  : (cross && (g->wmode != kUnit || o->tie == kRandom)) ? (1 << 30) : g->fuse_maxd;
    a.fuse_maxd = g->run_fuse >= (1 << 30) ? INT32_MAX
                  : (a.mid_max > 0 && g->run_fuse >= a.mid_max) ? a.mid_max
                  : g->run_fuse >= kSmallMax ? kSmallMax : 0;

    LP_CK(cudaMemsetAsync(g->counters, 0, kCtrCount * sizeof(unsigned long long), st));
    Prof prof;
    prof.on = (o->flags & LP_RAK_PROFILE) != 0;
    prof.pool = &g->event_pool;
    LP_CK(cudaEventRecord(g->ev0, st));
    int it = 0;
    int rounds = 0;
    int64_t gathered = 0;
    int64_t last_changed = n;
    while (it < o->max_iterations) {
        ++it;
        a.sweep = (uint32_t)it;
        a.L0 = L0;
        a.x = X;
        // (only after a sweep that changed few labels: marking the neighbours of
        // many changed rows costs more than one full round)
        const bool carry = track && it > 1 && last_changed <= (int64_t)(g->carry_frac * (double)P.S);
        if (carry) {
            // sweep boundary: a vertex is queued (with the changed weight, for the margin
            // test) when a neighbour whose sweep-start label it reads -- same or later
            // batch -- changed in the last sweep; an earlier-batch neighbour's change was
            // already read through the working labels, and if it moves again this sweep its
            // marks say so.  Only queued vertices can change in this sweep's first round
            LP_CK(cudaMemsetAsync(g->routes.len, 0, kLenCount * sizeof(int32_t), st));
            LP_CK(cudaMemsetAsync(g->mq_len, 0, sizeof(int32_t), st));
            a.mq_out = g->mq[0];
            a.mq_len = g->mq_len;
            prof.begin(st, -1);
            if (last_changed * g->push_div <= P.S) {
                // few changed rows: push from them (one atomic per neighbour)
                k_sweep_changes<<<g->num_sms * 8, 256, 0, st>>>(a, L0, X, (int32_t)P.S);  // L0 = last result
                a.mark_all = 2;
                const EvalArgs b = marks_mode(g, a, o->tie == kRandom ? g->n : last_changed);
                k_mark_pieces<<<g->num_sms * 16, 256, 0, st>>>(b);
                if (o->tie == kRandom) k_mark_ties<<<g->num_sms * 8, 256, 0, st>>>(b, (int32_t)P.S);
                bits_to_queue(g, b);
                a.mark_all = 0;
            } else {
                // many: every row pulls the changed flags of its neighbours (one flat
                // pass, one atomic per row piece with a changed neighbour)
                k_changed_flags<<<g->num_sms * 8, 256, 0, st>>>(L0, X, g->chg, n);
                const EvalArgs b = marks_mode(g, a, last_changed);
                k_pull_marks<<<g->num_sms * 16, 256, 0, st>>>(b, g->chg, P.dslot, P.dk0, P.dcount,
                                                             g->routes.len + kGatherCursor, 2);
                if (o->tie == kRandom) k_mark_ties<<<g->num_sms * 8, 256, 0, st>>>(b, (int32_t)P.S);
                bits_to_queue(g, b);
            }
            prof.end(st);
        }
        LP_CK(cudaMemcpyAsync(X, L0, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        LP_CK(cudaMemsetAsync(g->counters + kCtrChanged, 0, 2 * sizeof(unsigned long long), st));
        // first sweep from labels = ids: the dense round is trivial for unit
        // weights and scan-first / min-label ties on duplicate-free sorted rows
        const bool first_ids = it == 1 && !labels_init && (g->wmode == kUnit || g->wmode == kFixed) && g->rows_sorted &&
                               (o->tie == kScanFirst || o->tie == kMinLabel) && g->first_round_shortcut;
        // random ties, unit weights: the first round is the row's largest tie hash
        const bool first_random = it == 1 && !labels_init && g->wmode == kUnit && g->rows_sorted &&
                                  o->tie == kRandom && g->first_round_shortcut;
        // first sweep from labels = ids: unevaluated neighbours carry singleton labels
        a.id_single = (it == 1 && !labels_init && (g->wmode == kUnit || (g->wmode == kFixed && g->id_single_w)) &&
                       g->rows_sorted && n < (1 << 30) && (o->tie != kRandom || g->id_single_random) && g->id_single)
                          ? 1
                          : 0;
        a.two_team = a.id_single && (g->wmode == kUnit || (g->wmode == kFixed && g->two_team_w));
        // (the first round's low label estimates serve the next round's singleton
        // tallies of unit weights; with weights the labels stay diverse and the
        // small tables overflow: measured slower, so weighted rows estimate d)
        a.first_est_div = g->wmode == kFixed ? 1 : g->first_est_div;
        // (exact schedules, scan-first, unit weights: the first round follows first
        // arcs through earlier-batch neighbours, k_first_round)
        // (measured with fixed-point weights too: the weighted first sweep's
        // cascade of frontier rounds is not shortened, no gain)
        const bool first_chain = first_ids && cross && g->first_chain && g->wmode == kUnit && o->tie == kScanFirst;
        if (int rc = solve_sweep(g, a, cross, run_round, kGatherRak, &prof, &rounds, &gathered, first_ids || first_random,
                                 carry, first_random, first_chain))
            return rc;
        LP_CK(cudaMemcpyAsync(g->h_counters, g->counters, kCtrCount * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                              st));
        LP_CK(cudaStreamSynchronize(st));
        LP_CK(cudaGetLastError());
        if (g->h_counters[kCtrError])
            return lp_fail(LP_ERR_UNSUPPORTED, "a hub row's label partitions overflowed the team table split stack");
        const int64_t changed = (int64_t)g->h_counters[kCtrChanged];
        if (changed_per_iter) changed_per_iter[it - 1] = changed;
        last_changed = changed;
        std::swap(L0, X);  // L0 now holds this sweep's labels
        if ((double)changed <= o->tolerance * (double)n) break;  // rak.py:114-115
    }
    LP_CK(cudaEventRecord(g->ev1, st));
    LP_CK(cudaEventSynchronize(g->ev1));
    float ms = 0.f;
    LP_CK(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
    g->cur = L0;
    g->labels_valid = true;
    if (int rc = finish_stats(g, prof, S, it, rounds, gathered, ms)) return rc;
    S->arcs_dense = g->m * it;
    if (g->run_fuse >= (1 << 30)) S->flags |= LP_STATS_FUSED;
#ifdef LP_PATH_STATS
    {
        unsigned long long h[8];
        cudaMemcpy(h, g->counters + 20, sizeof(h), cudaMemcpyDeviceToHost);
        fprintf(stderr, "[lp] k_warp paths: majority %llu, majority-miss %llu, register %llu, hashed %llu, "
                "hashed-tied %llu, overflow %llu\n", h[0], h[5], h[1], h[2], h[3], h[4]);
        cudaMemset(g->counters + 20, 0, sizeof(h));
    }
#endif
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
    // int32 labels into a pinned staging buffer (full-speed DMA, half the
    // bytes), widened to the caller's int64 array by host threads -- instead
    // of a pageable int64 copy
    // (the staging buffer is process-wide and grow-only: pinned allocations
    // cost milliseconds, handles come and go)
    static std::mutex mu;
    static int32_t* stage = nullptr;
    static size_t stage_cap = 0;
    std::lock_guard<std::mutex> lock(mu);
    const int64_t n = g->n;
    if ((size_t)n > stage_cap) {
        if (stage) cudaFreeHost(stage);
        stage = nullptr;
        stage_cap = 0;
        LP_CK(cudaMallocHost((void**)&stage, (size_t)n * sizeof(int32_t)));
        stage_cap = (size_t)n;
    }
    LP_CK(cudaMemcpyAsync(stage, g->cur, n * sizeof(int32_t), cudaMemcpyDeviceToHost, g->stream));
    LP_CK(cudaStreamSynchronize(g->stream));
    const int32_t* src = stage;
#pragma omp parallel for schedule(static) if (n > (1 << 16))
    for (int64_t v = 0; v < n; ++v) labels_out[v] = src[v];
    return LP_OK;
}

extern "C" int lp_rak_run(lp_graph* g, const lp_rak_opts* opts, const int64_t* order, const int64_t* labels_init,
                          int64_t* labels_out, int64_t* changed_per_iter, lp_run_stats* stats) {
    if (!labels_out) return lp_fail(LP_ERR_INVALID, "labels_out is NULL");
    if (int rc = rak_core(g, opts, order, labels_init, changed_per_iter, stats)) return rc;
    return lp_labels_download(g, labels_out);
}

// ---------------------------------------------------------------------------
// SLPA driver (slpa.py:91-111 _slpa_seq, :166-193 _detect_full)
// ---------------------------------------------------------------------------
// Round t = 1 .. T-1 is a RAK sweep over the INDEX plan (identity order, no
// self arcs) with the SLPA phase-1 gather; the working array x starts from
// a guess (the previous round's appends; own ids in round 1) and is solved
// exactly under the batched schedule, then appended to the memories.
extern "C" int lp_slpa_run(lp_graph* g, const lp_slpa_opts* o, int64_t* labels_out, int64_t* slots_out,
                           int64_t* repeats_per_iter, lp_run_stats* stats) {
    if (!g || !o) return lp_fail(LP_ERR_INVALID, "NULL argument");
    if (o->memory_size < 2) return lp_fail(LP_ERR_INVALID, "memory_size must be >= 2");
    if (!(o->tolerance > 0.0 && o->tolerance <= 1.0)) return lp_fail(LP_ERR_INVALID, "tolerance must be in (0, 1]");
    if (o->tie < 0 || o->tie > 2) return lp_fail(LP_ERR_INVALID, "unknown tie rule");
    if (o->batches < 0) return lp_fail(LP_ERR_INVALID, "batches must be >= 0");
    LP_CK(cudaSetDevice(g->device));
    StreamScope ss(g->stream);
    lp_run_stats st_local;
    lp_run_stats* S = stats ? stats : &st_local;
    memset(S, 0, sizeof(*S));
    const int64_t n = g->n;
    const int T = o->memory_size;
    g->labels_valid = false;
    if (n == 0) return LP_OK;
    if ((double)n * T >= 2147483647.0 * 4) return lp_fail(LP_ERR_UNSUPPORTED, "memories too large");
    float plan_ms = 0.f;
    if (int rc = build_plan(g, kPlanIndex, nullptr, 0, &plan_ms)) return rc;
    const int64_t B = (o->batches == 0 || o->batches > n) ? n : o->batches;
    const int64_t bs = (n + B - 1) / B;
    const bool cross = bs < n;
    if (int rc = ensure_flags(g, bs, &plan_ms)) return rc;
    S->plan_ms = plan_ms;
    set_l2_window(g);
    Plan& P = g->plan();
    cudaStream_t st = g->stream;
    round_fn run_round = nullptr;
    setup_fn setup = nullptr;
    if (g->wmode == kFixed)
        pick_fns<kFixed>(o->tie, &run_round, &setup);
    else if (g->wmode == kFloat)
        pick_fns<kFloat>(o->tie, &run_round, &setup);
    else
        pick_fns<kUnit>(o->tie, &run_round, &setup);
    LP_CK(setup(g->device));
    g->loop_run = g->wmode == kFixed   ? pick_loop<kFixed>(o->tie)
                  : g->wmode == kFloat ? pick_loop<kFloat>(o->tie)
                                       : pick_loop<kUnit>(o->tie);
    const size_t cells = (size_t)n * T;
    if (cells > g->slots_cap) {
        dfree(g->slots);
        g->slots = nullptr;
        g->slots_cap = 0;
        LP_CK(pool_alloc(&g->slots, cells * sizeof(int32_t)));
        g->slots_cap = cells;
    }
    int32_t* A = g->labA;  // previous appends (round 1: own ids, the guess)
    int32_t* X = g->labB;  // working appends of this round
    LP_CK(cudaMemsetAsync(g->slots, 0, cells * sizeof(int32_t), st));
    k_slpa_init<<<g->num_sms * 8, 256, 0, st>>>(g->slots, A, n, T);
    if (P.S > 0) k_reset_ndist<<<g->num_sms * 8, 256, 0, st>>>(P.soff, P.ndist, P.S);
    LP_CK(cudaGetLastError());
    EvalArgs a;
    memset(&a, 0, sizeof(a));
    a.soff = P.soff;
    a.snbr = P.snbr;
    a.sw = P.sw;
    a.swsum = P.swsum;
    a.svid = P.svid;
    a.lbuf = P.lbuf;
    a.mark = cross ? g->mark : nullptr;
    a.gap = (cross && g->wmode != kFloat && g->margin_skip) ? g->gap : nullptr;
    a.pos = P.pos;
    a.horizon = INT32_MAX;
    a.ndist = P.ndist;
    a.counters = g->counters;
    a.r = g->routes;
    a.seed = o->seed;
    a.slots = g->slots;
    a.T = T;
    a.cap_route = g->cap_route;
    a.id_single = 0;
    a.two_team = 0;
    a.mbits = g->mbits;  // (per marking pass: marks_mode)
    a.first_est_min = g->first_est_min;
    a.first_est_div = g->first_est_div;
    // (unit weights only: with weights the bucketed arcs' weight loads are
    // indirect, measured slower on R-MAT-22 float32 weights)
    const bool buckets = g->hub_bucket && g->wmode == kUnit;
    a.hb_lab = buckets ? P.hb_lab : nullptr;
    a.hb_pos = buckets ? P.hb_pos : nullptr;
    a.hb_off = buckets ? g->hb_off : nullptr;
    a.warp_maxd[0] = g->warp_maxd[0];
    a.warp_maxd[1] = g->warp_maxd[1];
    a.reg_est = g->reg_est;
    a.mid_max = g->mid_max > kSmallMax ? g->mid_max : 0;
    LP_CK(cudaMemsetAsync(g->counters, 0, kCtrCount * sizeof(unsigned long long), st));
    unsigned long long* rep_ctr = g->counters + kCtrCount;  // spare counter slot
    Prof prof;
    prof.on = (o->flags & LP_RAK_PROFILE) != 0;
    prof.pool = &g->event_pool;
    LP_CK(cudaEventRecord(g->ev0, st));
    int it = 0, rounds = 0;
    int64_t gathered = 0;
    for (int t = 1; t < T; ++t) {  // slpa.py:98
        ++it;
        a.sweep = (uint32_t)t;
        a.L0 = A;
        a.x = X;
        LP_CK(cudaMemcpyAsync(X, A, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        LP_CK(cudaMemsetAsync(g->counters + kCtrChanged, 0, 2 * sizeof(unsigned long long), st));
        if (P.S < n) {
            prof.begin(st, -1);
            k_slpa_idle<<<grid_for(n - P.S, 256, g->num_sms * 8), 256, 0, st>>>(P.svid, P.S, n, g->slots, T, t, X);
            prof.end(st);
        }
        if (P.S > 0)
            if (int rc = solve_sweep(g, a, cross, run_round, kGatherSlpa, &prof, &rounds, &gathered)) return rc;
        LP_CK(cudaMemsetAsync(rep_ctr, 0, sizeof(unsigned long long), st));
        prof.begin(st, -1);
        k_slpa_commit<<<g->num_sms * 8, 256, 0, st>>>(X, A, g->slots, n, T, t, t >= 2 ? 1 : 0, rep_ctr);
        prof.end(st);
        LP_CK(cudaMemcpyAsync(g->h_counters, g->counters, (kCtrCount + 1) * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
        LP_CK(cudaGetLastError());
        const int64_t repeats = (int64_t)g->h_counters[kCtrCount];
        if (repeats_per_iter) repeats_per_iter[t - 1] = repeats;
        std::swap(A, X);  // A = this round's appends (the next round's prev)
        if (t >= 2 && (double)repeats >= (1.0 - o->tolerance) * (double)n) break;  // slpa.py:109-110
    }
    // projection (slpa.py:147-150) inside the timed region like the reference (:183-185)
    if (labels_out) k_slpa_project<<<g->num_sms * 8, 256, 0, st>>>(g->slots, n, T, it + 1, g->out64);
    LP_CK(cudaEventRecord(g->ev1, st));
    LP_CK(cudaEventSynchronize(g->ev1));
    float ms = 0.f;
    LP_CK(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
    if (int rc = finish_stats(g, prof, S, it, rounds, gathered, ms)) return rc;
    if (labels_out) {
        LP_CK(cudaMemcpyAsync(labels_out, g->out64, n * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
    }
    if (slots_out) {
        int64_t* tmp = nullptr;
        LP_CK(pool_alloc(&tmp, cells * sizeof(int64_t)));
        k_slots_to64<<<g->num_sms * 8, 256, 0, st>>>(g->slots, tmp, (int64_t)cells);
        cudaError_t e = cudaMemcpyAsync(slots_out, tmp, cells * sizeof(int64_t), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        dfree(tmp);
        LP_CK(e);
    }
    return LP_OK;
}

// ---------------------------------------------------------------------------
// COPRA driver (copra.py:124-176 _copra_seq, :240-283 _detect_full)
// ---------------------------------------------------------------------------
static int copra_buffers(lp_graph* g, int K) {
    const int64_t n = g->n;
    const size_t cells = (size_t)n * K;
    if (cells > g->ccap) {
        for (int i = 0; i < 2; ++i) {
            dfree(g->clabs[i]);
            dfree(g->cbels[i]);
            g->clabs[i] = nullptr;
            g->cbels[i] = nullptr;
        }
        g->ccap = 0;
        for (int i = 0; i < 2; ++i) {
            LP_CK(pool_alloc(&g->clabs[i], cells * sizeof(int32_t)));
            LP_CK(pool_alloc(&g->cbels[i], cells * sizeof(double)));
        }
        g->ccap = cells;
    }
    if (!g->csize[0]) {
        for (int i = 0; i < 2; ++i) {
            LP_CK(pool_alloc(&g->csize[i], std::max<int64_t>(n, 1) * sizeof(int32_t)));
            LP_CK(pool_alloc(&g->cbest[i], std::max<int64_t>(n, 1) * sizeof(int32_t)));
        }
        LP_CK(pool_alloc(&g->ccur, 8 * sizeof(int32_t)));
        LP_CK(pool_alloc(&g->cbig, std::max<int64_t>(n, 1) * sizeof(int32_t)));
        LP_CK(pool_alloc(&g->cmid, std::max<int64_t>(n, 1) * sizeof(int32_t)));
        LP_CK(pool_alloc(&g->croute, std::max<int64_t>(n, 1) * sizeof(int32_t)));
        LP_CK(pool_alloc(&g->croute_mark, std::max<int64_t>(n, 1) * sizeof(int32_t)));
        LP_CK(cudaMemsetAsync(g->croute_mark, 0, std::max<int64_t>(n, 1) * sizeof(int32_t), g->stream));
    }
    // team scratch: a row sees at most min(n, max_degree * K) distinct labels and
    // max_degree * K contributions; blocks bounded by a 4 GiB budget
    const size_t con = (size_t)std::max<int64_t>(1, g->max_degree) * K;
    const size_t ent = std::min<size_t>((size_t)n, con);
    if (ent > g->gent || con > g->gcon) {
        dfree(g->gelab);
        dfree(g->geval);
        dfree(g->gefirst);
        dfree(g->grlab);
        dfree(g->grval);
        dfree(g->gfmap);
        dfree(g->gblab);
        dfree(g->gbval);
        dfree(g->gbc);
        dfree(g->gwc);
        dfree(g->gqs);
        dfree(g->gslab);
        dfree(g->gsval);
        g->gelab = g->gefirst = g->grlab = g->gfmap = g->gblab = g->gbc = g->gwc = g->gqs = g->gslab = nullptr;
        g->geval = g->grval = g->gbval = g->gsval = nullptr;
        g->gent = g->gcon = 0;
        const size_t parts = (size_t)kCopraTeamWarps * kCopraMaxParts + kCopraMaxParts + 1;
        const size_t per = ent * (3 * sizeof(int32_t) + 2 * sizeof(double)) +
                           con * (4 * sizeof(int32_t) + 2 * sizeof(double)) + parts * sizeof(int32_t);
        const int blocks = (int)std::max<size_t>(1, std::min<size_t>(2 * g->num_sms, ((size_t)6 << 30) / per));
        LP_CK(pool_alloc(&g->gelab, ent * blocks * sizeof(int32_t)));
        LP_CK(pool_alloc(&g->geval, ent * blocks * sizeof(double)));
        LP_CK(pool_alloc(&g->gefirst, ent * blocks * sizeof(int32_t)));
        LP_CK(pool_alloc(&g->grlab, ent * blocks * sizeof(int32_t)));
        LP_CK(pool_alloc(&g->grval, ent * blocks * sizeof(double)));
        LP_CK(pool_alloc(&g->gfmap, con * blocks * sizeof(int32_t)));
        LP_CK(pool_alloc(&g->gblab, con * blocks * sizeof(int32_t)));
        LP_CK(pool_alloc(&g->gbval, con * blocks * sizeof(double)));
        LP_CK(pool_alloc(&g->gbc, con * blocks * sizeof(int32_t)));
        LP_CK(pool_alloc(&g->gslab, con * blocks * sizeof(int32_t)));
        LP_CK(pool_alloc(&g->gsval, con * blocks * sizeof(double)));
        LP_CK(pool_alloc(&g->gwc, (size_t)kCopraTeamWarps * kCopraMaxParts * blocks * sizeof(int32_t)));
        LP_CK(pool_alloc(&g->gqs, (size_t)(kCopraMaxParts + 1) * blocks * sizeof(int32_t)));
        k_fill_i32<<<g->num_sms * 8, 256, 0, g->stream>>>(g->gfmap, -1, (int64_t)(con * blocks));
        LP_CK(cudaGetLastError());
        g->gent = ent;
        g->gcon = con;
        g->gblocks = blocks;
    }
    return LP_OK;
}

// COPRA tiers: warp + 512-slot table (8 warps/block), warp + 4096-slot
// table (1 warp/block), team (16 warps, partitioned; lp_copra_kernels.cuh)
#define COPRA_T0 kCopraBits, kCopraWarps, 3
#define COPRA_T1 11, 2, 3

extern "C" int lp_copra_run(lp_graph* g, const lp_copra_opts* o, int64_t* labs_out, double* bels_out,
                            int64_t* sizes_out, int64_t* best_out, int64_t* changed_per_iter, lp_run_stats* stats) {
    if (!g || !o) return lp_fail(LP_ERR_INVALID, "NULL argument");
    if (!(o->tolerance > 0.0 && o->tolerance <= 1.0)) return lp_fail(LP_ERR_INVALID, "tolerance must be in (0, 1]");
    if (o->max_labels < 1) return lp_fail(LP_ERR_INVALID, "max_labels must be >= 1");
    if (o->max_iterations < 1) return lp_fail(LP_ERR_INVALID, "max_iterations must be >= 1");
    if (o->batches < 0) return lp_fail(LP_ERR_INVALID, "batches must be >= 0");
    if (o->max_labels > kCopraMaxLabels) return lp_fail(LP_ERR_UNSUPPORTED, "max_labels > 32 is not supported on the GPU");
    if (!best_out) return lp_fail(LP_ERR_INVALID, "best_out is NULL");
    if ((labs_out == nullptr) != (bels_out == nullptr)) return lp_fail(LP_ERR_INVALID, "labs_out and bels_out go together");
    LP_CK(cudaSetDevice(g->device));
    StreamScope ss(g->stream);
    lp_run_stats st_local;
    lp_run_stats* S = stats ? stats : &st_local;
    memset(S, 0, sizeof(*S));
    const int64_t n = g->n;
    const int K = o->max_labels;
    g->labels_valid = false;
    if (n == 0) return LP_OK;
    if ((double)n * K >= 2147483647.0) return lp_fail(LP_ERR_UNSUPPORTED, "n * max_labels must be < 2^31");
    float plan_ms = 0.f;
    if (int rc = build_plan(g, kPlanIndex, nullptr, 0, &plan_ms)) return rc;
    const int64_t B = (o->batches == 0 || o->batches > n) ? n : o->batches;
    const int64_t bs = (n + B - 1) / B;
    const bool cross = bs < n;
    if (int rc = ensure_flags(g, bs, &plan_ms)) return rc;
    S->plan_ms = plan_ms;
    set_l2_window(g);
    if (int rc = copra_buffers(g, K)) return rc;
    Plan& P = g->plan();
    cudaStream_t st = g->stream;
    static int smem_set_device = -1;
    if (smem_set_device != g->device) {
        LP_CK(cudaFuncSetAttribute(k_copra_warp<COPRA_T0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)copra_warp_smem_bytes<kCopraBits, kCopraWarps>()));
        LP_CK(cudaFuncSetAttribute(k_copra_warp<COPRA_T1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)copra_warp_smem_bytes<11, 2>()));
        LP_CK(cudaFuncSetAttribute(k_copra_team, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)copra_team_smem_bytes()));
        smem_set_device = g->device;
    }
    int occ = 1, occ1 = 1;
    LP_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_copra_warp<COPRA_T0>, kCopraWarps * 32,
                                                        copra_warp_smem_bytes<kCopraBits, kCopraWarps>()));
    LP_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, k_copra_warp<COPRA_T1>, 64,
                                                        copra_warp_smem_bytes<11, 2>()));
    occ = std::max(occ, 1);
    occ1 = std::max(occ1, 1);
    int c0 = 0, c1 = 1;  // L0 / X buffer index
    k_copra_init<<<g->num_sms * 8, 256, 0, st>>>(g->clabs[c0], g->cbels[c0], g->csize[c0], g->cbest[c0], n, K);
    if (P.S > 0) k_reset_ndist<<<g->num_sms * 8, 256, 0, st>>>(P.soff, P.ndist, P.S);
    LP_CK(cudaGetLastError());
    CopraArgs a;
    memset(&a, 0, sizeof(a));
    a.soff = P.soff;
    a.snbr = P.snbr;
    a.sw = P.sw;
    a.wmode = g->wmode;
    a.shift = g->fixed_shift;
    a.svid = P.svid;
    a.slot_of = P.slot_of;
    a.K = K;
    a.ndist = P.ndist;
    a.mark = cross ? g->mark : nullptr;
    a.S = (int32_t)P.S;
    a.cursor = g->ccur;
    a.big_len = g->ccur + 1;
    a.big_cursor = g->ccur + 2;
    a.big = g->cbig;
    a.gelab = g->gelab;
    a.geval = g->geval;
    a.gefirst = g->gefirst;
    a.grlab = g->grlab;
    a.grval = g->grval;
    a.gfmap = g->gfmap;
    a.gblab = g->gblab;
    a.gbval = g->gbval;
    a.gbc = g->gbc;
    a.gwc = g->gwc;
    a.gslab = g->gslab;
    a.gsval = g->gsval;
    a.gqs = g->gqs;
    a.gcap_entries = g->gent;
    a.gcap_contrib = g->gcon;
    a.counters = g->counters;
    a.seed = o->seed;
    a.long_row = g->copra_long;
    a.mbits = (cross && g->copra_bitmap) ? g->mbits : nullptr;
    Prof prof;
    prof.on = (o->flags & LP_RAK_PROFILE) != 0;
    prof.pool = &g->event_pool;
    LP_CK(cudaMemsetAsync(g->counters, 0, (kCtrCount + 2) * sizeof(unsigned long long), st));
    LP_CK(cudaEventRecord(g->ev0, st));
    int it = 0, rounds = 0;
    // One round: the team rows known up front (k_copra_route) run on an auxiliary stream beside the
    // warp tiers; rows the tiers spill (a table that overflowed its estimate) follow in a second,
    // usually empty, team pass.
    // (in-place schedules only: their rounds end in the tail of a few hub rows; a synchronous
    // sweep's team pass is throughput-bound and runs slower beside the warp tiers -- measured)
    const bool pre_route = g->copra_overlap && cross && g->aux[1] != nullptr;
    a.pre_routed = pre_route ? 1 : 0;
    auto launch = [&](int64_t work) -> int {
        LP_CK(cudaMemsetAsync(g->ccur, 0, 8 * sizeof(int32_t), st));
        // ccur: [0] tier-0 cursor [1] big length [2] big cursor [3] mid length [4] mid cursor
        //       [5] routed team length [6] routed team cursor
        cudaStream_t sT = g->aux[1];
        if (pre_route) {
            a.route_mark = g->croute_mark;
            a.route_id = ++g->copra_rid;
            prof.begin(st, -1);
            k_copra_route<<<grid_for(work, 256, g->num_sms * 8), 256, 0, st>>>(a, g->croute, g->ccur + 5);
            prof.end(st);
            cudaEventRecord(g->ev_fork, st);
            cudaStreamWaitEvent(sT, g->ev_fork, 0);
            CopraArgs b = a;
            b.big = g->croute;
            b.big_len = g->ccur + 5;
            b.big_cursor = g->ccur + 6;
            prof.begin(sT, kKHub);
            k_copra_team<<<g->gblocks, kCopraTeamWarps * 32, copra_team_smem_bytes(), sT>>>(b);
            prof.end(sT);
            cudaEventRecord(g->ev_join[1], sT);
        }
        prof.begin(st, kKWarp);
        k_copra_warp<COPRA_T0><<<grid_for(work, kCopraWarps, g->num_sms * occ), kCopraWarps * 32,
                                 copra_warp_smem_bytes<kCopraBits, kCopraWarps>(), st>>>(
            a, nullptr, nullptr, g->ccur, g->cmid, g->ccur + 3);
        prof.end(st);
        prof.begin(st, kKTeam);
        k_copra_warp<COPRA_T1><<<g->num_sms * occ1, 64, copra_warp_smem_bytes<11, 2>(), st>>>(
            a, g->cmid, g->ccur + 3, g->ccur + 4, g->cbig, g->ccur + 1);
        prof.end(st);
        if (pre_route) cudaStreamWaitEvent(st, g->ev_join[1], 0);  // (the team scratch is per block: one pass at a time)
        prof.begin(st, kKHub);
        k_copra_team<<<g->gblocks, kCopraTeamWarps * 32, copra_team_smem_bytes(), st>>>(a);  // gblocks <= 2 / SM
        prof.end(st);
        if (a.mbits) {
            // the vertices this round marked -> the next round's queue (bits cleared)
            const int64_t nwords = n / 32 + 1;
            prof.begin(st, -1);
            k_bits_to_queue<<<grid_for(nwords, 256, g->num_sms * 8), 256, 0, st>>>(g->mbits, nwords, a.mq_out, a.mq_len);
            prof.end(st);
        }
        ++rounds;
        return LP_OK;
    };
    const size_t cells = (size_t)n * K;
    while (it < o->max_iterations) {
        ++it;
        a.sweep = (uint32_t)it;
        a.labs0 = g->clabs[c0];
        a.bels0 = g->cbels[c0];
        a.size0 = g->csize[c0];
        a.labsX = g->clabs[c1];
        a.belsX = g->cbels[c1];
        a.sizeX = g->csize[c1];
        a.bestX = g->cbest[c1];
        LP_CK(cudaMemcpyAsync(g->clabs[c1], g->clabs[c0], cells * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        LP_CK(cudaMemcpyAsync(g->cbels[c1], g->cbels[c0], cells * sizeof(double), cudaMemcpyDeviceToDevice, st));
        LP_CK(cudaMemcpyAsync(g->csize[c1], g->csize[c0], n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        LP_CK(cudaMemcpyAsync(g->cbest[c1], g->cbest[c0], n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        // dense round over every active slot, then frontier rounds until nothing is marked
        int q = 0;
        a.queue = nullptr;
        a.queue_len = nullptr;
        a.mq_out = g->mq[q];
        a.mq_len = g->mq_len + q;
        LP_CK(cudaMemsetAsync(g->mq_len, 0, 2 * sizeof(int32_t), st));
        if (P.S > 0)
            if (int rc = launch(P.S)) return rc;
        while (cross && P.S > 0) {
            if (!a.mbits) {
                prof.begin(st, -1);
                k_clear_marks<<<g->num_sms * 4, 256, 0, st>>>(g->mq[q], g->mq_len + q, g->mark);
                prof.end(st);
            }
            LP_CK(cudaMemcpyAsync(g->h_len, g->mq_len + q, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
            LP_CK(cudaStreamSynchronize(st));
            const int32_t work = g->h_len[0];
            if (g->debug_rounds) fprintf(stderr, "[lp] copra sweep %d round %d: queue %d\n", it, rounds, work);
            if (work == 0) break;
            a.queue = g->mq[q];
            a.queue_len = g->mq_len + q;
            a.mq_out = g->mq[q ^ 1];
            a.mq_len = g->mq_len + (q ^ 1);
            LP_CK(cudaMemsetAsync(g->mq_len + (q ^ 1), 0, sizeof(int32_t), st));
            if (int rc = launch(work)) return rc;
            q ^= 1;
        }
        LP_CK(cudaMemsetAsync(g->counters + kCtrChanged, 0, sizeof(unsigned long long), st));
        k_count_changed<<<g->num_sms * 8, 256, 0, st>>>(g->cbest[c0], g->cbest[c1], n, g->counters + kCtrChanged);
        LP_CK(cudaMemcpyAsync(g->h_counters, g->counters, (kCtrCount + 2) * sizeof(unsigned long long),
                              cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
        LP_CK(cudaGetLastError());
        if (g->h_counters[kCtrCount + 1])
            return lp_fail(LP_ERR_UNSUPPORTED, "a row has more distinct labels than the team tables hold");
        if (g->h_counters[kCtrError])
            return lp_fail(LP_ERR_UNSUPPORTED, "a hub row's label partitions overflowed the team table split stack");
        const int64_t changed = (int64_t)g->h_counters[kCtrChanged];
        if (changed_per_iter) changed_per_iter[it - 1] = changed;
        std::swap(c0, c1);  // c0 = this sweep's state
        if ((double)changed <= o->tolerance * (double)n) break;  // copra.py:174-175
    }
    LP_CK(cudaEventRecord(g->ev1, st));
    LP_CK(cudaEventSynchronize(g->ev1));
    float ms = 0.f;
    LP_CK(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
    if (int rc = finish_stats(g, prof, S, it, rounds, 0, ms)) return rc;
    // download (int64 / float64 like the reference's arrays)
    int64_t* l64 = nullptr;
    double* b64 = nullptr;
    int64_t* s64 = nullptr;
    int64_t* best64 = g->out64;
    cudaError_t e = cudaSuccess;
    if (labs_out) {
        e = pool_alloc(&l64, cells * sizeof(int64_t));
        if (e == cudaSuccess) e = pool_alloc(&b64, cells * sizeof(double));
    }
    if (e == cudaSuccess && sizes_out) e = pool_alloc(&s64, n * sizeof(int64_t));
    if (e == cudaSuccess) {
        k_copra_download<<<g->num_sms * 8, 256, 0, st>>>(g->clabs[c0], g->cbels[c0], g->csize[c0], g->cbest[c0], l64,
                                                        b64, s64, best64, n, K, K);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(best_out, best64, n * sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && labs_out) e = cudaMemcpyAsync(labs_out, l64, cells * sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && labs_out) e = cudaMemcpyAsync(bels_out, b64, cells * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && sizes_out) e = cudaMemcpyAsync(sizes_out, s64, n * sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    dfree(l64);
    dfree(b64);
    dfree(s64);
    LP_CK(e);
    return LP_OK;
}

// ---------------------------------------------------------------------------
// modularity (quality.py:10-42) on the device, float64 accumulators
// ---------------------------------------------------------------------------
// warp per row of the input CSR: internal weight (self-loops twice) and the
// community degrees d_c (self-loops twice, graph.degree_weights)
__global__ void k_mod_arcs(const uint32_t* __restrict__ off, const int32_t* __restrict__ nbr,
                           const uint32_t* __restrict__ w, int wmode, int shift, const int32_t* __restrict__ lab,
                           int64_t n, double* __restrict__ dc, double* internal) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
    double in_sum = 0.0;
    for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; v < n; v += warps) {
        const int32_t lv = lab[v];
        double deg = 0.0;
        for (uint32_t e = off[v] + lane; e < off[v + 1]; e += 32) {
            const int32_t u = nbr[e];
            double we = 1.0;
            if (w) we = wmode == kFixed ? ldexp((double)w[e], -shift) : (double)__uint_as_float(w[e]);
            if (u == (int32_t)v) we *= 2.0;
            deg += we;
            if (lab[u] == lv) in_sum += we;
        }
        for (int o = 16; o >= 1; o >>= 1) deg += __shfl_xor_sync(0xffffffffu, deg, o);
        if (lane == 0 && deg != 0.0) atomicAdd(dc + lv, deg);
    }
    for (int o = 16; o >= 1; o >>= 1) in_sum += __shfl_xor_sync(0xffffffffu, in_sum, o);
    if (lane == 0 && in_sum != 0.0) atomicAdd(internal, in_sum);
}

__global__ void k_mod_squares(const double* __restrict__ dc, int64_t n, double inv_total, double* out) {
    double acc = 0.0;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
        const double x = dc[c] * inv_total;
        acc += x * x;
    }
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc != 0.0) atomicAdd(out, acc);
}

__global__ void k_labels_from64(const int64_t* __restrict__ in, int32_t* __restrict__ out, int64_t n) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        out[v] = (int32_t)in[v];
}

extern "C" int lp_modularity(lp_graph* g, const int64_t* labels, double total_weight, double* q_out) {
    if (!g || !q_out) return lp_fail(LP_ERR_INVALID, "NULL argument");
    *q_out = 0.0;
    if (g->n == 0 || !(total_weight > 0.0)) return LP_OK;
    LP_CK(cudaSetDevice(g->device));
    StreamScope ss(g->stream);
    cudaStream_t st = g->stream;
    const int64_t n = g->n;
    const int32_t* lab = nullptr;
    int32_t* tmp = nullptr;
    if (labels) {
        LP_CK(cudaMemcpyAsync(g->out64, labels, n * sizeof(int64_t), cudaMemcpyHostToDevice, st));
        LP_CK(cudaMemsetAsync(g->counters, 0, sizeof(unsigned long long), st));
        k_check_labels<<<g->num_sms * 4, 256, 0, st>>>(g->out64, n, g->counters);
        unsigned long long bad = 0;
        LP_CK(cudaMemcpyAsync(&bad, g->counters, sizeof(bad), cudaMemcpyDeviceToHost, st));
        LP_CK(cudaStreamSynchronize(st));
        if (bad) return lp_fail(LP_ERR_INVALID, "community labels must lie in [0, vertex_count)");
        LP_CK(pool_alloc(&tmp, n * sizeof(int32_t)));
        k_labels_from64<<<g->num_sms * 8, 256, 0, st>>>(g->out64, tmp, n);
        lab = tmp;
    } else {
        if (!g->labels_valid) return lp_fail(LP_ERR_INVALID, "no labels: run a detection first");
        lab = g->cur;
    }
    double* dc = nullptr;
    cudaError_t e = pool_alloc(&dc, (n + 2) * sizeof(double));
    if (e == cudaSuccess) e = cudaMemsetAsync(dc, 0, (n + 2) * sizeof(double), st);
    if (e == cudaSuccess) {
        k_mod_arcs<<<g->num_sms * 16, 256, 0, st>>>(g->off, g->nbr, g->w, g->wmode, g->fixed_shift, lab, n, dc,
                                                    dc + n);
        k_mod_squares<<<g->num_sms * 8, 256, 0, st>>>(dc, n, 1.0 / total_weight, dc + n + 1);
        e = cudaGetLastError();
    }
    double h[2] = {0.0, 0.0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(h, dc + n, 2 * sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    dfree(dc);
    dfree(tmp);
    LP_CK(e);
    *q_out = h[0] / total_weight - h[1];
    return LP_OK;
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

// ---------------------------------------------------------------------------
// calibration: memory-only passes over the storage CSR (no tally)
// ---------------------------------------------------------------------------
// mode 0: stream every neighbour index once (the compulsory DRAM traffic)
// mode 1: index + neighbour-label gather, per-row XOR (the sweep's memory
//         pattern without any hashing) -- the practical floor of a sweep
// mode 0/1: warp per row, plain loop (the naive structure)
// mode 2/3: flat arc-parallel stream, 8 loads in flight per thread (the floor)
// (the storage CSR packs neighbour id << 2; the original CSR holds plain ids)
__global__ void k_calib(const uint32_t* __restrict__ soff, const uint32_t* __restrict__ snbr, int shift,
                        const int32_t* __restrict__ lab, int64_t S, int mode, unsigned long long* sink) {
    const int lane = threadIdx.x & 31;
    unsigned acc = 0;
    if (mode < 2) {
        const int64_t warps = (int64_t)gridDim.x * blockDim.x / 32;
        for (int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; s < S; s += warps) {
            const uint32_t b = soff[s], e = soff[s + 1];
            for (uint32_t k = b + lane; k < e; k += 32) {
                const uint32_t u = __ldg(snbr + k) >> shift;
                acc ^= mode ? (unsigned)__ldg(lab + u) : u;
            }
        }
    } else {
        const int64_t m = soff[S];
        const int64_t stride = (int64_t)gridDim.x * blockDim.x;
        for (int64_t base = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; base < m; base += stride * 8) {
            uint32_t u[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int64_t e = base + j * stride;
                u[j] = e < m ? (__ldg(snbr + e) >> shift) : 0u;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) acc ^= mode == 3 ? (unsigned)__ldg(lab + u[j]) : u[j];
        }
    }
    acc = __reduce_xor_sync(0xffffffffu, acc);
    if (lane == 0 && acc == 0x12345678u) atomicAdd(sink, 1ull);
}

extern "C" int lp_calibrate(lp_graph* g, int32_t mode, int32_t reps, double* ms_out) {
    if (!g || !ms_out || reps < 1 || mode < 0 || mode > 5) return lp_fail(LP_ERR_INVALID, "bad arguments");
    if (!g->plan().valid) return lp_fail(LP_ERR_INVALID, "run a detection first (plan needed)");
    LP_CK(cudaSetDevice(g->device));
    const Plan& P = g->plan();
    cudaStream_t st = g->stream;
    k_init_labels<<<g->num_sms * 8, 256, 0, st>>>(nullptr, g->labA, g->n);
    // mode 4/5: the same flat passes over the ORIGINAL CSR (vertex-id order)
    const uint32_t* soff = mode >= 4 ? g->off : P.soff;
    const uint32_t* snbr = mode >= 4 ? (const uint32_t*)g->nbr : P.snbr;
    const int shift = mode >= 4 ? 0 : 2;
    const int64_t rows = mode >= 4 ? g->n : P.S;
    const int km = mode >= 4 ? mode - 2 : mode;
    k_calib<<<g->num_sms * 16, 256, 0, st>>>(soff, snbr, shift, g->labA, rows, km, g->counters);
    LP_CK(cudaEventRecord(g->ev0, st));
    for (int r = 0; r < reps; ++r)
        k_calib<<<g->num_sms * 16, 256, 0, st>>>(soff, snbr, shift, g->labA, rows, km, g->counters);
    LP_CK(cudaEventRecord(g->ev1, st));
    LP_CK(cudaEventSynchronize(g->ev1));
    float ms = 0.f;
    LP_CK(cudaEventElapsedTime(&ms, g->ev0, g->ev1));
    *ms_out = ms / reps;
    return LP_OK;
}
