// lp_build.cu -- graph builders on the GPU.
//
// The canonical preprocessed CSR of an undirected pair list -- symmetric,
// duplicates merged, generated self-loops dropped, one self-loop per vertex,
// rows sorted by neighbour id (what graph.preprocess(graph.from_arcs(...))
// returns for unit weights, graph.py:58-84,254-306) -- built with device
// sorts instead of numpy / the host builder: the same arrays arc for arc as
// lp_csr_build_undirected (tests/test_rak_gpu.py checks it).
//
//   keys  = (min << 32 | max) of every non-self pair, radix-sorted, unique
//   rev   = (max << 32 | min) of the unique keys, radix-sorted
//   row r = [rev keys of major r] ++ [r] ++ [fwd keys of major r]
#include <cuda_runtime.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <cstring>

#include "../../include/labelprop_cuda.h"
#include "lp_host.h"

namespace {

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

constexpr uint64_t kNoKey = ~0ull;

// the R-MAT draw of lp_gen_rmat (lp_gen.cpp), one thread per edge
__global__ void k_rmat_keys(int scale, int64_t edges, uint64_t ta, uint64_t tab, uint64_t tabc, uint64_t key,
                            uint64_t* __restrict__ keys) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < edges; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t s = 0, d = 0;
        const uint64_t base = key ^ ((uint64_t)i * 64ull);
        for (int l = scale - 1; l >= 0; --l) {
            const uint64_t r = splitmix64(base + (uint64_t)l) >> 11;
            const uint64_t sb = r >= tab, db = (r >= ta && r < tab) || r >= tabc;
            s |= sb << l;
            d |= db << l;
        }
        const uint64_t lo = s < d ? s : d, hi = s < d ? d : s;
        keys[i] = lo == hi ? kNoKey : (lo << 32) | hi;
    }
}

__global__ void k_pair_keys(const int64_t* __restrict__ u, const int64_t* __restrict__ v, int64_t pairs, int64_t n,
                            uint64_t* __restrict__ keys, unsigned long long* bad) {
    unsigned long long b = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < pairs; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = u[i], c = v[i];
        if (a < 0 || c < 0 || a >= n || c >= n) {
            ++b;
            keys[i] = kNoKey;
            continue;
        }
        const uint64_t lo = (uint64_t)(a < c ? a : c), hi = (uint64_t)(a < c ? c : a);
        keys[i] = lo == hi ? kNoKey : (lo << 32) | hi;
    }
    if (b) atomicAdd(bad, b);
}

__global__ void k_rev_and_counts(const uint64_t* __restrict__ fwd, int64_t k, uint64_t* __restrict__ rev,
                                 int32_t* __restrict__ fcount, int32_t* __restrict__ rcount) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = fwd[i];
        const uint64_t lo = key >> 32, hi = key & 0xffffffffull;
        rev[i] = (hi << 32) | lo;
        atomicAdd(fcount + lo, 1);
        atomicAdd(rcount + hi, 1);
    }
}

__global__ void k_degrees(const int32_t* __restrict__ fcount, const int32_t* __restrict__ rcount,
                          int64_t* __restrict__ deg, int64_t n) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        deg[r] = (int64_t)fcount[r] + rcount[r] + 1;
}

// row r: [rev of major r][r][fwd of major r]; run starts by exclusive scans
__global__ void k_fill(const uint64_t* __restrict__ fwd, const uint64_t* __restrict__ rev, int64_t k,
                       const int64_t* __restrict__ off, const int64_t* __restrict__ fstart,
                       const int64_t* __restrict__ rstart, const int32_t* __restrict__ rcount,
                       int64_t* __restrict__ nbr, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t f = fwd[i], rv = rev[i];
        const int64_t fr = (int64_t)(f >> 32), rr = (int64_t)(rv >> 32);
        nbr[off[fr] + rcount[fr] + 1 + (i - fstart[fr])] = (int64_t)(f & 0xffffffffull);
        nbr[off[rr] + (i - rstart[rr])] = (int64_t)(rv & 0xffffffffull);
    }
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
        nbr[off[r] + rcount[r]] = r;
}

__global__ void k_i32_to_i64(const int32_t* __restrict__ in, int64_t* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

struct DevBuf {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
};

#define B_CK(call)                                                                                            \
    do {                                                                                                      \
        cudaError_t _e = (call);                                                                              \
        if (_e != cudaSuccess)                                                                                \
            return lp_fail(_e == cudaErrorMemoryAllocation ? LP_ERR_NOMEM : LP_ERR_CUDA, "CUDA error %s at %s:%d", \
                           cudaGetErrorName(_e), __FILE__, __LINE__);                                         \
    } while (0)

template <typename T> cudaError_t balloc(DevBuf& b, T** p, size_t count, cudaStream_t st) {
    b.st = st;
    cudaError_t e = cudaMallocAsync(&b.p, std::max<size_t>(count, 1) * sizeof(T), st);
    *p = (T*)b.p;
    return e;
}

// keys[0..count) hold (lo << 32 | hi) or kNoKey; builds the CSR into the
// host arrays offsets[n+1] / neighbors[*m_out]
int build_from_keys(int64_t n, uint64_t* keys, int64_t count, cudaStream_t st, int sms, int64_t* offsets,
                    int64_t* neighbors, int64_t neighbors_cap, int64_t* m_out) {
    const int G = sms * 8;
    DevBuf b_sorted, b_tmp, b_rev, b_rev2, b_cnt, b_deg, b_off, b_fst, b_rst, b_nbr, b_k;
    uint64_t *sorted, *rev, *rev2;
    int32_t* cnt;
    int64_t *deg, *off, *fst, *rst, *nbr, *dk;
    B_CK(balloc(b_sorted, &sorted, count, st));
    size_t need = 0, need2 = 0, need3 = 0;
    B_CK(cub::DeviceRadixSort::SortKeys(nullptr, need, keys, sorted, (int)count, 0, 64, st));
    B_CK(cub::DeviceSelect::Unique(nullptr, need2, sorted, keys, (int64_t*)nullptr, (int)count, st));
    B_CK(cub::DeviceScan::ExclusiveSum(nullptr, need3, (int64_t*)nullptr, (int64_t*)nullptr, (int)(n + 1), st));
    void* tmp;
    B_CK(balloc(b_tmp, (char**)&tmp, std::max(need, std::max(need2, need3)), st));
    B_CK(cub::DeviceRadixSort::SortKeys(tmp, need, keys, sorted, (int)count, 0, 64, st));
    B_CK(balloc(b_k, &dk, 1, st));
    B_CK(cub::DeviceSelect::Unique(tmp, need2, sorted, keys, dk, (int)count, st));
    int64_t uniq = 0;
    B_CK(cudaMemcpyAsync(&uniq, dk, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    B_CK(cudaStreamSynchronize(st));
    int64_t k = uniq;
    if (k > 0) {
        uint64_t last = 0;
        B_CK(cudaMemcpyAsync(&last, keys + k - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        B_CK(cudaStreamSynchronize(st));
        if (last == kNoKey) --k;  // the self pairs
    }
    const int64_t m = 2 * k + n;
    if (m > neighbors_cap) return lp_fail(LP_ERR_INVALID, "neighbors buffer too small");
    B_CK(balloc(b_rev, &rev, k, st));
    B_CK(balloc(b_rev2, &rev2, k, st));
    B_CK(balloc(b_cnt, &cnt, 2 * n, st));
    B_CK(cudaMemsetAsync(cnt, 0, 2 * n * sizeof(int32_t), st));
    int32_t* fcount = cnt;
    int32_t* rcount = cnt + n;
    k_rev_and_counts<<<G, 256, 0, st>>>(keys, k, rev, fcount, rcount);
    B_CK(cub::DeviceRadixSort::SortKeys(tmp, need, rev, rev2, (int)k, 0, 64, st));
    B_CK(balloc(b_deg, &deg, n + 1, st));
    B_CK(balloc(b_off, &off, n + 1, st));
    B_CK(balloc(b_fst, &fst, n + 1, st));
    B_CK(balloc(b_rst, &rst, n + 1, st));
    k_degrees<<<G, 256, 0, st>>>(fcount, rcount, deg, n);
    B_CK(cudaMemsetAsync(deg + n, 0, sizeof(int64_t), st));
    B_CK(cub::DeviceScan::ExclusiveSum(tmp, need3, deg, off, (int)(n + 1), st));
    k_i32_to_i64<<<G, 256, 0, st>>>(fcount, deg, n);
    B_CK(cub::DeviceScan::ExclusiveSum(tmp, need3, deg, fst, (int)(n + 1), st));
    k_i32_to_i64<<<G, 256, 0, st>>>(rcount, deg, n);
    B_CK(cub::DeviceScan::ExclusiveSum(tmp, need3, deg, rst, (int)(n + 1), st));
    B_CK(balloc(b_nbr, &nbr, m, st));
    k_fill<<<G, 256, 0, st>>>(keys, rev2, k, off, fst, rst, rcount, nbr, n);
    B_CK(cudaGetLastError());
    B_CK(cudaMemcpyAsync(offsets, off, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    B_CK(cudaMemcpyAsync(neighbors, nbr, m * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    B_CK(cudaStreamSynchronize(st));
    *m_out = m;
    return LP_OK;
}

struct Ctx {
    cudaStream_t st = nullptr;
    int sms = 148;
    ~Ctx() {
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
    }
};

int open_ctx(Ctx& c, int32_t device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return lp_fail(LP_ERR_CUDA, "no CUDA device available (liblabelprop_cuda needs a B200)");
    if (device >= 0) B_CK(cudaSetDevice(device));
    int dev = 0;
    B_CK(cudaGetDevice(&dev));
    cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev);
    B_CK(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking));
    return LP_OK;
}

}  // namespace

extern "C" int lp_gen_rmat_csr(int32_t scale, int64_t edges, double a, double b, double c, uint64_t seed,
                               int32_t device, int64_t* offsets, int64_t* neighbors, int64_t neighbors_cap,
                               int64_t* m_out) {
    if (scale < 1 || scale > 30 || edges < 0 || !offsets || !neighbors || !m_out)
        return lp_fail(LP_ERR_INVALID, "bad R-MAT arguments");
    if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0)) return lp_fail(LP_ERR_INVALID, "bad R-MAT probabilities");
    Ctx ctx;
    if (int rc = open_ctx(ctx, device)) return rc;
    const int64_t n = (int64_t)1 << scale;
    const uint64_t ta = (uint64_t)(a * 9007199254740992.0), tab = (uint64_t)((a + b) * 9007199254740992.0),
                   tabc = (uint64_t)((a + b + c) * 9007199254740992.0);
    DevBuf bk;
    uint64_t* keys;
    B_CK(balloc(bk, &keys, edges, ctx.st));
    k_rmat_keys<<<ctx.sms * 8, 256, 0, ctx.st>>>(scale, edges, ta, tab, tabc, splitmix64(seed ^ 0x524D4154ull), keys);
    B_CK(cudaGetLastError());
    return build_from_keys(n, keys, edges, ctx.st, ctx.sms, offsets, neighbors, neighbors_cap, m_out);
}

extern "C" int lp_csr_build_undirected_gpu(int64_t n, int64_t pairs, const int64_t* u, const int64_t* v,
                                           int32_t device, int64_t* offsets, int64_t* neighbors,
                                           int64_t neighbors_cap, int64_t* m_out) {
    if (n < 0 || pairs < 0 || !offsets || !m_out || (pairs > 0 && (!u || !v)) || (n > 0 && !neighbors))
        return lp_fail(LP_ERR_INVALID, "bad CSR arguments");
    if (n >= (int64_t)1 << 31) return lp_fail(LP_ERR_UNSUPPORTED, "vertex count must be < 2^31");
    Ctx ctx;
    if (int rc = open_ctx(ctx, device)) return rc;
    DevBuf bk, bu, bv, bb;
    uint64_t* keys;
    int64_t *du, *dv;
    unsigned long long* bad;
    B_CK(balloc(bk, &keys, pairs, ctx.st));
    B_CK(balloc(bu, &du, pairs, ctx.st));
    B_CK(balloc(bv, &dv, pairs, ctx.st));
    B_CK(balloc(bb, &bad, 1, ctx.st));
    B_CK(cudaMemcpyAsync(du, u, pairs * sizeof(int64_t), cudaMemcpyHostToDevice, ctx.st));
    B_CK(cudaMemcpyAsync(dv, v, pairs * sizeof(int64_t), cudaMemcpyHostToDevice, ctx.st));
    B_CK(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), ctx.st));
    k_pair_keys<<<ctx.sms * 8, 256, 0, ctx.st>>>(du, dv, pairs, n, keys, bad);
    unsigned long long hb = 0;
    B_CK(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, ctx.st));
    B_CK(cudaStreamSynchronize(ctx.st));
    if (hb) return lp_fail(LP_ERR_INVALID, "pair endpoints must lie in [0, n)");
    return build_from_keys(n, keys, pairs, ctx.st, ctx.sms, offsets, neighbors, neighbors_cap, m_out);
}
