// lp_gen.cpp -- native graph builders (host, OpenMP).
//
// The benchmark graphs of BASELINE.json are tens to hundreds of millions of
// arcs; building them with numpy (sort-based dedupe, then the reference's
// from_arcs/preprocess path, graph.py:58-84,254-306) takes minutes.  These
// builders produce the same canonical CSR -- symmetric, duplicates merged,
// generated self-loops dropped, one weight-1 self-loop per vertex, rows
// sorted by neighbour id -- in seconds.  tests/test_host_abi.py checks them
// arc for arc against graph.preprocess(graph.from_arcs(...)).
#include <omp.h>
#include <parallel/algorithm>

#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/labelprop_cuda.h"
#include "lp_host.h"

static inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// R-MAT edge list: edge i, bit level l draws u = splitmix64(seed, i, l) in
// [0, 1) and picks the quadrant a | b | c | d; no noise, no id scrambling.
extern "C" int lp_gen_rmat(int32_t scale, int64_t edges, double a, double b, double c, uint64_t seed, int64_t* src,
                           int64_t* dst) {
    if (scale < 1 || scale > 30 || edges < 0 || !src || !dst) return lp_fail(LP_ERR_INVALID, "bad R-MAT arguments");
    if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0)) return lp_fail(LP_ERR_INVALID, "bad R-MAT probabilities");
    const uint64_t ta = (uint64_t)(a * 9007199254740992.0), tab = (uint64_t)((a + b) * 9007199254740992.0),
                   tabc = (uint64_t)((a + b + c) * 9007199254740992.0);
    const uint64_t key = splitmix64(seed ^ 0x524D4154ull);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < edges; ++i) {
        int64_t s = 0, d = 0;
        const uint64_t base = key ^ ((uint64_t)i * 64ull);
        for (int l = scale - 1; l >= 0; --l) {
            const uint64_t r = splitmix64(base + (uint64_t)l) >> 11;  // 53 bits
            const int64_t sb = r >= tab, db = (r >= ta && r < tab) || r >= tabc;
            s |= sb << l;
            d |= db << l;
        }
        src[i] = s;
        dst[i] = d;
    }
    return LP_OK;
}

// Canonical preprocessed CSR from an undirected pair list (unit weights).
// neighbors must hold 2*pairs + n entries; *m_out receives the arc count.
extern "C" int lp_csr_build_undirected(int64_t n, int64_t pairs, const int64_t* u, const int64_t* v, int64_t* offsets,
                                       int64_t* neighbors, int64_t* m_out) {
    if (n < 0 || pairs < 0 || !offsets || !m_out || (pairs > 0 && (!u || !v)) || (n > 0 && !neighbors))
        return lp_fail(LP_ERR_INVALID, "bad CSR arguments");
    if (n >= (int64_t)1 << 31) return lp_fail(LP_ERR_UNSUPPORTED, "vertex count must be < 2^31");
    std::vector<uint64_t> keys((size_t)pairs);
    int64_t bad = 0;
#pragma omp parallel for reduction(+ : bad)
    for (int64_t i = 0; i < pairs; ++i) {
        const int64_t a = u[i], b = v[i];
        if (a < 0 || b < 0 || a >= n || b >= n) {
            ++bad;
            keys[i] = ~0ull;
            continue;
        }
        const uint64_t lo = (uint64_t)(a < b ? a : b), hi = (uint64_t)(a < b ? b : a);
        keys[i] = lo == hi ? ~0ull : (lo << 32) | hi;  // self pairs sort last and are dropped
    }
    if (bad) return lp_fail(LP_ERR_INVALID, "pair endpoints must lie in [0, n)");
    __gnu_parallel::sort(keys.begin(), keys.end());
    int64_t k = 0;
    for (int64_t i = 0; i < pairs; ++i) {
        if (keys[i] == ~0ull) break;
        if (k == 0 || keys[i] != keys[k - 1]) keys[k++] = keys[i];
    }
    std::vector<int64_t> deg((size_t)n, 1);  // the self-loop
    for (int64_t i = 0; i < k; ++i) {
        ++deg[keys[i] >> 32];
        ++deg[keys[i] & 0xffffffffull];
    }
    offsets[0] = 0;
    for (int64_t r = 0; r < n; ++r) offsets[r + 1] = offsets[r] + deg[r];
    // row r = [lo < r ascending] + [r] + [hi > r ascending]; walking the
    // sorted (lo, hi) keys fills both blocks in ascending order
    std::vector<int64_t> cur(offsets, offsets + n);
    // reverse arcs first (row hi gets lo), then self-loop, then forward arcs
    for (int64_t i = 0; i < k; ++i) {
        const int64_t hi = (int64_t)(keys[i] & 0xffffffffull), lo = (int64_t)(keys[i] >> 32);
        neighbors[cur[hi]++] = lo;
    }
    for (int64_t r = 0; r < n; ++r) neighbors[cur[r]++] = r;
    for (int64_t i = 0; i < k; ++i) {
        const int64_t hi = (int64_t)(keys[i] & 0xffffffffull), lo = (int64_t)(keys[i] >> 32);
        neighbors[cur[lo]++] = hi;
    }
    *m_out = offsets[n];
    return LP_OK;
}
