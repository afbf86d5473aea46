// lp_host.cpp -- host utilities of liblabelprop_cuda.
//
// lp_shuffled_indices restates the reference's visit-order generator
// (prng.py:82-94): Fisher-Yates over range(n) driven by xorshift32
// (prng.py:29-44) seeded with mix_seed(seed, 0x4F524452) (prng.py:47-63,
// :79).  The engine consumes this order to define batches and positions,
// so it must match the reference byte for byte (tests/test_host_abi.py
// checks it against the golden fixture).
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "../../include/labelprop_cuda.h"
#include "lp_host.h"

static thread_local char g_err[512] = "";

void lp_set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int lp_fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

static inline uint32_t xs32(uint32_t x) {
    x ^= x << 13;
    x ^= x >> 17;
    x ^= x << 5;
    return x;
}

static inline uint32_t mix_seed(uint32_t seed, uint32_t k) {
    uint32_t x = seed + k * 0x9E3779B9u;
    x ^= x >> 16;
    x *= 0x85EBCA6Bu;
    x ^= x >> 13;
    x *= 0xC2B2AE35u;
    x ^= x >> 16;
    return x ? x : 2463534242u;
}

void lp_host_shuffled_indices(int64_t n, uint32_t seed, int64_t* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = i;
    uint32_t st = mix_seed(seed, 0x4F524452u);
    for (int64_t i = n - 1; i > 0; --i) {
        st = xs32(st);
        const int64_t j = (int64_t)(st % (uint32_t)(i + 1));
        const int64_t t = out[i];
        out[i] = out[j];
        out[j] = t;
    }
}

extern "C" int lp_shuffled_indices(int64_t n, uint32_t seed, int64_t* out) {
    if (n < 0 || (n > 0 && !out)) return lp_fail(LP_ERR_INVALID, "bad arguments");
    lp_host_shuffled_indices(n, seed, out);
    return LP_OK;
}

extern "C" const char* lp_last_error(void) { return g_err; }

extern "C" const char* lp_version(void) { return "labelprop-b200 0.1.0 (sm_100a)"; }
