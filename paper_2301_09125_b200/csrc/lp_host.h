// lp_host.h -- host-side helpers of liblabelprop_cuda (error slot, RNG).
#pragma once
#include <cstdint>

// thread-local error message for lp_last_error()
void lp_set_error(const char* fmt, ...);
// set the message and return `code`
int lp_fail(int code, const char* fmt, ...);
// prng.shuffled_indices (prng.py:82-94), byte-identical
void lp_host_shuffled_indices(int64_t n, uint32_t seed, int64_t* out);
