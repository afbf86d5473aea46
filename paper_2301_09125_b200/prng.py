"""xorshift32 generator and the seeded visit order (host side).

Same definitions as the reference's ``labelprop.prng``
(`pkg/src/labelprop/prng.py:29-120`): Marsaglia's (13, 17, 5) triple shift
on 32 bits, modulo-bounded draws, murmur3-fmix32 worker seeding and the
Fisher-Yates visit permutation ``shuffled_indices``.  The permutation is
computed by the C library (``lp_shuffled_indices``), byte-identical to the
reference's, because it defines the batch / position layout the CUDA
engine sweeps in.

Device-side randomness does not use this stream: a parallel sweep cannot
replay a sequential stream's draw order, so non-strict ties on the GPU use
the counter hash of ``csrc/lp_common.cuh``.
"""

from __future__ import annotations

import numpy as np

_MASK = 0xFFFFFFFF
ZERO_SEED_REPLACEMENT = 2463534242
ORDER_STREAM = 0x4F524452


def xs32_next(state: int) -> int:
    """One xorshift32 step; the new state is the output (ref prng.py:29-36)."""
    x = int(state) & _MASK
    x = (x ^ (x << 13)) & _MASK
    x ^= x >> 17
    x = (x ^ (x << 5)) & _MASK
    return x


def draw_bounded(states, slot: int, n: int) -> int:
    """Advance ``states[slot]`` and reduce modulo ``n`` (ref prng.py:39-44)."""
    x = xs32_next(states[slot])
    states[slot] = x
    return x % n


def mix_seed(seed: int, k: int) -> int:
    """murmur3 fmix32 over ``seed + k * 0x9E3779B9``; never 0 (ref prng.py:47-63)."""
    x = (int(seed) + int(k) * 0x9E3779B9) & _MASK
    x ^= x >> 16
    x = (x * 0x85EBCA6B) & _MASK
    x ^= x >> 13
    x = (x * 0xC2B2AE35) & _MASK
    x ^= x >> 16
    return x or ZERO_SEED_REPLACEMENT


def worker_states(seed: int, workers: int) -> np.ndarray:
    """Worker k starts at ``mix_seed(seed, k)`` (ref prng.py:66-74)."""
    return np.array([mix_seed(int(seed) & _MASK, k) for k in range(workers)], dtype=np.int64)


def shuffled_indices(n: int, seed: int) -> np.ndarray:
    """Seeded permutation of range(n) (ref prng.py:89-94), computed natively."""
    from . import _lib

    out = np.empty(int(n), dtype=np.int64)
    _lib.check(_lib.lib().lp_shuffled_indices(int(n), int(seed) & _MASK, out))
    return out


class XorShift32:
    """Single-stream generator (ref prng.py:97-120)."""

    def __init__(self, seed: int):
        s = int(seed) & _MASK
        self._state = np.array([s or ZERO_SEED_REPLACEMENT], dtype=np.int64)

    @property
    def state(self) -> int:
        return int(self._state[0])

    def next(self) -> int:
        x = xs32_next(self._state[0])
        self._state[0] = x
        return x

    def next_bounded(self, n: int) -> int:
        if n < 1:
            raise ValueError("bound must be a positive integer")
        return draw_bounded(self._state, 0, n)
