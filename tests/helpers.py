"""Shared test helpers: seeded configurations in the style of the reference's
property tests (proj/tests/test_async_sim.cpp:14-18, acceptance.cpp:37-65)."""
from __future__ import annotations

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


class SplitMix64:
    """rng.hpp:16-41, restated for test-input generation."""

    def __init__(self, seed: int):
        self.s = seed & M64

    def next(self) -> int:
        self.s = (self.s + GAMMA) & M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def next_bounded(self, b: int) -> int:
        return self.next() % (b + 1)


def random_field(rng: SplitMix64, n: int) -> np.ndarray:
    """test_async_sim.cpp:14-18: uniform in [-2, 2)."""
    return np.array([rng.next_double() * 4.0 - 2.0 for _ in range(n)], np.float64)


def random_divisor(rng: SplitMix64, n: int) -> int:
    """acceptance.cpp:59-65"""
    divs = [d for d in range(1, n + 1) if n % d == 0]
    return divs[rng.next_bounded(len(divs) - 1)]


def fnv1a64(v: np.ndarray) -> int:
    h = 1469598103934665603
    for b in np.ascontiguousarray(v, np.float64).tobytes():
        h ^= b
        h = (h * 1099511628211) & M64
    return h


def sine_field(n: int) -> np.ndarray:
    """BASELINE sine IC u_i = sin(pi*i/(N-1)) via libm sin (math.sin), ends snapped."""
    import math
    v = np.array([math.sin(math.pi * float(i) / float(n - 1)) for i in range(n)], np.float64)
    v[0] = 0.0
    v[-1] = 0.0
    return v


def bits_equal(a: np.ndarray, b: np.ndarray) -> bool:
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    return a.shape == b.shape and bool(np.all(a.view(np.uint64) == b.view(np.uint64)))
