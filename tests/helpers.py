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


def async_step_cases(seed: int, count: int, n_max: int = 60):
    """Random async_step inputs (async_sim.cpp:107-116): a ring at a random
    step with min(depth, step + 1) snapshots, a random partition / BC / law,
    and a random stream position.  One case in four has depth < q, so late
    draws can reach past the ring (HistoryRing::read's logic_error)."""
    gen = SplitMix64(seed)
    cases = []
    for _ in range(count):
        n = 3 + gen.next_bounded(n_max - 3)
        q = 1 + gen.next_bounded(7)
        depth = q if gen.next_bounded(3) else 1 + gen.next_bounded(q - 1) if q > 1 else 1
        step = gen.next_bounded(12)
        held = min(depth, step + 1)
        law = int(gen.next_bounded(2))
        cases.append(dict(
            snaps=np.stack([random_field(gen, n) for _ in range(held)]),
            depth=depth, step=step, r=0.5 * (gen.next_double() * 0.999 + 0.001),
            bc=int(gen.next() & 1), c1=gen.next_double(), c2=gen.next_double(),
            part_total=n, per_pe=random_divisor(gen, n), law=law, q=q,
            fixed_d=int(gen.next_bounded(q - 1)) if law == 1 else 0,
            p=0.05 + 0.9 * gen.next_double(), rng_state=gen.next()))
    return cases
