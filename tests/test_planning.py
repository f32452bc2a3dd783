"""Host-side planning logic, on the CPU (no device): the invariants the GPU
paths' correctness rests on.

* streamed sync_run (csrc/sync_host.cu stream_chunk_plan): boundaries start at
  0, end at N, increase, every chunk start is a 32-point unit (tensor-map
  coordinates), every chunk is wider than (passes + 1) x halo (the shifted
  ranges R(pi, c) stay non-empty and ordered), graded head/tail on big fields;
* K5 tile geometry (stream_host.cu stream_geometry): a PE spans >= 2 tiles and
  its last tile holds >= H points (an interior tile's window never reaches
  into the next PE), preferring 48x64 over 48x32 over 32x32;
* K3 layout (async_host.cu k3_layout): segments only in lockstep mode, S*V >=
  n, >= 4 warps when PEs share a warp, shared rings only for one CTA."""
import ctypes

import pytest

from paper_1510_08982_b200 import _lib

WAVE_B200 = 148 * 2 * 4 * 1408  # SMs x CTAs/SM x warps/CTA x exact points per 48x64 tile


def plan(n, wave):
    L = _lib.lib()
    cap = 4096
    out = (ctypes.c_size_t * cap)()
    cnt = ctypes.c_size_t(0)
    assert L.heat_stream_chunk_plan(n, wave, out, cap, ctypes.byref(cnt)) == 0
    return [out[i] for i in range(cnt.value)]


@pytest.mark.parametrize("n", [1 << 24, (1 << 24) + 12345, (1 << 28) + 4321, 1 << 30,
                               (1 << 30) + 777, 3 << 29, (1 << 31) - 32])
@pytest.mark.parametrize("wave", [WAVE_B200, 148 * 3 * 4 * 960, 1000 * 32])
def test_stream_chunk_plan_invariants(n, wave):
    B = plan(n, wave)
    assert B[0] == 0 and B[-1] == n
    assert all(a < b for a, b in zip(B, B[1:]))
    assert all(b % 32 == 0 for b in B[:-1])
    worst_passes = 128  # kStreamMaxPasses: the streamed path's limit
    for a, b in zip(B, B[1:]):
        assert b - a > (worst_passes + 1) * 64
    if n >= 128 * wave:  # graded: the head grows, the tail mirrors it
        sizes = [b - a for a, b in zip(B, B[1:])]
        assert sizes[0] == 4 * wave
        assert sizes[1] > sizes[0] and sizes[2] > sizes[1]
        assert sizes[1] <= 2 * sizes[0]  # growth below the compute/copy ratio ~1.8
        assert sizes[-1] >= 4 * wave and sizes[-1] < 4 * wave + 32
    else:
        assert len(B) - 1 <= 16


def k5(n):
    v, h = ctypes.c_int(), ctypes.c_int()
    assert _lib.lib().heat_k5_geometry(n, ctypes.byref(v), ctypes.byref(h)) == 0
    return v.value, h.value


def test_k5_geometry_invariants():
    seen = set()
    for n in range(1056, 200000, 32 * 37):  # PE widths the stream kernel takes (multiples of 32)
        V, H = k5(n)
        seen.add((V, H))
        out = 32 * V - 2 * H
        tiles = -(-n // out)
        assert tiles >= 2
        rem = n % out
        assert rem == 0 or rem >= H
        if (V, H) != (48, 64):  # the preferred geometry must really not fit
            assert n <= 1408 or 0 < n % 1408 < 64
    for n in (32768, 4256, 1056):
        seen.add(k5(n))
    assert k5(32768) == (48, 64) and k5(4256) == (48, 32) and k5(1056) == (32, 32)
    assert {(48, 64), (48, 32), (32, 32)} <= seen


def k3(n, P, q, mode):
    S, V, sh = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    w = ctypes.c_size_t()
    assert _lib.lib().heat_k3_geometry(n, P, q, mode, ctypes.byref(S), ctypes.byref(V),
                                       ctypes.byref(w), ctypes.byref(sh)) == 0
    return S.value, V.value, w.value, bool(sh.value)


@pytest.mark.parametrize("mode", [0, 1])
def test_k3_geometry_invariants(mode):
    for n in (1, 2, 3, 7, 16, 31, 32, 64, 100, 128, 256, 513, 1024):
        for P in (2, 3, 4, 8, 16, 17, 31, 46, 63, 64, 300):
            for q in (1, 2, 9, 40):
                S, V, warps, shared = k3(n, P, q, mode)
                assert S in (2, 4, 8, 16, 32) and V in (1, 2, 4, 8, 16, 32)
                assert S * V >= n
                assert warps == -(-P // (32 // S))
                if mode == 1 or not shared:
                    assert S == 32  # segments only in the lockstep barrier mode
                if S < 32:
                    assert warps >= 4
                if shared:
                    assert warps <= 16
    assert k3(128, 8, 2, 0)[:3] == (16, 8, 4)  # cfg2: two 16-lane PEs per warp, 4 warps
    assert k3(128, 8, 2, 1)[:3] == (32, 4, 8)  # free-running: one PE per warp


# ---- geometric-law thresholds (runtime.cu geometric_thresholds) -------------
GAMMA = 0x9E3779B97F4A7C15
M64 = (1 << 64) - 1


def _mix(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _unxorshift(y, s):
    x = y
    for _ in range(64 // s + 1):
        x = y ^ (x >> s)
    return x


def _unmix(x):
    z = _unxorshift(x, 31)
    z = _unxorshift((z * pow(0x94D049BB133111EB, -1, 1 << 64)) & M64, 27)
    return _unxorshift((z * pow(0xBF58476D1CE4E5B9, -1, 1 << 64)) & M64, 30)


def thresholds(p, q):
    out = (ctypes.c_uint64 * max(1, q - 1))()
    assert _lib.lib().heat_geometric_thresholds(p, q, out) == 0
    return [out[i] for i in range(q - 1)]


def rule(x, T, bound):
    m, d = x >> 11, 0
    while d < bound and m >= T[d]:
        d += 1
    return d


@pytest.mark.parametrize("p", [0.6, 0.3, 0.05, 0.999, 1e-6, 1.0])
@pytest.mark.parametrize("q", [2, 5, 40])
def test_geometric_thresholds_match_reference_draws(port, p, q):
    """The device rule d = #{T_j <= x >> 11} (capped at the bound) equals the
    reference's floor(log1p(-u)/log1p(-p)) (async_sim.cpp:64-69, through the
    oracle) on random draws and on draws crafted to sit at every threshold
    and one step either side of it."""
    T = thresholds(p, q)
    assert all(a <= b for a, b in zip(T, T[1:]))
    seed = 12345
    got = [rule(_mix((seed + (j + 1) * GAMMA) & M64), T, q - 1) for j in range(3000)]
    assert got == port.delay_stream(2, q, 0, p, seed, 10 ** 6, 3000)
    for t in T:
        if t >= 1 << 53:
            continue
        for m in (t - 1, t, t + 1):
            if not 0 <= m < 1 << 53:
                continue
            for low in (0, 0x7FF):
                x = (m << 11) | low
                s = (_unmix(x) - GAMMA) & M64  # the stream whose first draw is x
                for k in (10 ** 6, 1):
                    assert rule(x, T, min(q - 1, k)) == port.delay_stream(2, q, 0, p, s, k, 1)[0]


def free_geometry(N, n, q=8):
    L = _lib.lib()
    v = [ctypes.c_int(0) for _ in range(5)]
    st = L.heat_free_geometry(N, n, q, *[ctypes.byref(x) for x in v])
    return st, tuple(x.value for x in v)


@pytest.mark.parametrize("N,n,expect", [
    (100, 10, (4, 25, 1, 1, 0)), (1000, 100, (4, 25, 4, 3, 1)), (10000, 1000, (10, 25, 4, 10, 4)),
    (100, 5, (4, 25, 1, 1, 0)), (1000, 50, (5, 10, 4, 5, 1)), (10000, 500, (20, 25, 4, 5, 1)),
    (100, 25, (4, 25, 1, 1, 0)), (1024, 128, (4, 32, 4, 2, 1)), (4096, 32, (4, 8, 8, 16, 1)),
    (256, 2, (2, 1, 8, 16, 1)), (100, 1, (4, 25, 1, 1, 0)), (1000, 250, (10, 25, 4, 1, 1)), (10000, 2500, (25, 25, 4, 4, 4)),
    (10000, 2000, (20, 25, 4, 5, 4)), (10000, 5000, (50, 25, 4, 2, 4))])
def test_k10_free_geometry(N, n, expect):
    """K10 (exec_free.cu): Wp warps per PE of Lc lanes x V points, Wp*Lc*V = n
    exactly with 1 <= Lc <= 32 (Lc = 1: one thread per PE), chosen by the
    measured step-cost estimate; 4 warps per CTA (one per SM sub-partition) up
    to a 16-CTA cluster, then 8; Dirichlet fields of <= 160 points share one
    warp (K10w, Wp reported 0)."""
    st, got = free_geometry(N, n)
    assert st == 0 and got == expect
    V, Lc, W, C, Wp = got
    P = N // n
    if Wp == 0:  # K10w: a Dirichlet field of <= 160 points in one warp, V = 4 or 5
        assert V * Lc == N and V in (4, 5) and 2 <= Lc <= 32 and (W, C) == (1, 1)
        return
    assert V * Lc * Wp == n and 1 <= Lc <= 32 and W % Wp == 0
    assert W * C >= P * Wp and W * (C - 1) < P * Wp


@pytest.mark.parametrize("N,n,q", [(1031 * 2, 1031, 8),   # prime PE width: no lanes split
                                   (1000, 100, 17),       # q beyond the 32-slot ring
                                   (100, 100, 8),         # one PE: the sync path
                                   (129 * 4, 4, 8),       # 129 PEs > 16 x 8 warps
                                   (41 * 32 * 2, 41 * 32, 8)])  # 1312 = 41 x 32: no lanes split
def test_k10_free_geometry_refusals(N, n, q):
    st, got = free_geometry(N, n, q)
    assert st != 0 and got == (0, 0, 0, 0, 0)
