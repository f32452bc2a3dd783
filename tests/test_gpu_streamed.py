"""Streamed sync_run (csrc/sync_host.cu: sync_run_streamed): large Dirichlet
runs that only ask for the final state upload, advance and download the field
chunk by chunk, each pass on ranges shifted by 32 points.  It must be
bit-identical to the one-shot K1 path (HEAT_NO_STREAMED_SYNC=1, itself pinned
to the oracle in test_gpu_sync.py) and to the oracle's light cone at points
around every chunk boundary, and raise the reference's errors."""
import os

import numpy as np
import pytest

from helpers import bits_equal

pytestmark = pytest.mark.gpu

N = (1 << 24) + 12345  # not a multiple of the chunk, tile or 32-point chunk


@pytest.fixture(scope="module")
def H(gpu):
    from paper_1510_08982_b200 import heat
    return heat


def _field(seed, c1, c2):
    rng = np.random.default_rng(seed)
    u = rng.uniform(-1.0, 1.0, N)
    u[0], u[-1] = c1, c2
    return u


def _oneshot(H, u, r, bc, k):
    os.environ["HEAT_NO_STREAMED_SYNC"] = "1"
    try:
        return H.sync_final(u, H.SolverParams.from_r(r), bc, k)
    finally:
        del os.environ["HEAT_NO_STREAMED_SYNC"]


@pytest.mark.parametrize("k", [1, 31, 32, 33, 100, 1000, 10000])
def test_streamed_matches_one_shot(H, k):
    bc = H.BoundaryCondition.dirichlet(0.75, -0.25)
    u = _field(k, 0.75, -0.25)
    got = H.sync_final(u, H.SolverParams.from_r(0.4), bc, k)
    assert bits_equal(got, _oneshot(H, u, 0.4, bc, k))


def test_streamed_lightcone_at_chunk_boundaries(H, port):
    # 16 chunks of cp points; check points straddling every chunk start and
    # the shifted range edges of the first and last pass
    k = 1000
    bc = H.BoundaryCondition.dirichlet(0.5, 0.0)
    u = _field(7, 0.5, 0.0)
    got = H.sync_final(u, H.SolverParams.from_r(0.25), bc, k)
    cp = ((N + 15) // 16 + 31) // 32 * 32
    centres = {0, 1, 2, N - 3, N - 2, N - 1}
    for c in range(1, 16):
        for d in (-1024, -33, -32, -1, 0, 1, 31, 32, 960):
            centres.add(c * cp + d)
    prepared = u.copy()
    for i in sorted(centres):
        assert port.sync_lightcone(prepared, 0.25, 0, 0.5, 0.0, k, i) == got[i], i


def test_streamed_snaps_near_equal_ends(H):
    # ends within 1e-9 of the BC values are snapped exactly (sync_solver.cpp:25-37)
    bc = H.BoundaryCondition.dirichlet(1.0, 2.0)
    u = _field(3, 1.0 + 5e-10, 2.0 - 5e-10)
    got = H.sync_final(u, H.SolverParams.from_r(0.3), bc, 40)
    assert got[0] == 1.0 and got[-1] == 2.0
    assert bits_equal(got, _oneshot(H, u, 0.3, bc, 40))


def test_streamed_errors(H):
    bc = H.BoundaryCondition.dirichlet(0.0, 0.0)
    u = _field(5, 0.0, 0.0)
    u[N // 2 + 17] = np.nan  # inside a late chunk
    with pytest.raises(H.DomainError):
        H.sync_final(u, H.SolverParams.from_r(0.4), bc, 64)
    u = _field(5, 0.0, 0.0)
    u[0] = 1e-3  # end check fails -> the one-shot path reports it
    with pytest.raises(H.InvalidArgument):
        H.sync_final(u, H.SolverParams.from_r(0.4), bc, 64)
    # a good run afterwards is unaffected by the failed ones
    u = _field(6, 0.0, 0.0)
    assert bits_equal(H.sync_final(u, H.SolverParams.from_r(0.4), bc, 64),
                      _oneshot(H, u, 0.4, bc, 64))


def test_streamed_many_passes_pageable_and_pinned(H, port):
    # cfg3's pass count (10^4 steps: 157 passes of 64) on a 2^25-point field,
    # once from ordinary numpy buffers (the pinned staging ring) and once
    # from pinned ones: the same bits, and the oracle's light cone around
    # the field ends and a few interior points
    import torch
    n = (1 << 25) + 77
    k = 10000
    rng = np.random.default_rng(21)
    u = rng.uniform(-1.0, 1.0, n)
    u[0], u[-1] = 0.0, 0.0
    bc = H.BoundaryCondition.dirichlet(0.0, 0.0)
    p = H.SolverParams.from_r(0.4)
    got = H.sync_final(u, p, bc, k)
    pin_in = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    pin_out = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    pin_in[:] = u
    from paper_1510_08982_b200 import _lib
    _lib.check(_lib.lib().heat_sync_run(_lib.dptr(pin_in), n, 0.4, 0, 0.0, 0.0, k, k,
                                        _lib.dptr(pin_out), None, None, 0, None), "sync_run")
    assert bits_equal(got, pin_out)
    for i in (0, 1, 5, n // 3, n // 2 + 1, n - 6, n - 2, n - 1):
        assert port.sync_lightcone(u, 0.4, 0, 0.0, 0.0, k, i) == got[i], i


def test_streamed_graded_chunks_large(H):
    # >= 128 waves: graded head / middle / tail chunks (the bench's 2^30 plan)
    n = (1 << 28) + 4321
    rng = np.random.default_rng(11)
    u = rng.uniform(0.0, 1.0, n)
    u[0], u[-1] = 0.25, 0.5
    bc = H.BoundaryCondition.dirichlet(0.25, 0.5)
    got = H.sync_final(u, H.SolverParams.from_r(0.45), bc, 70)
    assert bits_equal(got, _oneshot(H, u, 0.45, bc, 70))
