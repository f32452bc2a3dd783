"""The bench's own configuration (BASELINE cfg3: N = 2^30, r = 0.4,
Dirichlet(0,0), sine IC, 10^4 steps), checked where it runs: the K1 sync run
and the K5 deterministic asynchronous run (512 PEs, uniform q = 2, seed 1) over
the full 10^4 steps, at the ends, the middle, K1 tile boundaries, K5 PE
boundaries and seeded random points -- every point of each light-cone window
that the window's held ends cannot reach, bit for bit against the oracle's
window runs (oracle/lightcone.py; the K loop replaced is sync_solver.cpp:70-75,
the asynchronous one async_sim.cpp:142-160)."""
import numpy as np
import pytest

from oracle import oracle as O
from oracle.lightcone import WindowCheck

pytestmark = pytest.mark.gpu

N = 1 << 30
K = 10_000
PES = 512


@pytest.fixture(scope="module")
def H(gpu):
    from paper_1510_08982_b200 import heat
    return heat


def centres(seed):
    rng = np.random.default_rng(seed)
    pe = N // PES
    c = [1, 2, N // 2, 1408 * 7777, 1408 * 7777 - 1, pe - 1, pe, 255 * pe - 1, 256 * pe,
         N - pe, N - 2]
    return c + [int(x) for x in rng.integers(0, N, 5)]


def test_cfg3_sync_and_async_full_length(H, port):
    bc = H.BoundaryCondition.dirichlet(0.0, 0.0)
    r = H.SolverParams.from_r(0.4).r()
    p = H.Plan(N, 0)
    try:
        p.fill_sine()
        chk = WindowCheck(N, K, centres(1))
        chk.capture(p.download_range)
        p.sync_advance(r, bc, K)
        res = chk.verify(p.download_range,
                         lambda w, lo: port.sync_window(w, lo, N, r, 0.0, 0.0, K))
        assert res["ok"], res["bad"]
        assert res["points"] > 10 * 64

        p.fill_sine()
        chk = WindowCheck(N, K, centres(2))
        chk.capture(p.download_range)
        st = p.async_replay(r, bc, N // PES, H.DelayModel.uniform(2, 1), K)
        assert st.max_delay == 1
        res = chk.verify(p.download_range,
                         lambda w, lo: port.async_window(w, lo, N, r, 0.0, 0.0, N // PES,
                                                         O.UNIFORM, 2, seed=1, k=K))
        assert res["ok"], res["bad"]
    finally:
        p.close()
