"""K5 tile geometries (csrc/stream_host.cu: stream_geometry): 48-point lanes
with a 64-point halo (64 steps per pass), 48x32, and 32x32 -- each chosen
automatically from the PE width -- all bit-exact with the oracle's async_run
in deterministic mode (the PE-boundary cut sits mid-lane in the first two).

    n = 32768: 32768 mod 1408 = 384 >= 64            -> 48x64
    n = 4256:  4256 mod 1408 = 32 < 64, mod 1472 = 1312 -> 48x32
    n = 1056:  a PE of <= 1472 points                 -> 32x32
"""
import numpy as np
import pytest

from helpers import bits_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H(gpu):
    from paper_1510_08982_b200 import heat
    return heat


@pytest.mark.parametrize("n", [32768, 4256, 1056])
@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("law,q,d", [(0, 3, 0), (1, 4, 2)])
def test_stream_geometries_bit_exact(H, port, n, periodic, law, q, d):
    P = 3
    N = P * n
    rng = np.random.default_rng(n + 7 * law + periodic)
    u0 = rng.uniform(-1.0, 1.0, N)
    c1, c2 = (0.0, 0.0) if periodic else (0.25, -0.5)
    if not periodic:
        u0[0], u0[-1] = c1, c2
    bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(c1, c2)
    k = 150  # two full passes of 64 and a partial one (or 4 of 32 and a partial one)
    model = H.DelayModel(q, H.Distribution(law), d, 0.5, 1234 + n)
    got = H.async_final(u0, H.SolverParams.from_r(0.4), bc, H.PartitionSpec(N, n), model, k)
    want = port.async_run(u0, 0.4, 1 if periodic else 0, c1, c2, n, law, q, d, 0.5, 1234 + n,
                          k_end=k)
    assert bits_equal(got, want)
