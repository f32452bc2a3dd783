"""K7c (sync_small.cu: sync_run of N = 8m <= 8192 over a thread-block cluster,
double-buffered field copies written with st.async, trajectory rows from the
exact lanes' registers, zero-copy I/O) against the oracle, bit for bit.

Shapes cover one warp (N <= 128, one CTA), the 2-CTA cfg1 cluster (N = 1000,
1024), partial last windows (N = 8 mod 128), 8-CTA clusters (4096, 8192),
both boundary conditions, strides that cut 64-step rounds (1, 7, 100) or
not (64), k = 0, 1, a round edge and beyond; the one-CTA variant
(HEAT_K7_NO_CLUSTER=1) and the round-1 K7 (HEAT_NO_K7C=1) in subprocesses."""
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import SplitMix64, bits_equal, random_field

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def H(gpu):
    from paper_1510_08982_b200 import heat
    return heat


def _check(H, port, n, periodic, k_end, stride, seed):
    gen = SplitMix64(seed)
    u0 = random_field(gen, n)
    r = 0.05 + 0.44 * gen.next_double()
    bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    p = H.SolverParams.from_r(r)
    t = H.sync_run(H.TemperatureField(u0), p, bc, k_end, stride)
    steps, snaps = port.sync_run(u0, p.r(), bc.kind, bc.c1, bc.c2, k_end, stride, record=True)
    assert t.steps == steps, (n, periodic, k_end, stride)
    for j, s in enumerate(t.snapshots):
        assert bits_equal(s.values(), snaps[j]), (n, periodic, k_end, stride, j)


@pytest.mark.parametrize("n", [8, 64, 128, 136, 520, 1000, 1024, 1032, 1544, 2048, 4096, 4104, 8192])
@pytest.mark.parametrize("periodic", [False, True])
def test_k7c_trajectories(H, port, n, periodic):
    for i, (k, stride) in enumerate([(0, 1), (1, 1), (64, 7), (130, 64), (333, 100), (200, 1)]):
        _check(H, port, n, periodic, k, stride, 1000 * n + 10 * i + periodic)


@pytest.mark.parametrize("n", [256, 1024, 8192])
def test_k7c_final_only_long(H, port, n):
    gen = SplitMix64(n)
    u0 = random_field(gen, n)
    p = H.SolverParams.from_r(0.45)
    bc = H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    got = H.sync_final(u0, p, bc, 2500)
    assert bits_equal(got, port.sync_run(u0, p.r(), bc.kind, bc.c1, bc.c2, 2500))


def test_k7c_rejects_nonfinite_and_bad_ends(H):
    u = np.sin(np.linspace(0, np.pi, 1024))
    u[-1] = 0.0
    bad = u.copy()
    bad[500] = np.nan
    p = H.SolverParams.from_r(0.25)
    bc = H.BoundaryCondition.dirichlet(0.0, 0.0)
    with pytest.raises(ValueError):
        H.sync_final(bad, p, bc, 10)
    off = u.copy()
    off[0] = 0.5
    with pytest.raises(ValueError):
        H.sync_final(off, p, bc, 10)
    # a good call right after the failures still works (no leaked flags)
    assert np.all(np.isfinite(H.sync_final(u, p, bc, 10)))


@pytest.mark.parametrize("env", ["HEAT_K7_NO_CLUSTER", "HEAT_NO_K7C"])
def test_variants_agree(env):
    code = (
        "import numpy as np, sys\n"
        "from paper_1510_08982_b200 import heat as H\n"
        "from oracle import oracle as O\n"
        "from helpers import SplitMix64, random_field, bits_equal\n"
        "port = O.port()\n"
        "for n in (1024, 4096):\n"
        "    u0 = random_field(SplitMix64(n), n)\n"
        "    p = H.SolverParams.from_r(0.3)\n"
        "    bc = H.BoundaryCondition.dirichlet(u0[0], u0[-1])\n"
        "    t = H.sync_run(H.TemperatureField(u0), p, bc, 300, 100)\n"
        "    st, sn = port.sync_run(u0, p.r(), 0, u0[0], u0[-1], 300, 100, record=True)\n"
        "    assert t.steps == st\n"
        "    assert all(bits_equal(s.values(), sn[j]) for j, s in enumerate(t.snapshots))\n"
        "print('ok')\n")
    env_ = dict(os.environ, **{env: "1"})
    env_["PYTHONPATH"] = os.pathsep.join([ROOT, os.path.join(ROOT, "tests"), env_.get("PYTHONPATH", "")])
    out = subprocess.run([sys.executable, "-c", code], env=env_, cwd=ROOT, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_k7c_and_k9_device_staging_fallback(H, port):
    # a trajectory larger than the pinned staging buffer (64 MB: 9001 rows of
    # 8 KB) takes the device-buffer path with copies instead of zero-copy
    n, k = 1024, 9000
    gen = SplitMix64(4242)
    u0 = random_field(gen, n)
    bc = H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    p = H.SolverParams.from_r(0.35)
    t = H.sync_run(H.TemperatureField(u0), p, bc, k, 1)
    steps, snaps = port.sync_run(u0, p.r(), bc.kind, bc.c1, bc.c2, k, 1, record=True)
    assert t.steps == steps
    for j in (0, 1, 63, 64, 65, 4500, k):
        assert bits_equal(t.snapshots[j].values(), snaps[j]), j
    m = H.DelayModel.uniform(3, 9)
    ta = H.async_run(H.TemperatureField(u0), p, bc, H.PartitionSpec(n, 128), m, k, 1)
    st, sn = port.async_run(u0, p.r(), bc.kind, bc.c1, bc.c2, 128, 0, 3, seed=9, k_end=k,
                            stride=1, record=True)
    assert ta.steps == st
    for j in (0, 1, 63, 64, 65, 4500, k):
        assert bits_equal(ta.snapshots[j].values(), sn[j]), j
