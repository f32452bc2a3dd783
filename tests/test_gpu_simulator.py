"""AsyncSimulator on the GPU (heat_async_sim_*, csrc/async_host.cu) against the
oracle's async_run: stepping in uneven slices must reproduce async_run(k)
bit-exactly after every slice -- K3 PEs (<= 1024 points) and K5 PEs (wider),
all three delay laws, both boundary conditions -- and the constructor must
raise the reference's errors in the reference's order (async_sim.cpp:122-134:
prepare_initial, then the partition check; HistoryRing rejects q = 0)."""
import numpy as np
import pytest

from helpers import SplitMix64, bits_equal, random_field

pytestmark = pytest.mark.gpu

SLICES = [1, 7, 30, 1, 50, 11]  # 100 steps


@pytest.fixture(scope="module")
def H(gpu):
    from paper_1510_08982_b200 import heat
    return heat


@pytest.mark.parametrize("N,n", [(1024, 128), (300, 1), (3 * 4096, 4096)])
@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("law,q,d,p", [(0, 3, 0, 0.5), (1, 4, 2, 0.5), (2, 4, 0, 0.6)])
def test_simulator_slices_match_async_run(H, port, N, n, periodic, law, q, d, p):
    gen = SplitMix64(N + 17 * law + periodic)
    u0 = random_field(gen, N)
    c1, c2 = (0.0, 0.0) if periodic else (float(u0[0]), float(u0[-1]))
    bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(c1, c2)
    seed = 4242 + N
    model = H.DelayModel(q, H.Distribution(law), d, p, seed)
    sim = H.AsyncSimulator(H.TemperatureField(u0), H.SolverParams.from_r(0.35), bc,
                           H.PartitionSpec(N, n), model)
    assert sim.step_index() == 0
    k = 0
    for s in SLICES:
        sim.step(s)
        k += s
        assert sim.step_index() == k
        want = port.async_run(u0, 0.35, 1 if periodic else 0, c1, c2, n, law, q, d, p, seed,
                              k_end=k)
        assert bits_equal(sim.current(), want), (k, s)
    sim.close()


def test_simulator_single_pe_is_sync(H, port):
    gen = SplitMix64(5)
    u0 = random_field(gen, 2000)
    bc = H.BoundaryCondition.dirichlet(float(u0[0]), float(u0[-1]))
    sim = H.AsyncSimulator(H.TemperatureField(u0), H.SolverParams.from_r(0.4), bc,
                           H.PartitionSpec(2000, 2000), H.DelayModel.uniform(3, 1))
    sim.step(40)
    sim.step(25)
    assert bits_equal(sim.current(), port.sync_run(u0, 0.4, 0, u0[0], u0[-1], 65))


def test_simulator_errors(H):
    u0 = H.cosine_init(100)
    p = H.SolverParams.from_r(0.4)
    bc = H.BoundaryCondition.dirichlet(1.0, 0.0)  # cosine_init(100) ends at 1, -1
    with pytest.raises(H.InvalidArgument):  # prepare_initial first ...
        H.AsyncSimulator(u0, p, bc, H.PartitionSpec(120, 10), H.DelayModel.uniform(2, 1))
    bc = H.BoundaryCondition.periodic()
    with pytest.raises(H.InvalidArgument):  # ... then the partition
        H.AsyncSimulator(u0, p, bc, H.PartitionSpec(120, 10), H.DelayModel.uniform(2, 1))
    with pytest.raises(H.DomainError):  # HistoryRing: depth >= 1
        H.AsyncSimulator(u0, p, bc, H.PartitionSpec(100, 10), H.DelayModel(0, H.Distribution(0),
                                                                           0, 0.5, 1))
