"""Device-boundary exchange of K5 on ONE GPU ("virtual devices").

HEAT_VIRTUAL_DEVICES=G splits a run into G device groups: PE boundaries between
groups go through exactly the multi-GPU path -- the reader's receive ring
filled by the neighbour's system-scope (P2P) stores and released/acquired at
.sys scope -- while everything stays in one kernel on one device (the
recommended emulation: ranks that wait on each other must not be separate
launches on one GPU).  Results must stay bit-exact with the reference."""
import os

import numpy as np
import pytest

from helpers import SplitMix64, bits_equal, random_field

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H(gpu):
    from paper_1510_08982_b200 import heat
    return heat


@pytest.fixture
def vdev():
    def set_groups(g):
        os.environ["HEAT_VIRTUAL_DEVICES"] = str(g)
    yield set_groups
    os.environ.pop("HEAT_VIRTUAL_DEVICES", None)


@pytest.mark.parametrize("groups", [2, 4])
@pytest.mark.parametrize("bc,law", [(0, 0), (1, 0), (0, 2), (1, 1)])
def test_virtual_devices_deterministic_bit_exact(H, port, vdev, groups, bc, law):
    vdev(groups)
    n_total, per_pe, q = 16384, 2048, 4
    gen = SplitMix64(groups * 10 + bc * 3 + law)
    u0 = random_field(gen, n_total)
    b = H.BoundaryCondition.periodic() if bc else H.BoundaryCondition.dirichlet(u0[0], u0[-1])
    p = H.SolverParams.from_r(0.4)
    fd = 2 if law == 1 else 0
    model = H.DelayModel(q, H.Distribution(law), fd, 0.6, 77)
    got = H.async_final(u0, p, b, H.PartitionSpec(n_total, per_pe), model, 150)
    exp = port.async_run(u0, p.r(), b.kind, b.c1, b.c2, per_pe, law, q, fd, 0.6, 77, 150)
    assert bits_equal(got, exp)


@pytest.mark.parametrize("groups", [2, 8])
def test_virtual_devices_exact_sync(H, port, vdev, groups):
    # free-running with q = 1 across device boundaries == the synchronous trajectory
    vdev(groups)
    n = 1 << 18
    gen = SplitMix64(groups)
    u0 = random_field(gen, n)
    u0[0] = u0[-1] = 0.0
    plan = H.Plan(n)
    plan.upload(u0)
    st = plan.async_advance(0.4, H.BoundaryCondition.dirichlet(0, 0), 1 << 13, 1, 170)
    assert bits_equal(plan.download(), port.sync_run(u0, 0.4, 0, 0.0, 0.0, 170))
    assert st.max_delay == 0


def test_virtual_devices_free_bounded(H, port, vdev):
    vdev(4)
    n = 1 << 18
    u0 = port.prepare_initial(port.sine_init(n), 1, 0.0, 0.0)
    plan = H.Plan(n)
    plan.upload(u0)
    st = plan.async_advance(0.3, H.BoundaryCondition.periodic(), 1 << 14, 3, 400)
    got = plan.download()
    assert st.max_delay <= 2 and st.reads > 0
    exp = port.sync_run(u0, 0.3, 1, 0.0, 0.0, 400)
    assert np.max(np.abs(got - exp)) < 1e-3
    assert abs(np.sum(got) - np.sum(u0)) < 1e-9 * n  # periodic: heat is conserved
