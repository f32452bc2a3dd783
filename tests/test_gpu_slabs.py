"""Multi-GPU slab path of K1 (heat_plan_create_slab / halo_pack / halo_unpack,
plan.cu) on ONE GPU: the G slabs of a world-G decomposition run one after
another in this process (no kernel waits on another), their H-point ghosts
moved between passes exactly as multigpu.halo_exchange moves them over NCCL
(send = [first H | last H] -> the neighbours' [left ghost | right ghost]).
The gathered field must be bit-identical to the single-domain oracle; the
slab advances run the default kernel when its halo fits the 64 ghost points
and the 32-point-halo variant otherwise (HEAT_SYNC_VARIANT=4 run)."""
import numpy as np
import pytest

from helpers import bits_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H(gpu):
    from paper_1510_08982_b200 import heat
    return heat


def _neighbours(rank, world, periodic):
    left = rank - 1 if rank > 0 else (world - 1 if periodic else None)
    right = rank + 1 if rank + 1 < world else (0 if periodic else None)
    return left, right


@pytest.mark.parametrize("world,periodic,n_local,k", [(2, False, 5037, 100), (3, False, 4096, 64),
                                                      (2, True, 3000, 97), (4, True, 2080, 33)])
def test_slabs_match_single_domain(H, port, world, periodic, n_local, k):
    import torch
    rng = np.random.default_rng(world * 1000 + n_local)
    N = world * n_local
    u0 = rng.uniform(-1.0, 1.0, N)
    c1, c2 = (0.0, 0.0) if periodic else (0.5, -0.25)
    if not periodic:
        u0[0], u0[-1] = c1, c2
    bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(c1, c2)
    r = 0.37
    Hh = H.Plan.halo()
    plans = []
    for g in range(world):
        p = H.Plan(n_local, 0, g, world)
        p.upload(u0[g * n_local:(g + 1) * n_local])
        plans.append(p)
    send = [torch.zeros(2 * Hh, dtype=torch.float64, device="cuda") for _ in range(world)]
    recv = [torch.zeros(2 * Hh, dtype=torch.float64, device="cuda") for _ in range(world)]
    left_steps = k
    while left_steps > 0:
        s = min(Hh, left_steps)
        for g, p in enumerate(plans):
            p.halo_pack(send[g].data_ptr())
            p.synchronize()
        for g in range(world):
            lft, rgt = _neighbours(g, world, periodic)
            if lft is not None:
                recv[g][:Hh].copy_(send[lft][Hh:])
            if rgt is not None:
                recv[g][Hh:].copy_(send[rgt][:Hh])
        torch.cuda.synchronize()
        for g, p in enumerate(plans):
            p.halo_unpack(recv[g].data_ptr())
            p.sync_advance(r, bc, s)
            p.synchronize()
        left_steps -= s
    got = np.concatenate([p.download() for p in plans])
    want = port.sync_run(u0, r, 1 if periodic else 0, c1, c2, k)
    assert bits_equal(got, want)
    for p in plans:
        p.close()


def test_slab_advance_caps_steps(H):
    p = H.Plan(1024, 0, 0, 2)
    p.upload(np.zeros(1024))
    with pytest.raises(H.InvalidArgument):
        p.sync_advance(0.25, H.BoundaryCondition.dirichlet(0.0, 0.0), H.Plan.halo() + 1)
    p.close()


def test_plan_gather_device_to_device(H):
    # the final gather's device path (heat_plan_download_device + NCCL
    # all_gather_into_tensor) on a one-rank group: the gathered field is the plan's
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_1510_08982_b200 import multigpu as M
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        p = H.Plan(5000, 0)
        u = np.linspace(0.0, 1.0, 5000)
        p.upload(u)
        p.sync_advance(0.3, H.BoundaryCondition.dirichlet(0.0, 1.0), 7)
        got = M.plan_gather(p, 1).cpu().numpy()
        assert bits_equal(got, p.download())
        p.close()
    finally:
        dist.destroy_process_group()
