"""Multi-GPU P2P plumbing (heat_plan_xlink_*) with two processes on ONE GPU.

Checks the parts the single-GPU emulation (test_gpu_xdevice.py) cannot: the
IPC export of each rank's receive rings, the handle exchange through
torch.distributed, opening the neighbours' mappings, and the seed P2P stores
landing in the right ring of the right rank.  No kernel that waits on another
rank runs here (two ranks that spin on each other must not share a GPU); the
in-kernel cross-device exchange itself is covered by the virtual-device tests."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, periodic, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_08982_b200 import heat as H
        from paper_1510_08982_b200 import multigpu as M
        torch.cuda.set_device(0)
        n_local, per_pe = 8192, 2048
        bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(0, 0)
        plan = H.Plan(n_local, 0, rank, world)
        u = np.arange(n_local, dtype=np.float64) + 1000.0 * (rank + 1)
        if not periodic:
            if rank == 0:
                u[0] = 0.0
            if rank == world - 1:
                u[-1] = 0.0
        plan.upload(u)
        plan.synchronize()
        handle = plan.xlink_setup(per_pe, 4, bc)
        left, right = M.exchange_handles(handle, rank, world, periodic)
        plan.xlink_connect(left, right)
        dist.barrier()
        plan.xlink_seed()
        torch.cuda.synchronize()
        dist.barrier()
        got = plan.xlink_debug_recv()  # [left neighbour's last, right neighbour's first]
        out = torch.tensor(got)
        allv = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allv, out)
        if rank == 0:
            torch.save([a.numpy() for a in allv], os.environ["XLINK_OUT"])
        dist.barrier()
        plan.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("periodic,world", [(False, 2), (True, 2), (True, 3)])
def test_xlink_ipc_seed(gpu, tmp_path, periodic, world):
    out = str(tmp_path / "recv.pt")
    os.environ["XLINK_OUT"] = out
    mp.start_processes(_worker, args=(world, _free_port(), periodic, 4), nprocs=world, join=True,
                       start_method="spawn")
    recv = torch.load(out, weights_only=False)
    n = 8192
    first = [1000.0 * (r + 1) for r in range(world)]
    last = [1000.0 * (r + 1) + n - 1 for r in range(world)]
    if not periodic:
        first[0] = 0.0
        last[-1] = 0.0
    for r in range(world):
        lft = (r - 1) % world if (periodic or r > 0) else None
        rgt = (r + 1) % world if (periodic or r < world - 1) else None
        if lft is not None:
            assert recv[r][0] == last[lft], (r, recv[r])
        if rgt is not None:
            assert recv[r][1] == first[rgt], (r, recv[r])
