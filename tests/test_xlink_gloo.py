"""Host logic of the P2P multi-GPU path (multigpu.AsyncSlabSolver over
heat_plan_xlink_*), on CPU with gloo, world size 2 and 3.

AsyncSlabSolver is the product's host protocol: the IPC handles are
all-gathered once and each rank opens its two neighbours' (periodic with two
ranks: the same rank on both sides); before every run each rank drains its
own stream, all meet, every rank seeds its step-0 edges into its neighbours'
receive rings, all meet again, and only then does any rank step.  Here the
device plan is replaced by ShmLink, a CPU stand-in that keeps the two receive
rings in POSIX shared memory (the "IPC handle" is the segment name) and
steps its slab with K5's boundary protocol (async_stream.cuh): before step k
it waits until the neighbour's progress word shows a value of step
>= k - (q - 1), takes the newest one of step <= k from ring slot step % R
(R = the power of two >= 2q + 2), and after the step it stores its new edge value into the
neighbour's ring, then the progress word (x86 keeps the two stores in order).
Random sleeps make the ranks drift.

* q = 1 is the exact synchronous scheme: two consecutive runs (the second
  reseeded from the first's result) gather to the single-domain oracle's
  sync_run, bit for bit, Dirichlet and periodic;
* q = 4 free-running: every consumed value is at most 3 steps old, the
  field stays inside the initial envelope (maximum principle).
"""
import os
import random
import socket
import time

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from multiprocessing import shared_memory

from paper_1510_08982_b200 import multigpu as M


class _Stats:
    def __init__(self):
        self.max_delay = 0
        self.reads = 0


class ShmLink:
    """CPU stand-in for a slab plan with xlink receive rings (see module doc)."""

    def __init__(self, u_local, r_unused, periodic, c1, c2, rank, world, seed):
        self.u = np.array(u_local, dtype=np.float64)
        self.periodic, self.c1, self.c2 = periodic, c1, c2
        self.rank, self.world = rank, world
        self.rng = random.Random(seed)
        self.left = self.right = None
        self._open = []

    # -- the five calls AsyncSlabSolver makes ---------------------------------
    def xlink_setup(self, per_pe, q, bc):
        self.q = q
        self.R = 1
        while self.R < 2 * q + 2:
            self.R *= 2
        self.shm = shared_memory.SharedMemory(create=True, size=2 * self.R * 8 + 2 * 8)
        self.rings, self.prog = self._views(self.shm)
        self.rings[:] = 0.0
        self.prog[:] = -1  # nothing published yet
        return self.shm.name.encode().ljust(64, b"\0")

    def xlink_connect(self, left, right):
        def open_(h):
            if h is None:
                return None
            seg = shared_memory.SharedMemory(name=h.rstrip(b"\0").decode())
            self._open.append(seg)
            return self._views(seg)
        self.left, self.right = open_(left), open_(right)

    def xlink_seed(self):
        # my step-0 edges into the neighbours' rings: the left neighbour's
        # side-1 ring holds my first point, the right one's side-0 my last
        if self.left is not None:
            rings, prog = self.left
            rings[1, 0] = self.u[0]
            prog[1] = 0
        if self.right is not None:
            rings, prog = self.right
            rings[0, 0] = self.u[-1]
            prog[0] = 0

    def xlink_advance(self, r, bc, steps, model=None):
        assert model is None  # free mode (q = 1: exact)
        st = _Stats()
        c = 1.0 - 2.0 * r
        R, q = self.R, self.q
        for k in range(steps):
            ghosts = []
            for side, nb in ((0, self.left), (1, self.right)):
                if nb is None:
                    ghosts.append(None)
                    continue
                need = k - (q - 1)
                t0 = time.monotonic()
                while int(self.prog[side]) < need:  # spin on the progress word
                    if time.monotonic() - t0 > 30:
                        raise TimeoutError(f"rank {self.rank}: no value >= step {need} on side {side}")
                    time.sleep(0)
                # the newest value not from the future (the neighbour may
                # already be one step ahead)
                m = min(int(self.prog[side]), k)
                v = float(self.rings[side, m % R])
                st.max_delay = max(st.max_delay, k - m)
                st.reads += 1
                ghosts.append(v)
            u = self.u
            ext = np.empty(u.size + 2)
            ext[1:-1] = u
            ext[0] = ghosts[0] if ghosts[0] is not None else 0.0
            ext[-1] = ghosts[1] if ghosts[1] is not None else 0.0
            nxt = (r * ext[2:] + c * ext[1:-1]) + r * ext[:-2]
            if not self.periodic and self.rank == 0:
                nxt[0] = self.c1
            if not self.periodic and self.rank == self.world - 1:
                nxt[-1] = self.c2
            self.u = nxt
            if self.rng.random() < 0.05:
                time.sleep(self.rng.random() * 2e-4)  # drift
            slot = (k + 1) % R
            if self.left is not None:  # value first, then the progress word
                rings, prog = self.left
                rings[1, slot] = nxt[0]
                prog[1] = k + 1
            if self.right is not None:
                rings, prog = self.right
                rings[0, slot] = nxt[-1]
                prog[0] = k + 1
        return st

    def synchronize(self):
        pass

    # -- helpers ---------------------------------------------------------------
    def _views(self, seg):
        R = self.R
        rings = np.ndarray((2, R), dtype=np.float64, buffer=seg.buf)
        prog = np.ndarray((2,), dtype=np.int64, buffer=seg.buf, offset=2 * R * 8)
        return rings, prog

    def close(self):
        for seg in self._open:
            seg.close()
        self.shm.close()
        self.shm.unlink()


def _worker(rank, world, port, u0, r, periodic, c1, c2, steps, q, runs, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_08982_b200 import heat as H
        n = u0.size // world
        link = ShmLink(u0[rank * n:(rank + 1) * n], r, periodic, c1, c2, rank, world, 77 + rank)
        bc = H.BoundaryCondition.periodic() if periodic else H.BoundaryCondition.dirichlet(c1, c2)
        solver = M.AsyncSlabSolver(n, n, q, bc, 0, rank, world, link=link)
        delay = 0
        for _ in range(runs):  # each run reseeds from the previous one's field
            st = solver.advance(r, steps)
            delay = max(delay, st.max_delay)
        full = M.gather_slabs(torch.from_numpy(link.u), world)
        d = torch.tensor([delay], dtype=torch.int64)
        dist.all_reduce(d, op=dist.ReduceOp.MAX)
        dist.barrier()
        link.close()
        if rank == 0:
            out.put((full.numpy(), int(d.item())))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, periodic, q, steps, runs, seed):
    from helpers import SplitMix64, random_field
    gen = SplitMix64(seed)
    u0 = random_field(gen, 40 * world)
    r = 0.3
    c1, c2 = (0.0, 0.0) if periodic else (float(u0[0]), float(u0[-1]))
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), u0, r, periodic, c1, c2, steps, q, runs,
                                      out), nprocs=world, join=True, start_method="spawn")
    got, delay = out.get(timeout=120)
    return u0, r, c1, c2, got, delay


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("periodic", [False, True])
def test_xlink_protocol_q1_is_sync(port, world, periodic):
    from helpers import bits_equal
    steps, runs = 60, 2
    u0, r, c1, c2, got, delay = _run(world, periodic, 1, steps, runs, 500 + world + 10 * periodic)
    exp = port.sync_run(u0, r, 1 if periodic else 0, c1, c2, steps * runs)
    assert delay == 0
    bad = np.nonzero(got != exp)[0]
    assert bits_equal(got, exp), (bad[:10], float(np.max(np.abs(got - exp))))


@pytest.mark.parametrize("world", [2, 3])
def test_xlink_protocol_free_bounded(world):
    q = 4
    u0, r, c1, c2, got, delay = _run(world, False, q, 80, 2, 900 + world)
    assert 0 <= delay <= q - 1
    assert np.all(np.isfinite(got))
    lo, hi = min(u0.min(), c1, c2), max(u0.max(), c1, c2)
    assert got.min() >= lo - 1e-12 and got.max() <= hi + 1e-12
