"""Host logic of the multi-GPU slab decomposition, on CPU with gloo.

The ranks run paper_1510_08982_b200.multigpu.run_passes / halo_exchange (the
product's exchange code) around a numpy stand-in for the GPU slab stepper, and
the gathered field must be bit-identical to the single-domain oracle sync_run
(SURVEY.md §8e).  world_size 2 and 4, Dirichlet and periodic."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1510_08982_b200 import multigpu as M


def test_neighbours_and_schedule():
    assert M.neighbours(0, 4, False) == (None, 1)
    assert M.neighbours(3, 4, False) == (2, None)
    assert M.neighbours(0, 4, True) == (3, 1)
    assert M.neighbours(1, 2, True) == (0, 0)
    assert M.neighbours(0, 1, True) == (None, None)
    assert M.pass_schedule(70, 32) == [32, 32, 6]
    assert M.pass_schedule(0, 32) == []


class NumpySlab(M.SlabEngine):
    """CPU stand-in for heat.Plan slabs: [ghost H | n | ghost H], same rounding
    sequence as the reference stencil ((r*R + c*S) + r*L), ends of the ghosted
    array held, true global ends pinned."""

    def __init__(self, u_local, r, periodic, c1, c2, rank, world, H=32):
        self.halo = H
        self.n = u_local.size
        self.ext = np.zeros(self.n + 2 * H)
        self.ext[H:H + self.n] = u_local
        self.r, self.c = r, 1.0 - 2.0 * r
        self.pin_lo = H if (not periodic and rank == 0) else None
        self.pin_hi = H + self.n - 1 if (not periodic and rank == world - 1) else None
        self.c1, self.c2 = c1, c2

    def halo_pack(self, dst):
        H = self.halo
        dst[:H] = torch.from_numpy(self.ext[H:2 * H].copy())
        dst[H:] = torch.from_numpy(self.ext[self.n:self.n + H].copy())

    def halo_unpack(self, src):
        H = self.halo
        s = src.numpy()
        self.ext[:H] = s[:H]
        self.ext[H + self.n:] = s[H:]

    def advance(self, steps):
        u = self.ext
        for _ in range(steps):
            nxt = u.copy()
            nxt[1:-1] = (self.r * u[2:] + self.c * u[1:-1]) + self.r * u[:-2]
            if self.pin_lo is not None:
                nxt[self.pin_lo] = self.c1
            if self.pin_hi is not None:
                nxt[self.pin_hi] = self.c2
            u = nxt
        self.ext = u

    def owned(self):
        return self.ext[self.halo:self.halo + self.n].copy()


def _worker(rank, world, port, u0, r, periodic, c1, c2, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = u0.size // world
        eng = NumpySlab(u0[rank * n:(rank + 1) * n], r, periodic, c1, c2, rank, world)
        send = torch.zeros(2 * eng.halo, dtype=torch.float64)
        recv = torch.zeros(2 * eng.halo, dtype=torch.float64)
        M.run_passes(eng, steps, rank, world, periodic, send, recv)
        # the product's final gather (multigpu.gather_slabs)
        full = M.gather_slabs(torch.from_numpy(eng.owned()), world)
        if rank == 0:
            q.put(full.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("periodic", [False, True])
def test_slab_decomposition_bit_exact(port, world, periodic):
    from helpers import SplitMix64, bits_equal, random_field
    n_total = 96 * world + (0 if world == 2 else 64)
    gen = SplitMix64(1000 + world + 10 * periodic)
    u0 = random_field(gen, n_total)
    r = 0.4
    c1, c2 = (0.0, 0.0) if periodic else (float(u0[0]), float(u0[-1]))
    steps = 75  # two full 32-step passes and a remainder
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_worker, args=(world, _free_port(), u0, r, periodic, c1, c2, steps, q),
                       nprocs=world, join=True, start_method="spawn")
    got = q.get(timeout=60)
    exp = port.sync_run(u0, r, 1 if periodic else 0, c1, c2, steps)
    assert bits_equal(got, exp)


# ---- ensembles across ranks (multigpu.ensemble_run_sharded) -----------------
def _ref_members(cfg, count, first_seed):
    """The reference's own ensemble_run for one rank's members (CPU stand-in
    for the GPU ensemble the product runs on each rank's device)."""
    from oracle import oracle as O
    from paper_1510_08982_b200 import heat as H
    m = cfg.model
    steps, norms, terms, mean, std, _ = O.ref().ensemble_run(
        cfg.u0.values(), cfg.params.r(), cfg.bc.kind, cfg.bc.c1, cfg.bc.c2, cfg.part.per_pe(),
        int(m.distribution), m.q, m.fixed_delay, cfg.k_end, cfg.stride, count, first_seed)
    return H.EnsembleResult(steps, [list(r) for r in norms], [H.TemperatureField(t) for t in terms],
                            list(mean), list(std), [first_seed + j for j in range(count)])


def _ens_worker(rank, world, port, runs, base_seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_08982_b200 import heat as H
        cfg = H.EnsembleConfig(H.cosine_init(100), H.SolverParams.from_r(0.45),
                               H.BoundaryCondition.dirichlet(1.0, 0.0), H.PartitionSpec(100, 1),
                               H.DelayModel.uniform(4, 0), k_end=500, stride=50)
        res = M.ensemble_run_sharded(cfg, runs, base_seed, member_fn=_ref_members)
        if rank == 0:
            q.put((res.steps, res.norm_series, res.mean_series, res.std_series,
                   [t.values() for t in res.terminal_fields], res.seeds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ensemble_sharded_bit_exact(world):
    from oracle import oracle as O
    if not O.Ref.available():
        pytest.skip("reference library not built here")
    runs, base = 7, 1000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_ens_worker, args=(world, _free_port(), runs, base, q), nprocs=world,
                       join=True, start_method="spawn")
    steps, norms, mean, std, terms, seeds = q.get(timeout=120)
    port_ = O.port()
    u0 = port_.cosine_init(100)
    e_steps, e_norms, e_terms, e_mean, e_std, _ = O.ref().ensemble_run(
        u0, 0.45, 0, 1.0, 0.0, 1, 0, 4, 0, 500, 50, runs, base)
    assert steps == e_steps and seeds == [base + j for j in range(runs)]
    assert np.array_equal(np.array(norms).view(np.uint64), e_norms.view(np.uint64))
    assert np.array_equal(np.array(mean).view(np.uint64), np.asarray(e_mean).view(np.uint64))
    assert np.array_equal(np.array(std).view(np.uint64), np.asarray(e_std).view(np.uint64))
    assert np.array_equal(np.array(terms).view(np.uint64), e_terms.view(np.uint64))


def _failing_members(cfg, count, first_seed):
    from paper_1510_08982_b200 import heat as H
    if first_seed != 1000:  # every rank but 0 fails, as a diverging shard would
        raise H.DivergenceError(f"shard at seed {first_seed} diverged")
    return _ref_members(cfg, count, first_seed)


def _ens_fail_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1510_08982_b200 import heat as H
        cfg = H.EnsembleConfig(H.cosine_init(100), H.SolverParams.from_r(0.45),
                               H.BoundaryCondition.dirichlet(1.0, 0.0), H.PartitionSpec(100, 1),
                               H.DelayModel.uniform(4, 0), k_end=50, stride=10)
        try:
            M.ensemble_run_sharded(cfg, 6, 1000, member_fn=_failing_members)
            q.put((rank, None))
        except Exception as exc:  # noqa: BLE001
            q.put((rank, f"{type(exc).__name__}: {exc}"))
    finally:
        dist.destroy_process_group()


def test_ensemble_sharded_error_reaches_every_rank():
    """one failing shard must not hang the others in the gather;
    every rank re-raises the first failing rank's error."""
    from oracle import oracle as O
    if not O.Ref.available():
        pytest.skip("reference library not built here")
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_ens_fail_worker, args=(world, _free_port(), q), nprocs=world, join=True,
                       start_method="spawn")
    got = sorted(q.get(timeout=60) for _ in range(world))
    assert [r for r, _ in got] == [0, 1, 2]
    for _, err in got:
        assert err == "DivergenceError: shard at seed 1002 diverged", err
