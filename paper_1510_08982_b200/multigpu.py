"""Multi-GPU 1-D slab decomposition of the FTCS field.

One process per GPU (torchrun).  Rank g owns points [g*n, (g+1)*n) of a global
field of G*n points.  Every pass of s <= H steps (H = heat_slab_halo() = 64)
each rank needs the H points beyond each of its ends at the pass's start
step: a nearest-neighbour halo exchange of 2 x H doubles (256 B each way),
not a collective.  Only the true global ends are pinned (Dirichlet on rank 0
and rank G-1); periodic domains wrap rank G-1 <-> rank 0 through the same
exchange.  The result is bit-identical to the single-domain sync_run: inside a
pass the slab's points never depend on anything further than H away.

The exchange uses torch.distributed point-to-point ops (NCCL over NVLink on the
GPU box, gloo in the CPU tests) on the plan's stream.  This module holds the
host logic only; the stepping is the sm_100a kernel behind heat.Plan.
"""
from __future__ import annotations

import math
from typing import Callable, Optional

import torch
import torch.distributed as dist

# tags: which ghost of the RECEIVER the message fills
_TAG_LEFT_GHOST = 0
_TAG_RIGHT_GHOST = 1


def neighbours(rank: int, world: int, periodic: bool):
    """(left, right) neighbour ranks, None at a Dirichlet global end."""
    left = rank - 1 if rank > 0 else (world - 1 if periodic and world > 1 else None)
    right = rank + 1 if rank < world - 1 else (0 if periodic and world > 1 else None)
    return left, right


def halo_exchange(send: torch.Tensor, recv: torch.Tensor, rank: int, world: int, periodic: bool,
                  group=None) -> None:
    """send = [my first H | my last H]; recv <- [left ghost H | right ghost H].

    Posting order is fixed (to-right before to-left; from-left before
    from-right) and tags name the receiver's ghost, so a 2-rank periodic ring
    -- where left and right are the same peer -- pairs correctly under both
    NCCL's in-order matching and gloo's tag matching."""
    H = send.numel() // 2
    left, right = neighbours(rank, world, periodic)
    ops = []
    if right is not None:
        ops.append(dist.P2POp(dist.isend, send[H:], right, group, _TAG_LEFT_GHOST))
    if left is not None:
        ops.append(dist.P2POp(dist.isend, send[:H], left, group, _TAG_RIGHT_GHOST))
    if left is not None:
        ops.append(dist.P2POp(dist.irecv, recv[:H], left, group, _TAG_LEFT_GHOST))
    if right is not None:
        ops.append(dist.P2POp(dist.irecv, recv[H:], right, group, _TAG_RIGHT_GHOST))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()


def pass_schedule(steps: int, halo: int):
    """Pass lengths: full passes of `halo` steps and one remainder."""
    out = []
    while steps > 0:
        s = min(steps, halo)
        out.append(s)
        steps -= s
    return out


class SlabEngine:
    """What a slab runner needs from its stepper (heat.Plan on the GPU)."""

    halo: int

    def halo_pack(self, dst: torch.Tensor) -> None: ...

    def halo_unpack(self, src: torch.Tensor) -> None: ...

    def advance(self, steps: int) -> None: ...


def run_passes(engine: SlabEngine, steps: int, rank: int, world: int, periodic: bool,
               send: torch.Tensor, recv: torch.Tensor, group=None,
               on_pass: Optional[Callable[[int], None]] = None) -> None:
    """Advance a slab by `steps`, exchanging ghosts before every pass."""
    for s in pass_schedule(steps, engine.halo):
        if world > 1:
            engine.halo_pack(send)
            halo_exchange(send, recv, rank, world, periodic, group)
            engine.halo_unpack(recv)
        engine.advance(s)
        if on_pass is not None:
            on_pass(s)


class PlanEngine(SlabEngine):
    """heat.Plan slab bound to torch device tensors for the exchange."""

    def __init__(self, plan, r: float, bc):
        self.plan, self.r, self.bc = plan, r, bc
        self.halo = plan.halo()

    def halo_pack(self, dst: torch.Tensor) -> None:
        self.plan.halo_pack(dst.data_ptr())

    def halo_unpack(self, src: torch.Tensor) -> None:
        self.plan.halo_unpack(src.data_ptr())

    def advance(self, steps: int) -> None:
        self.plan.sync_advance(self.r, self.bc, steps)


def gather_slabs(local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """The final gather: every rank's slab (equal sizes, rank order) -> the
    global field on every rank (all_gather_into_tensor; NCCL over NVLink on
    device tensors, gloo on CPU ones)."""
    out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    return out


def plan_gather(plan, world: int, group=None) -> torch.Tensor:
    """gather_slabs of a plan's owned points, device to device."""
    local = torch.empty(plan.n, dtype=torch.float64, device=f"cuda:{plan.device}")
    plan.download_device(local.data_ptr())
    plan.synchronize()
    return gather_slabs(local, world, group)


def exchange_handles(handle: bytes, rank: int, world: int, periodic: bool, group=None):
    """All-gather the 64-byte IPC handles (setup only) and pick the neighbours'."""
    handles = [None] * world
    dist.all_gather_object(handles, handle, group=group)
    left, right = neighbours(rank, world, periodic)
    return (handles[left] if left is not None else None,
            handles[right] if right is not None else None)


class AsyncSlabSolver:
    """Asynchronous FTCS over G GPUs: each rank runs K5 on its slab; the PE
    boundaries between ranks exchange edge values by P2P stores over NVLink
    into the neighbour's receive rings (heat_plan_xlink_*).  NCCL/gloo only
    ships the IPC handles and the per-run barriers around seeding; GPUs never
    barrier per step.  q = 1 free mode is the exact synchronous scheme.

    `link` is what holds the slab and its rings: the device plan (default), or
    for the CPU tests a stand-in with the same five calls (xlink_setup ->
    handle bytes, xlink_connect, xlink_seed, xlink_advance, synchronize) --
    the host protocol here (handle exchange, drain + barrier before seeding,
    barrier after) is the same for both."""

    def __init__(self, n_local: int, per_pe: int, q: int, bc, device: int, rank: int,
                 world: int, group=None, link=None):
        self.rank, self.world, self.group, self.bc = rank, world, group, bc
        self.periodic = not bc.is_dirichlet()
        if link is None:
            from .heat import Plan
            torch.cuda.set_device(device)
            link = Plan(n_local, device, rank, world)
            stream = torch.cuda.current_stream(device)
            if stream.cuda_stream == 0:
                raise ValueError("AsyncSlabSolver needs a non-default current stream")
            link.set_stream(stream.cuda_stream)
        self.plan = link
        handle = self.plan.xlink_setup(per_pe, q, bc)
        left, right = exchange_handles(handle, rank, world, self.periodic, group)
        self.plan.xlink_connect(left, right)
        dist.barrier(group=group)

    def _drain(self):
        self.plan.synchronize()
        if torch.cuda.is_available():
            torch.cuda.synchronize()

    def prepare(self):
        """Seed a fresh run from the current field (the only collectives of a
        run: two barriers).  No neighbour may still be consuming the previous
        run when seeding rewrites its receive ring and resets its progress
        words: every rank drains its own stream, then all meet, then all seed;
        and no rank may start stepping before every neighbour has seeded."""
        self._drain()
        dist.barrier(group=self.group)
        self.plan.xlink_seed()  # push my step-0 edges into the neighbours' rings
        self._drain()
        dist.barrier(group=self.group)

    def run(self, r: float, steps: int, model=None):
        """The seeded run: ONE persistent K5 launch per rank for all `steps`;
        the ranks couple only through P2P stores into each other's rings."""
        return self.plan.xlink_advance(r, self.bc, steps, model)

    def advance(self, r: float, steps: int, model=None):
        """One fresh run of `steps` steps from the current field."""
        self.prepare()
        return self.run(r, steps, model)

    def gather(self) -> torch.Tensor:
        """The global field (device tensor on every rank)."""
        return plan_gather(self.plan, self.world, self.group)


class SlabSolver:
    """Sync FTCS on a G-way slab decomposition, one rank per GPU."""

    def __init__(self, n_local: int, r: float, bc, device: int, rank: int, world: int,
                 group=None):
        from .heat import Plan
        torch.cuda.set_device(device)
        self.rank, self.world, self.group = rank, world, group
        self.periodic = not bc.is_dirichlet()
        self.plan = Plan(n_local, device, rank, world)
        stream = torch.cuda.current_stream(device)
        if stream.cuda_stream == 0:
            raise ValueError("SlabSolver needs a non-default current stream (torch.cuda.set_stream)")
        self.plan.set_stream(stream.cuda_stream)
        self.engine = PlanEngine(self.plan, r, bc)
        H = self.engine.halo
        self.send = torch.empty(2 * H, dtype=torch.float64, device=f"cuda:{device}")
        self.recv = torch.zeros(2 * H, dtype=torch.float64, device=f"cuda:{device}")

    def advance(self, steps: int) -> None:
        run_passes(self.engine, steps, self.rank, self.world, self.periodic, self.send,
                   self.recv, self.group)

    def gather(self) -> torch.Tensor:
        """The global field (device tensor on every rank)."""
        return plan_gather(self.plan, self.world, self.group)


# ---- ensembles across GPUs -------------------------------
def ensemble_run_sharded(cfg, runs: int, base_seed: int, device: Optional[int] = None,
                         group=None, member_fn: Optional[Callable] = None,
                         keep_terminals: bool = True):
    """ensemble_run (analysis.cpp:51-104) with the members split over the ranks:
    rank g runs members [g*M/G, (g+1)*M/G) (seeds base_seed + j) on its own GPU,
    with no communication while they run. One all_gather_object then assembles
    the norm series (and terminal fields) in member order, and every rank forms
    mean/std in the reference's order: sequential sums over j, population std.
    The result is bit-identical to a single-process ensemble_run of M members.

    member_fn(cfg, count, first_seed) -> EnsembleResult defaults to the GPU
    ensemble (heat.ensemble_run); the CPU tests pass the reference's."""
    from . import heat as H
    if runs == 0:
        raise H.DomainError("ensemble_run: M >= 1 required")
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if device is not None:
        H.set_device(device)
    if member_fn is None:
        def member_fn(c, count, first):
            return H.ensemble_run(c, count, first, keep_terminals=keep_terminals)
    start, end = rank * runs // world, (rank + 1) * runs // world
    # A failing shard (DivergenceError, OOM, ...) must not leave the other
    # ranks blocked in the gather: every rank gathers (ok, payload) and the
    # first error (in rank order) is re-raised on all of them.
    try:
        local = member_fn(cfg, end - start, base_seed + start) if end > start else None
        mine = (True, (start, local.steps if local else None,
                       [list(map(float, s)) for s in local.norm_series] if local else [],
                       [t.values() for t in local.terminal_fields]
                       if (local and keep_terminals) else []))
    except Exception as exc:  # noqa: BLE001 -- re-raised below on every rank
        if world == 1:
            raise
        mine = (False, exc)
    gathered = [mine]
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, mine, group=group)
    for ok, payload in gathered:
        if not ok:
            raise payload
    parts = [payload for _, payload in gathered]
    parts.sort(key=lambda x: x[0])
    steps = next(p[1] for p in parts if p[1] is not None)
    norms = [s for p in parts for s in p[2]]
    terms = [H.TemperatureField(t) for p in parts for t in p[3]]
    S = len(steps)
    mean_series, std_series = [0.0] * S, [0.0] * S
    for s in range(S):  # analysis.cpp:90-101
        mean = 0.0
        for j in range(runs):
            mean += norms[j][s]
        mean /= float(runs)
        var = 0.0
        for j in range(runs):
            d = norms[j][s] - mean
            var += d * d
        mean_series[s] = mean
        std_series[s] = math.sqrt(var / float(runs))
    return H.EnsembleResult(list(steps), norms, terms, mean_series, std_series,
                            [base_seed + j for j in range(runs)])
