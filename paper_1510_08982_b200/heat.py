"""Python mirror of the reference's solver API (namespace heat), running on the
B200 through the C-ABI in include/heat_b200.h.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/heat/{core,sync_solver,async_sim,async_exec}.hpp;
the exception classes in ``_lib`` stand in for the C++ exception types
(``DomainError`` ~ std::domain_error, ``InvalidArgument`` ~
std::invalid_argument, ``LogicError`` ~ std::logic_error, ``DivergenceError``).
Every solver call executes the sm_100a kernels; nothing here steps the field
on the CPU.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (DivergenceError, DomainError, InvalidArgument, LogicError,  # noqa: F401
                   NativeUnavailable, WatchdogTimeout)


# ---- core.hpp:11-35 -------------------------------------------------------
def derive_r(alpha: float, dt: float, dx: float) -> float:
    """core.cpp:7-11"""
    if not (alpha > 0.0) or not (dt > 0.0) or not (dx > 0.0):
        raise DomainError("derive_r: alpha, dt, dx must all be positive")
    return alpha * dt / (dx * dx)


class SolverParams:
    """core.hpp:13-35: r = alpha*dt/dx^2, always re-derived."""

    __slots__ = ("_alpha", "_dt", "_dx")

    def __init__(self, alpha: float, dt: float, dx: float, _token=None):
        if _token is not SolverParams._TOKEN:
            raise TypeError("use SolverParams.checked / unchecked / from_r")
        self._alpha, self._dt, self._dx = float(alpha), float(dt), float(dx)

    _TOKEN = object()

    @staticmethod
    def checked(alpha: float, dt: float, dx: float) -> "SolverParams":
        r = derive_r(alpha, dt, dx)
        if not (r > 0.0) or r > 0.5:
            raise DomainError("SolverParams: r = alpha*dt/dx^2 must lie in (0, 0.5]")
        return SolverParams(alpha, dt, dx, SolverParams._TOKEN)

    @staticmethod
    def unchecked(alpha: float, dt: float, dx: float) -> "SolverParams":
        derive_r(alpha, dt, dx)
        return SolverParams(alpha, dt, dx, SolverParams._TOKEN)

    @staticmethod
    def from_r(r: float, allow_unstable: bool = False) -> "SolverParams":
        return (SolverParams.unchecked if allow_unstable else SolverParams.checked)(r, 1.0, 1.0)

    def alpha(self) -> float:
        return self._alpha

    def dt(self) -> float:
        return self._dt

    def dx(self) -> float:
        return self._dx

    def r(self) -> float:
        return self._alpha * self._dt / (self._dx * self._dx)


class TemperatureField:
    """core.hpp:40-64 BasicField<double>: N >= 3, all values finite."""

    __slots__ = ("_v",)

    def __init__(self, values: Sequence[float] | np.ndarray):
        v = np.array(values, dtype=np.float64, copy=True).reshape(-1)
        if v.size < 3:
            raise DomainError("TemperatureField requires N >= 3")
        if not np.all(np.isfinite(v)):
            raise DomainError("TemperatureField values must be finite")
        v.setflags(write=False)
        self._v = v

    @classmethod
    def _adopt(cls, v: np.ndarray) -> "TemperatureField":
        """Wrap a read-only float64 row the library produced (its finiteness was
        checked on the device: a non-finite result raises before we get here)."""
        f = cls.__new__(cls)
        f._v = v
        return f

    def size(self) -> int:
        return int(self._v.size)

    def __len__(self) -> int:
        return int(self._v.size)

    def __getitem__(self, i):
        return self._v[i]

    def values(self) -> np.ndarray:
        return self._v

    def __eq__(self, other) -> bool:  # element-wise == like std::vector<double>
        return isinstance(other, TemperatureField) and self._v.shape == other._v.shape and bool(
            np.all(self._v == other._v))

    def __repr__(self) -> str:
        return f"TemperatureField(N={self._v.size})"


@dataclass(frozen=True)
class BoundaryCondition:
    """core.hpp:66-81"""

    kind: int = _lib.BC_DIRICHLET
    c1: float = 0.0
    c2: float = 0.0

    @staticmethod
    def dirichlet(c1: float, c2: float) -> "BoundaryCondition":
        return BoundaryCondition(_lib.BC_DIRICHLET, float(c1), float(c2))

    @staticmethod
    def periodic() -> "BoundaryCondition":
        return BoundaryCondition(_lib.BC_PERIODIC, 0.0, 0.0)

    def is_dirichlet(self) -> bool:
        return self.kind == _lib.BC_DIRICHLET


class PartitionSpec:
    """core.hpp:83-102, core.cpp:66-72"""

    def __init__(self, total_points: int, points_per_pe: int):
        if total_points < 3:
            raise DomainError("PartitionSpec: N >= 3 required")
        if points_per_pe == 0 or total_points % points_per_pe != 0:
            raise DomainError("PartitionSpec: n must divide N")
        self._total, self._per = int(total_points), int(points_per_pe)

    def total(self) -> int:
        return self._total

    def per_pe(self) -> int:
        return self._per

    def pe_count(self) -> int:
        return self._total // self._per

    def pe_of(self, i: int) -> int:
        return i // self._per

    def crosses(self, i: int, j: int) -> bool:
        return self.pe_of(i) != self.pe_of(j)


# ---- harness helpers (core.hpp:111-123); CPU, not on the hot path ----------
def cosine_init(n_points: int) -> TemperatureField:
    """core.cpp:29-39 (math.cos is the platform libm cos, as std::cos)."""
    if n_points < 3:
        raise DomainError("cosine_init: N >= 3 required")
    v = []
    for i in range(n_points):
        c = math.cos(3.0 * math.pi / 2.0 * float(i) / float(n_points - 1))
        v.append(c * c)
    return TemperatureField(v)


def linear_steady_state(n_points: int, c1: float, c2: float) -> TemperatureField:
    """core.cpp:41-48"""
    if n_points < 3:
        raise DomainError("linear_steady_state: N >= 3 required")
    return TemperatureField([c1 + (c2 - c1) * float(i) / float(n_points - 1)
                             for i in range(n_points)])


def l2_norm(u) -> float:
    """core.cpp:50-56 (sequential sum, same rounding order)."""
    v = u.values() if isinstance(u, TemperatureField) else np.asarray(u, np.float64)
    s = 0.0
    for x in v.tolist():
        s += x * x
    return math.sqrt(s)


def total_heat(u) -> float:
    """core.cpp:58-64"""
    v = u.values() if isinstance(u, TemperatureField) else np.asarray(u, np.float64)
    s = 0.0
    for x in v.tolist():
        s += x
    return s


# ---- sync_solver.hpp -------------------------------------------------------
@dataclass
class Trajectory:
    """sync_solver.hpp:12-20"""

    snapshots: list
    steps: list
    params: SolverParams
    bc: BoundaryCondition

    def initial(self) -> TemperatureField:
        return self.snapshots[0]

    def final(self) -> TemperatureField:
        return self.snapshots[-1]


K_DIRICHLET_END_TOL = 1e-9  # sync_solver.hpp:44


def default_stride(n_points: int) -> int:
    """sync_solver.hpp:52-54"""
    return 1 if n_points <= 1000 else 100


def set_device(device: int) -> None:
    """Device of this thread's one-shot calls (heat_set_device)."""
    _lib.check(_lib.lib().heat_set_device(int(device)), "set_device")


def set_strict_finite_checks(enabled: bool) -> None:
    _lib.lib().heat_set_strict_finite_checks(int(bool(enabled)))


def strict_finite_checks() -> bool:
    return bool(_lib.lib().heat_strict_finite_checks())


def prepare_initial(u0: TemperatureField, bc: BoundaryCondition) -> np.ndarray:
    """detail::prepare_initial (sync_solver.cpp:25-37): a copy of u0; for Dirichlet
    InvalidArgument if an end is off by more than 1e-9, else the ends snapped."""
    v = _field(u0)
    out = np.empty_like(v)
    _lib.check(_lib.lib().heat_prepare_initial(_lib.dptr(v), v.size, bc.kind, bc.c1, bc.c2,
                                               _lib.dptr(out)), "prepare_initial")
    return out


def _field(u0) -> np.ndarray:
    if isinstance(u0, TemperatureField):
        return np.ascontiguousarray(u0.values())
    return np.ascontiguousarray(TemperatureField(u0).values())


_NULL_PD = C.cast(None, _lib._pd)


def _trajectory(fn, what, u0, params, bc, k_end, stride, extra=()) -> Trajectory:
    v = _field(u0)
    n = v.size
    if stride == 0:
        stride = default_stride(n)  # as the library does (sync_solver.hpp:52-54)
    # rows 0, stride, ..., and k_end when it is not a multiple (heat_trajectory_length)
    count = 1 + k_end // stride + (1 if k_end % stride else 0)
    snaps = np.empty((count, n), np.float64)
    steps = np.empty(count, np.uintp)
    ns = C.c_size_t(0)
    _lib.check(fn(v.ctypes.data, n, params.r(), bc.kind, bc.c1, bc.c2, *extra, k_end, stride,
                  _NULL_PD, snaps.ctypes.data, steps.ctypes.data, count, C.byref(ns)), what)
    m = ns.value
    snaps.setflags(write=False)  # rows are shared by the snapshots, never copied
    adopt = TemperatureField._adopt
    return Trajectory([adopt(row) for row in snaps[:m]], steps[:m].tolist(), params, bc)


def sync_step(u: TemperatureField, params: SolverParams, bc: BoundaryCondition) -> TemperatureField:
    """sync_solver.hpp:60-62"""
    v = _field(u)
    out = np.empty_like(v)
    _lib.check(_lib.lib().heat_sync_step(_lib.dptr(v), v.size, params.r(), bc.kind, bc.c1, bc.c2,
                                         _lib.dptr(out)), "sync_step")
    return TemperatureField(out)


def sync_run(u0: TemperatureField, params: SolverParams, bc: BoundaryCondition, k_end: int,
             stride: int = 1) -> Trajectory:
    """sync_solver.hpp:64-67"""
    return _trajectory(_lib.lib().heat_sync_run, "sync_run", u0, params, bc, k_end, stride)


def sync_run_f32(u0: TemperatureField, params: SolverParams, bc: BoundaryCondition, k_end: int,
                 stride: int = 1) -> Trajectory:
    """sync_solver.hpp:69-73"""
    return _trajectory(_lib.lib().heat_sync_run_f32, "sync_run_f32", u0, params, bc, k_end, stride)


def sync_final(u0, params: SolverParams, bc: BoundaryCondition, k_end: int) -> np.ndarray:
    """Final state only (no snapshot copies): sync_run(...).final() without the trajectory."""
    v = _field(u0)
    out = np.empty_like(v)
    _lib.check(_lib.lib().heat_sync_run(_lib.dptr(v), v.size, params.r(), bc.kind, bc.c1, bc.c2,
                                        k_end, k_end or 1, _lib.dptr(out), None, None, 0, None),
               "sync_run")
    return out


# ---- async_sim.hpp -----------------------------------------------------------
class Distribution(enum.IntEnum):
    Uniform = _lib.DELAY_UNIFORM
    Fixed = _lib.DELAY_FIXED
    GeometricTruncated = _lib.DELAY_GEOMETRIC


@dataclass
class DelayModel:
    """async_sim.hpp:16-28, factories async_sim.cpp:7-23"""

    q: int = 1
    distribution: Distribution = Distribution.Uniform
    fixed_delay: int = 0
    geometric_p: float = 0.5
    seed: int = 0

    @staticmethod
    def uniform(q: int, seed: int) -> "DelayModel":
        if q == 0:
            raise DomainError("DelayModel: q >= 1 required")
        return DelayModel(q, Distribution.Uniform, 0, 0.5, seed)

    @staticmethod
    def fixed(q: int, d: int, seed: int) -> "DelayModel":
        if q == 0:
            raise DomainError("DelayModel: q >= 1 required")
        if d >= q:
            raise DomainError("DelayModel: fixed delay must satisfy d < q")
        return DelayModel(q, Distribution.Fixed, d, 0.5, seed)

    @staticmethod
    def geometric(q: int, p: float, seed: int) -> "DelayModel":
        if q == 0:
            raise DomainError("DelayModel: q >= 1 required")
        if not (p > 0.0) or p > 1.0:
            raise DomainError("DelayModel: geometric p must lie in (0, 1]")
        return DelayModel(q, Distribution.GeometricTruncated, 0, p, seed)

    def _args(self):
        return (self.q, int(self.distribution), self.fixed_delay, self.geometric_p,
                self.seed & 0xFFFFFFFFFFFFFFFF)


def sample_delay_at(model: DelayModel, j: int, k: int) -> int:
    """Counter form of sample_delay (async_sim.cpp:57-73): the j-th draw at step k."""
    d = C.c_size_t(0)
    _lib.check(_lib.lib().heat_sample_delay(*model._args(), j, k, C.byref(d)), "sample_delay")
    return d.value


_GAMMA = 0x9E3779B97F4A7C15
_M64 = 0xFFFFFFFFFFFFFFFF


class SplitMix64:
    """rng.hpp:16-41.  `state` is the stream position; async_step advances it
    on the device exactly as the reference's stream would be advanced."""

    def __init__(self, seed: int):
        self.state = int(seed) & _M64

    def next(self) -> int:
        self.state = (self.state + _GAMMA) & _M64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -53

    def next_bounded(self, bound: int) -> int:
        return self.next() % (bound + 1)


def sample_delay(rng: SplitMix64, model: DelayModel, k: int) -> int:
    """sample_delay (async_sim.cpp:57-73): one draw of `rng`'s stream at step k."""
    d = C.c_size_t(0)
    q, law, fd, p, _ = model._args()
    _lib.check(_lib.lib().heat_sample_delay(q, law, fd, p, rng.state, 0, k, C.byref(d)),
               "sample_delay")
    rng.state = (rng.state + _GAMMA) & _M64
    return d.value


class HistoryRing:
    """HistoryRing (async_sim.hpp:31-57, async_sim.cpp:25-55) with its snapshots
    in HBM: read(i, d) = u_i(current_step - d), LogicError when d >= depth,
    d > k or d >= snapshots held.  push() of a host state rotates the ring
    without moving device data; async_step() reads it on the device."""

    def __init__(self, depth: int, initial, device: int = -1):
        self._create(depth, 0, np.asarray(initial, np.float64).reshape(1, -1), device)

    @classmethod
    def at_step(cls, depth: int, step: int, snapshots, device: int = -1) -> "HistoryRing":
        """A ring at `step` holding min(depth, step + 1) snapshots, row d = u(step - d)."""
        ring = cls.__new__(cls)
        rows = np.asarray(snapshots, np.float64)
        ring._create(depth, step, rows.reshape(rows.shape[0], -1), device)
        return ring

    def _create(self, depth: int, step: int, rows: np.ndarray, device: int) -> None:
        rows = np.ascontiguousarray(rows)
        self._h = C.c_void_p()
        self._n = rows.shape[1]
        _lib.check(_lib.lib().heat_history_create(C.byref(self._h), depth, self._n, step,
                                                  _lib.dptr(rows), rows.shape[0], device),
                   "HistoryRing")

    def _info(self):
        d, k, n = C.c_size_t(), C.c_size_t(), C.c_size_t()
        _lib.check(_lib.lib().heat_history_info(self._h, C.byref(d), C.byref(k), C.byref(n)),
                   "HistoryRing")
        return d.value, k.value, n.value

    def depth(self) -> int:
        return self._info()[0]

    def current_step(self) -> int:
        return self._info()[1]

    def grid_size(self) -> int:
        return self._n

    def push(self, state) -> None:
        v = np.ascontiguousarray(np.asarray(state, np.float64).reshape(-1))
        _lib.check(_lib.lib().heat_history_push(self._h, _lib.dptr(v), v.size), "HistoryRing::push")

    def read(self, i: int, d: int) -> float:
        x = C.c_double()
        _lib.check(_lib.lib().heat_history_read(self._h, i, d, C.byref(x)), "HistoryRing::read")
        return x.value

    def snapshot(self, d: int) -> np.ndarray:
        out = np.empty(self._n, np.float64)
        _lib.check(_lib.lib().heat_history_snapshot(self._h, d, _lib.dptr(out)),
                   "HistoryRing::snapshot")
        return out

    def _step(self, params, bc, part, model, rng, out, push):
        st = C.c_uint64(rng.state)
        q, law, fd, p, _ = model._args()
        try:
            _lib.check(_lib.lib().heat_async_step(self._h, params.r(), bc.kind, bc.c1, bc.c2,
                                                  part.total(), part.per_pe(), q, law, fd, p,
                                                  C.byref(st), _lib.dptr(out), int(push)),
                       "async_step")
        finally:
            rng.state = int(st.value)

    def push_async_step(self, params: SolverParams, bc: BoundaryCondition, part: PartitionSpec,
                        model: DelayModel, rng: SplitMix64) -> None:
        """AsyncSimulator::step (async_sim.cpp:136-140) on this ring: async_step,
        then push its result, all on the device."""
        self._step(params, bc, part, model, rng, None, True)

    def close(self):
        if self._h:
            _lib.lib().heat_history_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def async_step(hist: HistoryRing, params: SolverParams, bc: BoundaryCondition,
               part: PartitionSpec, model: DelayModel, rng: SplitMix64) -> TemperatureField:
    """async_step (async_sim.hpp:68-71, async_sim.cpp:107-116): one step of Eq. (4)
    over the ring, drawing from `rng` in the reference's order (kernels K8a/K8b)."""
    out = np.empty(hist.grid_size(), np.float64)
    hist._step(params, bc, part, model, rng, out, False)
    return TemperatureField(out)


def async_run(u0: TemperatureField, params: SolverParams, bc: BoundaryCondition,
              part: PartitionSpec, model: DelayModel, k_end: int, stride: int = 1) -> Trajectory:
    """async_sim.hpp:97-101 -- the seeded delay stream replayed on the GPU."""
    v = _field(u0)
    if part.total() != v.size:
        raise InvalidArgument("AsyncSimulator: partition inconsistent with grid")
    return _trajectory(_lib.lib().heat_async_run, "async_run", v, params, bc, k_end, stride,
                       extra=(part.per_pe(), *model._args()))


class AsyncSimulator:
    """AsyncSimulator (async_sim.hpp:73-90, async_sim.cpp:122-140) on the GPU.

    The device holds the field, the PE edge rings and the draw offsets;
    step(count) = count x AsyncSimulator::step().  Any slicing of the steps
    is bit-identical to async_run over the whole run."""

    def __init__(self, u0, params: SolverParams, bc: BoundaryCondition, part: PartitionSpec,
                 model: DelayModel):
        v = _field(u0)
        self._h = C.c_void_p()
        self.n = v.size
        # prepare_initial runs before the partition check (async_sim.cpp:122-134):
        # a mismatched partition is checked after a one-PE create has validated u0
        per_pe = part.per_pe() if part.total() == v.size else v.size
        _lib.check(_lib.lib().heat_async_sim_create(C.byref(self._h), _lib.dptr(v), v.size,
                                                    params.r(), bc.kind, bc.c1, bc.c2, per_pe,
                                                    *model._args()), "AsyncSimulator")
        if part.total() != v.size:
            self.close()
            raise InvalidArgument("AsyncSimulator: partition inconsistent with grid")

    def step(self, count: int = 1) -> None:
        _lib.check(_lib.lib().heat_async_sim_step(self._h, count), "AsyncSimulator::step")

    def step_index(self) -> int:
        k = C.c_size_t(0)
        _lib.check(_lib.lib().heat_async_sim_current(self._h, None, C.byref(k)), "step_index")
        return int(k.value)

    def current(self) -> np.ndarray:
        out = np.empty(self.n, np.float64)
        _lib.check(_lib.lib().heat_async_sim_current(self._h, _lib.dptr(out), None), "current")
        return out

    def current_field(self) -> TemperatureField:
        return TemperatureField(self.current())

    def close(self):
        if self._h:
            _lib.lib().heat_async_sim_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def async_final(u0, params: SolverParams, bc: BoundaryCondition, part: PartitionSpec,
                model: DelayModel, k_end: int) -> np.ndarray:
    """Final state of async_run without the trajectory copies."""
    v = _field(u0)
    if part.total() != v.size:
        raise InvalidArgument("AsyncSimulator: partition inconsistent with grid")
    out = np.empty_like(v)
    _lib.check(_lib.lib().heat_async_run(_lib.dptr(v), v.size, params.r(), bc.kind, bc.c1, bc.c2,
                                         part.per_pe(), *model._args(), k_end, k_end or 1,
                                         _lib.dptr(out), None, None, 0, None), "async_run")
    return out


def async_free_run(u0, params: SolverParams, bc: BoundaryCondition, part: PartitionSpec,
                   q: int, k_end: int):
    """Free-running async with bounded staleness q and full edge logs (GPU only).

    Returns (final field as ndarray, AsyncStats); stats.residual_sum is the
    a-posteriori bound on ||u_async(K) - u_sync(K)||_inf."""
    v = _field(u0)
    if part.total() != v.size:
        raise InvalidArgument("async_free_run: partition inconsistent with grid")
    out = np.empty_like(v)
    st = _lib.AsyncStatsC()
    _lib.check(_lib.lib().heat_async_free_run(_lib.dptr(v), v.size, params.r(), bc.kind, bc.c1,
                                              bc.c2, part.per_pe(), q, k_end, _lib.dptr(out),
                                              C.byref(st)), "async_free_run")
    return out, AsyncStats(int(st.reads), int(st.max_delay), [int(x) for x in st.delay_histogram],
                           int(st.waits), float(st.residual_sum))


# ---- analysis.hpp: ensembles -------------------------------------------------
@dataclass
class EnsembleConfig:
    """analysis.hpp:14-23 (model.seed is ignored; members use base_seed + j)."""

    u0: TemperatureField
    params: SolverParams
    bc: BoundaryCondition
    part: PartitionSpec
    model: DelayModel
    k_end: int = 1
    stride: int = 1


@dataclass
class EnsembleResult:
    """analysis.hpp:25-32"""

    steps: list
    norm_series: list          # [run][recorded step]
    terminal_fields: list      # [run]
    mean_series: list
    std_series: list
    seeds: list


def ensemble_run(cfg: EnsembleConfig, runs: int, base_seed: int,
                 keep_terminals: bool = True) -> EnsembleResult:
    """analysis.cpp:51-104 on the GPU: one CTA per member (K6, csrc/ensemble.cu), or
    AsyncSimulator handles (K3/K5) when a member's history exceeds shared memory."""
    v = _field(cfg.u0)
    n = v.size
    if cfg.part.total() != n:
        raise InvalidArgument("AsyncSimulator: partition inconsistent with grid")
    stride = cfg.stride or default_stride(n)
    cap = 2 + cfg.k_end // stride
    steps = np.zeros(cap, np.uintp)
    ns = C.c_size_t(0)
    norms = np.zeros(max(1, runs) * cap, np.float64)
    terms = np.zeros((runs, n), np.float64) if keep_terminals and runs else None
    mean = np.zeros(cap, np.float64)
    std = np.zeros(cap, np.float64)
    m = cfg.model
    _lib.check(_lib.lib().heat_ensemble_run(
        _lib.dptr(v), n, cfg.params.r(), cfg.bc.kind, cfg.bc.c1, cfg.bc.c2, cfg.part.per_pe(),
        m.q, int(m.distribution), m.fixed_delay, m.geometric_p, cfg.k_end, stride, runs,
        base_seed & 0xFFFFFFFFFFFFFFFF, _lib.szptr(steps), cap, C.byref(ns), _lib.dptr(norms),
        _lib.dptr(terms), _lib.dptr(mean), _lib.dptr(std)), "ensemble_run")
    S = ns.value
    nrm = norms[:runs * S].reshape(runs, S)
    return EnsembleResult([int(s) for s in steps[:S]], [list(map(float, row)) for row in nrm],
                          [TemperatureField(t) for t in terms] if terms is not None else [],
                          [float(x) for x in mean[:S]], [float(x) for x in std[:S]],
                          [base_seed + j for j in range(runs)])


def _population_std(xs):
    mean = 0.0
    for x in xs:
        mean += x
    mean /= float(len(xs))
    var = 0.0
    for x in xs:
        var += (x - mean) * (x - mean)
    return math.sqrt(var / float(len(xs)))


def terminal_spread(res: EnsembleResult):
    """analysis.cpp:122-132: (std of terminal mean temperature, std of terminal norm)."""
    runs = len(res.terminal_fields)
    if runs < 2:
        raise DomainError("terminal_spread: M >= 2 required")
    temps = [total_heat(f) / float(f.size()) for f in res.terminal_fields]
    norms = [l2_norm(f) for f in res.terminal_fields]
    return _population_std(temps), _population_std(norms)


def convergence_check(traj: Trajectory, reference: TemperatureField, tol: float):
    """analysis.cpp:106-120: first recorded step within `tol` (max-abs) of `reference`."""
    if not (tol > 0.0):
        raise DomainError("convergence_check: tol > 0 required")
    for snap, k in zip(traj.snapshots, traj.steps):
        if snap.size() != reference.size():
            raise InvalidArgument("convergence_check: size mismatch")
        if float(np.max(np.abs(snap.values() - reference.values()))) <= tol:
            return k
    return None


# ---- async_exec.hpp ----------------------------------------------------------
class ExecMode(enum.IntEnum):
    Barriered = _lib.EXEC_BARRIERED
    BarrierFree = _lib.EXEC_BARRIER_FREE


def to_string(mode: ExecMode) -> str:
    return "barriered" if mode == ExecMode.Barriered else "barrier-free"


@dataclass
class LagStats:
    """async_exec.hpp:42-51"""

    reads: int = 0
    min_lag: int = 0
    max_lag: int = 0
    histogram: list = field(default_factory=list)
    overflow: int = 0

    def merge(self, other: "LagStats") -> None:
        if other.reads == 0:
            return
        if self.reads == 0:
            self.reads, self.min_lag, self.max_lag = other.reads, other.min_lag, other.max_lag
            self.histogram, self.overflow = list(other.histogram), other.overflow
            return
        self.min_lag = min(self.min_lag, other.min_lag)
        self.max_lag = max(self.max_lag, other.max_lag)
        self.reads += other.reads
        if len(self.histogram) < len(other.histogram):
            self.histogram += [0] * (len(other.histogram) - len(self.histogram))
        for i, c in enumerate(other.histogram):
            self.histogram[i] += c
        self.overflow += other.overflow

    def mean(self) -> float:
        if self.reads == 0:
            return 0.0
        return sum(float(d) * float(c) for d, c in enumerate(self.histogram)) / float(self.reads)


@dataclass
class AsyncStats:
    """Reader-relative delay log of the GPU free-running executor."""

    reads: int = 0
    max_delay: int = 0
    delay_histogram: list = field(default_factory=list)
    waits: int = 0
    residual_sum: float = 0.0


@dataclass
class ExecConfig:
    """async_exec.hpp:53-58 (+ q_free: the GPU free-running staleness bound)."""

    workers: int = 1
    k_end: int = 1
    mode: ExecMode = ExecMode.Barriered
    record_lag: bool = False
    q_free: int = 0


@dataclass
class ExecResult:
    """async_exec.hpp:60-66 (duration is GPU device time, ns)."""

    field: TemperatureField
    steps_per_pe: list
    duration_ns: int = 0
    oversubscribed: bool = False
    lag: Optional[LagStats] = None
    stats: Optional[AsyncStats] = None


def exec_run(u0: TemperatureField, params: SolverParams, bc: BoundaryCondition,
             part: PartitionSpec, cfg: ExecConfig, stats: bool = True) -> ExecResult:
    """async_exec.hpp:68-70 / async_exec.cpp:263-279.  `stats` (a B200
    extension, BarrierFree only): collect the kernel's delay histogram into
    `res.stats`; measure() times the runs without it, as the reference's
    exec_run collects nothing."""
    v = _field(u0)
    out = np.empty_like(v)
    dur = C.c_uint64(0)
    lag = _lib.LagStatsC()
    st = _lib.AsyncStatsC()
    _lib.check(_lib.lib().heat_exec_run(_lib.dptr(v), v.size, params.r(), bc.kind, bc.c1, bc.c2,
                                        part.per_pe(), cfg.workers, cfg.k_end, int(cfg.mode),
                                        int(cfg.record_lag), cfg.q_free, _lib.dptr(out),
                                        C.byref(dur), C.byref(lag), C.byref(st) if stats else None),
               "exec_run")
    res = ExecResult(TemperatureField(out), [cfg.k_end] * cfg.workers, int(dur.value))
    if cfg.record_lag:
        res.lag = LagStats(int(lag.reads), int(lag.min_lag), int(lag.max_lag),
                           [int(x) for x in lag.histogram], int(lag.overflow))
    if cfg.mode == ExecMode.BarrierFree and stats:
        res.stats = AsyncStats(int(st.reads), int(st.max_delay),
                               [int(x) for x in st.delay_histogram], int(st.waits),
                               float(st.residual_sum))
    return res


@dataclass
class BenchRow:
    """async_exec.hpp:72-78 (times are GPU device time, ns)."""

    n_points: int = 0
    mode: ExecMode = ExecMode.Barriered
    reps: int = 0
    median_ns: int = 0
    min_ns: int = 0


def measure(grid_sizes: Sequence[int], modes: Sequence[ExecMode], reps: int, k_end: int,
            workers: int) -> list:
    """measure (async_exec.cpp:281-307): cosine IC, r = 0.5, Dirichlet(1, 0),
    `workers` PEs; median = times[reps // 2] and min of `reps` exec_run calls."""
    if reps < 3:
        raise InvalidArgument("measure: reps >= 3 required")
    rows = []
    for n in grid_sizes:
        if n % workers != 0:
            raise InvalidArgument("measure: workers must divide every N")
        u0 = cosine_init(n)
        params = SolverParams.from_r(0.5)
        bc = BoundaryCondition.dirichlet(1.0, 0.0)
        part = PartitionSpec(n, n // workers)
        for mode in modes:
            cfg = ExecConfig(workers, k_end, mode, False)
            times = sorted(exec_run(u0, params, bc, part, cfg, stats=False).duration_ns
                           for _ in range(reps))
            rows.append(BenchRow(n, mode, reps, times[len(times) // 2], times[0]))
    return rows


def speedup_ratio(rows: Sequence[BenchRow], n_points: int) -> float:
    """speedup_ratio (async_exec.cpp:309-318): barriered median / barrier-free median."""
    barriered = free_running = 0
    for row in rows:
        if row.n_points != n_points:
            continue
        if row.mode == ExecMode.Barriered:
            barriered = row.median_ns
        else:
            free_running = row.median_ns
    if barriered == 0 or free_running == 0:
        raise InvalidArgument("speedup_ratio: missing mode for this N")
    return float(barriered) / float(free_running)


# ---- device-resident plan ------------------------------------------------------
class Plan:
    """A field resident in HBM (heat_plan_*): bench and multi-GPU slabs."""

    def __init__(self, n: int, device: int = 0, rank: int = 0, world: int = 1):
        self._h = C.c_void_p()
        if world == 1:
            _lib.check(_lib.lib().heat_plan_create(C.byref(self._h), n, device),
                       "heat_plan_create")
        else:
            _lib.check(_lib.lib().heat_plan_create_slab(C.byref(self._h), n, device, rank, world),
                       "heat_plan_create_slab")
        self.n = n
        self.device = device
        self.rank, self.world = rank, world

    @staticmethod
    def halo() -> int:
        """Ghost points per side of a slab = max steps per exchange."""
        return int(_lib.lib().heat_slab_halo())

    # ---- multi-GPU asynchronous slabs over NVLink P2P (heat_plan_xlink_*) ----
    def xlink_setup(self, per_pe: int, q: int, bc: BoundaryCondition) -> bytes:
        """Allocate the receive rings; returns this rank's IPC handle to share."""
        size = int(_lib.lib().heat_xlink_handle_size())
        buf = C.create_string_buffer(size)
        _lib.check(_lib.lib().heat_plan_xlink_setup(self._h, per_pe, q, bc.kind, buf),
                   "xlink_setup")
        return buf.raw

    def xlink_connect(self, left: Optional[bytes], right: Optional[bytes]):
        lb = C.create_string_buffer(left, len(left)) if left is not None else None
        rb = C.create_string_buffer(right, len(right)) if right is not None else None
        _lib.check(_lib.lib().heat_plan_xlink_connect(self._h, lb, rb), "xlink_connect")

    def xlink_seed(self):
        _lib.check(_lib.lib().heat_plan_xlink_seed(self._h), "xlink_seed")

    def xlink_advance(self, r: float, bc: BoundaryCondition, steps: int,
                      model: Optional["DelayModel"] = None):
        """mode free (model None, bound = the q of xlink_setup) or replay of `model`."""
        st = _lib.AsyncStatsC()
        if model is None:
            args = (1, int(Distribution.Uniform), 0, 0.5, 0)
        else:
            args = (0, int(model.distribution), model.fixed_delay, model.geometric_p,
                    model.seed & 0xFFFFFFFFFFFFFFFF)
        _lib.check(_lib.lib().heat_plan_xlink_advance(self._h, r, bc.c1, bc.c2, *args, steps,
                                                      C.byref(st)), "xlink_advance")
        return st

    def xlink_debug_recv(self):
        out = np.zeros(2, np.float64)
        _lib.check(_lib.lib().heat_plan_xlink_debug_recv(self._h, _lib.dptr(out)), "debug")
        return out

    def halo_pack(self, dst_device_ptr: int):
        _lib.check(_lib.lib().heat_plan_halo_pack(self._h, dst_device_ptr), "halo_pack")

    def halo_unpack(self, src_device_ptr: int):
        _lib.check(_lib.lib().heat_plan_halo_unpack(self._h, src_device_ptr), "halo_unpack")

    def close(self):
        if self._h:
            _lib.lib().heat_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int | None):
        _lib.check(_lib.lib().heat_plan_set_stream(self._h, stream_handle), "set_stream")

    def upload(self, host: np.ndarray):
        assert host.dtype == np.float64 and host.size == self.n and host.flags.c_contiguous
        _lib.check(_lib.lib().heat_plan_upload(self._h, host.ctypes.data), "upload")

    def download(self, host: Optional[np.ndarray] = None) -> np.ndarray:
        if host is None:
            host = np.empty(self.n, np.float64)
        _lib.check(_lib.lib().heat_plan_download(self._h, host.ctypes.data), "download")
        return host

    def download_range(self, offset: int, count: int) -> np.ndarray:
        """Points [offset, offset + count) of the owned field."""
        out = np.empty(count, np.float64)
        _lib.check(_lib.lib().heat_plan_download_range(self._h, offset, count, out.ctypes.data),
                   "download_range")
        return out

    def download_device(self, dst_device_ptr: int):
        """Owned points into device memory (stream-ordered on the plan's stream)."""
        _lib.check(_lib.lib().heat_plan_download_device(self._h, dst_device_ptr),
                   "download_device")

    def fill_sine(self):
        _lib.check(_lib.lib().heat_plan_fill_sine(self._h), "fill_sine")

    def sync_advance(self, r: float, bc: BoundaryCondition, steps: int):
        _lib.check(_lib.lib().heat_plan_sync_advance(self._h, r, bc.kind, bc.c1, bc.c2, steps),
                   "sync_advance")

    def async_advance(self, r: float, bc: BoundaryCondition, per_pe: int, q: int, steps: int):
        """Free-running bounded-staleness async (delays <= q-1), a fresh run."""
        st = _lib.AsyncStatsC()
        _lib.check(_lib.lib().heat_plan_async_advance(self._h, r, bc.kind, bc.c1, bc.c2, per_pe,
                                                      q, steps, C.byref(st)), "async_advance")
        return st

    def async_replay(self, r: float, bc: BoundaryCondition, per_pe: int, model: "DelayModel",
                     steps: int):
        """Deterministic async: replays `model`'s seeded delays (async_run semantics)."""
        st = _lib.AsyncStatsC()
        _lib.check(_lib.lib().heat_plan_async_replay(self._h, r, bc.kind, bc.c1, bc.c2, per_pe,
                                                     *model._args(), steps, C.byref(st)),
                   "async_replay")
        return st

    def synchronize(self):
        _lib.check(_lib.lib().heat_plan_synchronize(self._h), "synchronize")

    def device_ptr(self) -> int:
        p = C.c_void_p()
        _lib.check(_lib.lib().heat_plan_device_ptr(self._h, C.byref(p)), "device_ptr")
        return int(p.value or 0)


def kernel_launches() -> int:
    return int(_lib.lib().heat_kernel_launches())
