"""ctypes face of the CPU oracles.  TEST INFRASTRUCTURE ONLY.

Two libraries, both built by ``oracle/Makefile``:

* ``Port`` -- ``oracle/libheat_oracle.so``, our C restatement of the reference
  hot path (``oracle/heat_oracle.c``).  Always buildable (gcc only).
* ``Ref``  -- ``oracle/_ref/libheat_ref.so``, the reference's own sources from
  /root/reference/proj/src compiled with its own flags, behind ``ref_shim.cpp``.
  Built in the build container (where /root/reference exists) and shipped to the
  GPU box as a prebuilt file.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libheat_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libheat_ref.so")
REF_SRC = "/root/reference/proj"

DIRICHLET, PERIODIC = 0, 1
UNIFORM, FIXED, GEOMETRIC = 0, 1, 2
BARRIERED, BARRIER_FREE = 0, 1

_lock = threading.Lock()

_P = C.POINTER
_d = C.c_double
_sz = C.c_size_t
_u64 = C.c_uint64
_i = C.c_int
_pd = _P(C.c_double)
_psz = _P(C.c_size_t)
_pu64 = _P(C.c_uint64)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: status {code}")
        self.code = code


def build(ref: bool | None = None) -> None:
    """Build the port (always) and the reference library (when its sources exist)."""
    with _lock:
        subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
        if ref is None:
            ref = os.path.isdir(REF_SRC)
        if ref:
            subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
            lib = os.path.join(os.path.dirname(HERE), "paper_1510_08982_b200", "libheat_b200.so")
            if os.path.exists(lib):  # reference acceptance suite vs. the GPU library
                subprocess.run(["make", "-s", "-C", HERE, "acceptance"], check=True)


def _ptr(a: np.ndarray | None, ty=_pd):
    if a is None:
        return C.cast(None, ty)
    return a.ctypes.data_as(ty)


def _f64(u) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(u, dtype=np.float64))


class _Lib:
    path: str
    prefix: str

    def __init__(self):
        if not os.path.exists(self.path):
            build(ref=(self.prefix == "ref"))
        self.lib = C.CDLL(self.path)


class Port(_Lib):
    """Our C restatement (oracle/heat_oracle.c)."""

    path = PORT_SO
    prefix = "orc"

    def __init__(self):
        super().__init__()
        L = self.lib
        L.orc_splitmix_next.argtypes = [_pu64]
        L.orc_splitmix_next.restype = _u64
        L.orc_delay_stream.argtypes = [_i, _sz, _sz, _d, _u64, _sz, _sz, _pu64]
        L.orc_sync_run.argtypes = [_pd, _sz, _d, _i, _d, _d, _sz, _sz, _i, _pd, _pd, _psz, _sz, _psz]
        L.orc_sync_run_f32.argtypes = [_pd, _sz, _d, _i, _d, _d, _sz, _i, _pd]
        L.orc_async_run.argtypes = [_pd, _sz, _d, _i, _d, _d, _sz, _i, _sz, _sz, _d, _u64, _sz,
                                    _sz, _i, _pd, _pd, _psz, _sz, _psz]
        for f in ("orc_exec_barriered", "orc_exec_barrier_free"):
            getattr(L, f).argtypes = [_pd, _sz, _d, _i, _d, _d, _sz, _sz, _sz, _pd, _pu64]
        L.orc_sine_init.argtypes = [_sz, _pd, _i]
        L.orc_cosine_init.argtypes = [_sz, _pd]
        L.orc_linear_steady_state.argtypes = [_sz, _d, _d, _pd]
        L.orc_l2_norm.argtypes = [_pd, _sz]
        L.orc_l2_norm.restype = _d
        L.orc_total_heat.argtypes = [_pd, _sz]
        L.orc_total_heat.restype = _d
        L.orc_fnv1a64.argtypes = [_pd, _sz]
        L.orc_fnv1a64.restype = _u64
        L.orc_prepare_initial.argtypes = [_pd, _sz, _i, _d, _d, _pd]
        L.orc_sync_lightcone.argtypes = [_pd, _sz, _d, _i, _d, _d, _sz, _sz, _pd]
        L.orc_async_lightcone.argtypes = [_pd, _sz, _sz, _sz, _d, _d, _d, _sz, _i, _sz, _sz, _d,
                                          C.c_uint64, _sz, _sz, _pd]
        L.orc_sync_window.argtypes = [_pd, _sz, _sz, _sz, _d, _d, _d, _sz]
        L.orc_async_window.argtypes = [_pd, _sz, _sz, _sz, _d, _d, _d, _sz, _i, _sz, _sz, _d,
                                       C.c_uint64, _sz]
        L.orc_sync_step_into.argtypes = [_pd, _pd, _sz, _d, _i, _d, _d]
        L.orc_sync_step_into.restype = None
        L.orc_async_step.argtypes = [_pd, _sz, _sz, _sz, _sz, _d, _i, _d, _d, _sz, _sz, _i, _sz,
                                     _sz, _d, _pu64, _i, _pd]

    # --- initial conditions / norms --------------------------------------
    def sine_init(self, n: int, threads: int | None = None) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.orc_sine_init(n, _ptr(out), threads or os.cpu_count() or 1)
        return out

    def cosine_init(self, n: int) -> np.ndarray:
        out = np.empty(n, np.float64)
        if self.lib.orc_cosine_init(n, _ptr(out)):
            raise OracleError(1, "cosine_init")
        return out

    def linear_steady_state(self, n, c1, c2) -> np.ndarray:
        out = np.empty(n, np.float64)
        self.lib.orc_linear_steady_state(n, c1, c2, _ptr(out))
        return out

    def l2_norm(self, u) -> float:
        u = _f64(u)
        return self.lib.orc_l2_norm(_ptr(u), u.size)

    def total_heat(self, u) -> float:
        u = _f64(u)
        return self.lib.orc_total_heat(_ptr(u), u.size)

    def fnv1a64(self, u) -> int:
        u = _f64(u)
        return int(self.lib.orc_fnv1a64(_ptr(u), u.size))

    def prepare_initial(self, u0, bc=DIRICHLET, c1=0.0, c2=0.0) -> np.ndarray:
        u0 = _f64(u0)
        out = np.empty_like(u0)
        st = self.lib.orc_prepare_initial(_ptr(u0), u0.size, bc, c1, c2, _ptr(out))
        if st:
            raise OracleError(st, "prepare_initial")
        return out

    # --- rng -------------------------------------------------------------
    def delay_stream(self, law, q, fixed_d, p, seed, k, count) -> list[int]:
        out = np.empty(count, np.uint64)
        self.lib.orc_delay_stream(law, q, fixed_d, p, seed, k, count, _ptr(out, _pu64))
        return [int(x) for x in out]

    # --- solvers ---------------------------------------------------------
    def sync_step(self, u, r, bc=DIRICHLET, c1=0.0, c2=0.0) -> np.ndarray:
        u = _f64(u)
        out = np.empty_like(u)
        self.lib.orc_sync_step_into(_ptr(u), _ptr(out), u.size, r, bc, c1, c2)
        return out

    def sync_run(self, u0, r, bc=DIRICHLET, c1=0.0, c2=0.0, k_end=1, stride=None,
                 strict=False, record=False):
        u0 = _f64(u0)
        n = u0.size
        fin = np.empty(n, np.float64)
        snaps = steps = None
        cap = 0
        if record:
            s = stride if stride else (1 if n <= 1000 else 100)
            cap = k_end // s + 2
            snaps = np.empty((cap, n), np.float64)
            steps = np.empty(cap, np.uintp)
        ns = C.c_size_t(0)
        st = self.lib.orc_sync_run(_ptr(u0), n, r, bc, c1, c2, k_end,
                                   stride if stride is not None else (k_end or 1), int(strict),
                                   _ptr(fin), _ptr(snaps), _ptr(steps, _psz), cap, C.byref(ns))
        if st:
            raise OracleError(st, "sync_run")
        if record:
            return [int(x) for x in steps[:ns.value]], snaps[:ns.value].copy()
        return fin

    def sync_run_f32(self, u0, r, bc=DIRICHLET, c1=0.0, c2=0.0, k_end=1, strict=False):
        u0 = _f64(u0)
        fin = np.empty(u0.size, np.float64)
        st = self.lib.orc_sync_run_f32(_ptr(u0), u0.size, r, bc, c1, c2, k_end, int(strict), _ptr(fin))
        if st:
            raise OracleError(st, "sync_run_f32")
        return fin

    def async_run(self, u0, r, bc, c1, c2, per_pe, law, q, fixed_d=0, p=0.5, seed=0,
                  k_end=1, stride=None, strict=False, record=False):
        u0 = _f64(u0)
        n = u0.size
        fin = np.empty(n, np.float64)
        snaps = steps = None
        cap = 0
        if record:
            s = stride if stride else (1 if n <= 1000 else 100)
            cap = k_end // s + 2
            snaps = np.empty((cap, n), np.float64)
            steps = np.empty(cap, np.uintp)
        ns = C.c_size_t(0)
        st = self.lib.orc_async_run(_ptr(u0), n, r, bc, c1, c2, per_pe, law, q, fixed_d, p, seed,
                                    k_end, stride if stride is not None else (k_end or 1),
                                    int(strict), _ptr(fin), _ptr(snaps), _ptr(steps, _psz), cap,
                                    C.byref(ns))
        if st:
            raise OracleError(st, "async_run")
        if record:
            return [int(x) for x in steps[:ns.value]], snaps[:ns.value].copy()
        return fin

    def async_step(self, snaps, depth, step, r, bc, c1, c2, part_total, per_pe, law, q,
                   fixed_d=0, p=0.5, rng_state=0, strict=False):
        """async_step over a ring at `step` (rows of `snaps`: u(step - d)).
        Returns (status, field or None, rng state after the call)."""
        snaps = np.ascontiguousarray(np.asarray(snaps, np.float64))
        count, n = snaps.shape
        out = np.empty(n, np.float64)
        st_rng = C.c_uint64(rng_state)
        st = self.lib.orc_async_step(_ptr(snaps), count, depth, step, n, r, bc, c1, c2,
                                     part_total, per_pe, law, q, fixed_d, p, C.byref(st_rng),
                                     int(strict), _ptr(out))
        return st, (out if st == 0 else None), int(st_rng.value)

    def exec_run(self, u0, r, bc, c1, c2, per_pe, workers, k_end, mode=BARRIERED):
        u0 = _f64(u0)
        fin = np.empty(u0.size, np.float64)
        dur = C.c_uint64(0)
        f = self.lib.orc_exec_barriered if mode == BARRIERED else self.lib.orc_exec_barrier_free
        st = f(_ptr(u0), u0.size, r, bc, c1, c2, per_pe, workers, k_end, _ptr(fin), C.byref(dur))
        if st:
            raise OracleError(st, "exec_run")
        return fin, int(dur.value)

    def sync_lightcone(self, u0_prepared, r, bc, c1, c2, k, centre) -> float:
        u0 = _f64(u0_prepared)
        v = C.c_double(0.0)
        st = self.lib.orc_sync_lightcone(_ptr(u0), u0.size, r, bc, c1, c2, k, centre, C.byref(v))
        if st:
            raise OracleError(st, "sync_lightcone")
        return v.value

    def sync_window(self, win, lo, n, r, c1, c2, k) -> np.ndarray:
        """The window win = u[lo : lo + len(win)] of an n-point Dirichlet run
        advanced k steps with held window ends (heat_oracle.c orc_sync_window);
        points more than k from a held end are exact."""
        a = np.array(win, dtype=np.float64, copy=True)
        st = self.lib.orc_sync_window(_ptr(a), a.size, lo, n, r, c1, c2, k)
        if st:
            raise OracleError(st, "sync_window")
        return a

    def async_window(self, win, lo, n, r, c1, c2, per_pe, law, q, fixed_d=0, p=0.5, seed=0,
                     k=1) -> np.ndarray:
        """orc_async_window: the deterministic asynchronous run of k steps from
        step 0 on a window with held ends."""
        a = np.array(win, dtype=np.float64, copy=True)
        st = self.lib.orc_async_window(_ptr(a), a.size, lo, n, r, c1, c2, per_pe, law, q, fixed_d,
                                       p, seed & 0xFFFFFFFFFFFFFFFF, k)
        if st:
            raise OracleError(st, "async_window")
        return a

    def async_lightcone(self, win, lo, n, r, c1, c2, per_pe, law, q, fixed_d=0, p=0.5, seed=0,
                        k=1, centre=0) -> float:
        """u(k)[centre] of the deterministic async run (Dirichlet) from the window
        win = u0[lo : lo + len(win)] (heat_oracle.c orc_async_lightcone)."""
        w = _f64(win)
        v = C.c_double(0.0)
        st = self.lib.orc_async_lightcone(_ptr(w), w.size, lo, n, r, c1, c2, per_pe, law, q,
                                          fixed_d, p, seed & 0xFFFFFFFFFFFFFFFF, k, centre,
                                          C.byref(v))
        if st:
            raise OracleError(st, "async_lightcone")
        return v.value


class Ref(_Lib):
    """The reference itself (oracle/_ref/libheat_ref.so)."""

    path = REF_SO
    prefix = "ref"

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO) or os.path.isdir(REF_SRC)

    def __init__(self):
        super().__init__()
        L = self.lib
        L.ref_set_strict.argtypes = [_i]
        L.ref_set_strict.restype = None
        L.ref_params_checked_r.argtypes = [_d, _d, _d, _pd]
        L.ref_sync_step.argtypes = [_pd, _sz, _d, _i, _d, _d, _pd]
        L.ref_sync_run.argtypes = [_pd, _sz, _d, _i, _d, _d, _sz, _sz, _pd, _pd, _psz, _sz, _psz]
        L.ref_sync_run_f32.argtypes = [_pd, _sz, _d, _i, _d, _d, _sz, _pd]
        L.ref_async_run.argtypes = [_pd, _sz, _d, _i, _d, _d, _sz, _i, _sz, _sz, _d, _u64, _sz, _sz,
                                    _pd, _pd, _psz, _sz, _psz]
        L.ref_delay_stream.argtypes = [_i, _sz, _sz, _d, _u64, _sz, _sz, _pu64]
        L.ref_exec_run.argtypes = [_pd, _sz, _d, _i, _d, _d, _sz, _sz, _sz, _i, _i, _pd, _pu64, _pu64]
        L.ref_exec_run_reps.argtypes = [_pd, _sz, _d, _i, _d, _d, _sz, _sz, _sz, _i, _sz, _pu64,
                                         _pd]
        L.ref_sync_step_into_loop.argtypes = [_pd, _pd, _sz, _d, _i, _d, _d, _sz]
        L.ref_sync_step_into_loop.restype = _u64
        L.ref_prepare_initial.argtypes = [_pd, _sz, _i, _d, _d, _pd]
        L.ref_cosine_init.argtypes = [_sz, _pd]
        L.ref_async_step.argtypes = [_pd, _sz, _sz, _sz, _sz, _d, _i, _d, _d, _sz, _sz, _i, _sz,
                                     _sz, _d, _pu64, _pd]
        L.ref_hardware_concurrency.restype = C.c_uint

    def set_strict(self, on: bool):
        self.lib.ref_set_strict(int(on))

    def ensemble_run(self, u0, r, bc, c1, c2, per_pe, law, q, fixed_d, k_end, stride, runs,
                     base_seed, p=0.5):
        """heat::ensemble_run -> (steps, norms[runs][S], terminals[runs][n], mean, std, spread2)."""
        L = self.lib
        if not getattr(L.ref_ensemble_run, "argtypes", None):
            L.ref_ensemble_run.argtypes = [_pd, _sz, _d, _i, _d, _d, _sz, _i, _sz, _sz, _d, _sz,
                                           _sz, _sz, _u64, _psz, _psz, _pd, _pd, _pd, _pd, _pd]
        u0 = _f64(u0)
        n = u0.size
        s_ = stride if stride else (1 if n <= 1000 else 100)
        cap = 2 + k_end // s_
        steps = np.zeros(cap, np.uintp)
        ns = C.c_size_t(0)
        norms = np.zeros(runs * cap)
        terms = np.zeros((runs, n))
        mean = np.zeros(cap)
        std = np.zeros(cap)
        spread = np.zeros(2)
        st = L.ref_ensemble_run(_ptr(u0), n, r, bc, c1, c2, per_pe, law, q, fixed_d, p, k_end,
                                stride, runs, base_seed, _ptr(steps, _psz), C.byref(ns), _ptr(norms),
                                _ptr(terms), _ptr(mean), _ptr(std), _ptr(spread))
        if st:
            raise OracleError(st, "ensemble_run")
        S = ns.value
        return ([int(x) for x in steps[:S]], norms[:runs * S].reshape(runs, S), terms,
                mean[:S], std[:S], spread)

    def checked_r(self, alpha, dt, dx) -> float:
        r = C.c_double(0)
        st = self.lib.ref_params_checked_r(alpha, dt, dx, C.byref(r))
        if st:
            raise OracleError(st, "SolverParams::checked")
        return r.value

    def hardware_concurrency(self) -> int:
        return int(self.lib.ref_hardware_concurrency())

    def cosine_init(self, n) -> np.ndarray:
        out = np.empty(n, np.float64)
        st = self.lib.ref_cosine_init(n, _ptr(out))
        if st:
            raise OracleError(st, "cosine_init")
        return out

    def prepare_initial(self, u0, bc=DIRICHLET, c1=0.0, c2=0.0) -> np.ndarray:
        u0 = _f64(u0)
        out = np.empty_like(u0)
        st = self.lib.ref_prepare_initial(_ptr(u0), u0.size, bc, c1, c2, _ptr(out))
        if st:
            raise OracleError(st, "prepare_initial")
        return out

    def delay_stream(self, law, q, fixed_d, p, seed, k, count) -> list[int]:
        out = np.empty(count, np.uint64)
        st = self.lib.ref_delay_stream(law, q, fixed_d, p, seed, k, count, _ptr(out, _pu64))
        if st:
            raise OracleError(st, "delay_stream")
        return [int(x) for x in out]

    def sync_step(self, u, r, bc=DIRICHLET, c1=0.0, c2=0.0) -> np.ndarray:
        u = _f64(u)
        out = np.empty_like(u)
        st = self.lib.ref_sync_step(_ptr(u), u.size, r, bc, c1, c2, _ptr(out))
        if st:
            raise OracleError(st, "sync_step")
        return out

    def sync_run(self, u0, r, bc=DIRICHLET, c1=0.0, c2=0.0, k_end=1, stride=None, record=False):
        u0 = _f64(u0)
        n = u0.size
        fin = np.empty(n, np.float64)
        stride_v = stride if stride is not None else (k_end or 1)
        s = stride_v if stride_v else (1 if n <= 1000 else 100)
        cap = (k_end // s + 2) if record else 0
        snaps = np.empty((cap, n), np.float64) if record else None
        steps = np.empty(cap, np.uintp) if record else None
        ns = C.c_size_t(0)
        st = self.lib.ref_sync_run(_ptr(u0), n, r, bc, c1, c2, k_end, stride_v, _ptr(fin),
                                   _ptr(snaps), _ptr(steps, _psz), cap, C.byref(ns))
        if st:
            raise OracleError(st, "sync_run")
        if record:
            return [int(x) for x in steps[:ns.value]], snaps[:ns.value].copy()
        return fin

    def sync_run_f32(self, u0, r, bc=DIRICHLET, c1=0.0, c2=0.0, k_end=1):
        u0 = _f64(u0)
        fin = np.empty(u0.size, np.float64)
        st = self.lib.ref_sync_run_f32(_ptr(u0), u0.size, r, bc, c1, c2, k_end, _ptr(fin))
        if st:
            raise OracleError(st, "sync_run_f32")
        return fin

    def async_run(self, u0, r, bc, c1, c2, per_pe, law, q, fixed_d=0, p=0.5, seed=0, k_end=1,
                  stride=None, record=False):
        u0 = _f64(u0)
        n = u0.size
        fin = np.empty(n, np.float64)
        stride_v = stride if stride is not None else (k_end or 1)
        s = stride_v if stride_v else (1 if n <= 1000 else 100)
        cap = (k_end // s + 2) if record else 0
        snaps = np.empty((cap, n), np.float64) if record else None
        steps = np.empty(cap, np.uintp) if record else None
        ns = C.c_size_t(0)
        st = self.lib.ref_async_run(_ptr(u0), n, r, bc, c1, c2, per_pe, law, q, fixed_d, p, seed,
                                    k_end, stride_v, _ptr(fin), _ptr(snaps), _ptr(steps, _psz),
                                    cap, C.byref(ns))
        if st:
            raise OracleError(st, "async_run")
        if record:
            return [int(x) for x in steps[:ns.value]], snaps[:ns.value].copy()
        return fin

    def async_step(self, snaps, depth, step, r, bc, c1, c2, part_total, per_pe, law, q,
                   fixed_d=0, p=0.5, rng_state=0):
        """heat::async_step itself on a HistoryRing rebuilt at `step`; returns
        (status, field or None, rng state after the call)."""
        snaps = np.ascontiguousarray(np.asarray(snaps, np.float64))
        count, n = snaps.shape
        out = np.empty(n, np.float64)
        st_rng = C.c_uint64(rng_state)
        st = self.lib.ref_async_step(_ptr(snaps), count, depth, step, n, r, bc, c1, c2,
                                     part_total, per_pe, law, q, fixed_d, p, C.byref(st_rng),
                                     _ptr(out))
        return st, (out if st == 0 else None), int(st_rng.value)

    def exec_run(self, u0, r, bc, c1, c2, per_pe, workers, k_end, mode=BARRIERED,
                 record_lag=False):
        u0 = _f64(u0)
        fin = np.empty(u0.size, np.float64)
        dur = C.c_uint64(0)
        lag = np.zeros(70, np.uint64)
        st = self.lib.ref_exec_run(_ptr(u0), u0.size, r, bc, c1, c2, per_pe, workers, k_end, mode,
                                   int(record_lag), _ptr(fin), C.byref(dur), _ptr(lag, _pu64))
        if st:
            raise OracleError(st, "exec_run")
        return fin, int(dur.value), lag

    def exec_run_reps(self, u0, r, bc, c1, c2, per_pe, workers, k_end, mode, reps,
                      want_final=False):
        """exec_run called `reps` times on one field: (durations_ns list, final or None)."""
        u0 = _f64(u0)
        durs = np.zeros(reps, np.uint64)
        fin = np.empty(u0.size, np.float64) if want_final else None
        st = self.lib.ref_exec_run_reps(_ptr(u0), u0.size, r, bc, c1, c2, per_pe, workers, k_end,
                                        mode, reps, _ptr(durs, _pu64), _ptr(fin))
        if st:
            raise OracleError(st, "exec_run")
        return [int(x) for x in durs], fin

    def sync_step_into_loop(self, u_prepared, r, bc, c1, c2, k):
        """Runs detail::sync_step_into k times; returns (field, loop_ns)."""
        a = np.array(u_prepared, dtype=np.float64, copy=True)
        ns = self.lib.ref_sync_step_into_loop(_ptr(a), _ptr(None), a.size, r, bc, c1, c2, k)
        return a, int(ns)


_port = None
_ref = None


def port() -> Port:
    global _port
    with _lock:
        if _port is None:
            _port = Port.__new__(Port)
    if not hasattr(_port, "lib"):
        Port.__init__(_port)
    return _port


def ref() -> Ref:
    global _ref
    with _lock:
        if _ref is None:
            _ref = Ref.__new__(Ref)
    if not hasattr(_ref, "lib"):
        Ref.__init__(_ref)
    return _ref
