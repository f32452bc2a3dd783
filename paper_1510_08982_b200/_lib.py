"""ctypes binding of the C-ABI in include/heat_b200.h.

The shared library is built in-tree (``python -m paper_1510_08982_b200.build``)
and loaded from the package directory.  There is no CPU fallback: if the
library is missing or no B200 is visible, calls raise ``NativeUnavailable``.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
# HEAT_LIB_SUFFIX=x loads libheat_b200_x.so from the package (A/B builds only)
LIB_PATH = os.path.join(
    PKG, "libheat_b200" + ("_" + os.environ["HEAT_LIB_SUFFIX"] if os.environ.get("HEAT_LIB_SUFFIX") else "")
    + ".so")

HEAT_OK = 0
HEAT_EDOMAIN = 1
HEAT_EINVAL = 2
HEAT_ELOGIC = 3
HEAT_EDIVERGE = 4
HEAT_ECUDA = 5
HEAT_ETIMEOUT = 6
HEAT_ENOMEM = 7
HEAT_ENODEV = 8

BC_DIRICHLET = 0
BC_PERIODIC = 1
DELAY_UNIFORM, DELAY_FIXED, DELAY_GEOMETRIC = 0, 1, 2
EXEC_BARRIERED, EXEC_BARRIER_FREE = 0, 1


class HeatError(RuntimeError):
    """Base class; `.status` carries the C-ABI status code."""

    status = -1


class DomainError(HeatError, ValueError):
    """std::domain_error"""


class InvalidArgument(HeatError, ValueError):
    """std::invalid_argument"""


class LogicError(HeatError):
    """std::logic_error"""


class DivergenceError(HeatError):
    """heat::DivergenceError (a std::runtime_error)"""


class CudaError(HeatError):
    """CUDA runtime failure (std::runtime_error)"""


class WatchdogTimeout(HeatError):
    """An async halo-ring wait exceeded its deadline."""


class NativeUnavailable(HeatError):
    """The CUDA library is missing or no sm_100 device is visible."""


_EXC = {
    HEAT_EDOMAIN: DomainError,
    HEAT_EINVAL: InvalidArgument,
    HEAT_ELOGIC: LogicError,
    HEAT_EDIVERGE: DivergenceError,
    HEAT_ECUDA: CudaError,
    HEAT_ETIMEOUT: WatchdogTimeout,
    HEAT_ENOMEM: CudaError,
    HEAT_ENODEV: NativeUnavailable,
}


class LagStatsC(C.Structure):
    _fields_ = [("reads", C.c_uint64), ("min_lag", C.c_uint64), ("max_lag", C.c_uint64),
                ("overflow", C.c_uint64), ("histogram", C.c_uint64 * 64)]


class AsyncStatsC(C.Structure):
    _fields_ = [("reads", C.c_uint64), ("max_delay", C.c_uint64),
                ("delay_histogram", C.c_uint64 * 64), ("waits", C.c_uint64),
                ("residual_sum", C.c_double)]


_P = C.POINTER
_d, _sz, _i, _u64, _vp = C.c_double, C.c_size_t, C.c_int, C.c_uint64, C.c_void_p
_pd, _psz, _pu64 = _P(C.c_double), _P(C.c_size_t), _P(C.c_uint64)

# name -> (restype, argtypes); mirrors include/heat_b200.h exactly.
SIGNATURES = {
    "heat_last_error": (C.c_char_p, []),
    "heat_version": (C.c_char_p, []),
    "heat_device_count": (_i, []),
    "heat_set_device": (_i, [_i]),
    "heat_kernel_launches": (_u64, []),
    "heat_sync_kernel_info": (_i, [C.POINTER(_i), C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)]),
    "heat_stream_chunk_plan": (_i, [_sz, _sz, _P(_sz), _sz, _P(_sz)]),
    "heat_k3_geometry": (_i, [_sz, _sz, _sz, _i, _P(_i), _P(_i), _P(_sz), _P(_i)]),
    "heat_k5_geometry": (_i, [_sz, _P(_i), _P(_i)]),
    "heat_free_geometry": (_i, [_sz, _sz, _sz, _P(_i), _P(_i), _P(_i), _P(_i), _P(_i)]),
    "heat_geometric_thresholds": (_i, [_d, _sz, _pu64]),
    "heat_set_strict_finite_checks": (None, [_i]),
    "heat_strict_finite_checks": (_i, []),
    "heat_prepare_initial": (_i, [_pd, _sz, _i, _d, _d, _pd]),
    "heat_trajectory_length": (_sz, [_sz, _sz, _sz]),
    "heat_sync_step": (_i, [_pd, _sz, _d, _i, _d, _d, _pd]),
    "heat_sync_run": (_i, [_vp, _sz, _d, _i, _d, _d, _sz, _sz, _vp, _vp, _vp, _sz, _vp]),
    "heat_sync_run_f32": (_i, [_vp, _sz, _d, _i, _d, _d, _sz, _sz, _vp, _vp, _vp, _sz, _vp]),
    "heat_async_run": (_i, [_vp, _sz, _d, _i, _d, _d, _sz, _sz, _i, _sz, _d, _u64, _sz, _sz,
                            _vp, _vp, _vp, _sz, _vp]),
    "heat_sample_delay": (_i, [_sz, _i, _sz, _d, _u64, _u64, _sz, _psz]),
    "heat_async_free_run": (_i, [_pd, _sz, _d, _i, _d, _d, _sz, _sz, _sz, _pd, _P(AsyncStatsC)]),
    "heat_ensemble_run": (_i, [_pd, _sz, _d, _i, _d, _d, _sz, _sz, _i, _sz, _d, _sz, _sz, _sz, _u64,
                               _psz, _sz, _psz, _pd, _pd, _pd, _pd]),
    "heat_exec_run": (_i, [_pd, _sz, _d, _i, _d, _d, _sz, _sz, _sz, _i, _i, _sz, _pd, _pu64,
                           _P(LagStatsC), _P(AsyncStatsC)]),
    "heat_async_sim_create": (_i, [_P(_vp), _pd, _sz, _d, _i, _d, _d, _sz, _sz, _i, _sz, _d,
                                   _u64]),
    "heat_async_sim_step": (_i, [_vp, _sz]),
    "heat_history_create": (_i, [_P(_vp), _sz, _sz, _sz, _pd, _sz, _i]),
    "heat_history_destroy": (_i, [_vp]),
    "heat_history_info": (_i, [_vp, _psz, _psz, _psz]),
    "heat_history_push": (_i, [_vp, _pd, _sz]),
    "heat_history_read": (_i, [_vp, _sz, _sz, _pd]),
    "heat_history_snapshot": (_i, [_vp, _sz, _pd]),
    "heat_async_step": (_i, [_vp, _d, _i, _d, _d, _sz, _sz, _sz, _i, _sz, _d, _pu64, _pd, _i]),
    "heat_async_sim_current": (_i, [_vp, _pd, _P(_sz)]),
    "heat_async_sim_destroy": (_i, [_vp]),
    "heat_plan_create": (_i, [_P(_vp), _sz, _i]),
    "heat_plan_destroy": (_i, [_vp]),
    "heat_plan_set_stream": (_i, [_vp, _vp]),
    "heat_plan_upload": (_i, [_vp, _vp]),
    "heat_plan_download": (_i, [_vp, _vp]),
    "heat_plan_download_device": (_i, [_vp, _vp]),
    "heat_plan_download_range": (_i, [_vp, _sz, _sz, _vp]),
    "heat_plan_fill_sine": (_i, [_vp]),
    "heat_plan_sync_advance": (_i, [_vp, _d, _i, _d, _d, _sz]),
    "heat_plan_async_advance": (_i, [_vp, _d, _i, _d, _d, _sz, _sz, _sz, _P(AsyncStatsC)]),
    "heat_plan_async_replay": (_i, [_vp, _d, _i, _d, _d, _sz, _sz, _i, _sz, _d, _u64, _sz,
                                    _P(AsyncStatsC)]),
    "heat_plan_synchronize": (_i, [_vp]),
    "heat_plan_device_ptr": (_i, [_vp, _P(_vp)]),
    "heat_slab_halo": (_sz, []),
    "heat_plan_create_slab": (_i, [_P(_vp), _sz, _i, _i, _i]),
    "heat_plan_halo_pack": (_i, [_vp, _vp]),
    "heat_plan_halo_unpack": (_i, [_vp, _vp]),
    "heat_xlink_handle_size": (_sz, []),
    "heat_plan_xlink_setup": (_i, [_vp, _sz, _sz, _i, _vp]),
    "heat_plan_xlink_connect": (_i, [_vp, _vp, _vp]),
    "heat_plan_xlink_seed": (_i, [_vp]),
    "heat_plan_xlink_advance": (_i, [_vp, _d, _d, _d, _i, _i, _sz, _d, _u64, _sz,
                                     _P(AsyncStatsC)]),
    "heat_plan_xlink_debug_recv": (_i, [_vp, _pd]),
}

_lib = None
_lock = threading.Lock()


def lib() -> C.CDLL:
    """Load libheat_b200.so (raises NativeUnavailable when it is not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} is not built; run `python -m paper_1510_08982_b200.build` "
                    "(there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(status: int, what: str = "") -> None:
    if status == HEAT_OK:
        return
    msg = lib().heat_last_error().decode(errors="replace")
    exc = _EXC.get(status, HeatError)(f"{what}: {msg}" if what else msg)
    exc.status = status
    raise exc


def dptr(a: np.ndarray | None):
    return C.cast(None, _pd) if a is None else a.ctypes.data_as(_pd)


def szptr(a: np.ndarray | None):
    return C.cast(None, _psz) if a is None else a.ctypes.data_as(_psz)
