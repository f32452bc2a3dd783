"""K10 (exec_run BarrierFree, one cluster) vs K7 (Barriered) per-step device
time over the shapes the reference's measure() sweep uses, with and without
the delay statistics (async_exec.cpp:281-307)."""
import ctypes as C
import sys

import numpy as np

from paper_1510_08982_b200 import _lib
from paper_1510_08982_b200 import heat as H

lib = _lib.lib()
K = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
Q = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # exec_run's q_free (0: the default)


def run(N, P, mode, stats, q=Q):
    u0 = H.cosine_init(N).values()
    out = np.empty_like(u0)
    dur = C.c_uint64(0)
    st = _lib.AsyncStatsC()
    ts = []
    for _ in range(5):
        _lib.check(lib.heat_exec_run(_lib.dptr(u0), N, 0.5, 0, 1.0, 0.0, N // P, P, K, mode, 0, q,
                                     _lib.dptr(out), C.byref(dur), None,
                                     C.byref(st) if stats else None), "exec_run")
        ts.append(dur.value)
    return sorted(ts)[2] / K


for P in (4, 5, 10, 20):
    for N in (100, 1000, 10000):
        if N % P:
            continue
        geo = [C.c_int(0) for _ in range(5)]
        ok = lib.heat_free_geometry(N, N // P, Q or 8, *[C.byref(x) for x in geo]) == 0
        geo = [x.value for x in geo]
        b = run(N, P, 0, False)
        f = run(N, P, 1, False)
        fs = run(N, P, 1, True)
        print(f"P={P:2d} N={N:6d} K10={'y' if ok else 'n'} geo={geo} barriered {b:7.1f} ns/step"
              f"  free {f:7.1f}  free+stats {fs:7.1f}  ratio {b / f:5.2f}", flush=True)
