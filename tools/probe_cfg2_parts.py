"""Where a cfg2 async_run call's time goes: the public API, the bare C-ABI call
(same arguments, arrays allocated once), the C call without the trajectory,
and a 1-step call (fixed cost).  Best of 50 each."""
import ctypes as C
import time

import numpy as np

from paper_1510_08982_b200 import _lib
from paper_1510_08982_b200 import heat as H

n = 1024
u0 = np.sin(np.pi * np.arange(n) / (n - 1))
u0[-1] = 0.0
f = H.TemperatureField(u0)
p = H.SolverParams.from_r(0.25)
bc = H.BoundaryCondition.dirichlet(0.0, 0.0)
part = H.PartitionSpec(n, n // 8)
m = H.DelayModel.uniform(2, 1)
L = _lib.lib()
v = np.ascontiguousarray(f.values())
fin = np.empty(n)


def best(fn, reps=50):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e6


def c_call(k, stride, traj):
    count = L.heat_trajectory_length(n, k, stride)
    snaps = np.empty((count, n))
    steps = np.empty(count, np.uintp)
    ns = C.c_size_t(0)

    def go():
        _lib.check(L.heat_async_run(_lib.dptr(v), n, p.r(), bc.kind, bc.c1, bc.c2, n // 8,
                                    *m._args(), k, stride,
                                    _lib.dptr(fin) if not traj else C.cast(None, _lib._pd),
                                    _lib.dptr(snaps) if traj else None,
                                    _lib.szptr(steps) if traj else None, count if traj else 0,
                                    C.byref(ns)), "async_run")
    return go


print(f"api  k=1000 stride=100: {best(lambda: H.async_run(f, p, bc, part, m, 1000, 100).final()):.1f} us")
print(f"C    k=1000 stride=100: {best(c_call(1000, 100, True)):.1f} us")
print(f"C    k=1000 final only: {best(c_call(1000, 1000, False)):.1f} us")
print(f"C    k=1    final only: {best(c_call(1, 1, False)):.1f} us")
print(f"C    k=64   final only: {best(c_call(64, 64, False)):.1f} us")
print(f"sync k=1    final only: {best(lambda: H.sync_final(u0, p, bc, 1)):.1f} us")
