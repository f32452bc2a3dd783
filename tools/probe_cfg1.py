"""BASELINE configs[0] through the public API: sync_run N=1024, r=0.25,
Dirichlet 0/0, sine profile, 1000 steps with the default trajectory stride
(1 for N <= 1000, else 100), best of 30; the C-ABI call alone; and the
per-step cost at 20000 steps."""
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
L = _lib.lib()


def best(fn, reps=30):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e6


stride = H.default_stride(n)
print(f"sync_run cfg1 api k=1000 stride={stride}: {best(lambda: H.sync_run(f, p, bc, 1000, stride).final()):.1f} us")
fin = np.empty(n)
print(f"sync_run cfg1 C   k=1000 final:     {best(lambda: H.sync_final(u0, p, bc, 1000)):.1f} us")
t = best(lambda: H.sync_final(u0, p, bc, 20000), 5)
print(f"sync_run cfg1 k=20000: {t:.1f} us, {t / 20000 * 1e3:.1f} ns/step")
bp = H.BoundaryCondition.periodic()
t = best(lambda: H.sync_final(u0, p, bp, 20000), 5)
print(f"sync_run cfg1-periodic k=20000: {t:.1f} us, {t / 20000 * 1e3:.1f} ns/step")
