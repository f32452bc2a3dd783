"""Host-side phases of a pageable-buffer heat_sync_run at cfg3 (N = 2^30,
10^4 steps) against the pinned one: HEAT_STREAM_TRACE=1 prints them."""
import time

import numpy as np
import torch

from paper_1510_08982_b200 import _lib
from paper_1510_08982_b200 import heat as H

n = 1 << 30
K = 10000
r = 0.4
u = np.sin(np.pi * np.arange(n, dtype=np.float64) / (n - 1))
u[-1] = 0.0
out = np.empty(n)
out[:] = 0.0
L = _lib.lib()
for i in range(2):
    t0 = time.perf_counter()
    _lib.check(L.heat_sync_run(_lib.dptr(u), n, r, 0, 0.0, 0.0, K, K, _lib.dptr(out), None, None,
                               0, None), "sync_run")
    print(f"pageable run {i}: {time.perf_counter() - t0:.3f} s", flush=True)
pin_in = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
pin_out = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
pin_in[:] = u
for i in range(2):
    t0 = time.perf_counter()
    _lib.check(L.heat_sync_run(_lib.dptr(pin_in), n, r, 0, 0.0, 0.0, K, K, _lib.dptr(pin_out), None,
                               None, 0, None), "sync_run")
    print(f"pinned run {i}: {time.perf_counter() - t0:.3f} s", flush=True)
