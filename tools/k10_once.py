"""One exec_run(BarrierFree) call for ncu: N P K [stats]."""
import ctypes as C
import sys

import numpy as np

from paper_1510_08982_b200 import _lib
from paper_1510_08982_b200 import heat as H

N, P, K = (int(x) for x in sys.argv[1:4])
stats = len(sys.argv) > 4 and sys.argv[4] == "stats"
lib = _lib.lib()
u0 = H.cosine_init(N).values()
out = np.empty_like(u0)
dur = C.c_uint64(0)
st = _lib.AsyncStatsC()
_lib.check(lib.heat_exec_run(_lib.dptr(u0), N, 0.5, 0, 1.0, 0.0, N // P, P, K, 1, 0, 0,
                             _lib.dptr(out), C.byref(dur), None, C.byref(st) if stats else None),
           "exec_run")
print(N, P, K, stats, dur.value / K, "ns/step")
