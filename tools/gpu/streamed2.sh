#!/bin/bash
export PYTHONPATH=.
timeout 900 python -m pytest -x -q tests/test_gpu_streamed.py 2>&1 | tail -2
HEAT_STREAM_TRACE=1 timeout 300 python tools/pageable_trace.py 2>&1
cat > /tmp/pt1000.py <<'PY'
import time, numpy as np
from paper_1510_08982_b200 import _lib
n = 1 << 30
u = np.sin(np.pi * np.arange(n, dtype=np.float64) / (n - 1)); u[-1] = 0.0
out = np.empty(n); out[:] = 0.0
L = _lib.lib()
for i in range(3):
    t0 = time.perf_counter()
    _lib.check(L.heat_sync_run(_lib.dptr(u), n, 0.4, 0, 0.0, 0.0, 1000, 1000, _lib.dptr(out), None, None, 0, None), "x")
    print(f"pageable 1000 steps: {time.perf_counter() - t0:.3f} s", flush=True)
PY
HEAT_STREAM_TRACE=1 timeout 300 python /tmp/pt1000.py 2>&1
