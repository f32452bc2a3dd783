#!/bin/bash
export PYTHONPATH=.
timeout 600 python -m pytest -x -q tests/test_gpu_async.py tests/test_gpu_concurrency.py 2>&1 | tail -1
for i in 1 2; do
  timeout 120 python tools/probe_cfg2.py
  HEAT_K9_NO_WS=1 timeout 120 python tools/probe_cfg2.py | sed 's/^/no-ws /'
done
timeout 120 python tools/probe_k9_sizes.py
HEAT_K9_NO_WS=1 timeout 120 python tools/probe_k9_sizes.py | sed 's/^/no-ws /'
