#!/bin/bash
# K9: parity of the async tests, then cfg2 timings (cluster and one CTA).
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q tests/test_gpu_async.py 2>&1 | tail -3
timeout 600 python -m pytest -x -q tests/test_gpu_sync.py tests/test_gpu_acceptance.py tests/test_gpu_concurrency.py 2>&1 | tail -3
timeout 120 python tools/probe_cfg2_parts.py
HEAT_K9_NO_CLUSTER=1 timeout 120 python tools/probe_cfg2_parts.py | sed 's/^/one-cta /'
timeout 120 python tools/probe_cfg2.py
HEAT_K9_NO_CLUSTER=1 timeout 120 python tools/probe_cfg2.py | sed 's/^/one-cta /'
(cd tools/micro && ./call_floor && HEAT_K9_NO_CLUSTER=1 ./call_floor | grep heat_async | sed 's/^/one-cta /')
