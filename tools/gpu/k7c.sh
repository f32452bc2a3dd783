#!/bin/bash
# K7c: parity, cfg1 timings (cluster / one CTA / old K7), criterion-8 table.
export PYTHONPATH=.
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_sync.py tests/test_gpu_acceptance.py tests/test_gpu_concurrency.py tests/test_gpu_exec_free.py 2>&1 | tail -3
timeout 120 python tools/probe_cfg1.py
HEAT_K7_NO_CLUSTER=1 timeout 120 python tools/probe_cfg1.py | sed 's/^/one-cta /'
HEAT_NO_K7C=1 timeout 120 python tools/probe_cfg1.py | sed 's/^/old-k7 /'
timeout 300 python tools/probe_k10.py 2>&1 | tail -12
