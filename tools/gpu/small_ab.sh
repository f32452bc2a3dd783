#!/bin/bash
# K7c + K9 parity and cfg1/cfg2 timings
export PYTHONPATH=.
timeout 900 python -m pytest -x -q tests/test_gpu_k7c.py tests/test_gpu_async.py tests/test_gpu_sync.py 2>&1 | tail -2
timeout 120 python tools/probe_cfg1.py
timeout 120 python tools/probe_cfg2.py
