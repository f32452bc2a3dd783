#!/bin/bash
export PYTHONPATH=.
timeout 900 python -m pytest -x -q tests/test_gpu_async.py tests/test_gpu_ensemble.py tests/test_gpu_acceptance.py tests/test_gpu_history.py 2>&1 | tail -1
timeout 300 python tools/probe_member_vs_k3.py
HEAT_NO_MEMBER_ASYNC=1 timeout 300 python tools/probe_member_vs_k3.py | sed 's/^/k3 /'
