#!/bin/bash
export PYTHONPATH=.
timeout 900 python -m pytest -x -q tests/test_gpu_k7c.py tests/test_gpu_sync.py tests/test_gpu_async.py 2>&1 | tail -5
