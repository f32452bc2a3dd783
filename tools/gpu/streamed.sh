#!/bin/bash
export PYTHONPATH=.
timeout 900 python -m pytest -x -q tests/test_gpu_streamed.py tests/test_gpu_sync.py 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err; echo "bench rc=$?"
