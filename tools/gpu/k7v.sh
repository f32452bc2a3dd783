#!/bin/bash
export PYTHONPATH=.
for v in 8 4; do
  HEAT_K7C_V=$v timeout 600 python -m pytest -x -q tests/test_gpu_k7c.py 2>&1 | tail -1 | sed "s/^/V=$v /"
  HEAT_K7C_V=$v timeout 120 python tools/probe_cfg1.py | sed "s/^/V=$v /"
done
