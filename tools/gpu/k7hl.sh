#!/bin/bash
export PYTHONPATH=.
for hl in 8 10 12; do
  HEAT_K7C_HL=$hl timeout 600 python -m pytest -x -q tests/test_gpu_k7c.py 2>&1 | tail -1 | sed "s/^/HL=$hl /"
  HEAT_K7C_HL=$hl timeout 120 python tools/probe_cfg1.py | sed "s/^/HL=$hl /"
done
