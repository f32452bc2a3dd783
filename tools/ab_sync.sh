#!/bin/bash
# A/B the compile-time K1 variants on one GPU (device-timed probe at N=2^30).
for v in ${VARIANTS:-4 6 7 8}; do
  echo "variant $v"; HEAT_SYNC_VARIANT=$v PYTHONPATH=. python tools/probe_sync.py 1073741824 ${STEPS:-1024} 2>&1 | tail -4
done
