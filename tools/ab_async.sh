#!/bin/bash
# A/B of K5 (async_stream_kernel) done-signals per release fence (HEAT_K5_PEND)
# at N=2^30, 512 PEs, free q=8.  Each config is its own process (the knob is
# read once).   usage: tools/ab_async.sh "2 4 8" [steps]
PENDS=${1:-"2 8"}
STEPS=${2:-1024}
for pend in $PENDS; do
  echo "== PEND=$pend"
  PYTHONPATH=. HEAT_K5_PEND=$pend python tools/probe_async.py $((1 << 30)) $STEPS 512 8
done
