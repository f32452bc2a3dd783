#!/bin/bash
# A/B of K5 (async_stream_kernel) knobs at N=2^30, 512 PEs, free q=8:
# HEAT_K5_PEND (done-signals per release fence) x HEAT_K5_PREF (issue step of
# the next window).  Each config is its own process (the knobs are read once).
# usage: tools/ab_async.sh "2 4 8" "-1 4 8" [steps]
PENDS=${1:-"2 8"}
PREFS=${2:-"-1 4"}
STEPS=${3:-1024}
for pend in $PENDS; do
  for pref in $PREFS; do
    echo "== PEND=$pend PREF=$pref"
    PYTHONPATH=. HEAT_K5_PEND=$pend HEAT_K5_PREF=$pref python tools/probe_async.py $((1 << 30)) $STEPS 512 8
  done
done
