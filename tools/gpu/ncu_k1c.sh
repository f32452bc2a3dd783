set -x
export PYTHONPATH=.
HEAT_SYNC_VARIANT=18 timeout 300 ncu --set full --import-source on --clock-control none -k regex:sync_cta -c 1 -o gpurun_out/k1c python tools/probe_sync.py 268435456 64 > gpurun_out/ncu_k1c.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:exec_free -c 1 -o gpurun_out/k10v2_100_4 python tools/k10_once.py 100 4 20000 > gpurun_out/ncu_k10v2.log 2>&1
