set -x
export PYTHONPATH=.
timeout 300 ncu --set full --import-source on --clock-control none -k regex:exec_free -c 1 -o gpurun_out/k10v3_100_4 python tools/k10_once.py 100 4 20000 > gpurun_out/ncu_k10v3a.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:exec_free -c 1 -o gpurun_out/k10v3_10000_4 python tools/k10_once.py 10000 4 2000 > gpurun_out/ncu_k10v3b.log 2>&1
