export PYTHONPATH=.
timeout 300 ncu --set full --import-source on --clock-control none -k regex:exec_free -c 1 -o gpurun_out/k10t python tools/k10_once.py 100 10 20000 > gpurun_out/ncu_k10t.log 2>&1
