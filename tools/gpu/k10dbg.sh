export PYTHONPATH=.
for d in ${DBGS:-0 3}; do echo "dbg=$d"; HEAT_K10_DBG=$d timeout 300 python tools/probe_k10.py 2>&1 | grep "N=  1000" ; done > gpurun_out/k10dbg.txt
timeout 600 python -m pytest tests/test_gpu_exec_free.py -q > gpurun_out/k10_tests.log 2>&1; echo "k10 tests rc=$?" >> gpurun_out/k10dbg.txt
