export PYTHONPATH=.
for rep in 1 2; do timeout 300 python tools/probe_k10.py 2>&1 | grep "N=   100\|N=  1000"; done > gpurun_out/k10w.txt
timeout 600 python -m pytest tests/test_gpu_exec_free.py tests/test_gpu_acceptance.py -q -x > gpurun_out/k10w_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k10w_tests.log
