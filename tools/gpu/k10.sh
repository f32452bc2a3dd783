export PYTHONPATH=.
timeout 300 python tools/probe_k10.py > gpurun_out/probe_k10.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_exec_free.py -q > gpurun_out/k10_tests.log 2>&1; echo "k10 tests rc=$?"
