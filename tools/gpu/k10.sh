set -x
export PYTHONPATH=.
timeout 300 python tools/probe_k10.py > gpurun_out/probe_k10.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_exec_free.py -x -q > gpurun_out/k10_tests.log 2>&1; echo "k10 tests rc=$?"
HEAT_SYNC_VARIANT=18 timeout 600 python -m pytest tests/test_gpu_sync.py tests/test_gpu_streamed.py -x -q > gpurun_out/k1c_tests.log 2>&1; echo "k1c tests rc=$?"
tail -3 gpurun_out/k1c_tests.log
VARIANTS="15 18 19" bash tools/ab_sync.sh > gpurun_out/ab_k1c.txt 2>&1
