export PYTHONPATH=.
HEAT_SYNC_VARIANT=20 timeout 900 python -m pytest tests/test_gpu_sync.py tests/test_gpu_streamed.py tests/test_gpu_huge.py -q -x > gpurun_out/k1s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k1s_tests.log
VARIANTS="15 20 21 22 15 20" bash tools/ab_sync.sh > gpurun_out/ab_k1s.txt 2>&1
