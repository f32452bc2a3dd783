export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_streamed.py tests/test_gpu_sync.py -q -x > gpurun_out/streamed_tests.log 2>&1; echo "rc=$?" >> gpurun_out/streamed_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --skip-bound > gpurun_out/bench3.json 2> gpurun_out/bench3.err
