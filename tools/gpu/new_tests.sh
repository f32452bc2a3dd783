export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_async.py tests/test_gpu_concurrency.py tests/test_gpu_simulator.py -q -x > gpurun_out/new_tests.log 2>&1; echo "rc=$?" >> gpurun_out/new_tests.log
for i in 1 2 3 4 5; do timeout 300 python -m pytest tests/test_gpu_xlink_ipc.py -q 2>&1 | tail -1; done > gpurun_out/ipc_flake.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
