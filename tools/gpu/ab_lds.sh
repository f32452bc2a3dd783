export PYTHONPATH=.
for rep in 1 2; do for lib in old ""; do echo "lib=$lib"; HEAT_LIB_SUFFIX=$lib timeout 300 python tools/probe_async.py 1073741824 1024 2>&1 | tail -3; done; done > gpurun_out/ab_lds.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_sync.py tests/test_gpu_streamed.py tests/test_gpu_async.py tests/test_gpu_stream_geometry.py tests/test_gpu_xdevice.py -q -x > gpurun_out/lds_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lds_tests.log
