export PYTHONPATH=.
timeout 300 python tools/probe_k10.py > gpurun_out/probe_k10.txt 2>&1
