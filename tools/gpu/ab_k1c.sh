export PYTHONPATH=.
for lib in "" nr; do for v in 15 18; do echo "lib=$lib variant=$v"; HEAT_LIB_SUFFIX=$lib HEAT_SYNC_VARIANT=$v timeout 300 python tools/probe_sync.py 1073741824 1024 2>&1 | tail -2 | head -1; done; done > gpurun_out/ab_k1c.txt 2>&1
