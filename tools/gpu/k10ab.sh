export PYTHONPATH=.
for s in ${LIBS:-v2 ""}; do echo "lib=$s"; HEAT_LIB_SUFFIX=$s timeout 300 python tools/probe_k10.py 2>&1 | cat; done > gpurun_out/k10ab.txt 2>&1
