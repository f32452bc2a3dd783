#!/bin/bash
export PYTHONPATH=.
mkdir -p gpurun_out
rm -f gpurun_out/k9c.ncu-rep
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"async_small|sync_small_cl" -c 2 -o gpurun_out/k9c python tools/k7_k9_once.py > gpurun_out/ncu_k9c.log 2>&1
ncu -i gpurun_out/k9c.ncu-rep --page source --csv --print-source sass > gpurun_out/k9c_src.csv 2>/dev/null
ncu -i gpurun_out/k9c.ncu-rep --page raw --csv > gpurun_out/k9c_raw.csv 2>/dev/null
ncu -i gpurun_out/k9c.ncu-rep --page details --csv > gpurun_out/k9c_details.csv 2>/dev/null
