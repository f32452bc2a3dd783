#!/bin/bash
export PYTHONPATH=.
mkdir -p gpurun_out
rm -f gpurun_out/ens.ncu-rep
timeout 120 python tools/probe_ensemble.py
timeout 300 ncu --set full --import-source on --clock-control none -k regex:ensemble_ -c 1 -o gpurun_out/ens python tools/ens_once.py 20000 > gpurun_out/ncu_ens.log 2>&1
ncu -i gpurun_out/ens.ncu-rep --page source --csv --print-source sass > gpurun_out/ens_src.csv 2>/dev/null
ncu -i gpurun_out/ens.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,smsp__issue_active.avg.pct_of_peak_sustained_active > gpurun_out/ens_raw.csv 2>/dev/null
