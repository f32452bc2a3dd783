#!/bin/bash
# Round-end evidence: GPU tests, the bench line, the reference arm, smoke, and
# the ncu launch list of a short bench command (run after the plain one).
export PYTHONPATH=.
mkdir -p gpurun_out
nproc; lscpu | head -20 > gpurun_out/lscpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputests.log
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ref_f.json 2> gpurun_out/ref_f.err; echo "ref rc=$?"
timeout 600 python bench.py --steps 2 --warmup 1 --skip-e2e --skip-bound --skip-cpu > gpurun_out/b_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_f.csv \
    python bench.py --steps 2 --warmup 1 --skip-e2e --skip-bound --skip-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu rc=$?"
