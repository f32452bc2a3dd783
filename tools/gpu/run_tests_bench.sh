export PYTHONPATH=.
set -x
nproc; lscpu | head -20 > gpurun_out/lscpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ref1.json 2> gpurun_out/ref1.err; echo "ref rc=$?"
