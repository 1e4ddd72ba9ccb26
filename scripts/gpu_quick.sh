#!/bin/bash
# Quick GPU validation of a change: the named GPU tests, then a short bench (N=1) and the
# self-launched N=2 bench on one GPU (gloo plumbing).  usage: bash scripts/gpu_quick.sh TAG "pytest args"
TAG=${1:-q}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest ${2:-tests} -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/status
tail -3 $O/pytest_gpu.log
if [ "$3" != "skip-bench" ]; then
  timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" | tee -a $O/status
  cut -c1-600 $O/bench.json
fi
