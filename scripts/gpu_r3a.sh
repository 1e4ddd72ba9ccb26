#!/bin/bash
# Round-2 first validation pass: smoke, all GPU tests, bench (ours), reference arm (1 whole step)
O=gpurun_out/r3a
mkdir -p $O
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt 2>&1
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/status
tail -3 $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/status
tail -15 $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" | tee -a $O/status
cut -c1-1500 $O/bench.json; tail -5 $O/bench.err
timeout 1500 python bench.py --impl reference --ref-steps 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench_ref rc=$?" | tee -a $O/status
cut -c1-1500 $O/bench_ref.json; tail -5 $O/bench_ref.err
