#!/bin/bash
# One GPU validation pass: smoke, GPU tests, bench (both arms), ncu launch list + a full capture
# of the top kernel.  Outputs land in gpurun_out/ (merged back by gpurun).
# usage: bash scripts/gpu_round.sh TAG [skip-tests] [skip-ncu]
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/status
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/status
  tail -3 $O/pytest_gpu.log
fi
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" | tee -a $O/status
cat $O/bench.json
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench_ref rc=$?" | tee -a $O/status
cat $O/bench_ref.json
if [ "$3" != "skip-ncu" ]; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
      python bench.py --steps 3 --warmup 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "ncu-launch rc=$?" | tee -a $O/status
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_attention -s 40 -c 1 -o $O/attn_full \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu-full-attn rc=$?" | tee -a $O/status
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_gemm2 -s 150 -c 2 -o $O/gemm_full \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_full_gemm.log 2>&1; echo "ncu-full-gemm rc=$?" | tee -a $O/status
fi
