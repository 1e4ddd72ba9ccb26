#!/bin/bash
# ncu evidence for the current build: launch list of a bench run + --set full captures of
# the top kernels, mid-step.  usage: bash scripts/ncu_round.sh TAG
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 3 --warmup 1 --no-cpu-baseline > $O/ncu_bench.log 2>&1; echo "launch-list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_attention -s 40 -c 1 -o $O/attn_full \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_attn.log 2>&1; echo "attn rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm2 -s 400 -c 2 -o $O/gemm_full \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_gemm.log 2>&1; echo "gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_layernorm|k_rmsnorm|k_reconstruct|k_slice" -s 60 -c 4 -o $O/hbm_full \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu_hbm.log 2>&1; echo "hbm rc=$?"
