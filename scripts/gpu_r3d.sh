#!/bin/bash
# r3d: C4 / C5 through bench.py (clocks, roofline, e2e), the self-launched 2-rank bench on one GPU
# (gloo plumbing, peer exchange), the launch list + tcgen05-aware full captures of attention and
# the GEMMs at C2.
O=gpurun_out/r3d
mkdir -p $O
for c in c4 c5; do
  timeout 1200 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
  echo "bench $c rc=$?" | tee -a $O/status
  python -c "import json;d=json.load(open('$O/bench_$c.json'));print('$c', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['step'], d['clocks'])"
done
LP_BENCH_GLOO_TEST=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_n2_gloo.json 2> $O/bench_n2_gloo.err
echo "bench n2 gloo rc=$?" | tee -a $O/status; cut -c1-600 $O/bench_n2_gloo.json
M=sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.avg.pct_of_peak_sustained_elapsed
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 3 --warmup 1 --no-cpu-baseline --hbm-iters 1 --hbm-sets 1 > $O/ncu_bench.log 2>&1; echo "ncu-launch rc=$?" | tee -a $O/status
timeout 1200 ncu --set full --metrics $M --clock-control none --import-source on -k regex:k_attention -s 40 -c 2 -o $O/attn_full \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --hbm-iters 1 --hbm-sets 1 > $O/ncu_full.log 2>&1; echo "ncu-full-attn rc=$?" | tee -a $O/status
timeout 1200 ncu --set full --metrics $M --clock-control none --import-source on -k regex:k_gemm2 -s 150 -c 4 -o $O/gemm_full \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --hbm-iters 1 --hbm-sets 1 > $O/ncu_full_gemm.log 2>&1; echo "ncu-full-gemm rc=$?" | tee -a $O/status
