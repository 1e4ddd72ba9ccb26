#!/bin/bash
# r3v: ncu --set full of the CTA-pair GEMMs after the tempty handshake change (kbench shapes)
O=gpurun_out/r3v; mkdir -p $O
M=sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.avg.pct_of_peak_sustained_elapsed
KB_ROWS=28080 timeout 900 ncu --set full --metrics $M --clock-control none --import-source on -k regex:k_gemm2 -c 40 -o $O/gemm python scripts/kbench.py gemm epi > $O/ncu.log 2>&1; echo "gemm rc=$?" | tee -a $O/status
