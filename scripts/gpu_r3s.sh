#!/bin/bash
# r3s: ncu --set full of the CTA-pair attention vs the single-CTA kernel at the C2 K=4 max shard
O=gpurun_out/r3s; mkdir -p $O
M=sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum,sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.avg.pct_of_peak_sustained_elapsed
LP_TUNE_ATTN_PAIR=1 timeout 600 ncu --set full --metrics $M --clock-control none --import-source on -k regex:k_attention -c 2 -o $O/pair python scripts/kbench.py attn > $O/ncu_pair.log 2>&1; echo "pair rc=$?" | tee -a $O/status
timeout 600 ncu --set full --metrics $M --clock-control none --import-source on -k regex:k_attention -c 2 -o $O/single python scripts/kbench.py attn > $O/ncu_single.log 2>&1; echo "single rc=$?" | tee -a $O/status
