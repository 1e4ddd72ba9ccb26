#!/bin/bash
# r3t: GEMM tempty handshake (one plain remote arrive per warp vs release.cluster per thread),
# GEMM microbench + C2 bench A/B; CTA-pair attention with plain remote arrivals
O=gpurun_out/r3t; mkdir -p $O
timeout 600 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_dit_gpu.py -k "gemm or attention or forward" > $O/pytest.log 2>&1
rc=$?; echo "tests rc=$rc" | tee -a $O/status; tail -2 $O/pytest.log; [ $rc -ne 0 ] && exit 0
KB_ARGS="gemm epi" bash scripts/ab_so.sh r3t tw1 tw0
for rep in 1 2; do for v in 0 1; do
  LP_TUNE_ATTN_PAIR=$v timeout 300 python scripts/kbench.py attn > $O/kbp_$v_$rep.log 2>&1
  echo "pair=$v rep=$rep: $(grep -o '"tflops": [0-9.]*' $O/kbp_$v_$rep.log | tr '\n' ' ')" | tee -a $O/status
done; done
