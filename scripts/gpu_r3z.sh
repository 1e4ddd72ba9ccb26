#!/bin/bash
# r3z: GEMM two K sub-blocks per stage (gemm_ksub=2): tests, GEMM microbench, in-step A/B
O=gpurun_out/r3z; mkdir -p $O
timeout 600 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_dit_gpu.py -k "gemm" > $O/pytest.log 2>&1
rc=$?; echo "tests rc=$rc" | tee -a $O/status; tail -2 $O/pytest.log; [ $rc -ne 0 ] && { grep -E "^E " $O/pytest.log | head; exit 0; }
for rep in 1 2; do for v in 1 2; do
  LP_TUNE_GEMM_KSUB=$v KB_ROWS=28080 timeout 300 python scripts/kbench.py gemm epi > $O/kb_$v_$rep.log 2>&1
  echo "ksub=$v rep=$rep: $(grep -o '"gemm_[a-z0-9_]*": {"M": [0-9]*, "N": [0-9]*, "K": [0-9]*[^}]*"tflops": [0-9.]*' $O/kb_$v_$rep.log | sed -E 's/"M".*"tflops": / /' | tr '\n' ' ')" | tee -a $O/status
done; done
bash scripts/ab_knob.sh GEMM_KSUB 1 2 > $O/ab.txt 2>&1; cat $O/ab.txt
