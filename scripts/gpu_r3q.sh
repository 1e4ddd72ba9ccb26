#!/bin/bash
# r3q: attention MMA warp waiting for the whole P (attn_pwhole=1: one barrier check per tile and
# key block instead of two)
O=gpurun_out/r3q; mkdir -p $O
LP_TUNE_ATTN_PWHOLE=1 timeout 600 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_dit_gpu.py -k "attention" > $O/pytest_attn.log 2>&1
rc=$?; echo "attn tests (pwhole=1) rc=$rc" | tee -a $O/status; tail -2 $O/pytest_attn.log
[ $rc -ne 0 ] && exit 0
for rep in 1 2; do for v in 0 1; do
  LP_TUNE_ATTN_PWHOLE=$v timeout 300 python scripts/kbench.py attn > $O/kb_$v_$rep.log 2>&1
  echo "pwhole=$v rep=$rep: $(grep -o '"tflops": [0-9.]*' $O/kb_$v_$rep.log | tr '\n' ' ')" | tee -a $O/status
done; done
bash scripts/ab_knob.sh ATTN_PWHOLE 0 1 > $O/ab.txt 2>&1; cat $O/ab.txt
