#!/bin/bash
# r4i: TMEM-resident-Q CTA-pair attention (attn_qtm): correctness, standalone, in-step
O=gpurun_out/r4i; mkdir -p $O
timeout 600 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_dit_gpu.py -k "cta_pair or large_logits" > $O/pytest.log 2>&1
rc=$?; echo "tests rc=$rc" | tee -a $O/status; tail -3 $O/pytest.log; [ $rc -ne 0 ] && { grep -E "^E " $O/pytest.log | head -20; exit 0; }
for rep in 1 2; do for v in 0 1; do
  LP_TUNE_ATTN_QTM=$v timeout 300 python scripts/kbench.py attn > $O/kb_${v}_$rep.log 2>&1
  echo "qtm=$v rep=$rep: $(grep -o '"tflops": [0-9.]*' $O/kb_${v}_$rep.log | tr '\n' ' ')" | tee -a $O/status
done; done
bash scripts/ab_knob.sh ATTN_QTM 0 1 > $O/ab.txt 2>&1; cat $O/ab.txt
