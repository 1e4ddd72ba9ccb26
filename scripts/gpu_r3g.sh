#!/bin/bash
# r3g: CTA-pair self-attention (attn_pair): correctness, standalone A/B, in-step A/B
O=gpurun_out/r3g
mkdir -p $O
timeout 600 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_dit_gpu.py -k "attention" > $O/pytest_attn.log 2>&1
rc=$?; echo "attn tests rc=$rc" | tee -a $O/status; tail -3 $O/pytest_attn.log
if [ $rc -ne 0 ]; then grep -E "Error|assert" $O/pytest_attn.log | head -20; exit 0; fi
for rep in 1 2; do for v in 0 1; do
  LP_TUNE_ATTN_PAIR=$v KB_TAG=_pair$v timeout 300 python scripts/kbench.py attn > $O/kb_pair${v}_$rep.log 2>&1
  echo "pair=$v rep=$rep: $(grep -o '"tflops": [0-9.]*' $O/kb_pair${v}_$rep.log | tr '\n' ' ')" | tee -a $O/status
done; done
bash scripts/ab_knob.sh ATTN_PAIR 0 1 > $O/ab_pair.txt 2>&1; cat $O/ab_pair.txt
