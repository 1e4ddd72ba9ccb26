#!/bin/bash
# A/B of an attention compile-time variant: correctness tests + standalone attention + C2 bench,
# interleaved.  usage: bash scripts/ab_attn.sh "FLAGS_B"
for f in "" "$1"; do
  LP_NVCC_EXTRA="$f" python -c "from paper_2512_07350_b200 import build; build.build()" > /dev/null
  echo "== [$f] $(timeout 300 python -m pytest tests/test_dit_gpu.py -q -x -k 'attention or forward' 2>&1 | tail -1)"
  timeout 300 python scripts/kbench.py attn 2>&1 | grep "{" | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); k=list(d)[0]; v=d[k]; print('  ', k, round(v['tflops']), 'sdpa', round(v['sdpa_tflops']))"
done
bash scripts/ab_multi.sh "" "$1"
