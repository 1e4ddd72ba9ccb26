#!/bin/bash
# Interleaved bench A/B over several compile-time variants on one box.
# usage: bash scripts/ab_multi.sh "FLAGS_A" "FLAGS_B" ...   (each run twice, interleaved)
run() { timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'value': round(d['value'],4), 'sm_mhz': d['clocks']['sm_mhz'], 'tflops': {k: round(v['tflops']) for k, v in d['kernels'].items()}}))"; }
for rep in 1 2; do
  for f in "$@"; do
    LP_NVCC_EXTRA="$f" python -c "from paper_2512_07350_b200 import build; build.build()" > /dev/null
    echo "[$f] $(run)"
  done
done
python -c "from paper_2512_07350_b200 import build; build.build()" > /dev/null
