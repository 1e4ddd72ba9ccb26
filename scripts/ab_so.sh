#!/bin/bash
# Interleaved A/B of prebuilt library variants on one box.  Build each variant here first, e.g.
#   LP_NVCC_EXTRA="-DFLAG=0" python -m paper_2512_07350_b200.build && cp paper_2512_07350_b200/liblp_b200.so ab/liblp_v0.so
# then: bash scripts/ab_so.sh TAG v0 v1   (standalone kbench [KB_ARGS, default "attn"] + C2 bench,
# two rounds; output in gpurun_out/TAG/ab.txt).  The default build is restored at the end.
TAG=$1; shift
P=paper_2512_07350_b200/liblp_b200.so
O=gpurun_out/$TAG; mkdir -p $O
cp $P $O/.orig.so
for rep in 1 2; do for v in "$@"; do
  cp ab/liblp_$v.so $P
  echo "== $v"
  timeout 300 python scripts/kbench.py ${KB_ARGS:-attn} 2>&1 | grep "{" | python -c "
import sys, json
for l in sys.stdin:
    d=json.loads(l); k=list(d)[0]; x=d[k]; print('  ', k, round(x['tflops']))"
  timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  bench', json.dumps({'value': round(d['value'],4), 'sm_mhz': d['clocks']['sm_mhz'], 'reasons': d['clocks']['reasons'], 'tflops': {k: round(v['tflops']) for k, v in d['kernels'].items()}}))"
done; done 2>&1 | tee $O/ab.txt
cp $O/.orig.so $P && rm $O/.orig.so
