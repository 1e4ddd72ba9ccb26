#!/bin/bash
# Interleaved C2 bench A/B of prebuilt library variants (ab/liblp_<v>.so), bench only, R rounds.
# usage: bash scripts/ab_so_bench.sh TAG ROUNDS v0 v1 ...   (output gpurun_out/TAG/ab.txt)
TAG=$1; R=$2; shift 2
P=paper_2512_07350_b200/liblp_b200.so
O=gpurun_out/$TAG; mkdir -p $O
cp $P $O/.orig.so
for rep in $(seq $R); do for v in "$@"; do
  cp ab/liblp_$v.so $P
  timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', json.dumps({'value': round(d['value'],4), 'sm_mhz': d['clocks']['sm_mhz'], 'tflops': {k: round(v['tflops']) for k, v in d['kernels'].items()}}))"
done; done 2>&1 | tee $O/ab.txt
cp $O/.orig.so $P && rm $O/.orig.so
