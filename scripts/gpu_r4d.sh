#!/bin/bash
# r4d: CTA-pair attention ring depths (in-step, attn_pair=1) vs the single-CTA default
O=gpurun_out/r4d; mkdir -p $O
P=paper_2512_07350_b200/liblp_b200.so; cp $P $O/.orig.so
run() { cp ab/liblp_$1.so $P; timeout 600 env LP_TUNE_ATTN_PAIR=$2 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 pair=$2', json.dumps({'value': round(d['value'],4), 'sm_mhz': d['clocks']['sm_mhz'], 'tflops': {k: round(v['tflops']) for k, v in d['kernels'].items()}}))"; }
for rep in 1 2; do run p44 0; run p44 1; run p33 1; run p64 1; done 2>&1 | tee $O/ab.txt
cp $O/.orig.so $P
