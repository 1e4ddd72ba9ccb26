#!/bin/bash
# r3u: CTA-pair self-attention with plain remote arrivals, in-step A/B (3 rounds)
O=gpurun_out/r3u; mkdir -p $O
run() { timeout 600 env LP_TUNE_ATTN_PAIR=$1 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pair=$1', json.dumps({'value': round(d['value'],4), 'sm_mhz': d['clocks']['sm_mhz'], 'tflops': {k: round(v['tflops']) for k, v in d['kernels'].items()}, 'step_frac': round(d['roofline']['step']['frac'],3)}))"; }
for rep in 1 2 3; do run 0; run 1; done 2>&1 | tee $O/ab.txt
