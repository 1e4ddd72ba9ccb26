#!/bin/bash
# Interleaved bench A/B of a runtime knob (LP_TUNE_<KEY> env).  usage: bash scripts/ab_knob.sh KEY v1 v2 ...
KEY=$1; shift
run() { timeout 600 env LP_TUNE_${KEY}=$1 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'value': round(d['value'],4), 'sm_mhz': d['clocks']['sm_mhz'], 'tflops': {k: round(v['tflops']) for k, v in d['kernels'].items()}}))"; }
for rep in 1 2; do for v in "$@"; do echo "[$KEY=$v] $(run $v)"; done; done
