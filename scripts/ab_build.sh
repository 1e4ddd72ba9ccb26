#!/bin/bash
# A/B of a compile-time variant on one box: bench with the default build (A), with
# LP_NVCC_EXTRA="$1" (B), then A again.  usage: bash scripts/ab_build.sh "-DFLAG" [bench args]
FLAG="$1"; shift
run() { timeout 600 python bench.py --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'value': round(d['value'],4), 'sm_mhz': d['clocks']['sm_mhz'], 'reasons': d['clocks']['reasons'], 'tflops': {k: round(v['tflops']) for k, v in d['kernels'].items()}}))"; }
echo "A: $(run "$@")"
LP_NVCC_EXTRA="$FLAG" python -c "from paper_2512_07350_b200 import build; build.build()" > /dev/null
echo "B $FLAG: $(run "$@")"
python -c "from paper_2512_07350_b200 import build; build.build()" > /dev/null
echo "A: $(run "$@")"
