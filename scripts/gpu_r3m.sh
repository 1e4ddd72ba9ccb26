#!/bin/bash
# r3m: cross-attention instance probe: NT=1 persistent (default) vs NT=2 persistent (attn_nt1=0,
# attn_persist=2, which also makes self-attention persistent); fold test with the fold on
O=gpurun_out/r3m; mkdir -p $O
LP_TUNE_DIT_LNFOLD=1 timeout 900 python -m pytest -m gpu -q -p no:cacheprovider tests/test_dit_gpu.py -k "lnfold or forward" > $O/pytest_fold.log 2>&1; echo "fold tests rc=$?" | tee -a $O/status; tail -2 $O/pytest_fold.log
timeout 900 python -m pytest -m gpu -q -p no:cacheprovider tests/test_hybrid_gpu.py > $O/pytest_hybrid.log 2>&1; echo "hybrid tests rc=$?" | tee -a $O/status; tail -2 $O/pytest_hybrid.log
run() { timeout 600 env $2 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', json.dumps({'value': round(d['value'],4), 'sm_mhz': d['clocks']['sm_mhz'], 'tflops': {k: round(v['tflops']) for k, v in d['kernels'].items()}, 'ms': {k: round(v['ms'],1) for k, v in d['kernels'].items()}}))"; }
for rep in 1 2; do
  run default "LP_TUNE_X=0"; run cross_nt2p "LP_TUNE_ATTN_NT1=0 LP_TUNE_ATTN_PERSIST=2"; run nt1_nopersist "LP_TUNE_ATTN_PERSIST=0"
done 2>&1 | tee $O/ab.txt
