#!/bin/bash
# r3n: K10 W-axis rows in flight (recon_u 4 vs 8)
O=gpurun_out/r3n; mkdir -p $O
timeout 900 python -m pytest -m gpu -q -p no:cacheprovider tests/test_lp_gpu.py -k "w_axis" > $O/pytest_w.log 2>&1; echo "w tests rc=$?" | tee -a $O/status; tail -2 $O/pytest_w.log
for u in 4 8; do LP_TUNE_RECON_U=$u HB_TAG=_u$u timeout 600 python scripts/hbm_bench.py 4 > $O/hbm_u$u.log 2>&1; mv gpurun_out/hbm_bench_u$u.json $O/; done
python - <<'PY'
import json
a=json.load(open('gpurun_out/r3n/hbm_bench_u4.json'))['rows']; b=json.load(open('gpurun_out/r3n/hbm_bench_u8.json'))['rows']
for x,y in zip(a,b):
    if x['axis']=='W': print(x['config'],'W k10 u4 %.1fus %.2f fast %.2f | u8 %.1fus %.2f fast %.2f'%(x['k10_us'],x['k10_frac'],x['k10_fast_frac'],y['k10_us'],y['k10_frac'],y['k10_fast_frac']))
PY
