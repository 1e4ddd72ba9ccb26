#!/bin/bash
# r3h: K10 W-axis tile kernel v2 (warp per position, lane = row) + CTA-pair attention
O=gpurun_out/r3h
mkdir -p $O
timeout 900 python -m pytest -m gpu -q -p no:cacheprovider tests/test_lp_gpu.py -k "w_axis or reconstruct or nonfinite" > $O/pytest_k10.log 2>&1
echo "k10 tests rc=$?" | tee -a $O/status; tail -3 $O/pytest_k10.log
HB_TAG=_wt timeout 600 python scripts/hbm_bench.py 4 > $O/hbm_wt.log 2>&1; mv gpurun_out/hbm_bench_wt.json $O/
python - <<'PY'
import json
a=json.load(open('gpurun_out/r3h/hbm_bench_wt.json'))['rows']
for x in a: print(x['config'],x['axis'],'k1 %.1fus %.2f || k10 %.1fus %.2f | fast %.2f'%(x['k1_us'],x['k1_frac'],x['k10_us'],x['k10_frac'],x['k10_fast_frac']))
PY
HB_NCU=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_reconstruct_wt" \
   -o $O/wt_full python scripts/hbm_bench.py 4 > $O/ncu_wt.log 2>&1; echo "ncu-wt rc=$?" | tee -a $O/status
bash scripts/gpu_r3g.sh
