#!/bin/bash
# r3i: K10 W-axis branch-free x-stationary kernel (recon_xsb)
O=gpurun_out/r3i
mkdir -p $O
timeout 900 python -m pytest -m gpu -q -p no:cacheprovider tests/test_lp_gpu.py -k "w_axis or reconstruct or nonfinite" > $O/pytest_k10.log 2>&1
echo "k10 tests rc=$?" | tee -a $O/status; tail -3 $O/pytest_k10.log
for v in 1 0; do
LP_TUNE_RECON_XSB=$v HB_TAG=_xsb$v timeout 600 python scripts/hbm_bench.py 4 > $O/hbm_xsb$v.log 2>&1; mv gpurun_out/hbm_bench_xsb$v.json $O/
done
python - <<'PY'
import json
a=json.load(open('gpurun_out/r3i/hbm_bench_xsb1.json'))['rows']; b=json.load(open('gpurun_out/r3i/hbm_bench_xsb0.json'))['rows']
for x,y in zip(a,b): print(x['config'],x['axis'],'k10 xsb %.1fus %.2f fast %.2f | xs %.1fus %.2f'%(x['k10_us'],x['k10_frac'],x['k10_fast_frac'],y['k10_us'],y['k10_frac']))
PY
HB_NCU=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_reconstruct_xs" \
   -o $O/xsb_full python scripts/hbm_bench.py 4 > $O/ncu_xsb.log 2>&1; echo "ncu rc=$?" | tee -a $O/status
