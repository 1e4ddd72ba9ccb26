#!/bin/bash
# r3f: K1 TMA fix (16-byte aligned box starts) + K10 W-axis tile kernel + LN fold default off:
# targeted tests, the whole GPU suite, smoke, HBM replay bench, one bench line, then r3d's
# C4/C5 / N=2 / ncu work.
O=gpurun_out/r3f
mkdir -p $O
timeout 900 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_lp_gpu.py -k "tma or extract or w_axis or reconstruct" > $O/pytest_k1k10.log 2>&1
echo "k1/k10 tests rc=$?" | tee -a $O/status; tail -3 $O/pytest_k1k10.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/status
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/status
tail -5 $O/pytest_gpu.log
HB_TAG=_wt timeout 600 python scripts/hbm_bench.py 4 > $O/hbm_wt.log 2>&1; mv gpurun_out/hbm_bench_wt.json $O/
LP_TUNE_RECON_WT=0 HB_TAG=_xs timeout 600 python scripts/hbm_bench.py 4 > $O/hbm_xs.log 2>&1; mv gpurun_out/hbm_bench_xs.json $O/
python - <<'PY'
import json
a=json.load(open('gpurun_out/r3f/hbm_bench_wt.json'))['rows']; b=json.load(open('gpurun_out/r3f/hbm_bench_xs.json'))['rows']
for x,y in zip(a,b): print(x['config'],x['axis'],'k1 %.1fus %.2f || k10 wt %.1fus %.2f | xs %.1fus %.2f | fast %.2f'%(x['k1_us'],x['k1_frac'],x['k10_us'],x['k10_frac'],y['k10_us'],y['k10_frac'],x['k10_fast_frac']))
PY
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" | tee -a $O/status
python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['step'], d['clocks']); print({k:(v['GBps'],v['frac_of_hbm']) for k,v in d['hbm_kernels'].items() if isinstance(v,dict) and 'GBps' in v})"
HB_NCU=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gather|k_reconstruct" \
   -o $O/hbm_full python scripts/hbm_bench.py 4 > $O/ncu_hbm.log 2>&1; echo "ncu-hbm rc=$?" | tee -a $O/status
bash scripts/gpu_r3d.sh
