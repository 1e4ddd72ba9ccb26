#!/bin/bash
# r3c: LN fold + TMA K1 validation: all GPU tests, interleaved A/B of dit_lnfold, hbm bench
# (gather_tma on/off), one bench line.
O=gpurun_out/r3c
mkdir -p $O
timeout 600 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_lp_gpu.py -k "tma or extract" > $O/pytest_tma.log 2>&1
rc=$?; echo "tma tests rc=$rc" | tee -a $O/status; tail -3 $O/pytest_tma.log
if [ $rc -ne 0 ]; then export LP_TUNE_GATHER_TMA=0; echo "K1 TMA disabled for the rest" | tee -a $O/status; fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $O/status
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $O/status
tail -15 $O/pytest_gpu.log
bash scripts/ab_knob.sh DIT_LNFOLD 1 0 > $O/ab_lnfold.txt 2>&1; cat $O/ab_lnfold.txt
HB_TAG=_tma timeout 600 python scripts/hbm_bench.py 4 > $O/hbm_tma.log 2>&1; mv gpurun_out/hbm_bench_tma.json $O/
LP_TUNE_RECON_G=8 HB_TAG=_g8 timeout 600 python scripts/hbm_bench.py 4 > $O/hbm_g8.log 2>&1; mv gpurun_out/hbm_bench_g8.json $O/
grep '"C2"' $O/hbm_g8.log | cut -c1-330
LP_TUNE_GATHER_TMA=0 LP_TUNE_RECON_MK=0 HB_TAG=_vec timeout 600 python scripts/hbm_bench.py 4 > $O/hbm_vec.log 2>&1; mv gpurun_out/hbm_bench_vec.json $O/
python - <<'PY'
import json
a=json.load(open('gpurun_out/r3c/hbm_bench_tma.json'))['rows']; b=json.load(open('gpurun_out/r3c/hbm_bench_vec.json'))['rows']
for x,y in zip(a,b): print(x['config'],x['axis'],'k1 tma %.1fus %.2f | vec %.1fus %.2f || k10 mk %.1fus %.2f | div %.1fus %.2f | fast %.2f'%(x['k1_us'],x['k1_frac'],y['k1_us'],y['k1_frac'],x['k10_us'],x['k10_frac'],y['k10_us'],y['k10_frac'],x['k10_fast_frac']))
PY
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" | tee -a $O/status
python -c "import json;d=json.load(open('$O/bench.json'));print(d['value'], d['roofline']['step'], json.dumps(d['hbm_kernels'])[:1200])"
HB_NCU=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gather|k_reconstruct" \
   -o $O/hbm_full python scripts/hbm_bench.py 4 > $O/ncu_hbm.log 2>&1; echo "ncu-hbm rc=$?" | tee -a $O/status
