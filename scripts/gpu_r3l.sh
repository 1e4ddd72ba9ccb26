#!/bin/bash
# r3l: LN fold v2 (shifted-sum partials, TMA-staged xq): DiT/hybrid/parity tests with the fold ON,
# then the interleaved in-step A/B
O=gpurun_out/r3l; mkdir -p $O
LP_TUNE_DIT_LNFOLD=1 timeout 1500 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_dit_gpu.py tests/test_hybrid_gpu.py tests/test_parity_schedule_gpu.py > $O/pytest_fold.log 2>&1
rc=$?; echo "fold tests rc=$rc" | tee -a $O/status; tail -3 $O/pytest_fold.log
if [ $rc -ne 0 ]; then grep -E "^E |Error" $O/pytest_fold.log | head -20; fi
bash scripts/ab_knob.sh DIT_LNFOLD 0 1 > $O/ab_lnfold.txt 2>&1; cat $O/ab_lnfold.txt
