#!/bin/bash
# r4v: cross-attention q RMSNorm folded into attention (dit_xq_rms): DiT tests (floor parity,
# oracle, 14B shape, single-pass predict), the C2 full-size LP step vs the reference, in-step A/B
O=gpurun_out/r4v; mkdir -p $O
timeout 1500 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_dit_gpu.py tests/test_parity_schedule_gpu.py tests/test_integration_gpu.py > $O/pytest.log 2>&1
rc=$?; echo "tests rc=$rc" | tee -a $O/status; tail -2 $O/pytest.log; [ $rc -ne 0 ] && { grep -E "^E |FAILED" $O/pytest.log | head -20; exit 0; }
bash scripts/ab_knob.sh DIT_XQ_RMS 1 0 > $O/ab.txt 2>&1; bash scripts/ab_knob.sh DIT_XQ_RMS 1 0 >> $O/ab.txt 2>&1; cat $O/ab.txt
