#!/bin/bash
# r4f: row-order reversal of the LayerNorm / q/k RMSNorm passes (row_rev): identity test + in-step A/B
O=gpurun_out/r4f; mkdir -p $O
timeout 600 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_dit_gpu.py -k "row_order or forward" > $O/pytest.log 2>&1
rc=$?; echo "tests rc=$rc" | tee -a $O/status; tail -2 $O/pytest.log; [ $rc -ne 0 ] && exit 0
bash scripts/ab_knob.sh ROW_REV 0 1 > $O/ab.txt 2>&1; bash scripts/ab_knob.sh ROW_REV 0 1 >> $O/ab.txt 2>&1; cat $O/ab.txt
