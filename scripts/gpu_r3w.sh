#!/bin/bash
# r3w: attention p_half/p_full one arrive per softmax warp vs per thread
O=gpurun_out/r3w; mkdir -p $O
timeout 600 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_dit_gpu.py -k "attention" > $O/pytest.log 2>&1
rc=$?; echo "tests rc=$rc" | tee -a $O/status; tail -2 $O/pytest.log; [ $rc -ne 0 ] && exit 0
KB_ARGS="attn" bash scripts/ab_so.sh r3w wa1 wa0
