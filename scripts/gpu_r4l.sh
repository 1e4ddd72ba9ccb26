#!/bin/bash
# r4l: GELU epilogue with packed f32x2 math vs scalar: GEMM tests, kbench ffn1_gelu, in-step A/B
O=gpurun_out/r4l; mkdir -p $O
timeout 600 python -m pytest -m gpu -q -x -p no:cacheprovider tests/test_dit_gpu.py -k "gemm or forward" > $O/pytest.log 2>&1
rc=$?; echo "tests rc=$rc" | tee -a $O/status; tail -2 $O/pytest.log; [ $rc -ne 0 ] && { grep -E "^E " $O/pytest.log | head; exit 0; }
KB_ARGS="gemm epi" bash scripts/ab_so.sh r4l g2 g1 > /dev/null 2>&1
grep -E "==|gelu|bench" gpurun_out/r4l/ab.txt
bash scripts/ab_so_bench.sh r4l2 2 g2 g1 > /dev/null 2>&1; cat gpurun_out/r4l2/ab.txt
