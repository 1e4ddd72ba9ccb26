#!/bin/bash
# compute-sanitizer over this round's new kernel forms at small shapes: K1 TMA boxes (W) and bulk
# copies (T/H), K10 branch-free W kernel (xsb), the CTA-pair attention, the LN-fold v2 GEMM
# epilogue (TMA-staged xq). memcheck + synccheck + racecheck.
O=${1:-gpurun_out/sanitize_r3}
mkdir -p $O
T="tests/test_lp_gpu.py::test_extract_tma_paths_bitexact tests/test_lp_gpu.py::test_reconstruct_w_axis_bitexact
   tests/test_dit_gpu.py::test_attention_cta_pair_matches_torch"
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 50 --error-exitcode 99 \
     python -m pytest -m gpu -q -x -p no:cacheprovider $T -k "not dims0 and not dims3 and not shape3" > $O/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $O/status
  tail -3 $O/$tool.log
done
LP_TUNE_DIT_LNFOLD=1 timeout 900 compute-sanitizer --tool memcheck --target-processes all --print-limit 50 --error-exitcode 99 \
   python -m pytest -m gpu -q -x -p no:cacheprovider "tests/test_dit_gpu.py::test_lnfold_matches_layernorm_path_and_oracle" > $O/memcheck_lnfold.log 2>&1
echo "memcheck_lnfold rc=$?" | tee -a $O/status; tail -3 $O/memcheck_lnfold.log
