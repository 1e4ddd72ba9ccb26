#!/bin/bash
# compute-sanitizer over the hand-written kernels at small shapes (SURVEY §5 race detection):
# memcheck / racecheck / synccheck on the GEMM, attention, K1, K10, toy denoisers, a 1-block
# DiT forward through the engine, and the peer (CUDA-IPC) exchange with 2 ranks.
# usage: bash scripts/sanitize.sh OUTDIR
O=${1:-gpurun_out/sanitize}
mkdir -p $O
T="tests/test_dit_gpu.py::test_gemm_matches_torch tests/test_dit_gpu.py::test_attention_matches_torch
   tests/test_lp_gpu.py::test_extract_bitexact tests/test_lp_gpu.py::test_reconstruct_and_update_bitexact
   tests/test_lp_gpu.py::test_toy_denoisers_bitexact tests/test_dit_gpu.py::test_engine_dit_step_runs"
P="tests/test_peer_exchange_gpu.py::test_peer_exchange_toy_bitexact_vs_oracle"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 50 --error-exitcode 99 \
     python -m pytest -m gpu -q -x -p no:cacheprovider $T > $O/$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $O/status
  tail -4 $O/$tool.log
done
timeout 900 compute-sanitizer --tool memcheck --target-processes all --print-limit 50 --error-exitcode 99 \
   python -m pytest -m gpu -q -x -p no:cacheprovider "$P" > $O/memcheck_peer.log 2>&1
echo "memcheck_peer rc=$?" | tee -a $O/status; tail -4 $O/memcheck_peer.log
