"""Run scripts/micro/libmma_bench.so: cycles per tcgen05.mma per operand mode (all 148 SMs busy)."""
import ctypes as C
import json
import sys

import torch

L = C.CDLL("scripts/micro/libmma_bench.so")
out = torch.zeros(4, dtype=torch.int64, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
names = {0: "SS N128 (S=QK^T)", 1: "TS N128 B MN-major (PV)", 2: "SS N256", 3: "SS N64", 4: "TS N128 B K-major",
         5: "SS N128 B MN-major", 6: "SS N128 x2 sharing B", 7: "PV(TS) then S over P's columns (WAR)",
         8: "PV(TS) then S into other columns", 9: "SS N128 + commit per 8 MMAs", 10: "SS N128 + commit per 2 MMAs",
         11: "SS N128 + tcgen05.fence::after_thread_sync per 4 MMAs", 12: "SS N128 + try_wait(done)+fence per 4 MMAs",
         13: "SS N128 + test_wait(done)+fence per 4", 14: "SS N128 + try_wait(done) no fence per 4",
         15: "SS N128 + volatile smem flag poll+fence per 4"}
N = {0: 128, 1: 128, 2: 256, 3: 64, 4: 128, 5: 128, 6: 256, 7: 256, 8: 256, 9: 128, 10: 128, 11: 128, 12: 128, 13: 128, 14: 128, 15: 128}
res = {}
for mode in [0, 12, 13, 14, 15, 32]:
    iters = 200
    for rep in range(3):
        assert L.mma_bench(mode, iters, C.c_void_p(out.data_ptr()), st) == 0
        torch.cuda.synchronize()
    cyc = int(out[0])
    n_mma = iters * 8
    per = cyc / n_mma
    # FLOP per cycle per SM: 2*M*N*K per MMA (K=16)
    m = mode % 20
    key = names[m] + (" [warp+elect]" if mode % 100 >= 20 else " [lane 0]") + \
        {0: "", 1: " + 8 warps TMEM loads", 2: " + 8 warps TMEM loads+stores"}[mode // 100]
    res[key] = {"cycles_per_mma": round(per, 1), "frac_of_8192_flop_per_clk": round(2 * 128 * N[m] * 16 / per / 8192, 3)}
print(json.dumps(res, indent=1))
