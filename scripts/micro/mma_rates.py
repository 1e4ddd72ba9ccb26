"""Cycles per tcgen05.mma for the operand modes of scripts/micro/libmma_bench.so (all SMs busy):
SS N128 / TS N128 (MN-major B) / SS N256 / SS N64 — lane-0 issue and converged warp + elect."""
import ctypes as C
import json

import torch

L = C.CDLL("scripts/micro/libmma_bench.so")
out = torch.zeros(4, dtype=torch.int64, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
names = {0: "SS N128", 1: "TS N128 B MN-major", 2: "SS N256", 3: "SS N64", 4: "TS N128 B K-major"}
N = {0: 128, 1: 128, 2: 256, 3: 64, 4: 128}
res = {}
for mode in [0, 1, 2, 3, 4, 20, 21, 22, 23]:
    iters = 200
    for _ in range(3):
        assert L.mma_bench(mode, iters, C.c_void_p(out.data_ptr()), st) == 0
        torch.cuda.synchronize()
    per = int(out[0]) / (iters * 8)
    m = mode % 20
    res[names[m] + (" [warp+elect]" if mode >= 20 else " [lane 0]")] = {
        "cycles_per_mma": round(per, 1), "frac_of_8192_flop_per_clk": round(2 * 128 * N[m] * 16 / per / 8192, 3)}
print(json.dumps(res, indent=1))
