"""Run scripts/micro/libmma_bench.so: cycles per tcgen05.mma per operand mode (all 148 SMs busy)."""
import ctypes as C
import json
import sys

import torch

L = C.CDLL("scripts/micro/libmma_bench.so")
out = torch.zeros(4, dtype=torch.int64, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
names = {0: "SS N128 (S=QK^T)", 1: "TS N128 B MN-major (PV)", 2: "SS N256", 3: "SS N64", 4: "TS N128 B K-major",
         5: "SS N128 B MN-major", 6: "SS N128 x2 sharing B"}
N = {0: 128, 1: 128, 2: 256, 3: 64, 4: 128, 5: 128, 6: 256}
res = {}
for mode in list(names) + [m + 10 for m in names]:
    iters = 200
    for rep in range(3):
        assert L.mma_bench(mode, iters, C.c_void_p(out.data_ptr()), st) == 0
        torch.cuda.synchronize()
    cyc = int(out[0])
    n_mma = iters * 8
    per = cyc / n_mma
    # FLOP per cycle per SM: 2*M*N*K per MMA (K=16)
    m = mode % 10
    key = names[m] + (" [warp+elect]" if mode >= 10 else " [lane 0]")
    res[key] = {"cycles_per_mma": round(per, 1), "frac_of_8192_flop_per_clk": round(2 * 128 * N[m] * 16 / per / 8192, 3)}
print(json.dumps(res, indent=1))
