"""Run scripts/micro/libsm_bench.so: cycles per 64-key softmax chunk per warp."""
import ctypes as C
import json

import torch

L = C.CDLL("scripts/micro/libsm_bench.so")
out = torch.zeros(4, dtype=torch.int64, device="cuda")
sink = torch.zeros(148 * 1024, device="cuda")
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
names = {0: "tmem+mufu", 1: "regs+mufu", 2: "tmem+ffma", 3: "regs+ffma", 4: "tmem+mufu+prmt", 5: "regs+mufu+prmt",
         6: "tmem+ffma+prmt", 7: "regs+ffma+prmt", 0x40: "tmem+poly4", 0x60: "tmem+poly6", 0x80: "tmem+poly8",
         0x44: "tmem+poly4+prmt", 0x64: "tmem+poly6+prmt", 0x41: "regs+poly4", 0x61: "regs+poly6",
         0x100: "tmem+mufu +MMA load", 0x160: "tmem+poly6 +MMA load", 0x101: "regs+mufu +MMA load"}
res = {}
for mode in [0, 0x100, 0x60, 0x160, 1, 0x101]:
    for warps in (4, 8):
        iters = 400
        for _ in range(2):
            assert L.sm_bench(mode, warps, iters, C.c_void_p(out.data_ptr()), C.c_void_p(sink.data_ptr()), st) == 0
            torch.cuda.synchronize()
        cyc = int(out[0]) / iters
        res[f"{names[mode]} w{warps}"] = {"cycles_per_chunk_per_warp": round(cyc, 1),
                                          "cycles_per_mufu_instr_per_smsp": round(cyc / (64 * warps / 4), 2)}
print(json.dumps(res, indent=0))
