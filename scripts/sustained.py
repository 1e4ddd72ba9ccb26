"""Sustained (power-capped) throughput per SM clock: run one op back to back for ~4 s while
sampling the SM clock with NVML, for our GEMM / attention and for cuBLAS / SDPA at the same
shape.  Reports TF/s, the median SM clock under load, and TF/s per GHz (the per-clock
efficiency that survives the power cap).

usage: python scripts/sustained.py  ->  gpurun_out/sustained.json
"""
import ctypes as C
import json
import statistics
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, ".")
from paper_2512_07350_b200 import _lib  # noqa: E402

L = _lib.lib()
st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
pynvml.nvmlInit()
H = pynvml.nvmlDeviceGetHandleByIndex(0)


def sustained(fn, flops, secs=4.0):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    # calibrate a batch of ~50 ms
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    per = max(a.elapsed_time(b), 1e-3)
    batch = max(1, int(50 / per))
    clocks, power, stop = [], [], [False]

    def sample():
        while not stop[0]:
            clocks.append(pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM))
            power.append(pynvml.nvmlDeviceGetPowerUsage(H) / 1000.0)
            time.sleep(0.05)

    th = threading.Thread(target=sample)
    n = 0
    a.record()
    th.start()
    t0 = time.time()
    while time.time() - t0 < secs:
        for _ in range(batch):
            fn()
        n += batch
        torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    stop[0] = True
    th.join()
    ms = a.elapsed_time(b) / n
    tail = clocks[len(clocks) // 4:]  # drop the ramp
    mhz = statistics.median(tail)
    tf = flops / ms / 1e9
    return {"tflops": tf, "sm_mhz": mhz, "tflops_per_ghz": tf / (mhz / 1000), "power_w": statistics.median(power[len(power) // 4:]),
            "per_clock_frac": tf / (148 * 8192 * mhz * 1e6 / 1e12)}


out = {}
R = 2 * 14040
if "attn-knobs" in sys.argv:
    S = 14040
    q, k, v = (torch.randn(2, S, 12, 128, device="cuda").bfloat16() for _ in range(3))
    o = torch.empty_like(q)
    fl = 4 * 2 * 12 * S * S * 128
    for poly in (0, 4, 6, 8):
        _lib.check(L.lp_tune(b"attn_poly", poly))
        r = sustained(lambda: _lib.check(L.lp_attention_bf16(C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()),
                                                             C.c_void_p(v.data_ptr()), C.c_void_p(o.data_ptr()), 2, S, S,
                                                             12, 1 / 128 ** 0.5, st())), fl)
        out[f"attn_poly{poly}"] = r
        print(json.dumps({f"attn_poly{poly}": r}), flush=True)
    json.dump(out, open("gpurun_out/sustained_attn_knobs.json", "w"), indent=1)
    sys.exit(0)
for (M, N, K, name) in [(R, 4608, 1536, "qkv"), (R, 8960, 1536, "ffn1"), (R, 1536, 8960, "ffn2"), (8192, 8192, 8192, "sq8k")]:
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    fl = 2 * M * N * K
    ours = sustained(lambda: _lib.check(L.lp_gemm_bf16(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), None,
                                                       C.c_void_p(D.data_ptr()), M, N, K, st())), fl)
    cub = sustained(lambda: torch.matmul(A, B.t(), out=D), fl)
    out[f"gemm_{name}"] = {"ours": ours, "cublas": cub}
    print(json.dumps({f"gemm_{name}": out[f"gemm_{name}"]}), flush=True)
    del A, B, D
S = 14040
q, k, v = (torch.randn(2, S, 12, 128, device="cuda").bfloat16() for _ in range(3))
o = torch.empty_like(q)
fl = 4 * 2 * 12 * S * S * 128
ours = sustained(lambda: _lib.check(L.lp_attention_bf16(C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()),
                                                        C.c_void_p(o.data_ptr()), 2, S, S, 12, 1 / 128 ** 0.5, st())), fl)
qt, kt, vt = (x.transpose(1, 2) for x in (q, k, v))
sd = sustained(lambda: torch.nn.functional.scaled_dot_product_attention(qt, kt, vt), fl)
out["attn_14040"] = {"ours": ours, "sdpa": sd}
print(json.dumps({"attn_14040": out["attn_14040"]}), flush=True)
json.dump(out, open("gpurun_out/sustained.json", "w"), indent=1)
