"""Attention time vs key count at a fixed query count: the intercept of time = a + b * n_kv is
the per-CTA fixed cost (launch, Q/K fetch latency, pipeline ramp and drain, epilogue) times the
number of CTA waves.  usage: python scripts/attn_overhead.py"""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_07350_b200 import _lib  # noqa: E402

L = _lib.lib()
st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
nq, H, B = 14040, 12, 2
q = torch.randn(B, nq, H, 128, device="cuda").bfloat16()
o = torch.empty_like(q)
res = []
for nkv in (512, 1024, 2048, 4096, 8192, 14040):
    k = torch.randn(B, nkv, H, 128, device="cuda").bfloat16()
    v = torch.randn(B, nkv, H, 128, device="cuda").bfloat16()
    f = lambda: _lib.check(L.lp_attention_bf16(C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()),  # noqa: E731
                                               C.c_void_p(o.data_ptr()), B, nq, nkv, H, 1 / 128 ** 0.5, st()))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    ms = ts[5]
    res.append((nkv, ms))
    print(json.dumps({"n_kv": nkv, "ms": ms, "tflops": 4 * B * H * nq * nkv * 128 / ms / 1e9}), flush=True)
# least squares on the points with n_kv >= 1024
xs = [r[0] for r in res[1:]]
ys = [r[1] for r in res[1:]]
n = len(xs)
mx, my = sum(xs) / n, sum(ys) / n
b = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
a = my - b * mx
ctas = ((nq + 255) // 256) * H * B
waves = ctas / 148
print(json.dumps({"intercept_ms": a, "slope_ms_per_key": b, "ctas": ctas, "waves": waves,
                  "fixed_us_per_cta_wave": a * 1000 / waves}))
