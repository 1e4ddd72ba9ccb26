"""Interleaved A/B timing of kernel variants (lp_tune knobs) in one process.

usage: python scripts/abtest.py attn_poly 0,1,2 [S ...]
Each round times every variant once per shape (CUDA events, L2 flushed), rounds
alternate variants, medians are reported — robust to clock drift between runs."""
import ctypes as C
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_07350_b200 import _lib  # noqa: E402

L = _lib.lib()
knob = sys.argv[1]
variants = [int(v) for v in sys.argv[2].split(",")]
sizes = [int(s) for s in sys.argv[3:]] or [32760, 18720, 14040]
st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {(v, S): [] for v in variants for S in sizes}
bufs = {}
for S in sizes:
    bufs[S] = [torch.randn(2, S, 12, 128, device="cuda").bfloat16() for _ in range(4)]


def run(S):
    q, k, v, o = bufs[S]
    _lib.check(L.lp_attention_bf16(C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()),
                                   C.c_void_p(o.data_ptr()), 2, S, S, 12, 1 / 128 ** 0.5, st()))


# correctness of every variant against torch SDPA (fp32 softmax) at the first size
err = {}
S0 = 3000  # not a multiple of 128: exercises the key mask; small enough for an fp32 SDPA reference
bufs[S0] = [torch.randn(2, S0, 12, 128, device="cuda").bfloat16() for _ in range(4)]
q, k, v, o = bufs[S0]
ref = torch.nn.functional.scaled_dot_product_attention(*(x.transpose(1, 2).float() for x in (q, k, v))).transpose(1, 2)
for v_ in variants:
    _lib.check(L.lp_tune(knob.encode(), v_))
    run(S0)
    torch.cuda.synchronize()
    err[v_] = float((o.float() - ref).abs().max())
del ref
for rnd in range(6):
    for S in sizes:
        for v in variants:
            _lib.check(L.lp_tune(knob.encode(), v))
            run(S)
            flush.zero_()
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record()
            run(S)
            b.record()
            torch.cuda.synchronize()
            if rnd > 0:
                res[(v, S)].append(a.elapsed_time(b))
out = {}
for S in sizes:
    fl = 4 * 2 * 12 * S * S * 128
    out[S] = {v: round(fl / statistics.median(res[(v, S)]) / 1e9, 1) for v in variants}
print(json.dumps({"knob": knob, "tflops": out, "max_abs_err_vs_sdpa": err}))
