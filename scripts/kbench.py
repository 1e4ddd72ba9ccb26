"""Kernel micro-benchmarks (CUDA events, warm, L2-flushed between reps): tcgen05 GEMM at the
DiT's shapes and attention at the C2 shard sizes.  Prints TFLOP/s per shape."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_07350_b200 import _lib  # noqa: E402

L = _lib.lib()
st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


out = {}
R = int(os.environ.get("KB_ROWS", 2 * 32760))  # 2n rows (CFG batch 2); in-step shards: 2*14040 .. 2*18720
GEMMS = [(R, 4608, 1536, "qkv"), (R, 1536, 1536, "o"), (R, 8960, 1536, "ffn1"), (R, 1536, 8960, "ffn2"),
         (8192, 8192, 8192, "sq8k")]
for (M, N, K, name) in ([] if "attn" in sys.argv else GEMMS):
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    f = lambda: _lib.check(L.lp_gemm_bf16(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), None,  # noqa: E731
                                          C.c_void_p(D.data_ptr()), M, N, K, st()))
    ms = timeit(f)
    tc = timeit(lambda: torch.matmul(A, B.t(), out=D))
    out[f"gemm_{name}"] = {"M": M, "N": N, "K": K, "ms": ms, "tflops": 2 * M * N * K / ms / 1e9,
                           "cublas_ms": tc, "cublas_tflops": 2 * M * N * K / tc / 1e9}
    print(json.dumps({f"gemm_{name}": out[f"gemm_{name}"]}), flush=True)
    del A, B, D
# the DiT's fused epilogues at the shard size: GELU (ffn1) and the fp32 gated residual (o / co / ffn2)
for (M, N, K, mode, name) in ([] if "attn" in sys.argv or "gemm" in sys.argv and "epi" not in sys.argv else
                              [(R, 8960, 1536, 1, "ffn1_gelu"), (R, 1536, 1536, 2, "o_resid"),
                               (R, 1536, 8960, 2, "ffn2_resid")]):
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    bias = torch.randn(N, device="cuda")
    gate = torch.randn(N, device="cuda")
    D = torch.zeros(M, N, device="cuda", dtype=torch.float32 if mode >= 2 else torch.bfloat16)
    f = lambda: _lib.check(L.lp_gemm_bf16_epi(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()),  # noqa: E731
                                              C.c_void_p(bias.data_ptr()), C.c_void_p(gate.data_ptr()),
                                              C.c_void_p(D.data_ptr()), M, N, K, mode, st()))
    ms = timeit(f)
    out[f"gemm_{name}"] = {"M": M, "N": N, "K": K, "mode": mode, "ms": ms, "tflops": 2 * M * N * K / ms / 1e9,
                           "epilogue_GBps": (M * N * (8 if mode == 2 else 2)) / ms / 1e6}
    print(json.dumps({f"gemm_{name}": out[f"gemm_{name}"]}), flush=True)
    del A, B, D
for (S, name) in ([] if "gemm" in sys.argv else [(32760, "self_k1"), (18720, "self_k4max"), (14040, "self_k4min")]):
    q = torch.randn(2, S, 12, 128, device="cuda").bfloat16()
    k = torch.randn(2, S, 12, 128, device="cuda").bfloat16()
    v = torch.randn(2, S, 12, 128, device="cuda").bfloat16()
    o = torch.empty_like(q)
    f = lambda: _lib.check(L.lp_attention_bf16(C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()),  # noqa: E731
                                               C.c_void_p(v.data_ptr()), C.c_void_p(o.data_ptr()), 2, S, S, 12,
                                               1 / 128 ** 0.5, st()))
    ms = timeit(f, 5)
    fl = 4 * 2 * 12 * S * S * 128
    qt, kt, vt = (x.transpose(1, 2) for x in (q, k, v))
    tsd = timeit(lambda: torch.nn.functional.scaled_dot_product_attention(qt, kt, vt), 5)
    out[f"attn_{name}"] = {"S": S, "ms": ms, "tflops": fl / ms / 1e9, "sdpa_ms": tsd, "sdpa_tflops": fl / tsd / 1e9}
    print(json.dumps({f"attn_{name}": out[f"attn_{name}"]}), flush=True)
tag = os.environ.get("KB_TAG", "")
json.dump(out, open(f"gpurun_out/kbench{tag}.json", "w"), indent=1)
