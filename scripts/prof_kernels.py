"""Drive hot kernels once each at their C2 sizes, for `ncu --set full` captures.

usage: python scripts/prof_kernels.py [attn:S ...] [gemm] [lp]
  attn:S  self-attention, CFG batch 2, 12 heads, S tokens (18720 = K=4 T-axis shard)
  gemm    FFN1 GEMM at M = 2*18720
  lp      K1 gather + K10 reconstruct/update at the full C2 latent
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_07350_b200 import _lib, lp  # noqa: E402

L = _lib.lib()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
args = sys.argv[1:] or ["attn:18720", "gemm", "lp"]
for a in args:
    if a.startswith("attn"):
        S = int(a.split(":")[1])
        q = torch.randn(2, S, 12, 128, device="cuda").bfloat16()
        k = torch.randn(2, S, 12, 128, device="cuda").bfloat16()
        v = torch.randn(2, S, 12, 128, device="cuda").bfloat16()
        o = torch.empty_like(q)
        _lib.check(L.lp_attention_bf16(C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()),
                                       C.c_void_p(o.data_ptr()), 2, S, S, 12, 1 / 128 ** 0.5, st))
    elif a == "gemm":
        M, N, K = 2 * 18720, 8960, 1536
        A = torch.randn(M, K, device="cuda").bfloat16()
        B = torch.randn(N, K, device="cuda").bfloat16()
        D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        _lib.check(L.lp_gemm_bf16(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), None, C.c_void_p(D.data_ptr()),
                                  M, N, K, st))
    elif a == "lp":
        dims = (16, 21, 60, 104)
        z, cond = lp.synthetic_latent(dims, 4, 2025)
        plan = lp.build_plan(dims, (1, 2, 2), 1, 4, 0.5)
        subs = lp.extract_sublatents(z, plan)
        lp.reconstruct_update(subs, plan, z, 0.05)
torch.cuda.synchronize()
print("ok")
