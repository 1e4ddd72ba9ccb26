"""Drive each hot kernel once at its C2 size, for `ncu --set full` captures:
self-attention (S=18720, the K=4 T-axis shard, CFG batch 2), the FFN1 GEMM,
K1 gather and K10 reconstruct+update at the full C2 latent."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_07350_b200 import _lib, lp  # noqa: E402

L = _lib.lib()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
S = 18720
for rep in range(2):
    q = torch.randn(2, S, 12, 128, device="cuda").bfloat16()
    _lib.check(L.lp_attention_bf16(C.c_void_p(q.data_ptr()), C.c_void_p(q.data_ptr()), C.c_void_p(q.data_ptr()),
                                   C.c_void_p(q.data_ptr()), 2, S, S, 12, 1 / 128 ** 0.5, st))
    M, N, K = 2 * S, 8960, 1536
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    _lib.check(L.lp_gemm_bf16(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), None, C.c_void_p(D.data_ptr()),
                              M, N, K, st))
    dims = (16, 21, 60, 104)
    z, cond = lp.synthetic_latent(dims, 4, 2025)
    plan = lp.build_plan(dims, (1, 2, 2), 1, 4, 0.5)
    subs = lp.extract_sublatents(z, plan)
    lp.reconstruct_update(subs, plan, z, 0.05)
torch.cuda.synchronize()
print("ok")
