"""One fused-epilogue GEMM launch (for ncu): python scripts/gemm_epi_one.py M N K mode"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_07350_b200 import _lib  # noqa: E402

M, N, K, mode = (int(x) for x in sys.argv[1:5])
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
bias, gate = torch.randn(N, device="cuda"), torch.randn(N, device="cuda")
D = torch.zeros(M, N, device="cuda", dtype=torch.float32 if mode >= 2 else torch.bfloat16)
for _ in range(2):
    _lib.check(_lib.lib().lp_gemm_bf16_epi(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), C.c_void_p(bias.data_ptr()),
                                           C.c_void_p(gate.data_ptr()), C.c_void_p(D.data_ptr()), M, N, K, mode,
                                           C.c_void_p(torch.cuda.current_stream().cuda_stream)))
torch.cuda.synchronize()
