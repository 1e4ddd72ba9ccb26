"""Run one attention call (debug): python scripts/attn_one.py S [B] [H]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_07350_b200 import _lib  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
H = int(sys.argv[3]) if len(sys.argv) > 3 else 1
L = _lib.lib()
q, k, v, o = (torch.randn(B, S, H, 128, device="cuda").bfloat16() for _ in range(4))
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
_lib.check(L.lp_attention_bf16(C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()),
                               C.c_void_p(o.data_ptr()), B, S, S, H, C.c_double(1 / 128 ** 0.5), st))
torch.cuda.synchronize()
ref = torch.nn.functional.scaled_dot_product_attention(*(x.transpose(1, 2).float() for x in (q, k, v))).transpose(1, 2)
print("max err", float((o.float() - ref).abs().max()))
