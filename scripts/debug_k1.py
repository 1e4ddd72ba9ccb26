"""Isolate K1 TMA-path failures: one (dims, k, r, step, dtype) case per process.
usage: python scripts/debug_k1.py d step T H W k r"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle.oracle import Oracle  # noqa: E402
from paper_2512_07350_b200 import _lib, lp  # noqa: E402

d, step = int(sys.argv[1]), int(sys.argv[2])
dims = (16, int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]))
k, r = int(sys.argv[6]), float(sys.argv[7])
orc = Oracle()
z, _ = orc.synthetic(dims, d, 7)
zt = lp.LatentTensor.from_numpy(z, d)
L = _lib.lib()
plan = lp.build_plan(dims, (1, 2, 2), step, k, r)
n = sum(int(np.prod(plan.sub_shape(dims, e))) for e in range(plan.workers))
out = lp.LatentTensor(torch.empty(n, dtype=zt.data.dtype, device="cuda"), d)
_lib.check(L.lp_extract(C.byref(plan.raw), 0, plan.workers, zt.ptr(), _lib.i64arr(dims), d, out.ptr(),
                        C.c_void_p(torch.cuda.current_stream().cuda_stream)))
torch.cuda.synchronize()
want = orc.extract(z, orc.build_plan(dims, (1, 2, 2), step, k, r))
print("case", d, step, dims, k, r, "equal", np.array_equal(out.to_numpy(), want), flush=True)
