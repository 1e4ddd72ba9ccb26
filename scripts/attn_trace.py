"""Timeline of one attention CTA (clock64 stamps from the TR kernel variant).

usage: python scripts/attn_trace.py [S] [mode: 1 = real kernel, 2 = no softmax work (MMA/sync floor)]
Prints, per key block j and Q tile t, cycle offsets of: S ready, max done, p_half,
p_full (softmax side) and MMA-warp wakeups, plus the steady-state per-block period."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_07350_b200 import _lib  # noqa: E402

L = _lib.lib()
S = int(sys.argv[1]) if len(sys.argv) > 1 else 18720
q, k, v, o = (torch.randn(2, S, 12, 128, device="cuda").bfloat16() for _ in range(4))
buf = torch.zeros(64 * 2 * 16, dtype=torch.int64, device="cuda")
_lib.check(L.lp_attention_set_trace(C.c_void_p(buf.data_ptr())))
_lib.check(L.lp_tune(b"attn_trace", int(sys.argv[2]) if len(sys.argv) > 2 else 1))
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(3):
    _lib.check(L.lp_attention_bf16(C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()),
                                   C.c_void_p(o.data_ptr()), 2, S, S, 12, C.c_double(1 / 128 ** 0.5), st))
torch.cuda.synchronize()
tr = buf.view(64, 2, 16).cpu()
t0 = int(tr[0, 0, 0])
names = ["S_ready", "max", "p_half", "p_full", "mma_p_half", "mma_p_full", "mma_S_next", "ev7",
         "p_half_q0", "p_half_q1", "p_half_q2", "p_half_q3", "p_full_q0", "p_full_q1", "p_full_q2", "p_full_q3"]
rows = []
for j in range(min(64, -(-S // 128))):
    for t in range(2):
        rows.append({"j": j, "t": t, **{n: int(tr[j, t, e]) - t0 for e, n in enumerate(names)}})
for r in rows[:24]:
    print(r)
per = [(rows[2 * j + 2]["S_ready"] - rows[2 * j]["S_ready"]) for j in range(8, min(60, len(rows) // 2 - 1))]
dur = {n: sum(r[n] - r["S_ready"] for r in rows[16:100]) / len(rows[16:100]) for n in names[1:]}
summary = {"S": S, "period_cycles_per_block": sum(per) / len(per), "mean_offsets_from_S_ready": dur}
print(json.dumps(summary))
json.dump({"rows": rows, "summary": summary}, open("gpurun_out/attn_trace.json", "w"))
