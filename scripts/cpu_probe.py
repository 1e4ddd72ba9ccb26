"""Probe the GPU box's host CPU for the reference arm (CPU DiT sample sizing)."""
import os, time, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
print("nproc", os.cpu_count(), "sched_getaffinity", len(os.sched_getaffinity(0)))
print(subprocess.run(["lscpu"], capture_output=True, text=True).stdout)
print(torch.__config__.parallel_info())
from oracle.cpu_dit import CpuDiT
for threads in (len(os.sched_getaffinity(0)),):
    torch.set_num_threads(threads)
    for dt in (torch.float32, torch.bfloat16):
        a = torch.randn(14040, 1536, dtype=dt); b = torch.randn(8960, 1536, dtype=dt)
        a @ b.t()
        t0 = time.perf_counter(); a @ b.t(); dt_ = time.perf_counter() - t0
        print(f"threads {threads} {dt} gemm 14040x8960x1536: {2*14040*8960*1536/dt_/1e12:.2f} TF/s")
        q = torch.randn(1, 12, 14040, 128, dtype=dt)
        torch.nn.functional.scaled_dot_product_attention(q[:, :1], q[:, :1], q[:, :1])
        t0 = time.perf_counter(); torch.nn.functional.scaled_dot_product_attention(q, q, q); dt_ = time.perf_counter() - t0
        print(f"threads {threads} {dt} sdpa n=14040 h=12: {4*14040*14040*1536/dt_/1e12:.2f} TF/s ({dt_:.2f}s)")
    d = CpuDiT(num_layers=1)
    import numpy as np
    z = np.random.randn(16, 9, 60, 104).astype(np.float32)
    d.predict(z, 50, None, True)
    t0 = time.perf_counter(); d.predict(z, 50, None, True); print("1-block predict T-shard 9 frames", time.perf_counter() - t0)
