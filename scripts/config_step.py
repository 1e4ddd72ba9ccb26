"""One-GPU measurement of the other BASELINE.json configs through the engine (evidence, not
the bench line): C4 = WAN2.1-14B-shaped DiT (40 blocks, d=5120, 40 heads, FFN 13824) on the
720p/81-frame latent 16x21x90x160, 8-way LP; C5 = 1.3B-shaped DiT on the 161-frame latent
16x41x60x104, 8-way LP with the temporal-heavy schedule "TTHTTW".  All K shards run on one
GPU (2 streams), so steps/s here is the whole 8-way job on a single B200.

usage: python scripts/config_step.py c4|c5 [steps]
Writes gpurun_out/config_<name>.json.
"""
import json
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2512_07350_b200 import _lib, lp  # noqa: E402

CFG = {
    "c4": dict(dims=(16, 21, 90, 160), K=8, dit=dict(dim=5120, num_heads=40, ffn_dim=13824, num_layers=40),
               schedule=None, d=5120, F=13824, L=40),
    "c5": dict(dims=(16, 41, 60, 104), K=8, dit=dict(num_layers=30), schedule="TTHTTW", d=1536, F=8960, L=30),
}


def step_flops(dims, K, r, schedule, d, F, L, steps):
    axes = lp.parse_schedule(schedule) if schedule else [0, 1, 2]
    tot = []
    for i in range(len(axes)):
        p = lp.build_axis_plan(axes[i], dims[1 + axes[i]], (1, 2, 2)[axes[i]], i + 1, K, r)
        f = 0.0
        for k in range(p.workers):
            s = p.sub_shape(dims, k)
            n = s[1] * -(-s[2] // 2) * -(-s[3] // 2)
            f += L * (2 * 2 * n * (6 * d * d + 2 * d * F) + 2 * 4 * n * n * d + 2 * 4 * n * 512 * d)
        tot.append(f)
    return statistics.mean(tot[i % len(tot)] for i in range(steps)), tot


def main():
    name = sys.argv[1]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    c = CFG[name]
    torch.cuda.set_device(0)
    z, cond = lp.synthetic_latent_host(c["dims"], 4, 2025)
    t0 = time.time()
    dit = lp.DiTDenoiser(cond, **c["dit"])
    init_s = time.time() - t0
    eng = lp.LpEngine(c["dims"], (1, 2, 2), 4, c["K"], 0.5, 50, 0.05, 5.0, cond, denoiser="dit", dit=dit,
                      schedule=c["schedule"])
    eng.z.data.copy_(torch.from_numpy(z.astype("float32")))
    eng.run(1, 1)  # warm-up (also the first, T-axis step)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    eng.run(2, steps)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    per_step, per_axis = step_flops(c["dims"], c["K"], 0.5, c["schedule"], c["d"], c["F"], c["L"], steps)
    # the timed steps are 2..steps+1: recompute their mean exactly
    axes = lp.parse_schedule(c["schedule"]) if c["schedule"] else [0, 1, 2]
    fl = statistics.mean(per_axis[(i - 1) % len(axes)] for i in range(2, steps + 2))
    out = {"config": name, "dims": c["dims"], "K": c["K"], "schedule": c["schedule"] or "rotating T,H,W",
           "dit": c["dit"], "steps_timed": steps, "ms_per_step": ms, "steps_per_s": 1000.0 / ms,
           "algorithmic_tflop_per_step": fl / 1e12, "tflops": fl / (ms / 1000) / 1e12,
           "weights_init_s": init_s, "device_mem_used_gb": (lambda f: (f[1] - f[0]) / 1e9)(torch.cuda.mem_get_info()),
           "finite": bool(torch.isfinite(eng.z.data).all())}
    print(json.dumps(out))
    json.dump(out, open(f"gpurun_out/config_{name}.json", "w"), indent=1)
    eng.close()
    del per_step


if __name__ == "__main__":
    main()
