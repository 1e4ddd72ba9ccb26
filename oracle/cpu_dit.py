"""CPU WAN2.1-shaped DiT plugged into the UNMODIFIED reference run_lp (TEST / BASELINE
INFRASTRUCTURE ONLY: used by bench.py --impl reference and tests, never by the product).

The reference (`lpsim`) has no DiT: its Denoiser slot (include/lpsim/denoise.hpp:31-39)
only holds toy denoisers.  BASELINE.json's metric is quoted on a WAN-1.3B-shaped
denoiser, so the reference arm plugs this fp32 torch restatement (oracle/dit_fp32.py)
into the reference's own `run_lp` through its Denoiser interface (oracle/ref_harness.cpp
`ref_run_lp_callback`).  Weights are random (torch.Generator, fixed seed): the arm
measures time, not values.

Bounded sample: a full C2 step is ~630 TFLOP (hours on host cores), so one sample is
one reference `run_lp` step with a ONE-block DiT; the DiT wall time of that step is
scaled by the block count (all blocks have identical shapes and cost) and by the ratio
of the rotation-cycle mean DiT FLOPs to the sampled axis's FLOPs.
"""
from __future__ import annotations

import threading
import time
from types import SimpleNamespace

import numpy as np
import torch

from oracle.dit_fp32 import DiTReference, rms

WAN13B = dict(in_channels=16, dim=1536, ffn_dim=8960, num_heads=12, text_len=512, text_dim=4096, freq_dim=256,
              patch=(1, 2, 2), eps=1e-6, t_scale=1000.0 / 50.0)


def param_shapes(cfg):
    d, F, L = cfg.dim, cfg.ffn_dim, cfg.num_layers
    pfeat = cfg.in_channels * cfg.patch[0] * cfg.patch[1] * cfg.patch[2]
    s = {"patch.w": (d, pfeat), "patch.b": (d,), "text.w1": (d, cfg.text_dim), "text.b1": (d,), "text.w2": (d, d),
         "text.b2": (d,), "time.w1": (d, cfg.freq_dim), "time.b1": (d,), "time.w2": (d, d), "time.b2": (d,),
         "time.wp": (6 * d, d), "time.bp": (6 * d,), "blocks.mod": (L, 6, d)}
    for l in range(L):
        p = f"blocks.{l}."
        s.update({p + "qkv.w": (3 * d, d), p + "qkv.b": (3 * d,), p + "norm_q": (d,), p + "norm_k": (d,),
                  p + "o.w": (d, d), p + "o.b": (d,), p + "norm3.w": (d,), p + "norm3.b": (d,), p + "cq.w": (d, d),
                  p + "cq.b": (d,), p + "ck.w": (d, d), p + "ck.b": (d,), p + "cv.w": (d, d), p + "cv.b": (d,),
                  p + "cnorm_q": (d,), p + "cnorm_k": (d,), p + "co.w": (d, d), p + "co.b": (d,),
                  p + "ffn1.w": (F, d), p + "ffn1.b": (F,), p + "ffn2.w": (d, F), p + "ffn2.b": (d,)})
    s.update({"head.mod": (2, d), "head.w": (pfeat, d), "head.b": (pfeat,)})
    return s


class CpuDiT:
    """fp32 CPU DiT with the engine's architecture; predict() is one CFG pass
    (the reference's Denoiser::predict: uncond when the conditioning is null)."""

    def __init__(self, num_layers=1, seed=2025, **overrides):
        c = dict(WAN13B, **overrides)
        c["num_layers"] = num_layers
        self.cfg = SimpleNamespace(**c)
        g = torch.Generator().manual_seed(seed)
        params = {}
        for name, shape in param_shapes(self.cfg).items():
            fan_in = shape[-1]
            if name.endswith(("norm_q", "norm_k", "norm3.w")):
                params[name] = 1 + 0.1 * (2 * torch.rand(shape, generator=g) - 1)
            elif name.endswith(".w") or name == "time.wp":
                params[name] = (2 * torch.rand(shape, generator=g) - 1) * (3.0 / fan_in) ** 0.5
            else:
                params[name] = 0.02 * (2 * torch.rand(shape, generator=g) - 1)
        self.ref = DiTReference(SimpleNamespace(cfg=self.cfg, params=lambda: params))
        text = torch.zeros(2, self.cfg.text_len, self.cfg.text_dim)
        text[1] = torch.randn(self.cfg.text_len, self.cfg.text_dim, generator=g)
        with torch.no_grad():
            ctx = self.ref.context(text)
            p, d = self.ref.p, self.cfg.dim
            self.ck, self.cv = [], []
            for l in range(num_layers):
                pre = f"blocks.{l}."
                self.ck.append(rms(ctx @ p[pre + "ck.w"].t() + p[pre + "ck.b"], p[pre + "cnorm_k"], self.cfg.eps))
                self.cv.append(ctx @ p[pre + "cv.w"].t() + p[pre + "cv.b"])
        del d
        self._lock = threading.Lock()
        self.calls = []  # (start, end) perf_counter of every predict call

    def predict(self, z, t, cond, is_null):
        t0 = time.perf_counter()
        out = self.ref.predict(torch.from_numpy(np.asarray(z, np.float32)), int(t), self.ck, self.cv, 0 if is_null else 1)
        res = out.double().numpy()
        t1 = time.perf_counter()
        with self._lock:
            self.calls.append((t0, t1))
        return res


def dit_flops(shape, patch, dim=1536, ffn=8960, text_len=512):
    """Algorithmic FLOPs of one DiT block for one CFG pass on a shard (GEMM 2MNK, attention 4 n_q n_kv d)."""
    n = -(-shape[1] // patch[0]) * -(-shape[2] // patch[1]) * -(-shape[3] // patch[2])
    return 2 * n * (6 * dim * dim + 2 * dim * ffn) + 4 * n * n * dim + 4 * n * text_len * dim
