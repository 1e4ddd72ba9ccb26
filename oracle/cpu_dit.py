"""CPU WAN2.1-shaped DiT plugged into the UNMODIFIED reference run_lp (TEST / BASELINE
INFRASTRUCTURE ONLY: used by bench.py --impl reference and tests, never by the product).

The reference (`lpsim`) has no DiT: its Denoiser slot (include/lpsim/denoise.hpp:31-39)
only holds toy denoisers.  BASELINE.json's metric is quoted on a WAN-1.3B-shaped
denoiser, so the reference arm plugs this fp32 torch restatement (oracle/dit_fp32.py)
into the reference's own `run_lp` through its Denoiser interface (oracle/ref_harness.cpp
`ref_run_lp_callback`).  Weights are random (torch.Generator, fixed seed): the arm
measures time, not values.

Precision: `dtype=torch.bfloat16` (the arm's default) runs every GEMM and attention in bf16
with fp32 accumulation on the host's AMX tiles (oneDNN), residual stream and norms in fp32 —
the GPU arm's arithmetic, and ~2.5x faster on the box's 16 Sapphire-Rapids-class cores than
fp32 (probe: 11 vs 2.6 TF/s GEMM, 5 vs 2.3 TF/s SDPA; profiles/r3a).  A full C2 LP step is
~630 TFLOP, so bench.py --impl reference times whole reference run_lp steps (a T/H/W cycle)
with all 30 blocks; bench.py's in-line cpu_baseline uses a bounded one-block sample scaled to
the metric's unit instead (see bench.py).
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

    def __init__(self, num_layers=1, seed=2025, dtype=torch.float32, **overrides):
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
        self.dtype = dtype
        self.p = params
        if dtype != torch.float32:  # GEMM / attention operands in `dtype`, fp32 residual and norms
            self.w = {k: v.to(dtype) for k, v in params.items() if v.dim() == 2}
            self.ck = [k.to(dtype) for k in self.ck]
            self.cv = [v.to(dtype) for v in self.cv]
        self._lock = threading.Lock()
        self.calls = []  # (start, end) perf_counter of every predict call

    def predict(self, z, t, cond, is_null):
        t0 = time.perf_counter()
        zt = torch.from_numpy(np.asarray(z, np.float32))
        if self.dtype == torch.float32:
            out = self.ref.predict(zt, int(t), self.ck, self.cv, 0 if is_null else 1)
        else:
            out = self._predict_lowp(zt, int(t), 0 if is_null else 1)
        res = out.double().numpy()
        t1 = time.perf_counter()
        with self._lock:
            self.calls.append((t0, t1))
        return res

    @torch.no_grad()
    def _predict_lowp(self, z, t, b):
        """One CFG pass with bf16 GEMM / attention operands (fp32 accumulate), fp32 elsewhere:
        the forward of oracle/dit_fp32.DiTReference.run at the GPU arm's precision."""
        from oracle.dit_fp32 import apply_rope, rope_tables, sinusoid

        c, p, W, lp_ = self.cfg, self.p, self.w, self.dtype
        d, L, heads, eps = c.dim, c.num_layers, c.num_heads, c.eps

        def lin(x, name):
            return (x.to(lp_) @ W[name + ".w"].t()).float() + p[name + ".b"]

        def att(q, k, v):
            n = q.shape[0]
            q, k, v = (a.to(lp_).view(a.shape[0], heads, -1).transpose(0, 1)[None] for a in (q, k, v))
            return torch.nn.functional.scaled_dot_product_attention(q, k, v)[0].transpose(0, 1).reshape(n, d)

        pt, ph, pw = c.patch
        C, F, H, Wd = z.shape
        nf, nh, nw = -(-F // pt), -(-H // ph), -(-Wd // pw)
        zp = torch.zeros(C, nf * pt, nh * ph, nw * pw)
        zp[:, :F, :H, :Wd] = z
        x = lin(zp.view(C, nf, pt, nh, ph, nw, pw).permute(1, 3, 5, 0, 2, 4, 6).reshape(nf * nh * nw, -1), "patch")
        s = sinusoid(c.freq_dim, t * c.t_scale)
        silu = torch.nn.functional.silu
        e = silu(s[None] @ p["time.w1"].t() + p["time.b1"]) @ p["time.w2"].t() + p["time.b2"]
        e0 = (silu(e) @ p["time.wp"].t() + p["time.bp"]).view(6, d)
        mods = p["blocks.mod"].view(L, 6, d) + e0[None]
        cos, sin = rope_tables(nf, nh, nw, "cpu")
        ln = torch.nn.functional.layer_norm
        for l in range(L):
            pre, m = f"blocks.{l}.", mods[l]
            h = ln(x, (d,), eps=eps) * (1 + m[1]) + m[0]
            qkv = lin(h, pre + "qkv")
            q = apply_rope(rms(qkv[:, :d], p[pre + "norm_q"], eps), cos, sin, heads)
            k = apply_rope(rms(qkv[:, d:2 * d], p[pre + "norm_k"], eps), cos, sin, heads)
            x = x + lin(att(q, k, qkv[:, 2 * d:]), pre + "o") * m[2]
            h = ln(x, (d,), weight=p[pre + "norm3.w"], bias=p[pre + "norm3.b"], eps=eps)
            cq = rms(lin(h, pre + "cq"), p[pre + "cnorm_q"], eps)
            x = x + lin(att(cq, self.ck[l][b], self.cv[l][b]), pre + "co")
            h = ln(x, (d,), eps=eps) * (1 + m[4]) + m[3]
            f = torch.nn.functional.gelu(lin(h, pre + "ffn1"), approximate="tanh")
            x = x + lin(f, pre + "ffn2") * m[5]
        hm = p["head.mod"].view(2, d) + e
        head = lin(ln(x, (d,), eps=eps) * (1 + hm[1]) + hm[0], "head")
        out = head.view(nf, nh, nw, pt, ph, pw, C).permute(6, 0, 3, 1, 4, 2, 5).reshape(C, nf * pt, nh * ph, nw * pw)
        return out[:, :F, :H, :Wd]


def dit_flops(shape, patch, dim=1536, ffn=8960, text_len=512):
    """Algorithmic FLOPs of one DiT block for one CFG pass on a shard (GEMM 2MNK, attention 4 n_q n_kv d)."""
    n = -(-shape[1] // patch[0]) * -(-shape[2] // patch[1]) * -(-shape[3] // patch[2])
    return 2 * n * (6 * dim * dim + 2 * dim * ffn) + 4 * n * n * dim + 4 * n * text_len * dim
