"""Plain PyTorch fp32 restatement of the WAN2.1-shaped DiT denoiser (test infrastructure:
the tolerance oracle of tests/test_dit_gpu.py and the CPU DiT of bench.py --impl reference).

It consumes the engine's own (bf16/fp32) parameters, read back through the
C-ABI (lp_dit_param), and restates the forward described in
paper_2512_07350_b200/csrc/dit.cpp in fp32 torch ops.  It is the tolerance
oracle for the tcgen05 DiT (the reference repo has no DiT: SURVEY.md §8c).
"""
from __future__ import annotations

import math

import torch
import torch.nn.functional as Fn


def _f(t):
    return t.float()


def sinusoid(dim, t):
    half = dim // 2
    w = torch.pow(torch.tensor(10000.0, dtype=torch.float64), -torch.arange(half, dtype=torch.float64) / half)
    a = t * w
    return torch.cat([torch.cos(a), torch.sin(a)]).float()


def rope_tables(nf, nh, nw, device):
    def part(n, pairs):
        j = torch.arange(pairs, dtype=torch.float32, device=device)
        freq = torch.pow(torch.tensor(10000.0, device=device), -j / pairs)
        pos = torch.arange(n, dtype=torch.float32, device=device)
        return pos[:, None] * freq[None, :]  # [n, pairs]

    ft, fh, fw = part(nf, 22), part(nh, 21), part(nw, 21)
    ang = torch.cat([
        ft[:, None, None, :].expand(nf, nh, nw, 22),
        fh[None, :, None, :].expand(nf, nh, nw, 21),
        fw[None, None, :, :].expand(nf, nh, nw, 21),
    ], dim=-1).reshape(nf * nh * nw, 64)
    return torch.cos(ang), torch.sin(ang)


def apply_rope(x, cos, sin, heads):
    # x [n, heads*128]; pairs (2j, 2j+1) within each head
    n = x.shape[0]
    x = x.view(n, heads, 64, 2)
    a, b = x[..., 0], x[..., 1]
    c, s = cos[:, None, :], sin[:, None, :]
    return torch.stack([a * c - b * s, a * s + b * c], dim=-1).reshape(n, heads * 128)


def rms(x, g, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * g


def attention(q, k, v, heads):
    # q [nq, d], k/v [nk, d]
    nq, d = q.shape
    q = q.view(nq, heads, 128).transpose(0, 1)
    k = k.view(-1, heads, 128).transpose(0, 1)
    v = v.view(-1, heads, 128).transpose(0, 1)
    o = Fn.scaled_dot_product_attention(q[None], k[None], v[None])[0]
    return o.transpose(0, 1).reshape(nq, d)


class DiTReference:
    """act_bf16=True rounds every GEMM / attention operand to bf16 (fp32 math otherwise): the
    precision floor of any bf16-operand implementation, used to ground the test tolerances."""

    def __init__(self, dit, act_bf16=False):
        self.cfg = dit.cfg
        self.p = {k: _f(v) for k, v in dit.params().items()}
        self.r = (lambda x: x.bfloat16().float()) if act_bf16 else (lambda x: x)

    def lin(self, x, name):
        return x @ self.p[name + ".w"].view(-1, x.shape[-1]).t() + self.p[name + ".b"]

    @torch.no_grad()
    def context(self, cond_ctx_in):
        """cond_ctx_in: [2, T, text_dim] (uncond zeros, cond synthetic) -> [2, T, d]."""
        c = self.cfg
        h = Fn.gelu(cond_ctx_in @ self.p["text.w1"].view(c.dim, -1).t() + self.p["text.b1"], approximate="tanh")
        return h @ self.p["text.w2"].view(c.dim, -1).t() + self.p["text.b2"]

    @torch.no_grad()
    def forward(self, z, t, ctx_k, ctx_v, w):
        """z: [C, F, H, W] fp32 latent; ctx_k/ctx_v: per-layer [2, T, d] (the engine's cached
        cross K/V); returns (eps [C,F,H,W] fp32 computed with fp32 combine, head [2n, 64])."""
        out, head = self.run(z, t, ctx_k, ctx_v, (0, 1))
        u, cc = out[0].double(), out[1].double()
        return (u + w * (cc - u)).float(), head

    @torch.no_grad()
    def predict(self, z, t, ctx_k, ctx_v, b):
        """One CFG pass (b = 0 uncond / 1 cond): the Denoiser::predict of this DiT."""
        return self.run(z, t, ctx_k, ctx_v, (b,))[0][0]

    @torch.no_grad()
    def run(self, z, t, ctx_k, ctx_v, batches):
        c = self.cfg
        d, L, heads = c.dim, c.num_layers, c.num_heads
        pt, ph, pw = c.patch
        C, F, H, W = z.shape
        nf, nh, nw = -(-F // pt), -(-H // ph), -(-W // pw)
        zp = torch.zeros(C, nf * pt, nh * ph, nw * pw, device=z.device)
        zp[:, :F, :H, :W] = z
        patches = zp.view(C, nf, pt, nh, ph, nw, pw).permute(1, 3, 5, 0, 2, 4, 6).reshape(nf * nh * nw, -1)
        n = patches.shape[0]
        x0 = self.r(patches) @ self.p["patch.w"].view(d, -1).t() + self.p["patch.b"]
        B = len(batches)
        x = torch.cat([x0] * B, 0)
        s = sinusoid(c.freq_dim, t * c.t_scale).to(z.device)
        e = Fn.silu(s @ self.p["time.w1"].view(d, -1).t() + self.p["time.b1"]) @ self.p["time.w2"].view(d, d).t() + self.p["time.b2"]
        e0 = (Fn.silu(e) @ self.p["time.wp"].view(6 * d, d).t() + self.p["time.bp"]).view(6, d)
        mods = self.p["blocks.mod"].view(L, 6, d) + e0[None]
        cos, sin = rope_tables(nf, nh, nw, z.device)
        eps = c.eps
        for l in range(L):
            pre = f"blocks.{l}."
            m = mods[l]
            h = self.r(Fn.layer_norm(x, (d,), eps=eps) * (1 + m[1]) + m[0])
            qkv = h @ self.p[pre + "qkv.w"].view(3 * d, d).t() + self.p[pre + "qkv.b"]
            q, k, v = qkv[:, :d], qkv[:, d:2 * d], qkv[:, 2 * d:]
            q = rms(q, self.p[pre + "norm_q"], eps)
            k = rms(k, self.p[pre + "norm_k"], eps)
            outs = []
            for b in range(B):
                sl = slice(b * n, (b + 1) * n)
                outs.append(attention(self.r(apply_rope(q[sl], cos, sin, heads)), self.r(apply_rope(k[sl], cos, sin, heads)),
                                      self.r(v[sl]), heads))
            y = self.r(torch.cat(outs, 0)) @ self.p[pre + "o.w"].view(d, d).t() + self.p[pre + "o.b"]
            x = x + y * m[2]
            h = self.r(Fn.layer_norm(x, (d,), weight=self.p[pre + "norm3.w"], bias=self.p[pre + "norm3.b"], eps=eps))
            cq = rms(h @ self.p[pre + "cq.w"].view(d, d).t() + self.p[pre + "cq.b"], self.p[pre + "cnorm_q"], eps)
            outs = []
            for b in range(B):
                sl = slice(b * n, (b + 1) * n)
                outs.append(attention(self.r(cq[sl]), ctx_k[l][batches[b]], ctx_v[l][batches[b]], heads))
            x = x + self.r(torch.cat(outs, 0)) @ self.p[pre + "co.w"].view(d, d).t() + self.p[pre + "co.b"]
            h = self.r(Fn.layer_norm(x, (d,), eps=eps) * (1 + m[4]) + m[3])
            f = self.r(Fn.gelu(h @ self.p[pre + "ffn1.w"].view(c.ffn_dim, d).t() + self.p[pre + "ffn1.b"], approximate="tanh"))
            x = x + (f @ self.p[pre + "ffn2.w"].view(d, c.ffn_dim).t() + self.p[pre + "ffn2.b"]) * m[5]
        hm = self.p["head.mod"].view(2, d) + e[None]
        h = self.r(Fn.layer_norm(x, (d,), eps=eps) * (1 + hm[1]) + hm[0])
        head = h @ self.p["head.w"].view(-1, d).t() + self.p["head.b"]  # [2n, pt*ph*pw*C]
        out = head.view(B, nf, nh, nw, pt, ph, pw, C).permute(0, 7, 1, 4, 2, 5, 3, 6).reshape(B, C, nf * pt, nh * ph, nw * pw)
        return out[:, :, :F, :H, :W], head
