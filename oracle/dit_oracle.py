"""The DiT's parameters and synthetic text context restated from the engine's pinned generator
(TEST INFRASTRUCTURE ONLY: the tolerance oracle of the DiT tests; the product never imports it).

The reference (lpsim) has no DiT ("parity unpinned"), so the DiT's weights and
its text context are builder-defined, by a pinned generator in the engine:

* weights — paper_2512_07350_b200/csrc/dit.cpp `lp_dit_create` (parameter list, order and the
  init rule per name) and dit_kernels.cu `k_init_param`: value = fma(u, scale, offset) in fp32
  (one rounding: the SASS is FFMA), u = hash_uniform(seed, param_index + 1, element), bf16 by
  round-to-nearest-even for the GEMM operands;
* hash_uniform — dit_kernels.cu:17-26: splitmix64(splitmix64(seed ^ stream * 0xD1B54A32D192ED03)
  + i), top 24 bits -> [-1, 1) exactly;
* text context — dit.cpp (seed = seed * 0x9E3779B97F4A7C15, then (seed ^ bits(c_i)) * FNV prime
  over the ConditioningVector values) and dit_kernels.cu `k_text_context`: Box-Muller on two hash
  uniforms of stream 0x7e47 in fp32, bf16; the uncond (null-text) rows are zeros.

This module regenerates all of it independently (torch int64 / fp64 arithmetic, on any
device), so the DiT tests compare the engine against weights, text and cross-attention K/V the
oracle computed itself — never against tensors read back from the engine.
"""
from __future__ import annotations

import math
import struct
from types import SimpleNamespace

import torch

_M64 = (1 << 64) - 1


def _s64(x: int) -> int:
    """python int (mod 2^64) -> the int64 with the same bits."""
    x &= _M64
    return x - (1 << 64) if x >= (1 << 63) else x


def _splitmix64_int(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def _srl(x: torch.Tensor, k: int) -> torch.Tensor:
    """logical right shift of int64 bit patterns."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def _splitmix64_t(x: torch.Tensor) -> torch.Tensor:
    x = x + _s64(0x9E3779B97F4A7C15)
    x = (x ^ _srl(x, 30)) * _s64(0xBF58476D1CE4E5B9)
    x = (x ^ _srl(x, 27)) * _s64(0x94D049BB133111EB)
    return x ^ _srl(x, 31)


def hash_uniform(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """dit_kernels.cu hash_uniform for int64 element indices -> fp32 in [-1, 1) (exact)."""
    base = _splitmix64_int((seed ^ (stream * 0xD1B54A32D192ED03)) & _M64)
    h = _splitmix64_t(idx + _s64(base))
    return (_srl(h, 40).double() * (1.0 / 8388608.0) - 1.0).float()


def hash_uniform_int(seed: int, stream: int, i: int) -> float:
    """Scalar restatement with python ints (pins the tensor version in the CPU tests)."""
    base = _splitmix64_int((seed ^ (stream * 0xD1B54A32D192ED03)) & _M64)
    h = _splitmix64_int((base + i) & _M64)
    return (h >> 40) * (1.0 / 8388608.0) - 1.0


def param_table(cfg):
    """(name, numel, bf16?, scale, offset) in lp_dit_create's order (dit.cpp `add` calls and the
    init rule: weights sqrt(3/fan_in) u, norm gains 1 + 0.1u, modulation sqrt(3/d) u, else 0.02u)."""
    d, F, L = cfg.dim, cfg.ffn_dim, cfg.num_layers
    pfeat = cfg.in_channels * cfg.patch[0] * cfg.patch[1] * cfg.patch[2]
    rows = [("patch.w", d * pfeat, 2), ("patch.b", d, 4), ("text.w1", d * cfg.text_dim, 2), ("text.b1", d, 4),
            ("text.w2", d * d, 2), ("text.b2", d, 4), ("time.w1", d * cfg.freq_dim, 2), ("time.b1", d, 4),
            ("time.w2", d * d, 2), ("time.b2", d, 4), ("time.wp", 6 * d * d, 2), ("time.bp", 6 * d, 4),
            ("blocks.mod", L * 6 * d, 4)]
    for l in range(L):
        p = f"blocks.{l}."
        rows += [(p + "qkv.w", 3 * d * d, 2), (p + "qkv.b", 3 * d, 4), (p + "norm_q", d, 4), (p + "norm_k", d, 4),
                 (p + "o.w", d * d, 2), (p + "o.b", d, 4), (p + "norm3.w", d, 4), (p + "norm3.b", d, 4),
                 (p + "cq.w", d * d, 2), (p + "cq.b", d, 4), (p + "ck.w", d * d, 2), (p + "ck.b", d, 4),
                 (p + "cv.w", d * d, 2), (p + "cv.b", d, 4), (p + "cnorm_q", d, 4), (p + "cnorm_k", d, 4),
                 (p + "co.w", d * d, 2), (p + "co.b", d, 4), (p + "ffn1.w", F * d, 2), (p + "ffn1.b", F, 4),
                 (p + "ffn2.w", d * F, 2), (p + "ffn2.b", d, 4)]
    rows += [("head.mod", 2 * d, 4), ("head.w", pfeat * d, 2), ("head.b", pfeat, 4)]
    out = []
    f32 = lambda v: struct.unpack("f", struct.pack("f", v))[0]  # noqa: E731  (the kernel's float args)
    for n, numel, elem in rows:
        scale, offset = f32(0.02), 0.0
        if n.endswith(".w") and elem == 2:
            fan = {"patch.w": pfeat, "text.w1": cfg.text_dim, "time.w1": cfg.freq_dim}.get(n, F if n.endswith("ffn2.w") else d)
            scale = f32(math.sqrt(3.0 / fan))
        elif n.endswith(("norm_q", "norm_k", "norm3.w", "cnorm_q", "cnorm_k")):
            scale, offset = f32(0.1), 1.0
        elif n.endswith(".mod") or n == "time.wp":
            scale = f32(math.sqrt(3.0 / d))
        out.append((n, numel, elem == 2, scale, offset))
    return out


def generate_param(cfg, index, numel, bf16, scale, offset, device, chunk=1 << 24):
    """k_init_param for parameter `index` (stream index + 1): fma(u, scale, offset) with one
    rounding to fp32 (u * scale is exact in fp64 and the sum has <= 51 significant bits), then
    bf16 round-to-nearest-even for the GEMM operands."""
    out = torch.empty(numel, dtype=torch.bfloat16 if bf16 else torch.float32, device=device)
    for a in range(0, numel, chunk):
        i = torch.arange(a, min(numel, a + chunk), dtype=torch.int64, device=device)
        u = hash_uniform(int(cfg.seed), index + 1, i).double()
        v = (u * scale + offset).float()
        out[a:a + i.numel()] = v.to(out.dtype)
    return out


def text_seed(seed: int, cond) -> int:
    t = (seed * 0x9E3779B97F4A7C15) & _M64
    for c in cond:
        bits = struct.unpack("<Q", struct.pack("<d", float(c)))[0]
        t = ((t ^ bits) * 0x100000001B3) & _M64
    return t


def text_input(cfg, cond, device):
    """[2, text_len, text_dim] bf16: uncond = zeros (the null ConditioningVector, src/denoise.cpp:10-15),
    cond = k_text_context's Box-Muller in fp32 on hash uniforms of stream 0x7e47."""
    T, D = cfg.text_len, cfg.text_dim
    out = torch.zeros(2, T * D, dtype=torch.bfloat16, device=device)
    s = text_seed(int(cfg.seed), cond)
    i = torch.arange(T * D, dtype=torch.int64, device=device)
    u1 = 0.5 * (hash_uniform(s, 0x7E47, 2 * i) + 1.0)
    u2 = 0.5 * (hash_uniform(s, 0x7E47, 2 * i + 1) + 1.0)
    r = torch.sqrt(-2.0 * torch.log(torch.clamp(u1, min=1e-7)))
    out[1] = (r * torch.cos(torch.tensor(6.283185307179586, dtype=torch.float32) * u2)).to(torch.bfloat16)
    return out.view(2, T, D)


class OracleDiT:
    """The DiT as the oracle regenerates it: .cfg and .params() (the interface DiTReference
    consumes), .text_input() and .context_kv() (cross-attention K/V per layer, both CFG halves)."""

    FIELDS = ("in_channels", "dim", "ffn_dim", "num_heads", "num_layers", "text_len", "text_dim", "freq_dim", "eps",
              "t_scale", "seed")

    def __init__(self, cfg, cond, device="cuda"):
        self.cfg = SimpleNamespace(**{f: getattr(cfg, f) for f in self.FIELDS}, patch=tuple(cfg.patch))
        self.cond = list(cond)
        self.device = device
        self._p = {}
        for idx, (n, numel, bf16, scale, offset) in enumerate(param_table(self.cfg)):
            self._p[n] = generate_param(self.cfg, idx, numel, bf16, scale, offset, device)
        self._kv = None

    def params(self):
        return self._p

    def text_input(self):
        return text_input(self.cfg, self.cond, self.device)

    @torch.no_grad()
    def context_kv(self):
        """fp32 restatement of lp_dit_create's text MLP (GELU-tanh) and per-layer cross K (+ RMSNorm)
        and V projections: lists of [2, text_len, d] (row 0 = uncond, 1 = cond)."""
        if self._kv is None:
            from oracle.dit_fp32 import rms

            c, p = self.cfg, {k: v.float() for k, v in self._p.items() if k.startswith(("text.", "blocks."))}
            d = c.dim
            x = self.text_input().float()
            h = torch.nn.functional.gelu(x @ p["text.w1"].view(d, -1).t() + p["text.b1"], approximate="tanh")
            ctx = h @ p["text.w2"].view(d, d).t() + p["text.b2"]
            ck, cv = [], []
            for l in range(c.num_layers):
                pre = f"blocks.{l}."
                ck.append(rms(ctx @ p[pre + "ck.w"].view(d, d).t() + p[pre + "ck.b"], p[pre + "cnorm_k"], c.eps))
                cv.append(ctx @ p[pre + "cv.w"].view(d, d).t() + p[pre + "cv.b"])
            self._kv = (ck, cv)
        return self._kv
