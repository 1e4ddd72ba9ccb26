"""The oracle's restatement of the DiT's pinned generator (oracle/dit_oracle.py), on CPU: the
vectorised torch int64 splitmix64 / hash_uniform equals a python-int restatement, the parameter
table has lp_dit_create's layout, and the text generator is deterministic in the cond values.
(The engine's own parameter bits are compared with it on the GPU: tests/test_dit_gpu.py.)"""
from types import SimpleNamespace

import torch

from oracle.dit_oracle import generate_param, hash_uniform, hash_uniform_int, param_table, text_input, text_seed

CFG = SimpleNamespace(in_channels=16, dim=256, ffn_dim=512, num_heads=2, num_layers=2, text_len=8, text_dim=64,
                      freq_dim=32, patch=(1, 2, 2), eps=1e-6, t_scale=20.0, seed=2025)


def test_hash_uniform_tensor_equals_python_ints():
    idx = torch.tensor([0, 1, 2, 12345, (1 << 31) + 7, (1 << 40) + 3], dtype=torch.int64)
    for seed, stream in ((2025, 1), (42, 977), (0xFFFFFFFFFFFF, 0x7E47)):
        got = hash_uniform(seed, stream, idx)
        want = torch.tensor([hash_uniform_int(seed, stream, int(i)) for i in idx], dtype=torch.float64)
        assert torch.equal(got.double(), want)
        assert (got >= -1).all() and (got < 1).all()


def test_param_table_layout():
    t = param_table(CFG)
    assert len(t) == 13 + 22 * CFG.num_layers + 3
    names = [r[0] for r in t]
    assert names[:3] == ["patch.w", "patch.b", "text.w1"] and names[-1] == "head.b"
    rule = {r[0]: r[3:] for r in t}
    assert rule["blocks.0.norm_q"][1] == 1.0 and abs(rule["blocks.0.norm_q"][0] - 0.1) < 1e-7
    assert abs(rule["blocks.1.ffn2.w"][0] - (3 / CFG.ffn_dim) ** 0.5) < 1e-7
    assert abs(rule["time.wp"][0] - (3 / CFG.dim) ** 0.5) < 1e-7
    assert rule["blocks.0.norm3.b"] == (rule["patch.b"][0], 0.0)


def test_generate_param_fma_rule_and_ranges():
    s = torch.tensor(0.1, dtype=torch.float32).item()          # the kernel's float argument 0.1f
    v = generate_param(CFG, 7, 4096, False, s, 1.0, "cpu")     # a norm gain: 1 + 0.1 u in [0.9, 1.1)
    assert v.dtype == torch.float32 and (v >= 0.9).all() and (v < 1.1).all()
    u = hash_uniform(CFG.seed, 8, torch.arange(4096))
    # fma(u, s, 1): exact in fp64, one rounding to fp32; two roundings (mul, then add) differ somewhere
    assert torch.equal(v, (u.double() * s + 1.0).float())
    assert not torch.equal(v, (u * torch.tensor(s, dtype=torch.float32)) + 1.0)
    w = generate_param(CFG, 0, 1000, True, 0.25, 0.0, "cpu")
    assert w.dtype == torch.bfloat16 and w.float().abs().max() <= 0.25


def test_text_input_uncond_zero_cond_normal():
    x = text_input(CFG, [0.1 * i for i in range(8)], "cpu")
    assert x.shape == (2, CFG.text_len, CFG.text_dim) and x.dtype == torch.bfloat16
    assert (x[0] == 0).all()
    c = x[1].float()
    assert abs(c.mean().item()) < 0.2 and 0.7 < c.std().item() < 1.3
    assert text_seed(2025, [1.0]) != text_seed(2025, [2.0])
