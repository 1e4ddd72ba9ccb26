"""GPU numerics of the DiT kernels against plain PyTorch fp32 references.

Tolerances (bf16 operands, fp32 accumulation):
  GEMM       |D - ref| <= 2e-2 * max|ref| + 1e-2   (bf16 output rounding + K-long sums)
  attention  |O - ref| <= 2e-2                     (P in bf16, |O| <= max|V| ~ 3)
  DiT eps    rel. L2 error <= 5e-2 after 2 blocks  (bf16 activations through 2 blocks)
"""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2512_07350_b200 import _lib, lp

pytestmark = pytest.mark.gpu


def _gemm(A, B, bias):
    M, K = A.shape
    N = B.shape[0]
    D = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _lib.check(_lib.lib().lp_gemm_bf16(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()),
                                       C.c_void_p(bias.data_ptr()) if bias is not None else None,
                                       C.c_void_p(D.data_ptr()), M, N, K,
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return D


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 256, 128), (300, 1536, 1536), (130, 128, 4096),
                                   (1000, 64, 1536), (65, 4608, 1536), (4096, 8960, 1536), (2000, 1536, 8960)])
def test_gemm_matches_torch(cuda, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g)
    D = _gemm(A, B, bias).float()
    ref = A.float() @ B.float().t() + bias
    err = (D - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item() + 1e-2, err


@pytest.mark.parametrize("mode", [0, 1, 2, 3], ids=["bf16", "bf16-gelu", "f32-resid", "f32"])
@pytest.mark.parametrize("M,N,K", [(300, 1536, 1536), (1000, 8960, 512), (4097, 1536, 8960), (257, 256, 128)])
def test_gemm_fused_epilogues_match_torch(cuda, mode, M, N, K):
    """The DiT's fused epilogues (lp_gemm_bf16_epi): bias, tanh-GELU, fp32 gated residual."""
    g = torch.Generator(device="cuda").manual_seed(M + 3 * N + 7 * K + mode)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g)
    gate = torch.randn(N, device="cuda", generator=g)
    x0 = torch.randn(M, N, device="cuda", generator=g)
    D = x0.clone() if mode == 2 else torch.empty(M, N, device="cuda", dtype=torch.float32 if mode == 3 else torch.bfloat16)
    _lib.check(_lib.lib().lp_gemm_bf16_epi(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), C.c_void_p(bias.data_ptr()),
                                           C.c_void_p(gate.data_ptr()), C.c_void_p(D.data_ptr()), M, N, K, mode,
                                           C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    y = A.float() @ B.float().t() + bias
    ref = {0: y, 1: torch.nn.functional.gelu(y, approximate="tanh"), 2: x0 + gate * y, 3: y}[mode]
    err = (D.float() - ref).abs().max().item()
    assert err <= 2e-2 * ref.abs().max().item() + 1e-2, err


def _attn(q, k, v, scale):
    B, S, H, _ = q.shape
    Skv = k.shape[1]
    o = torch.empty_like(q)
    _lib.check(_lib.lib().lp_attention_bf16(C.c_void_p(q.data_ptr()), C.c_void_p(k.data_ptr()),
                                            C.c_void_p(v.data_ptr()), C.c_void_p(o.data_ptr()), B, S, Skv, H, scale,
                                            C.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return o


@pytest.mark.parametrize("mode", [0, 1], ids=["bf16", "bf16-gelu"])
@pytest.mark.parametrize("M,N,K", [(300, 1536, 1536), (1000, 8960, 512), (4097, 4608, 1536), (257, 256, 128)])
def test_gemm_two_subblock_stages_match_torch(cuda, mode, M, N, K):
    """CTA-pair GEMM with two 64-wide K sub-blocks per pipeline stage (knob gemm_ksub=2: 8 MMAs
    per full-barrier wait) vs torch fp32, and bit-identical to the one-sub-block pipeline (same
    MMAs in the same order)."""
    g = torch.Generator(device="cuda").manual_seed(M + 5 * N + K + mode)
    A = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    B = (torch.randn(N, K, device="cuda", generator=g) / K ** 0.5).bfloat16()
    bias = torch.randn(N, device="cuda", generator=g)
    outs = []
    for ks in (1, 2):
        _lib.check(_lib.lib().lp_tune(b"gemm_ksub", ks))
        D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        _lib.check(_lib.lib().lp_gemm_bf16_epi(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()),
                                               C.c_void_p(bias.data_ptr()), C.c_void_p(bias.data_ptr()),
                                               C.c_void_p(D.data_ptr()), M, N, K, mode,
                                               C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        outs.append(D)
    _lib.check(_lib.lib().lp_tune(b"gemm_ksub", 1))
    y = A.float() @ B.float().t() + bias
    ref = y if mode == 0 else torch.nn.functional.gelu(y, approximate="tanh")
    assert (outs[1].float() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item() + 1e-2
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("B,S,Skv,H", [(1, 128, 128, 1), (2, 200, 200, 3), (2, 300, 512, 2), (1, 1024, 1024, 2),
                                       (2, 1560, 1560, 12), (1, 129, 1000, 1)])
def test_attention_matches_torch(cuda, B, S, Skv, H):
    g = torch.Generator(device="cuda").manual_seed(S * 31 + Skv + H)
    q = torch.randn(B, S, H, 128, device="cuda", generator=g).bfloat16()
    k = torch.randn(B, Skv, H, 128, device="cuda", generator=g).bfloat16()
    v = torch.randn(B, Skv, H, 128, device="cuda", generator=g).bfloat16()
    scale = 1.0 / 128 ** 0.5
    o = _attn(q, k, v, scale).float()
    ref = torch.nn.functional.scaled_dot_product_attention(q.float().transpose(1, 2), k.float().transpose(1, 2),
                                                           v.float().transpose(1, 2)).transpose(1, 2)
    err = (o - ref).abs().max().item()
    assert err <= 2e-2, err


@pytest.mark.parametrize("knob", [b"attn_pair", b"attn_qtm"])
@pytest.mark.parametrize("B,S,H", [(1, 600, 1), (2, 1000, 3), (1, 1536, 2), (2, 1560, 12), (1, 130, 1)])
def test_attention_cta_pair_matches_torch(cuda, B, S, H, knob):
    """Self-attention on CTA pairs (knob attn_pair: cta_group::2, K split by rows and V by
    columns across the pair; knob attn_qtm: one Q tile per CTA resident in TMEM, S double-
    buffered) vs torch fp32 SDPA, and vs the single-CTA kernel.  Shapes cover an
    odd number of 256-row groups (the pair's second CTA past n_q), ragged key blocks and
    n_kv not a multiple of 64 (the second CTA's keys partly out of range)."""
    g = torch.Generator(device="cuda").manual_seed(S + 7 * H)
    q = torch.randn(B, S, H, 128, device="cuda", generator=g).bfloat16()
    k = torch.randn(B, S, H, 128, device="cuda", generator=g).bfloat16()
    v = torch.randn(B, S, H, 128, device="cuda", generator=g).bfloat16()
    scale = 1.0 / 128 ** 0.5
    single = _attn(q, k, v, scale).float()
    _lib.check(_lib.lib().lp_tune(knob, 1))
    try:
        o = _attn(q, k, v, scale).float()
        torch.cuda.synchronize()
    finally:
        _lib.check(_lib.lib().lp_tune(knob, 0))
    ref = torch.nn.functional.scaled_dot_product_attention(q.float().transpose(1, 2), k.float().transpose(1, 2),
                                                           v.float().transpose(1, 2)).transpose(1, 2)
    assert (o - ref).abs().max().item() <= 2e-2
    # same arithmetic per row as the single-CTA kernel: identical up to MMA accumulation order
    assert (o - single).abs().max().item() <= 1e-2


def test_attention_large_logits(cuda):
    # scores far from 0 exercise the lazy-rescale path (max jumps by > 8 in log2 units)
    g = torch.Generator(device="cuda").manual_seed(5)
    q = (torch.randn(1, 512, 1, 128, device="cuda", generator=g) * 4).bfloat16()
    k = (torch.randn(1, 512, 1, 128, device="cuda", generator=g) * 4).bfloat16()
    v = torch.randn(1, 512, 1, 128, device="cuda", generator=g).bfloat16()
    o = _attn(q, k, v, 1 / 128 ** 0.5).float()
    ref = torch.nn.functional.scaled_dot_product_attention(q.float().transpose(1, 2), k.float().transpose(1, 2),
                                                           v.float().transpose(1, 2)).transpose(1, 2)
    assert (o - ref).abs().max().item() <= 3e-2


def _oracle_ctx(dit, cond):
    """The oracle's own DiT: weights, text and cross-attention K/V regenerated from the pinned
    generator (oracle/dit_oracle.py) — nothing read back from the engine."""
    from oracle.dit_oracle import OracleDiT

    od = OracleDiT(dit.cfg, cond)
    ck, cv = od.context_kv()
    return od, ck, cv


def _dit_case(layers=2, shape=(16, 5, 16, 16), t=37, w=5.0):
    from tests.dit_reference import DiTReference

    z, cond = lp.synthetic_latent(shape, 4, 2025)
    dit = lp.DiTDenoiser(cond, num_layers=layers)
    eps = dit.cfg_predict(z, t, w)
    torch.cuda.synchronize()
    od, ck, cv = _oracle_ctx(dit, cond)
    want, head_ref = DiTReference(od).forward(z.data.float(), t, ck, cv, w)
    head = dit.debug_tensor("head", torch.float32).view(head_ref.shape)
    return eps, want, head, head_ref, dit


def test_dit_forward_matches_torch_fp32(cuda):
    eps, want, head, head_ref, _ = _dit_case()
    rel_head = ((head - head_ref).norm() / head_ref.norm()).item()
    rel = ((eps.data.float() - want).norm() / want.norm()).item()
    assert np.isfinite(rel) and rel <= 5e-2, (rel, rel_head)
    assert rel_head <= 5e-2


def test_dit_forward_odd_shard_shape(cuda):
    # remainder rows (W=19, H=9 not multiples of the patch) are zero-padded and cropped
    eps, want, _, _, _ = _dit_case(layers=1, shape=(16, 3, 9, 19), t=3, w=2.0)
    rel = ((eps.data.float() - want).norm() / want.norm()).item()
    assert rel <= 5e-2, rel


@pytest.mark.parametrize("kw", [dict(num_layers=2), dict(num_layers=1, dim=5120, ffn_dim=13824, num_heads=40)],
                         ids=["1.3B-2blocks", "14B-1block"])
def test_dit_params_bit_exact_vs_oracle_generator(cuda, kw):
    """Every engine parameter (k_init_param on the device) equals the oracle's host-side restatement
    of the pinned generator bit for bit (oracle/dit_oracle.py: splitmix64 hash, fma init rule, bf16 RNE)."""
    from oracle.dit_oracle import OracleDiT

    _, cond = lp.synthetic_latent_host((16, 3, 4, 4), 4, 2025)
    dit = lp.DiTDenoiser(list(cond), **kw)
    od = OracleDiT(dit.cfg, list(cond))
    mine, theirs = dit.params(), od.params()
    assert list(mine) == list(theirs)  # same names, same order
    for n, v in mine.items():
        o = theirs[n]
        assert v.dtype == o.dtype and v.numel() == o.numel(), n
        iv = torch.int16 if v.dtype == torch.bfloat16 else torch.int32
        assert torch.equal(v.view(iv), o.view(iv)), n


@pytest.mark.parametrize("d", [2, 4, 8])
def test_dit_single_pass_predict_reproduces_cfg_batch(cuda, d):
    """Denoiser::predict of the DiT (one CFG pass, lp_dit_predict) is bit-identical to the matching
    half of the CFG-batched forward: the reference's cfg_predict over two predict calls
    (src/denoise.cpp:24-39: u + w (c - u) in fp64 over quantized passes, quantized) equals the
    fused lp_dit_cfg_predict bit for bit, in every storage dtype."""
    z, cond = lp.synthetic_latent((16, 5, 16, 16), d, 2025)
    dit = lp.DiTDenoiser(cond, num_layers=2)
    t, w = 37, 5.0
    fused = dit.cfg_predict(z, t, w).to_numpy()
    u = dit.predict(z, t, null_text=True).to_numpy()
    c = dit.predict(z, t, null_text=False).to_numpy()
    want = lp._quantize_np(u + w * (c - u), d)
    assert np.array_equal(fused, want)
    assert not np.array_equal(u, c)


def test_dit_single_pass_predict_vs_oracle(cuda):
    from tests.dit_reference import DiTReference

    z, cond = lp.synthetic_latent((16, 5, 16, 16), 4, 2025)
    dit = lp.DiTDenoiser(cond, num_layers=2)
    od, ck, cv = _oracle_ctx(dit, cond)
    ref = DiTReference(od)
    for b in (0, 1):
        got = dit.predict(z, 21, null_text=(b == 0)).data.float()
        want = ref.predict(z.data.float(), 21, ck, cv, b).float()
        rel = ((got - want).norm() / want.norm()).item()
        assert np.isfinite(rel) and rel <= 5e-2, (b, rel)


@pytest.mark.parametrize("shape,t", [((16, 5, 16, 16), 37), ((16, 9, 30, 52), 4)])
def test_lnfold_matches_layernorm_path_and_oracle(cuda, shape, t):
    """The LayerNorm fold (knob dit_lnfold: LN partials + xq = bf16(x * g) written by the residual
    GEMM epilogues, rstd * (acc - mean * cs) + b' in the next GEMM's epilogue) against the
    separate-LayerNorm path and the fp32 oracle.  Both paths round differently (xq vs the
    normalised h), so the bound is bf16-level, not bitwise."""
    from tests.dit_reference import DiTReference

    z, cond = lp.synthetic_latent(shape, 4, 2025)
    dit = lp.DiTDenoiser(cond, num_layers=2)
    outs = {}
    for on in (0, 1):
        _lib.check(_lib.lib().lp_tune(b"dit_lnfold", on))
        outs[on] = dit.cfg_predict(z, t, 5.0).data.float().clone()
    _lib.check(_lib.lib().lp_tune(b"dit_lnfold", 0))  # the default
    rel = ((outs[1] - outs[0]).norm() / outs[0].norm()).item()
    assert np.isfinite(rel) and rel <= 2e-2, rel
    od, ck, cv = _oracle_ctx(dit, cond)
    want, _ = DiTReference(od).forward(z.data.float(), t, ck, cv, 5.0)
    for on in (0, 1):
        r = ((outs[on] - want).norm() / want.norm()).item()
        assert r <= 5e-2, (on, r)


def test_block0_self_attention_dedupe_is_bit_identical(cuda):
    """Block 0's self-attention sub-block runs once for the two identical CFG halves (knob
    dit_dedupe0); the result equals the duplicated computation bit for bit."""
    z, cond = lp.synthetic_latent((16, 5, 16, 16), 4, 2025)
    dit = lp.DiTDenoiser(cond, num_layers=2)
    outs = []
    for on in (0, 1):
        _lib.check(_lib.lib().lp_tune(b"dit_dedupe0", on))
        outs.append(dit.cfg_predict(z, 9, 5.0).data.clone())
    _lib.check(_lib.lib().lp_tune(b"dit_dedupe0", 1))
    assert torch.equal(outs[0], outs[1])


def test_row_order_reversal_is_bit_identical(cuda):
    """LayerNorm and q/k RMSNorm+RoPE passes walking rows last-to-first (knob row_rev, for L2
    reuse with the neighbouring GEMMs) give the same bits as the forward order."""
    z, cond = lp.synthetic_latent((16, 5, 16, 16), 4, 2025)
    dit = lp.DiTDenoiser(cond, num_layers=2)
    outs = []
    for on in (0, 1):
        _lib.check(_lib.lib().lp_tune(b"row_rev", on))
        outs.append(dit.cfg_predict(z, 9, 5.0).data.clone())
    _lib.check(_lib.lib().lp_tune(b"row_rev", 0))
    assert torch.equal(outs[0], outs[1])


def test_text_context_kv_all_layers_vs_oracle(cuda):
    """The cached cross-attention K/V of all 30 layers, uncond (null text) and cond (synthetic
    text) halves, vs the oracle's fp32 restatement: its own text generator, text MLP, K/V
    projections and K RMSNorm.  Tolerance: rel. L2 <= 2e-2 per layer and half (bf16 GEMM chain:
    text -> MLP (2 GEMMs) -> projection, each output rounded to bf16)."""
    _, cond = lp.synthetic_latent_host((16, 3, 4, 4), 4, 2025)
    dit = lp.DiTDenoiser(list(cond))
    od, ck, cv = _oracle_ctx(dit, list(cond))
    T = dit.cfg.text_len
    worst = 0.0
    for l in range(dit.cfg.num_layers):
        k = dit.debug_tensor(f"ctx_k.{l}", torch.bfloat16).float().view(2, T, -1)
        v = dit.debug_tensor(f"ctx_v.{l}", torch.bfloat16).float().view(2, T, -1)
        for b in (0, 1):
            for got, want in ((k[b], ck[l][b]), (v[b], cv[l][b])):
                rel = ((got - want).norm() / want.norm()).item()
                worst = max(worst, rel)
                assert np.isfinite(rel) and rel <= 2e-2, (l, b, rel)
    # the cond half really is the synthetic text (not zeros): the halves differ
    assert ((ck[0][1] - ck[0][0]).norm() / ck[0][0].norm()).item() > 0.1


def test_engine_dit_step_runs(cuda):
    z, cond = lp.synthetic_latent((16, 5, 16, 16), 4, 2025)
    dit = lp.DiTDenoiser(cond, num_layers=2)
    eng = lp.LpEngine((16, 5, 16, 16), (1, 2, 2), 4, 2, 0.5, 3, 0.05, 5.0, cond, denoiser="dit", dit=dit)
    eng.load(z)
    eng.run(1, 3)
    torch.cuda.synchronize()
    assert torch.isfinite(eng.z.data).all()
    assert eng.launches() > 0


def test_engine_dit_remainder_shard_shapes(cuda):
    """Shards that keep the reference's remainder rows (H=17 with patch 2) need ceil(H/p) token
    rows: the engine reserves the DiT workspace with the DiT's own patch and ceil division
    (ADVICE r1), so the forward never exceeds its reservation."""
    dims = (16, 5, 17, 16)
    z, cond = lp.synthetic_latent(dims, 4, 2025)
    dit = lp.DiTDenoiser(cond, num_layers=1)
    eng = lp.LpEngine(dims, (1, 2, 2), 4, 2, 0.5, 3, 0.05, 5.0, cond, denoiser="dit", dit=dit)
    eng.load(z)
    eng.run(1, 3)
    eng.sync(timeout_s=120)
    assert torch.isfinite(eng.z.data).all()
    eng.close()
    # an LP patch coarser than the DiT's: (1,4,4) LP windows on a (1,2,2) DiT
    eng = lp.LpEngine(dims, (1, 4, 4), 4, 2, 0.5, 3, 0.05, 5.0, cond, denoiser="dit", dit=dit)
    eng.load(z)
    eng.run(1, 3)
    eng.sync(timeout_s=120)
    assert torch.isfinite(eng.z.data).all()
    eng.close()


def test_lp_loop_with_dit_matches_reference_run_lp(cuda, reference):
    """The UNMODIFIED reference run_lp (oracle/_ref) driving the oracle's fp32 torch DiT through
    its Denoiser plugin slot, vs our engine (bf16 tcgen05 DiT, CFG batch 2, K1/K10 kernels).
    Tolerance: rel. L2 of the latent update <= 5e-2, max |dz| <= 1e-2 after 3 steps."""
    from tests.dit_reference import DiTReference

    dims, steps, K, r, eta, w = (16, 5, 16, 16), 3, 2, 0.5, 0.05, 5.0
    z, cond = lp.synthetic_latent(dims, 4, 2025)
    dit = lp.DiTDenoiser(cond, num_layers=2)
    od, ck, cv = _oracle_ctx(dit, cond)
    ref = DiTReference(od)

    def predict(zz, t, c, is_null):
        x = torch.from_numpy(zz).float().cuda()
        return ref.predict(x, t, ck, cv, 0 if is_null else 1).double().cpu().numpy()

    z0 = z.to_numpy()
    import os

    os.environ["LPSIM_THREADS"] = "0"  # serial worker pool: the callback drives the GPU from this thread
    want, ledger_ref = reference.run_lp_callback(predict, z0, 4, steps, eta, w, cond, (1, 2, 2), K, r)
    got, led = lp.run_lp("dit", (0, 0, 0), z, steps, eta, w, cond, (1, 2, 2), K, r, dit=dit)
    got = got.to_numpy()
    assert led["grand_total"] == ledger_ref
    rel = np.linalg.norm(got - want) / np.linalg.norm(want - z0)
    assert np.isfinite(rel) and rel <= 5e-2, rel
    assert np.abs(got - want).max() <= 1e-2


def test_dit_14b_shape_forward_matches_torch(cuda):
    """BASELINE config C4's DiT shape (WAN2.1-14B: d=5120, 40 heads, FFN 13824), one block."""
    from tests.dit_reference import DiTReference

    z, cond = lp.synthetic_latent((16, 3, 8, 12), 4, 7)
    dit = lp.DiTDenoiser(cond, dim=5120, ffn_dim=13824, num_heads=40, num_layers=1)
    eps = dit.cfg_predict(z, 11, 5.0)
    torch.cuda.synchronize()
    od, ck, cv = _oracle_ctx(dit, cond)
    want, _ = DiTReference(od).forward(z.data.float(), 11, ck, cv, 5.0)
    rel = ((eps.data.float() - want).norm() / want.norm()).item()
    assert np.isfinite(rel) and rel <= 5e-2, rel


def test_engine_graph_replay_bit_identical_to_eager(cuda):
    """DiT engines replay each axis's step as a captured CUDA graph (timestep written to the
    device before each replay); 7 steps cover capture (2nd occurrence) and replays of every
    axis and must match the eager launches bit for bit."""
    from paper_2512_07350_b200 import _lib

    z, cond = lp.synthetic_latent((16, 5, 16, 16), 4, 2025)
    dit = lp.DiTDenoiser(list(cond), num_layers=2)
    outs = []
    for graph in (0, 1):
        _lib.check(_lib.lib().lp_tune(b"engine_graph", graph))
        eng = lp.LpEngine((16, 5, 16, 16), (1, 2, 2), 4, 4, 0.5, 7, 0.05, 5.0, list(cond), denoiser="dit", dit=dit)
        eng.load(z)
        l0 = eng.launches()
        eng.run(1, 7)
        torch.cuda.synchronize()
        outs.append((eng.z.data.clone(), eng.launches() - l0, eng.comm()["ledger_bytes"]))
        eng.close()
    _lib.check(_lib.lib().lp_tune(b"engine_graph", 1))
    assert torch.equal(outs[0][0], outs[1][0])
    assert outs[0][2] == outs[1][2]  # same ledger either way
    # kernel counts differ only by the timestep writes (per forward eagerly, per slot before a replay)
    assert abs(outs[0][1] - outs[1][1]) <= 7 * 4



@pytest.mark.parametrize("shape", [(16, 5, 16, 16), (16, 3, 9, 19), (16, 9, 60, 104)])
def test_qk_rope_table_path_matches_per_element_path(cuda, shape):
    """q/k RMSNorm+RoPE has two independent implementations: the table kernel (per-lane
    (cos, sin) pairs hoisted per row; the default) and the per-element kernel (knob
    `rope_tab` 0).  Index errors in either would rotate the wrong pairs and move the DiT
    output by O(1); the two agree to bf16 rounding (different reduction order)."""
    z, cond = lp.synthetic_latent(shape, 4, 2025)
    dit = lp.DiTDenoiser(cond, num_layers=1)
    outs = []
    for tab in (0, 1):
        _lib.check(_lib.lib().lp_tune(b"rope_tab", tab))
        outs.append(dit.cfg_predict(z, 37, 5.0).data.clone().float())
        torch.cuda.synchronize()
    _lib.check(_lib.lib().lp_tune(b"rope_tab", 1))
    rel = ((outs[0] - outs[1]).norm() / outs[0].norm()).item()
    assert np.isfinite(rel) and rel <= 5e-3, rel
