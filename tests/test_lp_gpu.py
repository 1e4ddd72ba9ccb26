"""GPU parity of the LP kernels (K1 gather, K10 reconstruct+sampler, K11 toy
denoisers) and the engine loop against the CPU oracle — bit-exact (integer /
byte work and the fp64 "exact" path)."""
import hashlib

import numpy as np
import pytest

from oracle.oracle import sub_shape
from paper_2512_07350_b200 import lp

pytestmark = pytest.mark.gpu
H = lambda a: hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()[:16]  # noqa: E731


def _cases(seed, n):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        shape = tuple(int(v) for v in (rng.integers(1, 5), rng.integers(1, 14), rng.integers(1, 14), rng.integers(1, 14)))
        patch = tuple(int(v) for v in rng.integers(1, 4, size=3))
        k = int(rng.integers(1, 9))
        r = float(min(rng.choice([0.0, 0.25, 0.5, 1.0, 1.5]), k - 1))
        step = int(rng.integers(1, 4))
        d = int(rng.choice([2, 4, 8]))
        try:
            lp.build_plan(shape, patch, step, k, r)
        except lp.LpError:
            continue
        out.append((shape, patch, k, r, step, d, int(rng.integers(0, 1 << 30))))
    return out


def test_extract_bitexact(cuda, oracle):
    for shape, patch, k, r, step, d, seed in _cases(1, 60):
        z, _ = oracle.synthetic(shape, d, seed)
        plan = lp.build_plan(shape, patch, step, k, r)
        subs = lp.extract_sublatents(lp.LatentTensor.from_numpy(z, d), plan)
        want = oracle.extract(z, oracle.build_plan(shape, patch, step, k, r))
        got = np.concatenate([s.to_numpy().reshape(-1) for s in subs])
        assert np.array_equal(got, want), (shape, patch, k, r, step, d)


@pytest.mark.parametrize("d", [2, 4, 8])
@pytest.mark.parametrize("dims,k,r", [((16, 21, 60, 104), 4, 0.5), ((3, 7, 12, 40), 3, 1.0), ((2, 5, 9, 24), 8, 0.25),
                                      ((16, 41, 60, 104), 8, 0.5)])
def test_extract_tma_paths_bitexact(cuda, oracle, d, dims, k, r):
    """K1's TMA-staged forms (W axis: tensor-map boxes of R rows, repacked from shared memory;
    T/H axes: 1-D bulk copies) against the oracle and against the vector-copy kernel
    (knob gather_tma=0), all entries in one launch, on shapes whose geometry admits them."""
    from paper_2512_07350_b200 import _lib

    import ctypes as C

    import torch

    z, _ = oracle.synthetic(dims, d, 7)
    zt = lp.LatentTensor.from_numpy(z, d)
    L = _lib.lib()

    def packed(plan):  # every entry in ONE launch (the engine's K1), packed in entry order
        n = sum(int(np.prod(plan.sub_shape(dims, e))) for e in range(plan.workers))
        out = lp.LatentTensor(torch.empty(n, dtype=zt.data.dtype, device="cuda"), d)
        _lib.check(L.lp_extract(C.byref(plan.raw), 0, plan.workers, zt.ptr(), _lib.i64arr(dims), d, out.ptr(),
                                C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return out.to_numpy()

    for step in (1, 2, 3):
        plan = lp.build_plan(dims, (1, 2, 2), step, k, r)
        want = oracle.extract(z, oracle.build_plan(dims, (1, 2, 2), step, k, r))
        assert np.array_equal(packed(plan), want), (dims, step, d)
        one = np.concatenate([s.to_numpy().reshape(-1) for s in lp.extract_sublatents(zt, plan)])
        assert np.array_equal(one, want), (dims, step, d)
        _lib.check(L.lp_tune(b"gather_tma", 0))
        try:
            ref = packed(plan)
        finally:
            _lib.check(L.lp_tune(b"gather_tma", 1))
        assert np.array_equal(ref, want), (dims, step, d)


def test_toy_denoisers_bitexact(cuda, oracle):
    for shape, patch, k, r, step, d, seed in _cases(2, 40):
        z, cond = oracle.synthetic(shape, d, seed)
        zt = lp.LatentTensor.from_numpy(z, d)
        for kind, f in [(0, lp.BoxDenoiser((1, 2, 0))), (1, lp.GlobalMixDenoiser()), (2, lp.IdentityDenoiser())]:
            radius = f.radius
            t = 1 + seed % 50
            got = lp.cfg_predict(f, zt, t, list(cond), 5.0).to_numpy()
            want = oracle.cfg_predict(kind, radius, z, d, t, cond, 5.0)
            assert np.array_equal(got, want), (kind, shape, d)
            got = lp.denoiser_predict(f, zt, t, cond).to_numpy()
            want = oracle.toy_predict(kind, radius, z, d, t, float(np.mean(cond)) if False else sum(cond) / 8,
                                      t_coeff=f.t_coeff, cond_coeff=f.cond_coeff)
            if kind == 2:
                want = z
            assert np.array_equal(got, want), (kind, shape, d)


def test_reconstruct_and_update_bitexact(cuda, oracle):
    for shape, patch, k, r, step, d, seed in _cases(3, 60):
        z, cond = oracle.synthetic(shape, d, seed)
        plan = lp.build_plan(shape, patch, step, k, r)
        oplan = oracle.build_plan(shape, patch, step, k, r)
        rng = np.random.default_rng(seed)
        preds_np = [lp._quantize_np(rng.normal(size=sub_shape(shape, oplan, e)) * 3, d).astype(np.float64)
                    for e in range(oplan.n)]
        preds = [lp.LatentTensor.from_numpy(p, d) for p in preds_np]
        packed = np.concatenate([p.reshape(-1) for p in preds_np])
        want = oracle.reconstruct(packed, shape, d, oplan)
        got = lp.reconstruct(preds, plan, shape).to_numpy()
        assert np.array_equal(got, want), (shape, patch, k, r, step, d)
        zt = lp.LatentTensor.from_numpy(z, d)
        lp.reconstruct_update(preds, plan, zt, 0.05)
        assert np.array_equal(zt.to_numpy(), oracle.sampler_step(z, want, d, 0.05))
        fast = lp.reconstruct(preds, plan, shape, mode="fast").to_numpy()
        tol = {2: 2e-3, 4: 2e-6, 8: 2e-6}[d]
        np.testing.assert_allclose(fast, want, rtol=tol, atol=tol * 4)


def test_sampler_bitexact(cuda, oracle):
    for d in (2, 4, 8):
        z, _ = oracle.synthetic((3, 5, 7, 9), d, 1)
        e, _ = oracle.synthetic((3, 5, 7, 9), d, 2)
        got = lp.sampler_step(lp.LatentTensor.from_numpy(z, d), lp.LatentTensor.from_numpy(e, d), 1, 0.1).to_numpy()
        assert np.array_equal(got, oracle.sampler_step(z, e, d, 0.1))


@pytest.mark.parametrize("d,hash_", [(4, "3ad2d84ae75b30e9"), (8, "e7cbc9b6807bca2e")])
def test_engine_golden_crit1(cuda, d, hash_):
    # crit-1 config: 4x12x16x16 seed 2025, box rho=2, K=2, r=1, 6 steps, eta .05, w 2, p=2
    z, cond = lp.synthetic_latent((4, 12, 16, 16), d, 2025)
    out, ledger = lp.run_lp("box", (2, 2, 2), z, 6, 0.05, 2.0, cond, (2, 2, 2), 2, 1.0)
    assert H(out.to_numpy()) == hash_
    assert ledger["grand_total"] == 589824


def test_engine_golden_desk_default_and_c1(cuda):
    z, cond = lp.synthetic_latent((4, 12, 16, 16), 4, 42)
    out, ledger = lp.run_lp("box", (1, 1, 1), z, 60, 0.05, 3.0, cond, (2, 2, 2), 4, 0.5)
    assert H(out.to_numpy()) == "18f78847365f6597" and ledger["grand_total"] == 7700480
    z, cond = lp.synthetic_latent((16, 5, 16, 16), 4, 2025)
    out, ledger = lp.run_lp("box", (1, 1, 1), z, 4, 0.05, 5.0, cond, (1, 2, 2), 2, 0.5)
    assert H(out.to_numpy()) == "93a6824b0e691fdc" and ledger["grand_total"] == 442368


def test_engine_matches_oracle_sweep(cuda, oracle):
    for shape, patch, k, r, step, d, seed in _cases(4, 16):
        try:
            for s in (1, 2, 3):
                lp.build_plan(shape, patch, s, k, r)
        except lp.LpError:
            continue
        z, cond = oracle.synthetic(shape, d, seed)
        for kind, name in [(0, "box"), (1, "global"), (2, "identity")]:
            radius = (1, 0, 2)
            want, lw = oracle.run_lp(kind, radius, z, d, 4, 0.05, 3.0, cond, patch, k, r)
            got, lg = lp.run_lp(name, radius, lp.LatentTensor.from_numpy(z, d), 4, 0.05, 3.0, list(cond), patch, k, r)
            assert np.array_equal(got.to_numpy(), want) and lg["grand_total"] == lw, (name, shape, patch, k, r, d)


def test_single_worker_equals_centralized(cuda, reference):
    z, cond = lp.synthetic_latent((1, 8, 8, 8), 4, 11)
    central = reference.run_centralized(0, (1, 1, 1), z.to_numpy(), 4, 3, 0.1, 2.0, cond)
    final, ledger = lp.run_lp("box", (1, 1, 1), z, 3, 0.1, 2.0, cond, (2, 2, 2), 1, 0.0)
    assert ledger["grand_total"] == 0
    assert np.array_equal(final.to_numpy(), central)


def test_c2_full_size_engine_vs_oracle(cuda, oracle):
    # BASELINE config C2 shape (16x21x60x104, f32, seed 2025, K=4, r=0.5) through one
    # full T->H->W rotation with the box denoiser: bit-exact at full size.
    dims = (16, 21, 60, 104)
    z, cond = oracle.synthetic(dims, 4, 2025)
    want, lw = oracle.run_lp(0, (1, 1, 1), z, 4, 3, 0.05, 5.0, cond, (1, 2, 2), 4, 0.5)
    got, lg = lp.run_lp("box", (1, 1, 1), lp.LatentTensor.from_numpy(z, 4), 3, 0.05, 5.0, list(cond), (1, 2, 2), 4, 0.5)
    assert lg["grand_total"] == lw
    assert np.array_equal(got.to_numpy(), want)


def test_nonfinite_is_reported(cuda):
    """Non-finite values raise the device NonFinite flag (the reference's NonFinite,
    src/latent.cpp:72-77 / dtype.cpp quantize) in K10 and the sampler; f16 saturation does not."""
    import torch

    z = lp.LatentTensor.from_numpy(np.full((1, 2, 2, 2), 60000.0), 2)
    lp.device_flags(reset=True)
    lp.cfg_predict(lp.IdentityDenoiser(), z, 1, [1.0] * 8, 3.0)  # f16 saturates, stays finite
    assert lp.device_flags() == 0
    dims = (2, 4, 6, 6)
    for d, dt in ((4, torch.float32), (8, torch.float64)):
        plan = lp.build_plan(dims, (1, 1, 1), 1, 2, 0.5)
        preds = [lp.LatentTensor(torch.ones(plan.sub_shape(dims, k), dtype=dt, device="cuda"), d) for k in range(2)]
        assert np.isfinite(lp.reconstruct(preds, plan, dims).to_numpy()).all() and lp.device_flags() == 0
        preds[1].data[0, 1, 2, 3] = float("nan")
        lp.reconstruct(preds, plan, dims)
        assert lp.device_flags() & 1, d
        zt = lp.LatentTensor(torch.zeros(dims, dtype=dt, device="cuda"), d)
        eps = lp.LatentTensor(torch.zeros(dims, dtype=dt, device="cuda"), d)
        eps.data[1, 0, 0, 0] = float("inf")
        out = lp.sampler_step(zt, eps, 1, 0.05)
        if d == 4:  # the reference's F32 quantize saturates -inf to -FLT_MAX (src/dtype.cpp:106-111)
            assert lp.device_flags() == 0 and out.to_numpy()[1, 0, 0, 0] == -np.finfo(np.float32).max
        else:
            assert lp.device_flags() & 1, d
        eps.data[1, 0, 0, 0] = float("nan")  # NaN survives every quantize
        lp.sampler_step(zt, eps, 1, 0.05)
        assert lp.device_flags() & 1, d
        assert lp.device_flags() == 0  # reset by the read


@pytest.mark.gpu
@pytest.mark.parametrize("d", [2, 4])
def test_engine_nccl_exchange_path_single_rank(cuda, oracle, d):
    """The NCCL all-gather step of the engine (K9) on a 1-rank communicator: the same
    ncclAllGather call and buffer layout as world > 1, bit-exact vs the oracle loop."""
    dims = (16, 5, 16, 16)
    z, cond = oracle.synthetic(dims, d, 2025)
    want, ledger = oracle.run_lp(0, (1, 1, 1), z, d, 4, 0.05, 5.0, cond, (1, 2, 2), 2, 0.5)
    eng = lp.LpEngine(dims, (1, 2, 2), d, 2, 0.5, 4, 0.05, 5.0, list(cond), denoiser="box", radius=(1, 1, 1),
                      world=1, rank=0, nccl_id=lp.nccl_unique_id())
    eng.load(lp.LatentTensor.from_numpy(z, d))
    eng.run(1, 4)
    got = lp.LatentTensor(eng.z.data.clone(), d).to_numpy()
    comm = eng.comm()
    eng.close()
    assert np.array_equal(got, want)
    assert comm["ledger_bytes"] == ledger and comm["nccl_bytes_received"] == 0


@pytest.mark.parametrize("d", [2, 4, 8])
@pytest.mark.parametrize("shape,patch,k,r,step", [
    ((4, 9, 16, 24), (1, 2, 2), 4, 0.5, 1),   # T axis, inner = 384: 8-element vector path
    ((3, 6, 16, 24), (1, 2, 2), 4, 0.5, 2),   # H axis, inner = 24: vector path
    ((2, 5, 6, 52), (1, 2, 2), 4, 0.5, 3),    # W axis, inner = 1: x-stationary path
    ((2, 7, 6, 10), (1, 1, 1), 3, 0.25, 2),   # H axis, inner = 10: per-element path
    ((2, 16, 4, 8), (1, 1, 1), 8, 6.0, 1),    # every position covered by > 4 entries: table fallback
])
def test_reconstruct_paths_bitexact(cuda, oracle, shape, patch, k, r, step, d):
    """K10's code paths (lp_kernels.cu k_reconstruct_cov / k_reconstruct_xs and the fallback),
    exact mode, against the oracle bit for bit, with and without the fused sampler update."""
    z, _ = oracle.synthetic(shape, d, 11)
    plan = lp.build_plan(shape, patch, step, k, r)
    oplan = oracle.build_plan(shape, patch, step, k, r)
    rng = np.random.default_rng(7)
    preds_np = [lp._quantize_np(rng.normal(size=sub_shape(shape, oplan, e)) * 3, d).astype(np.float64)
                for e in range(oplan.n)]
    packed = np.concatenate([p.reshape(-1) for p in preds_np])
    want = oracle.reconstruct(packed, shape, d, oplan)
    preds = [lp.LatentTensor.from_numpy(p, d) for p in preds_np]
    assert np.array_equal(lp.reconstruct(preds, plan, shape).to_numpy(), want)
    zt = lp.LatentTensor.from_numpy(z, d)
    lp.reconstruct_update(preds, plan, zt, 0.05)
    assert np.array_equal(zt.to_numpy(), oracle.sampler_step(z, want, d, 0.05))


@pytest.mark.parametrize("d", [2, 4, 8])
@pytest.mark.parametrize("shape,k,r", [
    ((2, 5, 6, 52), 4, 0.5),       # 60 rows: one full 32-row tile + a ragged one
    ((3, 7, 5, 37), 3, 0.25),      # odd W: runs and the ragged tile not 16-byte aligned (cooperative copies)
    ((1, 3, 3, 40), 8, 1.0),       # 9 rows (< one tile), 8 workers, up to 3 covers per position
    ((16, 21, 60, 104), 4, 0.5),   # C2's W axis
])
@pytest.mark.parametrize("xsb,u", [(1, 4), (1, 8), (0, 4)])
def test_reconstruct_w_axis_bitexact(cuda, oracle, shape, k, r, d, xsb, u):
    """K10 on W-axis plans (inner == 1): the branch-free x-stationary kernel k_reconstruct_xsb
    (knob recon_xsb=1: every lane evaluates the plan's maximum cover count, absent covers
    dropped by selects; 4 or 8 rows in flight, knob recon_u) and the branching one
    (recon_xsb=0), exact mode, reconstruct and fused update, bit for bit vs the oracle."""
    from paper_2512_07350_b200 import _lib

    patch = (1, 1, 1) if shape[3] % 2 else (1, 2, 2)
    z, _ = oracle.synthetic(shape, d, 5)
    plan = lp.build_plan(shape, patch, 3, k, r)
    oplan = oracle.build_plan(shape, patch, 3, k, r)
    assert plan.raw.axis == 2
    rng = np.random.default_rng(3)
    preds_np = [lp._quantize_np(rng.normal(size=sub_shape(shape, oplan, e)) * 3, d).astype(np.float64)
                for e in range(oplan.n)]
    want = oracle.reconstruct(np.concatenate([p.reshape(-1) for p in preds_np]), shape, d, oplan)
    preds = [lp.LatentTensor.from_numpy(p, d) for p in preds_np]
    _lib.check(_lib.lib().lp_tune(b"recon_xsb", xsb))
    _lib.check(_lib.lib().lp_tune(b"recon_u", u))
    try:
        assert np.array_equal(lp.reconstruct(preds, plan, shape).to_numpy(), want)
        zt = lp.LatentTensor.from_numpy(z, d)
        lp.reconstruct_update(preds, plan, zt, 0.05)
        assert np.array_equal(zt.to_numpy(), oracle.sampler_step(z, want, d, 0.05))
    finally:
        _lib.check(_lib.lib().lp_tune(b"recon_xsb", 1))
        _lib.check(_lib.lib().lp_tune(b"recon_u", 4))
