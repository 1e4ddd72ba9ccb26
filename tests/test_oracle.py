"""Pins the CPU oracle (oracle/lp_oracle.c) before anything is checked against it.

1. The reference's own known-answer tests, restated here.
2. The golden checksums of reference runs (SURVEY.md §8c "Golden checksums").
3. Randomized sweeps against the compiled, unmodified reference (oracle/_ref).
"""
import hashlib

import numpy as np
import pytest

from oracle.oracle import LpError

H = lambda a: hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()[:16]  # noqa: E731


def test_rotation_axis_kat(oracle):
    # test_partition.cpp:26-39 / test_smoke.py:11-15
    import ctypes as C

    for step, axis in [(1, 0), (2, 1), (3, 2), (4, 0), (300, 2)]:
        a = C.c_int()
        assert oracle.lib.orc_rotation_axis(step, C.byref(a)) == 0 and a.value == axis
    assert oracle.lib.orc_rotation_axis(0, C.byref(C.c_int())) == 10  # InvalidArgument


def test_plan_kat_k2_r05(oracle):
    # test_smoke.py:31-39 / test_partition.cpp:92-137
    p = oracle.build_plan((1, 8, 8, 8), (2, 2, 2), 1, 2, 0.5)
    assert p.axis == 0 and p.meta[2] == 2 and p.meta[3] == 1
    assert p.latent(0) == (0, 6) and tuple(p.entries[0, 7:9]) == (0, 2)
    assert p.latent(1) == (2, 8) and tuple(p.entries[1, 7:9]) == (2, 0)


def test_plan_kat_idle_workers_and_remainder(oracle):
    # core_bounds 5 patches / 4 workers -> K_eff 3 (test_partition.cpp:41-62)
    p = oracle.build_axis_plan(0, 5, 1, 1, 4, 0.0)
    assert p.n == 3 and [p.latent(k) for k in range(3)] == [(0, 2), (2, 4), (4, 5)]
    # remainder rows go to the last entry: D=7, p=2 (test_partition.cpp:175-181)
    p = oracle.build_axis_plan(0, 7, 2, 1, 2, 0.0)
    assert p.latent(1) == (4, 7)
    with pytest.raises(LpError) as e:
        oracle.build_plan((1, 8, 8, 8), (2, 2, 2), 1, 2, 3.0)
    assert e.value.status == 4  # InvalidOverlapRatio
    with pytest.raises(LpError) as e:
        oracle.build_axis_plan(0, 1, 2, 1, 2, 0.0)
    assert e.value.status == 3  # DegenerateAxis


def test_weight_profile_kat(oracle):
    # test_smoke.py:42-45
    p = oracle.build_plan((1, 8, 8, 8), (2, 2, 2), 1, 2, 0.5)
    assert list(oracle.weight_profile(p, 0)) == [1.0, 1.0, 1.0, 1.0, 1.0, 0.5]
    assert list(oracle.weight_profile(p, 1)) == [0.0, 0.5, 1.0, 1.0, 1.0, 1.0]


def test_reconstruct_kat(oracle):
    # test_smoke.py:48-54 / test_reconstruct.cpp:101-129: rows [1,1,1,5/3,2,7/3,3,3]
    p = oracle.build_plan((1, 8, 2, 2), (2, 2, 2), 1, 2, 0.5)
    preds = np.concatenate([np.full(6 * 4, 1.0), np.full(6 * 4, 3.0)])
    out = oracle.reconstruct(preds, (1, 8, 2, 2), 8, p)
    np.testing.assert_allclose(out[0, :, 0, 0], [1, 1, 1, 5 / 3, 2, 7 / 3, 3, 3], atol=1e-12)


def test_cfg_and_sampler_kat(oracle):
    # sampler: eta=0.1, 1 -> 0.9 (test_denoise.cpp:156-180)
    z = np.ones((1, 2, 2, 2))
    assert np.all(oracle.sampler_step(z, z, 8, 0.1) == 1.0 - 0.1 * 1.0)
    # identity under CFG is exact for any w (u == c)
    for w in (0.0, 1.0, 5.0):
        out = oracle.cfg_predict(2, (0, 0, 0), z * 3, 8, 7, [1.0] * 8, w)
        assert np.all(out == 3.0)


def test_f16_kats(oracle, reference):
    # no double rounding: 9.269531296341157 -> 0x48a3 (test_latent.cpp:126-162)
    assert oracle.f16_encode(9.269531296341157) == 0x48A3
    assert oracle.f16_encode(1e9) == 0x7BFF and oracle.f16_encode(-1e9) == 0xFBFF
    # every binary16 pattern round-trips (finite ones) and decodes like the reference
    for b in range(0, 65536, 7):
        d = oracle.f16_decode(b)
        assert (np.isnan(d) and np.isnan(reference.f16_decode(b))) or d == reference.f16_decode(b)
        if np.isfinite(d):
            assert oracle.f16_encode(d) == b or (d == 0.0)
    rng = np.random.default_rng(5)
    vals = np.concatenate([rng.normal(size=3000) * 10.0 ** rng.integers(-9, 6, size=3000),
                           [65504.0, 65519.99, 65520.0, 2.0 ** -25, 2.0 ** -24 * 1.5, 5.960464477539063e-08]])
    for v in vals:
        assert oracle.f16_encode(v) == reference.f16_encode(v)
        for d in (2, 4, 8):
            assert oracle.quantize(v, d) == reference.quantize(v, d)


def test_golden_checksums(oracle):
    # SURVEY.md §8c, measured on the unmodified reference.
    z, c = oracle.synthetic((4, 12, 16, 16), 4, 2025)
    assert H(z) == "3889ec0d272812c2"
    out, ledger = oracle.run_lp(0, (2, 2, 2), z, 4, 6, 0.05, 2.0, c, (2, 2, 2), 2, 1.0)
    assert H(out) == "3ad2d84ae75b30e9" and ledger == 589824
    z, c = oracle.synthetic((4, 12, 16, 16), 8, 2025)
    out, _ = oracle.run_lp(0, (2, 2, 2), z, 8, 6, 0.05, 2.0, c, (2, 2, 2), 2, 1.0)
    assert H(out) == "e7cbc9b6807bca2e"
    z, c = oracle.synthetic((16, 5, 16, 16), 4, 2025)
    assert H(z) == "b51ffac38256406c"
    out, ledger = oracle.run_lp(0, (1, 1, 1), z, 4, 4, 0.05, 5.0, c, (1, 2, 2), 2, 0.5)
    assert H(out) == "93a6824b0e691fdc" and ledger == 442368
    z, c = oracle.synthetic((4, 12, 16, 16), 4, 42)
    out, ledger = oracle.run_lp(0, (1, 1, 1), z, 4, 60, 0.05, 3.0, c, (2, 2, 2), 4, 0.5)
    assert H(out) == "18f78847365f6597" and ledger == 7700480


def test_c2_latent_first_values(oracle):
    z, _ = oracle.synthetic((16, 21, 60, 104), 4, 2025)
    assert H(z) == "d3122ea6ca551a6a"
    assert z.reshape(-1)[0] == -1.6695451736450195 and z.reshape(-1)[1] == 0.2779560685157776


def _random_case(rng):
    shape = tuple(int(v) for v in (rng.integers(1, 4), rng.integers(1, 13), rng.integers(1, 13), rng.integers(1, 13)))
    patch = tuple(int(v) for v in rng.integers(1, 4, size=3))
    k = int(rng.integers(1, 9))
    r = float(rng.choice([0.0, 0.25, 0.5, 1.0, 1.5, 0.3333]))
    return shape, patch, k, min(r, k - 1)


def test_plans_match_reference_sweep(oracle, reference):
    # test_partition.cpp:183-238 style sweep (500 random plans)
    rng = np.random.default_rng(1)
    n = 0
    while n < 500:
        shape, patch, k, r = _random_case(rng)
        step = int(rng.integers(1, 7))
        try:
            a = reference.build_plan(shape, patch, step, k, r)
        except LpError as e:
            with pytest.raises(LpError) as e2:
                oracle.build_plan(shape, patch, step, k, r)
            assert e2.value.status == e.status
            continue
        b = oracle.build_plan(shape, patch, step, k, r)
        assert np.array_equal(a.meta, b.meta) and np.array_equal(a.entries, b.entries)
        for e in range(a.n):
            assert np.array_equal(oracle.weight_profile(b, e), reference.weight_profile(shape, patch, step, k, r, e))
        n += 1


def test_stages_match_reference_sweep(oracle, reference):
    # extract / toy cfg_predict / reconstruct / sampler: bitwise over random cases
    rng = np.random.default_rng(2)
    done = 0
    while done < 120:
        shape, patch, k, r = _random_case(rng)
        step = int(rng.integers(1, 4))
        d = int(rng.choice([2, 4, 8]))
        try:
            plan = reference.build_plan(shape, patch, step, k, r)
        except LpError:
            continue
        z, cond = reference.synthetic(shape, d, int(rng.integers(0, 1 << 30)))
        subs = oracle.extract(z, plan)
        assert np.array_equal(subs, reference.extract(z, d, patch, step, k, r))
        kind = int(rng.integers(0, 3))
        radius = tuple(int(v) for v in rng.integers(0, 3, size=3))
        w = float(rng.choice([1.0, 2.0, 5.0]))
        t = int(rng.integers(1, 60))
        preds = []
        off = 0
        for e in range(plan.n):
            from oracle.oracle import sub_shape

            ss = sub_shape(shape, plan, e)
            n = int(np.prod(ss))
            sub = subs[off: off + n].reshape(ss)
            a = oracle.cfg_predict(kind, radius, sub, d, t, cond, w)
            b = reference.cfg_predict(kind, radius, sub, d, t, cond, w)
            assert np.array_equal(a, b), (kind, ss, d)
            preds.append(a.reshape(-1))
            off += n
        packed = np.concatenate(preds)
        eps = oracle.reconstruct(packed, shape, d, plan)
        assert np.array_equal(eps, reference.reconstruct(packed, shape, d, patch, step, k, r))
        assert np.array_equal(oracle.sampler_step(z, eps, d, 0.05), reference.sampler_step(z, eps, d, 0.05))
        done += 1


def test_run_lp_matches_reference(oracle, reference):
    rng = np.random.default_rng(3)
    for _ in range(12):
        shape, patch, k, r = _random_case(rng)
        d = int(rng.choice([2, 4, 8]))
        try:
            reference.build_plan(shape, patch, 1, k, r)
            reference.build_plan(shape, patch, 2, k, r)
            reference.build_plan(shape, patch, 3, k, r)
        except LpError:
            continue
        z, c = reference.synthetic(shape, d, 7)
        kind = int(rng.integers(0, 3))
        a, la = reference.run_lp(kind, (1, 0, 1), z, d, 5, 0.05, 3.0, c, patch, k, r)
        b, lb = oracle.run_lp(kind, (1, 0, 1), z, d, 5, 0.05, 3.0, c, patch, k, r)
        assert np.array_equal(a, b) and la == lb
