"""CPU tests of the product's host side: the C-ABI library loads and exports every
symbol include/lp_b200.h declares; the host plan builder / weights / quantizer /
synthetic inputs are bit-exact with the reference (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle.oracle import LpError as OracleError
from paper_2512_07350_b200 import _lib, lp
from paper_2512_07350_b200._lib import LpError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "lp_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    names = set(re.findall(r"\b(lp_[a-z0-9_]+)\s*\(", hdr))
    L = _lib.lib()
    missing = [n for n in sorted(names) if not hasattr(L, n)]
    assert not missing, f"declared but not exported: {missing}"
    assert len(names) >= 40


def test_version():
    assert b"sm_100a" in _lib.lib().lp_version()


def test_rotation_axis():
    assert lp.rotation_axis(1).name == "temporal"
    assert lp.rotation_axis(2).name == "height"
    assert lp.rotation_axis(3).name == "width"
    assert lp.rotation_axis(300).name == "width"
    with pytest.raises(LpError) as e:
        lp.rotation_axis(0)
    assert e.value.kind == "InvalidArgument"


def test_plan_matches_reference_hand_bounds():
    # test_smoke.py:31-39
    d = lp.build_plan(dims=(1, 8, 8, 8), patch=(2, 2, 2), step=1, workers=2, overlap_ratio=0.5).to_dict()
    assert d["axis"] == "temporal" and d["L"] == 2 and d["O"] == 1
    assert d["entries"][0]["latent"] == (0, 6) and d["entries"][0]["delta"] == (0, 2)
    assert d["entries"][1]["latent"] == (2, 8) and d["entries"][1]["delta"] == (2, 0)


def test_weight_profile_kat():
    plan = lp.build_plan(dims=(1, 8, 8, 8), patch=(2, 2, 2), step=1, workers=2, overlap_ratio=0.5)
    assert lp.weight_profile(plan, 0) == [1.0, 1.0, 1.0, 1.0, 1.0, 0.5]
    assert lp.weight_profile(plan, 1) == [0.0, 0.5, 1.0, 1.0, 1.0, 1.0]


def test_c2_plans():
    # SURVEY.md §8 "C2 plans" table
    want = {
        1: [((0, 9), (0, 3)), ((3, 15), (3, 3)), ((9, 21), (3, 3)), ((15, 21), (3, 0))],
        2: [((0, 24), (0, 8)), ((8, 40), (8, 8)), ((24, 56), (8, 8)), ((40, 60), (8, 0))],
        3: [((0, 38), (0, 12)), ((14, 64), (12, 12)), ((40, 90), (12, 12)), ((66, 104), (12, 0))],
    }
    for step, ents in want.items():
        d = lp.build_plan((16, 21, 60, 104), (1, 2, 2), step, 4, 0.5).to_dict()
        assert [(e["latent"], e["delta"]) for e in d["entries"]] == ents
    d = lp.build_plan((16, 21, 60, 104), (1, 2, 2), 1, 8, 0.5).to_dict()
    assert len(d["entries"]) == 7  # K_eff = 7 on T at K=8


def test_invalid_overlap_ratio_raises():
    with pytest.raises(LpError) as e:
        lp.build_plan(dims=(1, 8, 8, 8), patch=(2, 2, 2), step=1, workers=2, overlap_ratio=3.0)
    assert e.value.kind == "InvalidOverlapRatio"


def test_plan_sweep_matches_reference(reference):
    rng = np.random.default_rng(11)
    lp_msgs = []
    _lib.lib().lp_set_warning_handler(None, None)
    for _ in range(800):
        shape = tuple(int(v) for v in rng.integers(1, 40, size=4))
        patch = tuple(int(v) for v in rng.integers(1, 5, size=3))
        k = int(rng.integers(1, 17))
        r = float(min(rng.choice([0.0, 0.1, 0.25, 0.5, 0.75, 1.0, 2.0, 2.5]), k - 1))
        step = int(rng.integers(1, 10))
        try:
            ref = reference.build_plan(shape, patch, step, k, r)
        except OracleError as e:
            with pytest.raises(LpError) as e2:
                lp.build_plan(shape, patch, step, k, r)
            assert e2.value.status == e.status
            continue
        ours = lp.build_plan(shape, patch, step, k, r).to_dict()
        assert [ref.meta[0], ref.meta[2], ref.meta[3], ref.meta[4], ref.meta[5], ref.meta[6]] == \
               [lp.Axis[ours["axis"]].value, ours["L"], ours["O"], ours["N"], ours["D"], ours["p"]]
        got = np.array([[e["k"], *e["core"], *e["ext"], *e["latent"], *e["delta"]] for e in ours["entries"]])
        assert np.array_equal(got, ref.entries)
        plan = lp.build_plan(shape, patch, step, k, r)
        for e in range(plan.workers):
            assert lp.weight_profile(plan, e) == list(reference.weight_profile(shape, patch, step, k, r, e))
    assert not lp_msgs


def test_quantizer_matches_reference(reference):
    rng = np.random.default_rng(4)
    vals = np.concatenate([rng.normal(size=5000) * 10.0 ** rng.integers(-10, 7, size=5000),
                           [0.0, -0.0, 65504.0, 65519.999, 65520.0, 1e40, -1e40, 3.4028235677973366e38,
                            9.269531296341157, 2.0 ** -25, 2.0 ** -24]])
    for v in vals:
        assert lp.f16_encode(v) == reference.f16_encode(v)
        for d in (2, 4, 8):
            assert lp.quantize(v, d) == reference.quantize(v, d)
    # the host-side numpy quantizer used by LatentTensor.from_numpy agrees too
    for d in (2, 4, 8):
        q = lp._quantize_np(vals, d).astype(np.float64)
        assert np.array_equal(q, np.array([reference.quantize(v, d) for v in vals]))


def test_synthetic_inputs_match_reference(reference):
    for shape, d, seed in [((2, 3, 4, 5), 2, 9), ((16, 5, 16, 16), 4, 2025), ((4, 12, 16, 16), 8, 42)]:
        z, c = lp.synthetic_latent_host(shape, d, seed)
        rz, rc = reference.synthetic(shape, d, seed)
        assert np.array_equal(z, rz) and np.array_equal(np.array(c), rc)


def test_shard_layout_and_comm_accounting(reference):
    dims = (16, 21, 60, 104)
    for step in (1, 2, 3):
        plan = lp.build_plan(dims, (1, 2, 2), step, 4, 0.5)
        offs = plan.offsets(dims)
        for world in (1, 2, 4):
            owned_all = []
            for rank in range(world):
                owned, slot = lp.shard_layout(plan, dims, world, rank)
                owned_all += owned
                assert all(e % world == rank for e in owned)
                assert slot >= sum(offs[e + 1] - offs[e] for e in owned)
            assert sorted(owned_all) == list(range(plan.workers))
        ledger, ag = lp.step_comm_bytes(plan, dims, 2, 4, 4)
        n = [offs[k + 1] - offs[k] for k in range(plan.workers)]
        assert ledger == 4 * sum(n[1:]) * 2  # cluster.cpp:186-209
        assert ag == 4 * 3 * max(n) * 4
    # the per-video ledger equals the reference cost model at C2 (1,162.7 MB)
    total = sum(lp.step_comm_bytes(lp.build_plan(dims, (1, 2, 2), i, 4, 0.5), dims, 2, 4, 4)[0] for i in range(1, 51))
    assert total == reference.cost(50, 4, 0.5, dims, (1, 2, 2))["C_LP_exact"]
    assert abs(total / 1e6 - 1162.7) < 0.1


def test_device_entry_points_fail_loudly_without_gpu():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("has a GPU")
    except Exception:
        pass
    st = _lib.lib().lp_device_check(0)
    assert st == 100  # LP_ERR_CUDA: no CPU fallback


def _same(a, b):
    return (a == b) or (np.isnan(a) and np.isnan(b))


def test_cost_report_matches_reference(reference):
    """cost_report bit-exact vs the reference (src/cost.cpp:215-248), incl. hybrid, over the
    BASELINE.json configs and a random sweep; and the BASELINE.md table values."""
    cases = [
        (60, 4, 0.5, (16, 13, 60, 104), (1, 2, 2), None),     # paper 49f
        (50, 4, 0.5, (16, 21, 60, 104), (1, 2, 2), None),     # C2
        (50, 8, 0.5, (16, 21, 90, 160), (1, 2, 2), None),     # C4 (hidden 5120 below)
        (50, 8, 0.5, (16, 41, 60, 104), (1, 2, 2), None),     # C5
        (60, 4, 0.5, (16, 13, 60, 104), (1, 2, 2), (2, [2, 2])),
        (50, 8, 1.0, (16, 21, 60, 104), (1, 2, 2), (3, [3, 3, 2])),
        (4, 1, 0.0, (16, 5, 16, 16), (1, 2, 2), (1, [1])),
    ]
    rng = np.random.default_rng(9)
    for _ in range(40):
        k = int(rng.integers(1, 9))
        g = int(rng.integers(1, k + 1))
        sizes = [1] * g
        for _ in range(k - g):
            sizes[int(rng.integers(0, g))] += 1
        cases.append((int(rng.integers(1, 70)), k, float(min(rng.choice([0, .25, .5, 1.0]), k - 1)),
                      tuple(int(v) for v in rng.integers(2, 40, size=4)), (1, 2, 2),
                      (g, sizes) if rng.random() < 0.5 else None))
    for steps, k, r, dims, patch, hyb in cases:
        hidden = 5120 if dims == (16, 21, 90, 160) else 1536
        try:
            want = reference.cost(steps, k, r, dims, patch, hidden, 2, hyb)
        except OracleError:
            continue
        got = lp.cost_report(steps, k, r, dims, patch, hybrid=hyb, hidden_dim=hidden, wire_bytes=2)
        for key in ("S_z", "S_H", "gamma", "C_NMP", "C_PP", "C_LP_exact", "C_LP_approx", "ratio_exact",
                    "ratio_approx", "Sz_over_SH"):
            assert _same(float(got[key]), float(want[key])), (key, got[key], want[key], dims, k, r)
        assert got["gamma_per_axis"] == want["gamma_per_axis"]
        assert ("hybrid" in got) == ("hybrid" in want)
        if "hybrid" in got:
            for key, v in want["hybrid"].items():
                assert _same(float(got["hybrid"][key]), float(v)), key
    # BASELINE.md §2 numbers
    c2 = lp.cost_report(50, 4, 0.5, (16, 21, 60, 104), (1, 2, 2))
    assert round(c2["C_LP_exact"] / 1e6, 1) == 1162.7 and round(c2["C_NMP"] / 1e6, 1) == 30191.6
    paper = lp.cost_report(60, 4, 0.5, (16, 13, 60, 104), (1, 2, 2))
    assert round(paper["ratio_exact"], 4) == 0.0381


def test_shard_layout_alignment_and_balanced_assignment():
    """Slots start 16-B aligned for every dtype (slot_elems % 8 == 0), round-robin is the
    default, and the balanced policy is longest-processing-time greedy on the cost model."""
    dims = (16, 21, 60, 104)
    for step in (1, 2, 3):
        for K in (4, 8):
            plan = lp.build_plan(dims, (1, 2, 2), step, K, 0.5)
            offs = plan.offsets(dims)
            n = [offs[k + 1] - offs[k] for k in range(plan.workers)]
            for world in (1, 2, 3, 4, 8):
                owned, slot = lp.shard_layout(plan, dims, world, 0)
                assert slot % 8 == 0
                o2, s2, owner, base = lp.shard_layout_ex(plan, dims, world, 0, "round-robin")
                assert (o2, s2) == (owned, slot) and owner == [k % world for k in range(plan.workers)]
                lin, quad = 1.0, 1e-6
                _, sb, ob, bb = lp.shard_layout_ex(plan, dims, world, 0, "balanced", lin, quad)
                cost = [lin * x + quad * x * x for x in n]
                load, want = [0.0] * world, [0] * plan.workers
                if plan.workers <= world:
                    want = list(range(plan.workers))
                else:
                    for k in sorted(range(plan.workers), key=lambda k: -cost[k]):
                        r = min(range(world), key=lambda r: load[r])
                        want[k] = r
                        load[r] += cost[k]
                assert ob == want
                assert sb % 8 == 0
                spans = sorted((bb[k], bb[k] + n[k]) for k in range(plan.workers))
                assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))
                assert all(ob[k] * sb <= bb[k] and bb[k] + n[k] <= (ob[k] + 1) * sb for k in range(plan.workers))
    # a one-channel latent whose per-rank sums are not multiples of 8 still gets aligned slots
    plan = lp.build_plan((1, 5, 6, 6), (1, 2, 2), 1, 4, 0.5)
    for world in (2, 3):
        _, slot = lp.shard_layout(plan, (1, 5, 6, 6), world, 1)
        assert slot % 8 == 0
