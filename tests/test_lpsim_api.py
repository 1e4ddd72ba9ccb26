"""The reference's own Python smoke test (proj/tests/python/test_smoke.py) run against
this engine's Python face: the same calls, arguments and expectations, with the import
switched from `lpsim` to `paper_2512_07350_b200.lp`.  Host-only calls
run on CPU; calls that touch tensors run on the GPU engine."""
import numpy as np
import pytest

import paper_2512_07350_b200 as pkg
from paper_2512_07350_b200 import lp as lpsim


def test_version():
    assert pkg.__version__ == "0.1.0"


def test_rotation_axis_cycles():
    assert lpsim.rotation_axis(1).name == "temporal"
    assert lpsim.rotation_axis(2).name == "height"
    assert lpsim.rotation_axis(3).name == "width"
    assert lpsim.rotation_axis(300).name == "width"


def test_build_plan_matches_hand_bounds():
    plan = lpsim.build_plan(dims=(1, 8, 8, 8), patch=(2, 2, 2), step=1, workers=2, overlap_ratio=0.5)
    d = plan.to_dict()
    assert d["axis"] == "temporal"
    assert d["L"] == 2 and d["O"] == 1
    assert tuple(d["entries"][0]["latent"]) == (0, 6)
    assert tuple(d["entries"][0]["delta"]) == (0, 2)
    assert tuple(d["entries"][1]["latent"]) == (2, 8)
    assert tuple(d["entries"][1]["delta"]) == (2, 0)


def test_weight_profile():
    plan = lpsim.build_plan(dims=(1, 8, 8, 8), patch=(2, 2, 2), step=1, workers=2, overlap_ratio=0.5)
    assert lpsim.weight_profile(plan, 0) == [1.0, 1.0, 1.0, 1.0, 1.0, 0.5]
    assert lpsim.weight_profile(plan, 1) == [0.0, 0.5, 1.0, 1.0, 1.0, 1.0]


def test_cost_report_formulas():
    report = lpsim.cost_report(steps=60, workers=4, overlap_ratio=0.5, dims=(16, 13, 60, 104), patch=(1, 2, 2),
                               preset="wan21-like")
    assert report["C_NMP"] == 2 * 60 * 3 * report["S_H"]
    assert report["C_PP"] == report["C_NMP"]
    assert report["ratio_exact"] <= 0.05


def test_cost_report_hybrid_bound():
    report = lpsim.cost_report(steps=60, workers=4, overlap_ratio=0.5, dims=(16, 13, 60, 104), patch=(1, 2, 2),
                               preset="wan21-like", hybrid=(2, [2, 2]))
    hybrid = report["hybrid"]
    assert hybrid["bound"] == pytest.approx(2 / 3)
    assert hybrid["ratio_vs_NMP"] < hybrid["bound"]
    assert hybrid["within_bound"]


def test_two_step_completeness():
    verdict = lpsim.verify_n_complete(grid=(4, 4, 4), workers=2, overlap_ratio=0.0, schedule="rotating", budget=2)
    assert verdict["complete"]
    assert verdict["complete_at"] == 2
    stuck = lpsim.verify_n_complete(grid=(4, 4, 4), workers=2, overlap_ratio=0.0, schedule="temporal", budget=50)
    assert not stuck["complete"]
    assert stuck["complete_at"] is None


def test_invalid_overlap_ratio_raises():
    with pytest.raises(Exception):
        lpsim.build_plan(dims=(1, 8, 8, 8), patch=(2, 2, 2), step=1, workers=2, overlap_ratio=3.0)


def test_presets_listed():
    names = [p["name"] for p in lpsim.presets()]
    assert "wan21-like" in names


# ---- tensor-touching calls: the GPU engine ----
@pytest.mark.gpu
def test_tensor_numpy_round_trip(cuda):
    rng = np.random.default_rng(7)
    arr = rng.normal(size=(2, 4, 4, 4))
    z = lpsim.LatentTensor.from_numpy(arr, dtype_bytes=8)
    assert z.shape == (2, 4, 4, 4)
    assert z.dtype_bytes == 8
    np.testing.assert_array_equal(z.to_numpy(), arr)
    z32 = lpsim.LatentTensor.from_numpy(arr, dtype_bytes=4)
    np.testing.assert_array_equal(z32.to_numpy(), arr.astype(np.float32).astype(np.float64))


@pytest.mark.gpu
def test_reconstruct_blends_overlaps(cuda):
    plan = lpsim.build_plan(dims=(1, 8, 2, 2), patch=(2, 2, 2), step=1, workers=2, overlap_ratio=0.5)
    ones = lpsim.LatentTensor.from_numpy(np.full((1, 6, 2, 2), 1.0), dtype_bytes=8)
    threes = lpsim.LatentTensor.from_numpy(np.full((1, 6, 2, 2), 3.0), dtype_bytes=8)
    out = lpsim.reconstruct([ones, threes], plan, (1, 8, 2, 2)).to_numpy()
    expected = np.array([1, 1, 1, 5 / 3, 2, 7 / 3, 3, 3])
    np.testing.assert_allclose(out[0, :, 0, 0], expected, atol=1e-12)


@pytest.mark.gpu
def test_single_worker_run_matches_centralized(cuda):
    z, cond = lpsim.synthetic_latent(dims=(1, 8, 8, 8), dtype_bytes=4, seed=11)
    central = lpsim.run_centralized("box", (1, 1, 1), z, steps=3, eta=0.1, guidance=2.0, cond=cond)
    final, ledger = lpsim.run_lp("box", (1, 1, 1), z, steps=3, eta=0.1, guidance=2.0, cond=cond, patch=(2, 2, 2),
                                 workers=1, overlap_ratio=0.0)
    assert ledger["grand_total"] == 0
    np.testing.assert_array_equal(final.to_numpy(), central.to_numpy())


@pytest.mark.gpu
def test_run_lp_meters_bytes(cuda):
    z, cond = lpsim.synthetic_latent(dims=(1, 8, 8, 8), dtype_bytes=4, seed=3)
    _, ledger = lpsim.run_lp("identity", (0, 0, 0), z, steps=1, eta=0.1, guidance=1.0, cond=cond, patch=(2, 2, 2),
                             workers=2, overlap_ratio=0.0)
    assert ledger["grand_total"] == 4 * (8 * 8 * 4) * 2


@pytest.mark.gpu
def test_latent_dump_round_trip(cuda, tmp_path):
    z, _ = lpsim.synthetic_latent(dims=(2, 3, 4, 5), dtype_bytes=2, seed=9)
    path = str(tmp_path / "z.bin")
    lpsim.save_latent(path, z)
    back = lpsim.load_latent(path)
    assert back.shape == z.shape
    assert back.dtype_bytes == 2
    np.testing.assert_array_equal(back.to_numpy(), z.to_numpy())
