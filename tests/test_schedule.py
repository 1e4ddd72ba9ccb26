"""Custom axis schedules (BASELINE config C5 "temporal-heavy rotation").

The reference hard-codes T->H->W (src/partition.cpp:38-43) but builds plans for any
axis (build_axis_plan) and checks arbitrary schedules for N-completeness
(verify_n_complete, src/completeness.cpp:104-160).  The engine takes an explicit
schedule; here the reference checker certifies the temporal-heavy one.
"""
import numpy as np
import pytest

from oracle.oracle import sub_shape, verify_n_complete
from paper_2512_07350_b200 import lp

TEMPORAL_HEAVY = "TTHTTW"   # 4 of every 6 steps cut time: long (161-frame) videos have the most tokens on T


def test_parse_schedule():
    assert lp.parse_schedule("TTHTTW") == [0, 0, 1, 0, 0, 2]
    assert lp.parse_schedule(["temporal", "width"]) == [0, 2]
    assert lp.parse_schedule([2, 1]) == [2, 1]
    with pytest.raises(lp.LpError):
        lp.parse_schedule("")


@pytest.mark.parametrize("grid,K", [((11, 8, 13), 8), ((9, 6, 8), 4), ((21, 6, 5), 8)])
def test_temporal_heavy_schedule_is_n_complete(reference, grid, K):
    sched = lp.parse_schedule(TEMPORAL_HEAVY)
    got = verify_n_complete(reference, grid, K, 0.5, sched, 24)
    assert got["complete"], got
    rot = verify_n_complete(reference, grid, K, 0.5, [0, 1, 2], 24)
    assert rot["complete"]
    # without overlap a constant temporal cut never connects its blocks (test_smoke.py:104-107 analogue)
    const = verify_n_complete(reference, grid, K, 0.0, [0], 24)
    assert not const["complete"]


def oracle_loop(orc, z, cond, dims, patch, K, r, steps, schedule, d, kind=0, radius=(1, 1, 1), eta=0.05, w=3.0):
    """run_lp restated with an explicit schedule from the oracle's per-stage functions."""
    z = z.copy()
    for i in range(1, steps + 1):
        t = steps + 1 - i
        a = schedule[(i - 1) % len(schedule)]
        plan = orc.build_axis_plan(a, dims[1 + a], patch[a], i, K, r)
        subs = orc.extract(z, plan)
        preds, off = [], 0
        for e in range(plan.n):
            ss = sub_shape(dims, plan, e)
            n = int(np.prod(ss))
            preds.append(orc.cfg_predict(kind, radius, subs[off:off + n].reshape(ss), d, t, cond, w).reshape(-1))
            off += n
        eps = orc.reconstruct(np.concatenate(preds), dims, d, plan)
        z = orc.sampler_step(z, eps, d, eta)
    return z


@pytest.mark.gpu
def test_engine_custom_schedule_bitexact(cuda, oracle):
    dims, patch, K, r, steps = (4, 10, 8, 12), (1, 2, 2), 4, 0.5, 7
    for d in (4, 8):
        z, cond = oracle.synthetic(dims, d, 31)
        sched = lp.parse_schedule(TEMPORAL_HEAVY)
        want = oracle_loop(oracle, z, cond, dims, patch, K, r, steps, sched, d)
        got, _ = lp.run_lp("box", (1, 1, 1), lp.LatentTensor.from_numpy(z, d), steps, 0.05, 3.0, list(cond), patch, K, r,
                           schedule=TEMPORAL_HEAVY)
        assert np.array_equal(got.to_numpy(), want)


def test_verify_n_complete_matches_reference_sweep(reference):
    """Our C++ checker (completeness.cpp) vs the reference's verify_n_complete on random
    grids, worker counts, overlap ratios and schedules (rotating, constant, custom)."""
    rng = np.random.default_rng(5)
    scheds = ["rotating", "temporal", "height", "width", "TTHTTW", "HW", "TWH"]
    for _ in range(60):
        grid = tuple(int(x) for x in rng.integers(1, 12, 3))
        K = int(rng.integers(1, 6))
        r = float(rng.choice([0.0, 0.25, 0.5, 1.0])) if K > 1 else 0.0
        r = min(r, K - 1)
        name = str(rng.choice(scheds))
        budget = int(rng.integers(1, 10))
        got = lp.verify_n_complete(grid, K, r, name, budget)
        if name == "rotating":
            axes = [lp.rotation_axis(i) for i in range(1, budget + 1)]
        elif name in ("temporal", "height", "width"):
            axes = [int(lp.Axis[name])] * budget
        else:
            cyc = lp.parse_schedule(name)
            axes = [cyc[i % len(cyc)] for i in range(budget)]
        want = verify_n_complete(reference, grid, K, r, axes, budget)
        assert (got["complete"], got["complete_at"], tuple(got["worst_position"])) == \
            (want["complete"], want["complete_at"], want["worst_position"]), (grid, K, r, name, budget)


def test_verify_n_complete_cap_and_lifted_cap():
    # the reference caps exhaustive analysis at 4096 positions (src/completeness.cpp:13,35-40)
    with pytest.raises(lp.LpError) as e:
        lp.verify_n_complete((17, 16, 16), 4, 0.5, "rotating", 8)
    assert e.value.status == 10 and "capped at 4096" in str(e.value)  # InvalidArgument
    # lifted: a C5-like grid (161 frames -> 41 latent frames, halved H/W patch grid) with the
    # temporal-heavy schedule is N-complete; so is the rotation
    grid = (41, 15, 26)
    th = lp.verify_n_complete(grid, 8, 0.5, TEMPORAL_HEAVY, 12, max_positions=grid[0] * grid[1] * grid[2])
    rot = lp.verify_n_complete(grid, 8, 0.5, "rotating", 12, max_positions=grid[0] * grid[1] * grid[2])
    assert th["complete"] and rot["complete"]
    assert th["complete_at"] <= 12 and min(th["min_steps"]) >= 1
