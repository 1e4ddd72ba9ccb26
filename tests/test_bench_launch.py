"""bench.py's launcher on CPU: `--gpus N` without a torchrun environment starts N ranks itself
(gloo plumbing for --plan-only), every rank reports, and rank 0 prints ONE line with n_gpus = N,
the per-rank shard assignment and the FLOP-ideal speedup bound."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [2, 4])
def test_gpus_n_self_launches_n_ranks(n):
    d = _run("--gpus", str(n), "--plan-only")
    assert d["n_gpus"] == n and [r["rank"] for r in d["ranks"]] == list(range(n))
    owned = sorted(k for r in d["ranks"] for k in r["owned_entries"]["T"])
    assert owned == [1, 2, 3, 4]  # C2 keeps its 4-way LP for N <= 4
    sm = d["scaling_model"]
    assert 1.0 < sm["flop_ideal_speedup_vs_1gpu"] <= n + 1e-9
    assert 0.0 < sm["rank_balance"] <= 1.0


def test_gpus_8_flop_ideal_bound_names_the_idle_rank():
    d = _run("--gpus", "8", "--plan-only")
    sm = d["scaling_model"]
    assert sm["k_eff_per_axis"] == [7, 8, 8]          # T axis: 21 frames, L = 3 -> 7 cores (partition.cpp:54-58)
    assert sm["owner_per_axis"][0] == list(range(7))   # rank 7 idles on T steps
    assert sm["flop_ideal_speedup_vs_1gpu"] > 8        # K = 8 shards carry less overlap work than K = 4


def test_single_gpu_plan_and_world_mismatch_fails_loudly():
    d = _run("--plan-only")
    assert d["n_gpus"] == 1 and d["scaling_model"]["flop_ideal_speedup_vs_1gpu"] == pytest.approx(1.0)
    env = dict(os.environ, WORLD_SIZE="1", RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--plan-only"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr
