"""bench.py's multi-rank path (torchrun, N=2) on one B200: LP_BENCH_GLOO_TEST=1 puts both
ranks on GPU 0 with gloo plumbing and the ε̂ exchange over CUDA IPC peer memory (NCCL refuses
two ranks on one device).  Checks the driver-facing contract of the N>1 line: one JSON line
from rank 0, n_gpus = 2, exchange "peer", measured exchange bytes > 0, finite numbers."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_two_ranks_peer_exchange(cuda):
    env = dict(os.environ, LP_BENCH_GLOO_TEST="1")
    port = 29400 + os.getpid() % 500
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--layers", "2"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["exchange"] == "peer"
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["comm"]["exchange_bytes_per_step_measured_all_ranks"] > 0
    assert d["allgather"]["in_step_launches"] > 0
    assert len(d["ranks"]) == 2 and all(r["exchange_bench"]["GBps"] > 0 for r in d["ranks"])


@pytest.mark.gpu
def test_bench_gpus_2_launches_its_own_ranks(cuda):
    """`python bench.py --gpus 2` WITHOUT torchrun starts both ranks itself (the driver's
    command line); under LP_BENCH_GLOO_TEST both sit on GPU 0."""
    env = dict(os.environ, LP_BENCH_GLOO_TEST="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3", "--layers", "2"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["exchange"] == "peer" and [x["rank"] for x in d["ranks"]] == [0, 1]
    assert d["scaling_model"]["flop_ideal_speedup_vs_1gpu"] > 1.5
