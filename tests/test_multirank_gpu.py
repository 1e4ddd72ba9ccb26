"""World-size-2 run of the ENGINE's multi-rank path on one GPU: two processes, each an
lp_engine with world=2 / rank=r and no NCCL id, driven through lp_engine_step_phase; the
padded rank slots are exchanged by gloo between phase 1 (K1 + cfg_predict of the rank's
own entries) and phase 3 (K10 on the gathered buffer).  That is the data path of the
NCCL run (engine.cpp step_exchange) with the transport swapped, so it covers the shard
ownership, slot bases and reconstruct-from-gathered code on the GPU (NCCL itself refuses
two ranks on one device; its call is covered by test_engine_nccl_exchange_path_single_rank).

Toy denoiser: both ranks must equal the oracle's single-process run_lp bit for bit.
DiT: both ranks must equal a world=1 engine run with the same DiT, bit for bit.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2
DIMS = (16, 5, 16, 16)
PATCH = (1, 2, 2)
K, R, STEPS = 4, 0.5, 4


def _engine(lp, denoiser, d, cond, world, rank, dit=None):
    return lp.LpEngine(DIMS, PATCH, d, K, R, STEPS, 0.05, 5.0, list(cond), denoiser=denoiser, radius=(1, 1, 1),
                       world=world, rank=rank, dit=dit)


def _worker(rank, port, q, denoiser, d):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        torch.cuda.set_device(0)
        from paper_2512_07350_b200 import lp

        z, cond = lp.synthetic_latent_host(DIMS, d, 2025)
        dit = lp.DiTDenoiser(list(cond), num_layers=2) if denoiser == "dit" else None
        eng = _engine(lp, denoiser, d, cond, WORLD, rank, dit)
        eng.load(lp.LatentTensor.from_numpy(z, d))
        for i in range(1, STEPS + 1):
            eng.step_phase(i, 1)
            buf, slot = eng.gather_buffer(i)
            torch.cuda.synchronize()
            mine = buf[rank * slot:(rank + 1) * slot].cpu()
            parts = [torch.empty_like(mine) for _ in range(WORLD)]
            dist.all_gather(parts, mine)
            buf[:WORLD * slot].copy_(torch.cat(parts).cuda())
            eng.step_phase(i, 3)
        torch.cuda.synchronize()
        out = eng.z.data.cpu().numpy().tobytes()
        eng.close()
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, repr(e)))


def _run(denoiser, d):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + (os.getpid() % 1000) + 7 * d
    procs = [ctx.Process(target=_worker, args=(r, port, q, denoiser, d)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=600) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
    for r, out in res:
        assert isinstance(out, bytes), out
    assert res[0][1] == res[1][1], "ranks disagree"
    return res[0][1]


@pytest.mark.gpu
@pytest.mark.parametrize("d", [2, 4])
def test_two_rank_engine_toy_bitexact_vs_oracle(cuda, oracle, d):
    got = _run("box", d)
    z, cond = oracle.synthetic(DIMS, d, 2025)
    want, _ = oracle.run_lp(0, (1, 1, 1), z, d, STEPS, 0.05, 5.0, cond, PATCH, K, R)
    dt = {2: np.float16, 4: np.float32}[d]
    assert np.frombuffer(got, dt).astype(np.float64).tobytes() == want.tobytes()


@pytest.mark.gpu
def test_two_rank_engine_dit_equals_single_process(cuda):
    from paper_2512_07350_b200 import lp

    got = _run("dit", 4)
    z, cond = lp.synthetic_latent_host(DIMS, 4, 2025)
    dit = lp.DiTDenoiser(list(cond), num_layers=2)
    eng = _engine(lp, "dit", 4, cond, 1, 0, dit)
    eng.load(lp.LatentTensor.from_numpy(z, 4))
    eng.run(1, STEPS)
    want = eng.z.data.cpu().numpy().tobytes()
    eng.close()
    assert got == want
