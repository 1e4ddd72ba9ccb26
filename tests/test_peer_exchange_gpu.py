"""K9 over NVLink peer memory: engines created without an NCCL id exchange their CUDA IPC
arena handles (gloo all_gather_object here) and attach; lp_engine_run then pushes each
rank's ε̂ slot into every peer's double-buffered gather buffer with remote stores, publishes
a per-step epoch flag (system-scope release) and starts K10 when every peer's flag has
arrived (engine.cpp step_exchange_peer, lp_kernels.cu k_peer_push / k_peer_wait).

Two processes share one B200 (CUDA IPC works within a device, so this runs the real push /
flag / wait kernels; across GPUs the same stores travel over NVLink).  Toy denoiser: both
ranks equal the oracle's single-process run_lp bit for bit.  DiT: both ranks equal a world=1
engine bit for bit.  No peer-timeout flag may be raised.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

DIMS = (16, 5, 16, 16)
PATCH = (1, 2, 2)
K, R = 4, 0.5


def _engine(lp, denoiser, d, cond, world, rank, dit=None, steps=5):
    return lp.LpEngine(DIMS, PATCH, d, K, R, steps, 0.05, 5.0, list(cond), denoiser=denoiser, radius=(1, 1, 1),
                       world=world, rank=rank, dit=dit)


def _worker(rank, port, q, denoiser, d, WORLD, STEPS):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        torch.cuda.set_device(0)
        from paper_2512_07350_b200 import lp

        z, cond = lp.synthetic_latent_host(DIMS, d, 2025)
        dit = lp.DiTDenoiser(list(cond), num_layers=2) if denoiser == "dit" else None
        eng = _engine(lp, denoiser, d, cond, WORLD, rank, dit, STEPS)
        eng.load(lp.LatentTensor.from_numpy(z, d))
        handles = [None] * WORLD
        dist.all_gather_object(handles, eng.ipc_handle())
        eng.ipc_attach(handles)
        dist.barrier()
        lp.device_flags(reset=True)
        eng.run(1, STEPS)
        torch.cuda.synchronize()
        flags = lp.device_flags(reset=True)
        out = eng.z.data.cpu().numpy().tobytes()
        comm = eng.comm()
        dist.barrier()  # keep the arenas mapped until every rank is done
        eng.close()
        q.put((rank, out, flags, comm))
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, repr(e), None, None))


def _run(denoiser, d, WORLD=2, STEPS=5):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 1000) + 13 * d + 3 * WORLD
    procs = [ctx.Process(target=_worker, args=(r, port, q, denoiser, d, WORLD, STEPS)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(WORLD)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for r, out, flags, _ in res:
        assert isinstance(out, bytes), out
        assert flags == 0, f"rank {r} raised device flags {flags} (4 = peer timeout)"
    assert all(r[1] == res[0][1] for r in res), "ranks disagree"
    assert res[0][3]["nccl_bytes_received"] > 0
    return res[0][1]


@pytest.mark.gpu
@pytest.mark.parametrize("world,steps", [(2, 5), (3, 9)])
def test_peer_exchange_toy_bitexact_vs_oracle(cuda, oracle, world, steps):
    got = _run("box", 4, world, steps)
    z, cond = oracle.synthetic(DIMS, 4, 2025)
    want, _ = oracle.run_lp(0, (1, 1, 1), z, 4, steps, 0.05, 5.0, cond, PATCH, K, R)
    assert np.frombuffer(got, np.float32).astype(np.float64).tobytes() == want.tobytes()


@pytest.mark.gpu
def test_peer_exchange_dit_equals_single_process(cuda):
    from paper_2512_07350_b200 import lp

    got = _run("dit", 4)
    z, cond = lp.synthetic_latent_host(DIMS, 4, 2025)
    dit = lp.DiTDenoiser(list(cond), num_layers=2)
    eng = _engine(lp, "dit", 4, cond, 1, 0, dit)
    eng.load(lp.LatentTensor.from_numpy(z, 4))
    eng.run(1, 5)
    want = eng.z.data.cpu().numpy().tobytes()
    eng.close()
    assert got == want
