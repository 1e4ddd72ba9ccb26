"""K9 over NVLink peer memory: engines created without an NCCL id exchange their CUDA IPC
arena handles (gloo all_gather_object here) and attach; lp_engine_run then pushes each
rank's ε̂ slot into every peer's double-buffered gather buffer with remote stores, publishes
a per-step epoch flag (system-scope release) and starts K10 when every peer's flag has
arrived (engine.cpp step_exchange_peer, lp_kernels.cu k_peer_push / k_peer_wait).

Two processes share one B200 (CUDA IPC works within a device, so this runs the real push /
flag / wait kernels; across GPUs the same stores travel over NVLink).  Toy denoiser: both
ranks equal the oracle's single-process run_lp bit for bit.  DiT: both ranks equal a world=1
engine bit for bit.  No peer-timeout flag may be raised.  Worlds 2-4, storage dtypes f16/f32/f64,
and a one-channel latent whose rank slots are not 16-byte multiples of the element count (every
slot still starts 16-byte aligned: lp_shard_layout rounds slot_elems to 8 elements).  A stalled
peer makes lp_engine_sync raise WorkerFailure naming the worker and step, with z left as it was.
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


def _engine(lp, denoiser, d, cond, world, rank, dit=None, steps=5, dims=DIMS):
    return lp.LpEngine(dims, PATCH, d, K, R, steps, 0.05, 5.0, list(cond), denoiser=denoiser, radius=(1, 1, 1),
                       world=world, rank=rank, dit=dit)


def _worker(rank, port, q, denoiser, d, WORLD, STEPS, dims=DIMS):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        torch.cuda.set_device(0)
        from paper_2512_07350_b200 import lp

        z, cond = lp.synthetic_latent_host(dims, d, 2025)
        dit = lp.DiTDenoiser(list(cond), num_layers=2) if denoiser == "dit" else None
        eng = _engine(lp, denoiser, d, cond, WORLD, rank, dit, STEPS, dims)
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


def _run(denoiser, d, WORLD=2, STEPS=5, dims=DIMS, target=_worker):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + (os.getpid() % 1000) + 13 * d + 3 * WORLD + dims[0]
    procs = [ctx.Process(target=target, args=(r, port, q, denoiser, d, WORLD, STEPS, dims)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(WORLD)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    if target is not _worker:
        return res
    for r, out, flags, _ in res:
        assert isinstance(out, bytes), out
        assert flags == 0, f"rank {r} raised device flags {flags} (4 = peer timeout)"
    assert all(r[1] == res[0][1] for r in res), "ranks disagree"
    assert res[0][3]["nccl_bytes_received"] > 0
    return res[0][1]


_NP = {2: np.float16, 4: np.float32, 8: np.float64}


@pytest.mark.gpu
@pytest.mark.parametrize("world,steps,d,dims", [
    (2, 5, 4, DIMS), (3, 9, 4, DIMS), (4, 6, 2, DIMS), (2, 6, 8, DIMS),
    # C=1: 5x6x6 slots of 1-channel shards, not 16-B multiples (rank > 0 offsets)
    (2, 6, 4, (1, 5, 6, 6)), (3, 6, 2, (1, 5, 6, 6)), (4, 6, 4, (1, 7, 10, 6)),
])
def test_peer_exchange_toy_bitexact_vs_oracle(cuda, oracle, world, steps, d, dims):
    got = _run("box", d, world, steps, dims)
    z, cond = oracle.synthetic(dims, d, 2025)
    want, _ = oracle.run_lp(0, (1, 1, 1), z, d, steps, 0.05, 5.0, cond, PATCH, K, R)
    assert np.frombuffer(got, _NP[d]).astype(np.float64).tobytes() == want.tobytes()


def _stall_worker(rank, port, q, denoiser, d, WORLD, STEPS, dims):
    """Rank 1 attaches and then never runs a step (a stalled peer); rank 0 runs one step."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        os.environ["LP_TUNE_PEER_TIMEOUT_MS"] = "1500"
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        torch.cuda.set_device(0)
        from paper_2512_07350_b200 import lp

        z, cond = lp.synthetic_latent_host(dims, d, 2025)
        eng = _engine(lp, denoiser, d, cond, WORLD, rank, None, STEPS, dims)
        eng.load(lp.LatentTensor.from_numpy(z, d))
        handles = [None] * WORLD
        dist.all_gather_object(handles, eng.ipc_handle())
        eng.ipc_attach(handles)
        dist.barrier()
        msg, same = "", None
        if rank == 0:
            before = eng.z.data.cpu().numpy().tobytes()
            eng.run(1, 1)
            try:
                eng.sync(timeout_s=120)
            except lp.LpError as ex:
                msg = f"{ex.kind}|{ex}"
            same = eng.z.data.cpu().numpy().tobytes() == before
            lp.device_flags(reset=True)
        dist.barrier()
        eng.close()
        q.put((rank, msg, same, None))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, "exception|" + repr(e), None, None))


@pytest.mark.gpu
def test_peer_exchange_stalled_peer_is_a_worker_failure(cuda):
    res = _run("box", 4, 2, 4, DIMS, target=_stall_worker)
    kind, _, text = res[0][1].partition("|")
    assert kind == "WorkerFailure", res[0][1]
    # K=4 round-robin over 2 ranks: rank 1 owns workers 2 and 4 -> the lowest is named
    assert "worker 2 failed at step 1" in text and "rank 1" in text, text
    assert res[0][2] is True, "K10 must leave z untouched when a shard never arrived"


@pytest.mark.gpu
@pytest.mark.parametrize("world,steps", [(2, 5), (2, 14), (3, 14), (4, 8)])
def test_peer_exchange_dit_equals_single_process(cuda, world, steps):
    """14 steps: every (axis, gather-parity) step graph is captured (steps 7-12) and replayed
    (13-14), with the exchange epoch on the device; the result stays bit-identical."""
    from paper_2512_07350_b200 import lp

    got = _run("dit", 4, world, steps)
    z, cond = lp.synthetic_latent_host(DIMS, 4, 2025)
    dit = lp.DiTDenoiser(list(cond), num_layers=2)
    eng = _engine(lp, "dit", 4, cond, 1, 0, dit, steps)
    eng.load(lp.LatentTensor.from_numpy(z, 4))
    eng.run(1, steps)
    want = eng.z.data.cpu().numpy().tobytes()
    eng.close()
    assert got == want
