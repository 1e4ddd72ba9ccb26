"""World-size-2 test of the multi-rank LP path on CPU (gloo).

Each rank takes the product's shard layout (lp_shard_layout / lp_shard_bases,
the layout engine.cpp uses for its ncclAllGather).  It computes ITS entries'
cfg predictions and packs them into its slot.  The ranks all-gather the padded
slots, reconstruct and apply the sampler from the gathered buffer.  Every rank
must hold the same latent as a single-process run_lp, bit for bit, and the
bytes moved must equal the product's accounting.  The oracle stands in for the
GPU compute here: it is the checker, not the thing measured.
"""
import os

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2
DIMS = (3, 9, 8, 10)
PATCH = (1, 2, 2)
K, R, STEPS, D = 4, 0.5, 6, 4


def _worker(rank, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=WORLD)
        from oracle.oracle import Oracle, sub_shape
        from paper_2512_07350_b200 import lp

        orc = Oracle()
        z, cond = orc.synthetic(DIMS, D, 77)
        moved = 0
        for i in range(1, STEPS + 1):
            t = STEPS + 1 - i
            plan = lp.build_plan(DIMS, PATCH, i, K, R)
            owned, slot = lp.shard_layout(plan, DIMS, WORLD, rank)
            bases = lp.shard_bases(plan, DIMS, WORLD)
            fp = orc.build_plan(DIMS, PATCH, i, K, R)
            subs = orc.extract(z, fp)
            offs = plan.offsets(DIMS)
            mine = np.zeros(slot, np.float64)
            for e in owned:
                s = subs[offs[e]:offs[e + 1]].reshape(sub_shape(DIMS, fp, e))
                pred = orc.cfg_predict(0, (1, 1, 1), s, D, t, cond, 3.0).reshape(-1)
                b = bases[e] - rank * slot
                mine[b:b + pred.size] = pred
            bufs = [torch.zeros(slot, dtype=torch.float64) for _ in range(WORLD)]
            dist.all_gather(bufs, torch.from_numpy(mine))
            moved += slot * (WORLD - 1) * D  # received by this rank (at storage width)
            gathered = torch.cat(bufs).numpy()
            packed = np.concatenate([gathered[bases[e]:bases[e] + offs[e + 1] - offs[e]] for e in range(plan.workers)])
            eps = orc.reconstruct(packed, DIMS, D, fp)
            z = orc.sampler_step(z, eps, D, 0.05)
            ledger, ag = lp.step_comm_bytes(plan, DIMS, 2, WORLD, D)
            assert ag == WORLD * (WORLD - 1) * slot * D
        q.put((rank, z.tobytes(), moved))
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, repr(e), -1))


def test_two_rank_gloo_matches_single_process(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    for r, zb, moved in res:
        assert moved >= 0, zb
    z, cond = oracle.synthetic(DIMS, D, 77)
    want, _ = oracle.run_lp(0, (1, 1, 1), z, D, STEPS, 0.05, 3.0, cond, PATCH, K, R)
    for r, zb, _ in res:
        assert np.frombuffer(zb, np.float64).reshape(DIMS).tobytes() == want.tobytes(), f"rank {r} differs"
    assert res[0][1] == res[1][1]


def test_shard_layout_round_robin_covers_all_entries():
    from paper_2512_07350_b200 import lp

    for world in (1, 2, 3, 4, 8):
        for step in (1, 2, 3):
            plan = lp.build_plan((16, 21, 60, 104), PATCH, step, 8, 0.5)
            bases = lp.shard_bases(plan, (16, 21, 60, 104), world)
            offs = plan.offsets((16, 21, 60, 104))
            spans = sorted((bases[e], bases[e] + offs[e + 1] - offs[e]) for e in range(plan.workers))
            assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:])), "slots overlap"
            _, slot = lp.shard_layout(plan, (16, 21, 60, 104), world, 0)
            assert spans[-1][1] <= world * slot
