"""Hybrid LP x intra-group model parallelism (the reference models its
traffic in src/cost.cpp:133-213 cost_hybrid): world = G LP groups x M pipeline stages.
Rank r is stage r % M of group r // M and runs DiT blocks [s*L/M, (s+1)*L/M); stage 0
gathers and embeds, the last stage writes the group's ε̂ slot.

Each case runs world processes sharing one GPU, each an lp_engine with group_size=M and no
NCCL id, driven stage by stage: the activation moves rank -> rank+1 by gloo send/recv where
the NCCL run uses ncclSend/Recv, and each group's ε̂ slot is broadcast from its last stage
where the NCCL run uses ncclBroadcast (engine.cpp hybrid_entry / step_exchange).

Checked: every rank ends with the latent of a plain world=1 engine, bit for bit (a stage
split moves the fp32 residual stream unchanged), and within the stated tolerance of the
UNMODIFIED reference run_lp driving the fp32 oracle DiT; the activation bytes all ranks sent
equal the reference's cost_hybrid intra-group bytes at hidden = d and 4-byte words.
"""
import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

DIMS = (16, 6, 16, 16)
PATCH = (1, 2, 2)
STEPS = 3


def _engine(lp, dit, cond, K, world, rank, M):
    return lp.LpEngine(DIMS, PATCH, 4, K, _r(K), STEPS, 0.05, 5.0, list(cond), denoiser="dit", dit=dit, world=world,
                       rank=rank, group_size=M)


def _r(K):
    return 0.0 if K == 1 else 0.5  # K = 1 requires r = 0 (src/partition.cpp:66)


def _worker(rank, world, M, K, layers, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2512_07350_b200 import lp

        z, cond = lp.synthetic_latent_host(DIMS, 4, 2025)
        dit = lp.DiTDenoiser(list(cond), num_layers=layers)
        eng = _engine(lp, dit, cond, K, world, rank, M)
        eng.load(lp.LatentTensor.from_numpy(z, 4))
        info = eng.hybrid()
        stage, G = info["stage"], world // M
        for i in range(1, STEPS + 1):
            for idx in range(eng.owned(i)):
                act = eng.stage_activation(i, idx)
                if stage > 0:
                    buf = torch.empty(act.numel(), dtype=torch.float32)
                    dist.recv(buf, src=rank - 1)
                    act.copy_(buf.cuda())
                eng.stage(i, idx)
                if stage < M - 1:
                    torch.cuda.synchronize()
                    dist.send(act.cpu(), dst=rank + 1)
            gbuf, slot = eng.gather_buffer(i)
            torch.cuda.synchronize()
            for g in range(G):
                part = gbuf[g * slot:(g + 1) * slot].cpu()
                dist.broadcast(part, src=g * M + M - 1)
                gbuf[g * slot:(g + 1) * slot].copy_(part.cuda())
            eng.step_phase(i, 3)
        torch.cuda.synchronize()
        out = eng.z.data.cpu().numpy().tobytes()
        q.put((rank, out, eng.hybrid()))
        eng.close()
        dist.destroy_process_group()
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, repr(e), None))


def _run(world, M, K, layers):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + (os.getpid() % 500) + 11 * world + M
    procs = [ctx.Process(target=_worker, args=(r, world, M, K, layers, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=900) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    for r, out, _ in res:
        assert isinstance(out, bytes), out
    return res


@pytest.mark.gpu
@pytest.mark.parametrize("world,M,K,layers", [(2, 2, 1, 2), (4, 2, 2, 3), (3, 3, 1, 3)],
                         ids=["1group-2stages", "2groups-2stages-uneven", "1group-3stages"])
def test_hybrid_groups_equal_plain_lp_and_cost_model(cuda, reference, world, M, K, layers):
    import numpy as np

    from paper_2512_07350_b200 import lp
    from tests.test_parity_schedule_gpu import _oracle

    res = _run(world, M, K, layers)
    outs = {out for _, out, _ in res}
    assert len(outs) == 1, "ranks disagree"
    z, cond = lp.synthetic_latent_host(DIMS, 4, 2025)
    dit = lp.DiTDenoiser(list(cond), num_layers=layers)
    ref = _engine(lp, dit, cond, K, 1, 0, 1)
    ref.load(lp.LatentTensor.from_numpy(z, 4))
    ref.run(1, STEPS)
    want = ref.z.data.cpu().numpy().tobytes()
    ref.close()
    assert res[0][1] == want
    # and against the oracle: the UNMODIFIED reference run_lp driving the fp32 oracle DiT (its own
    # regenerated weights and text), at the stated per-step tolerance of
    # tests/test_parity_schedule_gpu.py after the last step
    torch.backends.cuda.matmul.allow_tf32 = False
    refd, ck, cv, _ = _oracle(dit, cond)

    def predict(zz, t, c, is_null):
        return refd.predict(torch.from_numpy(zz).float().cuda(), t, ck, cv, 0 if is_null else 1).double().cpu().numpy()

    os.environ["LPSIM_THREADS"] = "0"
    final, _ = reference.run_lp_callback(predict, z, 4, STEPS, 0.05, 5.0, cond, PATCH, K, _r(K))
    got = np.frombuffer(res[0][1], dtype=np.float32).reshape(DIMS).astype(np.float64)
    rel = np.linalg.norm(got - final) / np.linalg.norm(final - np.asarray(z, np.float64))
    assert np.isfinite(rel) and rel <= 1.5e-2, rel
    assert np.abs(got - final).max() <= 5e-3 + 1e-3 * STEPS
    # stage layer ranges tile [0, L) and the activation traffic matches cost_hybrid
    spans = sorted((h["stage"], h["layer_begin"], h["layer_end"]) for _, _, h in res if h["group"] == 0)
    assert spans[0][1] == 0 and spans[-1][2] == layers
    assert all(spans[j][2] == spans[j + 1][1] for j in range(len(spans) - 1))
    sent = sum(h["intra_bytes_sent"] for _, _, h in res)
    cr = lp.cost_report(STEPS, world, _r(K), DIMS, PATCH, preset="custom", hidden_dim=dit.cfg.dim, wire_bytes=4,
                        hybrid=(world // M, [M] * (world // M)))
    assert sent == cr["hybrid"]["C_intra_total"], (sent, cr["hybrid"])


def test_hybrid_config_validation():
    from paper_2512_07350_b200 import lp

    z, cond = lp.synthetic_latent_host(DIMS, 4, 2025)
    with pytest.raises(lp.LpError, match="DiT"):  # toy denoisers cannot be pipelined
        lp.LpEngine(DIMS, PATCH, 4, 2, 0.5, STEPS, 0.05, 5.0, list(cond), denoiser="box", world=2, rank=0,
                    group_size=2)


def test_hybrid_world_must_divide():
    from paper_2512_07350_b200 import lp

    z, cond = lp.synthetic_latent_host(DIMS, 4, 2025)
    with pytest.raises(lp.LpError, match="multiple of group_size"):  # checked before any device work
        lp.LpEngine(DIMS, PATCH, 4, 1, 0.0, STEPS, 0.05, 5.0, list(cond), denoiser="box", world=3, rank=0,
                    group_size=2)
