"""Measured DiT / LP-loop errors against the fp32 oracles (evidence for the tolerances written
in tests/test_dit_gpu.py and tests/test_parity_schedule_gpu.py).

1. One CFG forward (eps) of our bf16 tcgen05 DiT vs the fp32 torch restatement, beside the
   same restatement with every GEMM / attention operand rounded to bf16 (the precision floor
   of any bf16-operand implementation), at C1 size (2 and 30 blocks) and on a full-size C2
   shard (30 blocks, 14040 tokens, CFG batch 2).
2. Per-step trajectory errors of the LP loop: the UNMODIFIED reference run_lp (oracle/_ref)
   driving the fp32 DiT through its Denoiser slot, traced per step, vs our engine stepped
   one timestep at a time, for the C1 config (4 steps, K=2) and a 12-step K=2/K=4 schedule.

usage: python scripts/parity_report.py [--no-c2]  ->  gpurun_out/parity_report.json
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle.dit_fp32 import DiTReference  # noqa: E402
from paper_2512_07350_b200 import lp  # noqa: E402


def rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm())


def oracle_dit(dit, cond):
    """The oracle's own DiT (weights, text, cross K/V regenerated: oracle/dit_oracle.py)."""
    from oracle.dit_oracle import OracleDiT

    od = OracleDiT(dit.cfg, cond)
    return od, *od.context_kv()


def forward_case(shape, layers, t=37, w=5.0, seed=2025):
    z, cond = lp.synthetic_latent(shape, 4, seed)
    dit = lp.DiTDenoiser(cond, num_layers=layers)
    eps = dit.cfg_predict(z, t, w)
    torch.cuda.synchronize()
    od, ck, cv = oracle_dit(dit, cond)
    t0 = time.time()
    want, _ = DiTReference(od).forward(z.data.float(), t, ck, cv, w)
    emul, _ = DiTReference(od, act_bf16=True).forward(z.data.float(), t, ck, cv, w)
    torch.cuda.synchronize()
    out = {"shape": list(shape), "layers": layers, "t": t, "w": w,
           "rel_l2_ours_vs_fp32": rel(eps.data, want), "rel_l2_bf16_operands_vs_fp32": rel(emul, want),
           "rel_l2_ours_vs_bf16_operands": rel(eps.data, emul),
           "max_abs_ours_vs_fp32": float((eps.data.float() - want).abs().max()), "ref_seconds": time.time() - t0}
    out["ratio_to_bf16_floor"] = out["rel_l2_ours_vs_fp32"] / max(out["rel_l2_bf16_operands_vs_fp32"], 1e-30)
    dit.close() if hasattr(dit, "close") else None
    return out


def trajectory_case(ref, dims, K, r, steps, eta=0.05, w=5.0, layers=2, seed=2025):
    os.environ["LPSIM_THREADS"] = "0"
    z, cond = lp.synthetic_latent(dims, 4, seed)
    dit = lp.DiTDenoiser(cond, num_layers=layers)
    od, ck, cv = oracle_dit(dit, cond)
    dr = DiTReference(od)

    def predict(zz, t, c, is_null):
        return dr.predict(torch.from_numpy(zz).float().cuda(), t, ck, cv, 0 if is_null else 1).double().cpu().numpy()

    z0 = z.to_numpy()
    want, ledger, tr = ref.run_lp_callback(predict, z0, 4, steps, eta, w, cond, (1, 2, 2), K, r, trace=True)
    eng = lp.LpEngine(dims, (1, 2, 2), 4, K, r, steps, eta, w, cond, denoiser="dit", dit=dit)
    eng.load(z)
    per = []
    for i in range(1, steps + 1):
        eng.run(i, 1)
        torch.cuda.synchronize()
        got = eng.z.data.double().cpu().numpy()
        upd = np.linalg.norm(tr[i - 1] - z0)
        per.append({"step": i, "rel_l2_of_update": float(np.linalg.norm(got - tr[i - 1]) / upd),
                    "max_abs": float(np.abs(got - tr[i - 1]).max())})
    ledger_ours = eng.comm()["ledger_bytes"]
    eng.close()
    return {"dims": list(dims), "K": K, "r": r, "steps": steps, "layers": layers, "ledger_equal": ledger_ours == ledger,
            "per_step": per, "final_rel_l2_of_update": per[-1]["rel_l2_of_update"], "final_max_abs": per[-1]["max_abs"]}


def main():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    from oracle.oracle import Reference

    rep = {"forward": [], "trajectory": []}
    rep["forward"].append(forward_case((16, 5, 16, 16), 2))
    rep["forward"].append(forward_case((16, 5, 16, 16), 30))
    if "--no-c2" not in sys.argv:
        # C2's first T-axis shard at K=4 (frames [0,9) of 16x21x60x104): 9x30x52 = 14040 tokens
        rep["forward"].append(forward_case((16, 9, 60, 104), 30, t=50))
    ref = Reference()
    rep["trajectory"].append(trajectory_case(ref, (16, 5, 16, 16), 2, 0.5, 4))  # C1: the full 4-step schedule
    rep["trajectory"].append(trajectory_case(ref, (16, 5, 16, 16), 2, 0.5, 12))
    rep["trajectory"].append(trajectory_case(ref, (16, 6, 16, 24), 4, 0.5, 12))
    for f in rep["forward"]:
        print(json.dumps(f))
    for t in rep["trajectory"]:
        print(json.dumps({k: v for k, v in t.items() if k != "per_step"}))
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(rep, open("gpurun_out/parity_report.json", "w"), indent=1)


if __name__ == "__main__":
    main()
