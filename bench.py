"""LP denoise benchmark (BASELINE.json metric: LP denoise steps/s, WAN-1.3B-shape 480p 81f,
1/2/4/8 B200; comm bytes/video).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config c2|c4|c5]
    torchrun --nproc-per-node N bench.py --gpus N ...

`--gpus N` with N > 1 and no torchrun environment launches N ranks itself (torchrun on
127.0.0.1, one process per GPU) and fails loudly when fewer than N GPUs are visible; it never
reports fewer ranks than asked for.  `--plan-only` prints the per-rank shard assignment, the
exchange bytes and the FLOP-ideal speedup bound for N ranks without touching a GPU.

Workload (BASELINE.json configs[1], "C2", the default): WAN2.1-1.3B-shaped random-init DiT
(30 blocks, d=1536, 12 heads, FFN 8960, CFG batch 2) on the 480p/81-frame latent 16x21x60x104
(f32 storage), patch (1,2,2), LP with K = max(4, N) workers, r = 0.5, T = 50-step schedule,
eta 0.05, w 5.0, synthetic_inputs seed 2025.  Entries are dealt to the N ranks round-robin
(or balanced by DiT FLOPs, --assign balanced); N=1 runs all 4 shards on one GPU.  A "step" is
one LP denoise step: plan, K1 gather, DiT cfg_predict on this rank's shards, the ε̂ exchange
(N>1: NVLink peer stores fused into the DiT epilogue, or NCCL all-gather), K10 blend + sampler
update.  --config c4 / c5 run BASELINE configs[3] / [4] the same way (K = 8).

`value` is device-timed (CUDA events on the engine stream, max over ranks); `e2e` is the same
steps through the C-ABI engine with the latent copied in from pinned host memory and the result
copied back every step.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PATCH = (1, 2, 2)
T_SCHED = 50
ETA, W_CFG, SEED = 0.05, 5.0, 2025
UNIT = "steps/s"

# BASELINE.json configs: [1] = C2 (the metric's workload, default), [3] = C4, [4] = C5.
CONFIGS = {
    "c2": dict(dims=(16, 21, 60, 104), K=None, schedule=None, dit=dict(), d=1536, F=8960, layers=30, heads=12,
               metric="LP denoise steps/s, WAN-1.3B-shape 480p 81f (C2)",
               name="C2: WAN2.1-1.3B-shaped DiT ({L} blocks, d=1536, 12 heads, ffn 8960, CFG batch 2) on 480p81f "
                    "latent 16x21x60x104 f32"),
    "c4": dict(dims=(16, 21, 90, 160), K=8, schedule=None, dit=dict(dim=5120, num_heads=40, ffn_dim=13824), d=5120,
               F=13824, layers=40, heads=40, metric="LP denoise steps/s, WAN-14B-shape 720p 81f (C4)",
               name="C4: WAN2.1-14B-shaped DiT ({L} blocks, d=5120, 40 heads, ffn 13824, CFG batch 2) on 720p81f "
                    "latent 16x21x90x160 f32"),
    "c5": dict(dims=(16, 41, 60, 104), K=8, schedule="TTHTTW", dit=dict(), d=1536, F=8960, layers=30, heads=12,
               metric="LP denoise steps/s, WAN-1.3B-shape 480p 161f (C5)",
               name="C5: WAN2.1-1.3B-shaped DiT ({L} blocks, d=1536, 12 heads, ffn 8960, CFG batch 2) on 480p161f "
                    "latent 16x41x60x104 f32, temporal-heavy schedule TTHTTW"),
}

# LP_BENCH_GLOO_TEST=1 (on a ONE-GPU box): every rank on GPU 0, gloo plumbing, no NCCL
# communicator, ε̂ exchange over CUDA IPC peer memory.  Validates the multi-rank bench path where
# NCCL refuses two ranks on one device; its numbers are not scaling numbers.
GLOO_TEST = os.environ.get("LP_BENCH_GLOO_TEST") == "1"


class Cfg:
    """The run's workload: a BASELINE config, the LP worker count for N ranks, the DiT depth."""

    def __init__(self, args, world):
        c = CONFIGS[args.config]
        self.key = args.config
        self.dims = c["dims"]
        self.metric = c["metric"]
        self.r = args.overlap if args.overlap is not None else 0.5
        self.M = max(1, args.hybrid)
        self.K = args.workers or c["K"] or (world // self.M if self.M > 1 else max(4, world))
        self.K1 = args.workers or c["K"] or 4  # the same job's K on one GPU (FLOP-ideal baseline)
        self.layers = args.layers or c["layers"]
        self.schedule = c["schedule"]
        self.d, self.F, self.heads = c["d"], c["F"], c["heads"]
        self.dit_kwargs = dict(c["dit"], num_layers=self.layers)
        self.name = c["name"].format(L=self.layers)
        self.assign = args.assign

    def axes(self):
        from paper_2512_07350_b200 import lp

        return lp.parse_schedule(self.schedule) if self.schedule else [0, 1, 2]

    def axis_of(self, step):
        a = self.axes()
        return a[(step - 1) % len(a)]

    def plan(self, step, K=None):
        from paper_2512_07350_b200 import lp

        a = self.axis_of(step)
        return lp.build_axis_plan(a, self.dims[1 + a], PATCH[a], step, K or self.K, self.r)

    def tokens(self, shape):
        return -(-shape[1] // PATCH[0]) * -(-shape[2] // PATCH[1]) * -(-shape[3] // PATCH[2])

    def entry_flops(self, shape):
        """Algorithmic FLOPs of the CFG-batched DiT on one shard: GEMM 2MNK with M = 2n over QKV, O,
        cross-Q, cross-O, FFN1, FFN2; self-attention 4 n^2 d per batch; cross-attention 4 n 512 d;
        minus block 0's self-attention sub-block of one half (QKV + O GEMMs, attention): both CFG
        halves are identical there, so the engine computes it once (knob dit_dedupe0)."""
        n, d = self.tokens(shape), self.d
        full = self.layers * (2 * 2 * n * (6 * d * d + 2 * d * self.F) + 2 * 4 * n * n * d + 2 * 4 * n * 512 * d)
        return full - (2 * n * 4 * d * d + 4 * n * n * d)

    def cost_model(self):
        """lp_shard_layout_ex cost per element (balanced assignment): linear ~ n, attention ~ n^2."""
        per_tok = self.dims[0] * PATCH[0] * PATCH[1] * PATCH[2]
        return 4.0 * (6 * self.d ** 2 + 2 * self.d * self.F) / per_tok, 8.0 * self.d / per_tok ** 2

    def layout(self, step, world, K=None):
        """owner rank of every entry at `step` (the engine's assignment)."""
        from paper_2512_07350_b200 import lp

        p = self.plan(step, K)
        lin, quad = self.cost_model()
        _, _, owner, _ = lp.shard_layout_ex(p, self.dims, world, 0, self.assign, lin, quad)
        return p, owner

    def workload(self, world):
        return {
            "workload": f"{self.name}, patch (1,2,2), LP K={self.K} r={self.r}, T={T_SCHED}, eta {ETA}, w {W_CFG}",
            "lp_workers": self.K, "overlap_ratio": self.r, "latent": list(self.dims), "patch": list(PATCH),
            "schedule_steps": T_SCHED, "axis_schedule": self.schedule or "rotating T,H,W", "ranks": world,
            "shard_assignment": f"{self.assign} entries over ranks",
            "scaling_note": "strong: one fixed video job; C2 uses K = max(4, N) LP workers, so N = 8 re-partitions "
                            "the job into 8 shards (the FLOP-ideal bound in scaling_model accounts for it)",
            "parallelism": f"lp{self.K} over {world} GPU(s)" if self.M == 1 else
            f"hybrid: {world // self.M} LP groups x {self.M} pipeline stages",
            "l2": "working set > L2 (2.6 GB of bf16 weights streamed per forward, >100 MB activations)",
            "cuda_graphs": "each step graph captured before the warm-up (priming steps on a scratch copy of z, "
                           "restored after); warm-up and timed steps replay graphs",
        }


def step_index(s):
    return (s - 1) % T_SCHED + 1


def scaling_model(cfg, world):
    """Per-rank DiT FLOPs of the rotation cycle under the engine's assignment, and the FLOP-ideal
    speedup over the same job on one GPU: mean_axis(total FLOPs at K1) / mean_axis(max-rank FLOPs).
    It bounds what the N-rank step can reach if every rank ran at the one-GPU throughput."""
    axes = cfg.axes()
    per_rank = [[0.0] * world for _ in axes]
    one_gpu, keff, owners = [], [], []
    for i in range(len(axes)):
        p, owner = cfg.layout(i + 1, world)
        keff.append(p.workers)
        owners.append(owner)
        for k in range(p.workers):
            per_rank[i][owner[k]] += cfg.entry_flops(p.sub_shape(cfg.dims, k))
        p1 = cfg.plan(i + 1, cfg.K1)
        one_gpu.append(sum(cfg.entry_flops(p1.sub_shape(cfg.dims, k)) for k in range(p1.workers)))
    mx = [max(r) for r in per_rank]
    tot = [sum(r) for r in per_rank]
    return {
        "axes": "".join("THW"[a] for a in axes), "k_eff_per_axis": keff,
        "owner_per_axis": owners,
        "rank_tflop_per_cycle": [sum(per_rank[i][r] for i in range(len(axes))) / 1e12 for r in range(world)],
        "max_rank_tflop_per_step_mean": statistics.mean(mx) / 1e12,
        "one_gpu_tflop_per_step_mean": statistics.mean(one_gpu) / 1e12,
        "flop_ideal_speedup_vs_1gpu": statistics.mean(one_gpu) / statistics.mean(mx),
        "rank_balance": statistics.mean(t / world / m for t, m in zip(tot, mx)),
    }


# ---------------------------------------------------------------------------
# clocks (NVML) sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, v in self.REASONS.items():
                    if mask & v and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# The reference's CPU path: the UNMODIFIED reference run_lp (oracle/_ref) with a CPU DiT
# ---------------------------------------------------------------------------
def cpu_reference_run(cfg, steps, threads):
    """LP machinery alone: the reference run_lp with its own box denoiser (rho=1) at the shape."""
    from oracle.oracle import Oracle, Reference, reference_available

    os.environ["LPSIM_THREADS"] = str(threads)
    kind = "reference" if reference_available() else "port"
    lib = Reference() if kind == "reference" else Oracle()
    z, cond = lib.synthetic(cfg.dims, 4, SEED)
    t0 = time.perf_counter()
    lib.run_lp(0, (1, 1, 1), z, 4, steps, ETA, W_CFG, cond, PATCH, cfg.K, cfg.r)
    dt = time.perf_counter() - t0
    used = min(threads, cfg.K) if kind == "reference" else 1
    sample = (f"reference run_lp (box denoiser rho=1 in place of the DiT: the reference has none), latent "
              f"{'x'.join(map(str, cfg.dims))} f32, K={cfg.K}, r={cfg.r}, {steps} steps; LPSIM_THREADS={threads} "
              f"(the pool uses min(threads, K) workers; extract/reconstruct/sampler are single-threaded)")
    return steps / dt, {"kind": kind, "cores": used, "sample": sample, "seconds": dt}


def _cpu_dit(cfg, layers):
    import torch

    from oracle.cpu_dit import CpuDiT

    kw = dict(cfg.dit_kwargs)
    kw.pop("num_layers", None)
    return CpuDiT(num_layers=layers, dtype=torch.bfloat16, **kw)


def reference_full_steps(cfg, steps, threads):
    """The reference arm's measurement: the UNMODIFIED reference run_lp (oracle/_ref) for `steps`
    whole LP steps (step 1 = T axis, then H, W ...) with the full-depth bf16 CPU DiT in its
    Denoiser slot (oracle/cpu_dit.py).  Nothing is scaled: the wall time is what ran."""
    import torch

    from oracle.oracle import Reference

    os.environ["LPSIM_THREADS"] = "0"  # serial workers: each predict() gets every host thread
    torch.set_num_threads(threads)
    ref = Reference()
    z, cond = ref.synthetic(cfg.dims, 4, SEED)
    dit = _cpu_dit(cfg, cfg.layers)
    # warm-up outside the timing: page in oneDNN's AMX kernels on a small shard, one block's shape
    dit.predict(z[:, :1, :8, :8], 1, cond, True)
    dit.calls.clear()
    t0 = time.perf_counter()
    _, _, trace = ref.run_lp_callback(dit.predict, z, 4, steps, ETA, W_CFG, cond, PATCH, cfg.K, cfg.r, trace=True)
    wall = time.perf_counter() - t0
    dit_s = sum(e - s for s, e in dit.calls)
    return wall, dit_s, len(dit.calls)


def reference_sample(cfg, threads):
    """Bounded sample for our arm's cpu_baseline (about 10-30 s of CPU work): the reference run_lp
    for one step (T axis) with a ONE-block bf16 CPU DiT in its Denoiser slot; the DiT's share is
    scaled to the full depth (all blocks have one shape) and to the cycle-mean shard FLOPs."""
    import torch

    from oracle.oracle import Reference

    os.environ["LPSIM_THREADS"] = "0"
    torch.set_num_threads(threads)
    ref = Reference()
    z, cond = ref.synthetic(cfg.dims, 4, SEED)
    dit = _cpu_dit(cfg, 1)
    dit.predict(z[:, :1, :8, :8], 1, cond, True)
    dit.calls.clear()
    t0 = time.perf_counter()
    ref.run_lp_callback(dit.predict, z, 4, 1, ETA, W_CFG, cond, PATCH, cfg.K, cfg.r)
    wall = time.perf_counter() - t0
    dit_s = sum(e - s for s, e in dit.calls)

    def axis_flops(step):
        p = cfg.plan(step)
        return sum(cfg.entry_flops(p.sub_shape(cfg.dims, k)) for k in range(p.workers))

    cyc = statistics.mean(axis_flops(i + 1) for i in range(len(cfg.axes())))
    scale = cfg.layers * cyc / axis_flops(1)
    est = (wall - dit_s) + dit_s * scale
    sample = (f"UNMODIFIED reference run_lp (oracle/_ref), 1 step (T axis) of {cfg.key.upper()} with a ONE-block "
              f"bf16 CPU DiT (oracle/cpu_dit.py, AMX) in its Denoiser slot: wall {wall:.2f} s of which DiT {dit_s:.2f} s; "
              f"DiT share scaled x{scale:.2f} ({cfg.layers} blocks x cycle-mean/T-axis shard FLOPs); serial workers, "
              f"{threads} torch threads.  bench.py --impl reference times whole {cfg.layers}-block steps instead")
    return 1.0 / est, sample


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    from oracle.oracle import reference_available

    cfg = Cfg(args, world)
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (the compiled reference) was not built"}))
        return
    cpu_reference_run(cfg, 1, threads)
    lp_only, lp_info = cpu_reference_run(cfg, 20, threads)
    # whole steps of the metric's workload, nothing extrapolated.  Default: ONE step (step 1, the
    # T axis: ~210 s on 16 cores, so the arm ends within a few minutes); its shards carry ~7% more
    # DiT FLOPs than the T/H/W cycle mean, so one T step slightly understates the reference's
    # cycle throughput.  --ref-steps 3 times a whole cycle.
    n = args.ref_steps or 1
    wall, dit_s, calls = reference_full_steps(cfg, n, threads)
    value = n / wall
    sample = (f"UNMODIFIED reference run_lp (oracle/_ref) for {n} whole LP steps (steps 1..{n}: axes "
              f"{''.join('THW'[cfg.axis_of(i)] for i in range(1, n + 1))}) of {cfg.key.upper()} "
              f"({'x'.join(map(str, cfg.dims))} f32, K={cfg.K}, r={cfg.r}, eta {ETA}, w {W_CFG}) with the full "
              f"{cfg.layers}-block WAN-shaped DiT (bf16 GEMM/attention on AMX, fp32 residual; random weights) in its "
              f"Denoiser slot, {calls} predict() calls; wall {wall:.1f} s of which DiT {dit_s:.1f} s; serial workers "
              f"(LPSIM_THREADS=0), {threads} torch threads.  Timed once: the requested --steps {args.steps} "
              f"--warmup {args.warmup} would take {(args.steps + args.warmup) * wall / n / 60:.0f} min")
    line = {
        "impl": "reference", "metric": cfg.metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": n,
        "warmup": 0, "ms_per_step": 1000.0 * wall / n, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16 (CPU DiT GEMM/attention) / f64 (LP machinery)",
        "data": "synthetic (synthetic_inputs seed 2025; random-init weights)",
        "config": cfg.workload(world),
        "requested": {"steps": args.steps, "warmup": args.warmup},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "lp_machinery_only": {"value": lp_only, "unit": UNIT, "cores": lp_info["cores"], "sample": lp_info["sample"]},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# plan only (no GPU): the assignment, exchange bytes and FLOP-ideal bound for N ranks
# ---------------------------------------------------------------------------
def run_plan_only(args, rank, world):
    import torch.distributed as dist

    from paper_2512_07350_b200 import lp

    cfg = Cfg(args, world)
    mine = {"rank": rank, "owned_entries": {}, "tokens": {}}
    for a in sorted(set(cfg.axes())):
        p, owner = cfg.layout(cfg.axes().index(a) + 1, world)
        ks = [k for k in range(p.workers) if owner[k] == rank]
        mine["owned_entries"]["THW"[a]] = [k + 1 for k in ks]
        mine["tokens"]["THW"[a]] = [cfg.tokens(p.sub_shape(cfg.dims, k)) for k in ks]
    ranks = [mine]
    if world > 1:
        ranks = [None] * world
        dist.all_gather_object(ranks, mine)
    if rank != 0:
        return
    ag = led = 0
    for i in range(1, T_SCHED + 1):
        a, b = lp.step_comm_bytes(cfg.plan(i), cfg.dims, 2, world // cfg.M, 4)
        led += a
        ag += b
    print(json.dumps({"mode": "plan-only", "metric": cfg.metric, "n_gpus": world, "config": cfg.workload(world),
                      "ranks": ranks, "scaling_model": scaling_model(cfg, world),
                      "comm": {"allgather_bytes_per_video": ag, "reference_ledger_bytes_per_video": led}}), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2512_07350_b200 import _lib, lp

    L = _lib.lib()
    torch.cuda.set_device(local_rank)
    _lib.check(L.lp_device_check(local_rank))
    cfg = Cfg(args, world)
    M = cfg.M
    if world % M:
        raise SystemExit(f"--hybrid {M} must divide the number of GPUs {world}")
    dims, K = cfg.dims, cfg.K
    z_host_np, cond = lp.synthetic_latent_host(dims, 4, SEED)
    dit = lp.DiTDenoiser(cond, **cfg.dit_kwargs)
    nccl_id = None
    if world > 1 and not GLOO_TEST and (args.exchange == "nccl" or M > 1):
        obj = [lp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    eng = lp.LpEngine(dims, PATCH, 4, K, cfg.r, T_SCHED, ETA, W_CFG, cond, denoiser="dit", dit=dit, world=world,
                      rank=rank, nccl_id=nccl_id, group_size=M, schedule=cfg.schedule, assign=cfg.assign)
    exchange = "nccl" if nccl_id is not None else "none"
    if world > 1 and M == 1 and args.exchange == "peer":
        # K9 over NVLink peer memory (CUDA IPC); every rank must map every peer, else fall back to NCCL
        handles = [None] * world
        dist.all_gather_object(handles, eng.ipc_handle())
        ok = 1
        try:
            eng.ipc_attach(handles)
        except Exception as ex:  # noqa: BLE001
            print(f"rank {rank}: peer attach failed ({ex}); exchanging through NCCL", file=sys.stderr)
            ok = 0
        t = torch.tensor([ok], dtype=torch.int32, device="cpu" if GLOO_TEST else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if int(t.item()) == 1:
            exchange = "peer"
        else:
            if ok:
                eng.ipc_detach()
            if GLOO_TEST:
                raise SystemExit("peer attach failed under LP_BENCH_GLOO_TEST (no NCCL fallback on one GPU)")
            eng.close()
            obj = [lp.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            eng = lp.LpEngine(dims, PATCH, 4, K, cfg.r, T_SCHED, ETA, W_CFG, cond, denoiser="dit", dit=dit,
                              world=world, rank=rank, nccl_id=obj[0], schedule=cfg.schedule, assign=cfg.assign)
            exchange = "nccl"
    z0 = torch.from_numpy(z_host_np.astype("float32")).pin_memory()
    eng.z.data.copy_(z0)
    stream = torch.cuda.current_stream()
    tmo = args.sync_timeout

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if GLOO_TEST else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # One-time setup, outside every timed region: the engine captures each step graph (one per
    # schedule axis, and per exchange-buffer parity on the peer path) on that graph's second
    # occurrence.  Run those occurrences now on a scratch copy of the latent, so the W warm-up
    # steps and the K timed steps replay captured graphs (otherwise the first cycle of timed
    # steps would include the eager runs and graph instantiation).
    n_graph_keys = len(cfg.axes()) * (2 if exchange == "peer" else 1)
    z_keep = eng.z.data.clone()
    for s in range(1, 2 * n_graph_keys + 1):
        eng.run(step_index(s), 1)
    eng.sync(tmo)
    eng.z.data.copy_(z_keep)
    del z_keep

    # warm-up
    for s in range(1, args.warmup + 1):
        eng.run(step_index(s), 1)
    eng.sync(tmo)

    # ---- device-timed region: K steps, inputs resident in HBM ----
    first = args.warmup + 1
    c0, l0 = eng.comm(), L.lp_launch_count()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        for s in range(first, first + args.steps):
            eng.run(step_index(s), 1)
        ev1.record(stream)
        eng.sync(tmo)  # a dead or stalled peer raises WorkerFailure instead of hanging
    barrier()
    launches = int(L.lp_launch_count() - l0)
    my_ms = ev0.elapsed_time(ev1)
    ms = max_over_ranks(my_ms)
    c1 = eng.comm()

    # ---- end-to-end through the C-ABI engine with host buffers ----
    zin = torch.empty(dims, dtype=torch.float32).pin_memory()
    zin.copy_(z0)
    zout = torch.empty_like(zin).pin_memory()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(first, first + args.steps):
        eng.z.data.copy_(zin, non_blocking=True)          # H2D: the step's input latent
        eng.run(step_index(s), 1)
        zout.copy_(eng.z.data, non_blocking=True)         # D2H: the step's result
    e1.record(stream)
    eng.sync(tmo)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    assert torch.isfinite(zout).all(), "non-finite latent"
    if lp.device_flags(reset=True) & 4:
        raise SystemExit(f"rank {rank}: peer exchange watchdog fired (a peer's epoch flag never arrived)")
    if world > 1:
        # z is replicated: every rank must hold the same bits after the exchanges (catches a
        # broken exchange that still yields finite numbers)
        chk = torch.tensor([int(eng.z.data.view(torch.int32).to(torch.int64).sum().item())], dtype=torch.int64,
                           device="cpu" if GLOO_TEST else "cuda")
        lo, hi = chk.clone(), chk.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        if int(lo.item()) != int(hi.item()):
            raise SystemExit(f"rank {rank}: replicated latent differs across ranks after the run")

    # ---- K9 alone: back-to-back exchanges of the first timed step's full slots (NVLink GB/s) ----
    xbench = None
    if world > 1 and M == 1:
        barrier()
        xms, xbytes = eng.exchange_bench(step_index(first), args.exchange_iters)
        xbench = {"iters": args.exchange_iters, "ms": xms, "bytes_received": xbytes,
                  "GBps": xbytes / xms / 1e6 if xms else None}

    # ---- per-kernel roofline pass: one rotation cycle with the shard streams serialised, so
    # each kernel's CUDA-event duration is its own (in the timed region two shards' DiT
    # forwards overlap on two streams and per-kernel durations would overlap) ----
    nl = (C.c_uint64 * 6)()
    kms, kfl, kby = (C.c_double * 6)(), (C.c_double * 6)(), (C.c_double * 6)()
    ncyc = len(cfg.axes())
    barrier()
    L.lp_tune(b"engine_serial", 1)
    L.lp_profile_enable(1)
    pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pe0.record(stream)
    for s in range(first, first + ncyc):
        eng.run(step_index(s), 1)
    pe1.record(stream)
    eng.sync(tmo)
    L.lp_profile_enable(0)
    L.lp_tune(b"engine_serial", 0)
    prof_ms = pe0.elapsed_time(pe1)
    _lib.check(L.lp_profile_collect(nl, kms, kfl, kby))
    # ---- K1 / K10 alone (HBM roofline): back-to-back replays per axis of the cycle ----
    hb = {}
    for s in range(first, first + ncyc):
        ax = "THW"[cfg.axis_of(step_index(s))]
        if ax not in hb:
            hb[ax] = eng.hbm_bench(step_index(s), args.hbm_iters, args.hbm_sets)

    # ---- per-rank report ----
    owned = {}
    for a in sorted(set(cfg.axes())):
        p, owner = cfg.layout(cfg.axes().index(a) + 1, world)
        owned["THW"[a]] = [k + 1 for k in range(p.workers) if owner[k] == rank]
    mine = {"rank": rank, "owned_entries": owned, "ms_timed": my_ms, "exchange": exchange,
            "bytes_received_timed": (c1["nccl_bytes_received"] - c0["nccl_bytes_received"]),
            "exchange_bench": xbench, "launches_timed": launches,
            "exchange_in_step": {"ms": kms[3], "launches": int(nl[3]), "bytes": kby[3],
                                 "note": "push+flag+wait inside the serialised profiling cycle: includes peer skew"}}
    ranks = [mine]
    if world > 1:
        ranks = [None] * world
        dist.all_gather_object(ranks, mine)
    if rank != 0:
        eng.close()
        return
    names = ["self_attention", "cross_attention", "gemm"]
    kern = {names[i]: {"launches": int(nl[i]), "ms": kms[i], "tflops": (kfl[i] / kms[i] / 1e9) if kms[i] else None,
                       "share_of_step": kms[i] / prof_ms if prof_ms else None} for i in range(3)}
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peaks_hbm = peaks.get("hbm_gbs") or 7700.0
    hbm = {}
    for i, nm, key in ((4, "k1_gather", "k1"), (5, "k10_reconstruct_update", "k10")):
        per_axis = {}
        for ax, r in hb.items():
            gbps = r[key + "_bytes"] / r[key + "_ms"] / 1e6 if r[key + "_ms"] else None
            per_axis[ax] = {"us_per_launch": 1000.0 * r[key + "_ms"], "algorithmic_bytes": r[key + "_bytes"],
                            "GBps": gbps, "frac_of_hbm": gbps / peaks_hbm if gbps else None}
        tb = sum(r[key + "_bytes"] for r in hb.values())
        tm = sum(r[key + "_ms"] for r in hb.values())
        hbm[nm] = {"per_axis": per_axis, "GBps": tb / tm / 1e6 if tm else None,
                   "frac_of_hbm": tb / tm / 1e6 / peaks_hbm if tm else None,
                   "share_of_step": kms[i] / prof_ms if prof_ms else None,
                   "in_step_event_timed": {"launches": int(nl[i]), "ms": kms[i], "algorithmic_bytes": kby[i]}}
    hbm["timing"] = (f"per axis: {args.hbm_iters} back-to-back launches over {args.hbm_sets} private buffer copies "
                     f"used round robin (working set > L2, so launches stream from HBM), CUDA events around the "
                     f"whole run on the launching stream; share_of_step from the serialised profiling cycle")
    hbm["peak_GBps"] = peaks_hbm
    hbm["peak_source"] = "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)" if peaks.get("hbm_gbs") else "fallback 7700"
    ag = None
    if world > 1 and xbench:
        ag = {"exchange": exchange, "bench_GBps_per_rank": [r["exchange_bench"]["GBps"] for r in ranks],
              "nvlink_peak_GBps_per_direction": 900.0,
              "frac": min(r["exchange_bench"]["GBps"] for r in ranks) / 900.0,
              "bytes_received_per_rank_per_step": ranks[0]["exchange_bench"]["bytes_received"] / args.exchange_iters,
              "in_step_launches": int(nl[3])}
    dom = max(range(3), key=lambda i: kms[i])
    peak = peaks.get("bf16_tflops_sustained") or 1400.0
    achieved = kfl[dom] / kms[dom] / 1e9 if kms[dom] else None
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        traffic = prof.get(names[dom], {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    sm = scaling_model(cfg, world)
    # whole-step algorithmic FLOPs per rank (the max-loaded rank sets the step), CFG batch 2
    step_flops = sm["max_rank_tflop_per_step_mean"] * 1e12
    step_tflops = step_flops / (ms / args.steps / 1000.0) / 1e12
    # communication per video (50 steps): measured exchange bytes, exact all-gather layout, reference ledger, NMP
    per_step_x = sum(r["bytes_received_timed"] for r in ranks) / args.steps
    led = ag_video = 0
    for i in range(1, T_SCHED + 1):
        a, b = lp.step_comm_bytes(cfg.plan(i), dims, 2, world // M, 4)
        led += a
        ag_video += b
    tokens = cfg.tokens(dims)
    nmp = 2 * T_SCHED * (K - 1) * tokens * cfg.d * 2
    value = args.steps / (ms / 1000.0)
    line = {
        "metric": cfg.metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic (synthetic_inputs seed 2025; random-init weights, pinned generator)",
        "config": cfg.workload(world),
        "e2e": {"value": args.steps / (e2e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": zin.numel() * 4,
                "d2h_bytes_per_step": zout.numel() * 4},
        "gpu_launches": launches,
        "roofline": {"bound": "tensor", "kernel": names[dom], "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if achieved else None, "traffic": traffic,
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (kernel timed inside a long step)",
                     "timing": "CUDA events around every launch on its stream, over one schedule cycle "
                               "run right after the timed region with the shard streams serialised",
                     "step": {"algorithmic_tflop_per_step_max_rank": step_flops / 1e12, "achieved": step_tflops,
                              "frac": step_tflops / peak}},
        "kernels": kern,
        "hbm_kernels": hbm,
        "allgather": ag,
        "clocks": clk.summary(),
        "exchange": exchange,
        "ranks": ranks,
        "scaling_model": sm,
        "comm": {"exchange_bytes_per_step_measured_all_ranks": per_step_x,
                 "allgather_bytes_per_video": ag_video, "reference_ledger_bytes_per_video": led,
                 "reference_nmp_bytes_per_video": nmp, "wire": "f32 eps shards (ledger counts the 2-B preset width)"},
    }
    if M > 1:
        hy = eng.hybrid()
        cr = lp.cost_report(T_SCHED, world, cfg.r, dims, PATCH, preset="custom", hidden_dim=dit.cfg.dim,
                            wire_bytes=4, hybrid=(world // M, [M] * (world // M)))
        line["hybrid"] = {"group_size": M, "groups": world // M, "rank0_layers": [hy["layer_begin"], hy["layer_end"]],
                          "reference_cost_hybrid_intra_bytes_per_video_fp32": cr["hybrid"]["C_intra_total"],
                          "reference_cost_hybrid_bound": cr["hybrid"]["bound"]}
    if world == 1 and not args.no_cpu_baseline:
        from oracle.oracle import reference_available

        threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
        v_lp, info = cpu_reference_run(cfg, args.cpu_steps, threads)
        line["cpu_baseline_lp_machinery_only"] = {"value": v_lp, "unit": UNIT, "cores": info["cores"],
                                                  "kind": info["kind"], "sample": info["sample"]}
        if reference_available():
            v, sample = reference_sample(cfg, threads)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample}
        else:
            line["cpu_baseline"] = dict(line["cpu_baseline_lp_machinery_only"])
    print(json.dumps(line), flush=True)
    eng.close()


# ---------------------------------------------------------------------------
# launch
# ---------------------------------------------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args):
    """--gpus N without a torchrun environment: start N ranks with torchrun ourselves (one
    process per GPU, rendezvous on 127.0.0.1).  Fails loudly when N GPUs are not visible."""
    n = args.gpus
    if not args.plan_only and not GLOO_TEST and not (args.impl == "reference"):
        import torch

        have = torch.cuda.device_count()
        if have < n:
            raise SystemExit(f"bench.py --gpus {n}: only {have} CUDA device(s) visible; refusing to report fewer ranks")
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # the communicator's nranks shows in the log
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    r = subprocess.run(cmd, env=env)
    if r.returncode:
        raise SystemExit(f"bench.py --gpus {n}: a rank failed (torchrun exit {r.returncode})")


def run_guarded(args):
    """N = 1: run the measurement in a child process (same arguments) and retry it once if it
    stalls or fails, printing the child's JSON line.  Two stalls were seen in ~60 runs of this
    round's A/B loops (both in runs of the default kernels, neither reproduced in 36 watched
    runs, profiles/r4r); a stalled CUDA context cannot be recovered in-process, so the guard
    restarts the whole measurement.  A retried line carries "attempts": 2."""
    import signal

    budget = args.attempt_timeout or (600 if args.config == "c2" else 3000)
    # the engine library is mapped into this process too (no CUDA call here: the child measures)
    from paper_2512_07350_b200 import _lib

    _lib.lib()
    env = dict(os.environ, LP_BENCH_CHILD="1")
    for attempt in (1, 2):
        p = subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]], stdout=subprocess.PIPE,
                             env=env, start_new_session=True)
        try:
            out, _ = p.communicate(timeout=budget)
        except subprocess.TimeoutExpired:
            os.killpg(p.pid, signal.SIGKILL)
            p.wait()
            print(f"bench.py: attempt {attempt} stalled ({budget} s)", file=sys.stderr, flush=True)
            continue
        lines = [x for x in out.decode().splitlines() if x.strip()]
        if p.returncode == 0 and lines:
            line = json.loads(lines[-1])
            if attempt > 1:
                line["attempts"] = attempt
            print(json.dumps(line), flush=True)
            return
        print(f"bench.py: attempt {attempt} failed (exit {p.returncode})", file=sys.stderr, flush=True)
    raise SystemExit("bench.py: the measurement failed twice")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS), help="BASELINE config (default c2 = configs[1])")
    ap.add_argument("--workers", type=int, default=0, help="LP workers K (default max(4, N); C4/C5: 8)")
    ap.add_argument("--layers", type=int, default=0, help="DiT blocks (default: the config's)")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="N > 1: eps exchange over NVLink peer memory fused into the DiT epilogue (default), or NCCL")
    ap.add_argument("--assign", default="round-robin", choices=["round-robin", "balanced"],
                    help="entry -> rank assignment (balanced: longest-processing-time on DiT FLOPs)")
    ap.add_argument("--hybrid", type=int, default=1,
                    help="M > 1: hybrid LP x model parallelism, N/M LP groups of M pipeline stages (K = N/M)")
    ap.add_argument("--overlap", type=float, default=None,
                    help="LP overlap ratio r (BASELINE configs[2] sweep; default 0.5 = configs[1])")
    ap.add_argument("--cpu-steps", type=int, default=24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-steps", type=int, default=0, help="reference arm: whole LP steps to time (default 1: step 1, the T axis, ~210 s on 16 cores; 3 = one T/H/W cycle)")
    ap.add_argument("--exchange-iters", type=int, default=20)
    ap.add_argument("--hbm-iters", type=int, default=64, help="K1/K10 replays per axis for the HBM roofline")
    ap.add_argument("--hbm-sets", type=int, default=8, help="buffer copies the K1/K10 replays cycle through")
    ap.add_argument("--sync-timeout", type=float, default=600.0, help="seconds before a stalled step is a WorkerFailure")
    ap.add_argument("--plan-only", action="store_true", help="print the N-rank assignment and FLOP-ideal bound (no GPU)")
    ap.add_argument("--attempt-timeout", type=float, default=0.0,
                    help="N = 1: seconds before a stalled measurement is restarted (default 600 for c2, 3000 otherwise)")
    args = ap.parse_args()
    if ("WORLD_SIZE" not in os.environ and args.gpus == 1 and args.impl == "ours" and not args.plan_only
            and not os.environ.get("LP_BENCH_CHILD")):
        run_guarded(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        self_launch(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} launched with WORLD_SIZE={world}")
    local_rank = 0 if GLOO_TEST else int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch.distributed as dist

        if args.plan_only or GLOO_TEST:  # CPU plumbing / validation of the multi-rank bench on ONE GPU
            dist.init_process_group("gloo")
        else:
            import torch

            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.plan_only:
        run_plan_only(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
