"""Python face of the B200 LP engine — mirrors the reference's python module
(``lpsim``, proj/python/lpsim_bindings.cpp:119-289) and its C++ API
(include/lpsim/{partition,reconstruct,denoise,cluster}.hpp) so that the
parity tests read like the reference's own tests.

Tensors live on the GPU (torch CUDA tensors holding the storage dtype's exact
bits: 2 -> float16, 4 -> float32, 8 -> float64); every operation is a kernel in
liblp_b200.so called through the C-ABI.  There is no CPU path: without a GPU the
device entry points raise.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import LpError, check, i64arr, lib

__all__ = [
    "Axis", "LpError", "LatentTensor", "PartitionPlan", "rotation_axis", "build_plan", "build_axis_plan",
    "weight_profile", "synthetic_latent", "extract_sublatents", "BoxDenoiser", "GlobalMixDenoiser",
    "IdentityDenoiser", "DiTDenoiser", "cfg_predict", "sampler_step", "reconstruct", "reconstruct_update",
    "run_lp", "run_centralized", "LpEngine", "quantize", "f16_encode", "step_comm_bytes", "shard_layout",
    "PRESETS", "presets", "verify_n_complete", "save_latent", "load_latent", "cli",
]

# ModelPreset (src/latent.cpp:197-205): wire width used by the comm ledger.
PRESETS = {"wan21-like": {"hidden_dim": 1536, "dtype_bytes": 2}, "fp32-small": {"hidden_dim": 256, "dtype_bytes": 4}}


class Axis(enum.IntEnum):
    temporal = 0
    height = 1
    width = 2


_TORCH_DT = {2: "float16", 4: "float32", 8: "float64"}


def _torch():
    import torch

    return torch


def _stream():
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def quantize(v: float, dtype_bytes: int) -> float:
    return lib().lp_quantize(float(v), int(dtype_bytes))


def f16_encode(v: float) -> int:
    return lib().lp_f16_encode(float(v))


def _quantize_np(a: np.ndarray, dtype_bytes: int) -> np.ndarray:
    """quantize() of src/dtype.cpp:102-116 over an array (host)."""
    a = np.asarray(a, np.float64)
    if dtype_bytes == 8:
        return a.copy()
    if dtype_bytes == 4:
        lim = float(np.finfo(np.float32).max)
        return np.clip(a, -lim, lim).astype(np.float32)
    if dtype_bytes == 2:
        return np.clip(a, -65504.0, 65504.0).astype(np.float16)
    raise LpError(10, f"dtype_bytes must be 2, 4 or 8, got {dtype_bytes}")


# --------------------------------------------------------------------------
# Tensors
# --------------------------------------------------------------------------
class LatentTensor:
    """Dense (c, t, h, w) latent on the GPU — LatentTensor (include/lpsim/latent.hpp:72-110)."""

    def __init__(self, data, dtype_bytes: int):
        self.data = data  # torch tensor, cuda, storage dtype
        self.dtype_bytes = int(dtype_bytes)

    @staticmethod
    def from_numpy(arr, dtype_bytes: int = 4, device="cuda"):
        torch = _torch()
        arr = np.asarray(arr, np.float64)
        if arr.ndim != 4:
            raise ValueError("expected a 4-d array (C, T, H, W)")
        q = _quantize_np(arr, dtype_bytes)
        if not np.all(np.isfinite(q)):
            raise LpError(11, "tensor element is not finite")
        return LatentTensor(torch.from_numpy(np.ascontiguousarray(q)).to(device), dtype_bytes)

    @staticmethod
    def empty(shape, dtype_bytes: int, device="cuda"):
        torch = _torch()
        return LatentTensor(torch.empty(tuple(shape), dtype=getattr(torch, _TORCH_DT[dtype_bytes]), device=device),
                            dtype_bytes)

    def to_numpy(self) -> np.ndarray:
        return self.data.detach().cpu().numpy().astype(np.float64)

    @property
    def shape(self):
        return tuple(int(s) for s in self.data.shape)

    def ptr(self):
        return C.c_void_p(self.data.data_ptr())

    def size(self) -> int:
        return int(self.data.numel())


def synthetic_latent(dims, dtype_bytes: int, seed: int, device="cuda"):
    """synthetic_inputs (src/run_config.cpp:258-301): (latent, cond values)."""
    n = int(np.prod(dims))
    z = np.zeros(n, np.float64)
    cond = np.zeros(8, np.float64)
    check(lib().lp_synthetic_inputs(i64arr(dims), dtype_bytes, seed, z.ctypes.data_as(_lib._f64p),
                                    cond.ctypes.data_as(_lib._f64p)))
    return LatentTensor.from_numpy(z.reshape(dims), dtype_bytes, device), list(cond)


def synthetic_latent_host(dims, dtype_bytes: int, seed: int):
    """Host-only variant (no GPU needed): numpy latent + cond list."""
    n = int(np.prod(dims))
    z = np.zeros(n, np.float64)
    cond = np.zeros(8, np.float64)
    check(lib().lp_synthetic_inputs(i64arr(dims), dtype_bytes, seed, z.ctypes.data_as(_lib._f64p),
                                    cond.ctypes.data_as(_lib._f64p)))
    return z.reshape(dims), list(cond)


# --------------------------------------------------------------------------
# Plans
# --------------------------------------------------------------------------
class PartitionPlan:
    """PartitionPlan (include/lpsim/partition.hpp:32-46) as the lp_plan POD."""

    def __init__(self, raw: _lib.Plan):
        self.raw = raw

    @property
    def axis(self) -> str:
        return Axis(self.raw.axis).name

    @property
    def workers(self) -> int:
        return int(self.raw.n_entries)

    def entries(self):
        return [self.raw.entries[k] for k in range(self.raw.n_entries)]

    def latent(self, k):
        e = self.raw.entries[k]
        return int(e.latent_begin), int(e.latent_end)

    def to_dict(self):
        p = self.raw
        return {
            "axis": self.axis, "step": p.step_index, "L": p.patches_per_core, "O": p.overlap_patches,
            "N": p.axis_patches, "D": p.axis_extent, "p": p.patch_size,
            "entries": [{"k": e.worker_id, "core": (e.core_begin, e.core_end), "ext": (e.ext_begin, e.ext_end),
                         "latent": (e.latent_begin, e.latent_end), "delta": (e.delta_start, e.delta_end)}
                        for e in self.entries()],
        }

    def sub_shape(self, full_shape, k):
        s = list(full_shape)
        b, e = self.latent(k)
        s[1 + self.raw.axis] = e - b
        return tuple(s)

    def offsets(self, full_shape):
        off = (C.c_int64 * (self.workers + 1))()
        check(lib().lp_plan_offsets(C.byref(self.raw), i64arr(full_shape), off))
        return list(off)


def rotation_axis(step_index: int) -> Axis:
    a = C.c_int32()
    check(lib().lp_rotation_axis(step_index, C.byref(a)))
    return Axis(a.value)


def build_plan(dims, patch, step, workers, overlap_ratio) -> PartitionPlan:
    p = _lib.Plan()
    check(lib().lp_build_plan(i64arr(dims), i64arr(patch), step, workers, float(overlap_ratio), C.byref(p)))
    return PartitionPlan(p)


def build_axis_plan(axis, extent, patch, step, workers, overlap_ratio) -> PartitionPlan:
    p = _lib.Plan()
    check(lib().lp_build_axis_plan(int(axis), extent, patch, step, workers, float(overlap_ratio), C.byref(p)))
    return PartitionPlan(p)


def weight_profile(plan: PartitionPlan, entry: int):
    if entry < 0 or entry >= plan.workers:
        raise IndexError("entry out of range")
    b, e = plan.latent(entry)
    out = (C.c_double * (e - b))()
    check(lib().lp_weight_profile(C.byref(plan.raw), entry, out))
    return list(out)


def shard_layout(plan: PartitionPlan, dims, world: int, rank: int):
    owned = (C.c_int32 * _lib.LP_MAX_WORKERS)()
    n = C.c_int32()
    slot = C.c_int64()
    check(lib().lp_shard_layout(C.byref(plan.raw), i64arr(dims), world, rank, owned, C.byref(n), C.byref(slot)))
    return list(owned[: n.value]), int(slot.value)


def shard_bases(plan: PartitionPlan, dims, world: int):
    """Offsets (elements) of every entry's shard in the gathered buffer."""
    out = (C.c_int64 * plan.workers)()
    check(lib().lp_shard_bases(C.byref(plan.raw), i64arr(dims), world, out))
    return list(out)


def cost_report(steps, workers, overlap_ratio, dims, patch, preset="wan21-like", hybrid=None, hidden_dim=None,
                wire_bytes=None):
    """cost_report of the reference (src/cost.cpp:215-248; python binding lpsim_bindings.cpp:234-245):
    same keys as the reference module's dict."""
    pr = PRESETS[preset] if preset in PRESETS else None
    if pr is None and (hidden_dim is None or wire_bytes is None):
        raise ValueError(f"unknown preset '{preset}'")
    hd = hidden_dim if hidden_dim is not None else pr["hidden_dim"]
    wb = wire_bytes if wire_bytes is not None else pr["dtype_bytes"]
    groups, sizes = (0, []) if hybrid is None else (int(hybrid[0]), list(hybrid[1]))
    arr = (C.c_int32 * max(1, len(sizes)))(*sizes) if sizes else (C.c_int32 * 1)()
    r = _lib.CostReport()
    check(lib().lp_cost_report(steps, workers, float(overlap_ratio), i64arr(dims), i64arr(patch), hd, wb, groups, arr,
                               C.byref(r)))
    d = {"S_z": r.latent_bytes, "S_H": r.activation_bytes, "gamma": r.gamma, "C_NMP": r.nmp_bytes, "C_PP": r.pp_bytes,
         "C_LP_exact": r.lp_exact_bytes, "C_LP_approx": r.lp_approx_bytes, "ratio_exact": r.ratio_exact,
         "ratio_approx": r.ratio_approx, "Sz_over_SH": r.latent_activation_ratio,
         "gamma_per_axis": tuple(r.gamma_per_axis)}
    if r.has_hybrid:
        d["hybrid"] = {"C_inter": r.hybrid_inter_bytes, "C_intra_total": r.hybrid_intra_bytes,
                       "C_hyb": r.hybrid_total_bytes, "ratio_vs_NMP": r.hybrid_ratio_vs_nmp, "bound": r.hybrid_bound,
                       "within_bound": bool(r.hybrid_within_bound)}
    return d


def shard_layout_ex(plan: PartitionPlan, dims, world: int, rank: int, policy="round-robin", lin=1.0, quad=0.0):
    """lp_shard_layout_ex: (owned entries, slot_elems, owner per entry, base per entry)."""
    n = plan.workers
    owned = (C.c_int32 * _lib.LP_MAX_WORKERS)()
    cnt, slot = C.c_int32(), C.c_int64()
    owner, base = (C.c_int32 * n)(), (C.c_int64 * n)()
    check(lib().lp_shard_layout_ex(C.byref(plan.raw), i64arr(dims), world, rank,
                                   {"round-robin": 0, "balanced": 1}[policy], float(lin), float(quad), owned,
                                   C.byref(cnt), C.byref(slot), owner, base))
    return list(owned[:cnt.value]), slot.value, list(owner), list(base)


def step_comm_bytes(plan: PartitionPlan, dims, wire_bytes: int, world: int, dtype_bytes: int):
    a, b = C.c_uint64(), C.c_uint64()
    check(lib().lp_step_comm_bytes(C.byref(plan.raw), i64arr(dims), wire_bytes, world, dtype_bytes, C.byref(a),
                                   C.byref(b)))
    return int(a.value), int(b.value)


# --------------------------------------------------------------------------
# Stages
# --------------------------------------------------------------------------
def extract_sublatents(z: LatentTensor, plan: PartitionPlan):
    """extract_sublatents (src/partition.cpp:136-148) — K1 gather, one launch per entry."""
    outs = []
    for k in range(plan.workers):
        sub = LatentTensor.empty(plan.sub_shape(z.shape, k), z.dtype_bytes)
        check(lib().lp_extract(C.byref(plan.raw), k, 1, z.ptr(), i64arr(z.shape), z.dtype_bytes, sub.ptr(), _stream()))
        outs.append(sub)
    return outs


@dataclass
class BoxDenoiser:
    """make_box_denoiser (include/lpsim/denoise.hpp:54-56)."""

    radius: tuple = (1, 1, 1)
    t_coeff: float = 0.01
    cond_coeff: float = 0.1
    kind: int = field(default=0, init=False)

    def receptive_radius(self):
        return tuple(self.radius)


@dataclass
class GlobalMixDenoiser:
    t_coeff: float = 0.01
    cond_coeff: float = 0.1
    kind: int = field(default=1, init=False)
    radius: tuple = field(default=(0, 0, 0), init=False)

    def receptive_radius(self):
        return None


@dataclass
class IdentityDenoiser:
    kind: int = field(default=2, init=False)
    radius: tuple = field(default=(0, 0, 0), init=False)
    t_coeff: float = 0.0
    cond_coeff: float = 0.0

    def receptive_radius(self):
        return (0, 0, 0)


def _mean(cond):
    return sum(0.0 + v for v in cond) / len(cond) if len(cond) else 0.0


def _toy_ws(z: LatentTensor):
    torch = _torch()
    return torch.empty(int(lib().lp_toy_workspace_bytes(i64arr(z.shape))) // 8 + 8, dtype=torch.float64,
                       device=z.data.device)


def denoiser_predict(f, z: LatentTensor, timestep: int, cond, is_null=False) -> LatentTensor:
    """Denoiser::predict (include/lpsim/denoise.hpp:36) for the toy denoisers."""
    out = LatentTensor.empty(z.shape, z.dtype_bytes)
    mean = 0.0 if is_null else _mean(cond)
    check(lib().lp_toy_predict(f.kind, i64arr(f.radius), f.t_coeff, f.cond_coeff, z.ptr(), i64arr(z.shape),
                               z.dtype_bytes, timestep, mean, out.ptr(), _stream()))
    return out


def cfg_predict(f, z: LatentTensor, timestep: int, cond, guidance_scale: float) -> LatentTensor:
    """cfg_predict (src/denoise.cpp:24-39): uncond + w (cond - uncond), quantized."""
    if cond is None:
        raise LpError(10, "cfg_predict requires a non-null conditioning vector")
    out = LatentTensor.empty(z.shape, z.dtype_bytes)
    if isinstance(f, DiTDenoiser):
        return f.cfg_predict(z, timestep, guidance_scale)
    ws = _toy_ws(z)
    check(lib().lp_toy_cfg_predict(f.kind, i64arr(f.radius), f.t_coeff, f.cond_coeff, z.ptr(), i64arr(z.shape),
                                   z.dtype_bytes, timestep, _mean(cond), float(guidance_scale), out.ptr(),
                                   C.c_void_p(ws.data_ptr()), _stream()))
    return out


def sampler_step(z: LatentTensor, eps: LatentTensor, timestep: int, eta: float) -> LatentTensor:
    """sampler_step (src/denoise.cpp:41-52)."""
    if z.shape != eps.shape or z.dtype_bytes != eps.dtype_bytes:
        raise LpError(7, f"sampler_step: latent {z.shape} vs prediction {eps.shape}")
    out = LatentTensor.empty(z.shape, z.dtype_bytes)
    check(lib().lp_sampler_step(z.ptr(), eps.ptr(), z.size(), z.dtype_bytes, float(eta), out.ptr(), _stream()))
    return out


def _pack(preds, plan: PartitionPlan, full_dims):
    torch = _torch()
    if len(preds) != plan.workers:
        raise LpError(7, f"got {len(preds)} predictions for {plan.workers} partitions")
    d = preds[0].dtype_bytes
    for k, p in enumerate(preds):
        if p.shape != plan.sub_shape(full_dims, k) or p.dtype_bytes != d:
            raise LpError(7, f"prediction {k + 1} has shape {p.shape}, expected {plan.sub_shape(full_dims, k)}")
    return torch.cat([p.data.reshape(-1) for p in preds]), d


def reconstruct(predictions, plan: PartitionPlan, full_dims, mode: str = "exact") -> LatentTensor:
    """reconstruct (src/reconstruct.cpp:42-121) on the GPU (K10 without the update)."""
    packed, d = _pack(predictions, plan, tuple(full_dims))
    out = LatentTensor.empty(tuple(full_dims), d)
    check(lib().lp_reconstruct(C.byref(plan.raw), C.c_void_p(packed.data_ptr()), i64arr(full_dims), d,
                               0 if mode == "exact" else 1, out.ptr(), _stream()))
    return out


def reconstruct_update(predictions, plan: PartitionPlan, z: LatentTensor, eta: float, mode: str = "exact"):
    """K10: z <- sampler_step(z, reconstruct(predictions)) in one pass (in place)."""
    packed, d = _pack(predictions, plan, z.shape)
    check(lib().lp_reconstruct_update(C.byref(plan.raw), C.c_void_p(packed.data_ptr()), i64arr(z.shape), d,
                                      0 if mode == "exact" else 1, float(eta), z.ptr(), _stream()))
    return z


def device_flags(reset=True) -> int:
    f = C.c_uint32()
    check(lib().lp_device_flags(C.byref(f), int(reset)))
    return int(f.value)


# --------------------------------------------------------------------------
# DiT denoiser
# --------------------------------------------------------------------------
class DiTDenoiser:
    """WAN2.1-shaped DiT behind the Denoiser plugin slot (include/lpsim/denoise.hpp:31-39)."""

    def __init__(self, cond, **overrides):
        cfg = _lib.DitConfig()
        lib().lp_dit_default_config(C.byref(cfg))
        for k, v in overrides.items():
            if k == "patch":
                for i in range(3):
                    cfg.patch[i] = int(v[i])
            else:
                setattr(cfg, k, v)
        self.cfg = cfg
        c = (C.c_double * len(cond))(*cond)
        h = C.c_void_p()
        check(lib().lp_dit_create(C.byref(cfg), c, len(cond), C.byref(h)))
        self.handle = h
        self.reserved = 0

    def reserve(self, tokens):
        if tokens > self.reserved:
            check(lib().lp_dit_reserve(self.handle, int(tokens)))
            self.reserved = tokens

    def tokens(self, shape):
        p = self.cfg.patch
        return -(-shape[1] // p[0]) * -(-shape[2] // p[1]) * -(-shape[3] // p[2])

    def cfg_predict(self, z: LatentTensor, timestep: int, guidance: float) -> LatentTensor:
        self.reserve(self.tokens(z.shape))
        out = LatentTensor.empty(z.shape, z.dtype_bytes)
        check(lib().lp_dit_cfg_predict(self.handle, z.ptr(), i64arr(z.shape), z.dtype_bytes, int(timestep),
                                       float(guidance), out.ptr(), _stream()))
        return out

    def predict(self, z: LatentTensor, timestep: int, null_text: bool = False) -> LatentTensor:
        """Denoiser::predict: ONE CFG pass (null text = the uncond pass), quantized to z's dtype."""
        self.reserve(self.tokens(z.shape))
        out = LatentTensor.empty(z.shape, z.dtype_bytes)
        check(lib().lp_dit_predict(self.handle, z.ptr(), i64arr(z.shape), z.dtype_bytes, int(timestep),
                                   1 if null_text else 0, out.ptr(), _stream()))
        return out

    def params(self):
        torch = _torch()
        out = {}
        for i in range(lib().lp_dit_num_params(self.handle)):
            name, ptr, n, eb = C.c_char_p(), C.c_void_p(), C.c_int64(), C.c_int32()
            check(lib().lp_dit_param(self.handle, i, C.byref(name), C.byref(ptr), C.byref(n), C.byref(eb)))
            out[name.value.decode()] = _wrap_device(ptr.value, n.value, torch.bfloat16 if eb.value == 2 else torch.float32)
        return out

    def debug_tensor(self, name, dtype):
        ptr, n = C.c_void_p(), C.c_int64()
        check(lib().lp_dit_debug_tensor(self.handle, name.encode(), C.byref(ptr), C.byref(n)))
        return _wrap_device(ptr.value, n.value, dtype)

    def receptive_radius(self):
        return None

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                lib().lp_dit_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def _wrap_device(ptr, numel, dtype):
    """Non-owning torch view of a device buffer owned by the library."""
    torch = _torch()
    typestr = {torch.bfloat16: "<i2", torch.float32: "<f4", torch.float16: "<f2", torch.float64: "<f8"}[dtype]

    class _H:
        __cuda_array_interface__ = {"shape": (int(numel),), "typestr": typestr, "data": (int(ptr), False),
                                    "version": 2}

    t = torch.as_tensor(_H(), device="cuda")
    return t.view(torch.bfloat16) if dtype == torch.bfloat16 else t


# --------------------------------------------------------------------------
# The loop
# --------------------------------------------------------------------------
class LpEngine:
    """The run_lp step loop (src/cluster.cpp:166-225) as one engine per rank.

    world/rank select this rank's round-robin share of the K entries; for
    world > 1 pass the NCCL unique id rank 0 obtained from ``nccl_unique_id()``.
    """

    def __init__(self, dims, patch, dtype_bytes, workers, overlap_ratio, steps, eta, guidance, cond,
                 denoiser="box", radius=(1, 1, 1), wire_bytes=2, world=1, rank=0, nccl_id=None, mode="exact",
                 dit: DiTDenoiser | None = None, t_coeff=0.01, cond_coeff=0.1, schedule=None, group_size=1,
                 assign="round-robin"):
        cfg = _lib.EngineConfig()
        for i in range(4):
            cfg.shape[i] = int(dims[i])
        for i in range(3):
            cfg.patch[i] = int(patch[i])
            cfg.radius[i] = int(radius[i])
        cfg.dtype_bytes = dtype_bytes
        cfg.workers = workers
        cfg.overlap_ratio = float(overlap_ratio)
        cfg.total_steps = steps
        cfg.mode = 0 if mode == "exact" else 1
        cfg.eta = float(eta)
        cfg.guidance = float(guidance)
        kinds = {"box": 0, "global": 1, "identity": 2, "dit": -1}
        cfg.denoiser = kinds[denoiser]
        cfg.wire_bytes = wire_bytes
        if denoiser != "box":
            t_coeff, cond_coeff = (0.01, 0.1) if denoiser == "global" else (t_coeff, cond_coeff)
        cfg.t_coeff = t_coeff
        cfg.cond_coeff = cond_coeff
        cfg.world = world
        cfg.rank = rank
        cfg.dit = dit.handle if dit is not None else None
        cfg.group_size = int(group_size)
        cfg.assign = {"round-robin": 0, "balanced": 1}[assign]
        if schedule:
            axes = parse_schedule(schedule)
            cfg.schedule_len = len(axes)
            for i, a in enumerate(axes):
                cfg.schedule[i] = a
        self.dit = dit
        self.world = int(world)
        self.group_size = max(1, int(group_size))
        self.groups = self.world // self.group_size
        self.dims = tuple(int(d) for d in dims)
        self.dtype_bytes = dtype_bytes
        c = (C.c_double * len(cond))(*cond)
        idp = None
        if nccl_id is not None:
            idp = (C.c_uint8 * 128)(*nccl_id)
        h = C.c_void_p()
        check(lib().lp_engine_create(C.byref(cfg), idp, c, len(cond), C.byref(h)))
        self.handle = h
        zp = C.c_void_p()
        check(lib().lp_engine_latent(h, C.byref(zp)))
        torch = _torch()
        self.z = LatentTensor(_wrap_latent(zp.value, self.dims, dtype_bytes), dtype_bytes)

    def load(self, z: LatentTensor):
        self.z.data.copy_(z.data)

    def run(self, first_step, count, stream=None):
        st = C.c_void_p(stream) if stream is not None else _stream()
        check(lib().lp_engine_run(self.handle, first_step, count, st))

    def sync(self, timeout_s=0.0, stream=None):
        """lp_engine_sync: wait for the enqueued steps; a dead/stalled peer or an NCCL async
        error raises LpError(WorkerFailure) naming the step (and the worker, for the peer path)."""
        st = C.c_void_p(stream) if stream is not None else _stream()
        check(lib().lp_engine_sync(self.handle, st, int(timeout_s * 1000)))

    def exchange_bench(self, step, iters, stream=None):
        """lp_engine_exchange_bench: (ms, bytes received by this rank) of `iters` K9 exchanges."""
        st = C.c_void_p(stream) if stream is not None else _stream()
        ms, nb = C.c_double(), C.c_uint64()
        check(lib().lp_engine_exchange_bench(self.handle, int(step), int(iters), st, C.byref(ms), C.byref(nb)))
        return ms.value, int(nb.value)

    def hbm_bench(self, step, iters=50, sets=8, stream=None):
        """lp_engine_hbm_bench: K1 / K10 of `step` replayed back to back over `sets` buffer copies.
        Returns {"k1_ms", "k1_bytes", "k10_ms", "k10_bytes"} per launch."""
        st = C.c_void_p(stream) if stream is not None else _stream()
        out = (C.c_double * 4)()
        check(lib().lp_engine_hbm_bench(self.handle, int(step), int(iters), int(sets), st, out))
        return {"k1_ms": out[0], "k1_bytes": out[1], "k10_ms": out[2], "k10_bytes": out[3]}

    def step_phase(self, step, phase, stream=None):
        """lp_engine_step_phase: 1 = compute this rank's shards, 2 = NCCL exchange, 3 = reconstruct."""
        st = C.c_void_p(stream) if stream is not None else _stream()
        check(lib().lp_engine_step_phase(self.handle, int(step), int(phase), st))

    def gather_buffer(self, step):
        """(torch view of the gather buffer [world * slot_elems], slot_elems) for step's layout."""
        ptr, slot = C.c_void_p(), C.c_int64()
        check(lib().lp_engine_gather_buffer(self.handle, int(step), C.byref(ptr), C.byref(slot)))
        torch = _torch()
        dt = getattr(torch, _TORCH_DT[self.dtype_bytes])
        return _wrap_device(ptr.value, self.groups * slot.value, dt), slot.value

    # --- K9 over NVLink peer memory (CUDA IPC) instead of NCCL ---
    def ipc_handle(self) -> bytes:
        h = (C.c_uint8 * 64)()
        check(lib().lp_engine_ipc_handle(self.handle, h))
        return bytes(h)

    def ipc_attach(self, handles):
        """handles: the world ranks' ipc_handle() bytes, by rank."""
        buf = (C.c_uint8 * (64 * len(handles)))(*b"".join(handles))
        check(lib().lp_engine_ipc_attach(self.handle, buf))

    def ipc_detach(self):
        check(lib().lp_engine_ipc_detach(self.handle))

    # --- hybrid LP x model-parallel groups (group_size > 1), SURVEY.md §8 f2 ---
    def owned(self, step):
        n = C.c_int32()
        check(lib().lp_engine_owned(self.handle, int(step), C.byref(n)))
        return int(n.value)

    def stage(self, step, idx, stream=None):
        """This rank's pipeline stage for the idx-th entry its group owns (no-NCCL driving)."""
        st = C.c_void_p(stream) if stream is not None else _stream()
        check(lib().lp_engine_stage(self.handle, int(step), int(idx), st))

    def stage_activation(self, step, idx):
        """torch float32 view of the activation handed between stages for that entry."""
        ptr, nb = C.c_void_p(), C.c_int64()
        check(lib().lp_engine_stage_activation(self.handle, int(step), int(idx), C.byref(ptr), C.byref(nb)))
        return _wrap_device(ptr.value, nb.value // 4, _torch().float32)

    def hybrid(self):
        v = [C.c_int32() for _ in range(5)]
        intra = C.c_uint64()
        check(lib().lp_engine_hybrid(self.handle, *[C.byref(x) for x in v], C.byref(intra)))
        keys = ("group_size", "group", "stage", "layer_begin", "layer_end")
        out = {k: int(x.value) for k, x in zip(keys, v)}
        out["intra_bytes_sent"] = int(intra.value)
        return out

    def comm(self):
        a, b = C.c_uint64(), C.c_uint64()
        check(lib().lp_engine_comm(self.handle, C.byref(a), C.byref(b)))
        return {"nccl_bytes_received": int(a.value), "ledger_bytes": int(b.value)}

    def launches(self):
        a = C.c_uint64()
        check(lib().lp_engine_launches(self.handle, C.byref(a)))
        return int(a.value)

    def close(self):
        if getattr(self, "handle", None):
            lib().lp_engine_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _wrap_latent(ptr, dims, dtype_bytes):
    torch = _torch()
    typestr = {2: "<f2", 4: "<f4", 8: "<f8"}[dtype_bytes]

    class _H:
        __cuda_array_interface__ = {"shape": tuple(dims), "typestr": typestr, "data": (int(ptr), False),
                                    "version": 2}

    return torch.as_tensor(_H(), device="cuda")


def parse_schedule(schedule):
    """'TTHTTW' / ['temporal', 'height', ...] / [0, 1, 2] -> axis ids (T=0, H=1, W=2)."""
    if isinstance(schedule, str):
        m = {"T": 0, "H": 1, "W": 2}
        axes = [m[ch] for ch in schedule.upper() if ch in m]
    else:
        axes = [Axis[a].value if isinstance(a, str) else int(a) for a in schedule]
    if not 1 <= len(axes) <= 64:
        raise LpError(10, "schedule must have 1..64 axes")
    return axes


def nccl_unique_id():
    buf = (C.c_uint8 * 128)()
    check(lib().lp_nccl_unique_id(C.byref(buf)))
    return bytes(buf)


def run_lp(denoiser, radius, z: LatentTensor, steps, eta, guidance, cond, patch, workers, overlap_ratio,
           preset="wan21-like", mode="exact", dit: DiTDenoiser | None = None, schedule=None):
    """Same signature as the reference binding's run_lp (lpsim_bindings.cpp:199-232);
    returns (final latent, ledger summary)."""
    if preset not in PRESETS:
        raise ValueError(f"unknown preset '{preset}'")
    eng = LpEngine(z.shape, patch, z.dtype_bytes, workers, overlap_ratio, steps, eta, guidance, cond,
                   denoiser=denoiser, radius=radius, wire_bytes=PRESETS[preset]["dtype_bytes"], mode=mode, dit=dit,
                   schedule=schedule)
    eng.load(z)
    eng.run(1, steps)
    out = LatentTensor(eng.z.data.clone(), z.dtype_bytes)
    comm = eng.comm()
    eng.close()
    flags = device_flags(reset=True)
    if flags & 1:
        raise LpError(11, "tensor element is not finite")
    return out, {"grand_total": comm["ledger_bytes"], "nccl_bytes_received": comm["nccl_bytes_received"]}


def run_centralized(denoiser, radius, z: LatentTensor, steps, eta, guidance, cond, dit: DiTDenoiser | None = None):
    """run_centralized (src/denoise.cpp:158-174) ≡ run_lp at K=1 (test_cluster.cpp:75-92)."""
    out, _ = run_lp(denoiser, radius, z, steps, eta, guidance, cond, (1, 1, 1), 1, 0.0, dit=dit)
    return out


# --------------------------------------------------------------------------
# Completeness, latent dumps, presets, CLI
# --------------------------------------------------------------------------
def presets():
    """builtin_presets (src/latent.cpp:197-206), as the binding's presets() (lpsim_bindings.cpp:277-289)."""
    return [{"name": k, "hidden_dim": v["hidden_dim"], "dtype_bytes": v["dtype_bytes"]} for k, v in PRESETS.items()]


def verify_n_complete(grid, workers, overlap_ratio, schedule="rotating", budget=8, max_positions=0):
    """verify_n_complete (src/completeness.cpp:104-160) with the binding's signature
    (lpsim_bindings.cpp:247-271); `schedule` may also be an explicit axis list / string
    ("TTHTTW", repeated cyclically).  Returns {complete, complete_at, worst_position, min_steps}."""
    if isinstance(schedule, str) and schedule in ("rotating", "temporal", "height", "width"):
        axes = [rotation_axis(i) for i in range(1, budget + 1)] if schedule == "rotating" else \
            [int(Axis[schedule])] * budget
    else:
        cyc = parse_schedule(schedule)
        axes = [cyc[i % len(cyc)] for i in range(budget)]
    n = int(grid[0]) * int(grid[1]) * int(grid[2])
    sched = (C.c_int32 * len(axes))(*axes)
    comp, at = C.c_int32(), C.c_int32()
    worst = (C.c_int64 * 3)()
    mins = (C.c_int32 * max(n, 1))()
    check(lib().lp_verify_n_complete(i64arr(grid), int(workers), float(overlap_ratio), sched, len(axes), int(budget),
                                     int(max_positions), C.byref(comp), C.byref(at), worst, mins))
    return {"complete": bool(comp.value), "complete_at": at.value if comp.value else None,
            "worst_position": (worst[0], worst[1], worst[2]), "min_steps": list(mins[:n])}


def save_latent(path, tensor: LatentTensor):
    """write_latent_dump (src/io.cpp:39-79): LPLT header + storage-width payload."""
    host = tensor.data.contiguous().cpu()
    check(lib().lp_latent_dump_write(str(path).encode(), C.c_void_p(host.data_ptr()), i64arr(tensor.shape),
                                     tensor.dtype_bytes))


def load_latent(path, device="cuda") -> LatentTensor:
    """read_latent_dump (src/io.cpp:81-139)."""
    torch = _torch()
    shape, db = (C.c_int64 * 4)(), C.c_int32()
    check(lib().lp_latent_dump_read(str(path).encode(), shape, C.byref(db), None, 0))
    dims = tuple(shape)
    dt = getattr(torch, _TORCH_DT[db.value])
    host = torch.empty(dims, dtype=dt)
    check(lib().lp_latent_dump_read(str(path).encode(), shape, C.byref(db), C.c_void_p(host.data_ptr()),
                                    host.numel() * db.value))
    return LatentTensor(host.to(device) if device else host, db.value)


def cli(argv):
    """The `lpsim` command line on this engine (lp_cli_main); returns the exit code."""
    args = ["lpsim_b200", *[str(a) for a in argv]]
    arr = (C.c_char_p * len(args))(*[a.encode() for a in args])
    return lib().lp_cli_main(len(args), arr)
