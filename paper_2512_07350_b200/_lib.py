"""ctypes binding of liblp_b200.so (the C-ABI declared in include/lp_b200.h).

The library is built in-tree by ``python -m paper_2512_07350_b200.build``.  There
is no fallback: importing a device entry point without the library raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "liblp_b200.so")
LP_MAX_WORKERS = 256

# lp_status -> reference ErrorKind name (include/lpsim/errors.hpp:10-24)
ERROR_KINDS = {
    1: "OutOfBounds", 2: "EmptyRange", 3: "DegenerateAxis", 4: "InvalidOverlapRatio", 5: "OutsideExtent",
    6: "ZeroWeight", 7: "ShapeMismatch", 8: "WorkerFailure", 9: "InvalidGrouping", 10: "InvalidArgument",
    11: "NonFinite", 12: "Config", 13: "Io", 100: "Cuda", 101: "Nccl",
}


class LpError(RuntimeError):
    """Mirror of lpsim::Error: carries the ErrorKind (python binding: LpsimError)."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.kind = ERROR_KINDS.get(status, f"Status{status}")
        super().__init__(f"{self.kind}: {message}")


class Entry(C.Structure):
    _fields_ = [("worker_id", C.c_int32), ("reserved", C.c_int32),
                ("core_begin", C.c_int64), ("core_end", C.c_int64),
                ("ext_begin", C.c_int64), ("ext_end", C.c_int64),
                ("latent_begin", C.c_int64), ("latent_end", C.c_int64),
                ("delta_start", C.c_int64), ("delta_end", C.c_int64)]


class Plan(C.Structure):
    _fields_ = [("axis", C.c_int32), ("step_index", C.c_int32), ("overlap_ratio", C.c_double),
                ("patches_per_core", C.c_int64), ("overlap_patches", C.c_int64), ("axis_patches", C.c_int64),
                ("axis_extent", C.c_int64), ("patch_size", C.c_int64), ("n_entries", C.c_int32),
                ("reserved", C.c_int32), ("entries", Entry * LP_MAX_WORKERS)]


class DitConfig(C.Structure):
    _fields_ = [("in_channels", C.c_int32), ("dim", C.c_int32), ("ffn_dim", C.c_int32), ("num_heads", C.c_int32),
                ("num_layers", C.c_int32), ("text_len", C.c_int32), ("text_dim", C.c_int32),
                ("freq_dim", C.c_int32), ("patch", C.c_int32 * 3), ("reserved", C.c_int32),
                ("eps", C.c_double), ("t_scale", C.c_double), ("seed", C.c_uint64)]


class EngineConfig(C.Structure):
    _fields_ = [("shape", C.c_int64 * 4), ("patch", C.c_int64 * 3), ("dtype_bytes", C.c_int32),
                ("workers", C.c_int32), ("overlap_ratio", C.c_double), ("total_steps", C.c_int32),
                ("mode", C.c_int32), ("eta", C.c_double), ("guidance", C.c_double), ("denoiser", C.c_int32),
                ("wire_bytes", C.c_int32), ("radius", C.c_int64 * 3), ("t_coeff", C.c_double),
                ("cond_coeff", C.c_double), ("world", C.c_int32), ("rank", C.c_int32), ("dit", C.c_void_p),
                ("schedule_len", C.c_int32), ("schedule", C.c_int32 * 64), ("group_size", C.c_int32),
                ("assign", C.c_int32)]


class CostReport(C.Structure):
    _fields_ = [("latent_bytes", C.c_uint64), ("activation_bytes", C.c_uint64), ("ext_bytes_mean", C.c_double),
                ("gamma", C.c_double), ("gamma_per_axis", C.c_double * 3), ("nmp_bytes", C.c_uint64),
                ("pp_bytes", C.c_uint64), ("lp_exact_bytes", C.c_uint64), ("lp_approx_bytes", C.c_double),
                ("ratio_exact", C.c_double), ("ratio_approx", C.c_double), ("latent_activation_ratio", C.c_double),
                ("has_hybrid", C.c_int32), ("hybrid_within_bound", C.c_int32), ("hybrid_inter_bytes", C.c_uint64),
                ("hybrid_intra_bytes", C.c_uint64), ("hybrid_total_bytes", C.c_uint64),
                ("hybrid_ratio_vs_nmp", C.c_double), ("hybrid_bound", C.c_double)]


_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p
_i = C.c_int
_i32 = C.c_int32
_i64 = C.c_int64
_d = C.c_double
_PlanP = C.POINTER(Plan)

_SIGS = {
    "lp_last_error": (C.c_char_p, []),
    "lp_version": (C.c_char_p, []),
    "lp_rotation_axis": (_i, [_i, C.POINTER(_i32)]),
    "lp_core_bounds": (_i, [_i64, _i, _i64p, C.POINTER(_i32)]),
    "lp_extend_overlap": (_i, [_i64p, _i32, _i64, _i64, _d, _i, _i64p]),
    "lp_build_axis_plan": (_i, [_i32, _i64, _i64, _i, _i, _d, _PlanP]),
    "lp_build_plan": (_i, [_i64p, _i64p, _i, _i, _d, _PlanP]),
    "lp_weight_profile": (_i, [_PlanP, _i32, _f64p]),
    "lp_plan_offsets": (_i, [_PlanP, _i64p, _i64p]),
    "lp_shard_layout": (_i, [_PlanP, _i64p, _i, _i, C.POINTER(_i32), C.POINTER(_i32), _i64p]),
    "lp_shard_bases": (_i, [_PlanP, _i64p, _i, _i64p]),
    "lp_shard_layout_ex": (_i, [_PlanP, _i64p, _i, _i, _i32, _d, _d, C.POINTER(_i32), C.POINTER(_i32), _i64p,
                                C.POINTER(_i32), _i64p]),
    "lp_step_comm_bytes":(_i, [_PlanP, _i64p, _i, _i, _i, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "lp_cost_report": (_i, [_i, _i, _d, _i64p, _i64p, _i64, _i, _i, C.POINTER(_i32), C.POINTER(CostReport)]),
    "lp_f16_encode": (C.c_uint16, [_d]),
    "lp_f16_decode": (_d, [C.c_uint16]),
    "lp_quantize": (_d, [_d, _i]),
    "lp_device_check": (_i, [_i]),
    "lp_device_flags": (_i, [C.POINTER(C.c_uint32), _i]),
    "lp_launch_count": (C.c_uint64, []),
    "lp_release_caches": (_i, []),
    "lp_profile_enable": (_i, [_i]),
    "lp_tune": (_i, [C.c_char_p, _i]),
    "lp_profile_collect": (_i, [C.POINTER(C.c_uint64), _f64p, _f64p, _f64p]),
    "lp_extract": (_i, [_PlanP, _i32, _i32, _vp, _i64p, _i, _vp, _vp]),
    "lp_toy_predict": (_i, [_i32, _i64p, _d, _d, _vp, _i64p, _i, _i, _d, _vp, _vp]),
    "lp_toy_cfg_predict": (_i, [_i32, _i64p, _d, _d, _vp, _i64p, _i, _i, _d, _d, _vp, _vp, _vp]),
    "lp_toy_workspace_bytes": (C.c_size_t, [_i64p]),
    "lp_cfg_combine": (_i, [_vp, _vp, _i64, _i, _d, _vp, _vp]),
    "lp_reconstruct": (_i, [_PlanP, _vp, _i64p, _i, _i32, _vp, _vp]),
    "lp_sampler_step": (_i, [_vp, _vp, _i64, _i, _d, _vp, _vp]),
    "lp_reconstruct_update": (_i, [_PlanP, _vp, _i64p, _i, _i32, _d, _vp, _vp]),
    "lp_synthetic_inputs": (_i, [_i64p, _i, C.c_uint64, _f64p, _f64p]),
    "lp_dit_default_config": (None, [C.POINTER(DitConfig)]),
    "lp_dit_create": (_i, [C.POINTER(DitConfig), _f64p, _i32, C.POINTER(_vp)]),
    "lp_dit_destroy": (_i, [_vp]),
    "lp_dit_reserve": (_i, [_vp, _i64]),
    "lp_dit_cfg_predict": (_i, [_vp, _vp, _i64p, _i, _i, _d, _vp, _vp]),
    "lp_dit_predict": (_i, [_vp, _vp, _i64p, _i, _i, _i32, _vp, _vp]),
    "lp_dit_predict_slot": (_i, [_vp, _i32, _vp, _i64p, _i, _i, _i32, _vp, _vp]),
    "lp_dit_reserve_slots": (_i, [_vp, _i64, _i32]),
    "lp_dit_cfg_predict_slot": (_i, [_vp, _i32, _vp, _i64p, _i, _i, _d, _vp, _vp]),
    "lp_dit_num_params": (_i, [_vp]),
    "lp_dit_param": (_i, [_vp, _i32, C.POINTER(C.c_char_p), C.POINTER(_vp), _i64p, C.POINTER(_i32)]),
    "lp_dit_debug_tensor": (_i, [_vp, C.c_char_p, C.POINTER(_vp), _i64p]),
    "lp_gemm_bf16": (_i, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp]),
    "lp_attention_bf16": (_i, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _d, _vp]),
    "lp_attention_set_trace": (_i, [_vp]),
    "lp_dit_set_time": (_i, [_vp, _i32, _i, _vp]),
    "lp_dit_time_on_device": (_i, [_vp, _i32]),
    "lp_engine_step_phase": (_i, [_vp, _i32, _i32, _vp]),
    "lp_engine_gather_buffer": (_i, [_vp, _i32, C.POINTER(_vp), C.POINTER(_i64)]),
    "lp_engine_stage": (_i, [_vp, _i32, _i32, _vp]),
    "lp_gemm_bf16_epi": (_i, [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _i32, _vp]),
    "lp_engine_ipc_handle": (_i, [_vp, C.POINTER(C.c_uint8)]),
    "lp_engine_ipc_attach": (_i, [_vp, C.POINTER(C.c_uint8)]),
    "lp_engine_ipc_detach": (_i, [_vp]),
    "lp_engine_stage_activation": (_i, [_vp, _i32, _i32, C.POINTER(_vp), C.POINTER(_i64)]),
    "lp_engine_owned": (_i, [_vp, _i32, C.POINTER(_i32)]),
    "lp_engine_hybrid": (_i, [_vp, C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32), C.POINTER(_i32),
                              C.POINTER(_i32), C.POINTER(C.c_uint64)]),
    "lp_dit_forward_layers": (_i, [_vp, _i32, _vp, _i64p, _i, _i, _d, _i32, _i32, _vp, _vp]),
    "lp_dit_activation": (_i, [_vp, _i32, _i64p, C.POINTER(_vp), C.POINTER(_i64)]),
    "lp_dit_get_config": (_i, [_vp, _vp]),
    "lp_verify_n_complete": (_i, [_i64p, _i32, _d, C.POINTER(_i32), _i32, _i32, _i64, C.POINTER(_i32),
                                  C.POINTER(_i32), _i64p, C.POINTER(_i32)]),
    "lp_coverage_trace": (_i, [_i64p, _i32, _d, C.POINTER(_i32), _i32, _i32, _i64, _i64p, _f64p, C.POINTER(_i32)]),
    "lp_latent_dump_write": (_i, [C.c_char_p, _vp, _i64p, _i32]),
    "lp_latent_dump_read": (_i, [C.c_char_p, _i64p, C.POINTER(_i32), _vp, _i64]),
    "lp_cli_main": (_i, [_i, C.POINTER(C.c_char_p)]),
    "lp_nccl_unique_id": (_i, [C.POINTER(C.c_uint8 * 128)]),
    "lp_engine_create": (_i, [C.POINTER(EngineConfig), _vp, _f64p, _i32, C.POINTER(_vp)]),
    "lp_engine_destroy": (_i, [_vp]),
    "lp_engine_latent": (_i, [_vp, C.POINTER(_vp)]),
    "lp_engine_run": (_i, [_vp, _i32, _i32, _vp]),
    "lp_engine_sync": (_i, [_vp, _vp, _i64]),
    "lp_engine_exchange_bench": (_i, [_vp, _i32, _i32, _vp, _f64p, C.POINTER(C.c_uint64)]),
    "lp_engine_hbm_bench": (_i, [_vp, _i32, _i32, _i32, _vp, _f64p]),
    "lp_engine_comm": (_i, [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "lp_engine_launches": (_i, [_vp, C.POINTER(C.c_uint64)]),
}

_lib = None


def lib():
    """Load liblp_b200.so (once).  Raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2512_07350_b200.build`")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def declared_symbols():
    return list(_SIGS)


def check(status: int) -> None:
    if status != 0:
        msg = lib().lp_last_error()
        raise LpError(status, msg.decode() if msg else "")


def i64arr(vals):
    vals = [int(v) for v in vals]
    return (C.c_int64 * len(vals))(*vals)
