"""ctypes access to the CPU oracles.  TEST INFRASTRUCTURE ONLY.

Two libraries, both built by ``oracle/Makefile``:

* ``Oracle``   — ``oracle/_build/liblp_oracle.so``: our plain-C restatement of the
  reference LP algorithm (``oracle/lp_oracle.c``).
* ``Reference`` — ``oracle/_ref/libref_harness.so``: the UNMODIFIED reference
  (lpsim, compiled from /root/reference/proj/src) behind a thin extern "C" harness.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl
reference`` legs may import this module, and only as the checker or the timed
CPU baseline.  The product (``paper_2512_07350_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liblp_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_harness.so")

_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


def build(quiet: bool = True) -> None:
    """Compile the oracle (and the reference harness when its sources exist)."""
    out = subprocess.run(["make", "-C", HERE, "-j8", "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
    if not quiet:
        print(out.stdout)


def _arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _p(a):
    if a is None:
        return None
    if a.dtype == np.float64:
        return a.ctypes.data_as(_f64p)
    return a.ctypes.data_as(_i64p)


class LpError(RuntimeError):
    """Carries the reference ErrorKind code (status - 1)."""

    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"status {status}: {msg}")
        self.status = status


@dataclass
class FlatPlan:
    meta: np.ndarray     # [axis, step, L, O, N, D, p, n]
    entries: np.ndarray  # [n, 9]

    @property
    def axis(self) -> int:
        return int(self.meta[0])

    @property
    def n(self) -> int:
        return int(self.meta[7])

    def latent(self, k):
        return int(self.entries[k, 5]), int(self.entries[k, 6])


def sub_shape(shape, plan: FlatPlan, k):
    s = list(shape)
    b, e = plan.latent(k)
    s[1 + plan.axis] = e - b
    return tuple(s)


def packed_size(shape, plan: FlatPlan) -> int:
    return int(sum(np.prod(sub_shape(shape, plan, k)) for k in range(plan.n)))


class _Lib:
    prefix = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(path + " (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        self.path = path

    def _check(self, st):
        if st != 0:
            msg = ""
            if hasattr(self.lib, "ref_last_error"):
                self.lib.ref_last_error.restype = C.c_char_p
                msg = self.lib.ref_last_error().decode()
            raise LpError(st, msg)

    def fn(self, name):
        return getattr(self.lib, self.prefix + name)

    # -- plan --
    def build_plan(self, shape, patch, step, workers, r, max_workers=None):
        meta = np.zeros(8, np.int64)
        ent = np.zeros((max(workers, 1), 9), np.int64)
        f = self.fn("build_plan")
        f.argtypes = [_i64p, _i64p, C.c_int, C.c_int, C.c_double, _i64p, _i64p]
        self._check(f(_p(_arr(shape, np.int64)), _p(_arr(patch, np.int64)), step, workers, r, _p(meta), _p(ent)))
        return FlatPlan(meta, ent[: meta[7]].copy())

    def build_axis_plan(self, axis, extent, patch, step, workers, r):
        meta = np.zeros(8, np.int64)
        ent = np.zeros((max(workers, 1), 9), np.int64)
        f = self.fn("build_axis_plan")
        f.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_double, _i64p, _i64p]
        self._check(f(axis, extent, patch, step, workers, r, _p(meta), _p(ent)))
        return FlatPlan(meta, ent[: meta[7]].copy())

    def quantize(self, v, dtype_bytes):
        f = self.fn("quantize")
        f.restype = C.c_double
        f.argtypes = [C.c_double, C.c_int]
        return f(v, dtype_bytes)

    def f16_encode(self, v):
        f = self.fn("f16_encode")
        f.restype = C.c_uint16
        f.argtypes = [C.c_double]
        return f(v)

    def f16_decode(self, b):
        f = self.fn("f16_decode")
        f.restype = C.c_double
        f.argtypes = [C.c_uint16]
        return f(b)

    def synthetic(self, shape, dtype_bytes, seed):
        z = np.zeros(int(np.prod(shape)), np.float64)
        c = np.zeros(8, np.float64)
        f = self.fn("synthetic")
        f.argtypes = [_i64p, C.c_int, C.c_uint64, _f64p, _f64p]
        self._check(f(_p(_arr(shape, np.int64)), dtype_bytes, seed, _p(z), _p(c)))
        return z.reshape(shape), c

    def sampler_step(self, z, eps, dtype_bytes, eta):
        z = _arr(z, np.float64)
        out = np.zeros_like(z)
        if self.prefix == "orc_":
            f = self.fn("sampler_step")
            f.argtypes = [_f64p, _f64p, C.c_int64, C.c_int, C.c_double, _f64p]
            self._check(f(_p(z), _p(_arr(eps, np.float64)), z.size, dtype_bytes, eta, _p(out)))
        else:
            f = self.fn("sampler_step")
            f.argtypes = [_f64p, _f64p, _i64p, C.c_int, C.c_double, _f64p]
            self._check(f(_p(z), _p(_arr(eps, np.float64)), _p(_arr(z.shape, np.int64)), dtype_bytes, eta, _p(out)))
        return out


class Oracle(_Lib):
    """Our C restatement (oracle/lp_oracle.c)."""

    prefix = "orc_"

    def __init__(self, path=ORACLE_SO):
        super().__init__(path)

    def weight_profile(self, plan: FlatPlan, k):
        b, e = plan.latent(k)
        out = np.zeros(e - b, np.float64)
        f = self.fn("weight_profile")
        f.argtypes = [_i64p, _f64p]
        f(_p(_arr(plan.entries[k], np.int64)), _p(out))
        return out

    def extract(self, z, plan: FlatPlan):
        z = _arr(z, np.float64)
        out = np.zeros(packed_size(z.shape, plan), np.float64)
        f = self.fn("extract")
        f.argtypes = [_f64p, _i64p, _i64p, _i64p, _f64p]
        self._check(f(_p(z), _p(_arr(z.shape, np.int64)), _p(plan.meta), _p(_arr(plan.entries, np.int64)), _p(out)))
        return out

    def toy_predict(self, kind, radius, z, dtype_bytes, t, cond_mean, t_coeff=0.01, cond_coeff=0.1):
        z = _arr(z, np.float64)
        out = np.zeros_like(z)
        f = self.fn("toy_predict")
        f.argtypes = [C.c_int, _i64p, C.c_double, C.c_double, _f64p, _i64p, C.c_int, C.c_int, C.c_double, _f64p]
        self._check(f(kind, _p(_arr(radius, np.int64)), t_coeff, cond_coeff, _p(z), _p(_arr(z.shape, np.int64)),
                      dtype_bytes, t, cond_mean, _p(out)))
        return out

    def cfg_predict(self, kind, radius, z, dtype_bytes, t, cond, w):
        z = _arr(z, np.float64)
        cond = _arr(cond, np.float64)
        out = np.zeros_like(z)
        f = self.fn("cfg_predict")
        f.argtypes = [C.c_int, _i64p, _f64p, _i64p, C.c_int, C.c_int, _f64p, C.c_int, C.c_double, _f64p]
        self._check(f(kind, _p(_arr(radius, np.int64)), _p(z), _p(_arr(z.shape, np.int64)), dtype_bytes, t,
                      _p(cond), cond.size, w, _p(out)))
        return out

    def reconstruct(self, preds_packed, shape, dtype_bytes, plan: FlatPlan):
        out = np.zeros(int(np.prod(shape)), np.float64)
        f = self.fn("reconstruct")
        f.argtypes = [_f64p, _i64p, C.c_int, _i64p, _i64p, _f64p]
        self._check(f(_p(_arr(preds_packed, np.float64)), _p(_arr(shape, np.int64)), dtype_bytes, _p(plan.meta),
                      _p(_arr(plan.entries, np.int64)), _p(out)))
        return out.reshape(shape)

    def run_lp(self, kind, radius, z, dtype_bytes, steps, eta, w, cond, patch, workers, r, wire_bytes=2):
        z = _arr(z, np.float64)
        cond = _arr(cond, np.float64)
        out = np.zeros_like(z)
        ledger = C.c_uint64(0)
        f = self.fn("run_lp")
        f.argtypes = [C.c_int, _i64p, _f64p, _i64p, C.c_int, C.c_int, C.c_double, C.c_double, _f64p, C.c_int,
                      _i64p, C.c_int, C.c_double, C.c_int, _f64p, C.POINTER(C.c_uint64)]
        self._check(f(kind, _p(_arr(radius, np.int64)), _p(z), _p(_arr(z.shape, np.int64)), dtype_bytes, steps, eta,
                      w, _p(cond), cond.size, _p(_arr(patch, np.int64)), workers, r, wire_bytes, _p(out),
                      C.byref(ledger)))
        return out, int(ledger.value)


class Reference(_Lib):
    """The unmodified reference (lpsim) through oracle/ref_harness.cpp."""

    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)
        self.lib.ref_silence_warnings.argtypes = [C.c_int]
        self.lib.ref_silence_warnings(1)

    def weight_profile(self, shape, patch, step, workers, r, k):
        plan = self.build_plan(shape, patch, step, workers, r)
        b, e = plan.latent(k)
        out = np.zeros(e - b, np.float64)
        f = self.fn("weight_profile")
        f.argtypes = [_i64p, _i64p, C.c_int, C.c_int, C.c_double, C.c_int, _f64p]
        self._check(f(_p(_arr(shape, np.int64)), _p(_arr(patch, np.int64)), step, workers, r, k, _p(out)))
        return out

    def extract(self, z, dtype_bytes, patch, step, workers, r):
        z = _arr(z, np.float64)
        plan = self.build_plan(z.shape, patch, step, workers, r)
        out = np.zeros(packed_size(z.shape, plan), np.float64)
        f = self.fn("extract")
        f.argtypes = [_f64p, _i64p, C.c_int, _i64p, C.c_int, C.c_int, C.c_double, _f64p]
        self._check(f(_p(z), _p(_arr(z.shape, np.int64)), dtype_bytes, _p(_arr(patch, np.int64)), step, workers, r,
                      _p(out)))
        return out

    def toy_predict(self, kind, radius, z, dtype_bytes, t, cond, is_null=False):
        z = _arr(z, np.float64)
        cond = _arr(cond, np.float64)
        out = np.zeros_like(z)
        f = self.fn("toy_predict")
        f.argtypes = [C.c_int, _i64p, _f64p, _i64p, C.c_int, C.c_int, _f64p, C.c_int, C.c_int, _f64p]
        self._check(f(kind, _p(_arr(radius, np.int64)), _p(z), _p(_arr(z.shape, np.int64)), dtype_bytes, t,
                      _p(cond), cond.size, int(is_null), _p(out)))
        return out

    def cfg_predict(self, kind, radius, z, dtype_bytes, t, cond, w):
        z = _arr(z, np.float64)
        cond = _arr(cond, np.float64)
        out = np.zeros_like(z)
        f = self.fn("cfg_predict")
        f.argtypes = [C.c_int, _i64p, _f64p, _i64p, C.c_int, C.c_int, _f64p, C.c_int, C.c_double, _f64p]
        self._check(f(kind, _p(_arr(radius, np.int64)), _p(z), _p(_arr(z.shape, np.int64)), dtype_bytes, t,
                      _p(cond), cond.size, w, _p(out)))
        return out

    def reconstruct(self, preds_packed, shape, dtype_bytes, patch, step, workers, r):
        out = np.zeros(int(np.prod(shape)), np.float64)
        f = self.fn("reconstruct")
        f.argtypes = [_f64p, _i64p, C.c_int, _i64p, C.c_int, C.c_int, C.c_double, _f64p]
        self._check(f(_p(_arr(preds_packed, np.float64)), _p(_arr(shape, np.int64)), dtype_bytes,
                      _p(_arr(patch, np.int64)), step, workers, r, _p(out)))
        return out.reshape(shape)

    def run_lp(self, kind, radius, z, dtype_bytes, steps, eta, w, cond, patch, workers, r, wire_bytes=2,
               trace=False):
        z = _arr(z, np.float64)
        cond = _arr(cond, np.float64)
        out = np.zeros_like(z)
        tr = np.zeros((steps,) + z.shape, np.float64) if trace else None
        ledger = C.c_uint64(0)
        f = self.fn("run_lp")
        f.argtypes = [C.c_int, _i64p, _f64p, _i64p, C.c_int, C.c_int, C.c_double, C.c_double, _f64p, C.c_int,
                      _i64p, C.c_int, C.c_double, C.c_int, _f64p, _f64p, C.POINTER(C.c_uint64)]
        self._check(f(kind, _p(_arr(radius, np.int64)), _p(z), _p(_arr(z.shape, np.int64)), dtype_bytes, steps, eta,
                      w, _p(cond), cond.size, _p(_arr(patch, np.int64)), workers, r, wire_bytes, _p(tr), _p(out),
                      C.byref(ledger)))
        return (out, int(ledger.value), tr) if trace else (out, int(ledger.value))

    def run_lp_callback(self, predict, z, dtype_bytes, steps, eta, w, cond, patch, workers, r, wire_bytes=2,
                        trace=False):
        """run_lp with an external Denoiser: predict(z: ndarray, t: int, cond: ndarray, is_null) -> ndarray."""
        CB = C.CFUNCTYPE(None, _f64p, _i64p, C.c_int, C.c_int, _f64p, C.c_int, C.c_int, _f64p, C.c_void_p)

        def _cb(zp, sp, db, t, cp, nc, isnull, outp, user):
            shape = tuple(sp[i] for i in range(4))
            n = int(np.prod(shape))
            zz = np.ctypeslib.as_array(zp, shape=(n,)).reshape(shape).copy()
            cc = np.ctypeslib.as_array(cp, shape=(nc,)).copy() if nc else np.zeros(0)
            res = np.asarray(predict(zz, t, cc, bool(isnull)), np.float64).reshape(-1)
            np.ctypeslib.as_array(outp, shape=(n,))[:] = res

        cb = CB(_cb)
        z = _arr(z, np.float64)
        cond = _arr(cond, np.float64)
        out = np.zeros_like(z)
        tr = np.zeros((steps,) + z.shape, np.float64) if trace else None
        ledger = C.c_uint64(0)
        f = self.fn("run_lp_callback")
        f.argtypes = [CB, C.c_void_p, _f64p, _i64p, C.c_int, C.c_int, C.c_double, C.c_double, _f64p, C.c_int,
                      _i64p, C.c_int, C.c_double, C.c_int, _f64p, _f64p, C.POINTER(C.c_uint64)]
        self._check(f(cb, None, _p(z), _p(_arr(z.shape, np.int64)), dtype_bytes, steps, eta, w, _p(cond), cond.size,
                      _p(_arr(patch, np.int64)), workers, r, wire_bytes, _p(tr), _p(out), C.byref(ledger)))
        return (out, int(ledger.value), tr) if trace else (out, int(ledger.value))

    def run_centralized(self, kind, radius, z, dtype_bytes, steps, eta, w, cond):
        z = _arr(z, np.float64)
        cond = _arr(cond, np.float64)
        out = np.zeros_like(z)
        f = self.fn("run_centralized")
        f.argtypes = [C.c_int, _i64p, _f64p, _i64p, C.c_int, C.c_int, C.c_double, C.c_double, _f64p, C.c_int,
                      _f64p, _f64p]
        self._check(f(kind, _p(_arr(radius, np.int64)), _p(z), _p(_arr(z.shape, np.int64)), dtype_bytes, steps, eta,
                      w, _p(cond), cond.size, None, _p(out)))
        return out

    def cost(self, steps, workers, r, shape, patch, hidden=1536, wire_bytes=2, hybrid=None):
        out = np.zeros(21, np.float64)
        groups, sizes = (0, [0]) if hybrid is None else (hybrid[0], list(hybrid[1]))
        sz = (C.c_int * len(sizes))(*sizes)
        f = self.fn("cost")
        f.argtypes = [C.c_int, C.c_int, C.c_double, _i64p, _i64p, C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int),
                      _f64p]
        self._check(f(steps, workers, r, _p(_arr(shape, np.int64)), _p(_arr(patch, np.int64)), hidden, wire_bytes,
                      groups, sz, _p(out)))
        d = {"S_z": out[0], "S_H": out[1], "gamma": out[3], "gamma_per_axis": tuple(out[4:7]), "C_NMP": out[7],
             "C_PP": out[8], "C_LP_exact": out[9], "C_LP_approx": out[10], "ratio_exact": out[11],
             "ratio_approx": out[12], "Sz_over_SH": out[13]}
        if out[14]:
            d["hybrid"] = {"C_inter": out[15], "C_intra_total": out[16], "C_hyb": out[17], "ratio_vs_NMP": out[18],
                           "bound": out[19], "within_bound": bool(out[20])}
        return d


def verify_n_complete(ref: "Reference", grid, workers, r, schedule, budget):
    out = np.zeros(5, np.int64)
    sched = (C.c_int * len(schedule))(*schedule)
    f = ref.fn("verify_n_complete")
    f.argtypes = [_i64p, C.c_int, C.c_double, C.POINTER(C.c_int), C.c_int, C.c_int, _i64p]
    ref._check(f(_p(_arr(grid, np.int64)), workers, r, sched, len(schedule), budget, _p(out)))
    return {"complete": bool(out[0]), "complete_at": int(out[1]) if out[0] else None,
            "worst_position": tuple(int(v) for v in out[2:5])}


def reference_available() -> bool:
    return os.path.exists(REF_SO)
