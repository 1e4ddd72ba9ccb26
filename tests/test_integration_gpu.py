"""The reference-side integration (integration/), built by integration/Makefile
from the reference's unmodified sources:

* drop-in mode — the reference archive with its hot-path symbols weakened, replaced at link time
  by integration/b200_backend.cpp: the reference's OWN acceptance suite (tests/acceptance.cpp,
  criteria 1-8, its CLI criterion on lpsim_b200) and its OWN python smoke test
  (tests/python/test_smoke.py, against its own pybind module) pass on the B200 engine;
* plugin mode — the UNMODIFIED reference run_lp / run_centralized driving the B200 denoisers
  (the WAN-shaped DiT's single-pass predict, the K11 toys) through the Denoiser slot.

run_lp through the drop-in returns the full LpRunResult: final latent, per-step trace and the
per-record CommLedger, all bit-identical to the unmodified reference (plugin mode with the
reference's own toy denoisers), in every storage dtype; the B200 DiT gives bit-identical
results under the unmodified reference loop and under the drop-in engine loop.
"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B = os.path.join(ROOT, "integration", "_build")
_f64p = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_u64p = C.POINTER(C.c_uint64)


def _lib(name):
    path = os.path.join(B, name)
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: build with `make -C integration` (needs /root/reference)")
    L = C.CDLL(path)
    L.check_run_lp.argtypes = [C.c_int, _i64p, C.c_int, _f64p, _i64p, C.c_int, C.c_int, C.c_double, C.c_double,
                               _f64p, C.c_int, _i64p, C.c_int, C.c_double, C.c_int, _f64p, _f64p, _u64p, _u64p,
                               C.c_int64]
    L.check_run_centralized.argtypes = [C.c_int, _i64p, C.c_int, _f64p, _i64p, C.c_int, C.c_int, C.c_double,
                                        C.c_double, _f64p, C.c_int, _f64p]
    L.check_dit_predict.argtypes = [C.c_int, _f64p, _i64p, C.c_int, C.c_int, _f64p, C.c_int, C.c_int, _f64p]
    L.check_last_error.restype = C.c_char_p
    return L


def run_lp(L, denoiser, z, d, steps, cond, patch, K, r, eta=0.05, w=3.0, layers=2, radius=(1, 1, 1), wire=2):
    shape = np.array(z.shape, np.int64)
    out = np.zeros(z.shape)
    trace = np.zeros((steps,) + z.shape)
    led = np.zeros(2, np.uint64)
    cap = 4 * steps * 256
    rec = np.zeros((cap, 7), np.uint64)
    rad, pt = np.array(radius, np.int64), np.array(patch, np.int64)
    zc, cc = np.ascontiguousarray(z, np.float64), np.ascontiguousarray(cond, np.float64)
    st = L.check_run_lp(denoiser, rad.ctypes.data_as(_i64p), layers, zc.ctypes.data_as(_f64p),
                        shape.ctypes.data_as(_i64p), d, steps, eta, w, cc.ctypes.data_as(_f64p), cc.size,
                        pt.ctypes.data_as(_i64p), K, r, wire, out.ctypes.data_as(_f64p), trace.ctypes.data_as(_f64p),
                        led.ctypes.data_as(_u64p), rec.ctypes.data_as(_u64p), cap)
    if st:
        return st, L.check_last_error().decode()
    return 0, (out, trace, int(led[0]), rec[: int(led[1])].copy())


@pytest.fixture(scope="module")
def libs(cuda):
    return _lib("libb200_plugin.so"), _lib("libb200_dropin.so")


@pytest.mark.gpu
def test_reference_acceptance_suite_on_the_b200_dropin(cuda):
    exe = os.path.join(B, "acceptance_b200")
    assert os.path.exists(exe), "build with make -C integration"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("[")]
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert len(lines) == 8 and all(l.startswith("[PASS]") for l in lines), r.stdout


@pytest.mark.gpu
def test_reference_python_smoke_test_on_the_b200_dropin(cuda):
    env = dict(os.environ, PYTHONPATH=B)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "test_smoke.py"], cwd=B,
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
    # the module really is the drop-in: its run_lp launches this engine's kernels
    probe = ("import lpsim, ctypes; L = ctypes.CDLL('" + os.path.join(ROOT, "paper_2512_07350_b200", "liblp_b200.so")
             + "'); L.lp_launch_count.restype = ctypes.c_uint64; z, c = lpsim.synthetic_latent((4, 6, 8, 8), 4, 3); "
             "n0 = L.lp_launch_count(); lpsim.run_lp('box', (1, 1, 1), z, 2, 0.1, 2.0, c, (2, 2, 2), 2, 0.5); "
             "print(L.lp_launch_count() - n0)")
    r = subprocess.run([sys.executable, "-c", probe], cwd=B, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert int(r.stdout.strip().splitlines()[-1]) > 0


@pytest.mark.gpu
@pytest.mark.parametrize("d", [2, 4, 8])
@pytest.mark.parametrize("denoiser,dims,patch,K,r,steps", [
    (0, (4, 12, 16, 16), (2, 2, 2), 2, 1.0, 6),      # acceptance criterion 1's config
    (0, (16, 5, 16, 16), (1, 2, 2), 4, 0.5, 5),      # C1 shape
    (1, (3, 7, 9, 5), (1, 2, 1), 3, 0.25, 4),        # global mix, remainder extents
    (2, (2, 9, 6, 11), (3, 2, 2), 8, 0.0, 3),        # identity, K_eff < K
])
def test_dropin_run_lp_equals_unmodified_reference(libs, oracle, d, denoiser, dims, patch, K, r, steps):
    """Drop-in run_lp (engine: K1, K11 fused CFG, K10) vs the unmodified reference run_lp with its
    own toy denoisers: final latent, every trace entry and every ledger record, bit for bit."""
    plugin, dropin = libs
    z, cond = oracle.synthetic(dims, d, 2025)
    a = run_lp(plugin, denoiser, z, d, steps, cond, patch, K, r)
    b = run_lp(dropin, denoiser, z, d, steps, cond, patch, K, r)
    assert a[0] == 0 and b[0] == 0, (a, b)
    (fa, ta, la, ra), (fb, tb, lb, rb) = a[1], b[1]
    assert fa.tobytes() == fb.tobytes()
    assert ta.tobytes() == tb.tobytes()
    assert la == lb and np.array_equal(ra, rb)
    assert len(ra) > 0 or K == 1


@pytest.mark.gpu
@pytest.mark.parametrize("d", [2, 4, 8])
def test_unmodified_reference_loop_drives_the_b200_dit(libs, d):
    """Plugin mode: the UNMODIFIED reference run_lp calls the B200 DiT's single-pass predict
    twice per shard (cfg_predict, src/denoise.cpp:24-39) and blends on the host; the drop-in
    runs the fused CFG-batch-2 engine.  Bit-identical latents, traces and ledgers."""
    from paper_2512_07350_b200 import lp

    plugin, dropin = libs
    dims = (16, 5, 16, 16)
    z, cond = lp.synthetic_latent_host(dims, d, 2025)
    os.environ["LPSIM_THREADS"] = "4"   # the reference pool calls predict() concurrently
    a = run_lp(plugin, -1, z, d, 4, cond, (1, 2, 2), 2, 0.5, w=5.0)
    b = run_lp(dropin, -1, z, d, 4, cond, (1, 2, 2), 2, 0.5, w=5.0)
    assert a[0] == 0 and b[0] == 0, (a, b)
    assert a[1][0].tobytes() == b[1][0].tobytes()
    assert a[1][1].tobytes() == b[1][1].tobytes()
    assert a[1][2] == b[1][2] and np.array_equal(a[1][3], b[1][3])
    # and the python engine (lp.LpEngine) agrees with both
    dit = lp.DiTDenoiser(list(cond), num_layers=2)
    eng = lp.LpEngine(dims, (1, 2, 2), d, 2, 0.5, 4, 0.05, 5.0, list(cond), denoiser="dit", dit=dit)
    eng.load(lp.LatentTensor.from_numpy(z, d))
    eng.run(1, 4)
    got = eng.z.data.double().cpu().numpy()
    eng.close()
    assert got.tobytes() == a[1][0].tobytes()


@pytest.mark.gpu
def test_dropin_run_centralized_and_errors_match_reference(libs, oracle):
    plugin, dropin = libs
    z, cond = oracle.synthetic((2, 6, 8, 8), 4, 11)
    outs = []
    for L in libs:
        out = np.zeros(z.shape)
        zc, cc = np.ascontiguousarray(z), np.ascontiguousarray(cond)
        rad, sh = np.array([1, 1, 1], np.int64), np.array(z.shape, np.int64)
        assert L.check_run_centralized(0, rad.ctypes.data_as(_i64p), 0, zc.ctypes.data_as(_f64p),
                                       sh.ctypes.data_as(_i64p), 4, 3, 0.1, 2.0, cc.ctypes.data_as(_f64p), cc.size,
                                       out.ctypes.data_as(_f64p)) == 0
        outs.append(out)
    assert outs[0].tobytes() == outs[1].tobytes()
    # error kinds (status = ErrorKind + 1) and messages agree on invalid inputs
    for args in [dict(K=2, r=1.5), dict(K=0, r=0.0), dict(K=2, r=0.5, patch=(9, 2, 2))]:
        a = run_lp(plugin, 0, z, 4, 2, cond, args.get("patch", (2, 2, 2)), args["K"], args["r"])
        b = run_lp(dropin, 0, z, 4, 2, cond, args.get("patch", (2, 2, 2)), args["K"], args["r"])
        assert a[0] != 0 and a == b, (args, a, b)
