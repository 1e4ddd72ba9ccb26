"""The `lpsim` command layer on the B200 engine: the same commands,
options, artifacts and exit codes as the reference CLI (tools/lpsim_main.cpp:42-113,
src/commands.cpp:46-216, src/run_config.cpp:85-247, src/io.cpp:37-244).

Artifacts are compared BYTE FOR BYTE with the unmodified reference's own command
functions (oracle/_ref, ref_command) run on the same config.  Host-only commands
(cost, completeness, partition-plan, config errors, LPLT dumps) run here; simulate /
compare need the GPU engine (marked gpu)."""
import ctypes as C
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2512_07350_b200 import lp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2512_07350_b200", "lpsim_b200")

# the reference's three shipped configs (proj/configs/*.json), restated
DESK = {"latent": {"C": 4, "T": 12, "H": 16, "W": 16, "dtype_bytes": 4}, "patch": {"p_T": 2, "p_H": 2, "p_W": 2},
        "sampler": {"steps": 60, "eta": 0.05, "guidance_w": 3.0},
        "denoiser": {"kind": "box", "radius": [1, 1, 1], "seed": 42}, "cluster": {"K": 4, "r": 0.5},
        "preset": "wan21-like", "output": {"dir": "out/desk_default", "formats": ["json", "csv", "bin"]}}
EQUIV = {"latent": {"C": 4, "T": 12, "H": 16, "W": 16, "dtype_bytes": 4}, "patch": {"p_T": 2, "p_H": 2, "p_W": 2},
         "sampler": {"steps": 6, "eta": 0.05, "guidance_w": 2.0},
         "denoiser": {"kind": "box", "radius": [2, 2, 2], "seed": 2025}, "cluster": {"K": 2, "r": 1.0},
         "preset": "wan21-like", "output": {"dir": "out/equivalence", "formats": ["json", "csv"]}}
WAN49 = {"latent": {"C": 16, "T": 13, "H": 60, "W": 104, "dtype_bytes": 2}, "patch": {"p_T": 1, "p_H": 2, "p_W": 2},
         "sampler": {"steps": 60, "eta": 0.05, "guidance_w": 5.0}, "denoiser": {"kind": "identity", "seed": 1},
         "cluster": {"K": 4, "r": 0.5}, "preset": "wan21-like", "hybrid": {"M": 2, "group_sizes": [2, 2]},
         "output": {"dir": "out/wan21_like_49f", "formats": ["json", "csv"]}}


def write_cfg(tmp_path, doc, name="cfg.json"):
    p = tmp_path / name
    p.write_text(json.dumps(doc) if isinstance(doc, dict) else doc)
    return str(p)


def ref_command(reference, cmd, cfg, out, seed=-1, schedule="rotating", max_steps=8, step=1):
    buf = C.create_string_buffer(1 << 22)
    f = reference.fn("command")
    f.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int64, C.c_char_p, C.c_int, C.c_int, C.c_char_p, C.c_int64]
    st = f(cmd.encode(), cfg.encode(), str(out).encode(), seed, schedule.encode(), max_steps, step, buf, len(buf))
    msg = reference.fn("last_error")
    msg.restype = C.c_char_p
    return st, (buf.value.decode() if st == 0 else msg().decode())


def ours(args):
    return subprocess.run([CLI, *args], capture_output=True, text=True)


def same_tree(a, b):
    fa, fb = sorted(os.listdir(a)), sorted(os.listdir(b))
    assert fa == fb, (fa, fb)
    for f in fa:
        assert open(os.path.join(a, f), "rb").read() == open(os.path.join(b, f), "rb").read(), f
    return fa


def run_both(reference, tmp_path, doc, cmd, extra=(), **kw):
    cfg = write_cfg(tmp_path, doc)
    mine, theirs = tmp_path / "ours", tmp_path / "ref"
    r = ours([cmd, "--config", cfg, "--out", str(mine), *extra])
    assert r.returncode == 0, r.stderr
    st, summary = ref_command(reference, cmd, cfg, theirs, **kw)
    assert st == 0, summary
    assert r.stdout == summary + "\n"
    return same_tree(mine, theirs)


@pytest.mark.parametrize("doc", [DESK, EQUIV, WAN49], ids=["desk", "equiv", "wan49"])
def test_cost_command_bytes_match_reference(reference, tmp_path, doc):
    files = run_both(reference, tmp_path, doc, "cost")
    assert "cost.json" in files


@pytest.mark.parametrize("doc", [DESK, EQUIV], ids=["desk", "equiv"])
@pytest.mark.parametrize("sched,steps", [("rotating", 8), ("temporal", 6), ("width", 3)])
def test_completeness_command_bytes_match_reference(reference, tmp_path, doc, sched, steps):
    files = run_both(reference, tmp_path, doc, "completeness", ["--schedule", sched, "--max-steps", str(steps)],
                     schedule=sched, max_steps=steps)
    assert set(files) == {"completeness.json", "coverage.csv"}


@pytest.mark.parametrize("doc", [DESK, EQUIV, WAN49], ids=["desk", "equiv", "wan49"])
@pytest.mark.parametrize("step", [1, 2, 3, 7])
def test_partition_plan_command_bytes_match_reference(reference, tmp_path, doc, step):
    run_both(reference, tmp_path, doc, "partition-plan", ["--step", str(step)], step=step)


def test_k_eff_warning_and_quiet(reference, tmp_path):
    # D_T = 5 patches for K = 8 -> K_eff < K warning on stderr (src/partition.cpp:100-110); --quiet silences
    doc = json.loads(json.dumps(EQUIV))
    doc["latent"]["T"] = 10
    doc["cluster"] = {"K": 8, "r": 0.5}
    cfg = write_cfg(tmp_path, doc)
    r = ours(["partition-plan", "--config", cfg, "--out", str(tmp_path / "a")])
    assert r.returncode == 0 and "lpsim: warning:" in r.stderr
    q = ours(["partition-plan", "--config", cfg, "--out", str(tmp_path / "b"), "--quiet"])
    assert q.returncode == 0 and q.stdout == "" and q.stderr == ""


BAD = [
    ('{"latent": 1}', "'latent' must be a JSON object"),
    ("{", None),
    (dict(DESK, extra=1), "unknown key 'extra' in 'config'"),
    (dict(DESK, cluster={"K": 4, "r": 3.5}), "'cluster.r' must lie in [0, K-1]"),
    (dict(DESK, preset="nope"), "unknown preset 'nope'"),
    (dict(DESK, sampler={"steps": 0, "eta": 0.05, "guidance_w": 1.0}), "'sampler.steps' must be >= 1"),
    (dict(DESK, denoiser={"kind": "gauss"}), "'denoiser.kind' must be one of box, global, identity"),
    (dict(DESK, output={"formats": ["xml"]}), "unknown output format 'xml'"),
    (dict(DESK, hybrid={"M": 2, "group_sizes": [1, 1]}), "'hybrid.group_sizes' must sum to cluster.K"),
    (dict(DESK, patch={"p_T": 20, "p_H": 2, "p_W": 2}), "latent axis temporal is smaller than its patch size"),
]


@pytest.mark.parametrize("doc,msg", BAD)
def test_config_errors_exit_2_with_reference_message(reference, tmp_path, doc, msg):
    cfg = write_cfg(tmp_path, doc)
    r = ours(["cost", "--config", cfg, "--out", str(tmp_path / "o")])
    st, ref_msg = ref_command(reference, "cost", cfg, tmp_path / "r")
    assert r.returncode == 2 and st == 12  # ErrorKind::Config + 1
    assert r.stderr == f"lpsim: error: {ref_msg}\n"
    if msg:
        assert msg in ref_msg


def test_usage_errors(tmp_path):
    assert ours([]).returncode == 2
    assert ours(["frobnicate"]).returncode == 2
    assert ours(["cost"]).returncode == 2                      # --config is required
    assert ours(["cost", "--config", "/nonexistent.json"]).returncode == 2
    assert ours(["partition-plan", "--config", "x", "--step", "0"]).returncode == 2
    assert ours(["cost", "--config", "x", "--backend", "cpu"]).returncode == 2
    assert ours(["--help"]).returncode == 0


def test_python_module_entry_point(reference, tmp_path):
    cfg = write_cfg(tmp_path, EQUIV)
    r = subprocess.run(["python", "-m", "paper_2512_07350_b200", "cost", "--config", cfg, "--out",
                        str(tmp_path / "o"), "--quiet"], capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    st, _ = ref_command(reference, "cost", cfg, tmp_path / "r")
    same_tree(tmp_path / "o", tmp_path / "r")


# ---- LPLT latent dumps (src/io.cpp:37-139) ----
def _bits(values, db):
    return values.astype({2: np.float16, 4: np.float32, 8: np.float64}[db])


@pytest.mark.parametrize("db", [2, 4, 8])
def test_latent_dump_bytes_match_reference(reference, oracle, tmp_path, db):
    z, _ = oracle.synthetic((3, 4, 5, 6), db, 7)
    shape = (C.c_int64 * 4)(*z.shape)
    mine, theirs = tmp_path / "a.bin", tmp_path / "b.bin"
    bits = np.ascontiguousarray(_bits(z, db))
    assert lp.lib().lp_latent_dump_write(str(mine).encode(), bits.ctypes.data, shape, db) == 0
    f = reference.fn("save_latent")
    f.argtypes = [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int]
    zz = np.ascontiguousarray(z, np.float64)
    assert f(str(theirs).encode(), zz.ctypes.data_as(C.POINTER(C.c_double)), shape, db) == 0
    assert mine.read_bytes() == theirs.read_bytes()
    # read back through ours: same bits and header
    sh, dt = (C.c_int64 * 4)(), C.c_int32()
    out = np.empty_like(bits)
    assert lp.lib().lp_latent_dump_read(str(theirs).encode(), sh, C.byref(dt), out.ctypes.data, out.nbytes) == 0
    assert tuple(sh) == z.shape and dt.value == db and out.tobytes() == bits.tobytes()


def test_latent_dump_read_errors(reference, tmp_path):
    sh, dt = (C.c_int64 * 4)(), C.c_int32()
    L = lp.lib()
    assert L.lp_latent_dump_read(str(tmp_path / "missing.bin").encode(), sh, C.byref(dt), None, 0) == 13
    (tmp_path / "junk.bin").write_bytes(b"NOTADUMP" * 8)
    assert L.lp_latent_dump_read(str(tmp_path / "junk.bin").encode(), sh, C.byref(dt), None, 0) == 13
    good = tmp_path / "g.bin"
    v = np.ones((1, 1, 2, 2), np.float32)
    assert L.lp_latent_dump_write(str(good).encode(), v.ctypes.data, (C.c_int64 * 4)(1, 1, 2, 2), 4) == 0
    (tmp_path / "trunc.bin").write_bytes(good.read_bytes()[:-1])
    assert L.lp_latent_dump_read(str(tmp_path / "trunc.bin").encode(), sh, C.byref(dt), None, 0) == 13
    nan = np.full((1, 1, 2, 2), np.nan, np.float32)
    (tmp_path / "nan.bin").write_bytes(good.read_bytes()[:32] + nan.tobytes())
    buf = np.empty(4, np.float32)
    assert L.lp_latent_dump_read(str(tmp_path / "nan.bin").encode(), sh, C.byref(dt), buf.ctypes.data, 16) == 11
    # the reference agrees on every one of these
    f = reference.fn("load_latent")
    f.argtypes = [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int), C.c_void_p]
    d = C.c_int()
    for name, code in (("missing.bin", 13), ("junk.bin", 13), ("trunc.bin", 13), ("nan.bin", 11)):
        assert f(str(tmp_path / name).encode(), sh, C.byref(d), None) == code, name


# ---- simulate / compare: the GPU engine behind the reference's command layer ----
@pytest.mark.gpu
@pytest.mark.parametrize("doc", [DESK, EQUIV], ids=["desk", "equiv"])
def test_simulate_command_bytes_match_reference(cuda, reference, tmp_path, doc):
    files = run_both(reference, tmp_path, doc, "simulate")
    assert "summary.json" in files and "ledger.csv" in files


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [2, 4, 8])
def test_simulate_z0_bin_all_dtypes(cuda, reference, tmp_path, dtype):
    doc = json.loads(json.dumps(EQUIV))
    doc["latent"]["dtype_bytes"] = dtype
    doc["output"]["formats"] = ["json", "csv", "bin"]
    assert "z0.bin" in run_both(reference, tmp_path, doc, "simulate")


@pytest.mark.gpu
@pytest.mark.parametrize("doc", [DESK, EQUIV], ids=["desk", "equiv"])
def test_compare_command_bytes_match_reference(cuda, reference, tmp_path, doc):
    assert set(run_both(reference, tmp_path, doc, "compare")) == {"diff.csv", "compare.json"}
