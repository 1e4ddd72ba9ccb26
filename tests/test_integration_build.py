"""The drop-in's link-time substitution (integration/Makefile), checked on CPU: the backend defines
exactly the reference hot-path functions it replaces, the reference archive carries them weakened,
and each drop-in artifact resolves every one of them to the backend's single strong definition."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B = os.path.join(ROOT, "integration", "_build")
REPLACED = {"lpsim::extract_sublatents", "lpsim::reconstruct", "lpsim::cfg_predict", "lpsim::sampler_step",
            "lpsim::make_box_denoiser", "lpsim::make_global_mix_denoiser", "lpsim::make_identity_denoiser",
            "lpsim::run_centralized", "lpsim::run_lp"}


def _nm(path, *flags):
    r = subprocess.run(["nm", "-C", *flags, path], capture_output=True, text=True, check=True)
    return r.stdout.splitlines()


def _names(lines, kinds):
    out = {}
    for l in lines:
        parts = l.split(None, 2)
        if len(parts) == 3 and parts[1] in kinds and "[clone" not in parts[2]:
            out.setdefault(parts[2].split("(")[0], []).append(parts[1])
    return out


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(os.path.join(B, "libb200_dropin.so")):
        pytest.skip("integration/_build not built (make -C integration needs /root/reference)")
    return B


def test_backend_defines_exactly_the_replaced_functions(built):
    strong = _names(_nm(os.path.join(B, "b200_backend.o"), "-g", "--defined-only"), {"T"})
    assert set(strong) == REPLACED


def test_reference_archive_carries_them_weakened(built):
    weak = _names(_nm(os.path.join(B, "liblpsim_dropin.a"), "--defined-only"), {"W"})
    assert REPLACED <= set(weak)
    plain = _names(_nm(os.path.join(B, "liblpsim_ref.a"), "--defined-only"), {"T"})
    assert REPLACED <= set(plain)  # the plugin build links the unmodified reference


@pytest.mark.parametrize("artifact", ["libb200_dropin.so", "acceptance_b200", "lpsim/_lpsim"])
def test_artifacts_resolve_to_one_strong_definition(built, artifact):
    path = os.path.join(B, artifact)
    if artifact.startswith("lpsim/"):
        path = [os.path.join(B, "lpsim", f) for f in os.listdir(os.path.join(B, "lpsim")) if f.endswith(".so")][0]
    defs = _names(_nm(path, "--defined-only"), {"T", "W"})
    for fn in REPLACED:
        assert defs.get(fn) == ["T"], (fn, defs.get(fn))
    assert "lp_engine_create" in " ".join(_nm(path, "-u"))  # bound to liblp_b200.so's C-ABI
