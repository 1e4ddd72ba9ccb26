"""Build liblp_b200.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2512_07350_b200.build

Objects go to paper_2512_07350_b200/_build/, the library to
paper_2512_07350_b200/liblp_b200.so (git-ignored; travels to the GPU box).
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "liblp_b200.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCS = ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC]

# (source, extra flags).  lp_kernels.cu must not contract FMAs (exact mode).
SOURCES = [
    ("lp_host.cpp", ["-Xcompiler", "-ffp-contract=off"]),
    ("cost.cpp", ["-Xcompiler", "-ffp-contract=off"]),
    ("lp_kernels.cu", ["-fmad=false"]),
    ("dit_kernels.cu", []),
    ("gemm_tcgen05.cu", []),
    ("attn_tcgen05.cu", []),
    ("dit.cpp", []),
    ("engine.cpp", ["-Xcompiler", "-ffp-contract=off"]),
    ("completeness.cpp", []),
    ("commands.cpp", None),  # host-only (g++): the lpsim command layer, nlohmann/json
]
GXX = shutil.which("g++") or "g++"
CUDA_INC = os.path.join(os.path.dirname(os.path.dirname(os.path.realpath(NVCC))), "include")
# nlohmann/json 3.11.3 — the header the reference's own build uses (vendored by cudnn_frontend in this image)
JSON_INC = os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}", "site-packages",
                        "include", "cudnn_frontend", "thirdparty", "nlohmann")
CLI = os.path.join(PKG, "lpsim_b200")


def _cmd(src, extra):
    path = os.path.join(CSRC, src)
    obj = os.path.join(OUT, src + ".o")
    if extra is None:  # host-only C++
        return path, obj, [GXX, "-std=c++17", "-O2", "-fPIC", "-I" + CUDA_INC, "-I" + JSON_INC, *INCS, "-c", path,
                           "-o", obj]
    lang = ["-x", "cu"]  # .cpp too: they share the device codec header
    cmd = [NVCC, *lang, "-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC", "-Xptxas", "-v",
           "--expt-relaxed-constexpr", *INCS, *extra, *os.environ.get("LP_NVCC_EXTRA", "").split(), "-c", path,
           "-o", obj]
    return path, obj, cmd


def _digest(cmd, path):
    h = hashlib.sha256(" ".join(cmd).encode())
    for f in sorted(os.listdir(CSRC)) + [os.path.join(ROOT, "include", "lp_b200.h")]:
        p = f if os.path.isabs(f) else os.path.join(CSRC, f)
        if p.endswith((".h", ".hpp", ".cuh")) or p == path:
            with open(p, "rb") as fh:
                h.update(fh.read())
    return h.hexdigest()


def _nccl_link():
    """Link the NCCL that torch ships (nvidia-nccl wheel) when present, with an rpath to it:
    libnccl.so.2 is one soname, so whichever copy loads first serves the whole process, and
    torch's libtorch_cuda needs symbols the older system NCCL lacks (ncclDevCommCreate)."""
    d = os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}", "site-packages",
                     "nvidia", "nccl", "lib")
    if os.path.exists(os.path.join(d, "libnccl.so.2")):
        return ["-L" + d, "-l:libnccl.so.2", "-Xlinker", "-rpath," + d]
    return ["-lnccl"]


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    jobs = []
    for src, extra in SOURCES:
        if not os.path.exists(os.path.join(CSRC, src)):
            continue
        path, obj, cmd = _cmd(src, extra)
        stamp = obj + ".sha"
        dig = _digest(cmd, path)
        if not force and os.path.exists(obj) and os.path.exists(stamp) and open(stamp).read() == dig:
            continue
        jobs.append((src, obj, cmd, stamp, dig))

    def run(job):
        src, obj, cmd, stamp, dig = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-8000:]}")
        with open(os.path.join(OUT, src + ".ptxas.txt"), "w") as fh:
            fh.write(r.stderr)
        with open(stamp, "w") as fh:
            fh.write(dig)
        return src

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for s in ex.map(run, jobs):
            if verbose:
                print("compiled", s)
    objs = [os.path.join(OUT, s + ".o") for s, _ in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    link = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, *_nccl_link(), "-Xlinker", "-rpath,$ORIGIN"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stderr[-8000:])
    cli = [GXX, "-O2", os.path.join(CSRC, "lpsim_main.cpp"), "-o", CLI, "-L" + PKG, "-llp_b200",
           "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cli, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("CLI link failed:\n" + r.stderr[-8000:])
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
