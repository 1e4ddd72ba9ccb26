"""K1 (partition gather) and K10 (reconstruct + sampler update) micro-benchmark at the BASELINE
latent sizes: per-launch device time, achieved algorithmic GB/s and fraction of the measured HBM
copy bandwidth.  Two timings per kernel: `*_us` = 64 back-to-back launches over 8 private
buffer copies used round robin (working set > L2), captured in one CUDA graph so host launch
gaps do not count (bench.py's engine replay does the same from C++), and `*_flush_us` = one launch between L2 flushes, CUDA events around it (~2 us event
granularity: an upper bound).

Algorithmic bytes: K1 = 2 * shard elements * b; K10 = (sum of shard elements +
2 * latent elements) * b (every prediction read once, z read and written).

usage: python scripts/hbm_bench.py [dtype_bytes=4]  ->  gpurun_out/hbm_bench.json
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2512_07350_b200 import _lib, lp  # noqa: E402

L = _lib.lib()
PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6452.5
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731
DT = {2: torch.int16, 4: torch.float32, 8: torch.float64}


def timed(fn, reps=20):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


SETS, ITERS = 8, 64


def replay(fn):
    """Per-launch ms of ITERS back-to-back launches fn(i % SETS), captured in one CUDA graph (no
    host launch gaps between these few-us kernels), one event pair around the graph replay."""
    for i in range(SETS):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(ITERS):
            fn(i % SETS)
    g.replay()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / ITERS


def case(name, dims, K, r, d):
    out = []
    n = 1
    for x in dims:
        n *= x
    zs = []
    for _ in range(SETS):
        zs.append(torch.randn(n, device="cuda").to(DT[d]) if d != 2 else
                  torch.randint(0, 0x3b00, (n,), device="cuda", dtype=torch.int16))
    z = zs[0]
    for step, axis in ((1, "T"), (2, "H"), (3, "W")):
        plan = lp.build_plan(dims, (1, 2, 2), step, K, r)
        subs = [plan.sub_shape(dims, k) for k in range(plan.workers)]
        vols = [s[0] * s[1] * s[2] * s[3] for s in subs]
        packs = []
        for _ in range(SETS):
            packed = torch.empty(sum(vols), device="cuda", dtype=DT[d])
            if d == 2:
                packed.copy_(torch.randint(0, 0x3b00, (sum(vols),), device="cuda", dtype=torch.int16))
            else:
                packed.normal_()
            packs.append(packed)
        packed = packs[0]
        shape = _lib.i64arr(dims)
        ex = lambda i: _lib.check(L.lp_extract(C.byref(plan.raw), 0, plan.workers, C.c_void_p(zs[i].data_ptr()),  # noqa: E731
                                               shape, d, C.c_void_p(packs[i].data_ptr()), st()))
        ru = lambda i, fast: _lib.check(L.lp_reconstruct_update(C.byref(plan.raw), C.c_void_p(packs[i].data_ptr()),  # noqa: E731
                                                               shape, d, fast, C.c_double(1e-30),
                                                               C.c_void_p(zs[i].data_ptr()), st()))
        k1r, k10r, k10fr = replay(ex), replay(lambda i: ru(i, 0)), replay(lambda i: ru(i, 1))
        # K1: gather every entry (one launch for all entries, as the engine does for its owned run)
        k1 = timed(lambda: _lib.check(L.lp_extract(C.byref(plan.raw), 0, plan.workers, C.c_void_p(z.data_ptr()), shape, d,
                                                   C.c_void_p(packed.data_ptr()), st())))
        k1_bytes = 2.0 * sum(vols) * d
        k10 = timed(lambda: _lib.check(L.lp_reconstruct_update(C.byref(plan.raw), C.c_void_p(packed.data_ptr()), shape, d, 0,
                                                              C.c_double(1e-30), C.c_void_p(z.data_ptr()), st())))
        k10_bytes = (sum(vols) + 2.0 * n) * d
        k10f = timed(lambda: _lib.check(L.lp_reconstruct_update(C.byref(plan.raw), C.c_void_p(packed.data_ptr()), shape, d, 1,
                                                               C.c_double(1e-30), C.c_void_p(z.data_ptr()), st())))
        row = {"config": name, "axis": axis, "K": K, "dtype_bytes": d, "latent_elems": n, "shard_elems": sum(vols),
               "k1_us": k1r * 1e3, "k1_GBps": k1_bytes / k1r / 1e6, "k1_frac": k1_bytes / k1r / 1e6 / PEAK,
               "k10_us": k10r * 1e3, "k10_GBps": k10_bytes / k10r / 1e6, "k10_frac": k10_bytes / k10r / 1e6 / PEAK,
               "k10_fast_us": k10fr * 1e3, "k10_fast_frac": k10_bytes / k10fr / 1e6 / PEAK,
               "k1_flush_us": k1 * 1e3, "k10_flush_us": k10 * 1e3, "k10_fast_flush_us": k10f * 1e3,
               "k1_bytes": k1_bytes, "k10_bytes": k10_bytes}
        print(json.dumps(row), flush=True)
        out.append(row)
    return out


def ncu_pass(d):
    """HB_NCU=1: each kernel once per C2 axis (K1, K10 exact, K10 fast), for ncu --set full."""
    dims, n = (16, 21, 60, 104), 16 * 21 * 60 * 104
    z = torch.randn(n, device="cuda").to(DT[d])
    shape = _lib.i64arr(dims)
    for step in (1, 2, 3):
        plan = lp.build_plan(dims, (1, 2, 2), step, 4, 0.5)
        vols = [s[0] * s[1] * s[2] * s[3] for s in (plan.sub_shape(dims, k) for k in range(plan.workers))]
        packed = torch.randn(sum(vols), device="cuda").to(DT[d])
        _lib.check(L.lp_extract(C.byref(plan.raw), 0, plan.workers, C.c_void_p(z.data_ptr()), shape, d,
                                C.c_void_p(packed.data_ptr()), st()))
        for fast in (0, 1):
            _lib.check(L.lp_reconstruct_update(C.byref(plan.raw), C.c_void_p(packed.data_ptr()), shape, d, fast,
                                               C.c_double(1e-30), C.c_void_p(z.data_ptr()), st()))
    torch.cuda.synchronize()


def main():
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    if os.environ.get("HB_NCU") == "1":
        return ncu_pass(d)
    rows = []
    rows += case("C2", (16, 21, 60, 104), 4, 0.5, d)
    rows += case("C4", (16, 21, 90, 160), 8, 0.5, d)
    rows += case("C5", (16, 41, 60, 104), 8, 0.5, d)
    tag = os.environ.get("HB_TAG", "")
    json.dump({"peak_GBps": PEAK, "rows": rows}, open(f"gpurun_out/hbm_bench{tag}.json", "w"), indent=1)


if __name__ == "__main__":
    main()
