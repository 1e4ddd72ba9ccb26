"""Summarise ncu outputs into profiles/ (tracked):
  - a launch list (--metrics gpu__time_duration.sum) -> per-kernel share of device time
  - a --set full report -> per-kernel duration, DRAM bytes, tensor-pipe / MUFU / DRAM utilisation

usage: python scripts/ncu_summary.py <launches.csv> <report.ncu-rep> <tag>
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict


def short(name):
    return name.split("(")[0].replace("void ", "")


def launches(path):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        k = short(r[ki])
        tot[k] += float(r[vi].replace(",", "")) * (scale.get(r[ui].strip().lower(), 1.0) if ui is not None else 1.0)
        cnt[k] += 1
    s = sum(tot.values())
    return {k: {"launches": cnt[k], "ns": tot[k], "share": tot[k] / s} for k in sorted(tot, key=lambda x: -tot[x])}


METRICS = {
    "duration_ms": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    # tcgen05-aware: bf16->fp32 UTCHMMA tensor ops (the kind::f16 MMAs of the GEMM and attention,
    # 1-CTA and CTA-pair alike) against their peak; the legacy pipe_tensor metric undercounts
    # cta_group::2 UTCHMMA and is kept only for comparison
    "utchmma_bf16_pct_of_peak": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.avg.pct_of_peak_sustained_elapsed",
    "utchmma_bf16_ops": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum",
    "tensor_pipe_active_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "mufu_xu_pct_active": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct_active": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "registers": "launch__registers_per_thread",
}


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")]), "grid": r[hdr.index("Grid Size")] if "Grid Size" in hdr else ""}
        for k, m in METRICS.items():
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                try:
                    x = float(v)
                except ValueError:
                    d[k] = v
                    continue
                # ncu auto-scales units per metric (the second CSV row): normalise to ms / MB
                u = units[hdr.index(m)].strip().lower()
                if k == "duration_ms":
                    x *= {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3,
                          "second": 1e3}.get(u, 1.0)
                elif k.endswith("_MB"):
                    x *= {"byte": 1e-6, "kbyte": 1e-3, "mbyte": 1.0, "gbyte": 1e3, "tbyte": 1e6}.get(u, 1.0)
                d[k] = x
        res.append(d)
    return res


if __name__ == "__main__":
    lpath, rpath, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    os.makedirs("profiles", exist_ok=True)
    summary = {"launch_list": launches(lpath) if os.path.exists(lpath) else {},
               "full": full(rpath) if os.path.exists(rpath) else []}
    json.dump(summary, open(f"profiles/{tag}_ncu.json", "w"), indent=1)
    with open(f"profiles/{tag}_ncu.md", "w") as f:
        f.write(f"# ncu summary — {tag}\n\n## Launch list (cold-cache, serialised; compare shares)\n\n")
        f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k, v in summary["launch_list"].items():
            f.write(f"| {k} | {v['launches']} | {v['ns'] / 1e6:.3f} | {100 * v['share']:.1f}% |\n")
        f.write("\n## `--set full` captures\n\n| kernel | " + " | ".join(METRICS) + " |\n|" + "---|" * (len(METRICS) + 1) + "\n")
        for d in summary["full"]:
            f.write(f"| {d['kernel']} | " + " | ".join(str(d.get(k, "")) for k in METRICS) + " |\n")
    print(open(f"profiles/{tag}_ncu.md").read())
