#!/usr/bin/env python3
"""Summarise an ncu report (.ncu-rep) or a launch-list CSV into a compact table.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep          # --set full capture
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv  # gpu__time_duration list
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("dur_us", "gpu__time_duration.sum"),
    ("dram_rd_MB", "dram__bytes_read.sum"),
    ("dram_wr_MB", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("tc_rt_pct", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("sm_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("occ_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("regs", "launch__registers_per_thread"),
    ("grid", "launch__grid_size"),
    ("smem_KB", "launch__shared_mem_per_block_dynamic"),
]


def to_base(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3,
             "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}
    return x * scale.get(unit, 1)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    print("| kernel | " + " | ".join(k for k, _ in KEYS) + " |")
    print("|---" * (len(KEYS) + 1) + "|")
    for r in data:
        name = r[idx["Kernel Name"]].replace("(anonymous namespace)::", "")[:60]
        vals = []
        for k, m in KEYS:
            if m not in idx:
                vals.append("-")
                continue
            v = to_base(r[idx[m]], units[idx[m]])
            if k.endswith("_MB") and isinstance(v, float):
                v = v / 1e6
            if k == "smem_KB" and isinstance(v, float):
                v = v / 1024
            vals.append(f"{v:.1f}" if isinstance(v, float) else str(v))
        print(f"| {name} | " + " | ".join(vals) + " |")


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    i_name, i_val, i_unit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= i_val:
            continue
        name = r[i_name].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        name = name.split("<")[0] if "k_gemm_tc" not in name else r[i_name].split("(")[0].split("::")[-1]
        tot[name] += to_base(r[i_val], r[i_unit])
        cnt[name] += 1
    s = sum(tot.values())
    print("| kernel | launches | total us | avg us | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| {k} | {cnt[k]} | {v:.1f} | {v / cnt[k]:.2f} | {v / s:.3f} |")


def hot(path, kernel_substr, top=25):
    """Top SASS instructions by warp-stall samples for the first kernel matching kernel_substr."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    blocks = raw.split('"Kernel Name",')
    for b in blocks[1:]:
        name = b.split("\n", 1)[0]
        if kernel_substr not in name:
            continue
        rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
        hdr = rows[0]
        i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
        reasons = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        tot = sum(float(r[i_s] or 0) for r in rows[1:] if len(r) > i_s)
        print(name[:100], "total samples", tot)
        best = sorted(rows[1:], key=lambda r: -float(r[i_s] or 0) if len(r) > i_s else 0)[:top]
        for r in best:
            rs = sorted(((float(r[i] or 0), hdr[i]) for i in reasons), reverse=True)[:2]
            print(f"{float(r[i_s]) / tot:6.3f}  {r[i_src][:70]:70s} {rs}")
        return


if __name__ == "__main__":
    if sys.argv[1] == "--hot":
        hot(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[1])
