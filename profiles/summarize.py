"""Summarise ncu outputs into markdown for profiles/ (run here, no GPU needed).

  python profiles/summarize.py launches gpurun_out/launches.csv > profiles/rNN_launches.md
  python profiles/summarize.py kernel gpurun_out/prof.ncu-rep   > profiles/rNN_<kernel>.md
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Compute (SM) Throughput", "Issue Slots Busy", "Executed Instructions",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Theoretical Active Warps per SM",
        "Achieved Active Warps Per SM", "No Eligible", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "lts__t_sectors_srcunit_tex_op_read.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    k = collections.OrderedDict()
    for r in rows[hi + 1:]:
        k.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
    out = ["| id | kernel | time (ms) | DRAM read (GB) | DRAM write (GB) | DRAM GB/s |", "|---|---|---|---|---|---|"]
    tot = collections.Counter()
    for (i, name), m in k.items():
        if name.startswith("void at::") or "at_cuda_detail" in name:
            continue  # torch's own setup kernels
        t = m.get("gpu__time_duration.sum", 0.0) / 1e6
        rd = m.get("dram__bytes_read.sum", 0.0) / 1e9
        wr = m.get("dram__bytes_write.sum", 0.0) / 1e9
        short = name.split("(")[0].replace("void ", "")[:70]
        tot[short] += t
        bw = (rd + wr) / (t * 1e-3) if t else 0.0
        out.append(f"| {i} | `{short}` | {t:.3f} | {rd:.2f} | {wr:.2f} | {bw:.0f} |")
    out.append("")
    out.append("Per kernel (summed over launches): " + ", ".join(f"`{k}` {v:.2f} ms" for k, v in tot.most_common()))
    return "\n".join(out)


def kernel(path: str) -> str:
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    ii, ki, mi, vi, ui = (h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"))
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    out = []
    by_id = collections.OrderedDict()
    for r in rows[1:]:
        by_id.setdefault(r[ii], []).append(r)
    for n, (kid, krows) in enumerate(by_id.items()):
        out.append(f"\n### kernel `{krows[0][ki][:150]}`\n")
        out.append("| metric | value |")
        out.append("|---|---|")
        seen = set()
        for r in krows:
            if r[mi] in KEYS and r[mi] not in seen:
                seen.add(r[mi])
                out.append(f"| {r[mi]} | {r[vi]} {r[ui]} |")
        if len(rr) > 2 + n:
            hdr, units, vals = rr[0], rr[1], rr[2 + n]
            for m in RAW:
                if m in hdr:
                    j = hdr.index(m)
                    out.append(f"| {m} | {vals[j]} {units[j]} |")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else kernel(path))
