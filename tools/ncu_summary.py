#!/usr/bin/env python3
"""Summarise an ncu --set full report into profiles/ (JSON + markdown).

usage: python tools/ncu_summary.py <report.ncu-rep | raw-page.csv> <out-prefix>
Writes <out-prefix>.json (per-kernel metrics, consumed by bench.py for roofline.traffic)
and <out-prefix>.md (human-readable table + top stall reasons).
"""
import csv
import io
import json
import subprocess
import sys

rep, prefix = sys.argv[1], sys.argv[2]
if rep.endswith(".csv"):  # a raw page exported on the GPU box (ncu -i rep --page raw --csv)
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_pct_peak": "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_bytes_per_s": "dram__bytes.sum.per_second",
    "fmaheavy_pct": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "alu_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "inst_executed": "smsp__inst_executed.sum",
}
SCALE = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0, "MB": 1e6, "GB": 1e9, "KB": 1e3,
         "B": 1.0, "msecond": 1e3, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "us": 1.0,
         "ns": 1e-3}


def val(r, key):
    i = idx.get(key)
    if i is None or r[i] in ("", "n/a"):
        return None
    try:
        v = float(r[i].replace(",", ""))
    except ValueError:  # "no data" etc.
        return None
    u = units[i]
    if key.startswith("dram__bytes"):
        v *= SCALE.get(u, 1.0)
    if key == "gpu__time_duration.sum":
        v *= SCALE.get(u, 1.0)
    return v


out = []
for r in data:
    d = {"kernel": r[idx["Kernel Name"]]}
    for k, m in KEYS.items():
        d[k] = val(r, m)
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    d["top_stalls"] = {n: round(v, 2) for v, n in sorted(stalls, reverse=True)[:6]}
    d["dram_bytes"] = (d["dram_read_bytes"] or 0) + (d["dram_write_bytes"] or 0)
    out.append(d)
json.dump({"report": rep, "kernels": out}, open(prefix + ".json", "w"), indent=1)
with open(prefix + ".md", "w") as fh:
    fh.write(f"# ncu --set full summary of `{rep}`\n\n")
    fh.write("| kernel | us | DRAM bytes | DRAM GB/s | fmaheavy % | alu % | issue % | warps % | regs | top stalls |\n")
    fh.write("|---|---|---|---|---|---|---|---|---|---|\n")
    for d in out:
        name = d["kernel"].split("(")[0].replace("void ", "")[-80:]
        f = lambda k, fmt: (format(d[k], fmt) if d.get(k) is not None else "-")
        fh.write(f"| `{name}` | {f('duration_us', '.1f')} | {d['dram_bytes']:.3e} | "
                 f"{d['dram_bytes'] / (d['duration_us'] or 1) / 1e3:.0f} | {f('fmaheavy_pct', '.1f')} | {f('alu_pct', '.1f')} | "
                 f"{f('issue_active_pct', '.1f')} | {f('warps_active_pct', '.1f')} | "
                 f"{f('registers', '.0f')} | "
                 + ", ".join(f"{k}={v}" for k, v in d["top_stalls"].items()) + " |\n")
print(open(prefix + ".md").read())
