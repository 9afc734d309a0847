"""Summarise an .ncu-rep: per kernel, the key metrics of the details page and
the top stall reasons from the source page.
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Registers Per Thread", "Achieved Occupancy", "Issued Warp Per Scheduler", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Dynamic Shared Memory Per Block",
        "Grid Size", "Block Size", "Mem Busy", "Max Bandwidth", "L1/TEX Hit Rate", "L2 Hit Rate"]


def details(rep, pat):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki, ni, vi, ui, ii = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                          hdr.index("Metric Unit"), hdr.index("ID"))
    seen = {}
    for r in rows[1:]:
        if not re.search(pat, r[ki]):
            continue
        key = (r[ii], r[ki][:60])
        seen.setdefault(key, [])
        if any(r[ni].startswith(k) for k in KEYS):
            seen[key].append(f"{r[ni]} = {r[vi]} {r[ui]}")
    for (i, k), ms in seen.items():
        print(f"=== [{i}] {k}")
        for m in ms:
            print("   ", m)


def raw(rep, pat, metrics):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    for r in rows[2:]:
        if not re.search(pat, r[hdr.index("Kernel Name")]):
            continue
        print("---", r[hdr.index("Kernel Name")][:60])
        for m in metrics:
            cols = [i for i, h in enumerate(hdr) if re.fullmatch(m, h)]
            for c in cols:
                print(f"    {hdr[c]} = {r[c]} {rows[1][c]}")


if __name__ == "__main__":
    rep = sys.argv[1]
    pat = sys.argv[2] if len(sys.argv) > 2 else "."
    details(rep, pat)
    raw(rep, pat, [r"dram__bytes_(read|write)\.sum", r"smsp__pcsamp_warps_issue_stalled_\w+",
                   r"sm__pipe_tensor\w*cycles_active\.avg\.pct_of_peak_sustained_active",
                   r"sm__inst_executed_pipe_\w+\.avg\.pct_of_peak_sustained_active"])
