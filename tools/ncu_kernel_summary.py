"""Key metrics of every kernel in an ncu --set full report (for profiles/):
    python tools/ncu_kernel_summary.py rep.ncu-rep > out.txt"""
import csv, io, subprocess, sys

rep = sys.argv[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, units = rr[0], rr[1]
print(f"# ncu --set full ({rep}), --clock-control none")
for r in rr[2:]:
    print("## " + r[h.index("Kernel Name")][:100])
    for m in want:
        if m in h:
            i = h.index(m)
            print(f"   {m} = {r[i]} {units[i]}")
    stalls = {c: r[i] for i, c in enumerate(h) if c.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not c.endswith("_not_issued") and r[i] not in ("", "0")}
    top = sorted(stalls.items(), key=lambda kv: -float(kv[1]))[:6]
    print("   top stall samples: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v}" for k, v in top))
