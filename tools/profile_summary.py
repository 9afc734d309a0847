"""Write a per-round profile summary for profiles/:
    python tools/profile_summary.py <launches.csv> <full.ncu-rep> <bench.json> <out.txt>
Launch-list shares (cold, serialised ncu durations), full-capture metrics
(duration, DRAM bytes, throughputs, tensor pipe, stalls) per kernel, and the
bench line's live per-kernel numbers for comparison."""
import collections
import csv
import io
import json
import subprocess
import sys

launches, rep, bench, out = sys.argv[1:5]
lines = []
P = lines.append

rows = list(csv.reader(open(launches)))
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            agg[d["Kernel Name"].split("(")[0].replace("void ", "")].append(float(d["Metric Value"]))
tot = sum(sum(v) for k, v in agg.items() if "wino" in k)
P(f"# ncu launch list ({launches}): gpu__time_duration.sum, --clock-control none, cold cache, serialised")
P(f"{'kernel':45s} {'launches':>8s} {'avg us':>9s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    if "wino" not in k:
        continue
    P(f"{k:45s} {len(v):8d} {sum(v) / len(v) / 1e3:9.2f} {sum(v) / tot:7.3f}")

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, units = rr[0], rr[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]
P("")
P(f"# ncu --set full ({rep}), one launch per kernel, --clock-control none")
for r in rr[2:]:
    P("## " + r[h.index("Kernel Name")][:90])
    for m in want:
        if m in h:
            i = h.index(m)
            P(f"   {m} = {r[i]} {units[i]}")
    stalls = {c: r[i] for i, c in enumerate(h) if c.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not c.endswith("_not_issued") and r[i] not in ("", "0")}
    top = sorted(stalls.items(), key=lambda kv: -float(kv[1]))[:6]
    P("   top stall samples: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v}" for k, v in top))
d = json.load(open(bench))
P("")
P(f"# bench.py live numbers ({bench}): value {d['value']} {d['unit']}, {d['ms_per_step']} ms/step")
for k, v in d["kernels"].items():
    P(f"   {k}: {v['us_per_launch']} us x{v['launches_per_step']}, share {v['share_of_step']}, "
      f"{v['achieved']} {v['unit']} = {v['frac']} of {v['peak']}")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
