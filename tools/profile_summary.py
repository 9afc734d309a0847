"""Write a per-round profile summary for profiles/:
    python tools/profile_summary.py <launches.csv> <a.ncu-rep[,b.ncu-rep..]> <bench.json> <out.txt> [traffic.json]
Launch-list per-step shares (cold, serialised ncu durations x launches per
step) beside the bench line's live shares, full-capture metrics (duration,
DRAM bytes, throughputs, tensor pipe, stalls) per kernel, and optionally a
traffic JSON {bench kernel key: dram read+write bytes per launch} that
bench.py reports as roofline.traffic."""
import collections
import csv
import io
import json
import subprocess
import sys

launches, reps, bench, out = sys.argv[1:5]
traffic_out = sys.argv[5] if len(sys.argv) > 5 else None
KEYS = {"k_filter": "k1_filter", "k_input": "k2_input", "k_gemm": "k3_gemm", "k_output": "k4_output",
        "k_fused": "k3_fused"}


def bench_key(name):
    for k, v in KEYS.items():
        if k in name:
            return v
    return None


d = json.load(open(bench))
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
        rec = dict(zip(hdr, r))
        if rec.get("Metric Name") == "gpu__time_duration.sum":
            agg[rec["Kernel Name"].split("(")[0].replace("void ", "")].append(float(rec["Metric Value"]))
per_step = {k: sum(v) / len(v) * d["kernels"][bench_key(k)]["launches_per_step"]
            for k, v in agg.items() if bench_key(k)}
tot = sum(per_step.values())
P(f"# ncu launch list ({launches}): gpu__time_duration.sum, --clock-control none, cold cache, serialised")
P("# share = avg launch x launches per step / sum over kernels (compare with the live share)")
P(f"{'kernel':40s} {'launches':>8s} {'avg us':>9s} {'share':>7s} {'live us':>8s} {'live share':>10s}")
for k, v in sorted(agg.items(), key=lambda kv: -per_step.get(kv[0], 0)):
    if not bench_key(k):
        continue
    lv = d["kernels"][bench_key(k)]
    P(f"{k:40s} {len(v):8d} {sum(v) / len(v) / 1e3:9.2f} {per_step[k] / tot:7.3f} {lv['us_per_launch']:8.2f} "
      f"{lv['share_of_step']:10.3f}")

want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
traffic, seen = {}, set()
for rep in reps.split(","):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h, units = rr[0], rr[1]
    P("")
    P(f"# ncu --set full ({rep}), --clock-control none")
    for r in rr[2:]:
        name = r[h.index("Kernel Name")]
        key = bench_key(name)
        if key in seen:
            continue
        seen.add(key)
        P("## " + name[:90])
        for m in want:
            if m in h:
                i = h.index(m)
                P(f"   {m} = {r[i]} {units[i]}")
        if key and "dram__bytes_read.sum" in h:
            ir, iw = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
            traffic[key] = int(float(r[ir]) * SCALE[units[ir]] + float(r[iw]) * SCALE[units[iw]])
            P(f"   traffic (dram read + write) = {traffic[key]} B per launch")
        stalls = {c: r[i] for i, c in enumerate(h) if c.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not c.endswith("_not_issued") and r[i] not in ("", "0")}
        top = sorted(stalls.items(), key=lambda kv: -float(kv[1]))[:6]
        P("   top stall samples: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')}={v}"
                                              for k, v in top))
P("")
P(f"# bench.py live numbers ({bench}): value {d['value']} {d['unit']}, {d['ms_per_step']} ms/step")
for k, v in d["kernels"].items():
    P(f"   {k}: {v['us_per_launch']} us x{v['launches_per_step']}, share {v['share_of_step']}, "
      f"{v['achieved']} {v['unit']} = {v['frac']} of {v['peak']}")
open(out, "w").write("\n".join(lines) + "\n")
if traffic_out:
    json.dump({"source": reps, "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch from ncu --set full "
               "(cold L2; writes still resident in L2 when the kernel ends are not counted)", "bytes": traffic},
              open(traffic_out, "w"), indent=1)
print("\n".join(lines))
