"""Per-kernel launches and time per step from an ncu --metrics gpu__time_duration.sum --csv launch list.
    python tools/launch_shares.py launches.csv [steps_in_capture]"""
import collections, csv, re, sys
path = sys.argv[1]; steps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
hdr = rows[0]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
t, n = collections.Counter(), collections.Counter()
for r in rows[1:]:
    if len(r) != len(hdr) or r[mi] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"^void ", "", r[ki]).split("<")[0].split("(")[0].split("::")[-1]
    unit_scale = 1e-3 if "ns" in hdr[vi + 0:vi + 1] else 1.0
    t[name] += float(r[vi].replace(",", "")); n[name] += 1
# gpu__time_duration is reported in ns or us depending on the ncu version: normalise by the unit column
ui = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
unit = next((r[ui] for r in rows[1:] if ui is not None and len(r) == len(hdr)), "us")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
tot = sum(t.values()) * scale / steps
print(f"# serialised per step: {tot:.1f} us")
print(f"{'kernel':40s} launches/step  us/step   share")
for k, v in t.most_common():
    print(f"{k:40s} {n[k] / steps:8.0f} {v * scale / steps:11.1f}  {v * scale / steps / tot:.3f}")
