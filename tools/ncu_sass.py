"""Aggregate the ncu source page (SASS) of one kernel: executed instructions and
stall samples per opcode, plus the hottest instructions.
    python tools/ncu_sass.py rep.ncu-rep kernel-regex [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{pat}"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
si, ei, ni = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
by_op = collections.defaultdict(lambda: [0, 0])
allr = []
for r in rows[1:]:
    if len(r) <= max(si, ei, ni):
        continue
    src = r[si].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    try:
        ex, smp = int(r[ei] or 0), int(r[ni] or 0)
    except ValueError:
        continue
    by_op[op][0] += ex
    by_op[op][1] += smp
    allr.append((smp, ex, r[0], src))
tot_e = sum(v[0] for v in by_op.values()); tot_s = sum(v[1] for v in by_op.values())
print(f"total warp-instructions {tot_e}, samples {tot_s}")
for op, (e, s) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:30]:
    print(f"  {op:12s} exec {e:10d} ({100*e/max(1,tot_e):5.1f}%)  samples {s:6d} ({100*s/max(1,tot_s):5.1f}%)")
print("hottest:")
for smp, ex, addr, src in sorted(allr, reverse=True)[:top]:
    print(f"  {smp:6d} {ex:9d}  {src[:90]}")
