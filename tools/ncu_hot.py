"""Top SASS instructions by warp-stall samples from an .ncu-rep source page.
    python tools/ncu_hot.py rep.ncu-rep [kernel-regex] [top]"""
import csv, io, re, subprocess, sys
rep = sys.argv[1]; pat = sys.argv[2] if len(sys.argv) > 2 else "."; top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + pat],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
si, ai, ei = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
body = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
tot = sum(int(r[si] or 0) for r in body)
print("total samples", tot, "instructions", len(body))
for idx, r in sorted(enumerate(body), key=lambda x: -int(x[1][si] or 0))[:top]:
    print(f"{idx:6d} {int(r[si] or 0):6d} {r[ei]:>8s}  {r[ai].strip()[:90]}")
