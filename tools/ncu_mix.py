"""Dynamic SASS opcode mix (warp instructions executed per opcode) from an .ncu-rep source page.
    python tools/ncu_mix.py rep.ncu-rep [kernel-regex] [top]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]; pat = sys.argv[2] if len(sys.argv) > 2 else "."; top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + pat],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hdr_i]
ai, ei = hdr.index("Source"), hdr.index("Instructions Executed")
body = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
mix = collections.Counter()
for r in body:
    toks = r[ai].split()
    op = next((t for t in toks if not t.startswith("@")), "?").split(".")[0]
    mix[op] += int(r[ei] or 0)
tot = sum(mix.values())
print("total warp instructions", tot)
for op, n in mix.most_common(top):
    print(f"{op:10s} {n:12d} {100 * n / tot:6.2f} %")
