"""Warp-stall samples and warp instructions executed per CUDA source line (inlined headers included) from an
.ncu-rep captured with --import-source on.
    python tools/ncu_lines.py rep.ncu-rep [kernel-regex] [top]"""
import collections, csv, io, os, subprocess, sys
rep = sys.argv[1]; pat = sys.argv[2] if len(sys.argv) > 2 else "."; top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + pat],
                     capture_output=True, text=True).stdout
samp, inst, text = collections.Counter(), collections.Counter(), {}
fname, line, hdr = "?", None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1]); continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        line = (fname, int(r[0])); text[line] = r[1].strip()[:80]; continue
    if line is None or r[4] in ("-", ""):
        continue
    samp[line] += int(r[4]); inst[line] += int(r[7] or 0)
ts, ti = sum(samp.values()), sum(inst.values())
print(f"samples {ts}  warp instructions {ti}")
for k, s in samp.most_common(top):
    print(f"{k[0]:>12s}:{k[1]:<5d} {100*s/ts:5.1f}% samp {100*inst[k]/ti:5.1f}% inst  {text.get(k, '')}")
