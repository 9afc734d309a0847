"""One line per bench JSON: value, ms/step, per-kernel us, roofline frac, self-check.
    python tools/brief_r02.py <bench json files>"""
import json
import signal
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)

for f in sys.argv[1:]:
    try:
        d = json.loads([l for l in open(f).read().splitlines() if l.startswith("{")][-1])
    except Exception as e:  # noqa: BLE001
        print(f, "n/a", e)
        continue
    ks = d.get("kernels") or {}
    kt = " ".join(f"{k}={v['us_per_launch']:.1f}" for k, v in ks.items())
    sc = (d.get("self_check") or {}).get("equal_to_oracle")
    lay = d.get("layers_kernels_us")
    print(f"{f}: {d['value']:.1f} TOPS {d['ms_per_step']} ms frac={d['roofline']['frac']} ({d['roofline']['kernel']}) "
          f"path_frac={d['path_roofline']['frac']} self_check={sc} {kt}")
    if lay:
        print("   layers:", " | ".join(" ".join(f"{k[:4]}={v:.0f}" for k, v in l.items()) for l in lay))
