import json, sys
d = json.load(open(sys.argv[1]))
print("value", d["value"], d["unit"], "ms/step", d["ms_per_step"], "launches", d["gpu_launches"], "clocks", d.get("clocks"))
for k, v in d["kernels"].items():
    print(f"  {k:10s} {v['us_per_launch']:8.2f} us x{v['launches_per_step']}  share {v['share_of_step']:.3f}  "
          f"{v['achieved']} {v['unit']} frac {v['frac']}" + (f"  hbm_view {v['hbm_view']}" if 'hbm_view' in v else ""))
print("  e2e", d["e2e"])
if "cpu_baseline" in d: print("  cpu", d["cpu_baseline"])
