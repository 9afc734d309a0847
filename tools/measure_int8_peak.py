"""Measure the dense int8 tensor peak of this B200 (cuBLAS via torch._int_mm,
8192^3, 2*N^3 ops): best of 10 (burst) and back-to-back for 4 s (sustained).
Writes gpurun_out/int8_peak.json.  Context for the roofline only."""
import json
import os
import time

import torch

N = 8192
a = torch.randint(-128, 128, (N, N), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 128, (N, N), dtype=torch.int8, device="cuda")
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); torch._int_mm(a, b); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e) / 1e3)
burst = 2 * N ** 3 / best / 1e12
t0 = time.time(); it = 0
s = torch.cuda.Event(True); e = torch.cuda.Event(True); s.record()
while time.time() - t0 < 4.0:
    torch._int_mm(a, b); it += 1
    if it % 20 == 0:
        torch.cuda.synchronize()
e.record(); torch.cuda.synchronize()
sus = 2 * N ** 3 * it / (s.elapsed_time(e) / 1e3) / 1e12
out = {"int8_tops_burst": round(burst, 1), "int8_tops_sustained": round(sus, 1),
       "how": "torch._int_mm int8 8192^3 (cuBLAS), 2*N^3 ops; best of 10 and 4 s back to back",
       "gpu": torch.cuda.get_device_name(0)}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/int8_peak.json", "w"), indent=1)
print(json.dumps(out))
