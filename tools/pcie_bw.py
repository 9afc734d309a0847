"""PCIe copy bandwidth between pinned host memory and HBM: H2D alone, D2H alone, both concurrently
(two streams), for the C2 step's buffer size (6.4 MB)."""
import time
import torch

n = 56 * 56 * 64 * 32
reps = 50
h = [torch.empty(n, dtype=torch.int8).pin_memory() for _ in range(2)]
d = [torch.empty(n, dtype=torch.int8, device="cuda") for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d[0].copy_(h[0], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h[1].copy_(d[1], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


run(True, True)
a, b, c = run(True, False), run(False, True), run(True, True)
print(f"H2D {n / a / 1e9:.1f} GB/s  D2H {n / b / 1e9:.1f} GB/s  both {2 * n / c / 1e9:.1f} GB/s aggregate "
      f"({c * 1e6:.0f} us per pair)")
