"""Per-layer A/B of the two kernel paths on one stream (CUDA graph of whole convs, K1 included):
    python tools/path_ab.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1901_01965_b200 as W


def t_conv(n, h, w, ci, co, path, reps=20):
    conv = W.WinoConv2d(n, h, w, ci, co, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8, path=path)
    rng = np.random.default_rng(2)
    x = torch.from_numpy(rng.integers(-128, 128, (n, h, w, ci)).astype(np.int8)).cuda()
    wt = torch.from_numpy(rng.integers(-60, 60, (co, 3, 3, ci)).astype(np.int8)).cuda()
    y = torch.empty(conv.y_shape, dtype=torch.int8, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        conv.transform_filter(wt, st); conv(x, 1, 10, y=y, stream=st)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                conv.transform_filter(wt, st); conv(x, 1, 10, y=y, stream=st)
        g.replay(); st.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st); g.replay(); e1.record(st); st.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    ops = 2 * n * h * w * ci * co * 9
    return float(np.median(ts)), ops


SHAPES = [(32, 56, 56, 64, 64), (64, 28, 28, 128, 128), (32, 56, 56, 64, 128), (32, 56, 56, 128, 128),
              (16, 56, 56, 128, 256), (64, 28, 28, 128, 256), (64, 28, 28, 256, 128), (128, 14, 14, 256, 256),
              (8, 112, 112, 64, 128), (8, 112, 112, 128, 128), (64, 28, 28, 256, 512), (64, 28, 28, 512, 512),
              (256, 14, 14, 512, 512)]
if len(sys.argv) > 1:   # e.g. python tools/path_ab.py fused 64,28,28,512,512 256,14,14,512,512
    paths = {"fused": W.WINO_PATH_FUSED, "staged": W.WINO_PATH_STAGED}
    for sh in sys.argv[2:]:
        shape = tuple(int(v) for v in sh.split(","))
        t, ops = t_conv(*shape, paths[sys.argv[1]])
        print(f"{shape}: {sys.argv[1]} {ops / t / 1e6:7.1f} TOPS (one stream)")
    sys.exit(0)
for shape in SHAPES:
    r = {}
    for name, p in (("fused", W.WINO_PATH_FUSED), ("staged", W.WINO_PATH_STAGED)):
        t, ops = t_conv(*shape, p)
        r[name] = ops / t / 1e6
    print(f"{shape}: fused {r['fused']:7.1f}  staged {r['staged']:7.1f} TOPS (one stream)")
