"""K3F time per unit as a function of the cout count (V re-reads per tile block = cout / 16) and of the
number of concurrently running CTAs: C2's tiles (32 x 56 x 56, c_in 64), c_out 16..64, and the same
problem with fewer images.   python tools/fused_scaling.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1901_01965_b200 as W
from paper_1901_01965_b200 import _lib as L


def time_k3f(n, h, w, ci, co, reps=30):
    conv = W.WinoConv2d(n, h, w, ci, co, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8, path=W.WINO_PATH_FUSED)
    rng = np.random.default_rng(1)
    x = torch.from_numpy(rng.integers(-128, 128, (n, h, w, ci)).astype(np.int8)).cuda()
    wt = torch.from_numpy(rng.integers(-60, 60, (co, 3, 3, ci)).astype(np.int8)).cuda()
    conv.transform_filter(wt)
    y = conv(x, 1, 10)
    st = torch.cuda.Stream(); sp = st.cuda_stream
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps):
                L.wino_conv2d_int8_stage(conv.plan, 3, 0, x.data_ptr(), conv.w_wino.data_ptr(), conv.codes.data_ptr(),
                                         1, 10, y.data_ptr(), conv.workspace.data_ptr(), sp)
        g.replay(); st.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st); g.replay(); e1.record(st); st.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    tiles = n * ((h + 3) // 4) * ((w + 3) // 4)
    units = ((tiles + 127) // 128) * ((co + 15) // 16)
    return float(np.median(ts)), units


for (n, co) in [(32, 16), (32, 32), (32, 64), (16, 64), (8, 64), (4, 64), (2, 64)]:
    t, u = time_k3f(n, 56, 56, 64, co)
    grid_rounds = -(-u // 148)
    print(f"n={n:2d} c_out={co:2d}: units {u:4d}, rounds {grid_rounds}, K3F {t:7.2f} us, per unit-round {t / grid_rounds:6.2f} us")
