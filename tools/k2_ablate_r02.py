"""K2 (NHWC int8 SWAR input transform) ablation on C2-shaped layers of growing batch (V from L2-resident to
HBM-sized): stage-2 launch time with WINO_K2_DBG = 0 full, 1 no V stores, 2 no x loads, 3 neither
(debug build -DWINO_K2_DBG).   python tools/k2_ablate_r02.py <batch>"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import paper_1901_01965_b200 as W
from paper_1901_01965_b200 import _lib as L

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
conv = W.WinoConv2d(n, 56, 56, 64, 64, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8, path=W.WINO_PATH_FUSED, workspace_mb=4096)
rng = np.random.default_rng(1)
x = torch.from_numpy(rng.integers(-128, 128, (n, 56, 56, 64)).astype(np.int8)).cuda()
wt = torch.from_numpy(rng.integers(-60, 60, (64, 3, 3, 64)).astype(np.int8)).cuda()
conv.transform_filter(wt)
y = conv(x, 1, 10)
st = torch.cuda.Stream()
sp = st.cuda_stream
reps = 20
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    with torch.cuda.graph(g, stream=st):
        for _ in range(reps):
            L.wino_conv2d_int8_stage(conv.plan, 2, 0, x.data_ptr(), conv.w_wino.data_ptr(), conv.codes.data_ptr(), 1,
                                     10, y.data_ptr(), conv.workspace.data_ptr(), sp)
    g.replay()
    st.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); g.replay(); e1.record(st); st.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
t = float(np.median(ts))
vb = conv.info.v_bytes
print(f"batch {n}: chunks {conv.info.n_chunks}, V {vb / 2**20:.0f} MiB, K2 {t:.1f} us, "
      f"x + V {(x.numel() + vb) / t / 1e3:.0f} GB/s  dbg={os.environ.get('WINO_K2_DBG', '0')}")
