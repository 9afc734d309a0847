"""C5 per-layer timing inside the real sequence: a CUDA graph per layer (K1 + conv + pool as the stack runs
it), replayed 10 times alone, against the whole-step graph; shows where the step's time goes beyond the
per-kernel isolated timings.   python tools/c5_layers_r02.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import synth
from paper_1901_01965_b200 import _lib as L
from paper_1901_01965_b200.stack import ConvStack

cfg = synth.CONFIGS["C5"]
shifts = synth.stack_shifts("C5")
x, ws = synth.stack_inputs("C5")
st = ConvStack(x.shape[0], cfg.layers, cfg.pools_after, shifts, workspace_mb=int(os.environ.get("CHUNK_MB", "1024")))
xd = torch.from_numpy(x).cuda()
wd = [torch.from_numpy(w).cuda() for w in ws]
stream = torch.cuda.Stream()
sp = stream.cuda_stream
with torch.cuda.stream(stream):
    st.transform_filters(wd, stream)
    st(xd, stream)
    stream.synchronize()


def layer_launch(i, k1=True, conv=True, pool=True):
    c = st.convs[i]
    cur = xd if i == 0 else st.pooled.get(i - 1, st.outs[i - 1])
    if k1:
        L.wino_transform_filter(c.plan, wd[i].data_ptr(), c.w_wino.data_ptr(), c.codes.data_ptr(), sp)
    if conv:
        L.wino_conv2d_int8(c.plan, cur.data_ptr(), c.w_wino.data_ptr(), c.codes.data_ptr(), 1, shifts[i],
                           st.outs[i].data_ptr(), st.workspace.data_ptr(), sp)
    if pool and i in st.pooled:
        y = st.outs[i]
        nn, hh, ww_, cc = y.shape
        L.wino_maxpool2_int8(y.data_ptr(), nn, hh, ww_, cc, 1, st.pooled[i].data_ptr(), sp)


def timed(fn, reps=10):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        with torch.cuda.graph(g, stream=stream):
            for _ in range(reps):
                fn()
        g.replay()
        stream.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream); g.replay(); e1.record(stream); stream.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    return float(np.median(ts))


tot = timed(lambda: [layer_launch(i) for i in range(13)], reps=3)
print(f"whole step (13 x (K1 + conv + pool)): {tot:.0f} us")
s = 0.0
for i in range(13):
    a = timed(lambda: layer_launch(i))
    b = timed(lambda: layer_launch(i, k1=False, pool=False))
    p = timed(lambda: layer_launch(i, k1=False, conv=False)) if i in st.pooled else 0.0
    s += a
    print(f"layer {i + 1:2d}: K1+conv+pool {a:8.1f} us   conv alone {b:8.1f}   pool {p:6.1f}   chunks {st.convs[i].info.n_chunks}")
print(f"sum of layers {s:.0f} us vs whole step {tot:.0f} us")
