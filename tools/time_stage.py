"""Time one stage of the conv (CUDA graph of back-to-back launches):
    python tools/time_stage.py C2 [fused|staged] [stage] [reps]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
import paper_1901_01965_b200 as W
from paper_1901_01965_b200 import _lib as L

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
path = W.WINO_PATH_STAGED if (len(sys.argv) > 2 and sys.argv[2] == "staged") else W.WINO_PATH_FUSED
stage = int(sys.argv[3]) if len(sys.argv) > 3 else 3
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 50
layer = synth.CONFIGS[cfg].layers[0]
x, w = synth.config_inputs(cfg)
conv = W.WinoConv2d(layer.n, layer.h, layer.w, layer.c_in, layer.c_out, layer.pad, W.WINO_NHWC, layer.scaling,
                    W.WINO_OUT_INT8, path=path)
wdv = torch.from_numpy(w).cuda()
conv.transform_filter(wdv)
xd = torch.from_numpy(x).cuda()
S = synth.requant_shift(layer)
y = conv(xd, 1, S)
st = torch.cuda.Stream()
sp = st.cuda_stream
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(st):
    with torch.cuda.graph(g, stream=st):
        for r in range(reps):
            if stage == 1:
                L.wino_transform_filter(conv.plan, wdv.data_ptr(), conv.w_wino.data_ptr(), conv.codes.data_ptr(), sp)
            else:
                L.wino_conv2d_int8_stage(conv.plan, stage, 0, xd.data_ptr(), conv.w_wino.data_ptr(),
                                         conv.codes.data_ptr(), 1, S, y.data_ptr(), conv.workspace.data_ptr(), sp)
    g.replay()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); g.replay(); e1.record(st); st.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
print(f"{cfg} path={path} stage={stage} dbg={os.environ.get('WINO_FUSED_DBG', '0')}: {sorted(ts)[2]:.2f} us/launch")
