"""Timeline of the fused kernel (build with WINO_NVCC_FLAGS=-DWINO_FUSED_TRACE):
    python tools/trace_fused.py C2 [cta]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import synth
import paper_1901_01965_b200 as W
from paper_1901_01965_b200 import _lib as L

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
cta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
layer = synth.CONFIGS[cfg].layers[0]
x, w = synth.config_inputs(cfg)
conv = W.WinoConv2d(layer.n, layer.h, layer.w, layer.c_in, layer.c_out, layer.pad, W.WINO_NHWC, layer.scaling,
                    W.WINO_OUT_INT8, path=W.WINO_PATH_FUSED)
conv.transform_filter(torch.from_numpy(w).cuda())
xd = torch.from_numpy(x).cuda()
S = synth.requant_shift(layer)
y = conv(xd, 1, S); y = conv(xd, 1, S)
buf = torch.zeros(148 * 96 * 4, dtype=torch.int64, device="cuda")
L.lib().wino_debug_set_trace(buf.data_ptr())
conv(xd, 1, S)
torch.cuda.synchronize()
L.lib().wino_debug_set_trace(None)
t = buf.cpu().numpy().reshape(148, 96, 4)[cta].astype(np.float64)
t0 = t[t > 0].min()
ns = lambda v: f"{(v - t0):8.0f}" if v > 0 else "       -"
print("stage: producer_issued  mma_saw_data  mma_committed  (SM cycles from the first event)")
for i in range(64):
    if t[i, 0] > 0:
        print(f"  st{i:2d}: {ns(t[i,0])} {ns(t[i,1])} {ns(t[i,2])}")
print("slot-group: mma_got_slot  epi_saw_acc  epi_released")
for i in range(32):
    if t[64 + i, 0] > 0:
        print(f"  sg{i:2d}: {ns(t[64+i,0])} {ns(t[64+i,1])} {ns(t[64+i,2])}")
print("unit end (warp 0): last slot taken, Y formed, barrier 1 passed, rows staged, barrier 2 passed, stored")
for u in range(4):
    row = t[u * 8: u * 8 + 6, 3]
    if row[0] > 0:
        print(f"  unit {u}: " + " ".join(ns(v) for v in row))
