"""Minimal C1 conv through the C ABI (for compute-sanitizer / debugging)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
import paper_1901_01965_b200 as W
cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
layer = synth.CONFIGS[cfg].layers[0]
x, w = synth.config_inputs(cfg, n=n)
conv = W.WinoConv2d(x.shape[0], layer.h, layer.w, layer.c_in, layer.c_out, 1, W.WINO_NHWC, True, W.WINO_OUT_INT32)
conv.transform_filter(torch.from_numpy(w).cuda())
y = conv(torch.from_numpy(x).cuda())
torch.cuda.synchronize()
print("ok", y.flatten()[:4].tolist())
