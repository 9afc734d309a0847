"""Run one config's conv a few times (for ncu captures): python tools/run_conv.py C2 [fused|staged] [reps]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synth
import paper_1901_01965_b200 as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
path = W.WINO_PATH_STAGED if (len(sys.argv) > 2 and sys.argv[2] == "staged") else W.WINO_PATH_FUSED
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
layer = synth.CONFIGS[cfg].layers[0]
x, w = synth.config_inputs(cfg)
conv = W.WinoConv2d(layer.n, layer.h, layer.w, layer.c_in, layer.c_out, layer.pad, W.WINO_NHWC, layer.scaling,
                    W.WINO_OUT_INT8, path=path)
conv.transform_filter(torch.from_numpy(w).cuda())
xd = torch.from_numpy(x).cuda()
S = synth.requant_shift(layer)
for _ in range(reps):
    y = conv(xd, 1, S)
torch.cuda.synchronize()
print("ok", cfg, "path", path, int(y.abs().sum()))
