"""Small runs of every kernel structure for compute-sanitizer (memcheck / racecheck / synccheck):
C1 and a two-tile-block case (3 images of 32 x 32 = 192 tiles: a full and a partial block of 128) on the fused
and staged complex F(4x4) paths (int8 and int32 output, the fused pool mode, two chunk lanes), the rational
F(2x2) paths, uint8 input, the int8-native target, the VGG pool kernel; each result checked against the oracle.
    compute-sanitizer --tool memcheck python tools/sanitize_r02.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import synth
import paper_1901_01965_b200 as W
from oracle import oracle as O

rng = np.random.default_rng(3)
cases = []
x1, w1 = synth.config_inputs("C1", O.NHWC)
cases.append(("C1", x1, w1))
x2, w2 = synth.random_layer(rng, 3, 32, 32, 40, 32, O.NHWC)   # 3 x 64 tiles = 192: two tile blocks of 128
cases.append(("2blocks", x2, w2))
ok = True
for name, x, w in cases:
    n, h, wd, ci = x.shape
    co = w.shape[0]
    xd, wdv = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    ref32 = O.wino_conv(x, w, 1, O.NHWC, True).out32
    ref8 = O.wino_conv(x, w, 1, O.NHWC, True, M0=1, S=8).y8
    for path in (W.WINO_PATH_FUSED, W.WINO_PATH_STAGED):
        c = W.WinoConv2d(n, h, wd, ci, co, 1, W.WINO_NHWC, True, W.WINO_OUT_INT32, path=path)
        c.transform_filter(wdv)
        ok &= np.array_equal(c(xd).cpu().numpy(), ref32)
        c = W.WinoConv2d(n, h, wd, ci, co, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8, path=path, workspace_mb=1, lanes=2)
        c.transform_filter(wdv)
        ok &= np.array_equal(c(xd, 1, 8).cpu().numpy(), ref8)
        if co % 16 == 0:
            c = W.WinoConv2d(n, h, wd, ci, co, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8_POOL2, path=path)
            c.transform_filter(wdv)
            ok &= np.array_equal(c(xd, 1, 8).cpu().numpy(), O.maxpool2(ref8, O.NHWC))
        c = W.WinoConv2d(n, h, wd, ci, co, 1, W.WINO_NHWC, True, W.WINO_OUT_INT32, path=path, algorithm=W.WINO_ALG_F2X2)
        c.transform_filter(wdv)
        ok &= np.array_equal(c(xd).cpu().numpy(), O.wino2_conv(x, w, 1, O.NHWC, True).out32)
        xu, wu = (x.astype(np.int16) + 128).astype(np.uint8), (w.astype(np.int16) + 128).astype(np.uint8)
        c = W.WinoConv2d(n, h, wd, ci, co, 1, W.WINO_NHWC, True, W.WINO_OUT_INT32, path=path,
                         input_type=W.WINO_IN_UINT8, x_zero_point=128, w_zero_point=128)
        c.transform_filter(torch.from_numpy(wu).cuda())
        ok &= np.array_equal(c(torch.from_numpy(xu).cuda()).cpu().numpy(), ref32)
    c = W.WinoConv2d(n, h, wd, ci, co, 1, W.WINO_NHWC, True, W.WINO_OUT_INT32, path=W.WINO_PATH_STAGED,
                     filter_target_max=127)
    c.transform_filter(wdv)
    ok &= np.array_equal(c(xd).cpu().numpy(), O.wino_conv(x, w, 1, O.NHWC, True, target=127).out32)
    ok &= np.array_equal(W.maxpool2(xd).cpu().numpy(), O.maxpool2(x, O.NHWC))
    torch.cuda.synchronize()
    print(name, "ok" if ok else "MISMATCH", flush=True)
print("sanitize run:", "all equal to the oracle" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
