"""Per-kernel launch times of one conv layer (CUDA graph of back-to-back launches per kernel, as bench.py):
    python tools/layer_kernels.py n h w c_in c_out [fused|staged|auto]"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_1901_01965_b200 as W
import bench

n, h, w, ci, co = (int(v) for v in sys.argv[1:6])
path = {"fused": W.WINO_PATH_FUSED, "staged": W.WINO_PATH_STAGED, "auto": W.WINO_PATH_AUTO}[
    sys.argv[6] if len(sys.argv) > 6 else "auto"]
conv = W.WinoConv2d(n, h, w, ci, co, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8, path=path)
rng = np.random.default_rng(3)
xs = [torch.from_numpy(rng.integers(-128, 128, (n, h, w, ci)).astype(np.int8)).cuda()]
ws = [torch.from_numpy(rng.integers(-60, 60, (co, 3, 3, ci)).astype(np.int8)).cuda()]
ys = [torch.empty(conv.y_shape, dtype=torch.int8, device="cuda")]
conv.transform_filter(ws[0])
st = torch.cuda.Stream()
k = bench.profile_kernels(conv, xs, ws, ys, 10, st, 1, 10)
ops = 2 * n * h * w * ci * co * 9
tot = sum(v["s_per_step"] for v in k.values())
print(f"({n},{h},{w},{ci},{co}) path {conv.info.path} chunks {conv.info.n_chunks}: " +
      " ".join(f"{name}={v['s_per_launch'] * 1e6:.1f}us x{v['launches_per_step']}" for name, v in k.items()) +
      f"  total {tot * 1e6:.0f} us  {ops / tot / 1e12:.1f} TOPS")
