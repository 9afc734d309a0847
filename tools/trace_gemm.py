"""Debug: timeline of the K3 GEMM pipeline (per CTA, per plane) for a config.
    python tools/trace_gemm.py [C2]   -> prints a summary, writes gpurun_out/trace_<cfg>.npy"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1901_01965_b200 as W  # noqa: E402
from paper_1901_01965_b200 import _lib as L  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
layer = synth.CONFIGS[cfg].layers[0]
conv = W.WinoConv2d(layer.n, layer.h, layer.w, layer.c_in, layer.c_out, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8)
x, w = synth.config_inputs(cfg)
xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
conv.transform_filter(wd)
S = synth.requant_shift(layer)
y = conv(xd, 1, S)
nsm = torch.cuda.get_device_properties(0).multi_processor_count
WORDS = 16 * 6
trace = torch.zeros(nsm * WORDS, dtype=torch.int64, device="cuda")
sp = torch.cuda.current_stream().cuda_stream
for rep in range(3):
    L.wino_conv2d_int8_stage(conv.plan, 2, 0, xd.data_ptr(), conv.w_wino.data_ptr(), conv.codes.data_ptr(), 1, S,
                             y.data_ptr(), conv.workspace.data_ptr(), sp)
    if rep == 2:
        L.lib().wino_debug_set_trace(trace.data_ptr())
    L.wino_conv2d_int8_stage(conv.plan, 3, 0, xd.data_ptr(), conv.w_wino.data_ptr(), conv.codes.data_ptr(), 1, S,
                             y.data_ptr(), conv.workspace.data_ptr(), sp)
    torch.cuda.synchronize()
L.lib().wino_debug_set_trace(None)
raw = trace.view(nsm, WORDS).cpu().numpy().astype(np.float64)
t0 = raw[raw > 0].min()
raw = np.where(raw > 0, (raw - t0) / 1e3, np.nan)   # us since first stamp
t = raw[:, :96].reshape(nsm, 16, 6)
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/trace_{cfg}.npy", t)
names = ["prod_issue", "mma_data", "mma_tmem", "mma_commit", "epi_acc", "epi_store"]
print(f"chunks {conv.info.n_chunks}  kernel span {np.nanmax(t):.2f} us")
for c in (0, 1, 74, 147):
    print(f"CTA {c}:")
    for p in range(16):
        row = t[c, p]
        if np.all(np.isnan(row)):
            continue
        print("   plane %2d " % p + "  ".join(f"{n}={v:7.2f}" for n, v in zip(names, row)))
d = lambda a, b: np.nanmean(t[:, :, b] - t[:, :, a])
print("mean  issue->data %.2f  data->tmem %.2f  tmem->commit %.2f  commit->epi %.2f" % (d(0, 1), d(1, 2), d(2, 3), d(3, 4)))
print("first stamps: prod_issue min %.2f max %.2f ; last epi_done max %.2f" % (
    np.nanmin(t[:, 0, 0]), np.nanmax(t[:, 0, 0]), np.nanmax(t[:, :, 5])))
