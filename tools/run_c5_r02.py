"""Run the C5 step (VGG-16 stack, batch 256, lanes 3, 256 MiB chunks, as bench.py) or one of its layers, for ncu
launch lists and --set full captures:
    python tools/run_c5_r02.py step [steps]     # whole steps (filter transforms on the side stream)
    python tools/run_c5_r02.py layer L [reps]   # conv of layer L (1-based) alone, on its synthetic input"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import synth
from paper_1901_01965_b200 import _lib as L
from paper_1901_01965_b200.stack import ConvStack

cfg = synth.CONFIGS["C5"]
shifts = synth.stack_shifts("C5")
x, ws = synth.stack_inputs("C5")
st = ConvStack(x.shape[0], cfg.layers, cfg.pools_after, shifts, workspace_mb=256, lanes=3)
xd = torch.from_numpy(x).cuda()
wd = [torch.from_numpy(w).cuda() for w in ws]
stream = torch.cuda.Stream()
mode = sys.argv[1] if len(sys.argv) > 1 else "step"
with torch.cuda.stream(stream):
    st.step(xd, wd, stream)           # warm-up (codes validated, outputs of every layer formed)
    stream.synchronize()
    if mode == "step":
        for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 1):
            st.step(xd, wd, stream)
    else:
        li = int(sys.argv[2]) - 1
        c = st.convs[li]
        cur = xd if li == 0 else st.pooled.get(li - 1, st.outs[li - 1])
        for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
            L.wino_conv2d_int8(c.plan, cur.data_ptr(), c.w_wino.data_ptr(), c.codes.data_ptr(), 1, shifts[li],
                               st.outs[li].data_ptr(), st.workspace.data_ptr(), stream.cuda_stream)
    stream.synchronize()
print("ok", mode)
