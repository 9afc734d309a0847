"""A stack of 3x3 int8 Winograd conv layers (the VGG-16 configuration of
BASELINE.json configs[4]): per layer one plan, the offline filter transform,
wino_conv2d_int8 with int8 requantisation (A14), and the 2x2/2 max
pool after layers 2, 4, 7, 10 (A22).  Sequencing only: every operation is a
call into libwino; one workspace is shared by all layers."""
from __future__ import annotations

import torch

from . import _lib as L
from .conv import WinoConv2d, maxpool2


class ConvStack:
    def __init__(self, n, layers, pools_after, shifts, layout=L.WINO_NHWC, device=None, workspace_mb=1024,
                 path=L.WINO_PATH_AUTO):
        """layers: sequence of objects with h, w, c_in, c_out, pad, scaling; shifts: requant
        shift per layer (multiplier 1)."""
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device)
        self.layout, self.pools_after, self.shifts = layout, set(pools_after), list(shifts)
        # one workspace sized for the largest layer
        sizes = []
        for l in layers:
            d = L.wino_conv_desc(n, l.h, l.w, l.c_in, l.c_out, l.pad, layout, int(l.scaling), 255, L.WINO_OUT_INT8,
                                 workspace_mb, path)
            plan = L.wino_plan(d, device)
            sizes.append(L.wino_workspace_bytes(plan))
            L.wino_plan_destroy(plan)
        self.workspace = torch.empty(max(sizes), dtype=torch.int8, device=self.device)
        self.convs = [WinoConv2d(n, l.h, l.w, l.c_in, l.c_out, l.pad, layout, l.scaling, L.WINO_OUT_INT8, device,
                                 workspace=self.workspace, workspace_mb=workspace_mb, path=path) for l in layers]
        self.outs = [torch.empty(c.y_shape, dtype=torch.int8, device=self.device) for c in self.convs]
        self.pooled = {}
        for i, c in enumerate(self.convs):
            if i in self.pools_after:
                if layout == L.WINO_NHWC:
                    nn, hh, ww, cc = c.y_shape
                    shape = (nn, hh // 2, ww // 2, cc)
                else:
                    nn, cc, hh, ww = c.y_shape
                    shape = (nn, cc, hh // 2, ww // 2)
                self.pooled[i] = torch.empty(shape, dtype=torch.int8, device=self.device)

    def transform_filters(self, weights, stream=None):
        for c, w in zip(self.convs, weights):
            c.transform_filter(w, stream)

    def __call__(self, x, stream=None):
        """Run all layers on x; returns the final activation (a view of an internal buffer)."""
        sp = (stream or torch.cuda.current_stream()).cuda_stream
        cur = x
        for i, c in enumerate(self.convs):
            y = self.outs[i]
            L.wino_conv2d_int8(c.plan, cur.data_ptr(), c.w_wino.data_ptr(), c.codes.data_ptr(), 1, self.shifts[i],
                               y.data_ptr(), self.workspace.data_ptr(), sp)
            if i in self.pools_after:
                p = self.pooled[i]
                if self.layout == L.WINO_NHWC:
                    nn, hh, ww, cc = y.shape
                else:
                    nn, cc, hh, ww = y.shape
                L.wino_maxpool2_int8(y.data_ptr(), nn, hh, ww, cc, self.layout, p.data_ptr(), sp)
                y = p
            cur = y
        return cur

    def launches(self):
        return sum(1 + c.info.stages * c.info.n_chunks for c in self.convs) + len(self.pooled)
