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
                 path=L.WINO_PATH_AUTO, lanes=0, fuse_pool=True):
        """layers: sequence of objects with h, w, c_in, c_out, pad, scaling; shifts: requant
        shift per layer (multiplier 1)."""
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device)
        self.layout, self.pools_after, self.shifts = layout, set(pools_after), list(shifts)
        # per layer: int8 output, and for a layer followed by a pool the pool fused into its output stage
        # (WINO_OUT_INT8_POOL2) where the plan supports it (fuse_pool), else a separate pool launch;
        # one workspace sized for the largest layer
        modes, sizes = [], []
        for i, l in enumerate(layers):
            mode = L.WINO_OUT_INT8
            for m in ((L.WINO_OUT_INT8_POOL2, L.WINO_OUT_INT8) if (fuse_pool and i in self.pools_after)
                      else (L.WINO_OUT_INT8,)):
                d = L.wino_conv_desc(n, l.h, l.w, l.c_in, l.c_out, l.pad, layout, int(l.scaling), 255, m,
                                     workspace_mb, path, 0, 0, 0, 0, lanes)
                try:
                    plan = L.wino_plan(d, device)
                except L.WinoError as e:
                    if m == L.WINO_OUT_INT8_POOL2 and e.status == L.WINO_ERR_UNSUPPORTED:
                        continue
                    raise
                mode = m
                sizes.append(L.wino_workspace_bytes(plan))
                L.wino_plan_destroy(plan)
                break
            modes.append(mode)
        self.workspace = torch.empty(max(sizes), dtype=torch.int8, device=self.device)
        self.convs = [WinoConv2d(n, l.h, l.w, l.c_in, l.c_out, l.pad, layout, l.scaling, m, device,
                                 workspace=self.workspace, workspace_mb=workspace_mb, path=path, lanes=lanes)
                      for l, m in zip(layers, modes)]
        self.fused_pool = {i for i, m in enumerate(modes) if m == L.WINO_OUT_INT8_POOL2}
        self.outs = [torch.empty(c.y_shape, dtype=torch.int8, device=self.device) for c in self.convs]
        self.pooled = {}
        for i, c in enumerate(self.convs):
            if i in self.fused_pool:
                self.pooled[i] = self.outs[i]       # the conv writes the pooled activation itself
            elif i in self.pools_after:
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

    def step(self, x, weights, stream=None):
        """One whole step: the 13 offline filter transforms on a side stream, forked at the start, so
        they overlap the first layers' convolutions instead of sitting between them; layer i's conv waits
        for its own filter transform only (event join).  Same launches and results as
        transform_filters(weights) followed by self(x)."""
        main = stream or torch.cuda.current_stream()
        if not hasattr(self, "_side"):
            self._side = torch.cuda.Stream(device=self.device)
        fork = torch.cuda.Event()
        fork.record(main)
        self._side.wait_event(fork)
        ready = []
        for c, w in zip(self.convs, weights):
            c.transform_filter(w, self._side)
            e = torch.cuda.Event()
            e.record(self._side)
            ready.append(e)
        out = self(x, main, ready)
        return out

    def __call__(self, x, stream=None, ready=None):
        """Run all layers on x; returns the final activation (a view of an internal buffer).  `ready`:
        optional per-layer CUDA events the layer's conv waits for (its filter transform)."""
        st_ = stream or torch.cuda.current_stream()
        sp = st_.cuda_stream
        cur = x
        for i, c in enumerate(self.convs):
            if ready is not None:
                st_.wait_event(ready[i])
            y = self.outs[i]
            L.wino_conv2d_int8(c.plan, cur.data_ptr(), c.w_wino.data_ptr(), c.codes.data_ptr(), 1, self.shifts[i],
                               y.data_ptr(), self.workspace.data_ptr(), sp)
            if i in self.pools_after and i not in self.fused_pool:
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
        return sum(1 + c.info.stages * c.info.n_chunks for c in self.convs) + len(self.pooled) - len(self.fused_pool)
