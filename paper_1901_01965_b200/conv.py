"""Torch-facing convenience wrapper over the C ABI.  PyTorch supplies device
memory and streams only; all arithmetic runs in libwino's CUDA kernels."""
from __future__ import annotations

import torch

from . import _lib as L


class WinoConv2d:
    """One 3x3 stride-1 int8 conv layer planned for a fixed shape.

    x / w / y are int8 (or int32 y) CUDA tensors in the plan's layout
    (NCHW with OIHW filters, or NHWC with OHWI filters).
    """

    def __init__(self, n, h, w, c_in, c_out, pad=1, layout=L.WINO_NHWC, filter_scaling=True,
                 out_mode=L.WINO_OUT_INT8, device=None, workspace=None, workspace_mb=0, path=L.WINO_PATH_AUTO,
                 algorithm=L.WINO_ALG_F4X4, input_type=L.WINO_IN_INT8, x_zero_point=0, w_zero_point=0,
                 filter_target_max=255, lanes=0):
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device)
        # filter_target_max: 255 = the paper's two-piece W'; 127 = int8-native single-piece W' (f3, A29)
        self.desc = L.wino_conv_desc(n, h, w, c_in, c_out, pad, layout, int(bool(filter_scaling)), filter_target_max,
                                     out_mode, workspace_mb, path, algorithm, input_type, x_zero_point, w_zero_point,
                                     lanes)
        self.in_dtype = torch.uint8 if input_type == L.WINO_IN_UINT8 else torch.int8
        self.plan = L.wino_plan(self.desc, device)
        self.info = L.wino_plan_query(self.plan)
        self.layout, self.out_mode = layout, out_mode
        ho, wo = self.info.ho, self.info.wo
        self.x_shape = (n, c_in, h, w) if layout == L.WINO_NCHW else (n, h, w, c_in)
        self.y_shape = (n, c_out, ho, wo) if layout == L.WINO_NCHW else (n, ho, wo, c_out)
        if out_mode == L.WINO_OUT_INT8_POOL2:   # the 2x2/2 max pool fused into the output stage (NHWC)
            self.y_shape = (n, ho // 2, wo // 2, c_out)
        self.w_shape = (c_out, c_in, 3, 3) if layout == L.WINO_NCHW else (c_out, 3, 3, c_in)
        self.y_dtype = torch.int32 if out_mode == L.WINO_OUT_INT32 else torch.int8
        self.w_wino = torch.empty(self.info.filter_bytes, dtype=torch.int8, device=self.device)
        self.codes = torch.empty((c_out, self.info.positions), dtype=torch.uint8, device=self.device)
        if workspace is not None:   # caller-shared scratch (e.g. one buffer for a layer stack)
            assert workspace.numel() >= self.info.workspace_bytes and workspace.dtype == torch.int8
            self.workspace = workspace
        else:
            self.workspace = torch.empty(self.info.workspace_bytes, dtype=torch.int8, device=self.device)

    def __del__(self):
        plan = getattr(self, "plan", None)
        if plan is not None and plan.value:
            try:
                L.wino_plan_destroy(plan)
            except Exception:
                pass
            self.plan = None

    @staticmethod
    def _stream(stream):
        return (stream or torch.cuda.current_stream()).cuda_stream

    def transform_filter(self, w: torch.Tensor, stream=None):
        assert w.dtype == self.in_dtype and w.is_cuda and tuple(w.shape) == self.w_shape and w.is_contiguous()
        L.wino_transform_filter(self.plan, w.data_ptr(), self.w_wino.data_ptr(), self.codes.data_ptr(),
                                self._stream(stream))
        return self.codes

    def __call__(self, x: torch.Tensor, requant_mult=1, requant_shift=0, y=None, codes=None, stream=None):
        assert x.dtype == self.in_dtype and x.is_cuda and tuple(x.shape) == self.x_shape and x.is_contiguous()
        if y is None:
            y = torch.empty(self.y_shape, dtype=self.y_dtype, device=self.device)
        c = self.codes if codes is None else codes
        L.wino_conv2d_int8(self.plan, x.data_ptr(), self.w_wino.data_ptr(), c.data_ptr(), requant_mult,
                           requant_shift, y.data_ptr(), self.workspace.data_ptr(), self._stream(stream))
        return y

    def call_host(self, x_host: torch.Tensor, y_host: torch.Tensor, x_dev: torch.Tensor, y_dev: torch.Tensor,
                  requant_mult=1, requant_shift=0, stream=None):
        """x_host / y_host: pinned CPU tensors; copies happen inside the C ABI call."""
        L.wino_conv2d_int8_host(self.plan, x_host.data_ptr(), self.w_wino.data_ptr(), self.codes.data_ptr(),
                                requant_mult, requant_shift, y_host.data_ptr(), x_dev.data_ptr(),
                                y_dev.data_ptr(), self.workspace.data_ptr(), self._stream(stream))
        return y_host

    # ---- workspace views (documented layouts, for tests) ----
    def v_image(self):
        return self.workspace[self.info.v_offset:self.info.v_offset + self.info.v_bytes]

    def m_raw(self):
        """Raw per-plane M of the last chunk (int32, layout in DESIGN.md / layout.cuh)."""
        i = self.info
        return self.workspace[i.m_offset:i.m_offset + i.m_bytes].view(torch.int32)


def maxpool2(x: torch.Tensor, layout=L.WINO_NHWC, stream=None):
    if layout == L.WINO_NHWC:
        n, h, w, c = x.shape; y = torch.empty((n, h // 2, w // 2, c), dtype=torch.int8, device=x.device)
    else:
        n, c, h, w = x.shape; y = torch.empty((n, c, h // 2, w // 2), dtype=torch.int8, device=x.device)
    L.wino_maxpool2_int8(x.data_ptr(), n, h, w, c, layout, y.data_ptr(),
                         (stream or torch.cuda.current_stream()).cuda_stream)
    return y
