"""B200-native complex-Winograd F(4x4,3x3) int8 convolution with the integer
filter-precision scaling of arXiv 1901.01965 (Meng & Brothers).

The computation lives in libwino.so (hand-written sm_100a CUDA kernels behind
the C ABI of include/wino.h); this package is a thin binding.  Importing it
does not load the library; the first call does, and raises if it is missing.
"""
from . import _lib  # noqa: F401
from ._lib import (WINO_NCHW, WINO_NHWC, WINO_OUT_INT8, WINO_OUT_INT32, WINO_OUT_INT8_POOL2, WINO_PATH_FUSED, WINO_PATH_STAGED, WINO_PATH_AUTO,  # noqa: F401
                   WINO_ALG_F4X4, WINO_ALG_F2X2, WINO_IN_INT8, WINO_IN_UINT8,
                   WinoError,
                   wino_conv_desc, wino_plan, wino_plan_destroy, wino_plan_query, wino_transform_filter,
                   wino_conv2d_int8, wino_conv2d_int8_host, wino_validate_codes)
from .conv import WinoConv2d, maxpool2  # noqa: F401
