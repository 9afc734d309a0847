"""Thin ctypes binding over libwino.so (include/wino.h).  Argument marshalling
only: every step of the path runs in the CUDA kernels behind the C ABI.
There is no fallback: if the library is missing or fails to load, every
entry point raises."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libwino.so")

WINO_OK, WINO_ERR_INVALID_ARG, WINO_ERR_UNSUPPORTED, WINO_ERR_SHAPE = 0, -1, -2, -3
WINO_ERR_RANGE, WINO_ERR_CUDA, WINO_ERR_NOMEM = -4, -5, -6
WINO_NCHW, WINO_NHWC = 0, 1
WINO_OUT_INT8, WINO_OUT_INT32, WINO_OUT_INT8_POOL2 = 0, 1, 2
WINO_PATH_AUTO, WINO_PATH_FUSED, WINO_PATH_STAGED = 0, 1, 2
WINO_ALG_F4X4, WINO_ALG_F2X2 = 0, 1
WINO_IN_INT8, WINO_IN_UINT8 = 0, 1

# every symbol include/wino.h declares
EXPORTS = ("wino_status_string", "wino_last_cuda_error", "wino_plan", "wino_plan_destroy", "wino_plan_query", "wino_filter_bytes",
           "wino_codes_bytes", "wino_workspace_bytes", "wino_output_bytes", "wino_transform_filter",
           "wino_conv2d_int8", "wino_conv2d_int8_host", "wino_conv2d_int8_stage", "wino_validate_codes", "wino_check_codes", "wino_maxpool2_int8",
           "wino_debug_set_trace", "wino_debug_fastdiv")


class wino_conv_desc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("h", ctypes.c_int), ("w", ctypes.c_int), ("c_in", ctypes.c_int),
                ("c_out", ctypes.c_int), ("pad", ctypes.c_int), ("layout", ctypes.c_int),
                ("filter_scaling", ctypes.c_int), ("filter_target_max", ctypes.c_int), ("out_mode", ctypes.c_int),
                ("workspace_mb", ctypes.c_int), ("path", ctypes.c_int), ("algorithm", ctypes.c_int),
                ("input_type", ctypes.c_int), ("x_zero_point", ctypes.c_int), ("w_zero_point", ctypes.c_int),
                ("lanes", ctypes.c_int)]


class wino_plan_info(ctypes.Structure):
    _fields_ = [("ho", ctypes.c_int), ("wo", ctypes.c_int), ("tiles_h", ctypes.c_int), ("tiles_w", ctypes.c_int),
                ("tiles", ctypes.c_longlong), ("cin_pad", ctypes.c_int), ("cout_pad", ctypes.c_int),
                ("n_block", ctypes.c_int), ("m_block", ctypes.c_int), ("planes", ctypes.c_int),
                ("pieces", ctypes.c_int), ("chunk_images", ctypes.c_int), ("n_chunks", ctypes.c_int),
                ("lanes", ctypes.c_int), ("lane_bytes", ctypes.c_size_t), ("packing", ctypes.c_int),
                ("chunk_tiles_pad", ctypes.c_longlong), ("path", ctypes.c_int), ("stages", ctypes.c_int),
                ("algorithm", ctypes.c_int), ("tile", ctypes.c_int), ("positions", ctypes.c_int),
                ("v_offset", ctypes.c_size_t), ("v_bytes", ctypes.c_size_t),
                ("m_offset", ctypes.c_size_t), ("m_bytes", ctypes.c_size_t), ("workspace_bytes", ctypes.c_size_t),
                ("filter_bytes", ctypes.c_size_t), ("codes_bytes", ctypes.c_size_t), ("x_bytes", ctypes.c_size_t),
                ("y_bytes", ctypes.c_size_t)]


class WinoError(RuntimeError):
    def __init__(self, status: int, where: str):
        extra = f": {lib().wino_last_cuda_error().decode()}" if status == WINO_ERR_CUDA else ""
        super().__init__(f"{where}: {status_string(status)} (status {status}){extra}")
        self.status = status


_lib = None


def lib():
    """Load libwino.so (raises if it is absent: no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P, I, I32, SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_int32, ctypes.c_size_t
        L.wino_status_string.argtypes = [I]; L.wino_status_string.restype = ctypes.c_char_p
        L.wino_last_cuda_error.argtypes = []; L.wino_last_cuda_error.restype = ctypes.c_char_p
        L.wino_plan.argtypes = [ctypes.POINTER(wino_conv_desc), I, ctypes.POINTER(P)]; L.wino_plan.restype = I
        L.wino_plan_destroy.argtypes = [P]; L.wino_plan_destroy.restype = I
        L.wino_plan_query.argtypes = [P, ctypes.POINTER(wino_plan_info)]; L.wino_plan_query.restype = I
        for f in ("wino_filter_bytes", "wino_codes_bytes", "wino_workspace_bytes", "wino_output_bytes"):
            getattr(L, f).argtypes = [P]; getattr(L, f).restype = SZ
        L.wino_transform_filter.argtypes = [P, P, P, P, P]; L.wino_transform_filter.restype = I
        L.wino_conv2d_int8.argtypes = [P, P, P, P, I32, I, P, P, P]; L.wino_conv2d_int8.restype = I
        L.wino_conv2d_int8_host.argtypes = [P, P, P, P, I32, I, P, P, P, P, P]; L.wino_conv2d_int8_host.restype = I
        L.wino_conv2d_int8_stage.argtypes = [P, I, I, P, P, P, I32, I, P, P, P]
        L.wino_conv2d_int8_stage.restype = I
        L.wino_validate_codes.argtypes = [P, P, P, P]; L.wino_validate_codes.restype = I
        L.wino_check_codes.argtypes = [P, P, P, P]; L.wino_check_codes.restype = I
        L.wino_maxpool2_int8.argtypes = [P, I, I, I, I, I, P, P]; L.wino_maxpool2_int8.restype = I
        L.wino_debug_set_trace.argtypes = [P]; L.wino_debug_set_trace.restype = I
        L.wino_debug_fastdiv.argtypes = [I, I]; L.wino_debug_fastdiv.restype = I
        _lib = L
    return _lib


def status_string(status: int) -> str:
    return lib().wino_status_string(int(status)).decode()


def _check(status: int, where: str):
    if status != WINO_OK:
        raise WinoError(status, where)


# ------------------------------------------------------------ same names as the C ABI
def wino_plan(desc: wino_conv_desc, device: int) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _check(lib().wino_plan(ctypes.byref(desc), int(device), ctypes.byref(h)), "wino_plan")
    return h


def wino_plan_destroy(plan) -> None:
    _check(lib().wino_plan_destroy(plan), "wino_plan_destroy")


def wino_plan_query(plan) -> wino_plan_info:
    info = wino_plan_info()
    _check(lib().wino_plan_query(plan, ctypes.byref(info)), "wino_plan_query")
    return info


def wino_filter_bytes(plan) -> int: return int(lib().wino_filter_bytes(plan))
def wino_codes_bytes(plan) -> int: return int(lib().wino_codes_bytes(plan))
def wino_workspace_bytes(plan) -> int: return int(lib().wino_workspace_bytes(plan))
def wino_output_bytes(plan) -> int: return int(lib().wino_output_bytes(plan))


def wino_transform_filter(plan, w_ptr: int, w_wino_ptr: int, codes_ptr: int, stream: int) -> None:
    _check(lib().wino_transform_filter(plan, w_ptr, w_wino_ptr, codes_ptr, stream), "wino_transform_filter")


def wino_conv2d_int8(plan, x_ptr: int, w_wino_ptr: int, codes_ptr: int, requant_mult: int, requant_shift: int,
                     y_ptr: int, ws_ptr: int, stream: int) -> None:
    _check(lib().wino_conv2d_int8(plan, x_ptr, w_wino_ptr, codes_ptr, int(requant_mult), int(requant_shift),
                                  y_ptr, ws_ptr, stream), "wino_conv2d_int8")


def wino_conv2d_int8_host(plan, x_host_ptr: int, w_wino_ptr: int, codes_ptr: int, requant_mult: int,
                          requant_shift: int, y_host_ptr: int, x_dev_ptr: int, y_dev_ptr: int, ws_ptr: int,
                          stream: int) -> None:
    _check(lib().wino_conv2d_int8_host(plan, x_host_ptr, w_wino_ptr, codes_ptr, int(requant_mult),
                                       int(requant_shift), y_host_ptr, x_dev_ptr, y_dev_ptr, ws_ptr, stream),
           "wino_conv2d_int8_host")


def wino_conv2d_int8_stage(plan, stage: int, chunk: int, x_ptr: int, w_wino_ptr: int, codes_ptr: int,
                           requant_mult: int, requant_shift: int, y_ptr: int, ws_ptr: int, stream: int) -> None:
    _check(lib().wino_conv2d_int8_stage(plan, int(stage), int(chunk), x_ptr, w_wino_ptr, codes_ptr,
                                        int(requant_mult), int(requant_shift), y_ptr, ws_ptr, stream),
           "wino_conv2d_int8_stage")


def wino_validate_codes(plan, codes_ptr: int, ws_ptr: int, stream: int) -> None:
    _check(lib().wino_validate_codes(plan, codes_ptr, ws_ptr, stream), "wino_validate_codes")


def wino_check_codes(plan, codes_ptr: int, bad_ptr: int, stream: int) -> None:
    _check(lib().wino_check_codes(plan, codes_ptr, bad_ptr, stream), "wino_check_codes")


def wino_maxpool2_int8(x_ptr: int, n: int, h: int, w: int, c: int, layout: int, y_ptr: int, stream: int) -> None:
    _check(lib().wino_maxpool2_int8(x_ptr, n, h, w, c, layout, y_ptr, stream), "wino_maxpool2_int8")
