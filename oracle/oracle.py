"""ctypes wrapper over oracle.c (TEST INFRASTRUCTURE ONLY -- see __init__.py).

Builds ``oracle/liboracle.so`` with gcc on first use.  All arrays are numpy;
the functions return numpy arrays.  Citations ``P:n`` are lines of PAPER.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

NCHW, NHWC = 0, 1


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (plain gcc, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int, ctypes.c_int64
        L.oracle_rha_shift.argtypes = [i64, i32]; L.oracle_rha_shift.restype = i64
        L.oracle_scale_factor.argtypes = [i64, i32, P, P]; L.oracle_scale_factor.restype = i32
        L.oracle_encode_code.argtypes = [i32, i32]; L.oracle_encode_code.restype = i32
        L.oracle_encode_code7.argtypes = [i32, i32]; L.oracle_encode_code7.restype = i32
        L.oracle_decode_code7.argtypes = [i32, P, P]; L.oracle_decode_code7.restype = None
        L.oracle_decode_code.argtypes = [i32, P, P]; L.oracle_decode_code.restype = None
        L.oracle_reverse_factor.argtypes = [i32, i32, P, P]; L.oracle_reverse_factor.restype = i32
        L.oracle_direct_conv.argtypes = [P, P, i32, i32, i32, i32, i32, i32, i32, P]
        L.oracle_direct_conv.restype = None
        L.oracle_filter_transform.argtypes = [P, i32, i32, i32, i32, i32, P, P, P]
        L.oracle_filter_transform.restype = i32
        L.oracle_input_transform.argtypes = [P, i32, i32, i32, i32, i32, i32, P]
        L.oracle_input_transform.restype = None
        L.oracle_wino_conv.argtypes = [P, P, i32, i32, i32, i32, i32, i32, i32, i32, i32,
                                       ctypes.c_int32, i32, P, P, P, P]
        L.oracle_wino_conv.restype = i32
        L.oracle_requant.argtypes = [P, i64, ctypes.c_int32, i32, P]; L.oracle_requant.restype = None
        L.oracle_maxpool2.argtypes = [P, i32, i32, i32, i32, i32, P]; L.oracle_maxpool2.restype = None
        L.oracle_matrices.argtypes = [P] * 6; L.oracle_matrices.restype = None
        L.oracle_filter_tile64.argtypes = [P, P]; L.oracle_filter_tile64.restype = None
        L.oracle_input_tile64.argtypes = [P, P]; L.oracle_input_tile64.restype = None
        L.oracle_output_tile64.argtypes = [P, P]; L.oracle_output_tile64.restype = i32
        L.oracle_filter_tile2_64.argtypes = [P, P]; L.oracle_filter_tile2_64.restype = None
        L.oracle_input_tile2_64.argtypes = [P, P]; L.oracle_input_tile2_64.restype = None
        L.oracle_output_tile2_64.argtypes = [P, P]; L.oracle_output_tile2_64.restype = None
        L.oracle_filter_transform2.argtypes = [P, i32, i32, i32, i32, i32, P, P, P]
        L.oracle_filter_transform2.restype = i32
        L.oracle_input_transform2.argtypes = [P, i32, i32, i32, i32, i32, i32, P]
        L.oracle_input_transform2.restype = None
        L.oracle_wino2_conv.argtypes = [P, P, i32, i32, i32, i32, i32, i32, i32, i32, i32,
                                        ctypes.c_int32, i32, P, P, P, P]
        L.oracle_wino2_conv.restype = i32
        L.oracle_direct_conv_u8.argtypes = [P, P, i32, i32, i32, i32, i32, i32, i32, i32, i32, P]
        L.oracle_direct_conv_u8.restype = None
        L.oracle_filter_transform_u8.argtypes = [P, i32, i32, i32, i32, i32, i32, P, P, P]
        L.oracle_filter_transform_u8.restype = i32
        L.oracle_input_transform_u8.argtypes = [P, i32, i32, i32, i32, i32, i32, i32, P]
        L.oracle_input_transform_u8.restype = None
        L.oracle_wino_conv_u8.argtypes = [P, P, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32,
                                          ctypes.c_int32, i32, P, P, P, P]
        L.oracle_wino_conv_u8.restype = i32
        L.oracle_filter_transform2_u8.argtypes = [P, i32, i32, i32, i32, i32, i32, P, P, P]
        L.oracle_filter_transform2_u8.restype = i32
        L.oracle_input_transform2_u8.argtypes = [P, i32, i32, i32, i32, i32, i32, i32, P]
        L.oracle_input_transform2_u8.restype = None
        L.oracle_wino2_conv_u8.argtypes = [P, P, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32,
                                           ctypes.c_int32, i32, P, P, P, P]
        L.oracle_wino2_conv_u8.restype = i32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------- scalars
def rha_shift(v: int, k: int) -> int:
    """round-half-away-from-zero of v / 2^k."""
    return int(lib().oracle_rha_shift(int(v), int(k)))


def scale_factor(mx: int, target: int = 255):
    """(n, p) per P:317-330 read as DESIGN.md A3; (0, 0) means unscaled."""
    n, p = ctypes.c_int(), ctypes.c_int()
    st = lib().oracle_scale_factor(int(mx), int(target), ctypes.byref(n), ctypes.byref(p))
    if st != 0:
        raise ValueError(f"scale factor out of range for max magnitude {mx}")
    return n.value, p.value


def encode_code(n: int, p: int) -> int:
    return int(lib().oracle_encode_code(int(n), int(p)))


def encode_code7(n: int, p: int) -> int:
    """7-bit code of the int8-native target (f3, A29)."""
    return int(lib().oracle_encode_code7(int(n), int(p)))


def decode_code7(code: int):
    n, p = ctypes.c_int(), ctypes.c_int()
    lib().oracle_decode_code7(int(code), ctypes.byref(n), ctypes.byref(p))
    return n.value, p.value


def decode_code(code: int):
    n, p = ctypes.c_int(), ctypes.c_int()
    lib().oracle_decode_code(int(code), ctypes.byref(n), ctypes.byref(p))
    return n.value, p.value


def reverse_factor(n: int, p: int):
    """(m, q) per P:366 read as DESIGN.md A8 / A27 (q in [3, 7]; q = 3 only for 8/128)."""
    m, q = ctypes.c_int(), ctypes.c_int()
    if lib().oracle_reverse_factor(int(n), int(p), ctypes.byref(m), ctypes.byref(q)) != 0:
        raise ValueError("no 8-bit inverse")
    return m.value, q.value


def matrices():
    """(B^T, G_int, A^T) as complex128 numpy arrays, as the oracle uses them."""
    bt_re = np.zeros((6, 6), np.int32); bt_im = np.zeros((6, 6), np.int32)
    g_re = np.zeros((6, 3), np.int32); g_im = np.zeros((6, 3), np.int32)
    at_re = np.zeros((4, 6), np.int32); at_im = np.zeros((4, 6), np.int32)
    lib().oracle_matrices(_p(bt_re), _p(bt_im), _p(g_re), _p(g_im), _p(at_re), _p(at_im))
    return bt_re + 1j * bt_im, g_re + 1j * g_im, at_re + 1j * at_im


# ---------------------------------------------------------------- tiles
def filter_tile(g) -> np.ndarray:
    """W = G_int g G_int^T for one 3x3 filter -> complex int (6,6,2) int64."""
    g = _c(np.asarray(g).reshape(9), np.int64)
    W = np.zeros(72, np.int64)
    lib().oracle_filter_tile64(_p(g), _p(W))
    return W.reshape(6, 6, 2)


def input_tile(d) -> np.ndarray:
    d = _c(np.asarray(d).reshape(36), np.int64)
    D = np.zeros(72, np.int64)
    lib().oracle_input_tile64(_p(d), _p(D))
    return D.reshape(6, 6, 2)


def output_tile(M):
    """Y = A^T M A for one 6x6 complex M (6,6,2) -> (Y (4,4) int64, im_is_zero)."""
    M = _c(np.asarray(M).reshape(72), np.int64)
    Y = np.zeros(16, np.int64)
    r = lib().oracle_output_tile64(_p(M), _p(Y))
    return Y.reshape(4, 4), r == 0


# ---------------------------------------------------------------- layers
def out_hw(H, W, pad):
    return H + 2 * pad - 2, W + 2 * pad - 2


def tiles(H, W, pad):
    Ho, Wo = out_hw(H, W, pad)
    return (Ho + 3) // 4, (Wo + 3) // 4


def direct_conv(x, w, pad=1, layout=NHWC) -> np.ndarray:
    """Exact correlation (int64), in the given layout (O1)."""
    x = _c(x, np.int8); w = _c(w, np.int8)
    if layout == NCHW:
        N, Cin, H, W = x.shape; Cout = w.shape[0]
    else:
        N, H, W, Cin = x.shape; Cout = w.shape[0]
    Ho, Wo = out_hw(H, W, pad)
    shape = (N, Cout, Ho, Wo) if layout == NCHW else (N, Ho, Wo, Cout)
    out = np.zeros(shape, np.int64)
    lib().oracle_direct_conv(_p(x), _p(w), N, H, W, Cin, Cout, pad, layout, _p(out))
    return out


def filter_transform(w, layout=NHWC, scaling=True, target=255):
    """Offline filter path -> (W [Cout][Cin][36][2], W' same, codes [Cout][36])."""
    w = _c(w, np.int8)
    Cout = w.shape[0]
    Cin = w.shape[1] if layout == NCHW else w.shape[3]
    W = np.zeros((Cout, Cin, 36, 2), np.int64)
    Wp = np.zeros((Cout, Cin, 36, 2), np.int64)
    codes = np.zeros((Cout, 36), np.uint8)
    st = lib().oracle_filter_transform(_p(w), Cout, Cin, layout, int(bool(scaling)), target,
                                       _p(W), _p(Wp), _p(codes))
    if st != 0:
        raise ValueError("scale factor out of range")
    return W, Wp, codes


def input_transform(x, pad=1, layout=NHWC) -> np.ndarray:
    """D for every (tile, cin) -> [T][Cin][36][2] int64."""
    x = _c(x, np.int8)
    if layout == NCHW:
        N, Cin, H, W = x.shape
    else:
        N, H, W, Cin = x.shape
    th, tw = tiles(H, W, pad)
    D = np.zeros((N * th * tw, Cin, 36, 2), np.int64)
    lib().oracle_input_transform(_p(x), N, H, W, Cin, pad, layout, _p(D))
    return D


class WinoResult:
    def __init__(self, out32, y8, M, Mpp, status):
        self.out32, self.y8, self.M, self.Mpp, self.status = out32, y8, M, Mpp, status


def wino_conv(x, w, pad=1, layout=NHWC, scaling=True, target=255, M0=1, S=0,
              want_y8=True, want_M=False) -> WinoResult:
    """The paper's pipeline end to end (O1-O12).  Raises on any invariant
    violation (Im Y != 0, 16 not dividing Y when unscaled, int32 range)."""
    x = _c(x, np.int8); w = _c(w, np.int8)
    if layout == NCHW:
        N, Cin, H, W = x.shape
    else:
        N, H, W, Cin = x.shape
    Cout = w.shape[0]
    Ho, Wo = out_hw(H, W, pad)
    th, tw = tiles(H, W, pad)
    T = N * th * tw
    shape = (N, Cout, Ho, Wo) if layout == NCHW else (N, Ho, Wo, Cout)
    out32 = np.zeros(shape, np.int32)
    y8 = np.zeros(shape, np.int8) if want_y8 else None
    M = np.zeros((T, Cout, 36, 2), np.int64) if want_M else None
    Mpp = np.zeros((T, Cout, 36, 2), np.int64) if want_M else None
    st = lib().oracle_wino_conv(_p(x), _p(w), N, H, W, Cin, Cout, pad, layout,
                                int(bool(scaling)), target, int(M0), int(S), _p(out32),
                                _p(y8) if y8 is not None else None,
                                _p(M) if M is not None else None,
                                _p(Mpp) if Mpp is not None else None)
    if st != 0:
        raise ValueError(f"oracle invariant violated (status {st})")
    return WinoResult(out32, y8, M, Mpp, st)


def requant(v, M0, S) -> np.ndarray:
    v = _c(v, np.int64)
    out = np.zeros(v.shape, np.int8)
    lib().oracle_requant(_p(v), v.size, int(M0), int(S), _p(out))
    return out


def maxpool2(x, layout=NHWC) -> np.ndarray:
    x = _c(x, np.int8)
    if layout == NCHW:
        N, C, H, W = x.shape; shape = (N, C, H // 2, W // 2)
    else:
        N, H, W, C = x.shape; shape = (N, H // 2, W // 2, C)
    y = np.zeros(shape, np.int8)
    lib().oracle_maxpool2(_p(x), N, H, W, C, layout, _p(y))
    return y


# ---------------------------------------------------------------- rational F(2x2,3x3)
def filter_tile2(g) -> np.ndarray:
    """W = G' g G'^T for one 3x3 filter -> (4,4) int64."""
    g = _c(np.asarray(g).reshape(9), np.int64)
    W = np.zeros(16, np.int64)
    lib().oracle_filter_tile2_64(_p(g), _p(W))
    return W.reshape(4, 4)


def input_tile2(d) -> np.ndarray:
    d = _c(np.asarray(d).reshape(16), np.int64)
    D = np.zeros(16, np.int64)
    lib().oracle_input_tile2_64(_p(d), _p(D))
    return D.reshape(4, 4)


def output_tile2(M) -> np.ndarray:
    M = _c(np.asarray(M).reshape(16), np.int64)
    Y = np.zeros(4, np.int64)
    lib().oracle_output_tile2_64(_p(M), _p(Y))
    return Y.reshape(2, 2)


def tiles2(H, W, pad):
    Ho, Wo = out_hw(H, W, pad)
    return (Ho + 1) // 2, (Wo + 1) // 2


def filter_transform2(w, layout=NHWC, scaling=True, target=255):
    """F(2x2) offline filter path -> (W [Cout][Cin][16], W', codes [Cout][16])."""
    w = _c(w, np.int8)
    Cout = w.shape[0]
    Cin = w.shape[1] if layout == NCHW else w.shape[3]
    W = np.zeros((Cout, Cin, 16), np.int64); Wp = np.zeros((Cout, Cin, 16), np.int64)
    codes = np.zeros((Cout, 16), np.uint8)
    if lib().oracle_filter_transform2(_p(w), Cout, Cin, layout, int(bool(scaling)), target,
                                      _p(W), _p(Wp), _p(codes)) != 0:
        raise ValueError("scale factor out of range")
    return W, Wp, codes


def input_transform2(x, pad=1, layout=NHWC) -> np.ndarray:
    """F(2x2) D for every (tile, cin) -> [T][Cin][16] int64."""
    x = _c(x, np.int8)
    if layout == NCHW:
        N, Cin, H, W = x.shape
    else:
        N, H, W, Cin = x.shape
    th, tw = tiles2(H, W, pad)
    D = np.zeros((N * th * tw, Cin, 16), np.int64)
    lib().oracle_input_transform2(_p(x), N, H, W, Cin, pad, layout, _p(D))
    return D


def wino2_conv(x, w, pad=1, layout=NHWC, scaling=True, target=255, M0=1, S=0,
               want_y8=True, want_M=False) -> WinoResult:
    """The rational F(2x2,3x3) pipeline with filter scaling; raises on
    invariant violations (4 not dividing Y when unscaled, int32 range)."""
    x = _c(x, np.int8); w = _c(w, np.int8)
    if layout == NCHW:
        N, Cin, H, W = x.shape
    else:
        N, H, W, Cin = x.shape
    Cout = w.shape[0]
    Ho, Wo = out_hw(H, W, pad)
    th, tw = tiles2(H, W, pad)
    T = N * th * tw
    shape = (N, Cout, Ho, Wo) if layout == NCHW else (N, Ho, Wo, Cout)
    out32 = np.zeros(shape, np.int32)
    y8 = np.zeros(shape, np.int8) if want_y8 else None
    M = np.zeros((T, Cout, 16), np.int64) if want_M else None
    Mpp = np.zeros((T, Cout, 16), np.int64) if want_M else None
    st = lib().oracle_wino2_conv(_p(x), _p(w), N, H, W, Cin, Cout, pad, layout, int(bool(scaling)), target,
                                 int(M0), int(S), _p(out32), _p(y8) if y8 is not None else None,
                                 _p(M) if M is not None else None, _p(Mpp) if Mpp is not None else None)
    if st != 0:
        raise ValueError(f"oracle invariant violated (status {st})")
    return WinoResult(out32, y8, M, Mpp, st)


# ---------------------------------------------------------------- uint8 + zero points
def _dims(x, w, layout):
    if layout == NCHW:
        N, Cin, H, W = x.shape
    else:
        N, H, W, Cin = x.shape
    return N, H, W, Cin, w.shape[0]


def direct_conv_u8(x, w, zx, zw, pad=1, layout=NHWC) -> np.ndarray:
    """Exact correlation of (x - zx) with (w - zw) (int64), uint8 tensors (O1 on int9 values)."""
    x = _c(x, np.uint8); w = _c(w, np.uint8)
    N, H, W, Cin, Cout = _dims(x, w, layout)
    Ho, Wo = out_hw(H, W, pad)
    out = np.zeros((N, Cout, Ho, Wo) if layout == NCHW else (N, Ho, Wo, Cout), np.int64)
    lib().oracle_direct_conv_u8(_p(x), _p(w), int(zx), int(zw), N, H, W, Cin, Cout, pad, layout, _p(out))
    return out


def filter_transform_u8(w, zw, layout=NHWC, scaling=True, target=255):
    w = _c(w, np.uint8)
    Cout = w.shape[0]
    Cin = w.shape[1] if layout == NCHW else w.shape[3]
    W = np.zeros((Cout, Cin, 36, 2), np.int64); Wp = np.zeros((Cout, Cin, 36, 2), np.int64)
    codes = np.zeros((Cout, 36), np.uint8)
    if lib().oracle_filter_transform_u8(_p(w), int(zw), Cout, Cin, layout, int(bool(scaling)), target,
                                        _p(W), _p(Wp), _p(codes)) != 0:
        raise ValueError("scale factor out of range")
    return W, Wp, codes


def input_transform_u8(x, zx, pad=1, layout=NHWC) -> np.ndarray:
    x = _c(x, np.uint8)
    if layout == NCHW:
        N, Cin, H, W = x.shape
    else:
        N, H, W, Cin = x.shape
    th, tw = tiles(H, W, pad)
    D = np.zeros((N * th * tw, Cin, 36, 2), np.int64)
    lib().oracle_input_transform_u8(_p(x), int(zx), N, H, W, Cin, pad, layout, _p(D))
    return D


def wino_conv_u8(x, w, zx, zw, pad=1, layout=NHWC, scaling=True, target=255, M0=1, S=0,
                 want_y8=True, want_M=False) -> WinoResult:
    """The complex F(4x4) pipeline on uint8 tensors with zero points (int9 values)."""
    x = _c(x, np.uint8); w = _c(w, np.uint8)
    N, H, W, Cin, Cout = _dims(x, w, layout)
    Ho, Wo = out_hw(H, W, pad)
    th, tw = tiles(H, W, pad)
    T = N * th * tw
    shape = (N, Cout, Ho, Wo) if layout == NCHW else (N, Ho, Wo, Cout)
    out32 = np.zeros(shape, np.int32)
    y8 = np.zeros(shape, np.int8) if want_y8 else None
    M = np.zeros((T, Cout, 36, 2), np.int64) if want_M else None
    Mpp = np.zeros((T, Cout, 36, 2), np.int64) if want_M else None
    st = lib().oracle_wino_conv_u8(_p(x), _p(w), int(zx), int(zw), N, H, W, Cin, Cout, pad, layout,
                                   int(bool(scaling)), target, int(M0), int(S), _p(out32),
                                   _p(y8) if y8 is not None else None, _p(M) if M is not None else None,
                                   _p(Mpp) if Mpp is not None else None)
    if st != 0:
        raise ValueError(f"oracle invariant violated (status {st})")
    return WinoResult(out32, y8, M, Mpp, st)



# ---------------------------------------------------------------- F(2x2) x uint8 (the paper's evaluated configuration)
def filter_transform2_u8(w, zw, layout=NHWC, scaling=True, target=255):
    """F(2x2) offline filter path on uint8 weights with zero point zw (int9 values)."""
    w = _c(w, np.uint8)
    Cout = w.shape[0]
    Cin = w.shape[1] if layout == NCHW else w.shape[3]
    W = np.zeros((Cout, Cin, 16), np.int64); Wp = np.zeros((Cout, Cin, 16), np.int64)
    codes = np.zeros((Cout, 16), np.uint8)
    if lib().oracle_filter_transform2_u8(_p(w), int(zw), Cout, Cin, layout, int(bool(scaling)), target,
                                         _p(W), _p(Wp), _p(codes)) != 0:
        raise ValueError("scale factor out of range")
    return W, Wp, codes


def input_transform2_u8(x, zx, pad=1, layout=NHWC) -> np.ndarray:
    x = _c(x, np.uint8)
    if layout == NCHW:
        N, Cin, H, W = x.shape
    else:
        N, H, W, Cin = x.shape
    th, tw = tiles2(H, W, pad)
    D = np.zeros((N * th * tw, Cin, 16), np.int64)
    lib().oracle_input_transform2_u8(_p(x), int(zx), N, H, W, Cin, pad, layout, _p(D))
    return D


def wino2_conv_u8(x, w, zx, zw, pad=1, layout=NHWC, scaling=True, target=255, M0=1, S=0,
                  want_y8=True, want_M=False) -> WinoResult:
    """The rational F(2x2) pipeline on uint8 tensors with zero points (int9 values)."""
    x = _c(x, np.uint8); w = _c(w, np.uint8)
    N, H, W, Cin, Cout = _dims(x, w, layout)
    Ho, Wo = out_hw(H, W, pad)
    th, tw = tiles2(H, W, pad)
    T = N * th * tw
    shape = (N, Cout, Ho, Wo) if layout == NCHW else (N, Ho, Wo, Cout)
    out32 = np.zeros(shape, np.int32)
    y8 = np.zeros(shape, np.int8) if want_y8 else None
    M = np.zeros((T, Cout, 16), np.int64) if want_M else None
    Mpp = np.zeros((T, Cout, 16), np.int64) if want_M else None
    st = lib().oracle_wino2_conv_u8(_p(x), _p(w), int(zx), int(zw), N, H, W, Cin, Cout, pad, layout,
                                    int(bool(scaling)), target, int(M0), int(S), _p(out32),
                                    _p(y8) if y8 is not None else None, _p(M) if M is not None else None,
                                    _p(Mpp) if Mpp is not None else None)
    if st != 0:
        raise ValueError(f"oracle invariant violated (status {st})")
    return WinoResult(out32, y8, M, Mpp, st)
