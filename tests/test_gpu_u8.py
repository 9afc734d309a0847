"""GPU parity of the uint8 + zero-point mode (staged complex F(4x4))
against the oracle's uint8 pipeline: codes, W', V and M'' exact, y bit-exact."""
import zlib

import numpy as np
import pytest
import torch

from oracle import oracle as O
import layout_decode as LD

pytestmark = pytest.mark.gpu


def _layer(rng, n, h, w, ci, co, layout):
    x = rng.integers(0, 256, (n, h, w, ci), dtype=np.int64).astype(np.uint8)
    wt = rng.integers(0, 256, (co, 3, 3, ci), dtype=np.int64).astype(np.uint8)
    if layout == O.NCHW:
        x = np.ascontiguousarray(x.transpose(0, 3, 1, 2)); wt = np.ascontiguousarray(wt.transpose(0, 3, 1, 2))
    return x, wt


def _check(x, w, zx, zw, layout, pad=1, scaling=True, intermediates=True, path=None):
    import paper_1901_01965_b200 as W
    path = W.WINO_PATH_STAGED if path is None else path
    intermediates = intermediates and path == W.WINO_PATH_STAGED   # V / W' / M'' decoders: staged layouts
    if layout == O.NCHW:
        n, ci, h, wd = x.shape
    else:
        n, h, wd, ci = x.shape
    co = w.shape[0]
    conv = W.WinoConv2d(n, h, wd, ci, co, pad, layout, scaling, W.WINO_OUT_INT32, path=path,
                        input_type=W.WINO_IN_UINT8, x_zero_point=zx, w_zero_point=zw)
    conv.transform_filter(torch.from_numpy(w).cuda())
    y = conv(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = O.wino_conv_u8(x, w, zx, zw, pad, layout, scaling=scaling, want_M=intermediates)
    np.testing.assert_array_equal(y, ref.out32)
    np.testing.assert_array_equal(conv.codes.cpu().numpy(), O.filter_transform_u8(w, zw, layout, scaling=scaling)[2])
    if not scaling:
        np.testing.assert_array_equal(y.astype(np.int64), O.direct_conv_u8(x, w, zx, zw, pad, layout))
    if intermediates:
        info = conv.info
        _, Wp, codes = O.filter_transform_u8(w, zw, layout, scaling=scaling)
        np.testing.assert_array_equal(conv.codes.cpu().numpy(), codes)
        wpl = LD.decode_w_staged(conv.w_wino.cpu().numpy(), info.cout_pad, info.n_block, info.cin_pad // 32,
                                 info.cin_pad)
        np.testing.assert_array_equal(wpl[:, :co, :ci], LD.complex_to_planes(Wp))
        if info.n_chunks == 1:
            T = int(info.tiles)
            vpl = LD.decode_v(conv.v_image().cpu().numpy(), T, info.cin_pad // 32, info.cin_pad)
            np.testing.assert_array_equal(vpl[:, :, :ci], LD.complex_to_planes(O.input_transform_u8(x, zx, pad, layout)))
            ms = LD.decode_m(conv.m_raw().cpu().numpy(), T, co, info.cout_pad, info.n_block, info.chunk_tiles_pad)
            Mo = ref.Mpp.transpose(2, 0, 1, 3)
            np.testing.assert_array_equal(ms[:16], Mo[LD.REAL_POS, :, :, 0])
            np.testing.assert_array_equal(ms[16:26], Mo[LD.CPX_POS, :, :, 0])
            np.testing.assert_array_equal(ms[26:36], Mo[LD.CPX_POS, :, :, 1])


@pytest.mark.parametrize("case", [
    (2, 40, 37, 17, 70, 1, O.NHWC, 128, 128), (1, 23, 30, 64, 16, 0, O.NHWC, 0, 255), (3, 13, 9, 3, 5, 1, O.NCHW, 255, 0),
    (1, 3, 3, 1, 1, 0, O.NHWC, 7, 200), (2, 1, 1, 2, 3, 1, O.NCHW, 128, 1), (4, 18, 18, 96, 128, 1, O.NHWC, 100, 140),
    (1, 9, 10, 224, 40, 1, O.NHWC, 128, 128)])
@pytest.mark.parametrize("scaling", [False, True])
@pytest.mark.parametrize("path", ["staged", "fused"])
def test_u8_random_shapes(case, scaling, path):
    import paper_1901_01965_b200 as W
    n, h, wd, ci, co, pad, layout, zx, zw = case
    rng = np.random.default_rng(zlib.crc32(repr((case, scaling, "u8")).encode()))
    x, w = _layer(rng, n, h, wd, ci, co, layout)
    _check(x, w, zx, zw, layout, pad, scaling, path=W.WINO_PATH_STAGED if path == "staged" else W.WINO_PATH_FUSED)


@pytest.mark.parametrize("xv,zx,wv,zw", [(0, 255, 255, 0), (255, 0, 0, 255), (255, 0, 255, 0), (0, 255, 0, 255)])
@pytest.mark.parametrize("scaling", [False, True])
@pytest.mark.parametrize("path", ["staged", "fused"])
def test_u8_int9_extremes(xv, zx, wv, zw, scaling, path):
    """The int9 corners: |x - zx| = |w - zw| = 255 everywhere (Winograd-domain values up to 4080, the
    8/128 scale factor and its q = 3 inverse, A27), at the plan's maximum c_in for some cases."""
    import paper_1901_01965_b200 as W
    p = W.WINO_PATH_STAGED if path == "staged" else W.WINO_PATH_FUSED
    for ci in (40, 224):
        x = np.full((1, 10, 11, ci), xv, np.uint8); w = np.full((8, 3, 3, ci), wv, np.uint8)
        _check(x, w, zx, zw, O.NHWC, 1, scaling, intermediates=ci == 40, path=p)


@pytest.mark.parametrize("path", ["staged", "fused"])
def test_u8_int8_requant(path):
    import paper_1901_01965_b200 as W
    rng = np.random.default_rng(51)
    x, w = _layer(rng, 2, 15, 14, 24, 32, O.NHWC)
    p = W.WINO_PATH_STAGED if path == "staged" else W.WINO_PATH_FUSED
    conv = W.WinoConv2d(2, 15, 14, 24, 32, 1, O.NHWC, True, W.WINO_OUT_INT8, path=p,
                        input_type=W.WINO_IN_UINT8, x_zero_point=120, w_zero_point=135)
    conv.transform_filter(torch.from_numpy(w).cuda())
    xd = torch.from_numpy(x).cuda()
    for M0, S in [(1, 0), (1, 13), (3, 14)]:
        np.testing.assert_array_equal(conv(xd, M0, S).cpu().numpy(),
                                      O.wino_conv_u8(x, w, 120, 135, 1, O.NHWC, True, M0=M0, S=S).y8)


@pytest.mark.parametrize("path", ["staged", "fused"])
def test_u8_with_zero_point_128_equals_int8_mode(path):
    """uint8 tensors x + 128, w + 128 with zero points 128 are the int8 tensors: identical outputs."""
    import paper_1901_01965_b200 as W
    import synth
    x, w = synth.config_inputs("C2", n=2)
    S = synth.requant_shift(synth.CONFIGS["C2"].layers[0])
    p = W.WINO_PATH_STAGED if path == "staged" else W.WINO_PATH_FUSED
    outs = []
    for it in (W.WINO_IN_INT8, W.WINO_IN_UINT8):
        conv = W.WinoConv2d(2, 56, 56, 64, 64, 1, W.WINO_NHWC, True, W.WINO_OUT_INT8, path=p,
                            input_type=it, x_zero_point=128 if it else 0, w_zero_point=128 if it else 0)
        sh = (lambda a: (a.astype(np.int16) + 128).astype(np.uint8)) if it else (lambda a: a)
        conv.transform_filter(torch.from_numpy(sh(w)).cuda())
        outs.append(conv(torch.from_numpy(sh(x)).cuda(), 1, S).cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])


# ---------------------------------------------------------------- F(2x2) x uint8 (the paper's evaluated configuration)
@pytest.mark.parametrize("case", [
    (2, 40, 37, 17, 70, 1, O.NHWC, 128, 128), (1, 23, 30, 64, 16, 0, O.NHWC, 0, 255), (3, 13, 9, 3, 5, 1, O.NCHW, 255, 0),
    (1, 3, 3, 1, 1, 0, O.NHWC, 7, 200), (4, 18, 18, 96, 128, 1, O.NHWC, 100, 140), (1, 9, 10, 224, 40, 1, O.NHWC, 128, 128)])
@pytest.mark.parametrize("scaling", [False, True])
@pytest.mark.parametrize("path", ["staged", "fused"])
def test_f2_u8_random_shapes(case, scaling, path):
    import paper_1901_01965_b200 as W
    n, h, wd, ci, co, pad, layout, zx, zw = case
    rng = np.random.default_rng(zlib.crc32(repr((case, scaling, "f2u8")).encode()))
    x, w = _layer(rng, n, h, wd, ci, co, layout)
    conv = W.WinoConv2d(n, h, wd, ci, co, pad, layout, scaling, W.WINO_OUT_INT32,
                        path=W.WINO_PATH_STAGED if path == "staged" else W.WINO_PATH_FUSED,
                        algorithm=W.WINO_ALG_F2X2, input_type=W.WINO_IN_UINT8, x_zero_point=zx, w_zero_point=zw)
    conv.transform_filter(torch.from_numpy(w).cuda())
    y = conv(torch.from_numpy(x).cuda()).cpu().numpy()
    np.testing.assert_array_equal(y, O.wino2_conv_u8(x, w, zx, zw, pad, layout, scaling=scaling).out32)
    np.testing.assert_array_equal(conv.codes.cpu().numpy(), O.filter_transform2_u8(w, zw, layout, scaling=scaling)[2])
    if not scaling:
        np.testing.assert_array_equal(y.astype(np.int64), O.direct_conv_u8(x, w, zx, zw, pad, layout))


@pytest.mark.parametrize("path", ["staged", "fused"])
def test_f2_u8_int9_extremes_and_requant(path):
    import paper_1901_01965_b200 as W
    p = W.WINO_PATH_STAGED if path == "staged" else W.WINO_PATH_FUSED
    for xv, zx, wv, zw in [(0, 255, 255, 0), (255, 0, 255, 0)]:
        x = np.full((1, 10, 11, 224), xv, np.uint8); w = np.full((8, 3, 3, 224), wv, np.uint8)
        conv = W.WinoConv2d(1, 10, 11, 224, 8, 1, O.NHWC, True, W.WINO_OUT_INT8, path=p, algorithm=W.WINO_ALG_F2X2,
                            input_type=W.WINO_IN_UINT8, x_zero_point=zx, w_zero_point=zw)
        conv.transform_filter(torch.from_numpy(w).cuda())
        for M0, S in [(1, 12), (3, 16)]:
            np.testing.assert_array_equal(conv(torch.from_numpy(x).cuda(), M0, S).cpu().numpy(),
                                          O.wino2_conv_u8(x, w, zx, zw, 1, O.NHWC, True, M0=M0, S=S).y8)
