"""GPU parity of the rational F(2x2,3x3) path (algorithm = WINO_ALG_F2X2, the staged
kernels and the fused k_fused2) against the oracle's F(2x2) pipeline, element by element: codes, W'
planes, V planes and M'' byte/int exact (staged), y bit-exact (both)."""
import zlib

import numpy as np
import pytest
import torch

import synth
from oracle import oracle as O
import layout_decode as LD

pytestmark = pytest.mark.gpu


PATHS = [pytest.param(2, id="staged"), pytest.param(1, id="fused")]   # WINO_PATH_STAGED / _FUSED


def _conv(n, h, w, ci, co, pad, layout, scaling, out_mode=1, chunk_mb=0, path=2):
    import paper_1901_01965_b200 as W
    return W.WinoConv2d(n, h, w, ci, co, pad, layout, scaling, out_mode, workspace_mb=chunk_mb,
                        path=path, algorithm=W.WINO_ALG_F2X2)


def _check(x, w, layout, pad=1, scaling=True, intermediates=True, path=2):
    intermediates = intermediates and path == 2   # V / W' / M'' decoders: staged layouts
    if layout == O.NCHW:
        n, ci, h, wd = x.shape
    else:
        n, h, wd, ci = x.shape
    co = w.shape[0]
    conv = _conv(n, h, wd, ci, co, pad, layout, scaling, path=path)
    conv.transform_filter(torch.from_numpy(w).cuda())
    y = conv(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = O.wino2_conv(x, w, pad, layout, scaling=scaling, want_M=intermediates)
    np.testing.assert_array_equal(y, ref.out32)
    np.testing.assert_array_equal(conv.codes.cpu().numpy(), O.filter_transform2(w, layout, scaling=scaling)[2])
    if not scaling:
        np.testing.assert_array_equal(y.astype(np.int64), O.direct_conv(x, w, pad, layout))
    if intermediates:
        info = conv.info
        assert info.positions == 16 and info.tile == 2 and info.planes == 16
        _, Wp, codes = O.filter_transform2(w, layout, scaling=scaling)
        np.testing.assert_array_equal(conv.codes.cpu().numpy(), codes)
        wpl = LD.decode_w_staged(conv.w_wino.cpu().numpy(), info.cout_pad, info.n_block, info.cin_pad // 32,
                                 info.cin_pad, nplanes=16)
        np.testing.assert_array_equal(wpl[:, :co, :ci], Wp.transpose(2, 0, 1))
        assert not wpl[:, co:, :].any() and not wpl[:, :, ci:].any()
        if info.n_chunks == 1:
            T = int(info.tiles)
            vpl = LD.decode_v(conv.v_image().cpu().numpy(), T, info.cin_pad // 32, info.cin_pad, nplanes=16)
            np.testing.assert_array_equal(vpl[:, :, :ci], O.input_transform2(x, pad, layout).transpose(2, 0, 1))
            ms = LD.decode_m(conv.m_raw().cpu().numpy(), T, co, info.cout_pad, info.n_block, info.chunk_tiles_pad,
                             slots=16)
            np.testing.assert_array_equal(ms, ref.Mpp.transpose(2, 0, 1))
    return conv


@pytest.mark.parametrize("layout", [O.NHWC, O.NCHW])
@pytest.mark.parametrize("scaling", [False, True])
@pytest.mark.parametrize("path", PATHS)
def test_f2_c1_shape(layout, scaling, path):
    x, w = synth.config_inputs("C1", layout)
    _check(x, w, layout, 1, scaling, path=path)


@pytest.mark.parametrize("case", [
    (2, 40, 37, 17, 70, 1, O.NHWC), (1, 23, 30, 64, 16, 0, O.NHWC), (3, 13, 9, 3, 5, 1, O.NCHW),
    (1, 3, 3, 1, 1, 0, O.NHWC), (2, 1, 1, 2, 3, 1, O.NCHW), (1, 57, 11, 40, 33, 1, O.NCHW),
    (4, 18, 18, 96, 128, 1, O.NHWC), (2, 11, 13, 200, 24, 1, O.NHWC), (1, 9, 9, 300, 40, 1, O.NCHW)])
@pytest.mark.parametrize("scaling", [False, True])
@pytest.mark.parametrize("path", PATHS)
def test_f2_random_shapes(case, scaling, path):
    n, h, wd, ci, co, pad, layout = case
    rng = np.random.default_rng(zlib.crc32(repr((case, scaling, "f2")).encode()))
    x, w = synth.random_layer(rng, n, h, wd, ci, co, layout)
    _check(x, w, layout, pad, scaling, path=path)


@pytest.mark.parametrize("xv,wv", [(-128, -128), (127, 127), (-128, 127)])
@pytest.mark.parametrize("scaling", [False, True])
@pytest.mark.parametrize("path", PATHS)
def test_f2_extremes(xv, wv, scaling, path):
    x = np.full((2, 12, 13, 40), xv, np.int8); w = np.full((24, 3, 3, 40), wv, np.int8)
    _check(x, w, O.NHWC, 1, scaling, path=path)


@pytest.mark.parametrize("path", PATHS)
def test_f2_max_cin(path):
    rng = np.random.default_rng(31)
    for ci, scaling in [(896, False), (768, True)]:
        x = rng.integers(-128, 128, (1, 6, 7, ci)).astype(np.int8)
        w = np.where(rng.integers(0, 2, (3, 3, 3, ci)) == 1, 127, -128).astype(np.int8)
        _check(x, w, O.NHWC, 1, scaling, intermediates=False, path=path)


@pytest.mark.parametrize("layout", [O.NHWC, O.NCHW])
@pytest.mark.parametrize("path", PATHS)
def test_f2_int8_requant_and_chunks(layout, path):
    rng = np.random.default_rng(32)
    x, w = synth.random_layer(rng, 24, 20, 20, 64, 48, layout)
    conv = _conv(24, 20, 20, 64, 48, 1, layout, True, out_mode=0, chunk_mb=1, path=path)
    assert conv.info.n_chunks > 1
    conv.transform_filter(torch.from_numpy(w).cuda())
    xd = torch.from_numpy(x).cuda()
    for M0, S in [(1, 0), (1, 9), (3, 11), (1, 24)]:
        np.testing.assert_array_equal(conv(xd, M0, S).cpu().numpy(),
                                      O.wino2_conv(x, w, 1, layout, True, M0=M0, S=S).y8)


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
@pytest.mark.parametrize("path", PATHS)
def test_f2_full_size_configs_sampled(name, path):
    """BASELINE config shapes with the F(2x2) algorithm, NHWC, int8 out: first, middle and last
    images compared bit-exactly with the oracle run on those images alone."""
    layer = synth.CONFIGS[name].layers[0]
    x, w = synth.config_inputs(name)
    S = synth.requant_shift(layer)
    conv = _conv(layer.n, layer.h, layer.w, layer.c_in, layer.c_out, 1, O.NHWC, True, out_mode=0, path=path)
    conv.transform_filter(torch.from_numpy(w).cuda())
    y = conv(torch.from_numpy(x).cuda(), 1, S).cpu().numpy()
    for i in sorted({0, layer.n // 2, layer.n - 1}):
        np.testing.assert_array_equal(y[i:i + 1], O.wino2_conv(x[i:i + 1], w, 1, O.NHWC, True, M0=1, S=S).y8)
    np.testing.assert_array_equal(conv.codes.cpu().numpy(), O.filter_transform2(w, O.NHWC, True)[2])


def test_f2_fused_plan_reports_its_shape():
    import paper_1901_01965_b200 as W
    conv = W.WinoConv2d(1, 8, 8, 4, 4, 1, W.WINO_NHWC, True, W.WINO_OUT_INT32, path=W.WINO_PATH_FUSED,
                        algorithm=W.WINO_ALG_F2X2)
    i = conv.info
    assert i.path == W.WINO_PATH_FUSED and i.stages == 2 and i.positions == 16 and i.tile == 2 and i.n_block == 32
