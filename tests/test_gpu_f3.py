"""GPU parity of the int8-native scaling target (A29; staged complex
F(4x4), filter_target_max = 127) against the oracle's target-127 pipeline: 7-bit codes, the
single-piece W' image, V and M'' exact, y bit-exact (int32 and requantised int8)."""
import zlib

import numpy as np
import pytest
import torch

import synth
from oracle import oracle as O
import layout_decode as LD

pytestmark = pytest.mark.gpu


def _conv(n, h, wd, ci, co, pad, layout, out_mode):
    import paper_1901_01965_b200 as W
    return W.WinoConv2d(n, h, wd, ci, co, pad, layout, True, out_mode, path=W.WINO_PATH_STAGED,
                        filter_target_max=127)


def _check(x, w, layout, pad=1, intermediates=True):
    import paper_1901_01965_b200 as W
    if layout == O.NCHW:
        n, ci, h, wd = x.shape
    else:
        n, h, wd, ci = x.shape
    co = w.shape[0]
    conv = _conv(n, h, wd, ci, co, pad, layout, W.WINO_OUT_INT32)
    conv.transform_filter(torch.from_numpy(w).cuda())
    y = conv(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = O.wino_conv(x, w, pad, layout, True, target=127, want_M=intermediates)
    _, Wp, codes = O.filter_transform(w, layout, True, target=127)
    np.testing.assert_array_equal(conv.codes.cpu().numpy(), codes)
    np.testing.assert_array_equal(y, ref.out32)
    if intermediates:
        info = conv.info
        assert info.filter_bytes == 46 * info.cout_pad * info.cin_pad   # one s8 piece per plane
        wpl = LD.decode_w1(conv.w_wino.cpu().numpy(), info.cout_pad, info.n_block, info.cin_pad // 32, info.cin_pad)
        np.testing.assert_array_equal(wpl[:, :co, :ci], LD.complex_to_planes(Wp))
        assert not wpl[:, co:, :].any() and not wpl[:, :, ci:].any()      # zero padding rows / channels
        if info.n_chunks == 1:
            T = int(info.tiles)
            ms = LD.decode_m(conv.m_raw().cpu().numpy(), T, co, info.cout_pad, info.n_block, info.chunk_tiles_pad)
            Mo = ref.Mpp.transpose(2, 0, 1, 3)
            np.testing.assert_array_equal(ms[:16], Mo[LD.REAL_POS, :, :, 0])
            np.testing.assert_array_equal(ms[16:26], Mo[LD.CPX_POS, :, :, 0])
            np.testing.assert_array_equal(ms[26:36], Mo[LD.CPX_POS, :, :, 1])
    return conv


@pytest.mark.parametrize("case", [
    (2, 40, 37, 17, 70, 1, O.NHWC), (1, 23, 30, 64, 16, 0, O.NHWC), (3, 13, 9, 3, 5, 1, O.NCHW),
    (1, 3, 3, 1, 1, 0, O.NHWC), (2, 1, 1, 2, 3, 1, O.NCHW), (4, 18, 18, 96, 128, 1, O.NHWC),
    (1, 9, 10, 200, 40, 1, O.NHWC), (2, 20, 20, 48, 33, 1, O.NCHW)])
def test_f3_random_shapes(case):
    n, h, wd, ci, co, pad, layout = case
    rng = np.random.default_rng(zlib.crc32(repr((case, "f3")).encode()))
    x, w = synth.random_layer(rng, n, h, wd, ci, co, layout)
    _check(x, w, layout, pad)


@pytest.mark.parametrize("xv,wv", [(-128, -128), (127, 127), (-128, 127)])
def test_f3_extremes_at_max_cin(xv, wv):
    """Constant extremes (every position scaled, the (15, 8) factor at the (0,0) corner, q = 3
    inverses) at c_in = 40 with intermediates and at the plan's scaled maximum 768."""
    for ci in (40, 768):
        x = np.full((1, 6, 7, ci), xv, np.int8); w = np.full((4, 3, 3, ci), wv, np.int8)
        _check(x, w, O.NHWC, 1, intermediates=ci == 40)


def test_f3_sign_vertex_filters():
    """Sign-vertex filters (the Appendix A extremes) over many couts: every code class appears."""
    rng = np.random.default_rng(63)
    co, ci = 96, 32
    w = np.where(rng.integers(0, 2, (co, 3, 3, ci)) == 1, 127, -128).astype(np.int8)
    x = rng.integers(-128, 128, (2, 17, 19, ci)).astype(np.int8)
    _check(x, w, O.NHWC, 1)


def test_f3_int8_requant_full_size_sampled():
    """C2's full layer shape (batch 16 here, chunked like bench) with int8 requantisation, y8 bit-exact
    on sampled output pixels recomputed by the oracle on their receptive fields."""
    import paper_1901_01965_b200 as W
    x, w = synth.config_inputs("C2", n=16)
    S = synth.requant_shift(synth.CONFIGS["C2"].layers[0])
    n, h, wd, ci = x.shape
    conv = _conv(n, h, wd, ci, w.shape[0], 1, O.NHWC, W.WINO_OUT_INT8)
    conv.transform_filter(torch.from_numpy(w).cuda())
    y = conv(torch.from_numpy(x).cuda(), 1, S).cpu().numpy()
    rng = np.random.default_rng(64)
    for _ in range(12):
        b, ty, tx = int(rng.integers(0, n)), int(rng.integers(0, h // 4)), int(rng.integers(0, wd // 4))
        # the 6x6 input patch of output tile (ty, tx) with its zero padding, as a 1-image 4x4-output layer
        xp = np.zeros((1, 6, 6, ci), np.int8)
        for r in range(6):
            for c in range(6):
                yy, xx = 4 * ty + r - 1, 4 * tx + c - 1
                if 0 <= yy < h and 0 <= xx < wd:
                    xp[0, r, c] = x[b, yy, xx]
        ref = O.wino_conv(xp, w, 0, O.NHWC, True, target=127, M0=1, S=S)
        np.testing.assert_array_equal(y[b, 4 * ty:4 * ty + 4, 4 * tx:4 * tx + 4], ref.y8[0])


def test_f3_error_close_to_paper_target():
    """The single-piece target costs accuracy: the GPU int32 outputs stay within 2 % mean |y| of direct
    convolution and are no closer than the paper's target 255 (same numbers as the oracle pin)."""
    import paper_1901_01965_b200 as W
    rng = np.random.default_rng(65)
    x, w = synth.random_layer(rng, 2, 16, 16, 64, 32, O.NHWC)
    ref = O.direct_conv(x, w, 1, O.NHWC)
    errs = []
    for tgt in (127, 255):
        conv = W.WinoConv2d(2, 16, 16, 64, 32, 1, O.NHWC, True, W.WINO_OUT_INT32, path=W.WINO_PATH_STAGED,
                            filter_target_max=tgt)
        conv.transform_filter(torch.from_numpy(w).cuda())
        errs.append(np.abs(conv(torch.from_numpy(x).cuda()).cpu().numpy() - ref).mean())
    assert errs[0] <= 0.02 * np.abs(ref).mean() and errs[0] >= errs[1]
