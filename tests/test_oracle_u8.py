"""Pins of the oracle's uint8 + zero-point mode (the paper's affine
quantisation model): int9 values after subtracting the zero points, the 13-bit
Winograd-domain weights of P:372 scaled back to 9 bits, and the q = 3 inverse corner
(A27).  Nothing here calls the CUDA path."""
from fractions import Fraction

import numpy as np
import pytest
import torch

from oracle import analysis as A
from oracle import oracle as O


def _u8_layer(rng, n, h, w, ci, co, layout):
    x = rng.integers(0, 256, (n, h, w, ci), dtype=np.int64).astype(np.uint8)
    wt = rng.integers(0, 256, (co, 3, 3, ci), dtype=np.int64).astype(np.uint8)
    if layout == O.NCHW:
        x = np.ascontiguousarray(x.transpose(0, 3, 1, 2)); wt = np.ascontiguousarray(wt.transpose(0, 3, 1, 2))
    return x, wt


@pytest.mark.parametrize("layout", [O.NHWC, O.NCHW])
@pytest.mark.parametrize("pad", [0, 1])
def test_direct_conv_u8_matches_torch_float64(layout, pad):
    """O1 on int9 values: torch conv2d in float64 on (x - zx), (w - zw); padding is real zero."""
    rng = np.random.default_rng(41)
    for zx, zw in [(0, 0), (128, 131), (255, 7)]:
        x, w = _u8_layer(rng, 2, 9, 8, 5, 3, layout)
        xt = torch.from_numpy(x.astype(np.float64) - zx); wt = torch.from_numpy(w.astype(np.float64) - zw)
        if layout == O.NHWC:
            xt = xt.permute(0, 3, 1, 2); wt = wt.permute(0, 3, 1, 2)
        ref = torch.nn.functional.conv2d(xt, wt, padding=pad)
        if layout == O.NHWC:
            ref = ref.permute(0, 2, 3, 1)
        np.testing.assert_array_equal(O.direct_conv_u8(x, w, zx, zw, pad, layout), ref.numpy().astype(np.int64))


@pytest.mark.parametrize("layout", [O.NHWC, O.NCHW])
def test_unscaled_u8_winograd_equals_direct(layout):
    rng = np.random.default_rng(42)
    for (n, h, w, ci, co, pad), (zx, zw) in zip([(1, 9, 7, 4, 3, 1), (2, 6, 11, 16, 5, 0), (1, 13, 13, 40, 2, 1)],
                                                 [(128, 128), (0, 255), (77, 3)]):
        x, wt = _u8_layer(rng, n, h, w, ci, co, layout)
        r = O.wino_conv_u8(x, wt, zx, zw, pad, layout, scaling=False)
        np.testing.assert_array_equal(r.out32.astype(np.int64), O.direct_conv_u8(x, wt, zx, zw, pad, layout))


def test_u8_extremes_unscaled():
    """int9 extremes (-255 / +255 after the zero points) through the complex F(4x4)."""
    for xv, zx, wv, zw in [(0, 255, 255, 0), (255, 0, 0, 255), (255, 0, 255, 0)]:
        x = np.full((1, 8, 9, 24), xv, np.uint8); w = np.full((3, 3, 3, 24), wv, np.uint8)
        np.testing.assert_array_equal(O.wino_conv_u8(x, w, zx, zw, 1, O.NHWC, scaling=False).out32.astype(np.int64),
                                      O.direct_conv_u8(x, w, zx, zw, 1, O.NHWC))


def test_int9_weights_reach_13_bits_and_scale_to_9():
    """P:372 on the complex F(4x4): int9 weights give |W| up to 4080 = 16*255 (13-bit signed, the
    corner positions) and the scaled W' fits 9 bits: the 30.77 % filter bit-width reduction."""
    w = np.zeros((2, 3, 3, 3), np.uint8)          # cout 0: corner taps at +255 (w = 255, zw = 0) -> g = 255
    w[0, 0, 0, :] = 255; w[1, :, :, :] = 0        # cout 1: all g = -255 (zw = 255)
    W, Wp, codes = O.filter_transform_u8(w[:1], 0, O.NHWC, scaling=True)
    assert np.abs(W).max() == 16 * 255 and A.signed_bits(16 * 255) == 13
    assert np.abs(Wp).max() <= 255 and A.signed_bits(int(np.abs(Wp).max())) <= 9
    W2, Wp2, _ = O.filter_transform_u8(w[1:], 255, O.NHWC, scaling=True)
    assert np.abs(Wp2).max() <= 255
    assert Fraction(13 - 9, 13) == Fraction(4, 13) and round(100 * 4 / 13, 2) == 30.77


def test_reverse_factor_q3_corner():
    """A27: the 8/128 factor (max magnitude 4080) needs q = 3: m = 128, 128/2^3 = 16 = 128/8 exactly;
    every factor emitted for int9 maxima in (255, 4080] has an 8-bit inverse with q maximal."""
    assert O.scale_factor(4080) == (8, 7)
    assert O.reverse_factor(8, 7) == (128, 3)
    for mx in range(256, 4081):
        n, p = O.scale_factor(mx)
        m, q = O.reverse_factor(n, p)
        assert 1 <= m <= 255 and 3 <= q <= 7
        assert abs(Fraction(m) - Fraction(2 ** (q + p), n)) <= Fraction(1, 2)
        if q < 7:
            assert int(Fraction(2 ** (q + 1 + p), n) + Fraction(1, 2)) > 255
        if (n, p) != (8, 7):
            assert q >= 4      # the int8 reading (A8) is unchanged


def test_scaled_u8_invariants_and_error():
    rng = np.random.default_rng(43)
    for zx, zw in [(128, 128), (10, 250)]:
        x, wt = _u8_layer(rng, 2, 10, 9, 12, 4, O.NHWC)
        W, Wp, codes = O.filter_transform_u8(wt, zw, O.NHWC, scaling=True)
        assert np.abs(Wp).max() <= 255 and (codes > 0).any()
        res = O.wino_conv_u8(x, wt, zx, zw, 1, O.NHWC, scaling=True)
        ref = O.direct_conv_u8(x, wt, zx, zw, 1, O.NHWC)
        assert np.abs(res.out32 - ref).mean() <= 0.01 * np.abs(ref).mean()


# ---------------------------------------------------------------- F(2x2) x uint8: the paper's evaluated configuration
@pytest.mark.parametrize("layout", [O.NHWC, O.NCHW])
def test_unscaled_f2_u8_equals_direct(layout):
    """Unscaled F(2x2) on uint8 tensors with zero points equals the direct correlation of the int9 values."""
    rng = np.random.default_rng(71)
    for (n, h, w, ci, co, pad, zx, zw) in [(1, 7, 9, 5, 3, 1, 128, 128), (2, 6, 5, 3, 4, 0, 0, 255),
                                           (1, 3, 3, 2, 2, 1, 255, 0), (1, 12, 11, 17, 9, 1, 7, 200)]:
        x = rng.integers(0, 256, (n, h, w, ci), dtype=np.int64).astype(np.uint8)
        wt = rng.integers(0, 256, (co, 3, 3, ci), dtype=np.int64).astype(np.uint8)
        if layout == O.NCHW:
            x = np.ascontiguousarray(x.transpose(0, 3, 1, 2)); wt = np.ascontiguousarray(wt.transpose(0, 3, 1, 2))
        r = O.wino2_conv_u8(x, wt, zx, zw, pad, layout, scaling=False)
        np.testing.assert_array_equal(r.out32.astype(np.int64), O.direct_conv_u8(x, wt, zx, zw, pad, layout))


def test_scaled_f2_u8_reaches_the_papers_section41_corner():
    """P:290-330 on int9 weights: the centre position reaches 9 * 255 = 2295 (12 bits), scaled by the 14/128
    factor the paper prints; every W' fits 9 bits; the error against direct convolution stays small."""
    x = np.full((1, 6, 6, 8), 255, np.uint8); w = np.full((4, 3, 3, 8), 255, np.uint8)
    W, Wp, codes = O.filter_transform2_u8(w, 0, O.NHWC, scaling=True)
    assert int(np.abs(W[..., 5]).max()) == 9 * 255 and int(np.abs(W[..., 0]).max()) == 4 * 255   # centre, corner
    assert O.decode_code(int(codes[0, 5])) == (14, 7)         # position (1,1): 2295 -> 14/128
    assert np.abs(Wp).max() <= 255
    rng = np.random.default_rng(72)
    x = rng.integers(0, 256, (2, 10, 9, 16), dtype=np.int64).astype(np.uint8)
    w = rng.integers(0, 256, (6, 3, 3, 16), dtype=np.int64).astype(np.uint8)
    ref = O.direct_conv_u8(x, w, 120, 130, 1, O.NHWC)
    res = O.wino2_conv_u8(x, w, 120, 130, 1, O.NHWC, scaling=True)
    assert np.abs(res.out32 - ref).mean() <= 0.01 * np.abs(ref).mean()
