"""Pins of the oracle's rational F(2x2,3x3) pipeline against what
the paper prints for its worked example and the closed forms.
Nothing here calls the CUDA path."""
import itertools
import os

import numpy as np
import pytest

import synth
from oracle import analysis as A
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _sec41():
    blocks, cur = {}, None
    for line in open(os.path.join(GOLD, "sec41_ranges.txt")):
        if line.startswith("#") or not line.strip():
            continue
        if line.strip()[0].isalpha():
            cur = line.strip(); blocks[cur] = []
        else:
            blocks[cur].append([int(v) for v in line.split()])
    return {k: np.array(v) for k, v in blocks.items()}


def test_filter_tile2_matches_printed_expansion():
    """G'g row by row (2g0j | g0j+g1j+g2j | g0j-g1j+g2j | 2g2j), p_i its
    elements row-major, and G'gG'^T row i = (2p_{3i}, p_{3i}+p_{3i+1}+p_{3i+2},
    p_{3i}-p_{3i+1}+p_{3i+2}, 2p_{3i+2})."""
    rng = np.random.default_rng(21)
    for _ in range(200):
        g = rng.integers(-255, 256, (3, 3))
        Gg = np.array([[2 * g[0, j] for j in range(3)],
                       [g[0, j] + g[1, j] + g[2, j] for j in range(3)],
                       [g[0, j] - g[1, j] + g[2, j] for j in range(3)],
                       [2 * g[2, j] for j in range(3)]])
        p = Gg.reshape(12)
        want = np.array([[2 * p[3 * i], p[3 * i] + p[3 * i + 1] + p[3 * i + 2], p[3 * i] - p[3 * i + 1] + p[3 * i + 2],
                          2 * p[3 * i + 2]] for i in range(4)])
        np.testing.assert_array_equal(O.filter_tile2(g), want)


def test_filter_tile2_worst_case_magnitudes_and_bits():
    """P:290-304 by vertex enumeration through the oracle's own F(2x2) filter tile
    (int9 weights in [-255, 255]): magnitude and bit-width matrices as printed."""
    b = _sec41()
    best = np.zeros((4, 4), np.int64)
    for signs in itertools.product((-1, 1), repeat=9):
        best = np.maximum(best, np.abs(O.filter_tile2(np.array(signs).reshape(3, 3) * 255)))
    np.testing.assert_array_equal(best, b["magnitude"])
    np.testing.assert_array_equal(np.vectorize(A.signed_bits)(best), b["bits"])
    assert best.max() == 2295 == 9 * 255


def test_input_tile2_fits_11_bits():
    """the activation transform B^T d B fits 11 bits for int9 (uint8 - zero point)
    activations, through the oracle's F(2x2) input tile."""
    best = 0
    for signs in itertools.product((-1, 1), repeat=16):
        best = max(best, int(np.abs(O.input_tile2(np.array(signs).reshape(4, 4) * 255)).max()))
    assert best == 4 * 255 and A.signed_bits(best) == 11


def _corr2(d, g):
    return np.array([[sum(d[i + u, j + v] * g[u, v] for u in range(3) for v in range(3)) for j in range(2)]
                     for i in range(2)])


def test_tile_identity_is_4_times_correlation():
    """A^T[(G'gG'^T) (.) (B^T d B)]A = 4 * (2x2 correlation of the 4x4 patch) exactly (G' = 2G);
    fails for the flipped (convolution) kernel."""
    rng = np.random.default_rng(22)
    flipped_ok = 0
    for _ in range(300):
        d = rng.integers(-128, 128, (4, 4)); g = rng.integers(-128, 128, (3, 3))
        Y = O.output_tile2(O.filter_tile2(g) * O.input_tile2(d))
        np.testing.assert_array_equal(Y, 4 * _corr2(d, g))
        flipped_ok += int(np.array_equal(Y, 4 * _corr2(d, g[::-1, ::-1])))
    assert flipped_ok < 5
    for signs in itertools.product((-1, 1), repeat=4):   # extremes on a few taps
        d = np.full((4, 4), 127); d[0, :] = np.array(signs) * 128 - (np.array(signs) > 0)
        g = np.full((3, 3), -128)
        np.testing.assert_array_equal(O.output_tile2(O.filter_tile2(g) * O.input_tile2(d)), 4 * _corr2(d, g))


@pytest.mark.parametrize("layout", [O.NHWC, O.NCHW])
def test_unscaled_f2_equals_direct(layout):
    rng = np.random.default_rng(23)
    for (n, h, w, ci, co, pad) in [(1, 5, 7, 3, 2, 1), (2, 9, 4, 5, 3, 0), (1, 3, 3, 1, 1, 0), (2, 1, 2, 2, 2, 1),
                                   (1, 12, 11, 17, 9, 1)]:
        x, wt = synth.random_layer(rng, n, h, w, ci, co, layout)
        r = O.wino2_conv(x, wt, pad, layout, scaling=False)
        np.testing.assert_array_equal(r.out32.astype(np.int64), O.direct_conv(x, wt, pad, layout))


def test_unscaled_f2_extremes():
    for xv, wv in [(-128, -128), (127, 127), (-128, 127)]:
        x = np.full((1, 6, 5, 40), xv, np.int8); w = np.full((3, 3, 3, 40), wv, np.int8)
        np.testing.assert_array_equal(O.wino2_conv(x, w, 1, O.NHWC, scaling=False).out32.astype(np.int64),
                                      O.direct_conv(x, w, 1, O.NHWC))


def test_scaled_f2_invariants():
    """Scaling on (P:312-330 with 16 positions): |W'| <= 255, every scaled code has n in [8,15]
    and p in [4,7], int8 weights reach the centre maximum 9*128 = 1152 > 255 so scaling happens,
    and the error against direct convolution is small."""
    rng = np.random.default_rng(24)
    for (n, h, w, ci, co) in [(1, 12, 9, 6, 5), (2, 8, 8, 16, 3)]:
        x, wt = synth.random_layer(rng, n, h, w, ci, co, O.NHWC)
        W, Wp, codes = O.filter_transform2(wt, O.NHWC, scaling=True)
        assert np.abs(W).max() <= 9 * 128 and np.abs(Wp).max() <= 255
        assert (codes > 0).any()
        for c in np.unique(codes):
            if c:
                nn, pp = O.decode_code(int(c)); assert 8 <= nn <= 15 and 4 <= pp <= 7
        res = O.wino2_conv(x, wt, 1, O.NHWC, scaling=True)
        ref = O.direct_conv(x, wt, 1, O.NHWC)
        assert np.abs(res.out32 - ref).mean() <= 0.01 * np.abs(ref).mean()


def test_scaled_f2_power_of_two_case_is_exact():
    """Single-tap filters with taps in {0, +-8, +-120}: G'gG'^T = a G'[:,k] G'[:,l]^T has entries
    a x {1, 2, 4}; a position whose max is 480 gets n/2^p = 8/16 = 1/2 (exact inverse 128/64) on
    even weights, every other position is unscaled -- scaling is lossless, so the scaled pipeline
    must equal direct convolution exactly."""
    rng = np.random.default_rng(25)
    seen = 0
    for _ in range(8):
        ci, co = int(rng.integers(1, 6)), int(rng.integers(1, 5))
        w = np.zeros((co, 3, 3, ci), np.int8)
        for o in range(co):
            for i in range(ci):
                k, l = rng.integers(0, 3, 2)
                w[o, k, l, i] = rng.choice([0, 8, -8, 120, -120])
        x = rng.integers(-128, 128, (2, 9, 10, ci)).astype(np.int8)
        _, _, codes = O.filter_transform2(w, O.NHWC, scaling=True)
        for c in np.unique(codes):
            if c:
                assert O.decode_code(int(c)) == (8, 4)
        seen += int((codes > 0).sum())
        np.testing.assert_array_equal(O.wino2_conv(x, w, 1, O.NHWC, scaling=True).out32.astype(np.int64),
                                      O.direct_conv(x, w, 1, O.NHWC))
    assert seen > 0
