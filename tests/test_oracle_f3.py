"""Pins of the oracle's int8-native scaling target (A29): target 127 on
|W| at real positions and 126 on |Re| + |Im| at complex positions, factors n/2^p with n in [8,15],
p in [4,8], 7-bit codes.  Not in the paper (it uses 255); nothing here calls the CUDA path."""
import itertools
from fractions import Fraction

import numpy as np

import synth
from oracle import oracle as O


def test_scale_factor_brute_force_int8_targets():
    """The A3 formula with targets 127 / 126 equals the largest n/2^p <= target/mx (n in [8,15],
    p in [4,8]) for every reachable max magnitude, and leaves mx <= target unscaled."""
    grid = sorted({(Fraction(n, 2 ** p), n, p) for n in range(8, 16) for p in range(4, 9)})
    for target in (127, 126):
        assert O.scale_factor(target, target) == (0, 0)
        for mx in range(target + 1, 2049):
            n, p = O.scale_factor(mx, target)
            best = max((g for g in grid if g[0] * mx <= target), key=lambda g: (g[0], -g[2]))
            assert Fraction(n, 2 ** p) == best[0], (target, mx)
            assert 8 <= n <= 15 and 4 <= p <= 8


def test_code7_round_trip():
    for n in range(8, 16):
        for p in range(4, 9):
            c = O.encode_code7(n, p)
            assert 64 <= c <= 127 and O.decode_code7(c) == (n, p)
    assert O.encode_code7(0, 0) == 0 and O.decode_code7(0) == (0, 0)


def test_reverse_factor_exists_for_every_int8_target_factor():
    for target in (127, 126):
        for mx in range(target + 1, 2049):
            n, p = O.scale_factor(mx, target)
            m, q = O.reverse_factor(n, p)
            assert 1 <= m <= 255 and 3 <= q <= 7


def _complex_positions():
    return [r * 6 + c for r in range(6) for c in range(6) if r in (3, 4) or c in (3, 4)]


def test_scaled_weights_fit_single_int8_pieces():
    """Every scaled real value fits s8 (|W'| <= 127) and every complex one keeps |Re'| + |Im'| <= 127,
    so Re', Im' and the Karatsuba sum Re' + Im' are single s8 operands -- on random layers and on
    sign-vertex filters (the extremes of Appendix A)."""
    rng = np.random.default_rng(61)
    cpx = _complex_positions()
    real = [p for p in range(36) if p not in cpx]
    filters = [synth.random_layer(rng, 1, 4, 4, ci, co, O.NHWC)[1] for ci, co in [(16, 8), (64, 4), (3, 5)]]
    for signs in itertools.islice(itertools.product((-128, 127), repeat=9), 0, 512, 7):
        filters.append(np.array(signs, np.int8).reshape(1, 3, 3, 1))
    for w in filters:
        _, Wp, codes = O.filter_transform(w, O.NHWC, True, target=127)
        assert np.abs(Wp[:, :, real, 0]).max() <= 127 and not Wp[:, :, real, 1].any()
        s = np.abs(Wp[:, :, cpx, 0]) + np.abs(Wp[:, :, cpx, 1])
        assert s.max() <= 127
        assert np.abs(Wp[:, :, cpx, 0] + Wp[:, :, cpx, 1]).max() <= 127
        for c in np.unique(codes):
            if c:
                n, p = O.decode_code7(int(c)); assert 8 <= n <= 15 and 4 <= p <= 8


def test_int8_target_pipeline_invariants_and_error():
    """Im Y == 0 and int32 ranges hold (asserted inside the oracle); the error against direct
    convolution stays below 2 % of mean |y| and exceeds the paper target's (the cost of the
    single-piece operands)."""
    rng = np.random.default_rng(62)
    for (n, h, w, ci, co) in [(1, 12, 9, 6, 5), (2, 16, 16, 32, 8)]:
        x, wt = synth.random_layer(rng, n, h, w, ci, co, O.NHWC)
        ref = O.direct_conv(x, wt, 1, O.NHWC)
        e127 = np.abs(O.wino_conv(x, wt, 1, O.NHWC, True, target=127).out32 - ref).mean()
        e255 = np.abs(O.wino_conv(x, wt, 1, O.NHWC, True).out32 - ref).mean()
        assert e127 <= 0.02 * np.abs(ref).mean()
        assert e127 >= e255
