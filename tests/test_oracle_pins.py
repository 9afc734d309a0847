"""Pins of the CPU oracle against what the paper and the mathematics fix.

Nothing here calls the CUDA path.  Each test names the passage it pins
(P:n = line n of PAPER.md) or the closed form / library routine used.
"""
import itertools
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

import synth
from oracle import analysis as A
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _read_figures():
    out = {}
    for line in open(os.path.join(GOLD, "paper_figures.txt")):
        if line.startswith("#") or not line.strip():
            continue
        k, v, _cite = line.split()
        out[k] = v
    return out


FIG = _read_figures()


# ----------------------------------------------------------- direct conv
@pytest.mark.parametrize("layout", [O.NCHW, O.NHWC])
@pytest.mark.parametrize("pad", [0, 1])
def test_direct_conv_matches_torch_float64(layout, pad):
    """O1 against torch.nn.functional.conv2d (an independent library routine,
    exact in float64 here since |values| < 2^53)."""
    rng = np.random.default_rng(11 + pad + 10 * layout)
    for n, h, w, ci, co in [(1, 5, 7, 3, 2), (2, 9, 6, 5, 4), (1, 3, 3, 1, 1), (2, 12, 11, 8, 3)]:
        x, wt = synth.random_layer(rng, n, h, w, ci, co, layout)
        got = O.direct_conv(x, wt, pad, layout)
        if layout == O.NHWC:
            xt = torch.from_numpy(x.astype(np.float64)).permute(0, 3, 1, 2)
            wtt = torch.from_numpy(wt.astype(np.float64)).permute(0, 3, 1, 2)
        else:
            xt = torch.from_numpy(x.astype(np.float64)); wtt = torch.from_numpy(wt.astype(np.float64))
        ref = torch.nn.functional.conv2d(xt, wtt, padding=pad)
        if layout == O.NHWC:
            ref = ref.permute(0, 2, 3, 1)
        np.testing.assert_array_equal(got, ref.numpy().astype(np.int64))


def test_direct_conv_hand_examples():
    # all-ones 3x3 input, one channel, no padding -> 9
    x = np.ones((1, 3, 3, 1), np.int8); w = np.ones((1, 3, 3, 1), np.int8)
    assert O.direct_conv(x, w, 0, O.NHWC).item() == 9
    # centre delta filter with pad 1 reproduces the input
    rng = np.random.default_rng(3)
    x = rng.integers(-128, 128, (1, 7, 5, 1)).astype(np.int8)
    w = np.zeros((1, 3, 3, 1), np.int8); w[0, 1, 1, 0] = 1
    np.testing.assert_array_equal(O.direct_conv(x, w, 1, O.NHWC), x.astype(np.int64))


# ----------------------------------------------------------- matrices
def test_bt_rows_match_printed_row_formulas():
    """The oracle's B^T reproduces the separately printed d' = B^T d row
    formulas of P:184-189 (guards against a typo in the P:146-151 matrix)."""
    BT, _, _ = O.matrices()
    rows = []
    for line in open(os.path.join(GOLD, "dtile_rows.txt")):
        if line.startswith("#") or not line.strip():
            continue
        left, right = line.split("|")
        vals = [int(v) for v in left.split()]
        rows.append((vals[0], np.array(vals[1:]), np.array([int(v) for v in right.split()])))
    for r, re, im in rows:
        np.testing.assert_array_equal(BT[r].real, re)
        np.testing.assert_array_equal(BT[r].imag, im)


def test_g_int_is_four_times_printed_g():
    """G_int = 4 G with G from P:154-160 (A2)."""
    _, G, _ = O.matrices()
    printed = np.array([[1, 0, 0], [.25, .25, .25], [.25, -.25, .25], [.25, .25j, -.25],
                        [.25, -.25j, -.25], [0, 0, 1]])
    np.testing.assert_array_equal(G, 4 * printed)


def _valid_corr(d, g):
    return np.array([[np.sum(d[i:i + 3, j:j + 3] * g) for j in range(4)] for i in range(4)])


def test_tile_identity_is_16_times_correlation():
    """Closed form: A^T[(G_int g G_int^T) (.) (B^T d B)]A = 16 * (valid
    correlation of d with g) for every integer tile (A1/A2).
    A kernel flip (true convolution) must NOT satisfy it."""
    rng = np.random.default_rng(5)
    flips_ok = 0
    for trial in range(300):
        g = rng.integers(-128, 128, (3, 3)); d = rng.integers(-128, 128, (6, 6))
        W = O.filter_tile(g); D = O.input_tile(d)
        Wc = W[..., 0] + 1j * W[..., 1]; Dc = D[..., 0] + 1j * D[..., 1]
        Mc = Wc * Dc
        M = np.stack([Mc.real, Mc.imag], -1).astype(np.int64)
        Y, im_zero = O.output_tile(M)
        assert im_zero
        np.testing.assert_array_equal(Y, 16 * _valid_corr(d, g))
        if np.array_equal(Y, 16 * _valid_corr(d, g[::-1, ::-1])):
            flips_ok += 1
    assert flips_ok < 5


def test_tile_identity_adversarial_vertices():
    """Same identity on the sign-vertex extremes that hit the Appendix-A
    range bounds (all -128 / 127 patterns)."""
    for bits in range(64):
        rng = np.random.default_rng(bits)
        g = np.where(rng.integers(0, 2, (3, 3)) == 1, 127, -128)
        d = np.where(rng.integers(0, 2, (6, 6)) == 1, 127, -128)
        if bits == 0:
            g[:] = -128; d[:] = -128
        W = O.filter_tile(g); D = O.input_tile(d)
        Mc = (W[..., 0] + 1j * W[..., 1]) * (D[..., 0] + 1j * D[..., 1])
        Y, ok = O.output_tile(np.stack([Mc.real, Mc.imag], -1).astype(np.int64))
        assert ok
        np.testing.assert_array_equal(Y, 16 * _valid_corr(d, g))


def test_conjugate_layout_of_D_and_W():
    """D and W hold 10 conjugate pairs and 16 real values at the
    positions of DS1 (rows/cols {0,1,2,5} real, 3<->4 mirrored)."""
    R = [0, 1, 2, 5]
    mirror = {0: 0, 1: 1, 2: 2, 5: 5, 3: 4, 4: 3}
    rng = np.random.default_rng(8)
    for _ in range(50):
        for T in (O.input_tile(rng.integers(-128, 128, (6, 6))), O.filter_tile(rng.integers(-128, 128, (3, 3)))):
            for r in range(6):
                for c in range(6):
                    if r in R and c in R:
                        assert T[r, c, 1] == 0
                    else:
                        mr, mc = mirror[r], mirror[c]
                        if (r, c) in ((3, 3), (4, 4)):
                            mr, mc = (4, 4) if r == 3 else (3, 3)
                        if (r, c) in ((3, 4), (4, 3)):
                            mr, mc = (4, 3) if r == 3 else (3, 4)
                        assert T[mr, mc, 0] == T[r, c, 0] and T[mr, mc, 1] == -T[r, c, 1]


def test_layout_read_from_matrices():
    BT, _, _ = O.matrices()
    real, pairs = A.conjugate_layout(BT)
    R = [0, 1, 2, 5]
    assert real == sorted((r, c) for r in R for c in R)
    assert len(pairs) == int(FIG["conjugate_pairs"]) and len(real) == int(FIG["real_positions"])
    prim = {p for p, _ in pairs}
    assert prim == {(0, 3), (1, 3), (2, 3), (5, 3), (3, 0), (3, 1), (3, 2), (3, 5), (3, 3), (3, 4)}


# ----------------------------------------------------------- counts / ratios
def test_general_multiplication_count_and_ratio():
    """46 general multiplications counted from the matrices, 144/46 = 3.13x."""
    BT, _, _ = O.matrices()
    muls = A.general_multiplications(BT)
    assert muls == int(FIG["general_multiplications"])
    direct = 4 * 4 * 3 * 3
    assert direct == int(FIG["direct_multiplications"])
    assert f"{float(A.reduction_ratio(4, 3, muls)):.2f}" == FIG["reduction_complex_f4"]
    assert float(A.reduction_ratio(2, 3, 16)) == float(FIG["reduction_f2"])
    assert float(A.reduction_ratio(4, 3, 36)) == float(FIG["reduction_rational_f4"])


def test_layer_multiplication_count_example():
    """1x8x8x16 input, 8 out channels, pad 1: 4 tiles * 16 * 8 * 46 = 23552 vs
    direct 73728 (ratio 3.13 of P:228)."""
    BT, _, _ = O.matrices()
    th, tw = O.tiles(8, 8, 1)
    wino = th * tw * 16 * 8 * A.general_multiplications(BT)
    assert wino == 23552 and 8 * 8 * 8 * 9 * 16 == 73728


def test_widening_bits():
    """ceil(log2(24^2)) = 10 for rational F(4x4); ceil(log2(4^2)) = 4
    for complex F(4x4); both read off the G matrices."""
    assert A.widening_bits(A.G_RATIONAL_F4) == int(FIG["widening_rational_f4_bits"])
    _, G, _ = O.matrices()
    Gc = [[complex(v) / 4 for v in row] for row in G]
    assert A.widening_bits(Gc) == int(FIG["widening_complex_f4_bits"])


def test_efficiency_gains():
    """33.33% bit-width, 17.37% and 15.93% (computed with the rounded 3.13)."""
    assert f"{100 * (1 - (8 + 4) / (8 + 10)):.2f}" == FIG["bitwidth_reduction_complex_vs_rational_pct"]
    r = round(144 / 46, 2)
    assert f"{100 * A.efficiency_gain(r, 12, 4.0, 18):.2f}" == FIG["efficiency_gain_vs_rational_f4_pct"]
    assert f"{100 * A.efficiency_gain(r, 8 + 4, 2.25, 8 + 2):.2f}" == FIG["efficiency_gain_vs_rational_f2_pct"]
    # exact 144/46 gives 17.39% / 15.94% (A19)
    assert f"{100 * A.efficiency_gain(144 / 46, 12, 4.0, 18):.2f}" == "17.39"


def test_complex_filter_width_is_8_plus_4_bits():
    """Symmetric int8 weights in [-127,127]: max |W| = 2032 -> 12 bits = 8 + 4."""
    mag = A.worst_case_magnitudes_complex(-127, 127)
    assert mag.max() == 2032 and A.signed_bits(int(mag.max())) == 12


# ----------------------------------------------------------- section 4.1
def _read_sec41():
    blocks, cur = {}, None
    for line in open(os.path.join(GOLD, "sec41_ranges.txt")):
        if line.startswith("#") or not line.strip():
            continue
        if line.strip() in ("G'", "magnitude", "bits"):
            cur = line.strip(); blocks[cur] = []; continue
        blocks[cur].append([int(v) for v in line.split()])
    return {k: np.array(v) for k, v in blocks.items()}


def test_section41_worst_case_ranges():
    """worst-case magnitudes / bits of G' g G'^T, int9 weights."""
    b = _read_sec41()
    np.testing.assert_array_equal(A.G_PRIME_F2, b["G'"])
    mag = A.worst_case_magnitudes_generic(A.G_PRIME_F2, 255)
    np.testing.assert_array_equal(mag, b["magnitude"])
    bits = np.vectorize(A.signed_bits)(mag)
    np.testing.assert_array_equal(bits, b["bits"])
    assert mag.max() == int(FIG["max_magnitude_f2_int9"])


def test_section41_activation_transform_bits():
    """the F(2x2) activation transform fits 11 bits (int9 inputs).
    B^T of F(2x2,3x3) with points {0,1,-1} (Lavin & Gray; not printed in the paper)."""
    BT2 = np.array([[1, 0, -1, 0], [0, 1, 1, 0], [0, -1, 1, 0], [0, 1, 0, -1]])
    best = 0
    for signs in itertools.product((-1, 1), repeat=16):
        d = np.array(signs).reshape(4, 4) * 255
        best = max(best, int(np.abs(BT2 @ d @ BT2.T).max()))
    assert A.signed_bits(best) == int(FIG["activation_transform_bits_f2"])


def test_filter_bitwidth_reduction_30_77():
    """13 -> 9 bits = 30.77% for int9 weights; also holds on the complex
    F(4x4) path (corner 16*255 = 4080 needs 13 bits) once scaled to <= 255."""
    assert A.signed_bits(int(FIG["max_magnitude_f2_int9"])) == int(FIG["unscaled_filter_bits_int9_f2"])
    mag = A.worst_case_magnitudes_complex(-255, 255)
    assert mag.max() == 4080 and A.signed_bits(4080) == 13
    assert A.signed_bits(255) == int(FIG["scaled_filter_bits"])
    assert f"{100 * (1 - 9 / 13):.2f}" == FIG["filter_bitwidth_reduction_pct"]
    # every magnitude up to 4080 gets a factor that lands it in [-255, 255]
    for mx in range(256, 4081):
        n, p = O.scale_factor(mx)
        assert Fraction(n, 2 ** p) * mx <= 255


# ----------------------------------------------------------- scale factors
def _brute_force_factor(mx):
    best = None
    for n in range(1, 16):
        for p in range(4, 8):
            v = Fraction(n, 2 ** p)
            if v * mx <= 255 and (best is None or v > best):
                best = v
    return best


def test_scale_factor_equals_brute_force():
    """DESIGN.md A3 reading of P:322-329: the largest 4-bit n over 2^p,
    p in [4,7], with n/2^p * mx <= 255 -- checked for every mx in [256, 4080]."""
    prev = Fraction(2)
    for mx in range(256, 4081):
        n, p = O.scale_factor(mx)
        assert 8 <= n <= 15 and 4 <= p <= 7
        v = Fraction(n, 2 ** p)
        assert v == _brute_force_factor(mx)
        assert v <= prev               # monotone in mx
        prev = v
        assert 0 < O.encode_code(n, p) < 64 and O.decode_code(O.encode_code(n, p)) == (n, p)
    for mx in (0, 1, 200, 255):
        assert O.scale_factor(mx) == (0, 0) and O.encode_code(0, 0) == 0
    assert O.scale_factor(2295) == (14, 7)                                    # P:314, Table 1
    assert FIG["scale_factor_2295"] == "14/128"


def test_table1():
    """Table 1: the 60 printed values and the gray set.  Gray
    cells are exactly the factors the scale-factor routine never emits for
    max magnitudes in (255, 2295] (A18)."""
    gold = {}
    for line in open(os.path.join(GOLD, "table1.txt")):
        if line.startswith("#") or not line.strip():
            continue
        N, P, val, gray = line.split()
        gold[(int(N), int(P))] = (val, gray == "1")
    rows = A.table1()
    assert len(rows) == 60 == len(gold)
    for N, P, printed, v, reachable in rows:
        assert printed == gold[(N, P)][0], (N, P)
        assert (not reachable) == gold[(N, P)][1], (N, P)
        assert (not reachable) == (v < Fraction(14, 128))
    assert sum(g for _, g in gold.values()) == 23


# ----------------------------------------------------------- reverse factor / rounding
def test_rha_shift_brute_force():
    for k in range(0, 9):
        for v in range(-1030, 1031):
            q = Fraction(v, 2 ** k)
            want = int(abs(q) + Fraction(1, 2)) * (1 if v >= 0 else -1)
            assert O.rha_shift(v, k) == want


def test_reverse_factor():
    """8-bit m, shift q in [4,7]; examples (8,5)->(128,5), (15,4)->(137,7),
    (14,7)->(146,4); exhaustive maximality of q over every emitted factor."""
    assert O.reverse_factor(8, 5) == (128, 5)
    assert O.reverse_factor(15, 4) == (137, 7)
    assert O.reverse_factor(14, 7) == (146, 4)
    emitted = {O.scale_factor(mx) for mx in range(256, 2049)}
    for n, p in emitted:
        m, q = O.reverse_factor(n, p)
        assert 1 <= m <= 255 and 4 <= q <= 7
        exact = Fraction(2 ** (q + p), n)
        assert abs(Fraction(m) - exact) <= Fraction(1, 2)
        if q < 7:   # a larger q would need m > 255
            assert int(Fraction(2 ** (q + 1 + p), n) + Fraction(1, 2)) > 255
        rel = abs(Fraction(m, 2 ** q) - Fraction(2 ** p, n)) / Fraction(2 ** p, n)
        assert rel <= Fraction(1, 2 * m)


def test_static_error_examples_and_sweep(capsys):
    """P:376 reports mean numerical error 1.12, proportional 0.1% over an
    unstated population (parity unpinned, A21): report ours on both
    of A21's populations.  Every weight's error stays within the bound derived
    from the three roundings (oracle/analysis.py `static_error_bound`), not a
    fitted constant."""
    n, p = O.scale_factor(2295); m, q = O.reverse_factor(n, p)
    down = O.rha_shift(2295 * n, p); up = O.rha_shift(down * m, q)
    assert (down, up) == (251, 2290)          # (SPEC S:405 prints 2291 -- an arithmetic slip)
    n, p = O.scale_factor(1020); m, q = O.reverse_factor(n, p)
    assert O.rha_shift(O.rha_shift(1020 * n, p) * m, q) == 1020
    for w in range(256, 2296):                # the derived per-weight bound holds everywhere
        n, p = O.scale_factor(w); m, q = O.reverse_factor(n, p)
        err = abs(O.rha_shift(O.rha_shift(w * n, p) * m, q) - w)
        assert err <= A.static_error_bound(w)
    uni = range(256, 2296)
    bound_mean = sum(A.static_error_bound(w) for w in uni) / len(uni)
    mean_num, mean_prop, mean_signed = A.static_error(uni)
    assert mean_num <= bound_mean
    f2 = A.f2_reachable_population()
    f2_num, f2_prop, _ = A.static_error(f2)
    f2x_num, f2x_prop, _ = A.static_error(f2, exact_inverse=True)
    # exact inverse: only the downscale's rha (|err| <= 2^(p-1)/n <= 8) remains
    assert f2x_num <= f2_num and f2x_num <= 8
    with capsys.disabled():
        print(f"\n[static error, uniform 256..2295] mean |err| {mean_num:.3f} (paper 1.12; derived bound of the "
              f"mean {float(bound_mean):.2f}), mean prop {100 * mean_prop:.3f}% (paper 0.1%), signed mean "
              f"{mean_signed:+.3f}\n[static error, F(2x2)-reachable multiset] 8-bit inverse: {f2_num:.3f}, "
              f"{100 * f2_prop:.3f}%; exact inverse: {f2x_num:.3f}, {100 * f2x_prop:.3f}% (paper 1.12, 0.1%)")


# ----------------------------------------------------------- whole layers
def _layers_sweep(rng, count):
    out = []
    while len(out) < count:
        n = int(rng.integers(1, 3)); pad = int(rng.integers(0, 2))
        h = int(rng.integers(3 - 2 * pad, 18)); w = int(rng.integers(3 - 2 * pad, 18))
        ci = int(rng.integers(1, 10)); co = int(rng.integers(1, 10))
        out.append((n, h, w, ci, co, pad))
    return out


@pytest.mark.parametrize("layout", [O.NCHW, O.NHWC])
def test_unscaled_winograd_equals_direct(layout):
    """Scaling off: the complex-Winograd pipeline equals direct correlation
    bit-exactly, incl. ragged maps and pad 0/1."""
    rng = np.random.default_rng(21 + layout)
    for (n, h, w, ci, co, pad) in _layers_sweep(rng, 60):
        x, wt = synth.random_layer(rng, n, h, w, ci, co, layout)
        res = O.wino_conv(x, wt, pad, layout, scaling=False)
        np.testing.assert_array_equal(res.out32.astype(np.int64), O.direct_conv(x, wt, pad, layout))


def test_unscaled_extremes():
    for xv, wv in [(-128, -128), (127, 127), (-128, 127), (127, -128)]:
        x = np.full((1, 9, 10, 7), xv, np.int8); w = np.full((5, 3, 3, 7), wv, np.int8)
        res = O.wino_conv(x, w, 1, O.NHWC, scaling=False)
        np.testing.assert_array_equal(res.out32.astype(np.int64), O.direct_conv(x, w, 1, O.NHWC))


def test_scaled_invariants():
    """Scaling on: |W'| <= 255 per component, codes valid and shared by
    mirrors, M'' conjugate-symmetric, Im Y == 0 (asserted inside the oracle),
    and a small error against direct convolution."""
    rng = np.random.default_rng(99)
    mirror = {(r, 3): (r, 4) for r in (0, 1, 2, 5)}
    mirror.update({(3, c): (4, c) for c in (0, 1, 2, 5)})
    mirror.update({(3, 3): (4, 4), (3, 4): (4, 3)})
    for (n, h, w, ci, co) in [(1, 12, 9, 6, 5), (2, 8, 8, 16, 3)]:
        x, wt = synth.random_layer(rng, n, h, w, ci, co, O.NHWC)
        W, Wp, codes = O.filter_transform(wt, O.NHWC, scaling=True)
        assert np.abs(Wp).max() <= 255
        assert (codes > 0).any()
        for c in np.unique(codes):
            if c:
                nn, pp = O.decode_code(int(c)); assert 8 <= nn <= 15 and 4 <= pp <= 7
        for (r, c), (r2, c2) in mirror.items():
            assert np.array_equal(codes[:, r * 6 + c], codes[:, r2 * 6 + c2])
        res = O.wino_conv(x, wt, 1, O.NHWC, scaling=True, want_M=True)
        for (r, c), (r2, c2) in mirror.items():
            a, b = res.Mpp[:, :, r * 6 + c], res.Mpp[:, :, r2 * 6 + c2]
            np.testing.assert_array_equal(a[..., 0], b[..., 0]); np.testing.assert_array_equal(a[..., 1], -b[..., 1])
        ref = O.direct_conv(x, wt, 1, O.NHWC)
        err = np.abs(res.out32 - ref)
        assert err.mean() <= 0.01 * np.abs(ref).mean()


def _pow2_filters(rng, co, ci):
    """Filters whose every scaled position gets a power-of-two factor (1/2 or
    1/8) and whose transformed weights are divisible by 8: scaling is then
    lossless, so scaled == unscaled == direct exactly (pins)."""
    w = np.zeros((co, 3, 3, ci), np.int8)
    for o in range(co):
        for i in range(ci):
            a = rng.choice([0, 1, -1, 15, -15])
            k, l = rng.integers(0, 3, 2)
            w[o, k, l, i] = 8 * a
    return w


def test_scaled_power_of_two_case_is_exact():
    rng = np.random.default_rng(7)
    seen_scaled = 0
    for trial in range(8):
        ci, co = int(rng.integers(1, 6)), int(rng.integers(1, 5))
        w = _pow2_filters(rng, co, ci)
        x = rng.integers(-128, 128, (2, 11, 10, ci)).astype(np.int8)
        _, _, codes = O.filter_transform(w, O.NHWC, scaling=True)
        seen_scaled += int((codes > 0).sum())
        for c in np.unique(codes):
            if c:
                assert O.decode_code(int(c))[0] == 8
        res = O.wino_conv(x, w, 1, O.NHWC, scaling=True)
        np.testing.assert_array_equal(res.out32.astype(np.int64), O.direct_conv(x, w, 1, O.NHWC))
    assert seen_scaled > 0


def test_requant_rounding_and_clamp():
    """DESIGN.md A14: y8 = clamp(rha(v * M0 / 2^S), -128, 127)."""
    v = np.array([24, -24, 23, -23, 8, -8, 7, 40000, -40000, 0], np.int64)
    np.testing.assert_array_equal(O.requant(v, 1, 4), [2, -2, 1, -1, 1, -1, 0, 127, -128, 0])
    np.testing.assert_array_equal(O.requant(np.array([3, -3]), 3, 1), [5, -5])   # 4.5 -> 5


def test_requant_inside_wino_matches_standalone():
    rng = np.random.default_rng(4)
    x, wt = synth.random_layer(rng, 1, 10, 10, 8, 4, O.NHWC)
    res = O.wino_conv(x, wt, 1, O.NHWC, scaling=True, M0=3, S=9)
    np.testing.assert_array_equal(res.y8, O.requant(res.out32.astype(np.int64), 3, 9))


def test_maxpool_reference():
    x = np.arange(-64, 64, dtype=np.int8).reshape(1, 4, 8, 4)
    y = O.maxpool2(x, O.NHWC)
    want = x.reshape(1, 2, 2, 4, 2, 4).max(axis=(2, 4))
    np.testing.assert_array_equal(y, want)


def test_config_inputs_are_deterministic():
    a = synth.config_inputs("C1"); b = synth.config_inputs("C1")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    x, w = synth.config_inputs("C2", n=2)
    assert x.shape == (2, 56, 56, 64) and w.shape == (64, 3, 3, 64) and np.abs(w.astype(int)).max() <= 127


def test_c1_scaling_off_then_on():
    """Config C1 (BASELINE.json configs[0]) through the oracle both ways."""
    for layout in (O.NCHW, O.NHWC):
        x, w = synth.config_inputs("C1", layout)
        direct = O.direct_conv(x, w, 1, layout)
        off = O.wino_conv(x, w, 1, layout, scaling=False)
        np.testing.assert_array_equal(off.out32.astype(np.int64), direct)
        on = O.wino_conv(x, w, 1, layout, scaling=True)
        assert np.abs(on.out32 - direct).max() < 0.02 * np.abs(direct).max()
