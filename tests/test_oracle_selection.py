"""Pins of the oracle's per-OFM filter-scale SELECTION.

P:312: "a downscale factor ... for each X-Y location of the transformed
filter"; "transform all the weights for the current OFM ...
find the maximum magnitude at each X-Y location across all channels".  The
oracle (`oracle_filter_transform16`) reads this as DESIGN.md A3 (the factor
grid n/2^p, n in [8, 15], p in [4, 7], largest with n/2^p <= 255/mx), A5
(magnitude of a complex W = max(|Re|, |Im|)), A15 (every position, mirrors
share) and A16 (mx = 0 -> unscaled).

What a plausible mistake would change, and the pin that catches it:
  * a max taken across ALL output channels (not per OFM)  -> per-OFM
    independence (codes of a bank == codes of each OFM alone) and the
    small-OFM-next-to-a-large-OFM case;
  * |Re| + |Im| (or the modulus) as the magnitude          -> the
    |Re| = |Im| = 200 position must stay unscaled (255/mx >= 1);
  * a factor that is valid but not the largest on the grid -> maximality:
    the next larger grid factor must push some channel above 255;
  * a max over a subset of channels                        -> every channel's
    W n / 2^p within 255 (exact rational product) at the chosen factor.
W itself (the unscaled transform the selection reads) is pinned elsewhere by
the closed-form identity A^T[(G g G^T) . (B^T d B)]A = 16 corr
(tests/test_oracle_pins.py), so these tests read W from the oracle.
"""
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import oracle as O

# the factor grid of P:322-330 read as A3: n/2^p, n in [8, 15], p in [4, 7]
GRID = sorted({Fraction(n, 2 ** p) for n in range(8, 16) for p in range(4, 8)})


def _factor(code):
    n, p = O.decode_code(int(code))
    return Fraction(n, 2 ** p)


def _bank(rng, co, ci, sigma):
    return np.clip(np.round(rng.normal(0, sigma, (co, 3, 3, ci))), -127, 127).astype(np.int8)


@pytest.mark.parametrize("seed,co,ci,sigma", [(1, 6, 5, 32.0), (2, 4, 17, 24.0), (3, 3, 2, 90.0), (4, 5, 1, 127.0)])
def test_codes_are_per_ofm(seed, co, ci, sigma):
    """P:319 'for the current OFM': the codes of output channel o depend on
    w[o] only -- the bank's codes equal each OFM transformed on its own."""
    w = _bank(np.random.default_rng(seed), co, ci, sigma)
    _, _, codes = O.filter_transform(w, O.NHWC, scaling=True)
    for o in range(co):
        _, _, alone = O.filter_transform(w[o:o + 1], O.NHWC, scaling=True)
        np.testing.assert_array_equal(codes[o], alone[0])


def test_small_ofm_next_to_large_ofm_stays_unscaled():
    """One OFM at the int8 extremes (every position scaled) next to one with
    |w| <= 3 (every |W| <= 16*3*... well below 255): a cross-OFM max would
    scale the small one; the paper's per-OFM max leaves it exact."""
    rng = np.random.default_rng(11)
    ci = 8
    big = np.where(rng.integers(0, 2, (1, 3, 3, ci)) == 0, -128, 127).astype(np.int8)
    small = rng.integers(-3, 4, (1, 3, 3, ci)).astype(np.int8)
    W, Wp, codes = O.filter_transform(np.concatenate([big, small]), O.NHWC, scaling=True)
    assert np.abs(W[1]).max() <= 255
    assert (codes[0] > 0).sum() >= 30          # the large OFM is scaled almost everywhere
    assert (codes[1] == 0).all()               # the small one not at all
    np.testing.assert_array_equal(Wp[1], W[1])


def test_magnitude_is_max_of_components():
    """A5: a complex position with |Re W| = |Im W| = 200 has magnitude 200
    <= 255 and stays unscaled (|Re| + |Im| = 400 or the modulus 283 would
    scale it).  g = [[50, 50, 0], 0, 0] gives W(0,3) = 4(g00 - g02) +
    4 g01 i = 200 + 200i (row 0 of G_int is (4, 0, 0), row 3 is (1, i, -1),
    P:155-160)."""
    g = np.zeros((1, 3, 3, 1), np.int8)
    g[0, 0, 0, 0] = 50
    g[0, 0, 1, 0] = 50
    W, Wp, codes = O.filter_transform(g, O.NHWC, scaling=True)
    pos03, pos04 = 0 * 6 + 3, 0 * 6 + 4
    assert tuple(W[0, 0, pos03]) == (200, 200) and tuple(W[0, 0, pos04]) == (200, -200)
    assert codes[0, pos03] == 0 and codes[0, pos04] == 0
    np.testing.assert_array_equal(Wp[0, 0, pos03], W[0, 0, pos03])
    # and the same magnitude pushed past 255 on one component only is scaled
    g[0, 0, 1, 0] = 64                        # Im = 256, Re = 200
    _, _, codes = O.filter_transform(g, O.NHWC, scaling=True)
    # mx = 256: the largest grid factor <= 255/256 is the grid's top, 15/16
    assert _factor(codes[0, pos03]) == Fraction(15, 16)


@pytest.mark.parametrize("seed,co,ci,sigma", [(5, 6, 9, 32.0), (6, 3, 33, 24.0), (7, 4, 4, 127.0), (8, 2, 64, 60.0)])
def test_factor_is_the_largest_valid_grid_factor(seed, co, ci, sigma):
    """P:312 / P:321-329 (A3): at every scaled (OFM, position), the chosen
    n/2^p keeps every channel's |Re W| n/2^p and |Im W| n/2^p within 255
    (exact rational products), and the NEXT LARGER factor on the grid does
    not -- some channel's component would exceed 255.  Unscaled positions
    have every component within 255 already."""
    w = _bank(np.random.default_rng(seed), co, ci, sigma)
    W, Wp, codes = O.filter_transform(w, O.NHWC, scaling=True)
    comp = np.abs(W)                                         # [co][ci][36][2]
    n_scaled = 0
    for o in range(co):
        for pos in range(36):
            c = int(codes[o, pos])
            peak = int(comp[o, :, pos, :].max())            # over channels and both components
            if c == 0:
                assert peak <= 255
                continue
            n_scaled += 1
            f = _factor(c)
            assert f in GRID
            assert f * peak <= 255
            larger = [h for h in GRID if h > f]
            if larger:                                       # f = 15/16 is the grid's top
                assert larger[0] * peak > 255
            # W' = rha(W n / 2^p) on both components (A7)
            n, p = O.decode_code(c)
            for ch in range(ci):
                for k in range(2):
                    v = int(W[o, ch, pos, k])
                    want = (abs(v) * n + (1 << (p - 1))) >> p
                    assert Wp[o, ch, pos, k] == (want if v >= 0 else -want)
    assert n_scaled > 0


def test_all_zero_position_is_unscaled():
    """A16: an OFM of zeros (mx = 0) has code 0 everywhere."""
    w = np.zeros((2, 3, 3, 4), np.int8)
    w[1] = 100
    _, _, codes = O.filter_transform(w, O.NHWC, scaling=True)
    assert (codes[0] == 0).all() and (codes[1] > 0).any()


def test_config_banks_selection_is_per_ofm_and_maximal():
    """The same two properties on the C2 bank (BASELINE configs[1]): 64 OFMs,
    64 channels, w ~ round(N(0, 32))."""
    _, w = synth.config_inputs("C2", n=1)
    W, _, codes = O.filter_transform(w, O.NHWC, scaling=True)
    peak = np.abs(W).max(axis=(1, 3))                        # [co][36]
    for o in range(0, 64, 7):
        _, _, alone = O.filter_transform(w[o:o + 1], O.NHWC, scaling=True)
        np.testing.assert_array_equal(codes[o], alone[0])
        for pos in range(36):
            c = int(codes[o, pos])
            if c == 0:
                assert peak[o, pos] <= 255
                continue
            f = _factor(c)
            assert f * int(peak[o, pos]) <= 255
            larger = [h for h in GRID if h > f]
            assert not larger or larger[0] * int(peak[o, pos]) > 255


def _error_bound_case(seed, n, h, w_, ci, co, sigma, xdist="uniform"):
    rng = np.random.default_rng(seed)
    x = rng.integers(-128, 128, (n, h, w_, ci)).astype(np.int8)
    if xdist == "relu":
        x = np.maximum(x, 0).astype(np.int8)
    w = _bank(rng, co, ci, sigma)
    return x, w


@pytest.mark.parametrize("case", [(31, 1, 9, 11, 7, 5, 32.0), (32, 2, 8, 8, 16, 4, 24.0),
                                  (33, 1, 6, 13, 3, 6, 127.0), (34, 1, 12, 12, 40, 3, 24.0)])
def test_scaled_pipeline_within_the_derived_error_bound(case):
    """The whole scaled pipeline (O1-O10) against direct convolution, within
    the error bound derived from its three roundings -- the check that the C
    pipeline's indexing, Karatsuba/complex products, reverse scaling and
    output transform are those of the paper (a transposed operand, a wrong
    position or a dropped term would leave it far outside).  Per position,
    with f = n/2^p, r = m/2^q:
      W' = f W + e, |e_re|, |e_im| <= 1/2                       (A7)
      M'' = rha(r M') = r M' + eps, |eps| <= 1/2 per component   (A9)
      M'' - M = (r f - 1) M + r sum_c e D + eps, so per component
      |d| <= |r f - 1| |M_comp| + r sum_c (|D_re| + |D_im|) / 2 + 1/2,
    M = sum_c W D the exact product of the pinned transforms.  Y = A^T M A
    adds |Re dM| + |Im dM| per nonzero A^T coefficient pair (|a| <= 1), and
    out32 = rha(Y / 16) adds 1/2."""
    seed, n, h, w_, ci, co, sigma = case
    x, w = _error_bound_case(seed, n, h, w_, ci, co, sigma)
    W, _, codes = O.filter_transform(w, O.NHWC, scaling=True)
    D = O.input_transform(x, 1, O.NHWC)                          # [T][ci][36][2]
    res = O.wino_conv(x, w, 1, O.NHWC, scaling=True)
    direct = O.direct_conv(x, w, 1, O.NHWC)
    _, _, AT = O.matrices()
    Wc = W[..., 0] + 1j * W[..., 1]                              # [co][ci][36]
    Dc = D[..., 0] + 1j * D[..., 1]                              # [T][ci][36]
    M = np.einsum("tcp,ocp->top", Dc, Wc)                        # exact product (|.| < 2^53)
    sumD = np.abs(D).sum(axis=3).sum(axis=1)                     # [T][36]: sum_c |D_re| + |D_im|
    rf1 = np.zeros((co, 36)); r = np.ones((co, 36))
    for o in range(co):
        for p_ in range(36):
            if codes[o, p_]:
                nn, pp = O.decode_code(int(codes[o, p_]))
                m, q = O.reverse_factor(nn, pp)
                r[o, p_] = m / 2 ** q
                rf1[o, p_] = abs(m / 2 ** q * nn / 2 ** pp - 1)
    scaled = codes > 0                                           # [co][36]
    dre = rf1[None] * np.abs(M.real) + scaled[None] * (r[None] * sumD[:, None, :] / 2 + 0.5)
    dim = rf1[None] * np.abs(M.imag) + scaled[None] * (r[None] * sumD[:, None, :] / 2 + 0.5)
    dM = (dre + dim).reshape(-1, co, 6, 6)                       # [T][co][6][6]
    absA = (np.abs(AT) > 0).astype(float)                        # |a| in {0, 1}
    dY = np.einsum("ir,tkrc,jc->tkij", absA, dM, absA)           # [T][co][4][4]
    Ho, Wo = h, w_
    th, tw = (Ho + 3) // 4, (Wo + 3) // 4
    bound = dY.reshape(n, th, tw, co, 4, 4).transpose(0, 1, 4, 2, 5, 3).reshape(n, 4 * th, 4 * tw, co)
    bound = bound[:, :Ho, :Wo] / 16 + 0.5 + 1e-6
    err = np.abs(res.out32.astype(np.int64) - direct)
    assert (err <= bound).all(), float((err - bound).max())
    assert (codes > 0).any() and err.max() > 0                   # the case really is scaled and lossy
