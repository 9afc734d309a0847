"""The paper's arithmetic-complexity and bit-width claims, recomputed from the
transform matrices (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

Nothing here is hard-coded from the paper's results: counts come from the
structure of the matrices the oracle uses, ranges from vertex enumeration,
factors from the oracle's scale-factor routine.  The tests compare these
against the values the paper prints (tests/golden/).
"""
from __future__ import annotations

import itertools
import math
from fractions import Fraction

import numpy as np

from . import oracle as O

# Rational F(4x4,3x3) filter matrix G, typed from P:126-132 (Lavin & Gray).
G_RATIONAL_F4 = [
    [Fraction(1, 4), Fraction(0), Fraction(0)],
    [Fraction(-1, 6), Fraction(-1, 6), Fraction(-1, 6)],
    [Fraction(-1, 6), Fraction(1, 6), Fraction(-1, 6)],
    [Fraction(1, 24), Fraction(1, 12), Fraction(1, 6)],
    [Fraction(1, 24), Fraction(-1, 12), Fraction(1, 6)],
    [Fraction(0), Fraction(0), Fraction(1)],
]
# Integer F(2x2,3x3) filter matrix G' = 2G, typed from P:261-268.
G_PRIME_F2 = np.array([[2, 0, 0], [1, 1, 1], [1, -1, 1], [0, 0, 2]], np.int64)


# ------------------------------------------------------------ structure
def position_coefficients(BT: np.ndarray):
    """Coefficient matrix of each D[r][c] = sum_kl BT[r][k] BT[c][l] d[k][l]."""
    t = BT.shape[0]
    return {(r, c): np.outer(BT[r], BT[c]) for r in range(t) for c in range(t)}


def conjugate_layout(BT: np.ndarray):
    """Partition the t x t positions into always-real ones and conjugate pairs,
    read off the coefficient matrices.  Returns (real, pairs)."""
    coef = position_coefficients(BT)
    real = sorted(p for p, C in coef.items() if np.all(np.imag(C) == 0))
    rest = [p for p in coef if p not in real]
    pairs, used = [], set()
    for p in sorted(rest):
        if p in used:
            continue
        mates = [q for q in rest if q != p and q not in used and np.array_equal(coef[q], np.conj(coef[p]))]
        if len(mates) != 1:
            raise AssertionError(f"position {p} has {len(mates)} conjugate mates")
        pairs.append((p, mates[0]))
        used.update({p, mates[0]})
    return real, pairs


def general_multiplications(BT: np.ndarray) -> int:
    """General multiplications per tile per (cin, cout): one per real position,
    three (Karatsuba) per conjugate pair."""
    real, pairs = conjugate_layout(BT)
    return len(real) * 1 + len(pairs) * 3


def filter_scale_of(G) -> int:
    """Smallest integer s with s*G integral (the widening source)."""
    s = 1
    for row in G:
        for v in row:
            if isinstance(v, complex):
                parts = [Fraction(v.real).limit_denominator(1000), Fraction(v.imag).limit_denominator(1000)]
            else:
                parts = [Fraction(v)]
            for f in parts:
                s = s * f.denominator // math.gcd(s, f.denominator)
    return s


def widening_bits(G) -> int:
    """ceil(log2(scale^2))."""
    s = filter_scale_of(G)
    return math.ceil(math.log2(s * s))


def signed_bits(mag: int) -> int:
    """1 + ceil(log2(mag + 1)) (A20)."""
    return 1 + math.ceil(math.log2(mag + 1))


def worst_case_magnitudes_generic(G: np.ndarray, bound: int) -> np.ndarray:
    """max over g in [-bound, bound]^{3x3} of |(G g G^T)[i][j]| by vertex
    enumeration (a linear function on a box peaks at a vertex)."""
    t = G.shape[0]
    best = np.zeros((t, t), np.int64)
    for signs in itertools.product((-1, 1), repeat=9):
        g = np.array(signs, np.int64).reshape(3, 3) * bound
        W = G @ g @ G.T
        best = np.maximum(best, np.abs(W))
    return best


def worst_case_magnitudes_complex(bound_lo: int, bound_hi: int) -> np.ndarray:
    """Per-position max of max(|Re W|, |Im W|) for the complex F(4x4) filter
    transform with g in [bound_lo, bound_hi]^{3x3}, by vertex enumeration
    through the oracle's own filter_tile."""
    best = np.zeros((6, 6), np.int64)
    for choice in itertools.product((bound_lo, bound_hi), repeat=9):
        W = O.filter_tile(np.array(choice, np.int64).reshape(3, 3))
        best = np.maximum(best, np.abs(W).max(axis=2))
    return best


# ------------------------------------------------------------ ratios
def reduction_ratio(m: int, r: int, muls: int) -> Fraction:
    return Fraction(m * m * r * r, muls)


def efficiency_gain(red_a: float, bits_a: int, red_b: float, bits_b: int) -> float:
    """(red_a / bits_a) / (red_b / bits_b) - 1."""
    return (red_a / bits_a) / (red_b / bits_b) - 1.0


# ------------------------------------------------------------ Table 1
def half_up_5dp(v: Fraction) -> str:
    """Decimal rounding half-up to 5 places (how Table 1 prints, A18)."""
    q = (v * 100000 * 2 + 1) // 2   # floor(v*1e5 + 0.5) for v >= 0
    return f"{q // 100000}.{q % 100000:05d}"


def table1():
    """The 60 (N, P) factors n/2^(P+4) with the set the oracle's scale-factor
    routine can ever emit for max magnitudes in (255, 2295]."""
    reachable = set()
    for mx in range(256, 2296):
        n, p = O.scale_factor(mx)
        reachable.add(Fraction(n, 2 ** p))
    rows = []
    for N in range(1, 16):
        for P in range(4):
            v = Fraction(N, 2 ** (P + 4))
            rows.append((N, P, half_up_5dp(v), v, v in reachable))
    return rows


# ------------------------------------------------------------ static error
def static_error(population, exact_inverse=False):
    """Down-then-up error of each weight: f = scale_factor(w),
    down = rha(w n / 2^p), up = rha(down m / 2^q) with the 8-bit inverse of
    P:366 (A8), or up = down 2^p / n exactly (`exact_inverse`).  Returns
    (mean |up - w|, mean |up - w| / |w|, mean (up - w)) over the scaled
    weights of the population."""
    num, prop, signed = [], [], []
    for w in population:
        n, p = O.scale_factor(int(w))
        if n == 0:
            continue
        down = O.rha_shift(int(w) * n, p)
        if exact_inverse:
            up = Fraction(down * 2 ** p, n)
        else:
            m, q = O.reverse_factor(n, p)
            up = O.rha_shift(down * m, q)
        num.append(abs(up - w)); prop.append(abs(up - w) / abs(w)); signed.append(up - w)
    return float(np.mean(num)), float(np.mean(prop)), float(np.mean(signed))


def static_error_bound(w):
    """Derived bound on |up - w| for one weight w > 255 (8-bit inverse):
    |down - w n/2^p| <= 1/2 (rha), |m - 2^(q+p)/n| <= 1/2 (rha) and the final
    rha adds <= 1/2, so
      |up - w| <= |down| |m/2^q - 2^p/n| + (2^p/n)|down - w n/2^p| + 1/2
               <= 255 / 2^(q+1) + 2^(p-1)/n + 1/2      (|down| <= 255)."""
    n, p = O.scale_factor(int(w))
    if n == 0:
        return Fraction(0)
    _, q = O.reverse_factor(n, p)
    return Fraction(255, 2 ** (q + 1)) + Fraction(2 ** (p - 1), n) + Fraction(1, 2)


def f2_reachable_population():
    """A21's second population: the magnitudes an F(2x2) Winograd-domain
    filter value can take from int8 weights (G' = 2G): the 4
    corner positions are 4 g (multiples of 4 up to 4*255 = 1020 for int9),
    the 8 edge positions 2 (g0 +- g1 + g2) (even values up to 1530), the 4
    centre positions any value up to 2295 (P:330's worst case); each kept
    above 255 (scaled), as a multiset."""
    corners = [v for v in range(256, 1021) if v % 4 == 0]
    edges = [v for v in range(256, 1531) if v % 2 == 0]
    centre = list(range(256, 2296))
    return corners * 4 + edges * 8 + centre * 4
