"""Pins of the oracle's mixed-precision rounding points.

tests/golden/mxp_rounding_points.json holds hand-derived Nt = 2..3, nb = 1
factorizations that separate the readings of SURVEY 8(c):
  * O3 / G14   -- the accumulator starts from the quantized input deq(q_p(A));
  * O4.2.5-6   -- quantize once per task, AFTER the TRSM;
  * O4.2.2-3   -- operands down-cast to the output tile's precision c with their
                  own power-of-two scale (G11, G12).
The oracle must reproduce each expected factor bit for bit.  Each case also
records the value one plausible misreading gives; a small exact-rational
re-derivation below (Fractions, written from the JSON's stated rule, not from
the oracle) confirms both the hand arithmetic and that the misreading lands
elsewhere -- so flipping any of the three rounding points in oracle.c turns
this file red.
"""
import math
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle
from mxp_pins import cases, embed, ij, num, scalar_case

BITS = {0: 53, 1: 24, 2: 11, 3: 4}  # significant bits per precision code


def rnd(x: Fr, p: int) -> Fr:
    """Round to nearest-even at BITS[p] significant bits (a scalar tile: the
    pow2 scale normalizes its one entry, so no subnormal/saturation case)."""
    if x == 0:
        return Fr(0)
    a, e = abs(x), 0
    while a >= 2:
        a, e = a / 2, e + 1
    while a < 1:
        a, e = a * 2, e - 1
    q = a * 2 ** (BITS[p] - 1)
    fl = q.numerator // q.denominator
    d = q - fl
    if d > Fr(1, 2) or (d == Fr(1, 2) and fl % 2):
        fl += 1
    return (1 if x > 0 else -1) * Fr(fl, 2 ** (BITS[p] - 1)) * Fr(2) ** e


def sqrt_exact(x: Fr):
    r = Fr(math.isqrt(x.numerator), math.isqrt(x.denominator))
    return r if r * r == x else None


def derive(c, skip_o3=False, quant_before=False, own_prec=False):
    """The JSON's stated rule (nb = 1) in exact rationals; a flag flips one reading.
    Returns {(i, j): L_ij} for the entries that stay exact (None otherwise)."""
    n = c["n"]
    A = {ij(k): Fr(num(v)) for k, v in c["A_lower"].items()}
    P = {ij(k): p for k, p in c["map"].items()}
    Ah = {k: (v if k[0] == k[1] or skip_o3 else rnd(v, P[k])) for k, v in A.items()}
    L = {}
    for k in range(n):
        s = Ah[(k, k)] - sum((L[(k, q)] ** 2 for q in range(k)), Fr(0))
        L[(k, k)] = sqrt_exact(s)
        if L[(k, k)] is None:
            return L
        for m in range(k + 1, n):
            cp = P[(m, k)]
            cast = (lambda t: t) if own_prec else (lambda t: rnd(t, cp))
            C = Ah[(m, k)] - sum((cast(L[(m, q)]) * cast(L[(k, q)]) for q in range(k)), Fr(0))
            L[(m, k)] = rnd(C, cp) / L[(k, k)] if quant_before else rnd(C / L[(k, k)], cp)
    return L


MISREAD = {"skip O3": dict(skip_o3=True), "quantize before TRSM": dict(quant_before=True),
           "operands used at their own": dict(own_prec=True)}


@pytest.mark.parametrize("case", cases(), ids=lambda c: c["name"])
def test_oracle_matches_hand_derivation(case):
    A, Lexp, pmap = scalar_case(case)
    L, info = oracle.factor(A, 1, pmap)
    assert info == 0
    assert np.array_equal(L, Lexp), (case["name"], L, Lexp)
    # the misreading's value differs from what the oracle computes
    i, j = ij(case["misreading"]["entry"])
    assert L[i, j] != num(case["misreading"]["value"])


@pytest.mark.parametrize("case", cases(), ids=lambda c: c["name"])
def test_hand_derivation_and_misreading_are_consistent(case):
    """Re-derive the JSON's arithmetic exactly: the stated reading gives L_lower,
    the named misreading gives the recorded (different) value."""
    L = derive(case)
    for k, v in case["L_lower"].items():
        assert L[ij(k)] == Fr(num(v)), (case["name"], k)
    mis = case["misreading"]
    flags = next(f for key, f in MISREAD.items() if mis["what"].startswith(key))
    Lm = derive(case, **flags)
    e = ij(mis["entry"])
    assert float(Lm[e]) == num(mis["value"]), (case["name"], float(Lm[e]))
    assert Lm[e] != L[e]
    # the other two readings agree with the stated one on this case's key entry
    # (each case isolates exactly one rounding point)
    for key, f in MISREAD.items():
        if f is flags:
            continue
        Lo = derive(case, **f)
        assert Lo.get(e) == L[e], (case["name"], key)


@pytest.mark.parametrize("case", cases(), ids=lambda c: c["name"])
@pytest.mark.parametrize("nb", [2, 4])
def test_oracle_identity_embedding(case, nb):
    """Tile (i,j) = A_ij I_nb: tiles stay diagonal, each tile's amax is |A_ij|,
    so the oracle's factor is L_ij I_nb bit for bit (the form the GPU test uses)."""
    A, Lexp, pmap = scalar_case(case)
    L, info = oracle.factor(embed(A, nb), nb, pmap)
    assert info == 0
    assert np.array_equal(L, embed(Lexp, nb))


def test_upcast_is_identity_even_when_the_stored_amax_crossed_a_binade():
    """O4.2.3 / P:42: an operand stored no more precisely than the compute
    precision c is used as stored (an exact up-cast), including c equal to
    its own precision.  Hand derivation (E4M3, nb = 2 tile [0.99, 2^-17]):
      q_FP8: amax = 0.99, floor(log2 0.99) = -1, s = 2^(7+1) = 2^8;
        0.99 * 256 = 253.44 in [2^7, 2^8), spacing 16 -> 15.84 -> 16 -> code 256 -> 1.0
        2^-17 * 256 = 2^-9 = the smallest E4M3 subnormal -> exact -> 2^-17
      stored T = [1.0, 2^-17].  cast_FP8(T) = T and cast_FP16(T) = T.
    The misreading 're-quantize with the stored amax' gives s' = 2^(7-0) = 2^7,
    2^-17 * 2^7 = 2^-10 = half the subnormal spacing -> tie -> even -> 0."""
    T, s = oracle.quantize_tile(3, np.array([0.99, 2.0 ** -17]))
    assert s == 2.0 ** 8 and T[0] == 1.0 and T[1] == 2.0 ** -17
    assert np.array_equal(oracle.cast_tile(3, 3, T), T)
    assert np.array_equal(oracle.cast_tile(2, 3, T), T)
    assert np.array_equal(oracle.cast_tile(0, 3, T), T)
    requant, _ = oracle.quantize_tile(3, T)      # the misreading
    assert requant[1] == 0.0 and requant[1] != T[1]
    # a genuine down-cast (stored FP32, c = FP8) rounds with the tile's own scale:
    # amax 1.03125 -> s = 2^7: 132 -> 128 -> 1.0;  0.1 * 128 = 12.8 in [2^3, 2^4), spacing 1 -> 13 -> 0.1015625
    D = oracle.cast_tile(3, 1, np.array([1.03125, 0.1]))
    assert D[0] == 1.0 and D[1] == 13 / 128
