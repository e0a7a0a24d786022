"""Pins for the oracle's quantizers (O2): exhaustive code points,
library cross-checks (numpy float16/float32, ml_dtypes E4M3), SPEC examples.
None of these re-use the oracle's own rounding code."""
import math

import ml_dtypes
import numpy as np
import pytest

import oracle
from oracle import FP8, FP16, FP32, FP64

PNAME = {"FP64": FP64, "FP32": FP32, "FP16": FP16, "FP8": FP8}


def test_spec_cast_examples(golden):
    for ex in golden["cast_scalar"]:
        assert oracle.round_scalar(PNAME[ex["prec"]], ex["x"]) == ex["expect"], ex["cite"]


def test_fp16_all_code_points_round_trip():
    codes = np.arange(1 << 16, dtype=np.uint16).view(np.float16).astype(np.float64)
    finite = codes[np.isfinite(codes)]
    out = oracle.round_array(FP16, finite)
    assert np.array_equal(out, finite)


def test_e4m3_all_code_points_round_trip():
    vals = np.arange(256, dtype=np.uint8).view(ml_dtypes.float8_e4m3fn).astype(np.float64)
    finite = vals[np.isfinite(vals)]
    assert len(finite) == 254  # 0x7f / 0xff are NaN in E4M3fn
    out = oracle.round_array(FP8, finite)
    assert np.array_equal(out, finite)
    assert finite.max() == 448.0 and np.min(np.abs(finite[finite != 0])) == 2.0 ** -9


def _samples(rng, n, lo, hi):
    mant = rng.uniform(1.0, 2.0, n)
    ex = rng.integers(lo, hi, n)
    sgn = rng.choice([-1.0, 1.0], n)
    return sgn * np.ldexp(mant, ex)


def test_fp16_matches_numpy():
    rng = np.random.default_rng(0)
    x = _samples(rng, 200_000, -28, 17)  # covers subnormals, normals and overflow
    ref = x.astype(np.float16).astype(np.float64)
    out = oracle.round_array(FP16, x)
    assert np.array_equal(out, ref)


def test_fp32_matches_numpy():
    rng = np.random.default_rng(1)
    x = _samples(rng, 200_000, -152, 129)
    with np.errstate(over="ignore"):
        ref = x.astype(np.float32).astype(np.float64)
    out = oracle.round_array(FP32, x)
    assert np.array_equal(out, ref)


def test_e4m3_matches_ml_dtypes_saturating():
    rng = np.random.default_rng(2)
    # float32-representable inputs so ml_dtypes' conversion rounds only once
    x = _samples(rng, 100_000, -12, 10).astype(np.float32).astype(np.float64)
    clamped = np.clip(x, -448.0, 448.0)  # ml_dtypes maps overflow to NaN; cvt.satfinite clamps
    ref = clamped.astype(np.float32).astype(ml_dtypes.float8_e4m3fn).astype(np.float64)
    out = oracle.round_array(FP8, x)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("prec,u", [(FP32, 2.0 ** -24), (FP16, 2.0 ** -11), (FP8, 2.0 ** -4)])
def test_unit_roundoff_bound_and_idempotence(prec, u):
    """|x - q(x)| <= u_p |x| for normal, non-saturated x; q(q(x)) = q(x)."""
    assert oracle.unit_roundoff(prec) == u
    rng = np.random.default_rng(3 + prec)
    lo, hi = {FP32: (-120, 120), FP16: (-13, 15), FP8: (-5, 8)}[prec]
    x = _samples(rng, 100_000, lo, hi)
    q = oracle.round_array(prec, x)
    if prec == FP8:
        keep = np.abs(x) <= 448.0
        x, q = x[keep], q[keep]
    assert np.all(np.abs(x - q) <= u * np.abs(x))
    assert np.array_equal(oracle.round_array(prec, q), q)


def test_ties_to_even():
    # FP16 around 1: spacing 2^-10; midpoint 1 + 2^-11 -> 1 (even), 1 + 3*2^-11 -> 1 + 2^-9
    assert oracle.round_scalar(FP16, 1 + 2.0 ** -11) == 1.0
    assert oracle.round_scalar(FP16, 1 + 3 * 2.0 ** -11) == 1 + 2.0 ** -9
    # E4M3 around 1: spacing 2^-3; 1 + 2^-4 -> 1, 1 + 3*2^-4 -> 1.25
    assert oracle.round_scalar(FP8, 1 + 2.0 ** -4) == 1.0
    assert oracle.round_scalar(FP8, 1 + 3 * 2.0 ** -4) == 1.25
    # FP16 overflow: 65520 is the midpoint between 65504 and 2^16 -> inf
    assert math.isinf(oracle.round_scalar(FP16, 65520.0))
    assert oracle.round_scalar(FP16, 65519.0) == 65504.0
    # E4M3 saturates, including far above the range
    assert oracle.round_scalar(FP8, -1e30) == -448.0
    assert oracle.round_scalar(FP64, 0.1) == 0.1


@pytest.mark.parametrize("prec,Ep", [(FP16, 14), (FP8, 7)])
def test_quantize_tile_pow2_scale(prec, Ep):
    """G11: s = 2^(E_p - floor(log2 amax)); amax*s in [2^Ep, 2^(Ep+1)); codes
    representable; deq = codes / s exactly."""
    rng = np.random.default_rng(10 + prec)
    for scale_exp in (-40, -12, 0, 9):
        T = rng.standard_normal(256) * 2.0 ** scale_exp
        deq, s = oracle.quantize_tile(prec, T)
        assert s == 2.0 ** round(math.log2(s))
        amax = np.max(np.abs(T))
        assert 2.0 ** Ep <= amax * s < 2.0 ** (Ep + 1)
        codes = deq * s
        ref = (codes.astype(np.float16).astype(np.float64) if prec == FP16 else
               codes.astype(np.float32).astype(ml_dtypes.float8_e4m3fn).astype(np.float64))
        assert np.array_equal(codes, ref)
        # codes are the library rounding of T*s
        lib = ((T * s).astype(np.float16).astype(np.float64) if prec == FP16 else
               (T * s).astype(np.float32).astype(ml_dtypes.float8_e4m3fn).astype(np.float64))
        if prec == FP16:
            assert np.array_equal(codes, lib)
        # error bound relative to amax: |T - deq| <= u * amax (normal range)
        u = oracle.unit_roundoff(prec)
        assert np.max(np.abs(T - deq)) <= u * amax


def test_quantize_tile_zero_and_clamp():
    deq, s = oracle.quantize_tile(FP8, np.zeros(16))
    assert s == 1.0 and np.all(deq == 0)
    deq, s = oracle.quantize_tile(FP8, np.full(4, 2.0 ** -200))
    assert s == 2.0 ** 127  # clamp to the UE8M0 range
    deq, s = oracle.quantize_tile(FP32, np.array([0.1, 1e-40]))
    assert s == 1.0 and deq[0] == float(np.float32(0.1)) and deq[1] == float(np.float32(1e-40))
    deq, s = oracle.quantize_tile(FP64, np.array([0.1]))
    assert s == 1.0 and deq[0] == 0.1
