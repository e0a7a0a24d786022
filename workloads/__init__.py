"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds none of the method's arithmetic: it only produces input
matrices (and the integer factors some of them are built from).  Both sides
may import it; neither side's arithmetic lives here.

Generators (recipes stated in DESIGN.md §4):
  * ``kms(n, rho)``              Kac-Murdock-Szego A_ij = rho^|i-j|  (C1)
  * ``plgsy(n, seed)``           PLASMA-plgsy-style random SPD: A_ij = A_ji =
                                 U(-0.5, 0.5) from a counter-based hash of
                                 (seed, max(i,j), min(i,j)), A_ii += n  (C2/C4)
  * ``matern_locations`` / ``matern_cov``  2-D Matern nu=0.5 covariance
                                 sigma^2 exp(-h/a) on uniform points, Morton
                                 sorted (C3/C5, G9)
  * ``integer_l0(n, seed)``      exact-recovery factor: unit-or-2 diagonal,
                                 +-1 entries only at (odd row, even col) so
                                 every Cholesky step is exact in fp64
  * ``banded(l0, bw)``           the same restricted to a band

The counter hash (``mix64``/``uniform``) is specified bit-exactly so a CUDA
generator can reproduce ``plgsy`` for bench-sized matrices without a host
copy: u = (mix64(key ^ mix64(seed + GOLDEN)) >> 11) * 2^-53.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
C1 = np.uint64(0xBF58476D1CE4E5B9)
C2 = np.uint64(0x94D049BB133111EB)


def mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * C1
        z = (z ^ (z >> np.uint64(27))) * C2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform(seed: int, i: np.ndarray, j: np.ndarray) -> np.ndarray:
    """U[0,1) from the counter (seed, i, j); i, j < 2^32."""
    with np.errstate(over="ignore"):
        s = mix64(np.uint64(seed) + GOLDEN)
        key = (np.asarray(i, dtype=np.uint64) << np.uint64(32)) | np.asarray(j, dtype=np.uint64)
        x = mix64(key ^ s)
    return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def pow_by_squaring(rho: float, d: np.ndarray) -> np.ndarray:
    """rho^d for integer d >= 0 by binary exponentiation (low bit first), the
    exact operation sequence the device generator uses, so both sides agree
    bit for bit (exact for rho = 0.5)."""
    d = np.asarray(d, dtype=np.int64)
    out = np.ones(d.shape, dtype=np.float64)
    base = np.full(d.shape, float(rho))
    e = d.copy()
    while np.any(e > 0):
        odd = (e & 1) == 1
        out = np.where(odd, out * base, out)
        e >>= 1
        base = np.where(e > 0, base * base, base)
    return out


def kms(n: int, rho: float) -> np.ndarray:
    idx = np.arange(n)
    return pow_by_squaring(rho, np.abs(idx[:, None] - idx[None, :]))


def plgsy(n: int, seed: int = 42) -> np.ndarray:
    """Random SPD: symmetric U(-0.5,0.5) plus n on the diagonal (fp64)."""
    i = np.arange(n, dtype=np.uint64)
    I, J = np.meshgrid(i, i, indexing="ij")
    hi = np.maximum(I, J)
    lo = np.minimum(I, J)
    A = uniform(seed, hi, lo) - 0.5
    A[np.arange(n), np.arange(n)] += float(n)
    return A


def _morton2(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    def spread(v):
        v = v.astype(np.uint64)
        v = (v | (v << np.uint64(8))) & np.uint64(0x00FF00FF)
        v = (v | (v << np.uint64(4))) & np.uint64(0x0F0F0F0F)
        v = (v | (v << np.uint64(2))) & np.uint64(0x33333333)
        v = (v | (v << np.uint64(1))) & np.uint64(0x55555555)
        return v
    return spread(x) | (spread(y) << np.uint64(1))


def matern_locations(n: int, seed: int = 1, morton: bool = True) -> np.ndarray:
    """n points uniform in [0,1]^2 from the counter hash; Morton (Z-order)
    sorted on a 2^16 grid per axis, ties broken by index (G9)."""
    idx = np.arange(n, dtype=np.uint64)
    xy = np.stack([uniform(seed, idx, np.zeros_like(idx)),
                   uniform(seed, idx, np.ones_like(idx))], axis=1)
    if morton:
        g = np.minimum((xy * 65536.0).astype(np.int64), 65535)
        code = _morton2(g[:, 0], g[:, 1])
        order = np.lexsort((np.arange(n), code))
        xy = xy[order]
    return xy


def matern_cov(xy: np.ndarray, sigma2: float = 1.0, a: float = 0.02627, nugget: float = 0.0) -> np.ndarray:
    """Matern nu = 0.5 (Eq. 2 closed form): sigma^2 exp(-h/a)."""
    d = xy[:, None, :] - xy[None, :, :]
    h = np.sqrt(d[..., 0] ** 2 + d[..., 1] ** 2)
    C = sigma2 * np.exp(-h / a)
    if nugget:
        C[np.arange(len(xy)), np.arange(len(xy))] += nugget
    return C


def integer_l0(n: int, seed: int = 7, density: float = 0.25, band: int | None = None) -> np.ndarray:
    """Exact-recovery factor L0 (fp64 lower-triangular).

    Diagonal entries are 1 or 2 (powers of two); off-diagonal entries are in
    {-1, 0, +1} and occur only at (i odd, j even), i > j (and |i - j| < band if
    given).  Then N = L0 - diag has N D^-1 N = 0, so L0^-1 and every block
    inverse are small dyadic matrices and every product, sum, square root and
    division met by any Cholesky ordering of A = L0 L0^T is exact in fp64.
    """
    i = np.arange(n, dtype=np.uint64)
    I, J = np.meshgrid(i, i, indexing="ij")
    u = uniform(seed, I, J)
    L = np.zeros((n, n), dtype=np.float64)
    mask = (I > J) & (I % np.uint64(2) == np.uint64(1)) & (J % np.uint64(2) == np.uint64(0))
    if band is not None:
        mask &= (I - J) < np.uint64(band)
    nz = mask & (u < density)
    sign = np.where(u < density / 2, -1.0, 1.0)
    L[nz] = sign[nz]
    d = np.where(uniform(seed + 1, i, i) < 0.5, 1.0, 2.0)
    L[np.arange(n), np.arange(n)] = d
    return L


def spd_from_l0(L0: np.ndarray) -> np.ndarray:
    """A = L0 L0^T (exact: small integers / dyadics)."""
    return L0 @ L0.T
