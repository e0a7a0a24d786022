"""CPU oracle for the MxP left-looking tile Cholesky (arxiv 2410.09819).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2410_09819_b200`` never imports it and
shares no code with it (no kernels, headers, helpers, tables or constants).

The arithmetic lives in plain C (``oracle.c``, fp64, naive loops, every
function citing the paper passage it follows); this module only compiles it
with gcc and marshals numpy arrays through ctypes.

Parity status: quantizers, norms, planner, the all-FP64
factorization, log-det and forward solve are pinned by tests that do not
re-use this code.  The mixed-precision factorization is pinned at each of its
rounding points (O3 input quantization, quantize-after-TRSM, operand down-cast)
by hand-derived cases in tests/golden/mxp_rounding_points.json, plus its exact
special cases (banded integer L0, reduction to the FP64 map).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

FP64, FP32, FP16, FP8 = 0, 1, 2, 3
PREC_NAMES = {FP64: "FP64", FP32: "FP32", FP16: "FP16", FP8: "FP8E4M3"}

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc -O2 -fopenmp).  Returns the path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        # -ffp-contract=off: no fused multiply-add, every product and sum is a
        # separately rounded fp64 operation, as the oracle's text reads.
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        lib = ctypes.CDLL(build())
        i64, dbl, u32 = ctypes.c_int64, ctypes.c_double, ctypes.c_uint32
        pd = ctypes.POINTER(ctypes.c_double)
        pu8 = ctypes.POINTER(ctypes.c_uint8)
        lib.orc_round.argtypes = [ctypes.c_int, dbl]
        lib.orc_round.restype = dbl
        lib.orc_unit_roundoff.argtypes = [ctypes.c_int]
        lib.orc_unit_roundoff.restype = dbl
        lib.orc_quantize_tile.argtypes = [ctypes.c_int, i64, pd, pd]
        lib.orc_quantize_tile.restype = dbl
        lib.orc_cast_tile.argtypes = [ctypes.c_int, ctypes.c_int, i64, pd, pd]
        lib.orc_cast_tile.restype = None
        lib.orc_tile_index.argtypes = [i64, i64, i64]
        lib.orc_tile_index.restype = i64
        lib.orc_tile_norms.argtypes = [i64, i64, pd, i64, pd]
        lib.orc_tile_norms.restype = None
        lib.orc_plan.argtypes = [i64, i64, pd, i64, dbl, u32, pu8]
        lib.orc_plan.restype = ctypes.c_int
        lib.orc_potrf_unblocked.argtypes = [i64, pd, i64]
        lib.orc_potrf_unblocked.restype = i64
        lib.orc_factor.argtypes = [i64, i64, pd, i64, pu8]
        lib.orc_factor.restype = i64
        lib.orc_logdet.argtypes = [i64, pd, i64]
        lib.orc_logdet.restype = dbl
        lib.orc_forward_solve.argtypes = [i64, pd, i64, pd]
        lib.orc_forward_solve.restype = None
        _lib = lib
        return lib


def _pd(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _colmajor(A: np.ndarray) -> np.ndarray:
    """fp64 Fortran-ordered copy (column-major, lda = n)."""
    return np.array(A, dtype=np.float64, order="F", copy=True)


def round_scalar(prec: int, x: float) -> float:
    """O2 scalar RNE rounding to precision ``prec`` (E4M3 saturating)."""
    return _load().orc_round(prec, float(x))


def round_array(prec: int, x) -> np.ndarray:
    lib = _load()
    x = np.asarray(x, dtype=np.float64)
    return np.vectorize(lambda v: lib.orc_round(prec, float(v)), otypes=[np.float64])(x)


def unit_roundoff(prec: int) -> float:
    return _load().orc_unit_roundoff(prec)


def quantize_tile(prec: int, T) -> tuple[np.ndarray, float]:
    """O2: returns (dequantized values, pow2 scale s); codes = deq * s."""
    T = np.ascontiguousarray(T, dtype=np.float64)
    out = np.empty_like(T)
    s = _load().orc_quantize_tile(prec, T.size, _pd(T), _pd(out))
    return out, s


def cast_tile(c: int, stored: int, T) -> np.ndarray:
    """O4.2.3: operand cast of a tile stored at ``stored`` to compute precision ``c``."""
    T = np.ascontiguousarray(T, dtype=np.float64)
    out = np.empty_like(T)
    _load().orc_cast_tile(c, stored, T.size, _pd(T), _pd(out))
    return out


def tile_index(Nt: int, i: int, j: int) -> int:
    return _load().orc_tile_index(Nt, i, j)


def tile_norms(A: np.ndarray, nb: int) -> np.ndarray:
    n = A.shape[0]
    Af = _colmajor(A)
    Nt = -(-n // nb)
    out = np.empty(Nt * (Nt + 1) // 2, dtype=np.float64)
    _load().orc_tile_norms(n, nb, _pd(Af), n, _pd(out))
    return out


def plan(A: np.ndarray, nb: int, eps: float, allowed: int = 0xF) -> np.ndarray:
    """O1 planner: uint8 precision map in column-major lower-tile order."""
    n = A.shape[0]
    Af = _colmajor(A)
    Nt = -(-n // nb)
    m = np.empty(Nt * (Nt + 1) // 2, dtype=np.uint8)
    rc = _load().orc_plan(n, nb, _pd(Af), n, float(eps), allowed,
                          m.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))
    if rc == -1:
        raise ZeroDivisionError("ZeroMatrix: ||A||_F = 0")
    if rc != 0:
        raise ValueError(f"orc_plan failed: {rc}")
    return m


def potrf_unblocked(A: np.ndarray) -> tuple[np.ndarray, int]:
    Af = _colmajor(A)
    info = _load().orc_potrf_unblocked(Af.shape[0], _pd(Af), Af.shape[0])
    return Af, int(info)


def factor(A: np.ndarray, nb: int, pmap: np.ndarray | None = None) -> tuple[np.ndarray, int]:
    """O4: tile left-looking MxP Cholesky.  Returns (L lower, zeros above), info."""
    n = A.shape[0]
    Af = _colmajor(A)
    if pmap is None:
        mp = None
    else:
        pmap = np.ascontiguousarray(pmap, dtype=np.uint8)
        mp = pmap.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    info = _load().orc_factor(n, nb, _pd(Af), n, mp)
    if info < 0:
        raise MemoryError("oracle allocation failed")
    return np.tril(Af), int(info)


def logdet(L: np.ndarray) -> float:
    Lf = _colmajor(L)
    return _load().orc_logdet(Lf.shape[0], _pd(Lf), Lf.shape[0])


def forward_solve(L: np.ndarray, y) -> np.ndarray:
    Lf = _colmajor(L)
    z = np.array(y, dtype=np.float64, copy=True)
    _load().orc_forward_solve(Lf.shape[0], _pd(Lf), Lf.shape[0], _pd(z))
    return z


def loglik(L: np.ndarray, y=None) -> float:
    """O6 / Eq. 1: -(n/2) log 2pi - 1/2 logdet - 1/2 ||L^-1 y||^2."""
    n = L.shape[0]
    ld = logdet(L)
    q = 0.0
    if y is not None:
        z = forward_solve(L, y)
        q = float(np.dot(z, z))
    return -0.5 * n * np.log(2.0 * np.pi) - 0.5 * ld - 0.5 * q


def kl_divergence(loglik_exact: float, loglik_approx: float) -> float:
    """Eq. 3, implemented as written (G17)."""
    return loglik_exact - loglik_approx
