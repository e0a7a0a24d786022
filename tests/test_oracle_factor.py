"""Pins for the oracle's factorization, planner and statistics.

Closed forms (KMS), exact recovery (integer L0), an independent
Cholesky-Banachiewicz brute force, LAPACK, and the SPEC worked examples.
"""
import math

import numpy as np
import pytest
import scipy.linalg

import oracle
import workloads as w
from oracle import FP8, FP16, FP32, FP64


def banachiewicz(A):
    """Row-by-row (Cholesky-Banachiewicz) brute force, pure Python, tiny n."""
    n = A.shape[0]
    L = [[0.0] * n for _ in range(n)]
    for i in range(n):
        for j in range(i + 1):
            s = sum(L[i][k] * L[j][k] for k in range(j))
            if i == j:
                L[i][j] = math.sqrt(A[i][i] - s)
            else:
                L[i][j] = (A[i][j] - s) / L[j][j]
    return np.array(L)


# ---------------------------------------------------------------- SPEC examples
def test_spec_potrf(golden):
    ex = golden["potrf"][0]
    A = np.array(ex["A"], float)
    for nb in (1, 2):
        L, info = oracle.factor(A, nb)
        assert info == 0 and np.array_equal(L, np.array(ex["L"], float)), ex["cite"]
    L, info = oracle.potrf_unblocked(A)
    assert info == 0 and np.array_equal(np.tril(L), np.array(ex["L"], float))


def test_spec_trsm_inside_factor(golden):
    """Embed the SPEC TRSM example (X Lkk^T = Amk) as tile (1,0) of a 4x4 factor."""
    ex = golden["trsm"][0]
    Lkk = np.array(ex["Lkk"], float)
    X = np.vstack([np.array(ex["X"], float), [[0.0, 1.0]]])
    L = np.zeros((4, 4))
    L[:2, :2] = Lkk
    L[2:, :2] = X
    L[2:, 2:] = np.eye(2)
    A = L @ L.T
    assert np.array_equal(A[2:3, :2], np.array(ex["Amk"], float)), ex["cite"]
    Lo, info = oracle.factor(A, 2)
    assert info == 0 and np.array_equal(Lo, L)


def test_spec_syrk_gemm_inside_factor(golden):
    """S:168 / S:177: with L(1,0) = I the SYRK of tile (1,1) gives 2I - I = I and
    the GEMM of tile (2,1) with zero input gives -I before its TRSM."""
    L = np.zeros((6, 6))
    for b in range(3):
        L[2 * b:2 * b + 2, 2 * b:2 * b + 2] = np.eye(2)
    L[2:4, 0:2] = np.eye(2)
    L[4:6, 0:2] = np.eye(2)
    L[4:6, 2:4] = -np.eye(2)   # C(2,1) = 0 - L(2,0) L(1,0)^T = -I, TRSM with I -> -I
    A = L @ L.T
    assert np.array_equal(A[2:4, 2:4], 2 * np.eye(2))
    assert np.array_equal(A[4:6, 2:4], np.zeros((2, 2)))
    Lo, info = oracle.factor(A, 2)
    assert info == 0 and np.array_equal(Lo, L)


def test_spec_norms(golden):
    assert oracle.tile_norms(np.array([[3.0, 0.0], [0.0, 4.0]]), 2)[0] == 5.0
    f = oracle.tile_norms(np.eye(4), 2)
    assert np.allclose(f, [math.sqrt(2), 0.0, math.sqrt(2)])
    # matrix norm with off-diagonal tiles counted twice equals the dense norm
    A = w.plgsy(24, seed=3)
    f = oracle.tile_norms(A, 8)
    Nt = 3
    F2 = sum((f[oracle.tile_index(Nt, i, j)] ** 2) * (1 if i == j else 2)
             for j in range(Nt) for i in range(j, Nt))
    assert math.isclose(math.sqrt(F2), np.linalg.norm(A), rel_tol=1e-14)


def test_spec_logdet_loglik(golden):
    for ex in golden["logdet"]:
        if "L_diag" in ex:
            L = np.diag(np.array(ex["L_diag"], float))
        else:
            L, info = oracle.factor(np.array(ex["Sigma"], float), 1)
            assert info == 0
        tol = ex.get("tol", 0.0)
        assert abs(oracle.logdet(L) - ex["expect"]) <= tol + 1e-15, ex["cite"]
    for ex in golden["loglik_y0"]:
        L, info = oracle.factor(np.array(ex["Sigma"], float), 2)
        assert abs(oracle.loglik(L) - ex["expect"]) <= ex["tol"], ex["cite"]
    assert math.isclose(golden["logdet"][1]["expect"], 6 * math.log(2), abs_tol=1e-4)


def test_task_order(golden):
    """Column-major lower-tile enumeration = oracle.tile_index."""
    order = golden["task_order_Nt3"]["order"]
    assert [oracle.tile_index(3, i, j) for i, j in order] == list(range(6))


# --------------------------------------------------------------- closed forms
def test_kms_closed_form_c1(golden):
    g = golden["kms_c1"]
    n, nb, rho = g["n"], g["nb"], g["rho"]
    A = w.kms(n, rho)
    L, info = oracle.factor(A, nb)
    assert info == 0
    i = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    Lc = np.where(i >= j, np.power(rho, (i - j).astype(float)), 0.0)
    Lc[:, 1:] *= math.sqrt(1 - rho * rho)
    assert np.max(np.abs(L - Lc)) <= 1e-14 * np.max(np.abs(Lc))
    ld = oracle.logdet(L)
    closed = (n - 1) * math.log(1 - rho * rho)
    assert math.isclose(closed, g["logdet"], rel_tol=1e-15)
    assert abs(ld - closed) <= 1e-12 * abs(closed)


def test_kms_strong_correlation():
    A = w.kms(300, 0.99)
    L, info = oracle.factor(A, 64)
    assert info == 0
    assert abs(oracle.logdet(L) - 299 * math.log(1 - 0.99 ** 2)) <= 1e-10 * 300


@pytest.mark.parametrize("n,nb", [(256, 64), (256, 256), (200, 48), (130, 16), (96, 7)])
def test_integer_l0_exact_recovery(n, nb):
    L0 = w.integer_l0(n, seed=n + nb)
    A = w.spd_from_l0(L0)
    L, info = oracle.factor(A, nb)
    assert info == 0
    assert np.array_equal(L, L0)


@pytest.mark.parametrize("n,nb", [(12, 4), (20, 5), (17, 4), (33, 8), (48, 48), (40, 64)])
def test_banachiewicz_brute_force(n, nb):
    A = w.plgsy(n, seed=n) + 0.0
    A = A + np.diag(np.linspace(0, 3, n))  # vary the diagonal a little
    Lb = banachiewicz(A)
    L, info = oracle.factor(A, nb)
    assert info == 0
    assert np.max(np.abs(L - Lb)) <= 1e-14 * np.max(np.abs(Lb))


def test_lapack_and_nb_invariance():
    n = 512
    A = w.plgsy(n, seed=42)
    Lref = np.linalg.cholesky(A)
    Ls = []
    for nb in (64, 128, 256, 100):
        L, info = oracle.factor(A, nb)
        assert info == 0
        assert np.max(np.abs(L - Lref)) <= 1e-13 * np.max(np.abs(Lref))
        Ls.append(L)
    for L in Ls[1:]:
        assert np.max(np.abs(L - Ls[0])) <= 1e-13 * np.max(np.abs(Ls[0]))
    be = np.linalg.norm(A - Ls[0] @ Ls[0].T) / np.linalg.norm(A)
    assert be <= 1e-15


def test_nb_equals_n_is_unblocked():
    A = w.plgsy(64, seed=9)
    L1, _ = oracle.factor(A, 64)
    L2, _ = oracle.potrf_unblocked(A)
    assert np.array_equal(L1, np.tril(L2))


def test_matern_factor_against_lapack():
    xy = w.matern_locations(1024, seed=1)
    S = w.matern_cov(xy, 1.0, 0.078809)
    L, info = oracle.factor(S, 128)
    assert info == 0
    Lref = np.linalg.cholesky(S)
    assert np.max(np.abs(L - Lref)) <= 1e-10 * np.max(np.abs(Lref))
    ld_ref = 2 * np.sum(np.log(np.diag(Lref)))
    assert abs(oracle.logdet(L) - ld_ref) <= 1e-9 * abs(ld_ref)


@pytest.mark.parametrize("n,nb,j", [(64, 16, 37), (64, 16, 0), (50, 16, 49), (33, 8, 8)])
def test_not_pd_info(n, nb, j):
    """info = global 1-based row of the first non-positive pivot (LAPACK)."""
    L0 = w.integer_l0(n, seed=5)
    A = w.spd_from_l0(L0)
    A[j, j] = -1.0 + np.sum(L0[j, :j] ** 2)  # pivot j becomes sqrt(-1)
    L, info = oracle.factor(A, nb)
    assert info == j + 1
    kfail = j // nb
    assert np.array_equal(L[:, : kfail * nb], L0[:, : kfail * nb])


# --------------------------------------------------------------- planner (O1)
def test_planner_spec_examples():
    nb, Nt = 4, 8
    n = nb * Nt
    A = np.eye(n)
    m = oracle.plan(A, nb, 1e-8)
    off = [oracle.tile_index(Nt, i, j) for j in range(Nt) for i in range(j + 1, Nt)]
    diag = [oracle.tile_index(Nt, i, i) for i in range(Nt)]
    assert np.all(m[off] == FP8)  # zero tiles -> lowest precision
    assert np.all(m[diag] == FP64)
    assert np.all(oracle.plan(A, nb, 1e-8, allowed=1 << FP64) == FP64)
    # one off-diagonal tile holds the entire norm: ratio = Nt*f/F = 8/sqrt(2)
    B = np.zeros((n, n))
    B[8:12, 0:4] = 1.0
    B[0:4, 8:12] = 1.0
    m = oracle.plan(B, nb, 1e-8)
    assert m[oracle.tile_index(Nt, 2, 0)] == FP64
    with pytest.raises(ZeroDivisionError):
        oracle.plan(np.zeros((n, n)), nb, 1e-8)


def test_planner_thresholds_exact():
    """Single tile with a known norm ratio lands exactly where eps/u_p puts it."""
    nb, Nt = 2, 2
    # diag tiles identity (norm sqrt2 each), off-diagonal tile value t in one entry
    for t, eps, expect in [(1e-9, 1e-5, FP8), (1e-6, 1e-5, FP8), (1e-3, 1e-5, FP16),
                           (1e-1, 1e-5, FP32), (1e-2, 1e-9, FP32), (0.5, 1e-9, FP64)]:
        A = np.eye(4)
        A[2, 0] = A[0, 2] = t
        F = math.sqrt(4 + 2 * t * t)
        ratio = Nt * t / F
        m = oracle.plan(A, nb, eps)
        p = m[oracle.tile_index(Nt, 1, 0)]
        assert p == expect, (t, eps, ratio)
        # the chosen p satisfies the criterion and every less precise one fails
        u = {FP64: 2.0 ** -53, FP32: 2.0 ** -24, FP16: 2.0 ** -11, FP8: 2.0 ** -4}
        assert p == FP64 or ratio < eps / u[p]
        for q in range(p + 1, 4):
            assert not ratio < eps / u[q]


def test_planner_monotone_and_correlation():
    xy = w.matern_locations(2048, seed=1)
    weak = w.matern_cov(xy, 1.0, 0.02627)
    strong = w.matern_cov(xy, 1.0, 0.210158)
    nb = 128
    mw5 = oracle.plan(weak, nb, 1e-5)
    mw8 = oracle.plan(weak, nb, 1e-8)
    ms5 = oracle.plan(strong, nb, 1e-5)
    assert np.all(mw8 <= mw5)  # tighter eps -> never less precise
    assert np.sum(mw5 == FP8) > np.sum(ms5 == FP8)
    f = oracle.tile_norms(weak, nb)
    order = np.argsort(f, kind="stable")
    Nt = 2048 // nb
    isdiag = np.zeros_like(f, dtype=bool)
    isdiag[[oracle.tile_index(Nt, i, i) for i in range(Nt)]] = True
    fo = order[~isdiag[order]]
    assert np.all(np.diff(mw5[fo].astype(int)) <= 0)  # larger norm -> more precise


# --------------------------------------------------------------- MxP reductions
def test_fp64_map_reduces_to_fp64_oracle():
    A = w.plgsy(256, seed=4)
    Nt = 4
    L1, _ = oracle.factor(A, 64)
    L2, _ = oracle.factor(A, 64, np.zeros(Nt * (Nt + 1) // 2, np.uint8))
    assert np.array_equal(L1, L2)


def test_banded_l0_mxp_exact():
    """Banded integer L0 (bandwidth < nb): far tiles are zero -> planned FP8 with
    s = 1; near tiles hold small integers representable in every precision the
    planner may pick -> L0 recovered bitwise through the MxP plumbing."""
    n, nb = 256, 32
    L0 = w.integer_l0(n, seed=11, band=20)
    A = w.spd_from_l0(L0)
    m = oracle.plan(A, nb, 1e-3)
    assert np.sum(m == FP8) > 0 and np.sum(m == FP64) >= n // nb
    L, info = oracle.factor(A, nb, m)
    assert info == 0 and np.array_equal(L, L0)


def test_mxp_accuracy_against_fp64():
    """Not a parity pin (the mixed factor has no closed form): the MxP log-det
    stays close to the FP64 one and the backward error is O(eps)."""
    xy = w.matern_locations(1024, seed=1)
    S = w.matern_cov(xy, 1.0, 0.02627)
    nb = 64
    L64, _ = oracle.factor(S, nb)
    for eps in (1e-5, 1e-8):
        m = oracle.plan(S, nb, eps)
        L, info = oracle.factor(S, nb, m)
        assert info == 0
        be = np.linalg.norm(S - L @ L.T) / np.linalg.norm(S)
        assert be < 50 * eps
        assert abs(oracle.logdet(L) - oracle.logdet(L64)) < 1e3 * eps * 1024


# --------------------------------------------------------------- stats
def test_forward_solve_and_loglik():
    A = w.plgsy(128, seed=8)
    L, _ = oracle.factor(A, 32)
    y = np.sin(np.arange(128))
    z = oracle.forward_solve(L, y)
    zr = scipy.linalg.solve_triangular(np.linalg.cholesky(A), y, lower=True)
    assert np.max(np.abs(z - zr)) <= 1e-13 * np.max(np.abs(zr))
    ll = oracle.loglik(L, y)
    sign, ld = np.linalg.slogdet(A)
    ref = -64 * math.log(2 * math.pi) - 0.5 * ld - 0.5 * y @ np.linalg.solve(A, y)
    assert math.isclose(ll, ref, rel_tol=1e-12)
    # block-diagonal additivity of log-det
    B = np.zeros((256, 256))
    B[:128, :128] = A
    B[128:, 128:] = w.kms(128, 0.3)
    Lb, _ = oracle.factor(B, 64)
    La, _ = oracle.factor(w.kms(128, 0.3), 64)
    assert math.isclose(oracle.logdet(Lb), oracle.logdet(L) + oracle.logdet(La), rel_tol=1e-13)


# --------------------------------------------------------------- generators
def test_generators(golden):
    assert int(w.mix64(np.uint64(0) + w.GOLDEN)) == int(golden["splitmix64_seed0_first"]["value"], 16)
    for ex in golden["matern"]:
        s2, a, nu = ex["theta"]
        xy = np.array([[0.0, 0.0], [ex["h"], 0.0]])
        C = w.matern_cov(xy, s2, a)
        assert abs(C[0, 1] - ex["expect"]) <= ex.get("tol", 0) + (1e-15 if ex["h"] else 0), ex["cite"]
    A = w.plgsy(64, 42)
    assert np.array_equal(A, A.T) and np.all(np.abs(A - np.diag(np.diag(A))) <= 0.5)
    xy = w.matern_locations(4096, seed=1)
    assert abs(xy[:, 0].mean() - 0.5) < 0.02 and xy.min() >= 0 and xy.max() < 1
    S = w.matern_cov(xy[:256], 1.0, 0.02627)
    assert np.all(np.diag(S) >= np.max(np.abs(S - np.diag(np.diag(S))), axis=1))
