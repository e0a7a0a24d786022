/*
 * oracle.c -- CPU oracle for the mixed-precision left-looking tile Cholesky of
 * arxiv 2410.09819 ("Accelerating Mixed-Precision Out-of-Core Cholesky
 * Factorization with Static Task Scheduling").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this
 * code.  The product path (paper_2410_09819_b200/) never links, imports or
 * executes anything under oracle/, and the two share no code: no headers,
 * helpers, tables or constants.
 *
 * Plain, slow, obviously correct: fp64 everywhere, naive loops, no blocking
 * beyond the paper's own tiles.  Every function cites the passage it follows.
 *   P:n  = /root/reference/PAPER.md line n   (the paper's LaTeX)
 *   S:n  = /root/reference/SPEC.md  line n   (interface/test ideas only)
 *   G<k> = the reading of an ambiguous passage, listed in DESIGN.md §3
 *
 * Parity status:
 *   orc_round / orc_quantize_tile ... pinned (exhaustive FP16/E4M3 code
 *        points, numpy float16 / ml_dtypes cross-check, SPEC examples)
 *   orc_tile_norms / orc_plan ....... pinned (SPEC planner examples, norm
 *        closed forms, monotonicity)
 *   orc_factor (all-FP64 map) ....... pinned (KMS closed form, integer-L0
 *        exact recovery, Cholesky-Banachiewicz brute force, LAPACK)
 *   orc_factor (mixed map) .......... pinned at its three rounding points
 *        (O3 input quantization, quantize once after the TRSM, operand
 *        down-cast cast_c with the operand's own scale) by hand-derived
 *        Nt = 2..3 cases (tests/golden/mxp_rounding_points.json) that each
 *        misreading fails; plus the exact banded-L0 case and the reduction
 *        to the FP64 map.  Its accuracy on real maps is bounded through
 *        log-det / log-likelihood vs the FP64 factor.
 *   orc_logdet / orc_forward_solve .. pinned (SPEC examples, KMS closed form)
 *
 * Layout: A is column-major with leading dimension lda; only the lower
 * triangle is referenced (LAPACK dpotrf('L') convention).  Tiles are nb x nb,
 * column-major inside a tile.  Lower tiles are enumerated in
 * column-major tile order (0,0),(1,0),...,(Nt-1,0),(1,1),....
 * Precision codes: 0 = FP64, 1 = FP32, 2 = FP16, 3 = FP8 E4M3 (G10).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_FP64 0
#define ORC_FP32 1
#define ORC_FP16 2
#define ORC_FP8 3

/* ------------------------------------------------------------------------ */
/* O2: scalar rounding to a binary format, round-to-nearest-even.            */
/* p = significand bits incl. the implicit one, emin = minimum normal        */
/* exponent, maxfin = largest finite value, sat = saturate instead of inf.   */
/* FP32: p=24 emin=-126; FP16: p=11 emin=-14 max 65504; E4M3 (OCP "fn"):     */
/* p=4 emin=-6 max 448, saturating like cvt.rn.satfinite (G10).     */
/* ------------------------------------------------------------------------ */
static double round_format(double x, int p, int emin, double maxfin, int sat) {
    if (x == 0.0 || x != x) return x;
    double a = fabs(x);
    if (isinf(a)) return sat ? copysign(maxfin, x) : x;
    int E;
    frexp(a, &E);            /* a = f * 2^E, f in [0.5, 1)  ->  floor(log2 a) = E-1 */
    int e = E - 1;
    if (e < emin) e = emin;  /* subnormal range: fixed quantum */
    double q = ldexp(1.0, e - (p - 1));     /* spacing of representable values */
    double r = a / q;                      /* exact: division by a power of two */
    double fl = floor(r);
    double d = r - fl;                     /* exact */
    double R;
    if (d > 0.5) R = fl + 1.0;
    else if (d < 0.5) R = fl;
    else R = (fmod(fl, 2.0) == 0.0) ? fl : fl + 1.0;   /* tie -> even */
    double v = R * q;
    if (v > maxfin) v = sat ? maxfin : INFINITY;
    return copysign(v, x);
}

double orc_round(int prec, double x) {
    switch (prec) {
    case ORC_FP64: return x;
    case ORC_FP32: return round_format(x, 24, -126, 0x1.fffffep127, 0);
    case ORC_FP16: return round_format(x, 11, -14, 65504.0, 0);
    case ORC_FP8:  return round_format(x, 4, -6, 448.0, 1);
    default: return NAN;
    }
}

/* Unit roundoffs u_p: FP64 2^-53, FP32 2^-24, FP16 2^-11, E4M3 2^-4. */
double orc_unit_roundoff(int prec) {
    switch (prec) {
    case ORC_FP64: return ldexp(1.0, -53);
    case ORC_FP32: return ldexp(1.0, -24);
    case ORC_FP16: return ldexp(1.0, -11);
    case ORC_FP8:  return ldexp(1.0, -4);
    default: return NAN;
    }
}

/* O2 (G11): quantize a tile of cnt values to precision prec.
 * FP64: identity, s = 1.  FP32: RNE to binary32, s = 1.
 * FP16 / E4M3: amax = max|T|; s = 1 if amax = 0, else
 *   s = 2^clamp(E_p - floor(log2 amax), -127, 127), E_FP16 = 14, E_E4M3 = 7;
 *   codes = RNE_p(T * s); dequantized value = codes / s (exact in fp64).
 * Writes the dequantized values to out (may alias in) and returns s. */
double orc_quantize_tile(int prec, int64_t cnt, const double* in, double* out) {
    double s = 1.0;
    if (prec == ORC_FP16 || prec == ORC_FP8) {
        double amax = 0.0;
        for (int64_t i = 0; i < cnt; ++i) {
            double a = fabs(in[i]);
            if (a > amax) amax = a;
        }
        if (amax > 0.0) {
            int E;
            frexp(amax, &E);
            int e = E - 1;
            int Ep = (prec == ORC_FP16) ? 14 : 7;
            int k = Ep - e;
            if (k > 127) k = 127;
            if (k < -127) k = -127;
            s = ldexp(1.0, k);
        }
    }
    for (int64_t i = 0; i < cnt; ++i) {
        double code = orc_round(prec, in[i] * s);
        out[i] = code / s;
    }
    return s;
}

/* O4.2.3 / G12: operand cast to the compute precision c of a GEMM,
 *   cast_c(T) = deq(q_c(deq(T)))  when T is stored MORE precise than c
 *                                  (down-cast with T's own new scale);
 *   cast_c(T) = T                  when T is stored no more precise than c
 *                                  (an exact up-cast, "up/down-casting").
 * (Re-quantizing an up-cast with a scale recomputed from the stored amax is
 * not always the identity: when the tile's amax rounded up into the next
 * binade its scale halves, and odd subnormal codes would round again.)
 * Codes: lower = more precise (FP64 0 ... FP8 3). */
void orc_cast_tile(int c, int stored, int64_t cnt, const double* in, double* out) {
    if (stored >= c) {
        if (out != in) memcpy(out, in, sizeof(double) * (size_t)cnt);
        return;
    }
    orc_quantize_tile(c, cnt, in, out);
}

/* ------------------------------------------------------------------------ */
/* O0 tiling helpers.  Tile (i,j) holds rows i*nb.., cols j*nb..; padding   */
/* is 0, with 1 on the padded diagonal.                              */
/* ------------------------------------------------------------------------ */
static int64_t n_tiles(int64_t n, int64_t nb) { return (n + nb - 1) / nb; }

/* column-major lower-tile index of (i, j), i >= j */
int64_t orc_tile_index(int64_t Nt, int64_t i, int64_t j) {
    return j * Nt - j * (j - 1) / 2 + (i - j);
}

static void load_tile(int64_t n, int64_t nb, const double* A, int64_t lda,
                      int64_t ti, int64_t tj, double* T) {
    for (int64_t c = 0; c < nb; ++c)
        for (int64_t r = 0; r < nb; ++r) {
            int64_t gi = ti * nb + r, gj = tj * nb + c;
            double v;
            if (gi < n && gj < n) v = (gi >= gj) ? A[gi + gj * lda] : A[gj + gi * lda];
            else v = (gi == gj) ? 1.0 : 0.0;
            T[r + c * nb] = v;
        }
}

static void store_tile(int64_t n, int64_t nb, double* A, int64_t lda,
                       int64_t ti, int64_t tj, const double* T) {
    for (int64_t c = 0; c < nb; ++c)
        for (int64_t r = 0; r < nb; ++r) {
            int64_t gi = ti * nb + r, gj = tj * nb + c;
            if (gi < n && gj < n && gi >= gj) A[gi + gj * lda] = T[r + c * nb];
        }
}

/* ------------------------------------------------------------------------ */
/* O1: tile Frobenius norms and the precision planner.    */
/* f_ij = sqrt(sum x^2) over the tile's real (non-padded) entries, fp64,     */
/* column-major element order.                                               */
/* ------------------------------------------------------------------------ */
void orc_tile_norms(int64_t n, int64_t nb, const double* A, int64_t lda, double* norms) {
    int64_t Nt = n_tiles(n, nb);
    for (int64_t j = 0; j < Nt; ++j)
        for (int64_t i = j; i < Nt; ++i) {
            double ss = 0.0;
            for (int64_t c = j * nb; c < (j + 1) * nb && c < n; ++c)
                for (int64_t r = i * nb; r < (i + 1) * nb && r < n; ++r) {
                    double v = (r >= c) ? A[r + c * lda] : A[c + r * lda];
                    ss += v * v;
                }
            norms[orc_tile_index(Nt, i, j)] = sqrt(ss);
        }
}

/* Planner, G6: p_ij = least precise p in `allowed` with
 *   Nt * f_ij / F < eps / u_p     (strict)
 * else the most precise allowed; diagonal tiles = most precise allowed.
 * F = sqrt(sum_i f_ii^2 + 2 sum_{i>j} f_ij^2).
 * allowed: bit p set => precision p allowed.  Returns 0, or -1 for F = 0
 * (ZeroMatrix), -2 for an empty mask. */
int orc_plan(int64_t n, int64_t nb, const double* A, int64_t lda, double eps,
             uint32_t allowed, uint8_t* map) {
    int64_t Nt = n_tiles(n, nb);
    int64_t T = Nt * (Nt + 1) / 2;
    if ((allowed & 0xF) == 0) return -2;
    double* f = (double*)malloc(sizeof(double) * (size_t)T);
    orc_tile_norms(n, nb, A, lda, f);
    double ss = 0.0;
    for (int64_t j = 0; j < Nt; ++j)
        for (int64_t i = j; i < Nt; ++i) {
            double v = f[orc_tile_index(Nt, i, j)];
            ss += (i == j) ? v * v : 2.0 * v * v;
        }
    double F = sqrt(ss);
    if (F == 0.0) { free(f); return -1; }
    int most = 3;
    for (int p = 0; p < 4; ++p) if (allowed & (1u << p)) { most = p; break; }
    for (int64_t j = 0; j < Nt; ++j)
        for (int64_t i = j; i < Nt; ++i) {
            int64_t t = orc_tile_index(Nt, i, j);
            int choice = most;
            if (i != j) {
                double ratio = (double)Nt * f[t] / F;
                for (int p = 3; p >= 0; --p) {          /* least precise first */
                    if (!(allowed & (1u << p))) continue;
                    if (ratio < eps / orc_unit_roundoff(p)) { choice = p; break; }
                }
            }
            map[t] = (uint8_t)choice;
        }
    free(f);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Unblocked Cholesky of an m x m block, kij order, lower.   */
/* Returns 0 or the 1-based index of the first non-positive / NaN pivot.    */
/* ------------------------------------------------------------------------ */
int64_t orc_potrf_unblocked(int64_t m, double* C, int64_t ldc) {
    for (int64_t k = 0; k < m; ++k) {
        double d = C[k + k * ldc];
        if (!(d > 0.0)) return k + 1;
        d = sqrt(d);
        C[k + k * ldc] = d;
        for (int64_t i = k + 1; i < m; ++i) C[i + k * ldc] /= d;
        for (int64_t j = k + 1; j < m; ++j)
            for (int64_t i = j; i < m; ++i)
                C[i + j * ldc] -= C[i + k * ldc] * C[j + k * ldc];
    }
    for (int64_t j = 1; j < m; ++j)
        for (int64_t i = 0; i < j; ++i) C[i + j * ldc] = 0.0;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* O4: the left-looking tile factorization (Alg. 1, Alg. 2        */
/* P:240-278), with per-tile precision.                        */
/*                                                                            */
/* Diagonal task (m == k), P:96 SYRK + POTRF:                                 */
/*   C <- A^_kk;  for n = 0..k-1:  C <- C - L_kn L_kn^T  (fp64, operands the  */
/*   stored values, exactly up-cast);  L_kk = chol(C) (kij, unblocked).       */
/* Off-diagonal task (m > k), P:96 GEMM + TRSM (G1, G2, G3):                  */
/*   c = p_mk;  C <- A^_mk;                                                    */
/*   for n = 0..k-1:  C <- C - cast_c(L_mn) cast_c(L_kn)^T   (G12)             */
/*   X solves X L_kk^T = C, column-wise forward substitution (G13);    */
/*   L_mk = deq(q_{p_mk}(X))   (quantize once per task, after TRSM).          */
/* A^_ij = deq(q_{p_ij}(A_ij)) is the stored input (O3, G14).                 */
/* cast_c(T): orc_cast_tile (down-cast deq(q_c(T)), up-cast identity). */
/*                                                                            */
/* A (n x n, lda, lower) is overwritten by L (dequantized values); the strict */
/* upper triangle is untouched.  map = NULL means all FP64.                   */
/* Returns info: 0, or the global 1-based row of the first non-PD pivot; on  */
/* failure the columns before the failing tile column hold L.                */
/* ------------------------------------------------------------------------ */
int64_t orc_factor(int64_t n, int64_t nb, double* A, int64_t lda, const uint8_t* map) {
    int64_t Nt = n_tiles(n, nb);
    int64_t T = Nt * (Nt + 1) / 2;
    int64_t tsz = nb * nb;
    double* tiles = (double*)malloc(sizeof(double) * (size_t)(T * tsz));
    if (!tiles) return -1;
#define TILE(i, j) (tiles + orc_tile_index(Nt, (i), (j)) * tsz)
#define PREC(i, j) (map ? (int)map[orc_tile_index(Nt, (i), (j))] : ORC_FP64)
    /* O0 + O3: tile, pad, and store every input tile at its precision */
    for (int64_t j = 0; j < Nt; ++j)
        for (int64_t i = j; i < Nt; ++i) {
            load_tile(n, nb, A, lda, i, j, TILE(i, j));
            orc_quantize_tile(PREC(i, j), tsz, TILE(i, j), TILE(i, j));
        }
    int64_t info = 0;
    for (int64_t k = 0; k < Nt && info == 0; ++k) {
        /* ---- diagonal task: SYRK chain then POTRF ---- */
        {
            double* C = TILE(k, k);
            for (int64_t nn = 0; nn < k; ++nn) {
                const double* Lkn = TILE(k, nn);
                for (int64_t c = 0; c < nb; ++c)
                    for (int64_t p = 0; p < nb; ++p) {
                        double y = Lkn[c + p * nb];
                        for (int64_t r = c; r < nb; ++r) C[r + c * nb] -= Lkn[r + p * nb] * y;
                    }
            }
            int64_t piv = orc_potrf_unblocked(nb, C, nb);
            if (piv) { info = k * nb + piv; break; }
            orc_quantize_tile(PREC(k, k), tsz, C, C);
        }
        /* ---- off-diagonal tasks of column k: GEMM chain then TRSM ---- */
        const double* Lkk = TILE(k, k);
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t m = k + 1; m < Nt; ++m) {
            int c_prec = PREC(m, k);
            double* C = TILE(m, k);
            double* X = (double*)malloc(sizeof(double) * (size_t)tsz);
            double* Y = (double*)malloc(sizeof(double) * (size_t)tsz);
            for (int64_t nn = 0; nn < k; ++nn) {
                orc_cast_tile(c_prec, PREC(m, nn), tsz, TILE(m, nn), X);   /* cast_c(L_mn) */
                orc_cast_tile(c_prec, PREC(k, nn), tsz, TILE(k, nn), Y);   /* cast_c(L_kn) */
                for (int64_t c = 0; c < nb; ++c)
                    for (int64_t p = 0; p < nb; ++p) {
                        double y = Y[c + p * nb];
                        for (int64_t r = 0; r < nb; ++r) C[r + c * nb] -= X[r + p * nb] * y;
                    }
            }
            /* TRSM: X Lkk^T = C, columns j = 0..nb-1 in order */
            for (int64_t j = 0; j < nb; ++j) {
                for (int64_t i = 0; i < j; ++i) {
                    double l = Lkk[j + i * nb];
                    for (int64_t r = 0; r < nb; ++r) C[r + j * nb] -= C[r + i * nb] * l;
                }
                double d = Lkk[j + j * nb];
                for (int64_t r = 0; r < nb; ++r) C[r + j * nb] /= d;
            }
            orc_quantize_tile(PREC(m, k), tsz, C, C);
            free(X);
            free(Y);
        }
    }
    /* O5: write back every finished tile column */
    for (int64_t j = 0; j < Nt; ++j) {
        if (info && j >= (info - 1) / nb) break;
        for (int64_t i = j; i < Nt; ++i) store_tile(n, nb, A, lda, i, j, TILE(i, j));
    }
#undef TILE
#undef PREC
    free(tiles);
    return info;
}

/* O5: logdet = 2 * sum_{i<n} log L_ii, ascending. */
double orc_logdet(int64_t n, const double* L, int64_t lda) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += log(L[i + i * lda]);
    return 2.0 * s;
}

/* O6: forward substitution L z = y in place (P:172 quadratic form). */
void orc_forward_solve(int64_t n, const double* L, int64_t lda, double* y) {
    for (int64_t j = 0; j < n; ++j) {
        y[j] /= L[j + j * lda];
        double v = y[j];
        for (int64_t i = j + 1; i < n; ++i) y[i] -= L[i + j * lda] * v;
    }
}
