// solve.cu -- forward substitution L z = y on the resident tile factor and the
// Gaussian log-likelihood (Eq. 1, the
// quadratic form y^T Sigma^-1 y = ||z||^2 with L z = y).
//
// HBM-bound: every lower tile of L is read once (nb^2 * 8 bytes per tile,
// n^2/2 * 8 bytes in all).  Tile column k: the diagonal solve
// z_k = L_kk^-1 r_k (one CTA, blocked by 128 with the inverses W_J = L_JJ^-1
// the POTRF left in wbuf), then r_m -= L_mk z_k for every m > k (one CTA per
// 128-row block).  Every sum runs in a fixed order: the result is bitwise
// reproducible.
#include "internal.h"
#include "quant.cuh"

namespace mxp {
namespace {

// r[m*nb + rows] -= L(m,k)[rows, :] z_k  for m = k+1 .. Nt-1, 128-row blocks
template <int P>
__device__ __forceinline__ double tile_elem(const double* L, const uint8_t* codes, int64_t e, double inv) {
    if constexpr (P == P_FP64) return __ldcs(L + e);
    else return decode_code(P, codes, e, inv);
}
// one thread's partial dot product over columns [c0, c1) of row `row` of a tile
template <int P>
__device__ __forceinline__ double row_dot(const double* L, const uint8_t* codes, double inv, int64_t nb, int64_t row,
                                          int64_t c0, int64_t c1, const double* sz) {
    // 8 chains, 16 loads in flight per thread (a CTA streams 1 MB: with 8 loads in flight it was
    // latency-bound at ~10 GB/s, which bounded every column's update)
    double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll 2
    for (int64_t c = c0; c < c1; c += 8) {
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] = fma(tile_elem<P>(L, codes, row + (c + q) * nb, inv), sz[c + q], s[q]);
    }
    return ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
}

constexpr int GEMV_T = 512;  // 4 column quarters x 128 rows
__global__ void __launch_bounds__(GEMV_T) k_trsv_gemv(const double* __restrict__ pool, const int32_t* __restrict__ slot,
                                                      int64_t Nt, int64_t nb, int64_t k, int64_t m0, double* r,
                                                      const double* __restrict__ z, TileCodes codes) {
    extern __shared__ double sz[];  // z_k (nb) + GEMV_T partial sums
    double* part = sz + nb;
    const int64_t RB = nb / 128;
    const int64_t m = m0 + blockIdx.x / RB, rb = blockIdx.x % RB;  // tile rows m0, m0+1, ...
    for (int64_t c = threadIdx.x; c < nb; c += blockDim.x) sz[c] = z[k * nb + c];
    __syncthreads();
    const int row = threadIdx.x & 127, h = threadIdx.x >> 7;
    const int64_t t = tile_index(Nt, m, k);
    const double* L = pool + (int64_t)slot[t] * nb * nb;
    const int64_t c0 = h * (nb / 4), c1 = c0 + nb / 4, grow = rb * 128 + row;
    // compact pool: tiles below FP64 are read at their storage precision (fewer bytes)
    const int p = (codes.sto && codes.sto[t] >= 0) ? codes.prec[t] : P_FP64;
    const uint8_t* cp = p != P_FP64 ? codes.shadow + codes.sto[t] : nullptr;
    const double inv = p != P_FP64 ? 1.0 / codes.scale[3 * t + 2] : 1.0;
    double dot;
    switch (p) {
    case P_FP32: dot = row_dot<P_FP32>(L, cp, inv, nb, grow, c0, c1, sz); break;
    case P_FP16: dot = row_dot<P_FP16>(L, cp, inv, nb, grow, c0, c1, sz); break;
    case P_FP8: dot = row_dot<P_FP8>(L, cp, inv, nb, grow, c0, c1, sz); break;
    default: dot = row_dot<P_FP64>(L, cp, inv, nb, grow, c0, c1, sz); break;
    }
    part[threadIdx.x] = dot;
    __syncthreads();
    if (h == 0) r[m * nb + rb * 128 + row] -= (part[row] + part[row + 128]) + (part[row + 256] + part[row + 384]);
}

// z_k = L_kk^-1 r_k: for J = 0..nb/128-1:  s = r_J - L[J, <J] z_<J;  z_J = W_J s
__global__ void __launch_bounds__(256) k_trsv_diag(const double* __restrict__ pool, const int32_t* __restrict__ slot,
                                                   const double* __restrict__ wbuf, int64_t Nt, int64_t nb,
                                                   int64_t k, const double* __restrict__ r, double* z) {
    extern __shared__ double sz[];  // z_k so far (nb) + s (128) + partials (256)
    double* s = sz + nb;
    double* part = s + 128;
    const int row = threadIdx.x & 127, h = threadIdx.x >> 7;
    const double* Lkk = pool + (int64_t)slot[tile_index(Nt, k, k)] * nb * nb;
    const int64_t S = nb / 128;
    for (int64_t J = 0; J < S; ++J) {
        const double* LJ = Lkk + J * 128 + row;
        const int64_t half = J * 64;  // columns [0, 128J) in two halves
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 2
        for (int64_t c = h * half; c < (h + 1) * half; c += 4) {
            a0 = fma(__ldcs(LJ + c * nb), sz[c], a0);
            a1 = fma(__ldcs(LJ + (c + 1) * nb), sz[c + 1], a1);
            a2 = fma(__ldcs(LJ + (c + 2) * nb), sz[c + 2], a2);
            a3 = fma(__ldcs(LJ + (c + 3) * nb), sz[c + 3], a3);
        }
        part[threadIdx.x] = (a0 + a1) + (a2 + a3);
        __syncthreads();
        if (h == 0) s[row] = r[k * nb + J * 128 + row] - (part[row] + part[row + 128]);
        __syncthreads();
        const double* W = wbuf + (k * S + J) * (128 * 128);  // column-major, lower triangular
        double b0 = 0.0;
        const int kk0 = h == 0 ? 0 : (row + 1) / 2, kk1 = h == 0 ? (row + 1) / 2 : row + 1;
        for (int kk = kk0; kk < kk1; ++kk) b0 = fma(W[row + kk * 128], s[kk], b0);
        part[threadIdx.x] = b0;
        __syncthreads();
        if (h == 0) sz[J * 128 + row] = part[row] + part[row + 128];
        __syncthreads();
    }
    for (int64_t c = threadIdx.x; c < nb; c += blockDim.x) z[k * nb + c] = sz[c];
}

// z_k = L_kk^-1 r_k with one CTA per 128-row block J of the tile (the blocks
// run concurrently): CTA J accumulates L[J, I] z_I for I < J as each z_I is
// published (flags[I] == tag, release/acquire), then z_J = W_J (r_J - sum).
// The single-CTA version streamed the whole half tile (~4.5 MB) through one SM
// on the critical path of every column.
__global__ void __launch_bounds__(256) k_trsv_diag_par(const double* __restrict__ pool,
                                                        const int32_t* __restrict__ slot,
                                                        const double* __restrict__ wbuf, int64_t Nt, int64_t nb,
                                                        int64_t k, const double* __restrict__ r, double* z,
                                                        int* flags, int tag) {
    __shared__ double zs[128], sv[128], part[256];
    const int J = blockIdx.x, tid = threadIdx.x, row = tid & 127, h = tid >> 7;
    const int64_t S = nb / 128;
    const double* Lkk = pool + (int64_t)slot[tile_index(Nt, k, k)] * nb * nb;
    const double* LJ = Lkk + J * 128 + row;  // row J*128 + row of the tile, column c at LJ[c * nb]
    double a0 = 0.0, a1 = 0.0;
    for (int I = 0; I < J; ++I) {
        const int64_t c0 = (int64_t)I * 128 + h * 64;
        double l[16];  // (the first loads of this block go out before the wait)
#pragma unroll
        for (int q = 0; q < 16; ++q) l[q] = __ldcs(LJ + (c0 + q) * nb);
        if (tid == 0) {
            int v;
            do {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flags + I) : "memory");
            } while (v != tag);
        }
        __syncthreads();
        if (tid < 128) zs[tid] = __ldcg(z + k * nb + I * 128 + tid);
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 16; q += 2) {
            a0 = fma(l[q], zs[h * 64 + q], a0);
            a1 = fma(l[q + 1], zs[h * 64 + q + 1], a1);
        }
#pragma unroll
        for (int c = 16; c < 64; c += 16) {
            double lv[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) lv[q] = __ldcs(LJ + (c0 + c + q) * nb);
#pragma unroll
            for (int q = 0; q < 16; q += 2) {
                a0 = fma(lv[q], zs[h * 64 + c + q], a0);
                a1 = fma(lv[q + 1], zs[h * 64 + c + q + 1], a1);
            }
        }
        __syncthreads();  // (zs is rewritten for the next block)
    }
    part[tid] = a0 + a1;
    __syncthreads();
    if (h == 0) sv[row] = r[k * nb + J * 128 + row] - (part[row] + part[row + 128]);
    __syncthreads();
    const double* W = wbuf + (k * S + J) * (128 * 128);  // column-major, lower triangular
    // (a fixed trip count with predicated loads, 4 chains: a data-dependent loop bound
    // serialized the 64 loads behind each other on every column's critical path)
    const int kk0 = h == 0 ? 0 : (row + 1) / 2, kk1 = h == 0 ? (row + 1) / 2 : row + 1;
    double bq[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 16
    for (int q = 0; q < 64; ++q) {
        const int kk = kk0 + q;  // <= 127
        const double w = kk < kk1 ? __ldg(W + row + kk * 128) : 0.0;
        bq[q & 3] = fma(w, sv[kk], bq[q & 3]);
    }
    part[tid] = (bq[0] + bq[1]) + (bq[2] + bq[3]);
    __syncthreads();
    if (h == 0) z[k * nb + J * 128 + row] = part[row] + part[row + 128];
    __threadfence();
    __syncthreads();
    if (tid == 0) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flags + J), "r"(tag) : "memory");
}

// out = sum z_i^2 over i < n (fixed-order tree in one CTA)
__global__ void __launch_bounds__(1024) k_sumsq(const double* __restrict__ z, int64_t n, double* out) {
    __shared__ double red[1024];
    double a = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a = fma(z[i], z[i], a);
    red[threadIdx.x] = a;
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

}  // namespace

void launch_forward_solve(const double* pool, const int32_t* slot, const double* wbuf, int64_t Nt, int64_t nb,
                          double* r, double* z, cudaStream_t s, TileCodes codes, int* flags, int seq, cudaStream_t s2,
                          cudaEvent_t* ev) {
    const size_t sm_diag = sizeof(double) * (nb + 128 + 256), sm_gemv = sizeof(double) * (nb + GEMV_T);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_trsv_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        cudaFuncSetAttribute(k_trsv_gemv, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        configured = true;
    }
    const unsigned RB = (unsigned)(nb / 128);
    // Two streams (ev: 2 Nt events, s2 != nullptr): s runs the chain -- diagonal solve of column
    // k, then the update of tile row k+1 by z_k -- and s2 the update of tile rows >= k+2, which
    // thus overlaps the next diagonal solves.  Each r_m still receives its updates in column
    // order: the s2 update by z_k (rows >= k+2) precedes the s update of row k+2 by z_{k+1}
    // (s waits for it), so the result is bitwise that of the one-stream order.
    for (int64_t k = 0; k < Nt; ++k) {
        if (s2 && k >= 2) cudaStreamWaitEvent(s, ev[Nt + k - 2], 0);  // r_k got its z_{k-2} share (s2)
        if (flags) {
            k_trsv_diag_par<<<RB, 256, 0, s>>>(pool, slot, wbuf, Nt, nb, k, r, z, flags, (int)(seq * Nt + k + 1));
        } else {
            MXP_CARVEOUT_MAX(k_trsv_diag);
            k_trsv_diag<<<1, 256, sm_diag, s>>>(pool, slot, wbuf, Nt, nb, k, r, z);
        }
        MXP_CARVEOUT_MAX(k_trsv_gemv);
        if (k + 1 >= Nt) continue;
        if (!s2) {
            k_trsv_gemv<<<(unsigned)(Nt - k - 1) * RB, GEMV_T, sm_gemv, s>>>(pool, slot, Nt, nb, k, k + 1, r, z, codes);
            continue;
        }
        if (k + 2 < Nt) {  // rows >= k+2 on s2, after z_k is final
            cudaEventRecord(ev[k], s);
            cudaStreamWaitEvent(s2, ev[k], 0);
            k_trsv_gemv<<<(unsigned)(Nt - k - 2) * RB, GEMV_T, sm_gemv, s2>>>(pool, slot, Nt, nb, k, k + 2, r, z,
                                                                              codes);
            cudaEventRecord(ev[Nt + k], s2);
        }
        if (k >= 1) cudaStreamWaitEvent(s, ev[Nt + k - 1], 0);  // row k+1's z_{k-1} share came first
        k_trsv_gemv<<<RB, GEMV_T, sm_gemv, s>>>(pool, slot, Nt, nb, k, k + 1, r, z, codes);
    }
    if (s2 && Nt >= 3) cudaStreamWaitEvent(s, ev[Nt + Nt - 3], 0);  // (the last s2 update)
}

void launch_sumsq(const double* z, int64_t n, double* out, cudaStream_t s) {
    MXP_CARVEOUT_MAX(k_sumsq);
    k_sumsq<<<1, 1024, 0, s>>>(z, n, out);
}


// Load every kernel of this file now (CUDA lazy loading would otherwise load a
// kernel at its first launch, which can wait for running kernels -- with ranks
// co-located on one GPU those spin on each other: a deadlock).
void preload_solve() {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void*)k_trsv_diag);
    cudaFuncGetAttributes(&fa, (const void*)k_trsv_diag_par);
    cudaFuncGetAttributes(&fa, (const void*)k_trsv_gemv);
    cudaFuncGetAttributes(&fa, (const void*)k_sumsq);
    cudaGetLastError();
}

}  // namespace mxp
