// kernels_f64.cu -- FP64 tile kernels for sm_100a (B200).
//
// FP64 has no tcgen05 kind: the dense contractions run on the
// FP64 tensor pipe through warp-level DMMA (mma.sync.m8n8k4.f64 -> SASS
// DMMA.8x8x4), operands staged global->shared with cp.async (LDGSTS) in a
// 4-stage pipeline, accumulators in registers (the V1 "accumulator stays
// resident" idea, held on-chip for the whole n-chain).
//
// Kernels (Alg. 2):
//   k_chain   GEMM/SYRK chain  C(m,k) -= sum_n A(m,n) A(k,n)^T      (a6/a7)
//   k_reduce  ordered reduction of split-K partials (deterministic)
//   k_potrf128 unblocked Cholesky of one 128x128 block in shared memory
//   k_trsm    X L^T = C, 64-row blocks, blocked forward substitution (G3)
//   k_trail   in-tile trailing update for the diagonal tile's POTRF
//   k_pack / k_unpack / k_logdet / k_tile_norms
#include <math.h>

#include "internal.h"

namespace mxp {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
// D(8x8) += A(8x4, row) * B(4x8, col); lane l holds A[l/4][l%4], B[l%4][l/4],
// D[l/4][2*(l%4)+{0,1}]  (PTX ISA, mma.m8n8k4 .f64 fragments).
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

constexpr int THREADS = 256;
constexpr int BK = 16;
constexpr int STAGES = 4;
constexpr int PAD = 4;  // doubles; makes the 4 k-rows of a fragment hit distinct banks

template <int BM, int BN>
struct GemmCfg {
    static constexpr int WARPS_M = 2, WARPS_N = 4;
    static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
    static constexpr int MI = WTM / 8, NI = WTN / 8;
    static constexpr int LDA_S = BM + PAD, LDB_S = BN + PAD;
    static constexpr int STAGE_DOUBLES = BK * (LDA_S + LDB_S);
    static constexpr int SMEM_BYTES = STAGES * STAGE_DOUBLES * 8;
    static constexpr int A_COPIES = BK * BM / 2 / THREADS;  // 16B copies per thread
    static constexpr int B_COPIES = BK * BN / 2 / THREADS;
};

// Operand source: for K-chunk `it` (BK columns), the address of element
// (row0, kcol) of the A and B panels; both column-major with ld.
// `src` is a functor: src(it, &pa, &pb).
template <int BM, int BN, class Src>
__device__ __forceinline__ void gemm_mainloop(double (&acc)[GemmCfg<BM, BN>::MI][GemmCfg<BM, BN>::NI][2],
                                              const Src& src, int64_t lda, int64_t ldb, int nk,
                                              double* smem) {
    using C = GemmCfg<BM, BN>;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
    const int g = lane >> 2, q = lane & 3;

    auto load_stage = [&](int stage, int it) {
        const double* pa;
        const double* pb;
        src(it, pa, pb);
        double* sA = smem + stage * C::STAGE_DOUBLES;
        double* sB = sA + BK * C::LDA_S;
#pragma unroll
        for (int i = 0; i < C::A_COPIES; ++i) {
            int c = t + i * THREADS;
            int col = c / (BM / 2), r2 = (c % (BM / 2)) * 2;
            cp_async16(sA + col * C::LDA_S + r2, pa + col * lda + r2);
        }
#pragma unroll
        for (int i = 0; i < C::B_COPIES; ++i) {
            int c = t + i * THREADS;
            int col = c / (BN / 2), r2 = (c % (BN / 2)) * 2;
            cp_async16(sB + col * C::LDB_S + r2, pb + col * ldb + r2);
        }
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) load_stage(s, s);
        cp_async_commit();
    }
    for (int it = 0; it < nk; ++it) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        int nxt = it + STAGES - 1;
        if (nxt < nk) load_stage(nxt % STAGES, nxt);
        cp_async_commit();
        const double* sA = smem + (it % STAGES) * C::STAGE_DOUBLES;
        const double* sB = sA + BK * C::LDA_S;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a[C::MI], b[C::NI];
            const double* pa = sA + (kk + q) * C::LDA_S + wm * C::WTM + g;
            const double* pb = sB + (kk + q) * C::LDB_S + wn * C::WTN + g;
#pragma unroll
            for (int mi = 0; mi < C::MI; ++mi) a[mi] = pa[mi * 8];
#pragma unroll
            for (int ni = 0; ni < C::NI; ++ni) b[ni] = pb[ni * 8];
#pragma unroll
            for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
                for (int ni = 0; ni < C::NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
        }
    }
    cp_async_wait<0>();
    __syncthreads();
}

// Element (row, col) of the CTA block owned by fragment (mi, ni, i) of this thread.
template <int BM, int BN>
__device__ __forceinline__ void frag_pos(int mi, int ni, int i, int& row, int& col) {
    using C = GemmCfg<BM, BN>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
    row = wm * C::WTM + mi * 8 + (lane >> 2);
    col = wn * C::WTN + ni * 8 + (lane & 3) * 2 + i;
}

__device__ __forceinline__ double* tile_ptr(double* pool, const int32_t* slot, int64_t Nt, int64_t nb,
                                            int64_t i, int64_t j) {
    return pool + (int64_t)slot[tile_index(Nt, i, j)] * nb * nb;
}

// ------------------------------------------------------------ GEMM chain
using CC = GemmCfg<128, 128>;

__global__ void __launch_bounds__(THREADS, 1) k_chain(ChainArgs a) {
    if (*a.dinfo != 0) return;
    extern __shared__ __align__(16) double smem[];
    const int64_t S = a.nb / 128;
    const int64_t bi = blockIdx.x % S, bj = blockIdx.x / S;
    const int64_t m = a.m0 + (int64_t)blockIdx.y * a.mstride;
    if (m == a.k && bi < bj) return;  // strict upper blocks of the diagonal tile: unused
    const int64_t chunk = blockIdx.z;
    const int64_t nbeg = a.n0 + chunk * a.chunk_tiles;
    int64_t nend = nbeg + a.chunk_tiles;
    if (nend > a.n1) nend = a.n1;
    if (nbeg >= nend) return;
    const int64_t kper = a.nb / BK;
    const int nk = (int)((nend - nbeg) * kper);
    double* pool = a.pool;
    const int32_t* slot = a.slot;
    const int64_t Nt = a.Nt, nb = a.nb, kc = a.k;
    auto src = [&](int it, const double*& pa, const double*& pb) {
        int64_t n = nbeg + it / kper;
        int64_t kcol = (it % kper) * BK;
        pa = tile_ptr(pool, slot, Nt, nb, m, n) + bi * 128 + kcol * nb;
        pb = tile_ptr(pool, slot, Nt, nb, kc, n) + bj * 128 + kcol * nb;
    };
    double acc[CC::MI][CC::NI][2];
#pragma unroll
    for (int mi = 0; mi < CC::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < CC::NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    gemm_mainloop<128, 128>(acc, src, nb, nb, nk, smem);

    if (a.nchunks == 1) {
        double* Ct = tile_ptr(pool, slot, Nt, nb, m, kc) + bi * 128 + bj * 128 * nb;
#pragma unroll
        for (int mi = 0; mi < CC::MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < CC::NI; ++ni)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    int r, c;
                    frag_pos<128, 128>(mi, ni, i, r, c);
                    double* p = Ct + r + (int64_t)c * nb;
                    *p = *p - acc[mi][ni][i];
                }
    } else {
        // partial layout: [item][chunk][e][thread], item = y*S*S + x
        int64_t item = (int64_t)blockIdx.y * S * S + blockIdx.x;
        double* P = a.partial + (item * a.nchunks + chunk) * (128 * 128);
        int e = 0;
#pragma unroll
        for (int mi = 0; mi < CC::MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < CC::NI; ++ni)
#pragma unroll
                for (int i = 0; i < 2; ++i, ++e) P[e * THREADS + threadIdx.x] = acc[mi][ni][i];
    }
}

__global__ void __launch_bounds__(THREADS) k_reduce(ChainArgs a) {
    if (*a.dinfo != 0) return;
    const int64_t S = a.nb / 128;
    const int64_t bi = blockIdx.x % S, bj = blockIdx.x / S;
    const int64_t m = a.m0 + (int64_t)blockIdx.y * a.mstride;
    if (m == a.k && bi < bj) return;
    int64_t item = (int64_t)blockIdx.y * S * S + blockIdx.x;
    const double* P = a.partial + item * a.nchunks * (128 * 128);
    double* Ct = tile_ptr(a.pool, a.slot, a.Nt, a.nb, m, a.k) + bi * 128 + bj * 128 * a.nb;
    // number of chunks that actually hold data (trailing chunks may be empty)
    int64_t nvalid = (a.n1 - a.n0 + a.chunk_tiles - 1) / a.chunk_tiles;
    int e = 0;
    for (int mi = 0; mi < CC::MI; ++mi)
        for (int ni = 0; ni < CC::NI; ++ni)
            for (int i = 0; i < 2; ++i, ++e) {
                double s = 0.0;
                for (int64_t c = 0; c < nvalid; ++c) s += P[c * (128 * 128) + e * THREADS + threadIdx.x];
                int r, cc;
                frag_pos<128, 128>(mi, ni, i, r, cc);
                double* p = Ct + r + (int64_t)cc * a.nb;
                *p = *p - s;
            }
}

void launch_chain_f64(const ChainArgs& a, cudaStream_t s) {
    int64_t S = a.nb / 128;
    dim3 grid((unsigned)(S * S), (unsigned)a.mcount, (unsigned)a.nchunks);
    k_chain<<<grid, THREADS, CC::SMEM_BYTES, s>>>(a);
}
void launch_reduce_partials(const ChainArgs& a, cudaStream_t s) {
    int64_t S = a.nb / 128;
    dim3 grid((unsigned)(S * S), (unsigned)a.mcount, 1);
    k_reduce<<<grid, THREADS, 0, s>>>(a);
}

// ------------------------------------------------- POTRF of a 128 block
// Unblocked right-looking Cholesky (kij order) of the 128x128 block
// D[J,J] of the diagonal tile, entirely in shared memory (128 KB).
__global__ void __launch_bounds__(THREADS) k_potrf128(PotrfArgs a, int J) {
    if (*a.dinfo != 0) return;
    extern __shared__ __align__(16) double sm[];
    __shared__ int fail;
    const int t = threadIdx.x;
    const int64_t nb = a.nb;
    double* D = tile_ptr(a.pool, a.slot, a.Nt, nb, a.k, a.k) + (int64_t)J * 128 + (int64_t)J * 128 * nb;
    for (int idx = t; idx < 128 * 128; idx += THREADS) {
        int c = idx >> 7, r = idx & 127;
        sm[idx] = D[r + (int64_t)c * nb];
    }
    if (t == 0) fail = 0;
    __syncthreads();
    for (int j = 0; j < 128; ++j) {
        if (t == 0) {
            double d = sm[j * 129];
            if (!(d > 0.0)) {
                fail = 1;
                *a.dinfo = a.k * nb + (int64_t)J * 128 + j + 1;
            } else {
                sm[j * 129] = sqrt(d);
            }
        }
        __syncthreads();
        if (fail) return;
        if (t > j && t < 128) sm[j * 128 + t] = sm[j * 128 + t] / sm[j * 129];
        __syncthreads();
        const int w = 127 - j;
        for (int idx = t; idx < w * w; idx += THREADS) {
            int c = j + 1 + idx / w, r = j + 1 + idx % w;
            if (r >= c) sm[c * 128 + r] -= sm[j * 128 + r] * sm[j * 128 + c];
        }
        __syncthreads();
    }
    for (int idx = t; idx < 128 * 128; idx += THREADS) {
        int c = idx >> 7, r = idx & 127;
        D[r + (int64_t)c * nb] = (r >= c) ? sm[idx] : 0.0;
    }
}

// ------------------------------------------------------------------- TRSM
// X L^T = C with L lower (nb x nb, the diagonal tile), X/C the rows
// [r0, r0+64) of a tile, both ld = nb.  Blocked by 128 columns J:
//   T = C[:, J] - X[:, J0*128 : J*128] L[J, J0*128 : J*128]^T   (DMMA)
//   T L_JJ^T = (that)   by column-wise forward substitution in smem
// In place: a CTA only touches its own 64 rows.
using TC = GemmCfg<64, 128>;
constexpr int TRSM_T_DOUBLES = 64 * 128;
constexpr int TRSM_SMEM = (TRSM_T_DOUBLES + (STAGES * TC::STAGE_DOUBLES > 128 * 128
                                                 ? STAGES * TC::STAGE_DOUBLES
                                                 : 128 * 128)) * 8;

__device__ void trsm_rows(double* X, const double* L, int64_t nb, int J0, int J1, double* sm) {
    double* T = sm;                    // [128 cols][64 rows]
    double* R = sm + TRSM_T_DOUBLES;   // mainloop stages, then L_JJ (col-major 128x128)
    const int t = threadIdx.x;
    for (int J = J0; J < J1; ++J) {
        double acc[TC::MI][TC::NI][2];
#pragma unroll
        for (int mi = 0; mi < TC::MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < TC::NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        int nk = (J - J0) * 128 / BK;
        if (nk > 0) {
            const int64_t kbase = (int64_t)J0 * 128;
            auto src = [&](int it, const double*& pa, const double*& pb) {
                int64_t kcol = kbase + (int64_t)it * BK;
                pa = X + kcol * nb;
                pb = L + (int64_t)J * 128 + kcol * nb;
            };
            gemm_mainloop<64, 128>(acc, src, nb, nb, nk, R);
        }
        // T = C[:, J] - acc
#pragma unroll
        for (int mi = 0; mi < TC::MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < TC::NI; ++ni)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    int r, c;
                    frag_pos<64, 128>(mi, ni, i, r, c);
                    T[c * 64 + r] = X[r + ((int64_t)J * 128 + c) * nb] - acc[mi][ni][i];
                }
        const double* Ljj = L + (int64_t)J * 128 + (int64_t)J * 128 * nb;
        for (int idx = t; idx < 128 * 128; idx += THREADS) {
            int c = idx >> 7, r = idx & 127;
            R[idx] = Ljj[r + (int64_t)c * nb];
        }
        __syncthreads();
        for (int j = 0; j < 128; ++j) {
            if (t < 64) T[j * 64 + t] = T[j * 64 + t] / R[j * 129];
            __syncthreads();
            const int w = 127 - j;
            for (int idx = t; idx < w * 64; idx += THREADS) {
                int c = j + 1 + (idx >> 6), r = idx & 63;
                T[c * 64 + r] -= T[j * 64 + r] * R[c + j * 128];
            }
            __syncthreads();
        }
        for (int idx = t; idx < 64 * 128; idx += THREADS) {
            int c = idx >> 6, r = idx & 63;
            X[r + ((int64_t)J * 128 + c) * nb] = T[idx];
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(THREADS, 1) k_trsm(TrsmArgs a) {
    if (*a.dinfo != 0) return;
    extern __shared__ __align__(16) double sm[];
    const int64_t m = a.m0 + (int64_t)blockIdx.y * a.mstride;
    double* X = tile_ptr(a.pool, a.slot, a.Nt, a.nb, m, a.k) + (int64_t)blockIdx.x * 64;
    const double* L = tile_ptr(a.pool, a.slot, a.Nt, a.nb, a.k, a.k);
    trsm_rows(X, L, a.nb, 0, (int)(a.nb / 128), sm);
}

// in-tile TRSM for the diagonal tile's POTRF: rows below block J, single J step
__global__ void __launch_bounds__(THREADS, 1) k_trsm_intile(PotrfArgs a, int J) {
    if (*a.dinfo != 0) return;
    extern __shared__ __align__(16) double sm[];
    double* D = tile_ptr(a.pool, a.slot, a.Nt, a.nb, a.k, a.k);
    double* X = D + (int64_t)(J + 1) * 128 + (int64_t)blockIdx.x * 64;
    trsm_rows(X, D, a.nb, J, J + 1, sm);
}

// in-tile trailing update: D[I,J'] -= D[I,J] D[J',J]^T, J < J' <= I < S
__global__ void __launch_bounds__(THREADS, 1) k_trail(PotrfArgs a, int J) {
    if (*a.dinfo != 0) return;
    extern __shared__ __align__(16) double smem[];
    const int S = (int)(a.nb / 128);
    int idx = blockIdx.x, Jp = J + 1, I = 0;
    // enumerate pairs column-major: Jp = J+1.., I = Jp..S-1
    while (true) {
        int cnt = S - Jp;
        if (idx < cnt) { I = Jp + idx; break; }
        idx -= cnt;
        ++Jp;
    }
    const int64_t nb = a.nb;
    double* D = tile_ptr(a.pool, a.slot, a.Nt, nb, a.k, a.k);
    const double* Ab = D + (int64_t)I * 128 + (int64_t)J * 128 * nb;
    const double* Bb = D + (int64_t)Jp * 128 + (int64_t)J * 128 * nb;
    auto src = [&](int it, const double*& pa, const double*& pb) {
        pa = Ab + (int64_t)it * BK * nb;
        pb = Bb + (int64_t)it * BK * nb;
    };
    double acc[CC::MI][CC::NI][2];
#pragma unroll
    for (int mi = 0; mi < CC::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < CC::NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    gemm_mainloop<128, 128>(acc, src, nb, nb, 128 / BK, smem);
    double* Ct = D + (int64_t)I * 128 + (int64_t)Jp * 128 * nb;
#pragma unroll
    for (int mi = 0; mi < CC::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < CC::NI; ++ni)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                int r, c;
                frag_pos<128, 128>(mi, ni, i, r, c);
                double* p = Ct + r + (int64_t)c * nb;
                *p = *p - acc[mi][ni][i];
            }
}

void launch_trsm_f64(const TrsmArgs& a, cudaStream_t s) {
    dim3 grid((unsigned)(a.nb / 64), (unsigned)a.mcount, 1);
    k_trsm<<<grid, THREADS, TRSM_SMEM, s>>>(a);
}

int launch_potrf_tile_f64(const PotrfArgs& a, cudaStream_t s) {
    const int S = (int)(a.nb / 128);
    int launches = 0;
    for (int J = 0; J < S; ++J) {
        k_potrf128<<<1, THREADS, 128 * 128 * 8, s>>>(a, J);
        ++launches;
        if (J + 1 < S) {
            k_trsm_intile<<<(unsigned)((S - J - 1) * 2), THREADS, TRSM_SMEM, s>>>(a, J);
            int pairs = (S - J - 1) * (S - J) / 2;
            k_trail<<<(unsigned)pairs, THREADS, CC::SMEM_BYTES, s>>>(a, J);
            launches += 2;
        }
    }
    return launches;
}

// ------------------------------------------------------- pack / unpack
// grid: (column-of-tile groups, tile columns j, tile rows i) -- one CTA per
// (tile, 8 columns); rows are contiguous in both layouts -> coalesced.
__global__ void k_pack(const double* __restrict__ A, int64_t lda, int64_t n, double* pool,
                       const int32_t* slot, int64_t Nt, int64_t nb, int64_t col0) {
    const int64_t j = col0 + blockIdx.y;
    const int64_t i = j + blockIdx.z;
    if (i >= Nt) return;
    double* T = pool + (int64_t)slot[tile_index(Nt, i, j)] * nb * nb;
    for (int64_t c = blockIdx.x * 8; c < (int64_t)blockIdx.x * 8 + 8; ++c) {
        int64_t gj = j * nb + c;
        for (int64_t r = threadIdx.x; r < nb; r += blockDim.x) {
            int64_t gi = i * nb + r;
            double v;
            if (gi < n && gj < n) v = (gi >= gj) ? A[gi + gj * lda] : 0.0;
            else v = (gi == gj) ? 1.0 : 0.0;
            T[r + c * nb] = v;
        }
    }
}
__global__ void k_unpack(double* __restrict__ A, int64_t lda, int64_t n, const double* pool,
                         const int32_t* slot, int64_t Nt, int64_t nb, int64_t col0) {
    const int64_t j = col0 + blockIdx.y;
    const int64_t i = j + blockIdx.z;
    if (i >= Nt) return;
    const double* T = pool + (int64_t)slot[tile_index(Nt, i, j)] * nb * nb;
    for (int64_t c = blockIdx.x * 8; c < (int64_t)blockIdx.x * 8 + 8; ++c) {
        int64_t gj = j * nb + c;
        if (gj >= n) return;
        for (int64_t r = threadIdx.x; r < nb; r += blockDim.x) {
            int64_t gi = i * nb + r;
            if (gi < n && gi >= gj) A[gi + gj * lda] = T[r + c * nb];
        }
    }
}
void launch_pack_f64(const double* A, int64_t lda, int64_t n, double* pool, const int32_t* slot,
                     int64_t Nt, int64_t nb, int64_t col0, int64_t col1, cudaStream_t s) {
    dim3 grid((unsigned)(nb / 8), (unsigned)(col1 - col0), (unsigned)(Nt - col0));
    k_pack<<<grid, 256, 0, s>>>(A, lda, n, pool, slot, Nt, nb, col0);
}
void launch_unpack_f64(double* A, int64_t lda, int64_t n, const double* pool, const int32_t* slot,
                       int64_t Nt, int64_t nb, int64_t col0, int64_t col1, cudaStream_t s) {
    dim3 grid((unsigned)(nb / 8), (unsigned)(col1 - col0), (unsigned)(Nt - col0));
    k_unpack<<<grid, 256, 0, s>>>(A, lda, n, pool, slot, Nt, nb, col0);
}

// -------------------------------------------------------------- log-det
// parts[j] = sum over the real diagonal entries of tile j of log L_ii (fixed
// tree order); out = 2 * sum_j parts[j] in ascending j.
__global__ void k_logdet_parts(const double* pool, const int32_t* slot, int64_t Nt, int64_t nb,
                               int64_t n, double* parts) {
    __shared__ double red[256];
    const int64_t j = blockIdx.x;
    const double* T = pool + (int64_t)slot[tile_index(Nt, j, j)] * nb * nb;
    double s = 0.0;
    for (int64_t r = threadIdx.x; r < nb; r += blockDim.x)
        if (j * nb + r < n) s += log(T[r + r * nb]);
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) parts[j] = red[0];
}
__global__ void k_logdet_final(const double* parts, int64_t Nt, double* out) {
    double s = 0.0;
    for (int64_t j = 0; j < Nt; ++j) s += parts[j];
    *out = 2.0 * s;
}
void launch_logdet(const double* pool, const int32_t* slot, int64_t Nt, int64_t nb, int64_t n,
                   double* parts, double* out, cudaStream_t s) {
    k_logdet_parts<<<(unsigned)Nt, 256, 0, s>>>(pool, slot, Nt, nb, n, parts);
    k_logdet_final<<<1, 1, 0, s>>>(parts, Nt, out);
}

// ----------------------------------------------------------- tile norms
// One CTA per lower tile; fp64 sum of squares over the real entries, fixed
// reduction order.  (Planner a2 / P:335.)
__global__ void k_tile_norms(const double* __restrict__ A, int64_t lda, int64_t n, int64_t nb,
                             int64_t Nt, double* norms) {
    __shared__ double red[256];
    const int64_t j = blockIdx.y;
    const int64_t i = j + blockIdx.x;
    if (i >= Nt) return;
    double s = 0.0;
    for (int64_t c = j * nb; c < (j + 1) * nb && c < n; ++c)
        for (int64_t r = i * nb + threadIdx.x; r < (i + 1) * nb && r < n; r += blockDim.x) {
            double v = (r >= c) ? A[r + c * lda] : A[c + r * lda];
            s += v * v;
        }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) norms[tile_index(Nt, i, j)] = sqrt(red[0]);
}
void launch_tile_norms(const double* A, int64_t lda, int64_t n, int64_t nb, double* norms, cudaStream_t s) {
    int64_t Nt = (n + nb - 1) / nb;
    dim3 grid((unsigned)Nt, (unsigned)Nt, 1);
    k_tile_norms<<<grid, 256, 0, s>>>(A, lda, n, nb, Nt, norms);
}

void configure_kernels() {
    static bool done = false;
    if (done) return;
    cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM_BYTES);
    cudaFuncSetAttribute(k_trail, cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM_BYTES);
    cudaFuncSetAttribute(k_potrf128, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 128 * 8);
    cudaFuncSetAttribute(k_trsm, cudaFuncAttributeMaxDynamicSharedMemorySize, TRSM_SMEM);
    cudaFuncSetAttribute(k_trsm_intile, cudaFuncAttributeMaxDynamicSharedMemorySize, TRSM_SMEM);
    done = true;
}

}  // namespace mxp
