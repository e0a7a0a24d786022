// kernels_f64.cu -- layout and reduction kernels of the FP64 path (sm_100a):
// pack/unpack between the caller's lda matrix and the tile pool (a1), the
// log-det reduction (a11) and the planner's tile norms (a2).
// The factorization itself lives in sched_f64.cu.
#include <math.h>

#include "dmma_gemm.cuh"
#include "quant.cuh"

namespace mxp {

// ------------------------------------------------------- pack / unpack
// grid: (column-of-tile groups, tile columns j, tile rows i) -- one CTA per
// (tile, 8 columns); rows are contiguous in both layouts -> coalesced.
__global__ void k_pack(const double* __restrict__ A, int64_t lda, int64_t n, double* pool,
                       const int32_t* slot, int64_t Nt, int64_t nb, int64_t col0, int rank, int nranks) {
    const int64_t j = col0 + blockIdx.y;
    const int64_t i = j + blockIdx.z;
    if (i >= Nt || i % nranks != rank) return;  // only this rank's rows (peers push the rest)
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
                         const int32_t* slot, int64_t Nt, int64_t nb, int64_t col0, TileCodes codes) {
    const int64_t j = col0 + blockIdx.y;
    const int64_t i = j + blockIdx.z;
    if (i >= Nt) return;
    const int64_t t = tile_index(Nt, i, j);
    const double* T = pool + (int64_t)slot[t] * nb * nb;
    // compact pool: a tile stored below FP64 is decoded from its storage image
    const bool coded = codes.sto && codes.sto[t] >= 0;
    const uint8_t* cp = coded ? codes.shadow + codes.sto[t] : nullptr;
    const int p = coded ? codes.prec[t] : P_FP64;
    const double inv = coded ? 1.0 / codes.scale[3 * t + 2] : 1.0;
    for (int64_t c = blockIdx.x * 8; c < (int64_t)blockIdx.x * 8 + 8; ++c) {
        int64_t gj = j * nb + c;
        if (gj >= n) return;
        for (int64_t r = threadIdx.x; r < nb; r += blockDim.x) {
            int64_t gi = i * nb + r;
            if (gi < n && gi >= gj) A[gi + gj * lda] = coded ? decode_code(p, cp, r + c * nb, inv) : T[r + c * nb];
        }
    }
}
void launch_pack_f64(const double* A, int64_t lda, int64_t n, double* pool, const int32_t* slot,
                     int64_t Nt, int64_t nb, int64_t col0, int64_t col1, cudaStream_t s, int rank, int nranks) {
    dim3 grid((unsigned)(nb / 8), (unsigned)(col1 - col0), (unsigned)(Nt - col0));
    MXP_CARVEOUT_MAX(k_pack);
    k_pack<<<grid, 256, 0, s>>>(A, lda, n, pool, slot, Nt, nb, col0, rank, nranks);
}
void launch_unpack_f64(double* A, int64_t lda, int64_t n, const double* pool, const int32_t* slot,
                       int64_t Nt, int64_t nb, int64_t col0, int64_t col1, cudaStream_t s, TileCodes codes) {
    dim3 grid((unsigned)(nb / 8), (unsigned)(col1 - col0), (unsigned)(Nt - col0));
    MXP_CARVEOUT_MAX(k_unpack);
    k_unpack<<<grid, 256, 0, s>>>(A, lda, n, pool, slot, Nt, nb, col0, codes);
}

// -------------------------------------------------------------- log-det
// out = 2 * sum_j parts[j] in ascending j; parts[j] = sum of log L_ii
// over the real diagonal of tile j, written by the POTRF of column j.
__global__ void k_logdet_final(const double* parts, int64_t Nt, double* out) {
    double s = 0.0;
    for (int64_t j = 0; j < Nt; ++j) s += parts[j];
    *out = 2.0 * s;
}
void launch_logdet_final(const double* parts, int64_t Nt, double* out, cudaStream_t s) {
    MXP_CARVEOUT_MAX(k_logdet_final);
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
    MXP_CARVEOUT_MAX(k_tile_norms);
    k_tile_norms<<<grid, 256, 0, s>>>(A, lda, n, nb, Nt, norms);
}

// Tile norms of one tile column j from a device copy of the host matrix's panel
// (rows j*nb .. n-1, columns j*nb .. j*nb+nb-1, column-major with ld = ldp): the
// host planner streams A column panel by column panel (a2 with A in host memory).
__global__ void k_panel_norms(const double* __restrict__ P, int64_t ldp, int64_t n, int64_t nb, int64_t Nt,
                              int64_t j, double* norms) {
    __shared__ double red[256];
    const int64_t i = j + blockIdx.x;
    if (i >= Nt) return;
    const int64_t r0 = j * nb;  // global row of the panel's first row
    double s = 0.0;
    for (int64_t c = j * nb; c < (j + 1) * nb && c < n; ++c)
        for (int64_t r = i * nb + threadIdx.x; r < (i + 1) * nb && r < n; r += blockDim.x) {
            double v = (r >= c) ? P[(r - r0) + (c - r0) * ldp] : P[(c - r0) + (r - r0) * ldp];
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
void launch_panel_norms(const double* P, int64_t ldp, int64_t n, int64_t nb, int64_t j, double* norms,
                        cudaStream_t s) {
    const int64_t Nt = (n + nb - 1) / nb;
    MXP_CARVEOUT_MAX(k_panel_norms);
    k_panel_norms<<<(unsigned)(Nt - j), 256, 0, s>>>(P, ldp, n, nb, Nt, j, norms);
}

// Load every kernel of this file now (CUDA lazy loading would otherwise load a
// kernel at its first launch, which can wait for running kernels -- with ranks
// co-located on one GPU those spin on each other: a deadlock).
void preload_layout() {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void*)k_pack);
    cudaFuncGetAttributes(&fa, (const void*)k_unpack);
    cudaFuncGetAttributes(&fa, (const void*)k_logdet_final);
    cudaFuncGetAttributes(&fa, (const void*)k_tile_norms);
    cudaFuncGetAttributes(&fa, (const void*)k_panel_norms);
    cudaGetLastError();
}

}  // namespace mxp
