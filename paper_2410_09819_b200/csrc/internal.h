// internal.h -- shared declarations of the B200 engine (kernels <-> host runtime).
// Not part of the C ABI (see include/mxp_chol.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mxp {

// Tile pool: every lower tile (i,j) of the matrix lives in a pool slot of
// nb*nb elements, column-major inside the tile (ld = nb).  slot_of[t] maps
// the column-major lower-tile index t(i,j) to its slot (in-core: identity).
__host__ __device__ inline int64_t tile_index(int64_t Nt, int64_t i, int64_t j) {
    return j * Nt - j * (j - 1) / 2 + (i - j);
}

// ---- FP64 GEMM-chain update (Alg. 2, the hot loop P:265) -------
// C(m,k)[bi,bj] -= sum_{n in [n0,n1)} A(m,n)[bi,:] * A(k,n)[bj,:]^T for the
// rows m = m0 + y*mstride (y < mcount) of column k; 128x128 CTA blocks.
// nchunks > 1 writes per-chunk partial sums to `partial` (deterministic
// split-K), reduced in chunk order by launch_reduce_partials.
struct ChainArgs {
    double* pool;
    const int32_t* slot;
    const int64_t* dinfo;   // abort flag: kernels exit when *dinfo != 0
    double* partial;
    int64_t Nt, nb;
    int64_t k;              // output column
    int64_t m0, mstride, mcount;
    int64_t n0, n1;         // operand column range
    int64_t nchunks, chunk_tiles;
};
void launch_chain_f64(const ChainArgs& a, cudaStream_t s);
void launch_reduce_partials(const ChainArgs& a, cudaStream_t s);

// ---- diagonal-tile POTRF (Alg. 2), right-looking on 128 blocks
struct PotrfArgs {
    double* pool;
    const int32_t* slot;
    int64_t* dinfo;
    int64_t Nt, nb, k;
};
// Runs the whole in-tile sequence (base POTRF, in-tile TRSM, trailing update
// per 128-block); returns the number of kernels launched.
int launch_potrf_tile_f64(const PotrfArgs& a, cudaStream_t s);

// ---- TRSM of the tiles below the diagonal (Alg. 2, G3) --------
// X L_kk^T = C for the rows m = m0 + y*mstride of column k, in place.
struct TrsmArgs {
    double* pool;
    const int32_t* slot;
    const int64_t* dinfo;
    int64_t Nt, nb, k;
    int64_t m0, mstride, mcount;
};
void launch_trsm_f64(const TrsmArgs& a, cudaStream_t s);

// ---- layout / utility kernels --------------------------------------------
// lda matrix <-> pool tiles (padding: zeros, 1 on the padded diagonal)
void launch_pack_f64(const double* A, int64_t lda, int64_t n, double* pool, const int32_t* slot,
                     int64_t Nt, int64_t nb, int64_t col0, int64_t col1, cudaStream_t s);
void launch_unpack_f64(double* A, int64_t lda, int64_t n, const double* pool, const int32_t* slot,
                       int64_t Nt, int64_t nb, int64_t col0, int64_t col1, cudaStream_t s);
// logdet = 2 sum_{i<n} log L_ii, fixed reduction order (deterministic)
void launch_logdet(const double* pool, const int32_t* slot, int64_t Nt, int64_t nb, int64_t n,
                   double* parts, double* out, cudaStream_t s);
// planner: per-tile Frobenius norms (fp64) of the lower tiles of an lda matrix
void launch_tile_norms(const double* A, int64_t lda, int64_t n, int64_t nb, double* norms,
                       cudaStream_t s);

// Shared-memory bytes the kernels request (for attribute setup).
void configure_kernels();

}  // namespace mxp
