// dmma_gemm.cuh -- FP64 DMMA GEMM building blocks for sm_100a (B200).
//
// FP64 has no tcgen05 kind: dense FP64 contractions run on the FP64
// tensor pipe through warp-level DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4).
// Operands are staged global->shared with cp.async.cg (LDGSTS, L2-coherent) in
// a multi-stage pipeline; accumulators stay in registers.
#pragma once
#include <stdint.h>

#include "internal.h"

namespace mxp {

// ------------------------------------------------------------------ helpers
// CTA-internal barrier of the NT "worker" threads 0..NT-1 (named barrier 1).
// The task bodies shared by k_sched (128 threads) and the tensor-core kernel
// k_tc (128 workers + 2 tcgen05 producer / MMA warps that skip non-GEMM
// tasks) synchronize with it instead of __syncthreads; with NT = blockDim.x
// it is the same as __syncthreads.
template <int NT>
__device__ __forceinline__ void sync_nt() {
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}
__device__ __forceinline__ void sync_workers() { sync_nt<128>(); }
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

constexpr int BK = 16;
constexpr int PAD = 4;  // doubles; makes the 4 k-rows of a fragment hit distinct banks

// DMMA GEMM tile configuration.  Swept on B200 (tools/dmma_bench.cu,
// profiles/): 64x128 CTA tiles, 4 warps of 32x64, 3-stage cp.async, 3 CTAs
// per SM reaches 34.6 TF/s (cuBLAS DGEMM 36.2); the 1-CTA/SM 128x128 tile
// reached 31.0.
template <int BM_, int BN_, int WARPS_M_, int WARPS_N_, int STAGES_>
struct GemmCfg {
    static constexpr int BM = BM_, BN = BN_, WARPS_M = WARPS_M_, WARPS_N = WARPS_N_, STAGES = STAGES_;
    static constexpr int NT = 32 * WARPS_M * WARPS_N;
    static constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
    static constexpr int MI = WTM / 8, NI = WTN / 8;
    static constexpr int LDA_S = BM + PAD, LDB_S = BN + PAD;
    static constexpr int STAGE_DOUBLES = BK * (LDA_S + LDB_S);
    static constexpr int SMEM_BYTES = STAGES * STAGE_DOUBLES * 8;
    static constexpr int A_COPIES = BK * BM / 2 / NT;  // 16B copies per thread
    static constexpr int B_COPIES = BK * BN / 2 / NT;
};
using CC = GemmCfg<64, 128, 2, 2, 3>;   // chain / trailing update: 128 threads, 3 CTAs/SM
using PC = GemmCfg<128, 128, 2, 4, 3>;  // single-CTA POTRF kernel: 256 threads

// Operand source: for K-chunk `it` (BK columns), the address of element
// (row0, kcol) of the A and B panels; both column-major with ld.
// `src` is a functor: src(it, &pa, &pb).
struct NoPost {
    static constexpr bool active = false;
    __device__ void operator()(int, double*, double*) const {}
};

// `post(it, sA, sB)` (if Post::active) transforms stage `it` in shared memory
// after it has landed and before it is consumed (used for on-the-fly casts).
template <class C, class Src, class Post = NoPost>
__device__ __forceinline__ void gemm_mainloop(double (&acc)[C::MI][C::NI][2], const Src& src, int64_t lda,
                                              int64_t ldb, int nk, double* smem, const Post& post = Post()) {
    constexpr int BM = C::BM, BN = C::BN, STAGES = C::STAGES, NT = C::NT;
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
            int c = t + i * NT;
            int col = c / (BM / 2), r2 = (c % (BM / 2)) * 2;
            cp_async16(sA + col * C::LDA_S + r2, pa + col * lda + r2);
        }
#pragma unroll
        for (int i = 0; i < C::B_COPIES; ++i) {
            int c = t + i * NT;
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
        sync_nt<NT>();
        int nxt = it + STAGES - 1;
        if (nxt < nk) load_stage(nxt % STAGES, nxt);
        cp_async_commit();
        if constexpr (Post::active) {
            double* wA = smem + (it % STAGES) * C::STAGE_DOUBLES;
            post(it, wA, wA + BK * C::LDA_S);
            sync_nt<NT>();
        }
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
    sync_nt<NT>();
}

// Element (row, col) of the CTA block owned by fragment (mi, ni, i) of this thread.
template <class C>
__device__ __forceinline__ void frag_pos(int mi, int ni, int i, int& row, int& col) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int wm = warp / C::WARPS_N, wn = warp % C::WARPS_N;
    row = wm * C::WTM + mi * 8 + (lane >> 2);
    col = wn * C::WTN + ni * 8 + (lane & 3) * 2 + i;
}

__device__ __forceinline__ double* tile_ptr(double* pool, const int32_t* slot, int64_t Nt, int64_t nb,
                                            int64_t i, int64_t j) {
    return pool + (int64_t)slot[tile_index(Nt, i, j)] * nb * nb;
}


// ---- memory-model helpers for the device-side Ready table ----
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_add_release(int* p, int v) {
    int old;
    asm volatile("atom.add.release.gpu.global.s32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned s;
    asm volatile("mov.u32 %0, %smid;" : "=r"(s));
    return s;
}

}  // namespace mxp
