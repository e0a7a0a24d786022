// tc_block.cuh -- one 128x128 output block on tcgen05 (TF32 kind), used by the
// static-schedule kernel for GEMM tasks of tiles stored below FP64.
//
//   C(128x128, fp64, ldc) -= sum_k cast(A)[:, k] cast(B)[:, k]^T
//
// The K walk comes in 16-wide chunks from `src(step)` (operand pointers into
// column-major fp64 tiles + the cast to apply).  Each chunk is staged by all
// 128 threads (LDG -> cast_c -> fp32 [-> hi/lo] -> swizzled STS), then one
// thread issues the tcgen05.mma's for it and commits them to an mbarrier;
// two smem buffers alternate so staging of chunk s+1 overlaps the MMAs of
// chunk s.  THREE = 3xTF32 (FP32 compute: hi*hi + hi*lo + lo*hi), else 1xTF32
// (FP16 / E4M3 values are exact in TF32).
#pragma once
#include "quant.cuh"
#include "tc_tf32.cuh"

namespace mxp {
namespace tc {

constexpr int BUF_BYTES = 4 * SUB_BYTES;           // Ahi | Alo | Bhi | Blo  (32 KB)
constexpr int SMEM_BYTES = 1024 + 2 * BUF_BYTES;   // + alignment slack

struct Chunk {
    const double* a;  // element (row 0, k0) of A, column-major, lda
    const double* b;  // element (row 0, k0) of B, column-major, ldb
    Cast ca, cb;
};

// thread t stages 4 consecutive MN rows (t & 31)*4 .. +3 of columns (t >> 5) + 4j
__device__ __forceinline__ void load_chunk(const Chunk& ch, int64_t lda, int64_t ldb, double2 (&ra)[8],
                                           double2 (&rb)[8]) {
    const int t = threadIdx.x, mn = (t & 31) * 4, k0 = t >> 5;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const double* pa = ch.a + mn + (int64_t)(k0 + 4 * j) * lda;
        const double* pb = ch.b + mn + (int64_t)(k0 + 4 * j) * ldb;
        ra[2 * j] = __ldcg(reinterpret_cast<const double2*>(pa));
        ra[2 * j + 1] = __ldcg(reinterpret_cast<const double2*>(pa + 2));
        rb[2 * j] = __ldcg(reinterpret_cast<const double2*>(pb));
        rb[2 * j + 1] = __ldcg(reinterpret_cast<const double2*>(pb + 2));
    }
}

template <bool THREE>
__device__ __forceinline__ void store_operand(const Cast& c, const double2 (&r)[8], uint8_t* hi_buf,
                                              uint8_t* lo_buf) {
    const int t = threadIdx.x, mn = (t & 31) * 4, k0 = t >> 5;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        float x[4] = {(float)apply_cast(c, r[2 * j].x), (float)apply_cast(c, r[2 * j].y),
                      (float)apply_cast(c, r[2 * j + 1].x), (float)apply_cast(c, r[2 * j + 1].y)};
        const uint32_t off = sw_offset(mn, k0 + 4 * j);
        if (THREE) {
            float h[4], l[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) split_tf32(x[e], h[e], l[e]);
            *reinterpret_cast<float4*>(hi_buf + off) = make_float4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<float4*>(lo_buf + off) = make_float4(l[0], l[1], l[2], l[3]);
        } else {
            *reinterpret_cast<float4*>(hi_buf + off) = make_float4(x[0], x[1], x[2], x[3]);
        }
    }
}

// smem: >= SMEM_BYTES of dynamic shared memory (any 16-B aligned base);
// mbar: two 8-byte mbarriers in shared memory NOT inside smem's used range;
// tmem: this CTA's TMEM accumulator (>= 128 columns).  All 128 threads call.
template <bool THREE, class Src>
__device__ void block_gemm(double* C, int64_t ldc, const Src& src, int nsteps, int64_t lda, int64_t ldb,
                           uint8_t* smem, uint64_t* mbar, uint32_t tmem) {
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
    if (threadIdx.x == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    double2 ra[8], rb[8];
    Chunk ch = src(0);
    load_chunk(ch, lda, ldb, ra, rb);
    for (int s = 0; s < nsteps; ++s) {
        const int buf = s & 1;
        uint8_t* B0 = base + buf * BUF_BYTES;
        if (s >= 2) mbar_wait(&mbar[buf], ((s - 2) >> 1) & 1);  // MMAs of step s-2 released this buffer
        store_operand<THREE>(ch.ca, ra, B0, B0 + SUB_BYTES);
        store_operand<THREE>(ch.cb, rb, B0 + 2 * SUB_BYTES, B0 + 3 * SUB_BYTES);
        if (s + 1 < nsteps) {
            ch = src(s + 1);
            load_chunk(ch, lda, ldb, ra, rb);  // in flight while step s computes
        }
        fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
        __syncthreads();
        if (threadIdx.x == 0) {
            fence_after();
            const uint32_t a_hi = smem_u32(B0), a_lo = a_hi + SUB_BYTES;
            const uint32_t b_hi = a_hi + 2 * SUB_BYTES, b_lo = a_hi + 3 * SUB_BYTES;
#pragma unroll
            for (int kg = 0; kg < KS / 8; ++kg) {
                const uint32_t ko = kg * KSTEP_BYTES;
                const uint32_t acc0 = (s > 0 || kg > 0) ? 1u : 0u;
                mma_tf32(tmem, make_desc(a_hi + ko), make_desc(b_hi + ko), acc0);
                if (THREE) {
                    mma_tf32(tmem, make_desc(a_hi + ko), make_desc(b_lo + ko), 1u);
                    mma_tf32(tmem, make_desc(a_lo + ko), make_desc(b_hi + ko), 1u);
                }
            }
            commit(&mbar[buf]);
        }
    }
    // the last commit completes after every earlier MMA of this thread
    mbar_wait(&mbar[(nsteps - 1) & 1], ((nsteps - 1) >> 1) & 1);
    fence_after();
    const int warp = threadIdx.x >> 5, row = threadIdx.x;
    const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < N; c0 += 32) {
        float v[32];
        tmem_ld32(tl + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            double* p = C + row + (int64_t)(c0 + i) * ldc;
            __stcg(p, __ldcg(p) - (double)v[i]);
        }
    }
    fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_inval(&mbar[0]);
        mbar_inval(&mbar[1]);
    }
}

}  // namespace tc
}  // namespace mxp
