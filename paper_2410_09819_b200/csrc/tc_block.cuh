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
        for (int i0 = 0; i0 < 32; i0 += 8) {  // (loads first, then stores: aliasing would serialize)
            double cv[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) cv[i] = __ldcg(C + row + (int64_t)(c0 + i0 + i) * ldc);
#pragma unroll
            for (int i = 0; i < 8; ++i) __stcg(C + row + (int64_t)(c0 + i0 + i) * ldc, cv[i] - (double)v[i0 + i]);
        }
    }
    fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_inval(&mbar[0]);
        mbar_inval(&mbar[1]);
    }
}

// ---------------------------------------------------------------------------
// Operand-image variant: the operands arrive as pre-built fp32 images of
// cast_c(L) in exactly the shared-memory layout above (8 KB per 128 x 16
// chunk), written once per tile by the QUANT task (see sched_f64.cu), so the
// main loop is bulk copies (TMA engine, cp.async.bulk + mbarrier tx counts)
// feeding tcgen05.mma -- no per-element work on the SMs.
//
// Stage = 32 KB = 4 chunks: THREE: A_hi | A_lo | B_hi | B_lo of one K = 16
// step (lo chunks absent -> that product is skipped: the operand is exact in
// TF32); else A(s) | A(s+1) | B(s) | B(s+1) (K = 32 per stage).  Two stages;
// one elected thread issues copies and MMAs; all threads run the epilogue.
struct ImgStep {
    const uint8_t* ahi;
    const uint8_t* alo;  // nullptr: A exact in TF32
    const uint8_t* bhi;
    const uint8_t* blo;
};
constexpr int IMG_STAGE = 4 * SUB_BYTES;                     // 32 KB
constexpr int IMG_SMEM_BYTES = 1024 + 2 * IMG_STAGE + 64;    // + alignment slack + 5 mbarriers (NST = 2)

// NST stages: 2 in k_sched (3 CTAs per SM), 4 in k_tc (one CTA per SM).  Thread 0
// drives the pipeline (a warp-driven elect.sync variant measured slower).
template <bool THREE, int NST, class Src>
__device__ void block_gemm_img(double* C, int64_t ldc, const Src& src, int nsteps, uint8_t* smem, uint32_t tmem) {
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(base + NST * IMG_STAGE);
    uint64_t* done = full + NST;
    uint64_t* fin = done + NST;  // one-shot: every MMA of the block has completed
    const int nst = THREE ? nsteps : (nsteps + 1) / 2;  // stages to run
    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) mbar_init(&full[i], 1), mbar_init(&done[i], 1);
        mbar_init(fin, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // stage contents: which of the 4 chunks hold data (bit i = chunk i)
        auto issue = [&](int st, int stage) -> uint32_t {
            uint8_t* B0 = base + stage * IMG_STAGE;
            const uint8_t* srcs[4];
            if (THREE) {
                const ImgStep c = src(st);
                srcs[0] = c.ahi, srcs[1] = c.alo, srcs[2] = c.bhi, srcs[3] = c.blo;
            } else {
                const ImgStep c0 = src(2 * st);
                srcs[0] = c0.ahi, srcs[2] = c0.bhi;
                if (2 * st + 1 < nsteps) {
                    const ImgStep c1 = src(2 * st + 1);
                    srcs[1] = c1.ahi, srcs[3] = c1.bhi;
                } else {
                    srcs[1] = srcs[3] = nullptr;
                }
            }
            uint32_t mask = 0, bytes = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (srcs[i]) mask |= 1u << i, bytes += SUB_BYTES;
            mbar_expect_tx(&full[stage], bytes);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (srcs[i]) bulk_g2s(B0 + i * SUB_BYTES, srcs[i], SUB_BYTES, &full[stage]);
            return mask;
        };
        uint32_t masks[NST];
        for (int i = 0; i < NST && i < nst; ++i) masks[i] = issue(i, i);
        for (int st = 0; st < nst; ++st) {
            const int stage = st % NST;
            mbar_wait(&full[stage], (st / NST) & 1);
            fence_after();
            const uint32_t b0 = smem_u32(base + stage * IMG_STAGE);
            const uint32_t m = masks[stage];
#pragma unroll
            for (int kg = 0; kg < KS / 8; ++kg) {
                const uint32_t ko = kg * KSTEP_BYTES;
                if (THREE) {
                    const uint32_t acc0 = (st > 0 || kg > 0) ? 1u : 0u;
                    mma_tf32(tmem, make_desc(b0 + ko), make_desc(b0 + 2 * SUB_BYTES + ko), acc0);
                    if (m & 8u) mma_tf32(tmem, make_desc(b0 + ko), make_desc(b0 + 3 * SUB_BYTES + ko), 1u);
                    if (m & 2u) mma_tf32(tmem, make_desc(b0 + SUB_BYTES + ko), make_desc(b0 + 2 * SUB_BYTES + ko), 1u);
                } else {  // K step 2st first, then 2st + 1 (the register-staged engine's order)
                    const uint32_t acc0 = (st > 0 || kg > 0) ? 1u : 0u;
                    mma_tf32(tmem, make_desc(b0 + ko), make_desc(b0 + 2 * SUB_BYTES + ko), acc0);
                }
            }
            if (!THREE && (m & 2u)) {
#pragma unroll
                for (int kg = 0; kg < KS / 8; ++kg) {
                    const uint32_t ko = kg * KSTEP_BYTES;
                    mma_tf32(tmem, make_desc(b0 + SUB_BYTES + ko), make_desc(b0 + 3 * SUB_BYTES + ko), 1u);
                }
            }
            commit(&done[stage]);
            if (st + NST < nst) {
                mbar_wait(&done[stage], (st / NST) & 1);  // this stage's MMAs have read their operands
                masks[stage] = issue(st + NST, stage);
            }
        }
        commit(fin);  // tracks every earlier tcgen05 op of this thread
    }
    __syncwarp();
    if (threadIdx.x < 128) {  // TMEM lanes 0..127 (k_tc's warp 4 only join the barriers)
        // (a one-shot barrier: the per-stage ones may be several phases ahead of
        // a thread that starts waiting early, and parity waits would alias)
        mbar_wait(fin, 0);
        fence_after();
        const int warp = threadIdx.x >> 5, row = threadIdx.x;
        const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll 1
        for (int c0 = 0; c0 < N; c0 += 32) {
            float v[32];
            tmem_ld32(tl + c0, v);
#pragma unroll
            for (int i0 = 0; i0 < 32; i0 += 8) {  // (loads first, then stores: aliasing would serialize)
                double cv[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) cv[i] = __ldcg(C + row + (int64_t)(c0 + i0 + i) * ldc);
#pragma unroll
                for (int i = 0; i < 8; ++i) __stcg(C + row + (int64_t)(c0 + i0 + i) * ldc, cv[i] - (double)v[i0 + i]);
            }
        }
    }
    fence_before();
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) mbar_inval(&full[i]), mbar_inval(&done[i]);
        mbar_inval(fin);
    }
}

}  // namespace tc
}  // namespace mxp
