// tc_native.cuh -- GEMM tasks of tiles stored below FP64 at the operands'
// native width on the 5th-gen tensor cores (sm_100a):
//   output tile FP16 -> tcgen05.mma kind::f16    (fp16 codes, K = 16 / MMA)
//   output tile FP8  -> tcgen05.mma kind::f8f6f4 (E4M3 codes, K = 32 / MMA)
// with fp32 accumulation in TMEM (G12: "FP32 accumulation for FP16/FP8 tiles
// with per-tile scaling", BASELINE north_star; P:42 minimum bytes per word,
// P:46 low-precision tensor cores).
//
// Operands are the CODES of cast_c(L) (c = the output tile's precision, G12):
// every operand tile carries one power-of-two scale per image (G11), so the
// product of a K tile n is   sum_k codeA codeB = (A B^T)_n * sA_n * sB_n.
// Scales differ from K tile to K tile, so the TMEM partial of each K tile is
// drained and rescaled by 1/(sA_n sB_n) (exact: a power of two) into fp32
// registers; two TMEM accumulators alternate so the drain of tile n overlaps
// the MMAs of tile n+1 (one thread of warp 0 issues the bulk copies and the
// MMAs; warps 0-3 = TMEM lanes 0-127 drain).
//
// Image of a tile (written once by its QUANT tasks): 16 KB chunks of 128 rows
// x 128 bytes (64 fp16 or 128 E4M3 along K), chunk (rb, kc) at
// (rb * (nb / KE) + kc) * 16 KB, each in the canonical K-major SWIZZLE_128B
// layout: row r at r*128 B, its 16-byte unit u stored at unit u ^ (r % 8).
// An A operand (128 output rows) and a B operand (128 output columns) are
// both one row block of their tile's image.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "tc_tf32.cuh"

namespace mxp {
namespace nat {

// K_F32X2: FP32 outputs -- each operand as fp16 codes h = RN(x s) plus the
// remainder l = RN(x s - h) (both in the scale s: 22 bits, like 3xTF32 hi/lo),
// products h h + h l + l h on kind::f16 (l l, 2^-22 relative, dropped)
enum { K_F16 = 0, K_F8 = 1, K_F32X2 = 2 };
constexpr int BM = 128, BN = 128;
constexpr int CHUNK = 128 * 128;            // bytes per operand chunk
constexpr int STAGE_BYTES = 2 * CHUNK;      // A | B
constexpr int NST = 4;                      // stages
constexpr int SMEM_BYTES = 1024 + NST * STAGE_BYTES + 128;

__host__ __device__ constexpr int ke(int kind) { return kind == K_F8 ? 128 : 64; }  // K per chunk
__host__ __device__ constexpr int64_t image_bytes(int kind, int64_t nb) { return nb * nb * (kind == K_F8 ? 1 : 2); }
// stages and chunks per stage: A | B (| A remainder | B remainder for K_F32X2)
__host__ __device__ constexpr int nstages(int kind) { return kind == K_F32X2 ? 2 : NST; }
__host__ __device__ constexpr int stage_bytes(int kind) { return (kind == K_F32X2 ? 4 : 2) * CHUNK; }
__host__ __device__ constexpr int64_t chunk_offset(int kind, int64_t nb, int64_t rb, int64_t kc) {
    return (rb * (nb / ke(kind)) + kc) * CHUNK;
}
// byte offset of byte `kb` (0..127) of row `row` (0..127) inside a chunk
__host__ __device__ __forceinline__ uint32_t sw128(int row, int kb) {
    return (uint32_t)(row * 128 + ((((kb >> 4) ^ row) & 7) << 4) + (kb & 15));
}

// UMMA smem descriptor: K-major SWIZZLE_128B, 8-row groups 1024 B apart (SBO)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;    // SBO
    d |= (uint64_t)1 << 46;              // version 1 (sm100)
    d |= (uint64_t)2 << 61;              // SWIZZLE_128B
    return d;
}
// instruction descriptor: D f32, A/B F16 (kind::f16) or E4M3 (kind::f8f6f4)
// -- format code 0 in both kinds --, both K-major, M = 128, N = 128
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

template <int KIND>
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    if constexpr (KIND != K_F8)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
    else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}

// The 4 MMAs of one stage (K = 4 x 32 bytes: descriptors advance by 2 in their
// 16-byte address field) as one PTX block: the descriptor adds stay in uniform
// registers instead of a register-to-uniform move per MMA.
template <int KIND>
__device__ __forceinline__ void mma4(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    if constexpr (KIND != K_F8)
        asm volatile(
            "{\n\t.reg .pred p, t;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
            "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
            "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
            "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, t;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, t;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, t;\n\t}\n" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
    else
        asm volatile(
            "{\n\t.reg .pred p, t;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
            "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
            "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
            "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a1, b1, %3, t;\n\t"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a2, b2, %3, t;\n\t"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], a3, b3, %3, t;\n\t}\n" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
// one lane of a converged warp (the lowest active)
__device__ __forceinline__ bool elect1() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\t"
        "elect.sync rx|px, %1;\n\t"
        "@px mov.s32 %0, 1;\n\t}\n"
        : "+r"(pred)
        : "r"(0xFFFFFFFFu));
    return pred != 0;
}

// 32 consecutive fp32 columns of this thread's TMEM lane <- v (then wait for the store)
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
        "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
        "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
        "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(mbar)) : "memory");
}

// One K tile of the walk: the first chunk of the A rows / B rows of this
// block (consecutive K chunks follow at CHUNK strides) and 1/(sA sB) split
// into two powers of two that are each representable in fp32.
struct NatTile {
    const uint8_t* a;
    const uint8_t* b;
    const uint8_t* al;  // K_F32X2: remainder images (nullptr: the operand is exact in fp16 codes)
    const uint8_t* bl;
    float inv0, inv1;
};

// Drain of K tile i by this warp (its 32 TMEM lanes): R += P(buf) * inv.
// The running fp32 sum R lives in TMEM columns [256, 384) (no 128-register
// accumulator); partial P in columns [128 buf, 128 buf + 128).
__device__ __forceinline__ void drain_tile(uint32_t tl, int buf, bool first, const NatTile& t) {
    const uint32_t tr = tl + 2 * BN;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32], r[32];
        tc::tmem_ld32(tl + (uint32_t)(buf * BN + c0), v);
        if (!first) {
            tc::tmem_ld32(tr + (uint32_t)c0, r);
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = fmaf(v[j] * t.inv0, t.inv1, r[j]);
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = (v[j] * t.inv0) * t.inv1;
        }
        tmem_st32(tr + (uint32_t)c0, r);
    }
}

// C(128 x 128, fp64, column-major ldc) -= sum over ntiles K tiles of
// (A_n B_n^T) = codes products * inv;  kt = chunks per K tile (nb / KE).
// All 160 threads of k_tc call; tmem: >= 384 allocated columns (two
// accumulators + the running sum).  Warp 4 is the producer and MMA issuer (one
// lane: bulk copies into the ring, the MMAs of each step, refilling a stage as
// soon as the MMAs that read it complete); warps 0-3 (= TMEM lanes 0-127 =
// output rows) drain each K tile's accumulator while the tensor core runs the
// next one.  (Round 2 first had warp 0 issue and drain: while it drained, no
// MMA was issued -- the drains of the warp that feeds the tensor core were
// serialized with the MMAs.)
__device__ __forceinline__ uint64_t nat_clock() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
template <int KIND, class Src>
__device__ void block_gemm(double* C, int64_t ldc, const Src& src, int ntiles, int kt, uint8_t* smem, uint32_t tmem,
                           unsigned long long* stats = nullptr, int pf = 0) {
    uint64_t w_full = 0, w_empty = 0, w_tempty = 0, t_drain = 0, t_final = 0;
    constexpr int NS = nstages(KIND), SB = stage_bytes(KIND);
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(base + NS * SB);
    uint64_t* empty = full + NS;
    uint64_t* tfull = empty + NS;   // [2] accumulator ready for the drain
    uint64_t* tempty = tfull + 2;   // [2] accumulator drained (4 warps arrive)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int G = ntiles * kt;
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    if (tid == 0) {
        for (int i = 0; i < NS; ++i) tc::mbar_init(full + i, 1), tc::mbar_init(empty + i, 1);
        for (int i = 0; i < 2; ++i) tc::mbar_init(tfull + i, 1), tc::mbar_init(tempty + i, 4);
        tc::fence_mbar_init();
    }
    __syncthreads();
    if (warp == 4) {  // (all 32 lanes walk the loop converged; one elected lane issues)
        {
            NatTile cur{}, curm{}, pcur{};
            int cur_i = -1, pcur_i = -1;
            auto issue = [&](int g) {  // bulk copies of K step g into its stage
                const int st = g % NS, i = g / kt, kc = g - i * kt;
                if (i != cur_i) cur = src(i), cur_i = i;
                uint8_t* sa = base + st * SB;
                const int64_t o = (int64_t)kc * CHUNK;
                uint32_t bytes = 2 * CHUNK;
                if (KIND == K_F32X2) bytes += (cur.al ? CHUNK : 0) + (cur.bl ? CHUNK : 0);
                const int gp = g + pf;  // L2 prefetch of the operands pf K steps ahead (MXP_ATTR_OZ_PREFETCH)
                if (pf > 0 && gp < G) {
                    const int ip = gp / kt, kp = gp - ip * kt;
                    if (ip != pcur_i) pcur = src(ip), pcur_i = ip;
                    if (elect1()) {
                        const int64_t op = (int64_t)kp * CHUNK;
                        tc::bulk_prefetch_l2(pcur.a + op, CHUNK);
                        tc::bulk_prefetch_l2(pcur.b + op, CHUNK);
                        if (KIND == K_F32X2 && pcur.al) tc::bulk_prefetch_l2(pcur.al + op, CHUNK);
                        if (KIND == K_F32X2 && pcur.bl) tc::bulk_prefetch_l2(pcur.bl + op, CHUNK);
                    }
                    __syncwarp();
                }
                if (elect1()) {
                    tc::mbar_expect_tx(full + st, bytes);
                    tc::bulk_g2s(sa, cur.a + o, CHUNK, full + st);
                    tc::bulk_g2s(sa + CHUNK, cur.b + o, CHUNK, full + st);
                    if (KIND == K_F32X2 && cur.al) tc::bulk_g2s(sa + 2 * CHUNK, cur.al + o, CHUNK, full + st);
                    if (KIND == K_F32X2 && cur.bl) tc::bulk_g2s(sa + 3 * CHUNK, cur.bl + o, CHUNK, full + st);
                }
                __syncwarp();
            };
            for (int g = 0; g < NS && g < G; ++g) issue(g);
            for (int i = 0; i < ntiles; ++i) {
                const int buf = i & 1;
                if (KIND == K_F32X2) curm = src(i);
                const uint64_t q0 = stats ? nat_clock() : 0;
                if (i >= 2) tc::mbar_wait(tempty + buf, (uint32_t)(((i >> 1) - 1) & 1));
                if (stats) w_tempty += nat_clock() - q0;
                tc::fence_after();
                const uint32_t d = tmem + (uint32_t)(buf * BN);
                for (int kc = 0; kc < kt; ++kc) {
                    const int g = i * kt + kc, st = g % NS;
                    const uint64_t q1 = stats ? nat_clock() : 0;
                    tc::mbar_wait(full + st, (uint32_t)((g / NS) & 1));
                    if (stats) w_full += nat_clock() - q1;
                    tc::fence_after();
                    const uint32_t sa = tc::smem_u32(base + st * SB);
                    const uint64_t ad = make_desc(sa), bd = make_desc(sa + CHUNK);
                    if (elect1()) {
                        if constexpr (KIND != K_F32X2) {
                            mma4<KIND>(d, ad, bd, kc ? 1u : 0u);
                        } else {
                            mma4<KIND>(d, ad, bd, kc ? 1u : 0u);  // h h
                            if (curm.bl) mma4<KIND>(d, ad, make_desc(sa + 3 * CHUNK), 1u);  // h l
                            if (curm.al) mma4<KIND>(d, make_desc(sa + 2 * CHUNK), bd, 1u);  // l h
                        }
                        tc::commit(empty + st);
                    }
                    __syncwarp();
                    // refill the previous step's stage once its MMAs have read it (this
                    // step's MMAs stay queued behind them meanwhile)
                    const int pg = g - 1;
                    if (pg >= 0 && pg + NS < G) {
                        const uint64_t q2 = stats ? nat_clock() : 0;
                        tc::mbar_wait(empty + (pg % NS), (uint32_t)((pg / NS) & 1));
                        if (stats) w_empty += nat_clock() - q2;
                        issue(pg + NS);
                    }
                }
                if (elect1()) tc::commit(tfull + buf);
                __syncwarp();
            }
        }
        __syncwarp();
    } else {  // warps 0-3: drain every K tile as soon as it is complete
        for (int i = 0; i < ntiles; ++i) {
            const int buf = i & 1;
            const NatTile t = src(i);
            tc::mbar_wait(tfull + buf, (uint32_t)((i >> 1) & 1));
            tc::fence_after();
            __syncwarp();
            const uint64_t q3 = stats ? nat_clock() : 0;
            drain_tile(tl, buf, i == 0, t);
            tc::fence_before();
            __syncwarp();
            if (stats) t_drain += nat_clock() - q3;
            if (lane == 0) mbar_arrive(tempty + buf);
        }
        // C -= R (fp64 read-modify-write of this thread's output row)
        const uint64_t q4 = stats ? nat_clock() : 0;
        const uint32_t tr = tl + 2 * BN;
        const int row = tid;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
            float r[32];
            tc::tmem_ld32(tr + (uint32_t)c0, r);
            // loads first, then the stores: interleaved load-subtract-store per element was
            // serialized by possible aliasing (~1 L2 round trip per element: measured 58 us per
            // 128 x 128 block, 45 % of the native engine's time at C3)
#pragma unroll
            for (int j0 = 0; j0 < 32; j0 += 16) {
                double cv[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) cv[j] = __ldcg(C + row + (int64_t)(c0 + j0 + j) * ldc);
#pragma unroll
                for (int j = 0; j < 16; ++j) __stcg(C + row + (int64_t)(c0 + j0 + j) * ldc, cv[j] - (double)r[j0 + j]);
            }
        }
        tc::fence_before();
        if (stats) t_final += nat_clock() - q4;
    }
    __syncthreads();
    if (stats && (tid == 0 || tid == 128)) {  // (warp 0: drains; warp 4: issuer)
        atomicAdd(stats + STAT_NAT_FULL, (unsigned long long)w_full);
        atomicAdd(stats + STAT_NAT_EMPTY, (unsigned long long)w_empty);
        atomicAdd(stats + STAT_NAT_TEMPTY, (unsigned long long)w_tempty);
        atomicAdd(stats + STAT_NAT_DRAIN, (unsigned long long)t_drain);
        atomicAdd(stats + STAT_NAT_FINAL, (unsigned long long)t_final);
    }
    if (tid == 0) {
        for (int i = 0; i < NS; ++i) tc::mbar_inval(full + i), tc::mbar_inval(empty + i);
        for (int i = 0; i < 2; ++i) tc::mbar_inval(tfull + i), tc::mbar_inval(tempty + i);
    }
}

// ---------------------------------------------------------------- images
// Codes of 16 consecutive K elements [k0, k0+16) of row `row` of a tile into
// its image (values x already on the grid of cast_c with scale s: x*s is an
// exact fp16 / E4M3 code).
__device__ __forceinline__ void write_f16_16(uint8_t* img, int64_t nb, int row, int k0, const double (&x)[16],
                                             double s) {
    uint32_t w[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const unsigned short lo = __half_as_ushort(__double2half(x[2 * e] * s));
        const unsigned short hi = __half_as_ushort(__double2half(x[2 * e + 1] * s));
        w[e] = (uint32_t)lo | ((uint32_t)hi << 16);
    }
    const int64_t rb = row >> 7, kc = k0 >> 6;
    const int kb = (k0 & 63) * 2;
    uint8_t* ch = img + chunk_offset(K_F16, nb, rb, kc);
    __stcg(reinterpret_cast<uint4*>(ch + sw128(row & 127, kb)), make_uint4(w[0], w[1], w[2], w[3]));
    __stcg(reinterpret_cast<uint4*>(ch + sw128(row & 127, kb + 16)), make_uint4(w[4], w[5], w[6], w[7]));
}
// fp16 remainders l = RN(x s - RN(x s)) of 16 consecutive K elements (K_F32X2)
__device__ __forceinline__ void write_f16rem_16(uint8_t* img, int64_t nb, int row, int k0, const double (&x)[16],
                                                double s) {
    double r[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        const double y = x[e] * s;
        r[e] = y - (double)__half2float(__double2half(y));
    }
    write_f16_16(img, nb, row, k0, r, 1.0);
}
__device__ __forceinline__ void write_f8_16(uint8_t* img, int64_t nb, int row, int k0, const double (&x)[16],
                                            double s) {
    uint32_t w[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        uint32_t b = 0;
#pragma unroll
        for (int q = 0; q < 4; q += 2) {
            unsigned short pair;
            asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;"
                : "=h"(pair)
                : "f"((float)(x[4 * e + q + 1] * s)), "f"((float)(x[4 * e + q] * s)));
            b |= (uint32_t)pair << (8 * q);
        }
        w[e] = b;
    }
    const int64_t rb = row >> 7, kc = k0 >> 7;
    uint8_t* ch = img + chunk_offset(K_F8, nb, rb, kc);
    __stcg(reinterpret_cast<uint4*>(ch + sw128(row & 127, k0 & 127)), make_uint4(w[0], w[1], w[2], w[3]));
}

// 1/(sA sB) as two fp32 powers of two (sA, sB = 2^kA, 2^kB with |kA|, |kB| <= 127)
__device__ __forceinline__ void inv_scales(double sa, double sb, float& inv0, float& inv1) {
    int ea = ilogb(sa), eb = ilogb(sb);
    int e = -(ea + eb);
    int e0 = e > 120 ? 120 : (e < -120 ? -120 : e);
    inv0 = scalbnf(1.f, e0);
    inv1 = scalbnf(1.f, e - e0);
}

}  // namespace nat
}  // namespace mxp
