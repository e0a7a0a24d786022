// oz_i8.cuh -- FP64 tile GEMM emulated on the int8 tensor cores (Ozaki scheme,
// "scheme I": error-free splitting into integer slices), sm_100a tcgen05.
//
// B200's FP64 tensor pipe (DMMA, ~37 TF/s) is the bottleneck
// of the FP64 tiles (all of C2, the FP64 share of the MxP maps), while its int8
// tensor cores run ~60x faster.  An FP64 operand tile X (rows r, K = tile
// columns) is split row by row, exactly, into s int8 slices:
//
//   E_r = exponent with max_c |X_rc| < 2^E_r          (frexp of the row max)
//   M = rint(X_rc 2^(8s-2-E_r))                        (|M| <= 2^(8s-2): 8s-2 bits + sign)
//   balanced base-256 digits of M from the low end: d_{s-1}, ..., d_1 in [-128, 127]
//   (d = ((M + 128) mod 256) - 128, M <- (M - d) / 256, exact integer steps), d_0 = the rest
//   X_rc ~= 2^(E_r - 6) sum_t d_t 2^(-8t)             (|d_0| <= 64; error <= 2^(E_r - 8s + 1))
//
// A product of two tiles is then a sum of int8 GEMMs with exact int32
// accumulation; pairs of equal weight (t + u = c) share one TMEM accumulator
// ("level" c), and the pairs of weight below 2^-8(s-1) are dropped
// (t + u <= s - 1: s(s+1)/2 int8 GEMMs):
//
//   (A B^T)_rj ~= sA_r sB_j sum_{c=0}^{s-1} 2^(-8c) ACC_c[r][j],
//   ACC_c = sum_{t+u=c} D^A_t D^B_u^T,   sA_r = 2^(EA_r - 6),  sB_j = 2^(EB_j - 6).
//
// Each tile of K carries its own row scales, so the levels are drained (int32
// -> fp64, scaled) after every tile of K into an fp64 register accumulator:
// the accumulation across tiles is FP64, as in a DGEMM.  s = 7 (default) gives
// 54 bits per operand (vs 53 for FP64) with 28 products; the dropped pairs weigh
// <= (s-1) 2^(14-8s) of the product of the two row maxima' scales (~1e-15 worst
// case, random-signed in practice).  |ACC_c| <= s * 2^14 * nb < 2^31 for
// nb <= 16384: no overflow.  (Round 1 used base-128 digits |d| <= 64, s = 8:
// 36 products for 55 bits; the full int8 range carries one more bit per slice.)
//
// Block shape: 128 (M, rows of A) x 64 (N, rows of B).  s levels x 64 int32
// columns live in TMEM (s <= 8 -> <= 512 columns: the whole TMEM of the SM;
// one such CTA per SM), level c at columns [64c, 64c+64).  Stacking B slices
// along N maps onto consecutive levels, so one MMA of N = 64m covers m pairs
// (s = 7: 10 MMAs per 32-K step).
//
// Operand image of a tile (written once by the tile's QUANT tasks): for slice
// t (0-based), 128-row block rb, 32-column K chunk kc, a 4 KB chunk at
//   ((t * (nb/128) + rb) * (nb/32) + kc) * 4096
// holding 128 rows x 32 int8 in the canonical K-major SWIZZLE_32B layout
// (8-row groups of 256 B, row r8 at r8*32, 16-byte half h at h ^ ((r8 >> 2) & 1));
// after the s slices, nb doubles of row scales 2^(E_r - 6).  A B-operand
// (64 rows) is one half of a chunk: rows [64h, 64h+64) = bytes [2048h, 2048h+2048).
#pragma once
#include <stdint.h>

#include "tc_tf32.cuh"

namespace mxp {
namespace oz {

constexpr int MAX_S = 8;
constexpr int BM = 128, BN = 64, KB = 32;  // block rows / cols, K per stage (int8 elements = bytes)
constexpr int CHUNK = BM * KB;             // 4096 B: one slice chunk of 128 rows x 32 K
constexpr int CHUNK_B = BN * KB;           // 2048 B
constexpr int STAGES = 3;
constexpr int STAGE_BYTES = MAX_S * (CHUNK + CHUNK_B);  // 48 KB
constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 128 + BN * 8;  // + align slack, mbarriers, B scales
constexpr int TMEM_COLS = 512;


__host__ __device__ constexpr int64_t image_bytes(int s, int64_t nb) {
    return (((int64_t)s * nb * nb + 8 * nb) + 1023) / 1024 * 1024;
}
__host__ __device__ constexpr int64_t slice_stride(int64_t nb) { return nb * nb; }
__host__ __device__ constexpr int64_t chunk_offset(int64_t nb, int t, int64_t rb, int64_t kc) {
    return ((t * (nb / 128) + rb) * (nb / 32) + kc) * CHUNK;
}
// byte offset of element (row, k) inside a 128 x 32 chunk (row < 128, k < 32)
__host__ __device__ __forceinline__ uint32_t sw32_offset(int row, int k) {
    const int r8 = row & 7;
    return (uint32_t)((row >> 3) * 256 + r8 * 32 + ((((k >> 4) ^ (r8 >> 2)) & 1) << 4) + (k & 15));
}

// smem descriptor: K-major, SWIZZLE_32B, 8-row groups 256 B apart (SBO), LBO unused (1)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(256 >> 4) << 32;
    d |= (uint64_t)1 << 46;  // version 1 (sm100)
    d |= (uint64_t)6 << 61;  // SWIZZLE_32B
    return d;
}
// instruction descriptor: D s32, A/B signed int8, both K-major, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
    return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// The 10 MMAs of one 32-K step for S = 7 as ONE PTX block: the descriptors
// and TMEM addresses are formed by adds inside it, so the uniform-register
// moves happen once per step instead of once per MMA (the per-MMA form cost
// ~100 issue cycles each).  (t, u0, m): A slice t against the m stacked B
// slices u0 .. u0+m-1 into levels t+u0 .. t+u0+m-1 -- the same list as the
// generic loop of block_gemm_t.
__device__ __forceinline__ void mma_step7(uint32_t tmem, uint64_t ad0, uint64_t bd0, uint32_t acc0) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t.reg .b64 a, b;\n\t.reg .b32 d;\n\t"
        "setp.ne.b32 p, %3, 0;\n\tsetp.eq.b32 q, 0, 0;\n\t"
        // t = 0: (u0 0, m 4) -> level 0; (u0 4, m 3) -> level 4
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %4, p;\n\t"
        "add.s64 b, %2, 512;\n\tadd.u32 d, %0, 256;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [d], %1, b, %5, p;\n\t"
        // t = 1: (0, 4) -> level 1; (4, 2) -> level 5
        "add.s64 a, %1, 256;\n\tadd.u32 d, %0, 64;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [d], a, %2, %4, q;\n\t"
        "add.u32 d, %0, 320;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [d], a, b, %6, q;\n\t"
        // t = 2: (0, 4) -> level 2; (4, 1) -> level 6
        "add.s64 a, %1, 512;\n\tadd.u32 d, %0, 128;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [d], a, %2, %4, q;\n\t"
        "add.u32 d, %0, 384;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [d], a, b, %7, q;\n\t"
        // t = 3: (0, 4) -> level 3
        "add.s64 a, %1, 768;\n\tadd.u32 d, %0, 192;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [d], a, %2, %4, q;\n\t"
        // t = 4: (0, 3) -> level 4
        "add.s64 a, %1, 1024;\n\tadd.u32 d, %0, 256;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [d], a, %2, %5, q;\n\t"
        // t = 5: (0, 2) -> level 5
        "add.s64 a, %1, 1280;\n\tadd.u32 d, %0, 320;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [d], a, %2, %6, q;\n\t"
        // t = 6: (0, 1) -> level 6
        "add.s64 a, %1, 1536;\n\tadd.u32 d, %0, 384;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [d], a, %2, %7, q;\n\t}\n" ::"r"(tmem),
        "l"(ad0), "l"(bd0), "r"(acc0), "r"(idesc_i8(256)), "r"(idesc_i8(192)), "r"(idesc_i8(128)),
        "r"(idesc_i8(64)));
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, int (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// exact int32 -> fp64 on the FP64 pipe: 2^52 + 2^31 + x  minus the constant
__device__ __forceinline__ double i2d(int x) {
    return __hiloint2double(0x43300000, (int)((unsigned)x ^ 0x80000000u)) - 4503601774854144.0;
}

// ---------------------------------------------------------------- slicing
// The s int8 digits of y = x * 2^-E in (-1, 1) (see the header comment):
// M = rint(y 2^(8s-2)) then balanced base-256 digits, every step exact.
__device__ __forceinline__ void slice_digits(double y, int s, int (&d)[MAX_S]) {
    long long M = __double2ll_rn(y * __longlong_as_double((long long)(1023 + 8 * s - 2) << 52));
#pragma unroll
    for (int t = MAX_S - 1; t >= 1; --t) {
        if (t < s) {
            const int dt = (int)((M + 128) & 255) - 128;  // in [-128, 127]
            d[t] = dt;
            M = (M - dt) >> 8;  // exact: M - dt is a multiple of 256
        } else {
            d[t] = 0;
        }
    }
    d[0] = (int)M;  // |d_0| <= 64
}
// 2^(E-6) for the row max m (E: m < 2^E, from frexp); m = 0 -> scale 1 (all digits 0)
__device__ __forceinline__ double row_scale(double m, double& inv) {
    if (!(m > 0.0) || !isfinite(m)) {
        inv = 1.0;
        return 1.0;
    }
    int e;
    frexp(m, &e);  // m = f 2^e, f in [0.5, 1)  ->  |x| <= m < 2^e
    inv = scalbn(1.0, -e);
    return scalbn(1.0, e - 6);
}

// Slices of 16 consecutive columns [k0, k0 + 16) (k0 % 16 == 0) of row `row`
// of a tile into its image (x: the 16 values; inv = 2^-E of the row).
__device__ __forceinline__ void write_slices16(uint8_t* img, int64_t nb, int s, int row, int k0,
                                               const double (&x)[16], double inv) {
    uint32_t w[MAX_S][4];
#pragma unroll
    for (int t = 0; t < MAX_S; ++t) w[t][0] = w[t][1] = w[t][2] = w[t][3] = 0u;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
        int d[MAX_S];
        slice_digits(x[e] * inv, s, d);
#pragma unroll
        for (int t = 0; t < MAX_S; ++t) w[t][e >> 2] |= ((uint32_t)d[t] & 0xFFu) << (8 * (e & 3));
    }
    const int64_t rb = row >> 7, kc = k0 >> 5;
    const uint32_t off = sw32_offset(row & 127, k0 & 31);
#pragma unroll
    for (int t = 0; t < MAX_S; ++t)
        if (t < s)
            __stcg(reinterpret_cast<uint4*>(img + chunk_offset(nb, t, rb, kc) + off),
                   make_uint4(w[t][0], w[t][1], w[t][2], w[t][3]));
}

// sum_c 2^(-8c) ACC_c of one element.  S = 7: levels 0-2 and 3-5 are first
// combined exactly in int64 (|.| < 2^47) and converted with the 2^52 + 2^51
// magic number, so 3 conversions and 3 fma replace 7 + 7 on the FP64 pipe (the
// drain is ~15 % of a C2 GEMM task); the value differs from the per-level sum
// only in the order of exact partial sums (no extra rounding below 2^-53 of
// the partials).  Other S: the per-level sum, smallest weight first.
template <int S>
__device__ __forceinline__ double combine_levels(const int (&x)[S][8], int j) {
    if constexpr (S == 7) {
        const long long hi = ((long long)x[0][j] << 16) + ((long long)x[1][j] << 8) + (long long)x[2][j];
        const long long lo = ((long long)x[3][j] << 16) + ((long long)x[4][j] << 8) + (long long)x[5][j];
        const double m = 6755399441055744.0;  // 2^52 + 2^51
        const double hd = __longlong_as_double(0x4338000000000000LL + hi) - m;
        const double ld = __longlong_as_double(0x4338000000000000LL + lo) - m;
        return fma(hd, 0x1p-16, fma(ld, 0x1p-40, i2d(x[6][j]) * 0x1p-48));
    } else {
        double v = 0.0;
#pragma unroll
        for (int c = S - 1; c >= 0; --c)  // smallest weight first; 2^(-8c) exact
            v = fma(i2d(x[c][j]), __longlong_as_double((long long)(1023 - 8 * c) << 52), v);
        return v;
    }
}

// ------------------------------------------------------------ block GEMM
// One operand tile of the K walk: chunk (t = 0, kc = 0) of the A rows / B rows
// of this block, the byte stride between slices, and the row scales.
struct OzTile {
    const uint8_t* a;   // A: image + chunk_offset(nb, 0, rbA, 0)
    const uint8_t* b;   // B: image + chunk_offset(nb, 0, rbB, 0) + 2048 * half
    const double* sa;   // 128 row scales of A's rows
    const double* sb;   // 64 row scales of B's rows
};

// one lane of a converged warp (the same lane every time: the lowest active)
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .b32 rx;\n\t.reg .pred px;\n\t"
        "elect.sync rx|px, %1;\n\t"
        "@px mov.s32 %0, 1;\n\t}\n"
        : "+r"(pred)
        : "r"(0xFFFFFFFFu));
    return pred != 0;
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, int* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}

// C(128 x 64, fp64, column-major ldc) -= sum over ntiles tiles of A_n B_n^T,
// each tile of K = 32 * kt (kt = nb / 32) emulated with S slices (kt * 32 <= 16384);
// C is updated once per tile of K (C <- C - P_n, one fp64 rounding each, in the
// fixed tile order): no 64-double register accumulator, so k_tc fits 5 warps
// beside a k_sched CTA (the 5th warp issues the native engine's MMAs).
// smem: >= SMEM_BYTES dynamic shared memory; tmem: 512 allocated columns.
// All 128 threads call; thread 0 issues the bulk copies and the MMAs (S
// compile-time: the S(S+1)/2 MMAs of a K step are straight-line code on
// precomputed descriptors).
__device__ __forceinline__ uint64_t oz_clock() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// stats (MXP_ATTR_PROFILE): [STAT_OZ_FULL], [STAT_OZ_DONE], [STAT_OZ_DRAIN] in ns, or nullptr
// RACC (the 4-warp k_tc of FP64 maps): the tiles' products accumulate in 64
// fp64 registers per thread and C is updated once per task; otherwise (the
// 5-warp k_tc of MxP maps, 168 registers) C is updated once per tile of K.
// uniform: every tile of the chunk carries the same row scales (running row scales, no flagged
// tile after the first): the int32 level accumulators run across up to `maxt` tiles of K before one drain
// (|ACC_c| <= S 2^14 K must stay below 2^31), instead of one drain per tile of K.
template <int S, bool RACC, class Src>
__device__ void block_gemm_t(double* C, int64_t ldc, const Src& src, int ntiles, int kt, int64_t nb, uint8_t* smem,
                             uint32_t tmem, int pf, unsigned long long* stats, bool uniform) {
    const long long lim = 2147483647LL / ((long long)S * 16384 * 32 * kt);
    const int maxt = uniform ? (lim < 1 ? 1 : (int)lim) : 1;
    int ndrain = 0;
    uint64_t t_full = 0, t_done = 0, t_drain = 0, t_mma = 0, t_copy = 0, t_loop = 0, t_tbar = 0;
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * STAGE_BYTES);
    uint64_t* done = full + STAGES;
    uint64_t* tbar = done + STAGES;
    double* s_sb = reinterpret_cast<double*>(base + STAGES * STAGE_BYTES + 128);
    const int tid = threadIdx.x;
    const int G = ntiles * kt;  // K steps (32 each)
    const int64_t sstride = slice_stride(nb);
    if (tid == 0) {
        for (int i = 0; i < STAGES; ++i) tc::mbar_init(full + i, 1), tc::mbar_init(done + i, 1);
        tc::mbar_init(tbar, 1);
        tc::fence_mbar_init();
    }
    __syncthreads();
    // producer (warp 0): copies of K step g into its stage
    OzTile cur{};
    int cur_i = -1;
    // L2 prefetch of K step g + pf (pf > 0): the operand chunks that miss L2 (~25 % of the
    // sectors at C2) then wait one DRAM latency less than the 3-stage smem ring can hide
    OzTile pcur{};
    int pcur_i = -1;
    auto issue = [&](int g) {
        const uint64_t c0 = stats ? oz_clock() : 0;
        const int i = g / kt, kc = g - i * kt;
        if (i != cur_i) cur = src(i), cur_i = i;
        uint8_t* st = base + (g % STAGES) * STAGE_BYTES;
        uint64_t* fb = full + (g % STAGES);
        const int gp = g + pf;
        if (pf > 0 && gp < G) {
            const int ip = gp / kt, kp = gp - ip * kt;
            if (ip != pcur_i) pcur = src(ip), pcur_i = ip;
            if (elect_one()) {
#pragma unroll
                for (int t = 0; t < S; ++t) {
                    tc::bulk_prefetch_l2(pcur.a + t * sstride + (int64_t)kp * CHUNK, CHUNK);
                    tc::bulk_prefetch_l2(pcur.b + t * sstride + (int64_t)kp * CHUNK, CHUNK_B);
                }
            }
            __syncwarp();
        }
        if (elect_one()) {
            tc::mbar_expect_tx(fb, (uint32_t)(S * (CHUNK + CHUNK_B)));
#pragma unroll
            for (int t = 0; t < S; ++t) {
                tc::bulk_g2s(st + t * CHUNK, cur.a + t * sstride + (int64_t)kc * CHUNK, CHUNK, fb);
                tc::bulk_g2s(st + MAX_S * CHUNK + t * CHUNK_B, cur.b + t * sstride + (int64_t)kc * CHUNK, CHUNK_B,
                             fb);
            }
        }
        __syncwarp();
        if (stats) t_copy += oz_clock() - c0;
    };
    // Warp-specialized: warp 1 produces (bulk copies into the ring, refilling a
    // stage once the MMAs that read it have completed), warp 0 issues the MMAs;
    // one elected lane each.  (A single thread doing both spent ~650 cycles per
    // 32-K step issuing the 10 MMAs and ~630 issuing the 14 copies: more than
    // the ~900 cycles of tensor work they feed -- measured, DESIGN 5.7.)
    const int warp = tid >> 5;
    if (warp == 1) {
        __syncwarp();
        for (int g = 0; g < STAGES && g < G; ++g) issue(g);
    }

    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    double acc[RACC ? BN : 1];
#pragma unroll
    for (int j = 0; j < (RACC ? BN : 1); ++j) acc[j] = 0.0;

    for (int i = 0; i < ntiles; ++i) {
        if (warp == 0) {
            __syncwarp();
            const uint64_t l0 = stats ? oz_clock() : 0;
            for (int kc = 0; kc < kt; ++kc) {
                const int g = i * kt + kc, stage = g % STAGES;
                const uint64_t w0 = stats ? oz_clock() : 0;
                tc::mbar_wait(full + stage, (uint32_t)((g / STAGES) & 1));
                if (stats) t_full += oz_clock() - w0;
                tc::fence_after();
                const uint32_t sa = tc::smem_u32(base + stage * STAGE_BYTES);
                const uint64_t ad0 = make_desc(sa), bd0 = make_desc(sa + MAX_S * CHUNK);
                const uint32_t acc0 = (kc > 0 || i % maxt != 0) ? 1u : 0u;
                const uint64_t m0 = stats ? oz_clock() : 0;
                // A slice t meets B slices u = 0 .. S-1-t, i.e. levels t .. S-1.  The B
                // slices sit 2 KB apart in smem (64 rows each): B slices u0 .. u0+m-1
                // stacked are ONE K-major operand of N = 64 m rows, and its product
                // lands in the m consecutive level accumulators (t+u0) .. (t+u0+m-1)
                // -- so each A slice needs ceil((S-t)/4) MMAs of N <= 256 instead of
                // S-t MMAs of N = 64 (12 instead of 36 for S = 8; A read 12x, not 36x).
                if (elect_one()) {
                    if constexpr (S == 7) {
                        mma_step7(tmem, ad0, bd0, acc0);
                    } else {
#pragma unroll
                        for (int t = 0; t < S; ++t)
#pragma unroll
                            for (int u0 = 0; u0 + t < S; u0 += 4) {
                                const int m = (S - t - u0) < 4 ? (S - t - u0) : 4;
                                mma_i8(tmem + (uint32_t)((t + u0) * BN), ad0 + (uint64_t)(t * (CHUNK >> 4)),
                                       bd0 + (uint64_t)(u0 * (CHUNK_B >> 4)), idesc_i8(BN * m), t > 0 ? 1u : acc0);
                            }
                    }
                    tc::commit(done + stage);
                }
                __syncwarp();
                if (stats) t_mma += oz_clock() - m0;
            }
            if ((i + 1) % maxt == 0 || i + 1 == ntiles) {
                if (elect_one()) tc::commit(tbar);  // every MMA up to tile i
                __syncwarp();
            }
            if (stats) t_loop += oz_clock() - l0;
        } else if (warp == 1) {
            // refill the stage of step g - 1 once its MMAs have read it (step g's MMAs
            // stay queued behind them meanwhile)
            __syncwarp();
            for (int kc = 0; kc < kt; ++kc) {
                const int g = i * kt + kc;
                if (g >= 1 && g - 1 + STAGES < G) {
                    const int pg = g - 1;
                    const uint64_t w1 = stats ? oz_clock() : 0;
                    tc::mbar_wait(done + (pg % STAGES), (uint32_t)((pg / STAGES) & 1));
                    if (stats) t_done += oz_clock() - w1;
                    issue(pg + STAGES);
                }
            }
        }
        // drain: ACC levels of tile i (of tiles i-maxt+1 .. i when uniform) -> fp64, scaled by
        // the row scales (threads 0..127 = TMEM lanes; in k_tc warp 4 only join the barriers)
        if ((i + 1) % maxt != 0 && i + 1 != ntiles) continue;
        const bool wk = tid < 128;
        const uint64_t d0 = (stats && tid == 0) ? oz_clock() : 0;
        if (tid < BN) s_sb[tid] = __ldcg(src(i).sb + tid);
        const double sa_r = wk ? __ldcg(src(i).sa + tid) : 0.0;
        if (wk) tc::mbar_wait(tbar, (uint32_t)(ndrain & 1));
        ++ndrain;
        tc::fence_after();
        __syncthreads();  // s_sb visible
        __syncwarp();     // (converged warp for the .sync.aligned TMEM loads)
        if (stats && tid == 0) t_tbar += oz_clock() - d0;
        if (wk && RACC) {
#pragma unroll
        for (int g8 = 0; g8 < BN / 8; ++g8) {
            int x[S][8];
#pragma unroll
            for (int c = 0; c < S; ++c) tmem_ld8(tl + (uint32_t)(c * BN + g8 * 8), x[c]);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const double v = combine_levels<S>(x, j);
                acc[(g8 * 8 + j) % (RACC ? BN : 1)] =
                    fma(v * sa_r, s_sb[g8 * 8 + j], acc[(g8 * 8 + j) % (RACC ? BN : 1)]);
            }
        }
        } else if (wk) {  // C -= (this tile's product), one fp64 rounding per tile of K
            double* crow = C + tid;
#pragma unroll
        for (int g8 = 0; g8 < BN / 8; ++g8) {
            int x[S][8];
#pragma unroll
            for (int c = 0; c < S; ++c) tmem_ld8(tl + (uint32_t)(c * BN + g8 * 8), x[c]);
            double cv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) cv[j] = __ldcg(crow + (int64_t)(g8 * 8 + j) * ldc);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const double v = combine_levels<S>(x, j);
                __stcg(crow + (int64_t)(g8 * 8 + j) * ldc, fma(-(v * sa_r), s_sb[g8 * 8 + j], cv[j]));
            }
        }
        }
        tc::fence_before();
        __syncthreads();  // TMEM and s_sb free for tile i + 1
        if (stats && tid == 0) t_drain += oz_clock() - d0;
    }
    if (RACC && tid < 128) {  // (16 loads in flight, then the stores: see tc_native.cuh)
#pragma unroll
        for (int j0 = 0; j0 < (RACC ? BN : 1); j0 += 16) {
            double cv[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) cv[j] = __ldcg(C + tid + (int64_t)(j0 + j) * ldc);
#pragma unroll
            for (int j = 0; j < 16; ++j) __stcg(C + tid + (int64_t)(j0 + j) * ldc, cv[j] - acc[(j0 + j) % (RACC ? BN : 1)]);
        }
    }
    if (stats && (tid == 0 || tid == 32)) {  // (warp 0: MMA side; warp 1: copy side)
        atomicAdd(stats + STAT_OZ_FULL, (unsigned long long)t_full);
        atomicAdd(stats + STAT_OZ_DONE, (unsigned long long)t_done);
        atomicAdd(stats + STAT_OZ_DRAIN, (unsigned long long)t_drain);
        atomicAdd(stats + STAT_OZ_MMA, (unsigned long long)t_mma);
        atomicAdd(stats + STAT_OZ_COPY, (unsigned long long)t_copy);
        atomicAdd(stats + STAT_OZ_LOOP, (unsigned long long)t_loop);
        atomicAdd(stats + STAT_OZ_TBAR, (unsigned long long)t_tbar);
    }
    __syncthreads();
    if (tid == 0) {
        for (int i = 0; i < STAGES; ++i) tc::mbar_inval(full + i), tc::mbar_inval(done + i);
        tc::mbar_inval(tbar);
    }
}

constexpr int MIN_S = 4;  // slices supported by the compiled variants: MIN_S..MAX_S
template <bool RACC, class Src>
__device__ __forceinline__ void block_gemm(double* C, int64_t ldc, const Src& src, int ntiles, int s, int kt,
                                           int64_t nb, uint8_t* smem, uint32_t tmem, int pf,
                                           unsigned long long* stats, bool uniform) {
    switch (s) {
    case 4: block_gemm_t<4, RACC>(C, ldc, src, ntiles, kt, nb, smem, tmem, pf, stats, uniform); break;
    case 5: block_gemm_t<5, RACC>(C, ldc, src, ntiles, kt, nb, smem, tmem, pf, stats, uniform); break;
    case 6: block_gemm_t<6, RACC>(C, ldc, src, ntiles, kt, nb, smem, tmem, pf, stats, uniform); break;
    case 7: block_gemm_t<7, RACC>(C, ldc, src, ntiles, kt, nb, smem, tmem, pf, stats, uniform); break;
    default: block_gemm_t<8, RACC>(C, ldc, src, ntiles, kt, nb, smem, tmem, pf, stats, uniform); break;
    }
}

}  // namespace oz
}  // namespace mxp
