// tc_tf32.cuh -- tcgen05 (5th-gen tensor core) TF32 building blocks for sm_100a.
//
// Used for the GEMM tasks whose output tile is stored below FP64 (G12): the
// operands are staged as fp32 VALUES of cast_c(L) (exact for FP16/E4M3
// values; FP32 values are split hi + lo for 3xTF32), multiplied with
// tcgen05.mma.cta_group::1.kind::tf32 (M = 128, N = 128, K = 8 per
// instruction) into an fp32 accumulator in TMEM, and drained with tcgen05.ld.
//
// Shared-memory operand layout (both A and B are MN-major, like the tiles):
// fp32/tf32 MN-major operands use the canonical SWIZZLE_128B_BASE32B layout
// (layout type 1, CuTe Swizzle<2,5,2>): 512-byte atoms of 4 K-rows x 128 B
// (32 fp32 along MN) in which the 32-byte chunk c of row r sits at chunk
// (c ^ r).  A 128 (MN) x 16 (K) sub-buffer is 16 atoms: atom(mb, ka) at
// mb*512 + ka*2048, so LBO (MN-block stride) = 512 B and SBO (K-atom stride)
// = 2048 B; one K = 8 instruction spans two K-atoms.
#pragma once
#include <stdint.h>

namespace mxp {
namespace tc {

constexpr int M = 128, N = 128;        // UMMA shape
constexpr int KS = 16;                 // K per sub-buffer (two K-groups of 8)
constexpr int SUB_BYTES = 128 * KS * 4;  // 8 KB
constexpr uint32_t LBO = 512, SBO = 2048;
constexpr uint32_t KSTEP_BYTES = 2 * SBO;  // advance of the descriptor per K = 8 instruction
constexpr int TMEM_COLS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of element (mn, k) inside a 128 x KS sub-buffer
__device__ __forceinline__ uint32_t sw_offset(int mn, int k) {
    const int mb = mn >> 5, c32 = (mn & 31) >> 3, ka = k >> 2, r = k & 3;
    return (uint32_t)(mb * LBO + ka * SBO + r * 128 + ((c32 ^ r) << 5) + ((mn & 7) << 2));
}

// UMMA shared-memory descriptor (sm100 version 1, SWIZZLE_128B_BASE32B)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((LBO >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((SBO >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;  // version = 1 (Blackwell)
    d |= (uint64_t)1 << 61;  // SWIZZLE_128B_BASE32B
    return d;
}

// instruction descriptor: D f32, A/B tf32, both MN-major, M = 128, N = 128
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
        ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}
__device__ __forceinline__ void commit(uint64_t* mbar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 ::"r"(smem_u32(mbar)) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_inval(uint64_t* mbar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(mbar)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
    uint32_t a = smem_u32(mbar);
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(a), "r"(parity) : "memory");
}

// TMEM allocation by one full warp; the base address is written to *dst (smem)
__device__ __forceinline__ void tmem_alloc(uint32_t* dst, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(dst)), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

// 32 consecutive accumulator columns of this thread's TMEM lane (row)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// mbarrier transaction count for bulk copies (tx bytes), then arrive
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
}
// TMA-engine bulk copy global -> this CTA's shared memory, completing on mbar
// L2 prefetch of a global range (no smem, no completion tracking)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(mbar))
        : "memory");
}

// round-to-nearest-even to TF32 (10 explicit mantissa bits); the result is
// exact as a tensor-core TF32 operand
__device__ __forceinline__ float rne_tf32(float x) {
    uint32_t b = __float_as_uint(x);
    if ((b & 0x7F800000u) == 0x7F800000u) return x;  // inf / nan
    b += 0x0FFFu + ((b >> 13) & 1u);
    return __uint_as_float(b & 0xFFFFE000u);
}

// 3xTF32 split: x = hi + lo, hi = RNE_tf32(x), lo = RNE_tf32(x - hi) (both
// exact TF32 operands; the same split the operand images store)
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
    hi = rne_tf32(x);
    lo = rne_tf32(x - hi);
}

}  // namespace tc
}  // namespace mxp
