// tc_diag.cu -- minimal tcgen05 diagnostics (dev tool)
#include <cuda_runtime.h>
#include <stdio.h>
#include "tc_tf32.cuh"
using namespace mxp;

__device__ void mma_any(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc, int kind) {
    if (kind == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                     ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                     ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__global__ void k_diag(float* out, uint32_t idesc, int kind, int swz, int delay) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t taddr;
    uint8_t* base = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
    if (threadIdx.x < 32) tc::tmem_alloc(&taddr, 128);
    tc::fence_before(); __syncthreads(); tc::fence_after();
    uint32_t tmem = taddr;
    const int warp = threadIdx.x >> 5;
    uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
    uint32_t* f = (uint32_t*)base;
    uint32_t one = kind == 0 ? 0x3f800000u : 0x3C003C00u;
    for (int i = threadIdx.x; i < 8192; i += 128) f[i] = one;  // 32 KB of ones
    if (threadIdx.x == 0) { tc::mbar_init(&mbar, 1); tc::fence_mbar_init(); }
    tc::fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
        tc::fence_after();
        uint32_t a = tc::smem_u32(base), b = a + 16384;
        uint64_t da = 0, db = 0;
        da |= (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(512 >> 4) << 16) | ((uint64_t)(2048 >> 4) << 32) | (1ull << 46) | ((uint64_t)swz << 61);
        db |= (uint64_t)((b >> 4) & 0x3FFF) | ((uint64_t)(512 >> 4) << 16) | ((uint64_t)(2048 >> 4) << 32) | (1ull << 46) | ((uint64_t)swz << 61);
        mma_any(tmem, da, db, idesc, 0u, kind);
        tc::commit(&mbar);
    }
    tc::mbar_wait(&mbar, 0);
    tc::fence_after();
    if (delay) { long t0 = clock64(); while (clock64() - t0 < 2000000) {} }
    float v[32];
    for (int c = 0; c < 4; ++c) {
        tc::tmem_ld32(tl + c * 32, v);
        for (int i = 0; i < 32; ++i) out[threadIdx.x * 128 + c * 32 + i] = v[i];
    }
    tc::fence_before(); __syncthreads();
    if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 128);
}

int main() {
    float* d; cudaMalloc(&d, 128 * 128 * 4);
    static float h[128 * 128];
    cudaFuncSetAttribute(k_diag, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    struct V { const char* name; uint32_t idesc; int kind, swz, delay; } vs[] = {
        {"tf32 MN/MN base32", tc::IDESC, 0, 1, 0},
        {"tf32 MN/MN base32 +delay", tc::IDESC, 0, 1, 1},
    };
    for (auto& v : vs) {
        cudaMemset(d, 0xff, sizeof(h));
        k_diag<<<1, 128, 40000>>>(d, v.idesc, v.kind, v.swz, v.delay);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        int nz = 0; for (int i = 0; i < 128 * 128; ++i) nz += h[i] != 0.0f;
        printf("%-26s %-14s d[0,0]=%g d[0,127]=%g d[127,0]=%g d[64,77]=%g nonzero=%d\n", v.name, cudaGetErrorString(e),
               h[0], h[127], h[127 * 128], h[64 * 128 + 77], nz);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
