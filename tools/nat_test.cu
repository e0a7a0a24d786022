// nat_test.cu -- dev harness for tc_native.cuh (fp16 / E4M3 code GEMM blocks on tcgen05).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2410_09819_b200/csrc -o tools/nat_test tools/nat_test.cu
//   ./tools/nat_test [kind 0=f16 1=f8] [ntiles] [reps]   exactness check, then throughput
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "tc_native.cuh"

using namespace mxp;

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);   \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

// small-integer values (exact in fp16 / E4M3 and in fp32 sums) -> code images
__global__ void k_fill(uint8_t* img, int kind, int64_t nb, int ntile, unsigned seed) {
    const int64_t tile = blockIdx.y;
    const int row = blockIdx.x;  // one CTA per row
    for (int k0 = threadIdx.x * 16; k0 < nb; k0 += blockDim.x * 16) {
        double x[16];
        for (int e = 0; e < 16; ++e) {
            unsigned h = (unsigned)(tile * 1315423911u) ^ (unsigned)(row * 2654435761u) ^ (unsigned)((k0 + e) * 97u) ^ seed;
            h ^= h >> 13;
            h *= 0x5bd1e995u;
            h ^= h >> 15;
            x[e] = (double)((int)(h % 9u) - 4);
        }
        uint8_t* t = img + tile * nat::image_bytes(kind, nb);
        if (kind == nat::K_F16) nat::write_f16_16(t, nb, row, k0, x, 1.0);
        else nat::write_f8_16(t, nb, row, k0, x, 1.0);
    }
}

__host__ __device__ inline double hval(int64_t tile, int row, int k, unsigned seed) {
    unsigned h = (unsigned)(tile * 1315423911u) ^ (unsigned)(row * 2654435761u) ^ (unsigned)(k * 97u) ^ seed;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    return (double)((int)(h % 9u) - 4);
}

template <int KIND>
__global__ void __launch_bounds__(128, 1) k_gemm(double* Cb, const uint8_t* imgA, const uint8_t* imgB, int ntiles,
                                                 int64_t nb, int reps) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t taddr;
    if (threadIdx.x < 32) tc::tmem_alloc(&taddr, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = taddr;
    const int64_t S = nb / 128;
    const int rbA = blockIdx.x % S, rbB = (blockIdx.x / S) % S;
    double* C = Cb + (int64_t)blockIdx.x * 128 * 128;
    const int64_t ib = nat::image_bytes(KIND, nb);
    auto src = [&](int i) {
        nat::NatTile t;
        t.a = imgA + (int64_t)i * ib + nat::chunk_offset(KIND, nb, rbA, 0);
        t.b = imgB + (int64_t)i * ib + nat::chunk_offset(KIND, nb, rbB, 0);
        t.inv0 = 1.f;
        t.inv1 = 1.f;
        return t;
    };
    for (int r = 0; r < reps; ++r) nat::block_gemm<KIND>(C, 128, src, ntiles, (int)(nb / nat::ke(KIND)), smem, tmem);
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 512);
}

int main(int argc, char** argv) {
    const int kind = argc > 1 ? atoi(argv[1]) : 0;
    const int ntiles = argc > 2 ? atoi(argv[2]) : 8;
    const int reps = argc > 3 ? atoi(argv[3]) : 20;
    const int64_t nb = 1024;
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const int64_t ib = nat::image_bytes(kind, nb);
    uint8_t *A, *B;
    double* C;
    CK(cudaMalloc(&A, ib * ntiles));
    CK(cudaMalloc(&B, ib * ntiles));
    CK(cudaMalloc(&C, sizeof(double) * 128 * 128 * nsm));
    k_fill<<<dim3((unsigned)nb, ntiles), 64>>>(A, kind, nb, ntiles, 1u);
    k_fill<<<dim3((unsigned)nb, ntiles), 64>>>(B, kind, nb, ntiles, 2u);
    CK(cudaMemset(C, 0, sizeof(double) * 128 * 128 * nsm));
    auto kern = kind == 0 ? k_gemm<nat::K_F16> : k_gemm<nat::K_F8>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, nat::SMEM_BYTES));
    kern<<<nsm, 128, nat::SMEM_BYTES>>>(C, A, B, ntiles, nb, 1);
    CK(cudaDeviceSynchronize());
    // exactness: block 0 (rbA = 0, rbB = 0) and block 1 (rbA = 1, rbB = 0)
    std::vector<double> h(128 * 128 * 2);
    CK(cudaMemcpy(h.data(), C, sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
    double maxerr = 0.0;
    for (int blk = 0; blk < 2; ++blk)
        for (int i = 0; i < 128; ++i)
            for (int j = 0; j < 128; j += 17) {
                double ref = 0.0;
                for (int t = 0; t < ntiles; ++t)
                    for (int k = 0; k < nb; ++k) ref += hval(t, blk * 128 + i, k, 1u) * hval(t, j, k, 2u);
                maxerr = fmax(maxerr, fabs(h[blk * 128 * 128 + i + 128 * j] + ref));
            }
    printf("kind=%s ntiles=%d exact-check max|err|=%g\n", kind == 0 ? "f16" : "e4m3", ntiles, maxerr);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<nsm, 128, nat::SMEM_BYTES>>>(C, A, B, ntiles, nb, reps);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 128 * 128 * nb * ntiles * reps * (double)nsm;
    printf("  %d CTAs x %d reps: %.3f ms  %.1f TFLOP/s (operands %s L2-resident: %.1f MB)\n", nsm, reps, ms,
           fl / (ms * 1e-3) / 1e12, 2 * ib * ntiles < 100e6 ? "" : "NOT", 2.0 * ib * ntiles / 1e6);
    return 0;
}
