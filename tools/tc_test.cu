// tc_test.cu -- dev harness for tc_block.cuh (tcgen05 TF32 block GEMM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2410_09819_b200/csrc -o tc_test tools/tc_test.cu
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "tc_block.cuh"

using namespace mxp;

template <bool THREE>
__global__ void __launch_bounds__(128) k_test(double* C, const double* A, const double* B, int64_t ld, int K,
                                              int cmode, double amaxA, double amaxB) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint64_t mbar[2];
    __shared__ uint32_t taddr;
    if (threadIdx.x < 32) tc::tmem_alloc(&taddr, 128);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = taddr;
    const int64_t r0 = blockIdx.x * 128, c0 = blockIdx.y * 128;
    Cast ca = make_cast(P_FP64, cmode, amaxA), cb = make_cast(P_FP64, cmode, amaxB);
    int off = 0;
    auto src = [&](int s) {
        tc::Chunk ch;
        ch.a = A + r0 + (int64_t)(s + off) * 16 * ld;
        ch.b = B + c0 + (int64_t)(s + off) * 16 * ld;
        ch.ca = ca;
        ch.cb = cb;
        return ch;
    };
    const int total = K / 16, half = total / 2;
    for (int rep = 0; rep < 2; ++rep) {  // two tasks back to back: exercises mbarrier/TMEM reuse
        off = rep ? half : 0;
        tc::block_gemm<THREE>(C + r0 + c0 * ld, ld, src, rep ? total - half : half, ld, ld, smem, mbar, tmem);
    }
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_dealloc(tmem, 128);
}

int main(int argc, char** argv) {
    int M = 256, N = 256, K = 1024;
    int64_t ld = 8192 + 128;
    size_t el = (size_t)ld * 8192;
    double *A, *B, *C;
    cudaMalloc(&A, el * 8);
    cudaMalloc(&B, el * 8);
    cudaMalloc(&C, el * 8);
    std::vector<double> hA(el), hB(el), hC((size_t)ld * N);
    int fails = 0;
    for (int mode = 0; mode < 2; ++mode) {
        bool three = mode == 1;
        srand(3 + mode);
        for (size_t i = 0; i < (size_t)ld * K; ++i) {
            if (!three) {
                hA[i] = (double)(rand() % 17 - 8);
                hB[i] = (double)(rand() % 17 - 8) * 0.25;
            } else {
                hA[i] = (rand() / (double)RAND_MAX - 0.5);
                hB[i] = (rand() / (double)RAND_MAX - 0.5);
            }
        }
        cudaMemcpy(A, hA.data(), (size_t)ld * K * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(B, hB.data(), (size_t)ld * K * 8, cudaMemcpyHostToDevice);
        cudaMemset(C, 0, (size_t)ld * N * 8);
        dim3 g(M / 128, N / 128);
        int smem = tc::SMEM_BYTES;
        if (three) {
            cudaFuncSetAttribute(k_test<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_test<true><<<g, 128, smem>>>(C, A, B, ld, K, P_FP32, 0.5, 0.5);
        } else {
            cudaFuncSetAttribute(k_test<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_test<false><<<g, 128, smem>>>(C, A, B, ld, K, P_FP64, 8.0, 2.0);
        }
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %s: %s\n", three ? "3xTF32" : "1xTF32", cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        cudaMemcpy(hC.data(), C, (size_t)ld * N * 8, cudaMemcpyDeviceToHost);
        double maxerr = 0, maxref = 0;
        for (int i = 0; i < M; ++i)
            for (int j = 0; j < N; ++j) {
                double s = 0;
                for (int k = 0; k < K; ++k) {
                    double a = hA[i + (size_t)k * ld], b = hB[j + (size_t)k * ld];
                    if (three) { a = (double)(float)a; b = (double)(float)b; }
                    s += a * b;
                }
                double got = -hC[i + (size_t)j * ld];
                maxerr = fmax(maxerr, fabs(got - s));
                maxref = fmax(maxref, fabs(s));
            }
        double rel = maxerr / maxref;
        printf("  max|err| = %.3e  max|ref| = %.3e  rel = %.3e\n", maxerr, maxref, rel);
        if (!three && maxerr != 0.0) ++fails;
        if (three && rel > 1e-5) ++fails;
    }
    // throughput: 8192 x 8192 x K=8192 in 128x128 blocks (4096 CTAs)
    for (int mode = 0; mode < 2; ++mode) {
        int MM = 8192, NN = 8192, KK = 8192;
        dim3 g(MM / 128, NN / 128);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e9;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0);
            if (mode) k_test<true><<<g, 128, tc::SMEM_BYTES>>>(C, A, B, ld, KK, P_FP32, 0.5, 0.5);
            else k_test<false><<<g, 128, tc::SMEM_BYTES>>>(C, A, B, ld, KK, P_FP16, 0.5, 0.5);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        double tf = 2.0 * MM * NN * (double)KK / (best / 1e3) / 1e12;
        printf("throughput %s: %.2f ms  %.1f TF/s  (%s)\n", mode ? "3xTF32" : "1xTF32 (FP16 cast)", best, tf,
               cudaGetErrorString(cudaGetLastError()));
    }
    printf(fails ? "FAIL\n" : "PASS\n");
    return fails;
}
