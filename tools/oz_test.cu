// oz_test.cu -- dev harness for oz_i8.cuh (FP64 GEMM block emulated on int8 tcgen05).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2410_09819_b200/csrc -o tools/oz_test tools/oz_test.cu
//   ./tools/oz_test [s]      accuracy vs a long-double reference, then throughput
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "oz_i8.cuh"

using namespace mxp;

#define CK(x)                                                                               \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) {                                                            \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);        \
            exit(1);                                                                        \
        }                                                                                   \
    } while (0)

// one CTA per tile: row scales (thread per row), then slices
__global__ void k_slice(const double* X, int64_t nb, int s, uint8_t* img_base, int64_t img_bytes) {
    const double* T = X + (int64_t)blockIdx.x * nb * nb;
    uint8_t* img = img_base + (int64_t)blockIdx.x * img_bytes;
    double* rs = reinterpret_cast<double*>(img + (int64_t)s * nb * nb);
    for (int row = threadIdx.x; row < nb; row += blockDim.x) {
        double m = 0.0;
        for (int c = 0; c < nb; ++c) m = fmax(m, fabs(T[row + (int64_t)c * nb]));
        double inv;
        rs[row] = oz::row_scale(m, inv);
        for (int k0 = 0; k0 < nb; k0 += 16) {
            double x[16];
            for (int e = 0; e < 16; ++e) x[e] = T[row + (int64_t)(k0 + e) * nb];
            oz::write_slices16(img, nb, s, row, k0, x, inv);
        }
    }
}

// block (rbA, hB) of every tile: C(128 x 64) -= sum_n A_n[rows] B_n[rows]^T
__global__ void __launch_bounds__(128, 1) k_gemm(double* Cb, const uint8_t* imgA, const uint8_t* imgB,
                                                 int64_t img_bytes, int ntiles, int s, int64_t nb, int rbA_mod,
                                                 int reps) {
    extern __shared__ __align__(16) uint8_t smem[];
    __shared__ uint32_t taddr;
    if (threadIdx.x < 32) tc::tmem_alloc(&taddr, oz::TMEM_COLS);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = taddr;
    const int rbA = blockIdx.x % rbA_mod, hB = (blockIdx.x / rbA_mod) % (int)(2 * nb / 128);
    const int rbB = hB >> 1, half = hB & 1;
    double* C = Cb + (int64_t)blockIdx.x * 128 * 64;
    auto src = [&](int i) {
        const uint8_t* ia = imgA + (int64_t)i * img_bytes;
        const uint8_t* ib = imgB + (int64_t)i * img_bytes;
        oz::OzTile t;
        t.a = ia + oz::chunk_offset(nb, 0, rbA, 0);
        t.b = ib + oz::chunk_offset(nb, 0, rbB, 0) + 2048 * half;
        t.sa = reinterpret_cast<const double*>(ia + (int64_t)s * nb * nb) + rbA * 128;
        t.sb = reinterpret_cast<const double*>(ib + (int64_t)s * nb * nb) + rbB * 128 + half * 64;
        return t;
    };
    for (int r = 0; r < reps; ++r) oz::block_gemm(C, 128, src, ntiles, s, (int)(nb / 32), nb, smem, tmem);
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tc::tmem_dealloc(tmem, oz::TMEM_COLS);
}

static double frand(unsigned long long& st) {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    return ((st >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

int main(int argc, char** argv) {
    const int s = argc > 1 ? atoi(argv[1]) : 8;
    CK(cudaFuncSetAttribute(k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, oz::SMEM_BYTES));
    // ---- accuracy: nb = 256, 5 tiles, rows with wildly different scales
    {
        const int64_t nb = 256;
        const int nt = 5;
        const int64_t ib = oz::image_bytes(s, nb);
        std::vector<double> A(nt * nb * nb), B(nt * nb * nb);
        unsigned long long st = 12345;
        for (int n = 0; n < nt; ++n)
            for (int64_t c = 0; c < nb; ++c)
                for (int64_t r = 0; r < nb; ++r) {
                    const int ea = (int)((r * 7 + n * 3) % 41) - 20, eb = (int)((r * 5 + n * 11) % 37) - 18;
                    double va = frand(st), vb = frand(st);
                    if ((r + c) % 13 == 0) va *= 1e-9;  // small entries inside a row
                    A[n * nb * nb + r + c * nb] = ldexp(va, ea);
                    B[n * nb * nb + r + c * nb] = ldexp(vb, eb);
                }
        double *dA, *dB, *dC;
        uint8_t *iA, *iB;
        CK(cudaMalloc(&dA, sizeof(double) * A.size()));
        CK(cudaMalloc(&dB, sizeof(double) * B.size()));
        CK(cudaMalloc(&iA, ib * nt));
        CK(cudaMalloc(&iB, ib * nt));
        const int nblk = 2 * 4;  // rbA in {0,1}, hB in {0..3}
        CK(cudaMalloc(&dC, sizeof(double) * 128 * 64 * nblk));
        CK(cudaMemcpy(dA, A.data(), sizeof(double) * A.size(), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dB, B.data(), sizeof(double) * B.size(), cudaMemcpyHostToDevice));
        CK(cudaMemset(dC, 0, sizeof(double) * 128 * 64 * nblk));
        k_slice<<<nt, 256>>>(dA, nb, s, iA, ib);
        k_slice<<<nt, 256>>>(dB, nb, s, iB, ib);
        k_gemm<<<nblk, 128, oz::SMEM_BYTES>>>(dC, iA, iB, ib, nt, s, nb, 2, 1);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        std::vector<double> C(128 * 64 * nblk);
        CK(cudaMemcpy(C.data(), dC, sizeof(double) * C.size(), cudaMemcpyDeviceToHost));
        double worst = 0.0, worst_abs = 0.0;
        for (int blk = 0; blk < nblk; ++blk) {
            const int rbA = blk % 2, hB = blk / 2;
            for (int i = 0; i < 128; ++i)
                for (int j = 0; j < 64; ++j) {
                    long double ref = 0.0L, mag = 0.0L;
                    const int64_t ra = rbA * 128 + i, rb = hB * 64 + j;
                    for (int n = 0; n < nt; ++n)
                        for (int64_t c = 0; c < nb; ++c) {
                            long double a = A[n * nb * nb + ra + c * nb], b = B[n * nb * nb + rb + c * nb];
                            ref += a * b;
                            mag += fabsl(a * b);
                        }
                    const double got = -C[blk * 128 * 64 + i + j * 128];
                    const double err = (double)fabsl((long double)got - ref);
                    if (mag > 0 && err / (double)mag > worst) worst = err / (double)mag;
                    if (err > worst_abs) worst_abs = err;
                }
        }
        printf("accuracy s=%d: max |C - ref| / sum|a b| = %.3e  (2^-53 = 1.1e-16)\n", s, worst);
        cudaFree(dA), cudaFree(dB), cudaFree(dC), cudaFree(iA), cudaFree(iB);
    }
    // ---- throughput: nb = 1024, 8 tiles, 148 CTAs x reps
    {
        const int64_t nb = 1024;
        const int nt = 8, reps = 4;
        const int64_t ib = oz::image_bytes(s, nb);
        int nsm = 0;
        CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
        double *dX, *dC;
        uint8_t *iA, *iB;
        CK(cudaMalloc(&dX, sizeof(double) * nt * nb * nb));
        CK(cudaMalloc(&iA, ib * nt));
        CK(cudaMalloc(&iB, ib * nt));
        CK(cudaMalloc(&dC, sizeof(double) * 128 * 64 * nsm));
        std::vector<double> X(nt * nb * nb);
        unsigned long long st = 7;
        for (auto& v : X) v = frand(st);
        CK(cudaMemcpy(dX, X.data(), sizeof(double) * X.size(), cudaMemcpyHostToDevice));
        k_slice<<<nt, 256>>>(dX, nb, s, iA, ib);
        k_slice<<<nt, 256>>>(dX, nb, s, iB, ib);
        CK(cudaMemset(dC, 0, sizeof(double) * 128 * 64 * nsm));
        k_gemm<<<nsm, 128, oz::SMEM_BYTES>>>(dC, iA, iB, ib, nt, s, nb, 8, 1);
        CK(cudaDeviceSynchronize());
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0), cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_gemm<<<nsm, 128, oz::SMEM_BYTES>>>(dC, iA, iB, ib, nt, s, nb, 8, reps);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double blocks = (double)nsm * reps;
        const double f64 = blocks * 2.0 * 128 * 64 * nt * nb;  // emulated FP64 flops
        const double i8 = f64 * s * (s + 1) / 2;               // int8 ops issued
        printf("throughput s=%d: %.3f ms  FP64-equivalent %.1f TF/s  int8 %.0f TOPS  (CTAs %d x %d reps, K=%lld)\n", s,
               ms, f64 / ms / 1e9, i8 / ms / 1e9, nsm, reps, (long long)(nt * nb));
    }
    return 0;
}
