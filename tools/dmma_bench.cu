// dmma_bench.cu -- dev microbenchmark: FP64 DMMA GEMM tile configurations on
// B200 (C -= A B^T, column-major panels like the chain kernel).  Not product code.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_bench tools/dmma_bench.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>
#include <vector>

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// PERM: rows of a warp tile permuted so a lane's MI fragments are contiguous
// (row = g*MI + mi) -> LDS.128 loads two fragments at once.
template <int BM, int BN, int WM, int WN, int BK, int STAGES, int MINB, bool PERM>
struct K {
    static constexpr int THREADS = WM * WN * 32;
    static constexpr int WTM = BM / WM, WTN = BN / WN, MI = WTM / 8, NI = WTN / 8;
    static constexpr int PAD = PERM ? 2 : 4;
    static constexpr int LDA_S = BM + PAD, LDB_S = BN + PAD;
    static constexpr int STAGE = BK * (LDA_S + LDB_S);
    static constexpr int SMEM = STAGES * STAGE * 8;
};

template <int BM, int BN, int WM, int WN, int BK, int STAGES, int MINB, bool PERM>
__global__ void __launch_bounds__(WM * WN * 32, MINB)
gemm(const double* __restrict__ A, const double* __restrict__ B, double* C, int M, int N, int Kd, int ld) {
    using C_ = K<BM, BN, WM, WN, BK, STAGES, MINB, PERM>;
    extern __shared__ __align__(16) double smem[];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int wm = warp / WN, wn = warp % WN, g = lane >> 2, q = lane & 3;
    const int row0 = blockIdx.x * BM, col0 = blockIdx.y * BN;
    double acc[C_::MI][C_::NI][2];
#pragma unroll
    for (int i = 0; i < C_::MI; ++i)
#pragma unroll
        for (int j = 0; j < C_::NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int nk = Kd / BK;
    auto load = [&](int st, int it) {
        double* sA = smem + st * C_::STAGE;
        double* sB = sA + BK * C_::LDA_S;
        const double* pa = A + row0 + (int64_t)it * BK * ld;
        const double* pb = B + col0 + (int64_t)it * BK * ld;
        constexpr int AC = BK * BM / 2, BC = BK * BN / 2;
#pragma unroll
        for (int c = t; c < AC; c += C_::THREADS) {
            int col = c / (BM / 2), r2 = (c % (BM / 2)) * 2;
            cp_async16(sA + col * C_::LDA_S + r2, pa + (int64_t)col * ld + r2);
        }
#pragma unroll
        for (int c = t; c < BC; c += C_::THREADS) {
            int col = c / (BN / 2), r2 = (c % (BN / 2)) * 2;
            cp_async16(sB + col * C_::LDB_S + r2, pb + (int64_t)col * ld + r2);
        }
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nk) load(s, s);
        cp_async_commit();
    }
    for (int it = 0; it < nk; ++it) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        int nxt = it + STAGES - 1;
        if (nxt < nk) load(nxt % STAGES, nxt);
        cp_async_commit();
        const double* sA = smem + (it % STAGES) * C_::STAGE;
        const double* sB = sA + BK * C_::LDA_S;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double a[C_::MI], b[C_::NI];
            if (PERM) {
                const double2* pa = (const double2*)(sA + (kk + q) * C_::LDA_S + wm * C_::WTM + g * C_::MI);
                const double2* pb = (const double2*)(sB + (kk + q) * C_::LDB_S + wn * C_::WTN + g * C_::NI);
#pragma unroll
                for (int i = 0; i < C_::MI / 2; ++i) { double2 v = pa[i]; a[2 * i] = v.x; a[2 * i + 1] = v.y; }
#pragma unroll
                for (int i = 0; i < C_::NI / 2; ++i) { double2 v = pb[i]; b[2 * i] = v.x; b[2 * i + 1] = v.y; }
            } else {
                const double* pa = sA + (kk + q) * C_::LDA_S + wm * C_::WTM + g;
                const double* pb = sB + (kk + q) * C_::LDB_S + wn * C_::WTN + g;
#pragma unroll
                for (int i = 0; i < C_::MI; ++i) a[i] = pa[i * 8];
#pragma unroll
                for (int i = 0; i < C_::NI; ++i) b[i] = pb[i * 8];
            }
#pragma unroll
            for (int i = 0; i < C_::MI; ++i)
#pragma unroll
                for (int j = 0; j < C_::NI; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
    }
    cp_async_wait<0>();
#pragma unroll
    for (int i = 0; i < C_::MI; ++i)
#pragma unroll
        for (int j = 0; j < C_::NI; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                int r, c;
                if (PERM) { r = wm * C_::WTM + g * C_::MI + i; c = wn * C_::WTN + (2 * q + e) * C_::NI + j; }
                else { r = wm * C_::WTM + i * 8 + g; c = wn * C_::WTN + j * 8 + 2 * q + e; }
                double* p = C + (row0 + r) + (int64_t)(col0 + c) * ld;
                *p = *p - acc[i][j][e];
            }
}

template <int BM, int BN, int WM, int WN, int BK, int STAGES, int MINB, bool PERM>
void run(const char* name, const double* A, const double* B, double* C, int M, int N, int Kd, int ld,
         const double* Cref) {
    using C_ = K<BM, BN, WM, WN, BK, STAGES, MINB, PERM>;
    auto kern = gemm<BM, BN, WM, WN, BK, STAGES, MINB, PERM>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM) != cudaSuccess) {
        printf("%-40s smem %d too big\n", name, C_::SMEM);
        cudaGetLastError();
        return;
    }
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, C_::THREADS, C_::SMEM);
    dim3 grid(M / BM, N / BN);
    cudaMemset(C, 0, sizeof(double) * (size_t)ld * N);
    kern<<<grid, C_::THREADS, C_::SMEM>>>(A, B, C, M, N, Kd, ld);
    cudaDeviceSynchronize();
    // correctness vs the reference variant
    std::vector<double> h(8), r(8);
    double maxd = 0;
    if (Cref) {
        std::vector<double> hc((size_t)ld * 64), rc((size_t)ld * 64);
        cudaMemcpy(hc.data(), C, sizeof(double) * hc.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(rc.data(), Cref, sizeof(double) * rc.size(), cudaMemcpyDeviceToHost);
        for (size_t i = 0; i < hc.size(); ++i) { double d = fabs(hc[i] - rc[i]); if (d > maxd) maxd = d; }
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        kern<<<grid, C_::THREADS, C_::SMEM>>>(A, B, C, M, N, Kd, ld);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    double tf = 2.0 * M * N * (double)Kd / (best / 1e3) / 1e12;
    printf("%-44s occ=%d smem=%6d  %7.3f ms  %6.2f TF/s  maxdiff=%.2e  %s\n", name, occ, C_::SMEM, best, tf, maxd,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int M = 148 * 64 > 8192 ? 9472 : 8192;  // multiple of 128 and 256: 9472 = 74*128
    const int N = 8192, Kd = 8192, ld = 9472;
    double *A, *B, *C, *Cref;
    cudaMalloc(&A, sizeof(double) * (size_t)ld * Kd);
    cudaMalloc(&B, sizeof(double) * (size_t)ld * Kd);
    cudaMalloc(&C, sizeof(double) * (size_t)ld * N);
    cudaMalloc(&Cref, sizeof(double) * (size_t)ld * N);
    std::vector<double> h((size_t)ld * Kd);
    for (size_t i = 0; i < h.size(); ++i) h[i] = ((i * 2654435761u) % 1000) / 1000.0 - 0.5;
    cudaMemcpy(A, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
    for (size_t i = 0; i < h.size(); ++i) h[i] = ((i * 40503u + 7) % 997) / 997.0 - 0.5;
    cudaMemcpy(B, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
    printf("M=%d N=%d K=%d\n", M, N, Kd);
    run<128, 128, 2, 4, 16, 4, 1, false>("128x128 w2x4 bk16 s4 (current)", A, B, Cref, M, N, Kd, ld, nullptr);
    run<128, 128, 2, 4, 16, 4, 1, true>("128x128 w2x4 bk16 s4 perm", A, B, C, M, N, Kd, ld, Cref);
    run<128, 128, 4, 4, 16, 3, 1, false>("128x128 w4x4 bk16 s3", A, B, C, M, N, Kd, ld, Cref);
    run<128, 128, 4, 4, 16, 3, 1, true>("128x128 w4x4 bk16 s3 perm", A, B, C, M, N, Kd, ld, Cref);
    run<128, 64, 4, 2, 16, 3, 2, false>("128x64 w4x2 bk16 s3 2cta", A, B, C, M, N, Kd, ld, Cref);
    run<128, 64, 4, 2, 16, 3, 2, true>("128x64 w4x2 bk16 s3 2cta perm", A, B, C, M, N, Kd, ld, Cref);
    run<64, 128, 2, 2, 16, 3, 3, false>("64x128 w2x2 bk16 s3 (cutlass-like)", A, B, C, M, N, Kd, ld, Cref);
    run<64, 128, 2, 2, 16, 3, 3, true>("64x128 w2x2 bk16 s3 perm", A, B, C, M, N, Kd, ld, Cref);
    run<64, 128, 2, 2, 16, 4, 2, true>("64x128 w2x2 bk16 s4 perm occ2", A, B, C, M, N, Kd, ld, Cref);
    run<128, 128, 2, 2, 16, 3, 2, true>("128x128 w2x2 bk16 s3 perm", A, B, C, M, N, Kd, ld, Cref);
    run<128, 128, 2, 4, 32, 3, 1, true>("128x128 w2x4 bk32 s3 perm", A, B, C, M, N, Kd, ld, Cref);
    run<256, 128, 4, 4, 16, 3, 1, true>("256x128 w4x4 bk16 s3 perm", A, B, C, M, N, Kd, ld, Cref);
    run<128, 256, 4, 4, 16, 3, 1, true>("128x256 w4x4 bk16 s3 perm", A, B, C, M, N, Kd, ld, Cref);
    run<64, 64, 2, 2, 16, 4, 4, true>("64x64 w2x2 bk16 s4 perm occ4", A, B, C, M, N, Kd, ld, Cref);
    run<128, 64, 2, 2, 16, 4, 3, true>("128x64 w2x2 bk16 s4 perm occ3", A, B, C, M, N, Kd, ld, Cref);
    return 0;
}
