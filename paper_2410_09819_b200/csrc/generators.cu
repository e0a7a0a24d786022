// generators.cu -- AUX device generators for the synthetic inputs.
// Same counter hash as workloads/__init__.py (splitmix64 finaliser), so the
// device matrix is bit-identical to the host one; no method arithmetic here.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/mxp_chol.h"
#include "internal.h"

namespace {
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__global__ void k_gen_plgsy(int64_t n, uint64_t s, double* A, int64_t lda) {
    const int64_t j = blockIdx.y + (int64_t)blockIdx.z * gridDim.y;
    if (j >= n) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t hi = i > j ? i : j, lo = i > j ? j : i;
        uint64_t x = mix64(((hi << 32) | lo) ^ s);
        double v = (double)(x >> 11) * 0x1p-53 - 0.5;
        if (i == j) v += (double)n;
        A[i + j * lda] = v;
    }
}

__global__ void k_gen_kms(int64_t n, double rho, double* A, int64_t lda) {
    const int64_t j = blockIdx.y + (int64_t)blockIdx.z * gridDim.y;
    if (j >= n) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t e = i > j ? i - j : j - i;
        // rho^e by binary exponentiation, low bit first (same sequence as
        // workloads.pow_by_squaring, so host and device agree bitwise)
        double out = 1.0, base = rho;
        while (e > 0) {
            if (e & 1) out = out * base;
            e >>= 1;
            if (e > 0) base = base * base;
        }
        A[i + j * lda] = out;
    }
}

__global__ void k_gen_matern(int64_t n, const double* __restrict__ xy, double sigma2, double a, double nugget,
                             double* A, int64_t lda) {
    const int64_t j = blockIdx.y + (int64_t)blockIdx.z * gridDim.y;
    if (j >= n) return;
    const double xj = xy[2 * j], yj = xy[2 * j + 1];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double dx = xy[2 * i] - xj, dy = xy[2 * i + 1] - yj;
        const double h = sqrt(dx * dx + dy * dy);
        double v = sigma2 * exp(-h / a);
        if (i == j) v += nugget;
        A[i + j * lda] = v;
    }
}

void grid_for(int64_t n, dim3& g) {
    unsigned gy = (unsigned)(n < 65535 ? n : 65535);
    unsigned gz = (unsigned)((n + gy - 1) / gy);
    unsigned gx = (unsigned)((n + 255) / 256);
    if (gx > 64) gx = 64;
    g = dim3(gx, gy, gz);
}
}  // namespace

extern "C" int mxp_generate_plgsy_device(int64_t n, uint64_t seed, double* A, int64_t lda, void* stream) {
    if (n < 1) return -1;
    if (!A) return -3;
    if (lda < n) return -4;
    uint64_t s = seed + 0x9E3779B97F4A7C15ull;
    s = (s ^ (s >> 30)) * 0xBF58476D1CE4E5B9ull;
    s = (s ^ (s >> 27)) * 0x94D049BB133111EBull;
    s = s ^ (s >> 31);
    dim3 g;
    grid_for(n, g);
    MXP_CARVEOUT_MAX(k_gen_plgsy);
    k_gen_plgsy<<<g, 256, 0, (cudaStream_t)stream>>>(n, s, A, lda);
    return cudaGetLastError() == cudaSuccess ? MXP_OK : MXP_ECUDA;
}

extern "C" int mxp_generate_kms_device(int64_t n, double rho, double* A, int64_t lda, void* stream) {
    if (n < 1) return -1;
    if (!A) return -3;
    if (lda < n) return -4;
    dim3 g;
    grid_for(n, g);
    MXP_CARVEOUT_MAX(k_gen_kms);
    k_gen_kms<<<g, 256, 0, (cudaStream_t)stream>>>(n, rho, A, lda);
    return cudaGetLastError() == cudaSuccess ? MXP_OK : MXP_ECUDA;
}

extern "C" int mxp_generate_matern_device(int64_t n, const double* xy_dev, double sigma2, double range_a,
                                          double nugget, double* A, int64_t lda, void* stream) {
    if (n < 1) return -1;
    if (!xy_dev) return -2;
    if (!(sigma2 > 0.0)) return -3;
    if (!(range_a > 0.0)) return -4;
    if (!(nugget >= 0.0)) return -5;
    if (!A) return -6;
    if (lda < n) return -7;
    dim3 g;
    grid_for(n, g);
    MXP_CARVEOUT_MAX(k_gen_matern);
    k_gen_matern<<<g, 256, 0, (cudaStream_t)stream>>>(n, xy_dev, sigma2, range_a, nugget, A, lda);
    return cudaGetLastError() == cudaSuccess ? MXP_OK : MXP_ECUDA;
}

namespace mxp {
// (see preload_sched in sched_f64.cu)
void preload_generators() {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void*)k_gen_plgsy);
    cudaFuncGetAttributes(&fa, (const void*)k_gen_kms);
    cudaFuncGetAttributes(&fa, (const void*)k_gen_matern);
    cudaGetLastError();
}
}  // namespace mxp
