// solve.cu -- forward substitution L z = y on the resident tile factor and the
// Gaussian log-likelihood (Eq. 1, the
// quadratic form y^T Sigma^-1 y = ||z||^2 with L z = y).
//
// HBM-bound: every lower tile of L is read once (nb^2 * 8 bytes per tile,
// n^2/2 * 8 bytes in all).  One persistent kernel walks a fixed task order
// with a ticket, like the factorization's static schedule:
//   for k:  DIAG(k)                      z_k = L_kk^-1 (y_k - sum_{j<k} P(k,j))
//           GEMV(m, k, rb), m > k         P(m,k)[rows rb] = L_mk[rows rb, :] z_k
// DIAG(k) waits for the GEMV blocks of its row (pdone[k] = k * nb/128), GEMV(., k)
// for z_k (zready[k]); each partial P(m,k) is written once and summed in
// ascending k, so the result is bitwise reproducible and no two tasks write the
// same word -- the GEMVs of a column overlap the following diagonal solves.
// DIAG blocks by 128 with the inverses W_J = L_JJ^-1 the POTRF left in wbuf.
#include <algorithm>
#include <vector>

#include "internal.h"

namespace mxp {
namespace {

constexpr uint64_t SOLVE_TIMEOUT_NS = 20ull * 1000 * 1000 * 1000;

__device__ __forceinline__ int ld_acq(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// thread 0 waits for *f >= target; false on timeout (error flag set)
__device__ bool wait_ge(const int* f, int target, int* err) {
    if (ld_acq(f) >= target) return true;
    const uint64_t t0 = gtimer();
    unsigned ns = 32;
    while (ld_acq(f) < target) {
        if (*(volatile int*)err) return false;
        if (gtimer() - t0 > SOLVE_TIMEOUT_NS) {
            atomicExch(err, 1);
            return false;
        }
        __nanosleep(ns);
        if (ns < 1024) ns *= 2;
    }
    return true;
}

struct SolveArgs {
    const double* pool;
    const int32_t* slot;
    const double* wbuf;
    int64_t Nt, nb;
    const double* y;        // [Nt*nb], zero padded
    double* z;              // [Nt*nb]
    double* P;              // [T][nb] partial products (off-diagonal tiles)
    int* zready;            // [Nt]
    int* pdone;             // [Nt]
    int* counter;
    int* err;
    const int* colstart;    // [Nt+1] first ticket of column k
};

// P(m,k)[128 rows] = L(m,k)[rows, :] z_k
__device__ void task_gemv(const SolveArgs& a, int64_t m, int64_t k, int64_t rb, double* sz, double* part) {
    const int64_t nb = a.nb;
    for (int64_t c = threadIdx.x; c < nb; c += blockDim.x) sz[c] = __ldcg(a.z + k * nb + c);
    __syncthreads();
    const int row = threadIdx.x & 127, h = threadIdx.x >> 7;
    const double* L = a.pool + (int64_t)a.slot[tile_index(a.Nt, m, k)] * nb * nb + rb * 128 + row;
    const int64_t c0 = h * (nb / 2), c1 = c0 + nb / 2;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;  // 4 chains, 8 loads in flight per thread
#pragma unroll 2
    for (int64_t c = c0; c < c1; c += 4) {
        s0 = fma(__ldcs(L + c * nb), sz[c], s0);
        s1 = fma(__ldcs(L + (c + 1) * nb), sz[c + 1], s1);
        s2 = fma(__ldcs(L + (c + 2) * nb), sz[c + 2], s2);
        s3 = fma(__ldcs(L + (c + 3) * nb), sz[c + 3], s3);
    }
    part[threadIdx.x] = (s0 + s1) + (s2 + s3);
    __syncthreads();
    if (h == 0) __stcg(a.P + tile_index(a.Nt, m, k) * nb + rb * 128 + row, part[row] + part[row + 128]);
}

// z_k = L_kk^-1 (y_k - sum_{j<k} P(k,j)):  per 128 block J: s = r_J - L[J, <J] z_<J;  z_J = W_J s
__device__ void task_diag(const SolveArgs& a, int64_t k, double* sz, double* part) {
    const int64_t nb = a.nb, S = nb / 128, Nt = a.Nt;
    double* s = sz + nb;
    for (int64_t i = threadIdx.x; i < nb; i += blockDim.x) {  // r_k in sz (ascending j: deterministic)
        double r = a.y[k * nb + i];
        for (int64_t j = 0; j < k; ++j) r -= __ldcg(a.P + tile_index(Nt, k, j) * nb + i);
        sz[i] = r;
    }
    __syncthreads();
    const int row = threadIdx.x & 127, h = threadIdx.x >> 7;
    const double* Lkk = a.pool + (int64_t)a.slot[tile_index(Nt, k, k)] * nb * nb;
    for (int64_t J = 0; J < S; ++J) {
        const double* LJ = Lkk + J * 128 + row;
        const int64_t half = J * 64;  // columns [0, 128J) in two halves
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 2
        for (int64_t c = h * half; c < (h + 1) * half; c += 4) {
            a0 = fma(__ldcs(LJ + c * nb), sz[c], a0);
            a1 = fma(__ldcs(LJ + (c + 1) * nb), sz[c + 1], a1);
            a2 = fma(__ldcs(LJ + (c + 2) * nb), sz[c + 2], a2);
            a3 = fma(__ldcs(LJ + (c + 3) * nb), sz[c + 3], a3);
        }
        part[threadIdx.x] = (a0 + a1) + (a2 + a3);
        __syncthreads();
        if (h == 0) s[row] = sz[J * 128 + row] - (part[row] + part[row + 128]);
        __syncthreads();
        const double* W = a.wbuf + (k * S + J) * (128 * 128);  // column-major, lower triangular
        double b0 = 0.0;
        const int kk0 = h == 0 ? 0 : (row + 1) / 2, kk1 = h == 0 ? (row + 1) / 2 : row + 1;
        for (int kk = kk0; kk < kk1; ++kk) b0 = fma(W[row + kk * 128], s[kk], b0);
        part[threadIdx.x] = b0;
        __syncthreads();
        if (h == 0) sz[J * 128 + row] = part[row] + part[row + 128];
        __syncthreads();
    }
    for (int64_t c = threadIdx.x; c < nb; c += blockDim.x) __stcg(a.z + k * nb + c, sz[c]);
}

__global__ void __launch_bounds__(256) k_fsolve(const SolveArgs a) {
    extern __shared__ double sm[];  // z_k or r_k (nb) | s (128) | partials (256)
    double* part = sm + a.nb + 128;
    __shared__ int s_t, s_ok;
    const int64_t Nt = a.Nt, RB = a.nb / 128;
    const int total = a.colstart[Nt];
    while (true) {
        if (threadIdx.x == 0) s_t = atomicAdd(a.counter, 1);
        __syncthreads();
        const int t = s_t;
        __syncthreads();
        if (t >= total) break;
        int64_t k = 0;
        while (a.colstart[k + 1] <= t) ++k;
        const int64_t i = t - a.colstart[k];
        if (i == 0) {  // DIAG(k)
            if (threadIdx.x == 0) s_ok = wait_ge(a.pdone + k, (int)(k * RB), a.err);
            __syncthreads();
            if (s_ok) {
                task_diag(a, k, sm, part);
                __threadfence();
                __syncthreads();
                if (threadIdx.x == 0) atomicExch(a.zready + k, 1);  // (after the fence: release)
            }
        } else {  // GEMV(m, k, rb)
            const int64_t m = k + 1 + (i - 1) / RB, rb = (i - 1) % RB;
            if (threadIdx.x == 0) s_ok = wait_ge(a.zready + k, 1, a.err);
            __syncthreads();
            if (s_ok) {
                task_gemv(a, m, k, rb, sm, part);
                __threadfence();
                __syncthreads();
                if (threadIdx.x == 0) atomicAdd(a.pdone + m, 1);
            }
        }
        __syncthreads();
    }
}

// out = sum z_i^2 over i < n (fixed-order tree in one CTA)
__global__ void __launch_bounds__(1024) k_sumsq(const double* __restrict__ z, int64_t n, double* out) {
    __shared__ double red[1024];
    double a = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) a = fma(z[i], z[i], a);
    red[threadIdx.x] = a;
    __syncthreads();
    for (int w = 512; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0];
}

}  // namespace

size_t forward_solve_work_bytes(int64_t Nt, int64_t nb) {
    const int64_t T = Nt * (Nt + 1) / 2;
    return sizeof(double) * (size_t)(T * nb) + sizeof(int) * (size_t)(2 * Nt + 4 + Nt + 1);
}

// r: y padded to Nt*nb (read only here); work: forward_solve_work_bytes(Nt, nb) bytes
int launch_forward_solve(const double* pool, const int32_t* slot, const double* wbuf, int64_t Nt, int64_t nb,
                         double* r, double* z, void* work, cudaStream_t s) {
    const int64_t T = Nt * (Nt + 1) / 2, RB = nb / 128;
    double* P = reinterpret_cast<double*>(work);
    int* flags = reinterpret_cast<int*>(P + T * nb);  // zready[Nt] | pdone[Nt] | counter | err | pad | colstart
    int* colstart = flags + 2 * Nt + 4;
    static thread_local std::vector<int> cs;
    cs.assign(Nt + 1, 0);
    for (int64_t k = 0; k < Nt; ++k) cs[k + 1] = cs[k] + 1 + (int)((Nt - k - 1) * RB);
    if (cudaMemsetAsync(flags, 0, sizeof(int) * (2 * Nt + 4), s) != cudaSuccess) return -1;
    if (cudaMemcpyAsync(colstart, cs.data(), sizeof(int) * (Nt + 1), cudaMemcpyHostToDevice, s) != cudaSuccess)
        return -1;
    const size_t smem = sizeof(double) * (nb + 128 + 256);
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(k_fsolve, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        configured = true;
    }
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fsolve, 256, smem);
    SolveArgs a{pool, slot, wbuf, Nt, nb, r, z, P, flags, flags + Nt, flags + 2 * Nt, flags + 2 * Nt + 1, colstart};
    const int grid = std::max(1, std::min(occ, 4)) * nsm;  // all resident (the ticket order needs it)
    k_fsolve<<<grid, 256, smem, s>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

// the solve's error flag (1 = a wait timed out)
const int* forward_solve_err(void* work, int64_t Nt, int64_t nb) {
    const int64_t T = Nt * (Nt + 1) / 2;
    return reinterpret_cast<const int*>(reinterpret_cast<double*>(work) + T * nb) + 2 * Nt + 1;
}

void launch_sumsq(const double* z, int64_t n, double* out, cudaStream_t s) { k_sumsq<<<1, 1024, 0, s>>>(z, n, out); }

}  // namespace mxp
