// engine.cu -- host runtime of the B200 engine and the C ABI (include/mxp_chol.h).
//
// Static schedule (Alg. 1): tasks are enumerated column
// by column; the dependency table `Ready` of the paper becomes CUDA events
// between two streams:
//   stream U ("update", normal priority):  bulk GEMM chain of column k over
//       n in [0, k-1)  -- waits Ready(column k-2)
//   stream P ("panel", high priority):     last chain term n = k-1, POTRF(k),
//       TRSM(column k) -- waits the bulk of column k; records Ready(column k)
// so column k's latency-bound panel runs under column k+1's bulk update
// (lookahead).  The split of the chain into [0,k-1) + {k-1} and the split-K
// chunking are functions of (k, Nt, nb) only, so the result is bitwise
// identical with or without lookahead, for any stream timing.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mxp_chol.h"
#include "internal.h"

using namespace mxp;

namespace {
thread_local std::string g_last_error;

struct CudaError {
    cudaError_t e;
};

#define CK(expr)                                                                             \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess) {                                                             \
            g_last_error = std::string(#expr) + ": " + cudaGetErrorString(_e);               \
            throw CudaError{_e};                                                             \
        }                                                                                    \
    } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
}  // namespace

struct mxp_plan_s {
    int64_t n = 0, nb = 0, Nt = 0, T = 0;
    std::vector<uint8_t> map;
    int device = 0;
    cudaStream_t user_stream = 0;
    int64_t hbm_cap = 0;
    int64_t splitk_tiles = 16;
    int lookahead = 1;
    int debug_sync = 0;

    // workspace
    char* ws = nullptr;
    size_t ws_bytes = 0;
    bool ws_owned = false;
    int64_t* d_info = nullptr;
    double* d_logdet = nullptr;
    double* d_logdet_parts = nullptr;
    int32_t* d_slot = nullptr;
    double* d_partial = nullptr;
    double* pool = nullptr;
    size_t partial_doubles = 0;

    bool streams_ready = false;
    cudaStream_t sU = 0, sP = 0;
    std::vector<cudaEvent_t> ev_panel, ev_bulk;
    cudaEvent_t ev_start = nullptr, ev_done = nullptr;

    int64_t launches = 0, h2d = 0, d2h = 0;
    int profile = 0;
    struct Rec {
        int cls;
        cudaEvent_t a, b;
        double flops;
        int64_t n;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    int64_t st_launch[4] = {0, 0, 0, 0};
    double st_ms[4] = {0, 0, 0, 0}, st_flops[4] = {0, 0, 0, 0};
    bool have_result = false;
    double logdet = 0.0;

    ~mxp_plan_s();
};

mxp_plan_s::~mxp_plan_s() {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    if (ws_owned && ws) cudaFree(ws);
    for (auto e : ev_panel) cudaEventDestroy(e);
    for (auto e : ev_bulk) cudaEventDestroy(e);
    for (auto e : ev_pool) cudaEventDestroy(e);
    if (ev_start) cudaEventDestroy(ev_start);
    if (ev_done) cudaEventDestroy(ev_done);
    if (sU) cudaStreamDestroy(sU);
    if (sP) cudaStreamDestroy(sP);
    cudaSetDevice(cur);
}

namespace {

// Split-K chunking of the bulk chain of column k: a function of (k, Nt, nb)
// only (never of the GPU count or timing), so results are reproducible.
void bulk_chunks(const mxp_plan_s* p, int64_t k, int64_t& nchunks, int64_t& chunk_tiles) {
    int64_t nterms = k - 1;  // n in [0, k-1)
    if (nterms <= 0) {
        nchunks = 0;
        chunk_tiles = 1;
        return;
    }
    const int64_t S = p->nb / 128;
    int64_t blocks = (p->Nt - k) * S * S;
    const int64_t target = 2 * 148;
    int64_t want = blocks >= target ? 1 : (target + blocks - 1) / blocks;
    int64_t maxc = (nterms + p->splitk_tiles - 1) / p->splitk_tiles;  // at most this many
    want = std::min(want, std::max<int64_t>(1, std::min(maxc * 4, nterms)));
    chunk_tiles = (nterms + want - 1) / want;
    nchunks = (nterms + chunk_tiles - 1) / chunk_tiles;
}

size_t partial_need(const mxp_plan_s* p) {
    const int64_t S = p->nb / 128;
    size_t best = 0;
    for (int64_t k = 1; k < p->Nt; ++k) {
        int64_t nch, ct;
        bulk_chunks(p, k, nch, ct);
        if (nch > 1) best = std::max(best, (size_t)((p->Nt - k) * S * S * nch) * 128 * 128);
    }
    return best;
}

size_t workspace_need(const mxp_plan_s* p, size_t* pool_off, size_t* partial_off, size_t* slot_off) {
    size_t off = 0;
    off += 256;                                   // info
    off += align_up(sizeof(double) * (p->Nt + 2), 256);  // logdet + parts
    *slot_off = off;
    off += align_up(sizeof(int32_t) * p->T, 256);
    *partial_off = off;
    off += align_up(sizeof(double) * partial_need(p), 256);
    *pool_off = off;
    off += sizeof(double) * (size_t)p->T * p->nb * p->nb;
    return off;
}

void bind_workspace(mxp_plan_s* p) {
    size_t pool_off, partial_off, slot_off;
    size_t need = workspace_need(p, &pool_off, &partial_off, &slot_off);
    if (!p->ws) {
        void* ptr = nullptr;
        cudaError_t e = cudaMalloc(&ptr, need);
        if (e != cudaSuccess) {
            cudaGetLastError();
            g_last_error = std::string("cudaMalloc workspace: ") + cudaGetErrorString(e);
            throw CudaError{cudaErrorMemoryAllocation};
        }
        p->ws = (char*)ptr;
        p->ws_bytes = need;
        p->ws_owned = true;
    }
    p->d_info = (int64_t*)p->ws;
    p->d_logdet = (double*)(p->ws + 256);
    p->d_logdet_parts = p->d_logdet + 1;
    p->d_slot = (int32_t*)(p->ws + slot_off);
    p->d_partial = (double*)(p->ws + partial_off);
    p->pool = (double*)(p->ws + pool_off);
    p->partial_doubles = partial_need(p);
}

void ensure_streams(mxp_plan_s* p) {
    if (p->streams_ready) return;
    int lo, hi;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&p->sU, cudaStreamNonBlocking, lo));
    CK(cudaStreamCreateWithPriority(&p->sP, cudaStreamNonBlocking, hi));
    p->ev_panel.resize(p->Nt);
    p->ev_bulk.resize(p->Nt);
    for (int64_t k = 0; k < p->Nt; ++k) {
        CK(cudaEventCreateWithFlags(&p->ev_panel[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&p->ev_bulk[k], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming));
    configure_kernels();
    p->streams_ready = true;
}

void dbg(mxp_plan_s* p, cudaStream_t s, const char* what) {
    CK(cudaGetLastError());
    if (p->debug_sync) {
        cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
            throw CudaError{e};
        }
    }
}

// ---- launch profiling (MXP_ATTR_PROFILE): CUDA events on the launching stream
cudaEvent_t next_event(mxp_plan_s* p) {
    if (p->ev_used == p->ev_pool.size()) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        p->ev_pool.push_back(e);
    }
    return p->ev_pool[p->ev_used++];
}
struct Prof {
    mxp_plan_s* p;
    cudaStream_t s;
    int cls;
    double flops;
    int64_t nlaunch;
    cudaEvent_t a = nullptr;
    Prof(mxp_plan_s* p_, cudaStream_t s_, int cls_, double flops_, int64_t n_ = 1)
        : p(p_), s(s_), cls(cls_), flops(flops_), nlaunch(n_) {
        if (p->profile) {
            a = next_event(p);
            CK(cudaEventRecord(a, s));
        }
    }
    ~Prof() noexcept(false) {
        if (p->profile) {
            cudaEvent_t b = next_event(p);
            CK(cudaEventRecord(b, s));
            p->recs.push_back({cls, a, b, flops, nlaunch});
        }
    }
};
void prof_reset(mxp_plan_s* p) {
    p->recs.clear();
    p->ev_used = 0;
    for (int c = 0; c < 4; ++c) p->st_launch[c] = 0, p->st_ms[c] = 0, p->st_flops[c] = 0;
}
void prof_collect(mxp_plan_s* p) {
    for (auto& r : p->recs) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, r.a, r.b));
        p->st_ms[r.cls] += ms;
        p->st_flops[r.cls] += r.flops;
        p->st_launch[r.cls] += r.n;
    }
    p->recs.clear();
}

// In-core FP64 factorization of the tiles already packed in the pool.
// Streams sU / sP must already be ordered after the packing.
void factor_incore_f64(mxp_plan_s* p) {
    const int64_t Nt = p->Nt, nb = p->nb;
    cudaStream_t sU = p->lookahead ? p->sU : p->sP;
    cudaStream_t sP = p->sP;
    for (int64_t k = 0; k < Nt; ++k) {
        // ---- bulk chain of column k on U: n in [0, k-1), rows m in [k, Nt)
        if (k >= 2 && p->lookahead) CK(cudaStreamWaitEvent(sU, p->ev_panel[k - 2], 0));
        int64_t nch, ct;
        bulk_chunks(p, k, nch, ct);
        if (nch > 0) {
            ChainArgs a{};
            a.pool = p->pool;
            a.slot = p->d_slot;
            a.dinfo = p->d_info;
            a.partial = p->d_partial;
            a.Nt = Nt;
            a.nb = nb;
            a.k = k;
            a.m0 = k;
            a.mstride = 1;
            a.mcount = Nt - k;
            a.n0 = 0;
            a.n1 = k - 1;
            a.nchunks = nch;
            a.chunk_tiles = ct;
            const double nb3 = (double)nb * nb * nb;
            {
                Prof pr(p, sU, MXP_KCLASS_CHAIN, (double)(k - 1) * (2.0 * nb3 * (Nt - k - 1) + nb3),
                        nch > 1 ? 2 : 1);
                launch_chain_f64(a, sU);
                ++p->launches;
                dbg(p, sU, "chain bulk");
                if (nch > 1) {
                    launch_reduce_partials(a, sU);
                    ++p->launches;
                    dbg(p, sU, "reduce");
                }
            }
        }
        CK(cudaEventRecord(p->ev_bulk[k], sU));
        // ---- panel of column k on P
        CK(cudaStreamWaitEvent(sP, p->ev_bulk[k], 0));
        if (k >= 1) {
            ChainArgs a{};
            a.pool = p->pool;
            a.slot = p->d_slot;
            a.dinfo = p->d_info;
            a.partial = p->d_partial;
            a.Nt = Nt;
            a.nb = nb;
            a.k = k;
            a.m0 = k;
            a.mstride = 1;
            a.mcount = Nt - k;
            a.n0 = k - 1;
            a.n1 = k;
            a.nchunks = 1;
            a.chunk_tiles = 1;
            const double nb3 = (double)nb * nb * nb;
            Prof pr(p, sP, MXP_KCLASS_CHAIN, 2.0 * nb3 * (Nt - k - 1) + nb3);
            launch_chain_f64(a, sP);
            ++p->launches;
            dbg(p, sP, "chain last");
        }
        {
            PotrfArgs pa{p->pool, p->d_slot, p->d_info, Nt, nb, k};
            const int S = (int)(nb / 128);
            Prof pr(p, sP, MXP_KCLASS_POTRF, (double)nb * nb * nb / 3.0, 3 * S - 2);
            p->launches += launch_potrf_tile_f64(pa, sP);
            dbg(p, sP, "potrf");
        }
        if (k + 1 < Nt) {
            TrsmArgs ta{p->pool, p->d_slot, p->d_info, Nt, nb, k, k + 1, 1, Nt - k - 1};
            Prof pr(p, sP, MXP_KCLASS_TRSM, (double)nb * nb * nb * (Nt - k - 1));
            launch_trsm_f64(ta, sP);
            ++p->launches;
            dbg(p, sP, "trsm");
        }
        CK(cudaEventRecord(p->ev_panel[k], sP));
    }
    if (p->lookahead) {
        // U has nothing left after the final panel; make P's tail the join point
        CK(cudaStreamWaitEvent(sP, p->ev_bulk[Nt - 1], 0));
    }
}

int status_from_exception(const CudaError& e) {
    if (e.e == cudaErrorMemoryAllocation) return MXP_ENOMEM;
    return MXP_ECUDA;
}

}  // namespace

// =========================================================================
extern "C" {

int mxp_chol_abi_version(void) { return MXP_CHOL_ABI_VERSION; }

const char* mxp_strerror(int s) {
    switch (s) {
    case MXP_OK: return "success";
    case MXP_ECUDA: return "CUDA runtime error";
    case MXP_ENOMEM: return "device memory below the working-set bound";
    case MXP_EHOSTPIN: return "host memory pinning failed";
    case MXP_ESTATE: return "invalid plan state";
    case MXP_ENOTSUP: return "configuration not supported";
    case MXP_EZERO: return "zero matrix (||A||_F = 0)";
    case MXP_ENCCL: return "inter-GPU exchange failed";
    default: return s < 0 && s > -100 ? "invalid argument" : "unknown status";
    }
}

const char* mxp_last_error(void) { return g_last_error.c_str(); }

int mxp_chol_plan(int64_t n, int64_t nb, const uint8_t* precision_map, int ngpus, mxp_plan_t* out) {
    if (n < 1) return -1;
    if (nb < 128 || nb > 2048 || nb % 128 != 0) return -2;
    if (ngpus != 1) return -4;
    if (!out) return -5;
    int64_t Nt = (n + nb - 1) / nb;
    int64_t T = Nt * (Nt + 1) / 2;
    if (T > INT32_MAX) return -1;
    std::vector<uint8_t> map(T, MXP_FP64);
    if (precision_map) {
        for (int64_t j = 0; j < Nt; ++j)
            for (int64_t i = j; i < Nt; ++i) {
                uint8_t c = precision_map[tile_index(Nt, i, j)];
                if (c > MXP_FP8) return -3;
                if (i == j && c != MXP_FP64) return -3;
                map[tile_index(Nt, i, j)] = c;
            }
        for (auto c : map)
            if (c != MXP_FP64) return MXP_ENOTSUP;  // MxP kernels: not in this build yet
    }
    auto* p = new mxp_plan_s();
    p->n = n;
    p->nb = nb;
    p->Nt = Nt;
    p->T = T;
    p->map = std::move(map);
    cudaGetDevice(&p->device);
    *out = p;
    return MXP_OK;
}

int mxp_chol_plan_set(mxp_plan_t p, mxp_attr_t key, int64_t v) {
    if (!p) return -1;
    switch (key) {
    case MXP_ATTR_DEVICE:
        if (p->ws || p->streams_ready) return MXP_ESTATE;
        p->device = (int)v;
        return MXP_OK;
    case MXP_ATTR_STREAM: p->user_stream = (cudaStream_t)(intptr_t)v; return MXP_OK;
    case MXP_ATTR_HBM_BYTES_CAP:
        if (v < 0) return -3;
        p->hbm_cap = v;
        return MXP_OK;
    case MXP_ATTR_SPLITK_TILES:
        if (v < 1) return -3;
        if (p->ws && !p->ws_owned) return MXP_ESTATE;
        if (p->ws_owned) {
            cudaFree(p->ws);
            p->ws = nullptr;
            p->ws_owned = false;
        }
        p->splitk_tiles = v;
        return MXP_OK;
    case MXP_ATTR_LOOKAHEAD: p->lookahead = v ? 1 : 0; return MXP_OK;
    case MXP_ATTR_DEBUG_SYNC: p->debug_sync = v ? 1 : 0; return MXP_OK;
    case MXP_ATTR_PROFILE: p->profile = v ? 1 : 0; return MXP_OK;
    default: return -2;
    }
}

int mxp_chol_kernel_stats(mxp_plan_t p, int cls, int64_t* launches, double* ms, double* flops) {
    if (!p) return -1;
    if (cls < 0 || cls > 3) return -2;
    if (launches) *launches = p->st_launch[cls];
    if (ms) *ms = p->st_ms[cls];
    if (flops) *flops = p->st_flops[cls];
    return MXP_OK;
}

int mxp_chol_plan_get(mxp_plan_t p, mxp_attr_t key, int64_t* v) {
    if (!p) return -1;
    if (!v) return -3;
    switch (key) {
    case MXP_ATTR_DEVICE: *v = p->device; return MXP_OK;
    case MXP_ATTR_STREAM: *v = (int64_t)(intptr_t)p->user_stream; return MXP_OK;
    case MXP_ATTR_HBM_BYTES_CAP: *v = p->hbm_cap; return MXP_OK;
    case MXP_ATTR_SPLITK_TILES: *v = p->splitk_tiles; return MXP_OK;
    case MXP_ATTR_LOOKAHEAD: *v = p->lookahead; return MXP_OK;
    case MXP_ATTR_DEBUG_SYNC: *v = p->debug_sync; return MXP_OK;
    case MXP_ATTR_PROFILE: *v = p->profile; return MXP_OK;
    case MXP_ATTR_GPU_LAUNCHES: *v = p->launches; return MXP_OK;
    case MXP_ATTR_H2D_BYTES: *v = p->h2d; return MXP_OK;
    case MXP_ATTR_D2H_BYTES: *v = p->d2h; return MXP_OK;
    case MXP_ATTR_POOL_SLOTS: *v = p->T; return MXP_OK;
    case MXP_ATTR_NT: *v = p->Nt; return MXP_OK;
    default: return -2;
    }
}

int mxp_chol_workspace_size(mxp_plan_t p, size_t* bytes) {
    if (!p) return -1;
    if (!bytes) return -2;
    size_t a, b, c;
    *bytes = workspace_need(p, &a, &b, &c);
    return MXP_OK;
}

int mxp_chol_set_workspace(mxp_plan_t p, void* dev, size_t bytes) {
    if (!p) return -1;
    if (!dev || ((uintptr_t)dev & 255)) return -2;
    size_t a, b, c;
    if (bytes < workspace_need(p, &a, &b, &c)) return -3;
    if (p->ws_owned && p->ws) {
        cudaSetDevice(p->device);
        cudaFree(p->ws);
    }
    p->ws = (char*)dev;
    p->ws_bytes = bytes;
    p->ws_owned = false;
    return MXP_OK;
}

int mxp_chol_factor_device(mxp_plan_t p, double* A, int64_t lda, int64_t* info) {
    if (!p) return -1;
    if (!A) return -2;
    if (lda < p->n) return -3;
    if (!info) return -4;
    p->have_result = false;
    p->launches = p->h2d = p->d2h = 0;
    int cur = 0;
    cudaGetDevice(&cur);
    try {
        CK(cudaSetDevice(p->device));
        ensure_streams(p);
        bind_workspace(p);
        cudaStream_t s0 = p->user_stream;
        // slot table (identity in-core) + info reset, ordered on the user stream
        std::vector<int32_t> slot(p->T);
        for (int64_t t = 0; t < p->T; ++t) slot[t] = (int32_t)t;
        CK(cudaMemcpyAsync(p->d_slot, slot.data(), sizeof(int32_t) * p->T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemsetAsync(p->d_info, 0, sizeof(int64_t), s0));
        prof_reset(p);
        {
            Prof pr(p, s0, MXP_KCLASS_OTHER, 0.0);
            launch_pack_f64(A, lda, p->n, p->pool, p->d_slot, p->Nt, p->nb, 0, p->Nt, s0);
            ++p->launches;
            dbg(p, s0, "pack");
        }
        CK(cudaEventRecord(p->ev_start, s0));
        CK(cudaStreamWaitEvent(p->sU, p->ev_start, 0));
        CK(cudaStreamWaitEvent(p->sP, p->ev_start, 0));
        factor_incore_f64(p);
        CK(cudaEventRecord(p->ev_done, p->sP));
        CK(cudaStreamWaitEvent(s0, p->ev_done, 0));
        {
            Prof pr(p, s0, MXP_KCLASS_OTHER, 0.0, 3);
            launch_unpack_f64(A, lda, p->n, p->pool, p->d_slot, p->Nt, p->nb, 0, p->Nt, s0);
            launch_logdet(p->pool, p->d_slot, p->Nt, p->nb, p->n, p->d_logdet_parts, p->d_logdet, s0);
            p->launches += 3;
            dbg(p, s0, "unpack");
        }
        int64_t hinfo = 0;
        double ld = 0.0;
        CK(cudaMemcpyAsync(&hinfo, p->d_info, sizeof(int64_t), cudaMemcpyDeviceToHost, s0));
        CK(cudaMemcpyAsync(&ld, p->d_logdet, sizeof(double), cudaMemcpyDeviceToHost, s0));
        CK(cudaStreamSynchronize(s0));
        prof_collect(p);
        *info = hinfo;
        p->have_result = (hinfo == 0);
        p->logdet = ld;
    } catch (const CudaError& e) {
        cudaSetDevice(cur);
        return status_from_exception(e);
    }
    cudaSetDevice(cur);
    return MXP_OK;
}

int mxp_chol_factor(mxp_plan_t p, double* A_host, int64_t lda, int64_t* info) {
    if (!p) return -1;
    if (!A_host) return -2;
    if (lda < p->n) return -3;
    if (!info) return -4;
    // Host-resident path: stage the matrix through the device (column panels),
    // factor in core, write the lower triangle back.  Out-of-core caching
    // (HBM cap below the lower triangle) is handled by the OOC engine.
    p->have_result = false;
    int cur = 0;
    cudaGetDevice(&cur);
    double* dA = nullptr;
    int rc = MXP_OK;
    try {
        CK(cudaSetDevice(p->device));
        cudaPointerAttributes attr{};
        bool registered = false;
        size_t host_bytes = sizeof(double) * (size_t)lda * (size_t)(p->n - 1) + sizeof(double) * p->n;
        if (cudaPointerGetAttributes(&attr, A_host) == cudaSuccess && attr.type == cudaMemoryTypeHost) {
            // already pinned
        } else {
            cudaGetLastError();
            if (cudaHostRegister(A_host, host_bytes, cudaHostRegisterDefault) != cudaSuccess) {
                cudaGetLastError();
                cudaSetDevice(cur);
                return MXP_EHOSTPIN;
            }
            registered = true;
        }
        ensure_streams(p);
        cudaStream_t s0 = p->user_stream;
        size_t dbytes = sizeof(double) * (size_t)p->n * (size_t)p->n;
        cudaError_t e = cudaMallocAsync((void**)&dA, dbytes, s0);
        if (e != cudaSuccess) {
            cudaGetLastError();
            if (registered) cudaHostUnregister(A_host);
            cudaSetDevice(cur);
            return MXP_ENOMEM;
        }
        CK(cudaMemcpy2DAsync(dA, sizeof(double) * p->n, A_host, sizeof(double) * lda, sizeof(double) * p->n,
                             p->n, cudaMemcpyHostToDevice, s0));
        int64_t launches_before = 0;
        rc = mxp_chol_factor_device(p, dA, p->n, info);
        launches_before = p->launches;
        if (rc == MXP_OK) {
            CK(cudaMemcpy2DAsync(A_host, sizeof(double) * lda, dA, sizeof(double) * p->n, sizeof(double) * p->n,
                                 p->n, cudaMemcpyDeviceToHost, s0));
            CK(cudaStreamSynchronize(s0));
        }
        p->launches = launches_before;
        p->h2d = (int64_t)dbytes;
        p->d2h = rc == MXP_OK ? (int64_t)dbytes : 0;
        CK(cudaFreeAsync(dA, s0));
        CK(cudaStreamSynchronize(s0));
        if (registered) cudaHostUnregister(A_host);
    } catch (const CudaError& e) {
        cudaSetDevice(cur);
        return status_from_exception(e);
    }
    cudaSetDevice(cur);
    return rc;
}

int mxp_chol_logdet(mxp_plan_t p, double* logdet) {
    if (!p) return -1;
    if (!logdet) return -2;
    if (!p->have_result) return MXP_ESTATE;
    *logdet = p->logdet;
    return MXP_OK;
}

int mxp_precision_map_from_matrix_device(int64_t n, int64_t nb, const double* A, int64_t lda, double eps,
                                         uint32_t allowed, uint8_t* map_out, double* norms_out) {
    if (n < 1) return -1;
    if (nb < 1) return -2;
    if (!A) return -3;
    if (lda < n) return -4;
    if (!(eps > 0.0 && eps < 1.0)) return -5;
    if (!(allowed & 1u) || (allowed & ~0xFu)) return -6;
    if (!map_out) return -7;
    int64_t Nt = (n + nb - 1) / nb, T = Nt * (Nt + 1) / 2;
    double* dn = nullptr;
    std::vector<double> f(T);
    try {
        CK(cudaMalloc(&dn, sizeof(double) * T));
        launch_tile_norms(A, lda, n, nb, dn, 0);
        CK(cudaGetLastError());
        CK(cudaMemcpy(f.data(), dn, sizeof(double) * T, cudaMemcpyDeviceToHost));
        CK(cudaFree(dn));
    } catch (const CudaError& e) {
        if (dn) cudaFree(dn);
        return status_from_exception(e);
    }
    // F with off-diagonal tiles counted twice; criterion P:335 (G6)
    double ss = 0.0;
    for (int64_t j = 0; j < Nt; ++j)
        for (int64_t i = j; i < Nt; ++i) {
            double v = f[tile_index(Nt, i, j)];
            ss += (i == j ? 1.0 : 2.0) * v * v;
        }
    double F = std::sqrt(ss);
    if (F == 0.0) return MXP_EZERO;
    const double u[4] = {0x1p-53, 0x1p-24, 0x1p-11, 0x1p-4};
    for (int64_t j = 0; j < Nt; ++j)
        for (int64_t i = j; i < Nt; ++i) {
            int64_t t = tile_index(Nt, i, j);
            uint8_t c = MXP_FP64;
            if (i != j) {
                double ratio = (double)Nt * f[t] / F;
                for (int p = 3; p >= 0; --p) {
                    if (!(allowed & (1u << p))) continue;
                    if (ratio < eps / u[p]) {
                        c = (uint8_t)p;
                        break;
                    }
                }
            }
            map_out[t] = c;
            if (norms_out) norms_out[t] = f[t];
        }
    return MXP_OK;
}

void mxp_chol_plan_destroy(mxp_plan_t p) { delete p; }

int mxp_host_alloc(size_t bytes, void** ptr) {
    if (!ptr) return -2;
    if (cudaMallocHost(ptr, bytes) != cudaSuccess) {
        cudaGetLastError();
        return MXP_EHOSTPIN;
    }
    return MXP_OK;
}

int mxp_host_free(void* ptr) {
    if (!ptr) return MXP_OK;
    return cudaFreeHost(ptr) == cudaSuccess ? MXP_OK : MXP_ECUDA;
}

}  // extern "C"
