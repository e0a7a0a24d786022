// engine.cu -- host runtime of the B200 engine and the C ABI (include/mxp_chol.h).
//
// Static schedule (Alg. 1): the host enumerates the task
// list once per plan -- column by column, with one column of lookahead -- and
// uploads it; the device executes it with persistent CTAs that busy-wait on a
// device-resident Ready table (sched_f64.cu).  The diagonal POTRFs run as one
// small kernel per column on a high-priority stream on reserved SMs.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mxp_chol.h"
#include "internal.h"
#include "oz_i8.cuh"
#include "tc_native.cuh"

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

// Stream memory operations (executed by the GPU front-end, no SM needed):
// the copy streams publish "tile landed" and wait for "tile final" flags.
typedef CUresult (*PFN_streamValue32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
PFN_streamValue32 g_write32 = nullptr, g_wait32 = nullptr;
bool stream_memops() {
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamWriteValue32", (void**)&g_write32, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            g_write32 = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", (void**)&g_wait32, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            g_wait32 = nullptr;
        cudaGetLastError();
    });
    return g_write32 && g_wait32;
}
}  // namespace

struct mxp_plan_s {
    int64_t n = 0, nb = 0, Nt = 0, T = 0;
    std::vector<uint8_t> map;
    int device = 0;
    cudaStream_t user_stream = 0;
    int64_t hbm_cap = 0;
    int64_t splitk_tiles = 16;  // bulk K chunk of a GEMM task, in tiles (swept at C3 MxP: 4/8/16/32 -> 263/280/286/291 TF/s; C2 equal at 8 and 16)
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
    int32_t* d_prev = nullptr;     // previous tile of each tile's slot (out-of-core reuse)
    int* d_flags = nullptr;        // counter, err, ready[T], gemm_done[T], trsm_done[T], blk_chunk[T*NB]
    size_t flags_bytes = 0;
    int* d_expected = nullptr;     // gemm_expected[T]
    int4* d_items = nullptr;
    double* d_wbuf = nullptr;
    unsigned long long* d_stats = nullptr;  // diagnostics (profile=1)
    std::vector<unsigned long long> h_stats;
    double* pool = nullptr;
    std::vector<int4> items;       // host copy of the static task list
    std::vector<int> expected;
    bool list_uploaded = false;
    int reserved_sms = 1;
    int tc_engine = 3;             // non-FP64 GEMM tasks: 0 DMMA with casts, 1 tcgen05 on operand
                                   // images (register-staged when out of core), 2 tcgen05 register-staged
    // operand images (tcgen05 engine, in core): see SchedArgs::img
    std::vector<long long> img;    // [4T] byte offsets into the image arena, -1 = absent
    std::vector<uint8_t> qtile;    // [T] tile has QUANT tasks
    size_t shadow_bytes = 0;
    long long img_key = -1;        // (tc_engine, pool) state the image plan was computed for
    uint8_t* d_qtile = nullptr;
    long long* d_img = nullptr;
    uint8_t* d_shadow = nullptr;
    // FP64 engine (MXP_ATTR_FP64_ENGINE): 0 DMMA, 1 Ozaki int8 on tcgen05 (in core);
    // oz_on = the engine actually used by the current image plan
    int fp64_engine = 0, oz_slices = 7;
    int oz_prefetch = 0;            // MXP_ATTR_OZ_PREFETCH
    bool oz_on = false;
    bool nat_on = false;            // tiles below FP64 on the native-width engine (tc_engine 3, k_tc)
    // compact pool (with the native engine): only FP64 tiles keep a permanent fp64 slot; a tile
    // stored below FP64 keeps its fp64 accumulator slot from its input until its QUANT (a ring
    // recycled column by column) and then lives as its storage image (codes at its precision)
    bool compact = false;
    int compact_attr = 1;           // MXP_ATTR_COMPACT_POOL
    int64_t compact_slots = 0;
    std::vector<long long> sto;     // [T] byte offsets of the storage images in the shadow arena, -1 = none
    long long* d_sto = nullptr;
    void* const* tiles_io = nullptr;  // mxp_chol_factor_tiles: host tiles at storage precision (this call)
    double* d_in_scale = nullptr;     // [T] scales of those input tiles
    std::vector<long long> oz_img;  // [T] byte offsets of the int8 slice images, -1 = none
    long long* d_oz_img = nullptr;
    // Ozaki out of core (FP64 maps, one rank, HBM cap below the lower triangle): every tile keeps an
    // fp64 slot only while it is computed (a ring recycled column by column, plan_compact(all)),
    // and a final off-diagonal tile lives on as its slice image in an arena whose slots are
    // recycled when the tile's row dies (plan_oz_ooc; DESIGN 5.4)
    bool oz_ooc = false;
    int64_t ring_slots = 0, oz_img_slots = 0;
    std::vector<int32_t> ring_slot, ring_prev, img_prev;
    int32_t* d_img_prev = nullptr;
    int* d_oz_flag = nullptr;       // Ozaki: tiles whose row scales grew (SchedArgs::oz_flag)
    double* d_solve = nullptr;      // forward-solve work vectors (r | z | scalars)
    std::vector<int4> items2;       // GEMM list of k_tc (Ozaki mode)
    cudaStream_t sT = 0;
    bool mxp = false;              // any tile below FP64
    uint8_t* d_prec = nullptr;
    unsigned long long* d_amax_x = nullptr;
    double* d_amax_s = nullptr;
    double* d_iscale = nullptr;     // [3T] scales: native fp16 / E4M3 code images, storage image
    SchedArgs* d_args = nullptr;
    SchedArgs h_args{};
    bool host_mode = false;        // task list built for the host-streaming path (PREP tasks)
    int epoch = 0;                 // factorization counter: Ready entries equal to it are current
    int rank = 0, nranks = 1;      // row-cyclic distribution (tile (m, n) on rank m mod nranks)
    int sm_first = 0, sm_count = 0;  // SM partition of the scheduler (0 = all SMs)
    char* peer_ws[MAX_RANKS] = {};   // peers' workspaces (same layout), mapped in this process
    bool peer_ipc[MAX_RANKS] = {};
    cudaStream_t sPush = 0;
    int* d_epoch = nullptr;          // device word holding the current epoch (pushed to peers' Ready)
    int* d_entered = nullptr;        // [MAX_RANKS] epoch each peer has entered (start barrier)
    bool ready_dirty = false;        // Ready words may exceed the next epoch (probe / drained failure)
    int64_t slots = 0;             // tile slots in the device pool (T in core; fewer out of core)
    std::vector<int32_t> slot_plan, prev_owner;  // out-of-core slot assignment (host mode)
    cudaStream_t sH2D = 0, sD2H = 0, sAux = 0;
    double* h_stage = nullptr;     // pinned staging for the diagonal tiles (upper triangle untouched)
    size_t h_stage_bytes = 0;

    bool streams_ready = false;
    cudaStream_t sU = 0, sP = 0;
    std::vector<cudaEvent_t> ev_panel, ev_bulk;
    cudaEvent_t ev_start = nullptr, ev_done = nullptr, ev_join = nullptr;
    cudaEvent_t ev_sched_end = nullptr, ev_potrf_end = nullptr;  // schedule kernels finished (failure watcher)
    cudaStream_t sMain = nullptr;      // ordering stream of a multi-rank call (joined to user_stream)

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
    // copy/compute timeline of the last host-streaming factorization with MXP_ATTR_PROFILE = 1
    // (the paper's C2G / G2C / Work rows): per column k, events after its H2D loads,
    // after its D2H write-backs and after its POTRF; tl_ms = ms since the factorization start
    std::vector<cudaEvent_t> ev_tl;
    std::vector<cudaEvent_t> ev_solve;  // forward solve: two streams' column events
    std::vector<char> tl_rec;
    std::vector<double> tl_ms;
    bool tl_on = false;
    int64_t st_launch[4] = {0, 0, 0, 0};
    double st_ms[4] = {0, 0, 0, 0}, st_flops[4] = {0, 0, 0, 0};
    bool have_result = false;
    double logdet = 0.0;
    int solve_seq = 0;              // forward solves run on this plan (publication tags of the diagonal solves)
    // single-process multi-GPU (mxp_chol_plan with ngpus > 1): the group plan owns one sub-plan
    // per GPU (rank r, device r mod #devices) and runs them from one host thread each
    std::vector<mxp_plan_s*> group;
    bool in_group = false;  // a sub-plan: only rank 0 writes the factor back (factor_device)

    ~mxp_plan_s();
};

mxp_plan_s::~mxp_plan_s() {
    for (auto* c : group) delete c;
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    if (ws_owned && ws) cudaFree(ws);
    for (auto e : ev_panel) cudaEventDestroy(e);
    for (auto e : ev_bulk) cudaEventDestroy(e);
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (auto e : ev_tl) cudaEventDestroy(e);
    for (auto e : ev_solve) cudaEventDestroy(e);
    if (ev_start) cudaEventDestroy(ev_start);
    if (ev_done) cudaEventDestroy(ev_done);
    if (sU) cudaStreamDestroy(sU);
    if (sP) cudaStreamDestroy(sP);
    if (sH2D) cudaStreamDestroy(sH2D);
    if (sD2H) cudaStreamDestroy(sD2H);
    if (sAux) cudaStreamDestroy(sAux);
    if (sPush) cudaStreamDestroy(sPush);
    if (sMain) cudaStreamDestroy(sMain);
    if (sT) cudaStreamDestroy(sT);
    if (ev_join) cudaEventDestroy(ev_join);
    if (ev_sched_end) cudaEventDestroy(ev_sched_end);
    if (ev_potrf_end) cudaEventDestroy(ev_potrf_end);
    for (int q = 0; q < MAX_RANKS; ++q)
        if (peer_ipc[q] && peer_ws[q]) cudaIpcCloseMemHandle(peer_ws[q]);
    if (h_stage) cudaFreeHost(h_stage);
    cudaSetDevice(cur);
}

namespace {

int64_t blocks_per_tile(int64_t nb) { return (nb / 64) * (nb / 128); }

// 64x128 blocks of tile (m,k) that are computed: all of them off the diagonal,
// the lower(-intersecting) ones on it (strictly upper blocks are never read).
bool block_needed(int64_t m, int64_t k, int64_t b, int64_t nb) {
    if (m != k) return true;
    int64_t SR = nb / 64, bi = b % SR, bj = b / SR;
    return (bi + 1) * 64 > bj * 128;
}

// GEMM blocks of a tile: 64x128 DMMA blocks, or 128x128 tcgen05 blocks for
// tiles computed below FP64 when the tensor-core engine is on, or 128x64
// int8-tensor-core blocks for FP64 tiles in the Ozaki mode.
int64_t gemm_blocks(const mxp_plan_s* p, int64_t m, int64_t k) {
    const int64_t nb = p->nb;
    if (p->tc_engine && p->map[tile_index(p->Nt, m, k)] != MXP_FP64) return (nb / 128) * (nb / 128);
    return blocks_per_tile(nb);
}
// block b of tile (m,k) computed?  (strictly upper blocks of diagonal tiles are skipped)
bool gemm_block_needed(const mxp_plan_s* p, int64_t m, int64_t k, int64_t b) {
    const int64_t nb = p->nb;
    if (m != k) return true;
    if (p->oz_on) {  // 128x64 blocks: rows [128 bi, +128), cols [64 bj, +64)
        const int64_t SR = nb / 128, bi = b % SR, bj = b / SR;
        return (bi + 1) * 128 > bj * 64;
    }
    return block_needed(m, k, b, nb);
}

// chunks of column k: ceil((k-1)/KC) fixed-size chunks over [0, k-1), then {k-1}
int64_t nchunks(int64_t k, int64_t KC) {
    if (k == 0) return 0;
    int64_t nfull = k >= 2 ? (k - 1 + KC - 1) / KC : 0;
    return nfull + 1;
}

// The static task list (Alg. 1 enumerated column by column):
//   iteration k:  (a) last GEMM chunk (n = k-1) of column k, diagonal tile first
//                 (b) bulk GEMM chunks (n < k) of column k+1   [lookahead]
//                 (c) TRSM row tasks of column k
// POTRF(k) runs beside it (k_potrf_tile) once (a) has finished on tile (k,k).
void plan_images(mxp_plan_s* p);
void build_task_list(mxp_plan_s* p) {
    plan_images(p);
    const int64_t Nt = p->Nt, nb = p->nb, KC = p->splitk_tiles, NB = blocks_per_tile(nb);
    p->items.clear();
    p->items2.clear();
    p->expected.assign(p->T, 0);
    // Ozaki mode: k_tc walks the whole list (items2), k_sched its non-GEMM part (items)
    auto push = [&](const int4& it) {
        if (p->oz_on) {
            p->items2.push_back(it);
            if (it.x != ITEM_GEMM) p->items.push_back(it);
        } else {
            p->items.push_back(it);
        }
    };
    auto owned = [&](int64_t m) { return m % p->nranks == p->rank; };
    auto gemm_col = [&](int64_t k, int64_t c0, int64_t c1) {
        for (int64_t c = c0; c < c1; ++c)
            for (int64_t m = k; m < Nt; ++m)
                if (owned(m))
                for (int64_t b = 0; b < gemm_blocks(p, m, k); ++b)
                    if (gemm_block_needed(p, m, k, b)) {
                        push(make_int4(ITEM_GEMM, (int)m, (int)k, (int)((b << 16) | c)));
                        p->expected[tile_index(Nt, m, k)]++;
                    }
    };
    auto prep_col = [&](int64_t k) {
        for (int64_t m = k; m < Nt; ++m)
            if (owned(m)) push(make_int4(ITEM_PREP, (int)m, (int)k, 0));
    };
    if (p->host_mode) prep_col(0);
    for (int64_t k = 0; k < Nt; ++k) {
        if (p->host_mode && k + 1 < Nt) prep_col(k + 1);  // before any GEMM on column k+1
        if (k >= 1) {
            int64_t last = nchunks(k, KC) - 1;
            gemm_col(k, last, last + 1);
        }
        // POTRF(k): normally claimed by the dedicated kernel; listed so the
        // schedule can also complete on its own (fallback, see sched_f64.cu)
        if (owned(k)) push(make_int4(ITEM_POTRF, (int)k, (int)k, 0));
        if (k + 1 < Nt) {
            int64_t nb1 = nchunks(k + 1, KC) - 1;  // bulk chunks of column k+1
            gemm_col(k + 1, 0, nb1);
        }
        if (p->debug_sync == 2) continue;  // GEMM-throughput probe: no TRSM tasks
        for (int64_t m = k + 1; m < Nt; ++m)
            if (owned(m))
                for (int64_t r = 0; r < nb / 64; ++r)
                    push(make_int4(ITEM_TRSM, (int)m, (int)k, (int)r));
        for (int64_t m = k + 1; m < Nt; ++m)
            if (owned(m) && p->qtile[tile_index(Nt, m, k)])
                for (int64_t r = 0; r < nb / 64; ++r)
                    push(make_int4(ITEM_QUANT, (int)m, (int)k, (int)r));
    }
}

// Operand images (tcgen05 engine): tile t = (i, n) is an operand of the GEMMs
// of row i (outputs (i, k), n < k < i; A side) and of column i (outputs
// (m, i), m > i; B side).  Each such output of precision c != FP64 reads
// cast_c(L_t), i.e. the image e = max(c, p_t) (an operand stored at or below
// c is used as stored).  One fp32 image per distinct e, plus the TF32
// remainder for e = FP32.  Out of core (pool < T) the register-staged engine
// is used instead (images would be sized by the whole lower triangle).
int64_t pool_slots(const mxp_plan_s* p);
// Compact slot plan (the static schedule is known in advance): walking
// the columns in schedule order, tile (m, j) takes a slot freed by a tile of a
// column <= j-2 (those are final before column j's inputs are prepared, and
// their QUANT tasks come earlier in the task list, so waiting for them cannot
// deadlock) or a fresh one.  Tiles stored below FP64 (off the diagonal) free
// their slot when they are final; FP64 tiles keep theirs.  prev[t] = the tile
// whose death the preparation of t waits for.  Returns the slot count.
int64_t plan_compact(const mxp_plan_s* p, std::vector<int32_t>& slot, std::vector<int32_t>& prev, bool all = false) {
    const int64_t Nt = p->Nt, T = p->T;
    slot.assign(T, -1);
    prev.assign(T, -1);
    std::vector<int32_t> owner, freelist;
    std::vector<std::vector<int32_t>> freed_at(Nt);
    // all (Ozaki out of core): slots freed by columns <= j-3 -- the tiles of column j are
    // loaded during iteration j-2 (for the lookahead GEMMs of iteration j-1), while column
    // j-2's tiles become final and stream back (D2H) about one column later (measured)
    const int64_t lag = all ? 3 : 2;
    for (int64_t j = 0; j < Nt; ++j) {
        if (j >= lag)
            for (int32_t x : freed_at[j - lag]) freelist.push_back(x);
        for (int64_t m = j; m < Nt; ++m) {
            const int64_t t = tile_index(Nt, m, j);
            int32_t sl;
            if (!freelist.empty()) {
                sl = freelist.back();
                freelist.pop_back();
            } else {
                sl = (int32_t)owner.size();
                owner.push_back(-1);
            }
            slot[t] = sl;
            prev[t] = owner[sl];
            owner[sl] = (int32_t)t;
            // all (Ozaki out of core): every tile frees its slot -- off the diagonal once final
            // (its readers use the slice image), on the diagonal once its column is final
            if (all || (m != j && p->map[t] != MXP_FP64)) freed_at[j].push_back(sl);
        }
    }
    return (int64_t)owner.size();
}

// Slice-image arena of the Ozaki out-of-core mode: the image of tile (i, n)
// (i > n) is written by its QUANT (iteration n) and read by the GEMMs of row i
// (A side, columns n+1..i) and column i (B side): it dies with column i.  So
// the images born in column j take slots freed by rows <= j-2 (complete
// before the QUANTs of column j, which wait for them; those tasks are earlier
// in the list: no deadlock; one row of slack so a QUANT of column j rarely
// waits for the last QUANTs of column j-1).  prev[t] = the previous owner of t's image slot.
// Returns the slot count (the peak live set, ~Nt^2/4 tiles).
int64_t plan_oz_images(const mxp_plan_s* p, std::vector<int32_t>& slot, std::vector<int32_t>& prev) {
    const int64_t Nt = p->Nt, T = p->T;
    slot.assign(T, -1);
    prev.assign(T, -1);
    std::vector<int32_t> owner, freelist;
    for (int64_t j = 0; j < Nt; ++j) {
        if (j >= 2)  // row j-2 died with column j-2
            for (int64_t n = 0; n < j - 2; ++n) freelist.push_back(slot[tile_index(Nt, j - 2, n)]);
        for (int64_t m = j + 1; m < Nt; ++m) {
            const int64_t t = tile_index(Nt, m, j);
            int32_t sl;
            if (!freelist.empty()) {
                sl = freelist.back();
                freelist.pop_back();
            } else {
                sl = (int32_t)owner.size();
                owner.push_back(-1);
            }
            slot[t] = sl;
            prev[t] = owner[sl];
            owner[sl] = (int32_t)t;
        }
    }
    return (int64_t)owner.size();
}
// does a workspace of `need` bytes beside a pool of `pool_tiles` fp64 slots fit in this device's
// free memory (2 GB headroom; the plan's own current workspace counts as free)
bool fits_beside_pool(const mxp_plan_s* p, double need, int64_t pool_tiles = -1) {
    size_t fr = 0, tot = 0;
    int cur = 0;
    bool ok = true;
    cudaGetDevice(&cur);
    if (cudaSetDevice(p->device) == cudaSuccess && cudaMemGetInfo(&fr, &tot) == cudaSuccess) {
        const double pool = (double)sizeof(double) * p->nb * p->nb * (pool_tiles < 0 ? p->T : pool_tiles);
        ok = pool + need <= (double)fr + (double)p->ws_bytes - 2e9;
    }
    cudaGetLastError();
    cudaSetDevice(cur);
    return ok;
}
void plan_images_as(mxp_plan_s* p, bool native);
void plan_images(mxp_plan_s* p) {
    const long long key = (((((long long)p->oz_slices * 2 + p->fp64_engine) * 9 + p->nranks) * 4 + p->tc_engine) * 2 +
                           (pool_slots(p) == p->T ? 1 : 0)) * 2 + p->compact_attr +
                          1000003LL * (p->hbm_cap >> 20);  // (the out-of-core Ozaki plan depends on the cap)
    if (key == p->img_key) return;
    p->img_key = key;
    // native-width images (kind::f16 / kind::f8f6f4) run in the tensor-core kernel k_tc, which
    // exists with the Ozaki FP64 engine (in core, single rank); otherwise (or if the Ozaki
    // images do not fit) the fp32 tf32 images
    const bool try_native = p->mxp && p->tc_engine == 3 && p->fp64_engine == 1 && p->nranks == 1 &&
                            pool_slots(p) == p->T;
    plan_images_as(p, try_native);
    if (try_native && !p->oz_on) plan_images_as(p, false);
}
void plan_images_as(mxp_plan_s* p, bool native) {
    const int64_t Nt = p->Nt, T = p->T;
    p->img.assign(4 * T, -1);
    p->oz_img.assign(T, -1);
    p->sto.assign(T, -1);
    p->oz_on = false;
    p->oz_ooc = false;
    p->ring_slots = p->oz_img_slots = 0;
    p->img_prev.clear();
    p->nat_on = false;
    p->compact = false;
    p->qtile.assign(T, 0);
    p->shadow_bytes = 0;
    int64_t ptiles = T;  // fp64 pool slots (native: the compact plan)
    const bool compact = native && p->compact_attr;
    if (compact) {
        std::vector<int32_t> sl, pv;
        ptiles = plan_compact(p, sl, pv);
        // storage images (codes at the tile's precision, column-major) of the tiles below FP64
        for (int64_t j = 0; j < Nt; ++j)
            for (int64_t i = j + 1; i < Nt; ++i) {
                const int64_t t = tile_index(Nt, i, j);
                const int pt = p->map[t];
                if (pt == MXP_FP64) continue;
                p->sto[t] = (long long)p->shadow_bytes;
                p->shadow_bytes += (size_t)p->nb * p->nb * (pt == MXP_FP32 ? 4 : pt == MXP_FP16 ? 2 : 1);
            }
    }
    bool images = p->mxp && p->tc_engine != 0 && p->tc_engine != 2 && pool_slots(p) == T;
    const long long img_bytes = (long long)sizeof(float) * p->nb * p->nb;
    if (images) {  // lower bound of the image bytes (each non-FP64 tile at least its own image)
        long long need = 0;
        for (int64_t t = 0; t < T; ++t)
            need += p->map[t] == MXP_FP32 ? (native ? img_bytes : 2 * img_bytes)
                    : p->map[t] == MXP_FP16 ? (native ? img_bytes / 2 : img_bytes)
                    : p->map[t] == MXP_FP8 ? (native ? img_bytes / 4 : img_bytes) : 0;
        if (!fits_beside_pool(p, (double)need, ptiles)) images = false;
    }
    // Tile t = (i, n) is an operand of the GEMMs of row i (outputs (i, k), n < k < i) and of
    // column i (outputs (m, i), m > i).  tf32 engine: one fp32 image per distinct
    // e = max(c, p_t) (+ the TF32 remainder for e = FP32).  Native engine: slot 0 (+ 3) = fp32
    // values of cast_max(FP32, p_t) for FP32 outputs, slot 1 = fp16 codes for FP16 outputs,
    // slot 2 = E4M3 codes for FP8 outputs.
    for (int64_t n = 0; n < Nt; ++n)
        for (int64_t i = n + 1; i < Nt; ++i) {
            const int64_t t = tile_index(Nt, i, n);
            const int pt = p->map[t];
            bool need[4] = {false, false, false, false};  // by consumer precision c (native) / e (tf32)
            if (images) {
                auto consumer = [&](int c) {
                    if (c == MXP_FP64) return;
                    need[native ? c : std::max(c, pt)] = true;
                };
                for (int64_t k = n + 1; k < i; ++k) consumer(p->map[tile_index(Nt, i, k)]);
                for (int64_t m = i + 1; m < Nt; ++m) consumer(p->map[tile_index(Nt, m, i)]);
            }
            bool any = false;
            if (native) {
                // slot 1: fp16 codes h (FP16 consumers, and the high part for FP32 consumers);
                // slot 3: fp16 remainders l (FP32 consumers of operands stored at FP32 or finer);
                // slot 2: E4M3 codes (FP8 consumers)
                const bool n16 = need[MXP_FP16] || need[MXP_FP32], n8 = need[MXP_FP8];
                const bool nrem = need[MXP_FP32] && pt <= MXP_FP32;
                if (n16) p->img[4 * t + 1] = (long long)p->shadow_bytes, p->shadow_bytes += nat::image_bytes(nat::K_F16, p->nb);
                if (n8) p->img[4 * t + 2] = (long long)p->shadow_bytes, p->shadow_bytes += nat::image_bytes(nat::K_F8, p->nb);
                if (nrem) p->img[4 * t + 3] = (long long)p->shadow_bytes, p->shadow_bytes += nat::image_bytes(nat::K_F16, p->nb);
                any = n16 || n8;
            } else {
                for (int e = 1; e <= 3; ++e)
                    if (need[e]) {
                        any = true;
                        p->img[4 * t + e - 1] = (long long)p->shadow_bytes;
                        p->shadow_bytes += img_bytes;
                        if (e == MXP_FP32) {  // TF32 remainder of the FP32 image
                            p->img[4 * t + 3] = (long long)p->shadow_bytes;
                            p->shadow_bytes += img_bytes;
                        }
                    }
            }
            p->qtile[t] = (pt != MXP_FP64 || any) ? 1 : 0;
        }
    // Ozaki mode (in core; tiles below FP64 need the image engine): every
    // off-diagonal tile is an operand of the FP64 SYRK of its row's diagonal
    // tile, so each gets an int8 slice image (s bytes per element + row scales)
    // (single rank: with ranks co-located on one GPU the two kernels of each rank
    // did not all become resident and the schedule timed out -- DESIGN 5.7)
    if (p->fp64_engine == 1 && pool_slots(p) == T && p->nranks == 1 && (!p->mxp || images)) {
        const long long ob = oz::image_bytes(p->oz_slices, p->nb);
        const size_t before = p->shadow_bytes;
        for (int64_t n = 0; n < Nt; ++n)
            for (int64_t i = n + 1; i < Nt; ++i) {
                const int64_t t = tile_index(Nt, i, n);
                p->oz_img[t] = (long long)p->shadow_bytes;
                p->shadow_bytes += ob;
                p->qtile[t] = 1;
            }
        p->oz_on = true;
        if (!fits_beside_pool(p, (double)p->shadow_bytes, ptiles)) {  // does not fit: DMMA
            p->oz_img.assign(T, -1);
            p->shadow_bytes = before;
            p->oz_on = false;
            for (int64_t t = 0; t < T; ++t) p->qtile[t] = 0;
            for (int64_t t = 0; t < T; ++t)
                if (p->map[t] != MXP_FP64) p->qtile[t] = 1;
            for (int64_t t = 0; t < T; ++t)
                for (int e = 0; e < 4; ++e)
                    if (p->img[4 * t + e] >= 0) p->qtile[t] = 1;
            for (int64_t k = 0; k < Nt; ++k) p->qtile[tile_index(Nt, k, k)] = 0;
        }
    }
    // Ozaki out of core (FP64 map, one rank, cap below the fp64 lower triangle): an fp64 ring for
    // the tiles being computed + a slice-image arena sized by the live set; both under the cap
    if (!p->oz_on && p->fp64_engine == 1 && !p->mxp && p->nranks == 1 && pool_slots(p) < T) {
        const long long ob = oz::image_bytes(p->oz_slices, p->nb);
        std::vector<int32_t> islot, iprev;
        const int64_t ring = plan_compact(p, p->ring_slot, p->ring_prev, true);
        const int64_t ni = plan_oz_images(p, islot, iprev);
        const double need = (double)ring * sizeof(double) * p->nb * p->nb + (double)ni * ob;
        if (need <= (double)p->hbm_cap && fits_beside_pool(p, (double)ni * ob, ring)) {
            for (int64_t t = 0; t < T; ++t) {
                p->oz_img[t] = islot[t] >= 0 ? (long long)islot[t] * ob : -1;
                p->qtile[t] = islot[t] >= 0 ? 1 : 0;
            }
            p->img_prev = iprev;
            p->shadow_bytes = (size_t)ni * ob;
            p->oz_on = p->oz_ooc = true;
            p->ring_slots = ring;
            p->oz_img_slots = ni;
        }
    }
    p->nat_on = native && p->oz_on;
    p->compact = p->nat_on && compact;
    p->compact_slots = p->compact ? ptiles : 0;
    if (images && !p->oz_on && !fits_beside_pool(p, (double)p->shadow_bytes)) {
        // full size known now: does not fit -> the register-staged engine
        p->img.assign(4 * T, -1);
        p->shadow_bytes = 0;
        for (int64_t t = 0; t < T; ++t) p->qtile[t] = p->map[t] != MXP_FP64 ? 1 : 0;
        for (int64_t k = 0; k < p->Nt; ++k) p->qtile[tile_index(p->Nt, k, k)] = 0;
    }
}

size_t list_bytes(const mxp_plan_s* p) {
    // count without building: GEMM tasks + TRSM tasks
    const int64_t Nt = p->Nt, nb = p->nb, NB = blocks_per_tile(nb);
    int64_t diag_blocks = 0;
    for (int64_t b = 0; b < NB; ++b) diag_blocks += gemm_block_needed(p, 0, 0, b);
    int64_t cnt = 0;
    for (int64_t k = 1; k < Nt; ++k) {
        int64_t per = diag_blocks;
        for (int64_t m = k + 1; m < Nt; ++m) per += gemm_blocks(p, m, k);
        cnt += nchunks(k, p->splitk_tiles) * per;
    }
    cnt += (Nt * (Nt - 1) / 2) * (nb / 64);
    for (int64_t t = 0; t < p->T; ++t) cnt += p->qtile[t] * (nb / 64);
    cnt += p->T;   // PREP tasks (host-streaming mode)
    cnt += Nt;     // POTRF claims
    if (p->oz_on) cnt *= 2;  // the whole list for k_tc + its non-GEMM part for k_sched (upper bound)
    return sizeof(int4) * (size_t)cnt;
}

size_t flag_ints(const mxp_plan_s* p) {
    // + Ozaki-mode task claims (TRSM, QUANT: T * nb/64 each; PREP: T) + timeout diagnostics (8)
    // + per-SM claim words of k_sched in the Ozaki mode (256) + counter2 (last)
    return (size_t)(2 + 7 * p->T + p->T * blocks_per_tile(p->nb) + 2 * p->Nt + (2 * p->T * (p->nb / 64) + p->T) +
                    24 + 256 + 1);
}

// Tile slots of the device pool: every lower tile in core; with
// MXP_ATTR_HBM_BYTES_CAP the pool shrinks to the cap and the host-streaming
// path recycles the slots of dead tiles (out of core).
int64_t pool_slots(const mxp_plan_s* p) {
    if (p->hbm_cap <= 0) return p->T;
    const int64_t tile_bytes = (int64_t)sizeof(double) * p->nb * p->nb;
    return std::max<int64_t>(1, std::min<int64_t>(p->T, p->hbm_cap / tile_bytes));
}

// (m, n) of the column-major lower-tile index t
void tile_coords(int64_t Nt, int64_t t, int64_t& m, int64_t& n) {
    n = 0;
    while (t >= Nt - n) {
        t -= Nt - n;
        ++n;
    }
    m = n + t;
}

// Static slot plan for the streaming path (the schedule is known in advance,
// P:152): tile (c, n) is dead once column c is final (its last uses are
// column c's GEMMs as B operand / row c as A operand, and TRSM(., c) for the
// diagonal), so the tiles born for column j (loaded during iteration j-1)
// may take the slots freed by columns <= j-2.  prev_owner[t] is the tile whose
// death (and write-back) the H2D of t must wait for.  Returns false if the
// pool cannot hold the live set (re-fetching evicted live tiles, the paper's
// V2 regime, is not implemented: MXP_ENOMEM).
bool plan_slots(mxp_plan_s* p, int64_t C) {
    const int64_t Nt = p->Nt, T = p->T;
    if (p->compact) {  // (plan_images decided it: in core, native engine)
        plan_compact(p, p->slot_plan, p->prev_owner);
        return true;
    }
    if (p->oz_ooc) {  // Ozaki out of core: the fp64 ring (plan_images)
        p->slot_plan = p->ring_slot;
        p->prev_owner = p->ring_prev;
        return true;
    }
    p->slot_plan.assign(T, -1);
    p->prev_owner.assign(T, -1);
    if (C >= T) {  // in core: every tile keeps its own slot (L stays resident)
        for (int64_t t = 0; t < T; ++t) p->slot_plan[t] = (int32_t)t;
        return true;
    }
    std::vector<int32_t> owner(C, -1), freelist;
    for (int64_t s = C - 1; s >= 0; --s) freelist.push_back((int32_t)s);
    std::vector<std::vector<int32_t>> freed_at(Nt);
    for (int64_t j = 0; j < Nt; ++j) {
        if (j >= 2)
            for (int32_t s : freed_at[j - 2]) freelist.push_back(s);
        for (int64_t m = j; m < Nt; ++m) {
            if (freelist.empty()) return false;
            const int32_t s = freelist.back();
            freelist.pop_back();
            const int64_t t = tile_index(Nt, m, j);
            p->slot_plan[t] = s;
            p->prev_owner[t] = owner[s];
            owner[s] = (int32_t)t;
        }
        for (int64_t n = 0; n <= j; ++n) freed_at[j].push_back(p->slot_plan[tile_index(Nt, j, n)]);
    }
    return true;
}

struct Layout {
    size_t slot, prev, epoch, flags, flags_bytes, expected, items, wbuf, stats, prec, amax_x, amax_s, iscale, args,
        qtile, img, ozimg, imgprev, ozflag, sto, in_scale, solve, shadow, pool, total;
};

Layout layout(const mxp_plan_s* p) {
    plan_images(const_cast<mxp_plan_s*>(p));  // (cached; depends on map, engine and pool size)
    Layout L{};
    size_t off = 256 + align_up(sizeof(double) * (p->Nt + 2), 256);  // info, logdet parts
    L.slot = off;
    off += align_up(sizeof(int32_t) * p->T, 256);
    L.prev = off;
    off += align_up(sizeof(int32_t) * p->T, 256);
    L.epoch = off;
    off += 256;
    L.flags = off;
    // counter, err, ready, gemm_done, trsm_done, quant_done, loaded, prep_done, blk_chunk, potrf_claim,
    // col_ready, d2h_done; then amax_x
    L.flags_bytes = align_up(sizeof(int) * flag_ints(p), 8) + sizeof(unsigned long long) * (size_t)p->T;
    off += align_up(L.flags_bytes, 256);
    L.expected = off;
    off += align_up(sizeof(int) * p->T, 256);
    L.items = off;
    off += align_up(list_bytes(p), 256);
    L.wbuf = off;
    off += align_up(sizeof(double) * (size_t)p->Nt * p->nb * 128, 256);
    L.stats = off;
    off += align_up(sizeof(unsigned long long) * (size_t)(STAT_POTRF + 3 * p->Nt), 256);
    L.prec = off;
    off += align_up((size_t)p->T, 256);
    L.amax_s = off;
    off += align_up(sizeof(double) * (size_t)p->T, 256);
    L.iscale = off;
    off += align_up(sizeof(double) * 3 * (size_t)p->T, 256);
    L.args = off;
    off += align_up(sizeof(SchedArgs), 256);
    L.qtile = off;
    off += align_up((size_t)p->T, 256);
    L.img = off;
    off += align_up(sizeof(long long) * 4 * (size_t)p->T, 256);
    L.ozimg = off;
    off += align_up(sizeof(long long) * (size_t)p->T, 256);
    L.imgprev = off;
    off += align_up(sizeof(int32_t) * (size_t)p->T, 256);
    L.ozflag = off;
    off += align_up(sizeof(int) * (size_t)p->T, 256);
    L.sto = off;
    off += align_up(sizeof(long long) * (size_t)p->T, 256);
    L.in_scale = off;
    off += align_up(sizeof(double) * (size_t)p->T, 256);
    L.solve = off;  // forward solve: r, z (Nt*nb each) + scalars + 32 ints of diagonal-solve flags
    off += align_up(sizeof(double) * (2 * (size_t)p->Nt * p->nb + 8 + 16), 256);
    L.shadow = off;
    off += align_up(p->shadow_bytes, 1024);
    L.pool = off;
    off += sizeof(double) * (size_t)(p->oz_ooc ? p->ring_slots : p->compact ? p->compact_slots : pool_slots(p)) *
           p->nb * p->nb;
    L.total = off;
    return L;
}

size_t workspace_need(const mxp_plan_s* p) { return layout(p).total; }

void bind_workspace(mxp_plan_s* p) {
    Layout L = layout(p);
    if (p->ws && L.total > p->ws_bytes) {
        // the layout grew since the workspace was bound (e.g. RANK/NRANKS changed the image plan)
        if (!p->ws_owned) {
            g_last_error = "user workspace smaller than the plan's current layout (mxp_chol_workspace_size)";
            throw CudaError{cudaErrorInvalidValue};
        }
        cudaFree(p->ws);
        p->ws = nullptr;
        p->ws_owned = false;
        for (int q = 0; q < MAX_RANKS; ++q)  // peers must re-attach the new workspace
            if (p->peer_ws[q] && p->peer_ipc[q]) cudaIpcCloseMemHandle(p->peer_ws[q]);
        for (int q = 0; q < MAX_RANKS; ++q) p->peer_ws[q] = nullptr, p->peer_ipc[q] = false;
    }
    if (!p->ws) {
        void* ptr = nullptr;
        cudaError_t e = cudaMalloc(&ptr, L.total);
        if (e != cudaSuccess) {
            cudaGetLastError();
            g_last_error = std::string("cudaMalloc workspace: ") + cudaGetErrorString(e);
            throw CudaError{cudaErrorMemoryAllocation};
        }
        p->ws = (char*)ptr;
        p->ws_bytes = L.total;
        p->ws_owned = true;
        p->list_uploaded = false;
        p->epoch = 0;
        CK(cudaMemset(p->ws, 0, L.pool));  // Ready table and all metadata start at zero
    }
    p->d_info = (int64_t*)p->ws;
    p->d_logdet = (double*)(p->ws + 256);
    p->d_logdet_parts = p->d_logdet + 1;
    p->d_slot = (int32_t*)(p->ws + L.slot);
    p->d_prev = (int32_t*)(p->ws + L.prev);
    p->d_epoch = (int*)(p->ws + L.epoch);
    p->d_entered = (int*)(p->ws + L.epoch + 64);
    p->d_flags = (int*)(p->ws + L.flags);
    p->flags_bytes = L.flags_bytes;
    p->d_expected = (int*)(p->ws + L.expected);
    p->d_items = (int4*)(p->ws + L.items);
    p->d_wbuf = (double*)(p->ws + L.wbuf);
    p->d_stats = (unsigned long long*)(p->ws + L.stats);
    p->d_prec = (uint8_t*)(p->ws + L.prec);
    p->d_amax_s = (double*)(p->ws + L.amax_s);
    p->d_iscale = (double*)(p->ws + L.iscale);
    p->d_args = (SchedArgs*)(p->ws + L.args);
    p->d_qtile = (uint8_t*)(p->ws + L.qtile);
    p->d_img = (long long*)(p->ws + L.img);
    p->d_oz_img = (long long*)(p->ws + L.ozimg);
    p->d_img_prev = (int32_t*)(p->ws + L.imgprev);
    p->d_oz_flag = (int*)(p->ws + L.ozflag);
    p->d_sto = (long long*)(p->ws + L.sto);
    p->d_in_scale = (double*)(p->ws + L.in_scale);
    p->d_solve = (double*)(p->ws + L.solve);
    p->d_shadow = (uint8_t*)(p->ws + L.shadow);
    p->d_amax_x = (unsigned long long*)(p->ws + L.flags + align_up(sizeof(int) * flag_ints(p), 8));
    p->pool = (double*)(p->ws + L.pool);
}

void ensure_streams(mxp_plan_s* p) {
    if (p->streams_ready) return;
    int lo, hi;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&p->sU, cudaStreamNonBlocking, lo));
    CK(cudaStreamCreateWithPriority(&p->sP, cudaStreamNonBlocking, hi));
    CK(cudaStreamCreateWithFlags(&p->sH2D, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&p->sD2H, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&p->sAux, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&p->sPush, cudaStreamNonBlocking));
    p->ev_panel.resize(p->Nt);
    p->ev_bulk.resize(p->Nt);
    for (int64_t k = 0; k < p->Nt; ++k) {
        CK(cudaEventCreateWithFlags(&p->ev_panel[k], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&p->ev_bulk[k], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p->ev_sched_end, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p->ev_potrf_end, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&p->sMain, cudaStreamNonBlocking));
    p->streams_ready = true;
}

// The stream a call orders its work on.  Single rank: the user's stream.
// Several ranks: a private stream joined after the user's pending work --
// co-located ranks may share one user stream (e.g. the legacy default
// stream), and a rank's start-barrier wait must not block its peers' work.
// Every entry point synchronizes this stream before returning.
cudaStream_t entry_stream(mxp_plan_s* p) {
    if (p->nranks <= 1) return p->user_stream;
    CK(cudaEventRecord(p->ev_join, p->user_stream));
    CK(cudaStreamWaitEvent(p->sMain, p->ev_join, 0));
    return p->sMain;
}

void dbg(mxp_plan_s* p, cudaStream_t s, const char* what) {
    CK(cudaGetLastError());
    if (p->debug_sync == 1) {
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
void timeline_begin(mxp_plan_s* p) {
    const size_t need = 3 * (size_t)p->Nt + 1;  // + [3 Nt]: the start (timing event beside ev_start)
    while (p->ev_tl.size() < need) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        p->ev_tl.push_back(e);
    }
    p->tl_rec.assign(need, 0);
    p->tl_ms.clear();
    p->tl_on = true;
}
void timeline_mark(mxp_plan_s* p, int64_t k, int row, cudaStream_t s) {  // row 0 H2D, 1 D2H, 2 POTRF
    if (!p->tl_on) return;
    CK(cudaEventRecord(p->ev_tl[3 * k + row], s));
    p->tl_rec[3 * k + row] = 1;
}
void timeline_collect(mxp_plan_s* p) {  // after every stream of the run has been synchronized
    if (!p->tl_on) return;
    p->tl_on = false;
    const size_t n3 = 3 * (size_t)p->Nt;
    p->tl_ms.assign(n3, -1.0);
    if (!p->tl_rec[n3]) return;
    for (size_t i = 0; i < n3; ++i)
        if (p->tl_rec[i]) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, p->ev_tl[n3], p->ev_tl[i]));
            p->tl_ms[i] = ms;
        }
}
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

// In-core FP64 factorization of the tiles already packed in the pool: one
// persistent static-schedule kernel on U + the POTRF kernels on P.
// Multi-GPU exchange: every tile this rank finishes is
// pushed, in schedule order, into each peer's pool by the copy engines (D2D
// over NVLink P2P -- no SM is taken from the persistent schedules), followed
// by its Ready word (= epoch), so peers use it exactly like a local tile.
// Diagonal tiles carry their W blocks (TRSM inverses) and log-det share;
// MxP tiles their amax.  Tiles of row k are needed by every rank at column k.
template <class T>
T* peer_addr(const mxp_plan_s* p, int q, const T* local) {
    return (T*)(p->peer_ws[q] + ((const char*)local - p->ws));
}
void push_tiles(mxp_plan_s* p, const SchedArgs& a) {
    const int64_t Nt = p->Nt, nb = p->nb, S = nb / 128;
    if (!stream_memops()) {
        g_last_error = "cuStreamWaitValue32 unavailable";
        throw CudaError{cudaErrorNotSupported};
    }
    CK(cudaStreamWaitEvent(p->sPush, p->ev_start, 0));
    for (int64_t n = 0; n < Nt; ++n)
        for (int64_t k = n; k < Nt; ++k) {
            if (k % p->nranks != p->rank) continue;
            const int64_t t = tile_index(Nt, k, n);
            if (g_wait32((CUstream)p->sPush, (CUdeviceptr)(a.ready + t), (cuuint32_t)p->epoch,
                         CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                throw CudaError{cudaErrorUnknown};
            const double* tile = p->pool + (size_t)p->slot_plan[t] * nb * nb;
            for (int q = 0; q < p->nranks; ++q) {
                if (q == p->rank) continue;
                CK(cudaMemcpyAsync(peer_addr(p, q, tile), tile, sizeof(double) * nb * nb, cudaMemcpyDeviceToDevice,
                                   p->sPush));
                if (k == n) {
                    const double* W = p->d_wbuf + (size_t)k * S * 128 * 128;
                    CK(cudaMemcpyAsync(peer_addr(p, q, W), W, sizeof(double) * S * 128 * 128,
                                       cudaMemcpyDeviceToDevice, p->sPush));
                    CK(cudaMemcpyAsync(peer_addr(p, q, p->d_logdet_parts + k), p->d_logdet_parts + k, sizeof(double),
                                       cudaMemcpyDeviceToDevice, p->sPush));
                }
                if (p->mxp)
                    CK(cudaMemcpyAsync(peer_addr(p, q, p->d_amax_s + t), p->d_amax_s + t, sizeof(double),
                                       cudaMemcpyDeviceToDevice, p->sPush));
                for (int e = 0; e < 4 && p->shadow_bytes > 0; ++e)  // the tile's operand images
                    if (p->img[4 * t + e] >= 0) {
                        const uint8_t* im = p->d_shadow + p->img[4 * t + e];
                        CK(cudaMemcpyAsync(peer_addr(p, q, im), im, sizeof(float) * nb * nb,
                                           cudaMemcpyDeviceToDevice, p->sPush));
                    }
                if (p->oz_on && p->oz_img[t] >= 0) {  // int8 slice image + row scales (Ozaki engine)
                    const uint8_t* im = p->d_shadow + p->oz_img[t];
                    CK(cudaMemcpyAsync(peer_addr(p, q, im), im, (size_t)oz::image_bytes(p->oz_slices, nb),
                                       cudaMemcpyDeviceToDevice, p->sPush));
                }
                CK(cudaMemcpyAsync(peer_addr(p, q, a.ready + t), p->d_epoch, sizeof(int), cudaMemcpyDeviceToDevice,
                                   p->sPush));
            }
        }
}

// Ready words hold the epoch (factorization counter) of the run that made the
// tile final, so they are never cleared between runs: stale values compare
// below the current epoch (cuStreamWaitValue32 GEQ is a cyclic comparison).
// The rest of the flag area is reset per run.  With several ranks this is
// followed by a start barrier: every rank writes its epoch into each peer's
// entered[rank] word after its own resets (stream order on s0) and waits for
// all peers' words before any kernel of the run -- no peer pushes into this
// pool, or writes its Ready/info words, before they have been reset, and a
// peer enters run e+1 only after its run-e pushes into this pool completed.
void begin_epoch(mxp_plan_s* p, cudaStream_t s0) {
    // (ranks run the same sequence of factorizations, so their epochs agree)
    if (++p->epoch >= (1 << 24)) p->epoch = 1, p->ready_dirty = true;
    if (p->ready_dirty) {  // clear the table
        CK(cudaMemsetAsync(p->d_flags + 2, 0, sizeof(int) * p->T, s0));
        p->ready_dirty = false;
    }
    CK(cudaMemsetAsync(p->d_flags, 0, 2 * sizeof(int), s0));  // ticket, err
    const size_t rest = 2 * sizeof(int) + sizeof(int) * p->T;
    CK(cudaMemsetAsync((char*)p->d_flags + rest, 0, p->flags_bytes - rest, s0));
    if (p->nranks <= 1) {
        CK(cudaMemcpyAsync(p->d_epoch, &p->epoch, sizeof(int), cudaMemcpyHostToDevice, s0));
        return;
    }
    if (!stream_memops()) {
        g_last_error = "multi-rank factorization needs cuStreamWaitValue32";
        throw CudaError{cudaErrorNotSupported};
    }
    for (int q = 0; q < p->nranks; ++q)
        if (!p->peer_ws[q] && q != p->rank) {
            g_last_error = "peer workspace of rank " + std::to_string(q) + " not attached";
            throw CudaError{cudaErrorInvalidValue};
        }
    const cuuint32_t e = (cuuint32_t)p->epoch;
    if (g_write32((CUstream)s0, (CUdeviceptr)p->d_epoch, e, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
        throw CudaError{cudaErrorUnknown};
    for (int q = 0; q < p->nranks; ++q)
        if (q != p->rank &&
            g_write32((CUstream)s0, (CUdeviceptr)peer_addr(p, q, p->d_entered + p->rank), e,
                      CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
            throw CudaError{cudaErrorUnknown};
    for (int q = 0; q < p->nranks; ++q)
        if (q != p->rank &&
            g_wait32((CUstream)s0, (CUdeviceptr)(p->d_entered + q), e, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
            throw CudaError{cudaErrorUnknown};
}

// tile index of the last tile rank q pushes (push order of push_tiles), -1 if none
int64_t last_pushed_tile(const mxp_plan_s* p, int q) {
    int64_t last = -1;
    for (int64_t n = 0; n < p->Nt; ++n)
        for (int64_t k = n; k < p->Nt; ++k)
            if (k % p->nranks == q) last = tile_index(p->Nt, k, n);
    return last;
}

// where the final tiles of the compact pool live (storage images) for unpack / solve
TileCodes decode_args(const mxp_plan_s* p) {
    TileCodes d{};
    if (p->compact) {
        d.sto = p->d_sto;
        d.shadow = p->d_shadow;
        d.prec = p->d_prec;
        d.scale = p->d_iscale;
    }
    return d;
}

struct GenSource {  // fused on-device generation of the input tiles (N2)
    const double* xy = nullptr;
    double sigma2 = 1.0, range = 1.0, nugget = 0.0;
};

// what the first timed-out wait of the static schedule was waiting for
std::string sched_timeout_detail(mxp_plan_s* p) {
    const size_t nf = flag_ints(p);
    std::vector<int> f(nf);
    if (cudaMemcpy(f.data(), p->d_flags, sizeof(int) * nf, cudaMemcpyDeviceToHost) != cudaSuccess) {
        cudaGetLastError();
        return "";
    }
    const int* d = f.data() + nf - 1 - 256 - 24;
    if (!d[7]) return "";
    const int64_t T = p->T, NB = blocks_per_tile(p->nb);
    int64_t o = d[0];
    static const char* names[] = {"ready", "gemm_done", "trsm_done", "quant_done", "loaded", "prep_done"};
    std::string what;
    if (o >= 0 && o < 6 * T) {
        int64_t t = o % T, m = 0, n = 0;
        tile_coords(p->Nt, t, m, n);
        what = std::string(names[o / T]) + "(" + std::to_string(m) + "," + std::to_string(n) + ")";
    } else if (o >= 6 * T && o < 6 * T + T * NB) {
        int64_t t = (o - 6 * T) / NB, b = (o - 6 * T) % NB, m = 0, n = 0;
        tile_coords(p->Nt, t, m, n);
        what = "blk_chunk(" + std::to_string(m) + "," + std::to_string(n) + ") block " + std::to_string(b);
    } else {
        what = "flag offset " + std::to_string(o);
    }
    // progress of the first tile column (ready / trsm_done / quant_done / gemm_done of tiles (m, 0))
    std::string col0;
    for (int64_t m = 0; m < std::min<int64_t>(p->Nt, 4); ++m) {
        const int64_t t = tile_index(p->Nt, m, 0);
        col0 += " (" + std::to_string(m) + ",0):" + std::to_string(f[2 + t]) + "/" + std::to_string(f[2 + 2 * T + t]) +
                "/" + std::to_string(f[2 + 3 * T + t]) + "/" + std::to_string(f[2 + T + t]);
    }
    return " [first timeout: " + what + " target " + std::to_string(d[1]) + " value " + std::to_string(d[2]) +
           "; column 0 ready/trsm/quant/gemm" + col0 + "; k_tc CTAs started/ended " + std::to_string(d[8]) + "/" +
           std::to_string(d[9]) + ", k_sched " + std::to_string(d[10]) + "/" + std::to_string(d[11]) +
           ", k_tc GEMM tasks begun/done " + std::to_string(d[12]) + "/" + std::to_string(d[13]) +
           ", k_tc first start - k_sched first start " + std::to_string(d[14] - d[15]) + " us" +
           ", k_tc CTAs launched " + std::to_string(d[16]) + " first launch - k_sched start " +
           std::to_string(d[17] - d[15]) + " us" +
           " column " + std::to_string(d[6]) + " sm " + std::to_string(d[3]) + " block " + std::to_string(d[4]) + "/" +
           std::to_string(d[5]) + "; tickets k_sched " + std::to_string(f[0]) + "/" + std::to_string(p->items.size()) +
           " k_tc " + std::to_string(f[nf - 1]) + "/" + std::to_string(p->items2.size()) + "]";
}

void factor_incore_f64(mxp_plan_s* p, cudaStream_t s0, bool host_mode, double* A_host = nullptr,
                       int64_t lda = 0, const GenSource* gen = nullptr, const double* srcA = nullptr) {
    const int64_t Nt = p->Nt, T = p->T;
    if (p->host_mode != host_mode) {
        p->host_mode = host_mode;
        p->list_uploaded = false;
    }
    if (!p->list_uploaded) {
        build_task_list(p);
        CK(cudaMemcpyAsync(p->d_items, p->items.data(), sizeof(int4) * p->items.size(), cudaMemcpyHostToDevice, s0));
        if (!p->items2.empty())
            CK(cudaMemcpyAsync(p->d_items + p->items.size(), p->items2.data(), sizeof(int4) * p->items2.size(),
                               cudaMemcpyHostToDevice, s0));
        CK(cudaMemcpyAsync(p->d_oz_img, p->oz_img.data(), sizeof(long long) * T, cudaMemcpyHostToDevice, s0));
        if (p->oz_ooc)
            CK(cudaMemcpyAsync(p->d_img_prev, p->img_prev.data(), sizeof(int32_t) * T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemcpyAsync(p->d_expected, p->expected.data(), sizeof(int) * T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemcpyAsync(p->d_prec, p->map.data(), (size_t)T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemcpyAsync(p->d_qtile, p->qtile.data(), (size_t)T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemcpyAsync(p->d_img, p->img.data(), sizeof(long long) * 4 * T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemcpyAsync(p->d_sto, p->sto.data(), sizeof(long long) * T, cudaMemcpyHostToDevice, s0));
        CK(cudaStreamSynchronize(s0));
        p->list_uploaded = true;
    }
    begin_epoch(p, s0);
    if (p->mxp && !p->host_mode) {
        // O3: stored input A^ = deq(q_p(A)) per tile; amax_x is then reset for the TRSM outputs
        Prof pr(p, s0, MXP_KCLASS_OTHER, 0.0, 2);
        launch_input_quantize(p->pool, p->d_slot, p->d_prec, Nt, p->nb, p->d_amax_x, p->d_amax_s, s0, p->rank,
                              p->nranks);
        p->launches += 2;
        CK(cudaMemsetAsync(p->d_amax_x, 0, sizeof(unsigned long long) * T, s0));
    }
    if (p->debug_sync == 2) {  // GEMM-throughput probe: every tile "ready", no POTRF (values are garbage)
        CK(cudaMemsetAsync(p->d_flags + 2, 1, sizeof(int) * T, s0));
        p->ready_dirty = true;
    }
    CK(cudaEventRecord(p->ev_start, s0));
    if (p->tl_on) {  // timeline origin (ev_start has timing disabled)
        CK(cudaEventRecord(p->ev_tl[3 * Nt], s0));
        p->tl_rec[3 * Nt] = 1;
    }
    CK(cudaStreamWaitEvent(p->sU, p->ev_start, 0));
    CK(cudaStreamWaitEvent(p->sP, p->ev_start, 0));
    if (p->oz_on) {
        // The two persistent kernels of the Ozaki mode must share every SM (one
        // k_tc + one k_sched CTA).  When both wait on the same event (e.g. behind
        // the input quantization), k_sched CTAs were observed to land first and
        // keep k_tc off the SMs until the 20 s scheduler timeout; launched in host
        // order onto idle streams, k_tc lands first.  So the host waits for the
        // preceding work (a few microseconds after it ends) before the launches.
        CK(cudaEventSynchronize(p->ev_start));
        if (!p->sT) {  // created only when used: every stream takes a hardware queue, and parked
                       // streams (stream memory waits) must not share one with the others
            int lo = 0, hi = 0;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CK(cudaStreamCreateWithPriority(&p->sT, cudaStreamNonBlocking, lo));
        }
        CK(cudaStreamWaitEvent(p->sT, p->ev_start, 0));
    }

    SchedArgs a{};
    a.pool = p->pool;
    a.slot = p->d_slot;
    a.dinfo = p->d_info;
    a.counter = p->d_flags;
    a.err = p->d_flags + 1;
    a.ready = p->d_flags + 2;
    a.gemm_done = a.ready + T;
    a.trsm_done = a.gemm_done + T;
    a.quant_done = a.trsm_done + T;
    int* loaded = a.quant_done + T;
    a.prep_done = loaded + T;
    a.blk_chunk = a.prep_done + T;
    a.potrf_claim = a.blk_chunk + T * blocks_per_tile(p->nb);
    a.col_ready = a.potrf_claim + Nt;
    int* d2h_done = a.col_ready + Nt;
    a.logdet_parts = p->d_logdet_parts;
    a.loaded = (p->host_mode && !gen && !srcA) ? loaded : nullptr;
    a.src_A = srcA;  // compact device path: PREP copies tile (m, k) from the caller's matrix
    a.src_lda = lda;
    a.compact = p->compact ? 1 : 0;
    a.sto = p->compact ? p->d_sto : nullptr;
    a.tile_codes = p->tiles_io ? 1 : 0;  // input tiles arrive as codes in their storage images
    a.in_scale = p->d_in_scale;
    a.n = p->n;
    a.gen_mode = gen ? 1 : 0;
    a.prev_owner = p->d_prev;
    if (gen) {
        a.gen_xy = gen->xy;
        a.gen_sigma2 = gen->sigma2;
        a.gen_range = gen->range;
        a.gen_nugget = gen->nugget;
    }
    a.prec = (p->mxp || p->oz_on) ? p->d_prec : nullptr;
    a.oz_img = p->oz_on ? p->d_oz_img : nullptr;
    a.oz_slices = p->oz_slices;
    a.oz_flag = p->oz_on ? p->d_oz_flag : nullptr;
    if (a.oz_flag) CK(cudaMemsetAsync(p->d_oz_flag, 0, sizeof(int) * (size_t)T, s0));
    a.oz_prefetch = p->oz_prefetch;
    a.img_prev = p->oz_ooc ? p->d_img_prev : nullptr;
    a.ring_all = p->oz_ooc ? 1 : 0;
    a.items2 = p->d_items + p->items.size();
    a.nitems2 = (int)p->items2.size();
    a.counter2 = p->d_flags + flag_ints(p) - 1;
    a.sm_claim = a.counter2 - 256;
    a.tdiag = a.sm_claim - 24;
    a.task_claim = a.tdiag - (2 * T * (p->nb / 64) + T);
    a.qtile = p->d_qtile;
    a.img = (p->mxp && p->shadow_bytes > 0) ? p->d_img : nullptr;  // (null when no fp32 image exists)
    a.shadow = p->d_shadow;
    a.tc_engine = p->tc_engine;
    a.native = p->nat_on ? 1 : 0;
    a.iscale = p->d_iscale;
    a.amax_x = p->d_amax_x;
    a.amax_s = p->d_amax_s;
    a.gemm_expected = p->d_expected;
    a.Nt = Nt;
    a.nb = p->nb;
    a.KC = p->splitk_tiles;
    a.NB = blocks_per_tile(p->nb);
    a.items = p->d_items;
    a.nitems = (int)p->items.size();
    a.wbuf = p->d_wbuf;
    a.reserved_sms = p->reserved_sms;
    a.epoch = p->epoch;
    a.rank = p->rank;
    a.nranks = p->nranks;
    for (int q = 0; q < MAX_RANKS; ++q)
        a.peer_dinfo[q] = (q != p->rank && q < p->nranks && p->peer_ws[q]) ? (int64_t*)p->peer_ws[q] : nullptr;
    a.stats = nullptr;
    const size_t nstat = STAT_POTRF + 3 * (size_t)Nt;
    if (p->profile) {
        std::vector<unsigned long long> init(nstat, 0ull);
        init[STAT_T0] = ~0ull;
        CK(cudaMemcpyAsync(p->d_stats, init.data(), sizeof(unsigned long long) * nstat, cudaMemcpyHostToDevice, s0));
        CK(cudaStreamSynchronize(s0));
        a.stats = p->d_stats;
    }

    int dev = p->device, nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    a.sm_lo = p->sm_count > 0 ? p->sm_first : 0;
    a.sm_hi = p->sm_count > 0 ? std::min(nsm, p->sm_first + p->sm_count) : nsm;
    int occ = sched_ctas_per_sm();
    // algorithmic flops of this rank's tasks: row m of L costs (m^2 + m) nb^3
    // in GEMM/SYRK/TRSM (sum over all rows: n^3/3 - Nt nb^3/3) + nb^3/3 POTRF
    const double nb3 = (double)p->nb * p->nb * p->nb;
    double chain_flops = 0.0, potrf_flops = 0.0;
    for (int64_t m = p->rank; m < Nt; m += p->nranks) {
        chain_flops += ((double)m * m + (double)m) * nb3;
        potrf_flops += nb3 / 3.0;
    }
    if (!p->oz_on) {
        Prof pr(p, p->sU, MXP_KCLASS_CHAIN, chain_flops);
        p->h_args = a;
        CK(cudaMemcpyAsync(p->d_args, &p->h_args, sizeof(SchedArgs), cudaMemcpyHostToDevice, p->sU));
        launch_sched(a, p->d_args, p->mxp, occ * nsm, p->sU);
        ++p->launches;
        dbg(p, p->sU, "sched");
    } else {
        // Ozaki mode: the GEMM kernel (one CTA per SM, all TMEM) on sT beside
        // one k_sched CTA per SM (TRSM / QUANT / PREP / POTRF fallback) on sU
        // (measured: k_tc alone with a 5-stage ring and the TRSM / QUANT tasks
        // in its own list order ran C2 at 60.7 TF/s vs 65.0 co-scheduled)
        double trsm_flops = 0.0;
        for (int64_t m = p->rank; m < Nt; m += p->nranks) trsm_flops += (double)m * nb3;
        p->h_args = a;
        CK(cudaMemcpyAsync(p->d_args, &p->h_args, sizeof(SchedArgs), cudaMemcpyHostToDevice, p->sU));
        CK(cudaEventRecord(p->ev_join, p->sU));
        CK(cudaStreamWaitEvent(p->sT, p->ev_join, 0));
        {
            Prof pr(p, p->sT, MXP_KCLASS_CHAIN, chain_flops - trsm_flops);
            launch_tc(p->d_args, nsm, p->sT, p->nat_on);
            ++p->launches;
        }
        dbg(p, p->sT, "tc");  // (debug_sync = 1: k_tc then runs the whole schedule alone)
        {
            Prof pr(p, p->sU, MXP_KCLASS_TRSM, trsm_flops);
            launch_sched(a, p->d_args, true, nsm, p->sU);
            ++p->launches;
        }
        dbg(p, p->sU, "sched");
        CK(cudaEventRecord(p->ev_join, p->sT));
        CK(cudaStreamWaitEvent(p->sU, p->ev_join, 0));
    }
    {
        Prof pr(p, p->sP, MXP_KCLASS_POTRF, potrf_flops, (Nt - p->rank + p->nranks - 1) / p->nranks);
        if (p->debug_sync != 2 && p->debug_sync != 3) {  // 3: every POTRF by the scheduler fallback
            for (int64_t k = p->rank; k < Nt; k += p->nranks) {  // diagonal tiles this rank owns
                launch_potrf_tile(a, k, p->sP);
                ++p->launches;
                timeline_mark(p, k, 2, p->sP);
            }
        }
        CK(cudaGetLastError());
    }
    // The copy streams park on stream memory waits, and a stream's command
    // queue is finite: an enqueue into a full queue blocks the calling host
    // thread.  So each stream that can park is fed by its own host thread --
    // a blocked H2D enqueue (waiting for a slot to die) must never keep the D2H
    // writes or the peer pushes that make it die from being enqueued.
    std::vector<std::thread> feeders;
    std::vector<std::string> feeder_err;
    std::mutex feeder_mu;
    auto feed = [&](auto body) {
        feeders.emplace_back([&, body] {
            try {
                if (cudaSetDevice(p->device) != cudaSuccess) throw CudaError{cudaErrorInvalidDevice};
                body();
            } catch (const CudaError& e) {
                std::lock_guard<std::mutex> g(feeder_mu);
                feeder_err.push_back(g_last_error.empty() ? cudaGetErrorString(e.e) : g_last_error);
            }
        });
    };
    auto join_all = [&] {
        for (auto& th : feeders) th.join();
        feeders.clear();
    };
    int64_t d2h_bytes = 0;  // (outlives the feeders: they are joined on every path)
    // Failure watcher: the copy streams park on Ready / column words that a
    // failed column (info != 0) or a scheduler timeout never sets, and a
    // feeder blocked in an enqueue into a parked stream's full queue would
    // never return.  So the release is independent of the feeders: once the
    // schedule kernels have ended, a failed run's Ready and column words are
    // set to a value above every epoch, which drains every parked stream.
    CK(cudaEventRecord(p->ev_sched_end, p->sU));
    CK(cudaEventRecord(p->ev_potrf_end, p->sP));
    if (host_mode || p->nranks > 1)
        feed([&] {
            CK(cudaEventSynchronize(p->ev_sched_end));
            CK(cudaEventSynchronize(p->ev_potrf_end));
            int64_t hinfo = 0;
            int herr = 0;
            CK(cudaMemcpyAsync(&hinfo, p->d_info, sizeof(int64_t), cudaMemcpyDeviceToHost, p->sAux));
            CK(cudaMemcpyAsync(&herr, a.err, sizeof(int), cudaMemcpyDeviceToHost, p->sAux));
            CK(cudaStreamSynchronize(p->sAux));
            if (hinfo != 0 || herr || p->debug_sync == 2) {
                CK(cudaMemsetAsync(a.ready, 0x7f, sizeof(int) * T, p->sAux));
                CK(cudaMemsetAsync(a.col_ready, 0x7f, sizeof(int) * Nt, p->sAux));
                CK(cudaStreamSynchronize(p->sAux));
                p->ready_dirty = true;
            }
        });
    if (p->nranks > 1) feed([&] { push_tiles(p, a); });
    if (host_mode && !gen && !srcA) try {
        // H2D in schedule (column) order; the GPU front-end publishes loaded[t]
        CK(cudaStreamWaitEvent(p->sH2D, p->ev_start, 0));
        CK(cudaStreamWaitEvent(p->sD2H, p->ev_start, 0));
        const int64_t nb = p->nb, n = p->n;
        feed([&, nb, n] {
            // D2H of each finished tile as soon as Ready(t) flips (lower triangle only);
            // diagonal tiles go to a pinned stage and only their lower triangle is merged
            for (int64_t k = 0; k < Nt; ++k) {
                for (int64_t m = k; m < Nt; ++m) {
                    if (m % p->nranks != p->rank) continue;
                    const int64_t t = tile_index(Nt, m, k);
                    const int64_t rr = std::min(nb, n - m * nb), cr = std::min(nb, n - k * nb);
                    if (g_wait32((CUstream)p->sD2H, (CUdeviceptr)(a.ready + t), (cuuint32_t)p->epoch,
                                 CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                        throw CudaError{cudaErrorUnknown};
                    const double* src = p->pool + (size_t)p->slot_plan[t] * nb * nb;
                    if (p->tiles_io) {  // tile-packed host storage: the tile at its storage precision
                        const int pt = p->map[t];
                        const size_t bytes = (size_t)nb * nb * (pt == MXP_FP64 ? 8 : pt == MXP_FP32 ? 4 : pt == MXP_FP16 ? 2 : 1);
                        const void* s2 = pt == MXP_FP64 ? (const void*)src : (const void*)(p->d_shadow + p->sto[t]);
                        CK(cudaMemcpyAsync(p->tiles_io[t], s2, bytes, cudaMemcpyDeviceToHost, p->sD2H));
                        d2h_bytes += (int64_t)bytes;
                    } else if (m != k) {
                        CK(cudaMemcpy2DAsync(A_host + (size_t)k * nb * lda + (size_t)m * nb, sizeof(double) * lda, src,
                                             sizeof(double) * nb, sizeof(double) * rr, cr, cudaMemcpyDeviceToHost, p->sD2H));
                        d2h_bytes += (int64_t)(sizeof(double) * rr * cr);
                    } else {
                        CK(cudaMemcpyAsync(p->h_stage + (size_t)k * nb * nb, src, sizeof(double) * nb * nb,
                                           cudaMemcpyDeviceToHost, p->sD2H));
                        d2h_bytes += (int64_t)(sizeof(double) * nb * nb);
                    }
                    if (g_write32((CUstream)p->sD2H, (CUdeviceptr)(d2h_done + t), 1, CU_STREAM_WRITE_VALUE_DEFAULT) !=
                        CUDA_SUCCESS)
                        throw CudaError{cudaErrorUnknown};
                }
                timeline_mark(p, k, 1, p->sD2H);
            }
        });
        for (int64_t k = 0; k < Nt; ++k) {
            for (int64_t m = k; m < Nt; ++m) {
                if (m % p->nranks != p->rank) continue;  // peers stream their own rows
                const int64_t t = tile_index(Nt, m, k);
                const int64_t rr = std::min(nb, n - m * nb), cr = std::min(nb, n - k * nb);
                double* dst = p->pool + (size_t)p->slot_plan[t] * nb * nb;
                const double* src = A_host ? A_host + (size_t)k * nb * lda + (size_t)m * nb : nullptr;
                const int32_t prev = p->prev_owner[t];
                const bool coded = p->tiles_io && p->map[t] != MXP_FP64;
                if (coded) {  // codes into the tile's storage image; the PREP task waits for the slot
                    const int pt = p->map[t];
                    const size_t bytes = (size_t)nb * nb * (pt == MXP_FP32 ? 4 : pt == MXP_FP16 ? 2 : 1);
                    CK(cudaMemcpyAsync(p->d_shadow + p->sto[t], p->tiles_io[t], bytes, cudaMemcpyHostToDevice, p->sH2D));
                    if (g_write32((CUstream)p->sH2D, (CUdeviceptr)(a.loaded + t), 1, CU_STREAM_WRITE_VALUE_DEFAULT) !=
                        CUDA_SUCCESS)
                        throw CudaError{cudaErrorUnknown};
                    p->h2d += (int64_t)bytes;
                    continue;
                }
                if (prev >= 0) {  // out of core / compact: the slot's previous tile must be dead and written back
                    int64_t pm = 0, pc = 0;
                    tile_coords(Nt, prev, pm, pc);
                    // compact / Ozaki ring: an off-diagonal tile dies when it is final (its readers
                    // use images); out of core, and a diagonal tile of the Ozaki ring (read by the
                    // TRSMs of its column): when column pm is final
                    const bool ok = (p->compact || p->oz_ooc) && pm != pc
                        ? g_wait32((CUstream)p->sH2D, (CUdeviceptr)(a.ready + prev), (cuuint32_t)p->epoch,
                                   CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS
                        : g_wait32((CUstream)p->sH2D, (CUdeviceptr)(a.col_ready + (p->oz_ooc ? pc : pm)),
                                   (cuuint32_t)(Nt - (p->oz_ooc ? pc : pm)), CU_STREAM_WAIT_VALUE_GEQ) == CUDA_SUCCESS;
                    if (!ok ||
                        g_wait32((CUstream)p->sH2D, (CUdeviceptr)(d2h_done + prev), 1, CU_STREAM_WAIT_VALUE_GEQ) !=
                            CUDA_SUCCESS)
                        throw CudaError{cudaErrorUnknown};
                }
                if (p->tiles_io) {  // an FP64 tile: nb x nb doubles straight into its slot
                    CK(cudaMemcpyAsync(dst, p->tiles_io[t], sizeof(double) * nb * nb, cudaMemcpyHostToDevice, p->sH2D));
                    p->h2d += (int64_t)(sizeof(double) * nb * nb);
                } else {
                    CK(cudaMemcpy2DAsync(dst, sizeof(double) * nb, src, sizeof(double) * lda, sizeof(double) * rr, cr,
                                         cudaMemcpyHostToDevice, p->sH2D));
                    p->h2d += (int64_t)(sizeof(double) * rr * cr);
                }
                if (g_write32((CUstream)p->sH2D, (CUdeviceptr)(a.loaded + t), 1, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
                    throw CudaError{cudaErrorUnknown};
            }
            timeline_mark(p, k, 0, p->sH2D);
        }
        join_all();
        p->d2h += d2h_bytes;
    } catch (...) {
        join_all();
        throw;
    }
    join_all();
    if (!feeder_err.empty()) {
        g_last_error = "copy-stream feeder: " + feeder_err[0];
        throw CudaError{cudaErrorUnknown};
    }
    CK(cudaEventRecord(p->ev_done, p->sP));
    CK(cudaStreamWaitEvent(p->sU, p->ev_done, 0));
}

// Multi-rank epilogue: once this rank's schedule has ended, a failure (info)
// leaves Ready words unset that the push stream waits on -- release them so
// the stream drains -- then order the pushes before s0.
void finish_pushes(mxp_plan_s* p, cudaStream_t s0) {
    if (p->nranks <= 1) {
        return;
    }
    CK(cudaStreamSynchronize(p->sU));
    int64_t hinfo = 0;
    int herr = 0;
    CK(cudaMemcpy(&hinfo, p->d_info, sizeof(int64_t), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&herr, p->d_flags + 1, sizeof(int), cudaMemcpyDeviceToHost));
    const bool failed = hinfo != 0 || herr || p->debug_sync == 2;
    if (failed) {  // release the push stream's waits (the pushed tiles are not a result)
        CK(cudaMemsetAsync(p->d_flags + 2, 0x7f, sizeof(int) * p->T, p->sAux));
        CK(cudaStreamSynchronize(p->sAux));
    }
    CK(cudaEventRecord(p->ev_start, p->sPush));
    CK(cudaStreamWaitEvent(s0, p->ev_start, 0));
    if (!failed) {
        // every peer's pushes into this pool have landed: each peer pushes in
        // one stream, so its last Ready write orders all its earlier copies
        for (int q = 0; q < p->nranks; ++q) {
            const int64_t t = q == p->rank ? -1 : last_pushed_tile(p, q);
            if (t >= 0 && g_wait32((CUstream)s0, (CUdeviceptr)(p->d_flags + 2 + t), (cuuint32_t)p->epoch,
                                   CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                throw CudaError{cudaErrorUnknown};
        }
    } else {
        p->ready_dirty = true;  // drained words are ahead of every later epoch
    }
}

int status_from_exception(const CudaError& e) {
    if (e.e == cudaErrorMemoryAllocation) return MXP_ENOMEM;
    if (e.e == cudaErrorInvalidValue) return MXP_ESTATE;
    return MXP_ECUDA;
}

}  // namespace

// ---- single-process multi-GPU (a group plan: one sub-plan per GPU) ----------
bool is_group(const mxp_plan_s* p) { return p && !p->group.empty(); }
// attach every sub-plan to every other (in-process peer pools; re-done before
// every run: a sub-plan whose workspace was re-sized has dropped its peers)
int group_attach(mxp_plan_s* g) {
    const int P = (int)g->group.size();
    for (int r = 0; r < P; ++r)
        for (int q = 0; q < P; ++q)
            if (q != r) {
                const int rc = mxp_chol_attach_peer_plan(g->group[r], q, g->group[q]);
                if (rc != MXP_OK) return rc;
            }
    return MXP_OK;
}
// fn(sub-plan, &info) on every sub-plan, each from its own host thread (the
// sub-plans' schedules wait on each other's pushed tiles); first error wins
template <class F>
int group_run(mxp_plan_s* g, int64_t* info, F fn) {
    g->have_result = false;
    int rc = group_attach(g);
    if (rc != MXP_OK) return rc;
    const int P = (int)g->group.size();
    std::vector<int> st(P, MXP_OK);
    std::vector<int64_t> inf(P, 0);
    std::vector<std::string> err(P);
    std::vector<std::thread> th;
    for (int r = 0; r < P; ++r)
        th.emplace_back([&, r] {
            st[r] = fn(g->group[r], &inf[r]);
            if (st[r] != MXP_OK) err[r] = g_last_error;
        });
    for (auto& t : th) t.join();
    for (int r = 0; r < P; ++r)
        if (st[r] != MXP_OK) {
            g_last_error = "rank " + std::to_string(r) + ": " + err[r];
            return st[r];
        }
    *info = inf[0];  // (a failed pivot is propagated to every rank)
    g->have_result = g->group[0]->have_result;
    g->logdet = g->group[0]->logdet;
    return MXP_OK;
}

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
    if (ngpus < 1 || ngpus > MAX_RANKS) return -4;
    if (!out) return -5;
    if (ngpus > 1) {
        // Single-process multi-GPU: one sub-plan per GPU in the row-cyclic
        // distribution (rank r = GPU r mod #devices, tile row m on rank m mod ngpus), attached
        // to each other in process (peer access).  With fewer devices than ranks the ranks
        // sharing a device split its SMs (the co-located test setup).
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) {
            cudaGetLastError();
            g_last_error = "ngpus > 1: no CUDA device";
            return MXP_ECUDA;
        }
        std::vector<mxp_plan_s*> kids;
        for (int r = 0; r < ngpus; ++r) {
            mxp_plan_t c = nullptr;
            const int rc = mxp_chol_plan(n, nb, precision_map, 1, &c);
            if (rc != MXP_OK) {
                for (auto* k : kids) delete k;
                return rc;
            }
            c->rank = r;
            c->nranks = ngpus;
            c->device = r % ndev;
            c->in_group = true;
            kids.push_back(c);
        }
        for (int r = 0; r < ngpus; ++r) {  // SM partitions of co-located ranks
            int share = 0, idx = 0;
            for (int q = 0; q < ngpus; ++q)
                if (kids[q]->device == kids[r]->device) idx += (q < r), ++share;
            if (share > 1) {
                // one SM stays outside every partition: a device-to-device copy between two
                // pools on the same GPU runs as a copy kernel, which must find an SM that the
                // persistent schedules do not hold (on separate GPUs the copy engines move it)
                int nsm = 0;
                cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, kids[r]->device);
                cudaGetLastError();
                kids[r]->sm_first = idx * ((nsm - 1) / share);
                kids[r]->sm_count = (nsm - 1) / share;
            }
        }
        auto* g = new mxp_plan_s();
        g->n = n;
        g->nb = nb;
        g->Nt = kids[0]->Nt;
        g->T = kids[0]->T;
        g->map = kids[0]->map;
        g->mxp = kids[0]->mxp;
        g->device = kids[0]->device;
        g->group = std::move(kids);
        *out = g;
        return MXP_OK;
    }
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
    }
    {  // every kernel loaded now, before any persistent kernel can be running (CUDA lazy
       // loading at a first launch can wait for running kernels; co-located ranks deadlock)
        static std::once_flag once;
        std::call_once(once, [] {
            preload_sched();
            preload_layout();
            preload_solve();
            preload_generators();
        });
    }
    auto* p = new mxp_plan_s();
    p->n = n;
    p->nb = nb;
    p->Nt = Nt;
    p->T = T;
    p->map = std::move(map);
    for (auto c : p->map) p->mxp |= (c != MXP_FP64);
    cudaGetDevice(&p->device);
    *out = p;
    return MXP_OK;
}

int mxp_chol_plan_set(mxp_plan_t p, mxp_attr_t key, int64_t v) {
    if (!p) return -1;
    if (is_group(p)) {  // the group places its ranks itself; the user stream orders rank 0
        if (key == MXP_ATTR_DEVICE || key == MXP_ATTR_RANK || key == MXP_ATTR_NRANKS || key == MXP_ATTR_SM_FIRST ||
            key == MXP_ATTR_SM_COUNT)
            return MXP_ENOTSUP;
        if (key == MXP_ATTR_STREAM) return mxp_chol_plan_set(p->group[0], key, v);
        for (auto* c : p->group) {
            const int rc = mxp_chol_plan_set(c, key, v);
            if (rc != MXP_OK) return rc;
        }
        return MXP_OK;
    }
    switch (key) {
    case MXP_ATTR_DEVICE:
        if (p->ws || p->streams_ready) return MXP_ESTATE;
        p->device = (int)v;
        return MXP_OK;
    case MXP_ATTR_STREAM: p->user_stream = (cudaStream_t)(intptr_t)v; return MXP_OK;
    case MXP_ATTR_HBM_BYTES_CAP:
        if (v < 0) return -3;
        if (p->ws && !p->ws_owned) return MXP_ESTATE;  // changes the workspace size
        if (p->ws_owned) {
            cudaFree(p->ws);
            p->ws = nullptr;
            p->ws_owned = false;
        }
        p->hbm_cap = v;
        return MXP_OK;
    case MXP_ATTR_SPLITK_TILES:
        if (v < 1 || v > 4096) return -3;
        p->list_uploaded = false;
        if (p->ws && !p->ws_owned) return MXP_ESTATE;
        if (p->ws_owned) {
            cudaFree(p->ws);
            p->ws = nullptr;
            p->ws_owned = false;
        }
        p->splitk_tiles = v;
        return MXP_OK;
    case MXP_ATTR_LOOKAHEAD: p->lookahead = v ? 1 : 0; return MXP_OK;
    case MXP_ATTR_DEBUG_SYNC:
        if (v < 0 || v > 3) return -3;
        if ((v == 2) != (p->debug_sync == 2)) p->list_uploaded = false;
        p->debug_sync = (int)v;
        return MXP_OK;
    case MXP_ATTR_PROFILE: p->profile = v ? 1 : 0; return MXP_OK;
    case MXP_ATTR_RANK:
    case MXP_ATTR_NRANKS:
        if (key == MXP_ATTR_RANK && (v < 0 || v >= MAX_RANKS)) return -3;
        if (key == MXP_ATTR_NRANKS && (v < 1 || v > MAX_RANKS)) return -3;
        // nranks is part of the image plan (workspace layout): drop an owned
        // workspace, refuse a user one that may no longer fit
        if (p->ws && !p->ws_owned && key == MXP_ATTR_NRANKS && v != p->nranks) return MXP_ESTATE;
        if (p->ws_owned && (key == MXP_ATTR_NRANKS ? v != p->nranks : v != p->rank)) {
            cudaFree(p->ws);
            p->ws = nullptr;
            p->ws_owned = false;
            for (int q = 0; q < MAX_RANKS; ++q)
                if (p->peer_ws[q] && p->peer_ipc[q]) cudaIpcCloseMemHandle(p->peer_ws[q]);
            for (int q = 0; q < MAX_RANKS; ++q) p->peer_ws[q] = nullptr, p->peer_ipc[q] = false;
        }
        if (key == MXP_ATTR_RANK) p->rank = (int)v;
        else p->nranks = (int)v;
        p->list_uploaded = false;
        return MXP_OK;
    case MXP_ATTR_SM_FIRST:
        if (v < 0) return -3;
        p->sm_first = (int)v;
        return MXP_OK;
    case MXP_ATTR_SM_COUNT:
        if (v < 0) return -3;
        p->sm_count = (int)v;
        return MXP_OK;
    case MXP_ATTR_FP64_ENGINE:
    case MXP_ATTR_OZ_SLICES:
        if (key == MXP_ATTR_FP64_ENGINE && (v < 0 || v > 1)) return -3;
        if (key == MXP_ATTR_OZ_SLICES && (v < oz::MIN_S || v > oz::MAX_S)) return -3;
        if (p->ws && !p->ws_owned) return MXP_ESTATE;  // changes the task list / image sizes
        if (p->ws_owned) {
            cudaFree(p->ws);
            p->ws = nullptr;
            p->ws_owned = false;
        }
        if (key == MXP_ATTR_FP64_ENGINE) p->fp64_engine = (int)v;
        else p->oz_slices = (int)v;
        p->list_uploaded = false;
        return MXP_OK;
    case MXP_ATTR_OZ_PREFETCH:
        if (v < 0 || v > 64) return -3;
        p->oz_prefetch = (int)v;
        return MXP_OK;
    case MXP_ATTR_COMPACT_POOL:
        if (v < 0 || v > 1) return -3;
        if (p->ws && !p->ws_owned) return MXP_ESTATE;  // changes the workspace layout
        if (p->ws_owned) {
            cudaFree(p->ws);
            p->ws = nullptr;
            p->ws_owned = false;
        }
        p->compact_attr = (int)v;
        p->list_uploaded = false;
        return MXP_OK;
    case MXP_ATTR_TC_ENGINE:
        if (v < 0 || v > 3) return -3;
        if (p->ws && !p->ws_owned) return MXP_ESTATE;  // changes the task list / image sizes
        if (p->ws_owned) {
            cudaFree(p->ws);
            p->ws = nullptr;
            p->ws_owned = false;
        }
        p->tc_engine = (int)v;
        p->list_uploaded = false;
        return MXP_OK;
    default: return -2;
    }
}

int mxp_chol_sched_diagnostics(mxp_plan_t p, uint64_t* out, int64_t count, int64_t* written) {
    if (is_group(p)) return mxp_chol_sched_diagnostics(p->group[0], out, count, written);
    if (!p) return -1;
    if (!out && count) return -2;
    int64_t n = std::min<int64_t>(count, (int64_t)p->h_stats.size());
    for (int64_t i = 0; i < n; ++i) out[i] = p->h_stats[i];
    if (written) *written = (int64_t)p->h_stats.size();
    return MXP_OK;
}

int mxp_chol_timeline(mxp_plan_t p, double* ms, int64_t count, int64_t* written) {
    if (is_group(p)) return mxp_chol_timeline(p->group[0], ms, count, written);
    if (!p) return -1;
    if (!ms && count > 0) return -2;
    if (count < 0) return -3;
    if (p->tl_ms.empty()) return MXP_ESTATE;
    const int64_t w = std::min<int64_t>(count, (int64_t)p->tl_ms.size());
    for (int64_t i = 0; i < w; ++i) ms[i] = p->tl_ms[i];
    if (written) *written = (int64_t)p->tl_ms.size();
    return MXP_OK;
}

int mxp_chol_kernel_stats(mxp_plan_t p, int cls, int64_t* launches, double* ms, double* flops) {
    if (is_group(p)) return mxp_chol_kernel_stats(p->group[0], cls, launches, ms, flops);
    if (!p) return -1;
    if (cls < 0 || cls > 3) return -2;
    if (launches) *launches = p->st_launch[cls];
    if (ms) *ms = p->st_ms[cls];
    if (flops) *flops = p->st_flops[cls];
    return MXP_OK;
}

int mxp_chol_plan_get(mxp_plan_t p, mxp_attr_t key, int64_t* v) {
    if (is_group(p)) {
        if (!v) return -3;
        if (key == MXP_ATTR_GPU_LAUNCHES || key == MXP_ATTR_H2D_BYTES || key == MXP_ATTR_D2H_BYTES) {
            int64_t sum = 0;
            for (auto* c : p->group) {
                int64_t x = 0;
                const int rc = mxp_chol_plan_get(c, key, &x);
                if (rc != MXP_OK) return rc;
                sum += x;
            }
            *v = sum;
            return MXP_OK;
        }
        if (key == MXP_ATTR_NRANKS) {
            *v = (int64_t)p->group.size();
            return MXP_OK;
        }
        return mxp_chol_plan_get(p->group[0], key, v);
    }
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
    case MXP_ATTR_TC_ENGINE: *v = p->tc_engine; return MXP_OK;
    case MXP_ATTR_FP64_ENGINE: *v = p->fp64_engine; return MXP_OK;
    case MXP_ATTR_OZ_SLICES: *v = p->oz_slices; return MXP_OK;
    case MXP_ATTR_OZ_PREFETCH: *v = p->oz_prefetch; return MXP_OK;
    case MXP_ATTR_COMPACT_POOL: *v = p->compact_attr; return MXP_OK;
    case MXP_ATTR_COMPACT_USED: plan_images(p); *v = p->compact ? 1 : 0; return MXP_OK;
    case MXP_ATTR_OZ_IMAGE_SLOTS: plan_images(p); *v = p->oz_ooc ? p->oz_img_slots : 0; return MXP_OK;
    case MXP_ATTR_FP64_ENGINE_USED: plan_images(p); *v = p->oz_on ? 1 : 0; return MXP_OK;
    case MXP_ATTR_RANK: *v = p->rank; return MXP_OK;
    case MXP_ATTR_NRANKS: *v = p->nranks; return MXP_OK;
    case MXP_ATTR_SM_FIRST: *v = p->sm_first; return MXP_OK;
    case MXP_ATTR_SM_COUNT: *v = p->sm_count; return MXP_OK;
    case MXP_ATTR_GPU_LAUNCHES: *v = p->launches; return MXP_OK;
    case MXP_ATTR_H2D_BYTES: *v = p->h2d; return MXP_OK;
    case MXP_ATTR_D2H_BYTES: *v = p->d2h; return MXP_OK;
    case MXP_ATTR_POOL_SLOTS:
        plan_images(p);
        *v = p->oz_ooc ? p->ring_slots : p->compact ? p->compact_slots : pool_slots(p);
        return MXP_OK;
    case MXP_ATTR_NT: *v = p->Nt; return MXP_OK;
    case MXP_ATTR_IMAGE_BYTES: plan_images(p); *v = (int64_t)p->shadow_bytes; return MXP_OK;
    case MXP_ATTR_TC_ENGINE_USED: {
        plan_images(p);
        bool any_img = false;
        for (long long o : p->img) any_img |= o >= 0;
        *v = !p->mxp ? -1 : p->tc_engine == 0 ? 0 : p->nat_on ? 3 : any_img ? 1 : 2;
        return MXP_OK;
    }
    default: return -2;
    }
}

int mxp_chol_workspace_size(mxp_plan_t p, size_t* bytes) {
    if (is_group(p)) return mxp_chol_workspace_size(p->group[0], bytes);
    if (!p) return -1;
    if (!bytes) return -2;
    *bytes = workspace_need(p);
    return MXP_OK;
}

int mxp_chol_set_workspace(mxp_plan_t p, void* dev, size_t bytes) {
    if (is_group(p)) {
        g_last_error = "not for a group plan (ngpus > 1): it attaches its GPUs itself";
        return MXP_ENOTSUP;
    }
    if (!p) return -1;
    if (!dev || ((uintptr_t)dev & 255)) return -2;
    if (bytes < workspace_need(p)) return -3;
    if (p->ws_owned && p->ws) {
        cudaSetDevice(p->device);
        cudaFree(p->ws);
    }
    p->ws = (char*)dev;
    p->ws_bytes = bytes;
    p->ws_owned = false;
    p->list_uploaded = false;
    p->epoch = 0;
    {
        Layout L = layout(p);
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(p->device);
        cudaError_t e = cudaMemset(p->ws, 0, L.pool);
        cudaSetDevice(cur);
        if (e != cudaSuccess) return MXP_ECUDA;
    }
    return MXP_OK;
}

int mxp_chol_factor_device(mxp_plan_t p, double* A, int64_t lda, int64_t* info) {
    if (!p) return -1;
    if (!A) return -2;
    if (lda < p->n) return -3;
    if (!info) return -4;
    if (is_group(p))  // every rank packs its tile rows of A (peer reads), rank 0 writes L back
        return group_run(p, info, [&](mxp_plan_s* c, int64_t* inf) { return mxp_chol_factor_device(c, A, lda, inf); });
    p->have_result = false;
    p->launches = p->h2d = p->d2h = 0;
    int cur = 0;
    cudaGetDevice(&cur);
    try {
        CK(cudaSetDevice(p->device));
        if (pool_slots(p) < p->T) {
            g_last_error = "device-resident factorization needs every tile in the pool (HBM cap below the lower triangle)";
            cudaSetDevice(cur);
            return MXP_ENOMEM;
        }
        ensure_streams(p);
        bind_workspace(p);
        cudaStream_t s0 = entry_stream(p);
        // slot table (identity in core; the compact ring with the native engine) + info reset,
        // ordered on the user stream
        if (p->compact) {
            plan_slots(p, p->T);
        } else {
            p->slot_plan.resize(p->T);
            p->prev_owner.assign(p->T, -1);
            for (int64_t t = 0; t < p->T; ++t) p->slot_plan[t] = (int32_t)t;
        }
        CK(cudaMemcpyAsync(p->d_slot, p->slot_plan.data(), sizeof(int32_t) * p->T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemcpyAsync(p->d_prev, p->prev_owner.data(), sizeof(int32_t) * p->T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemsetAsync(p->d_info, 0, sizeof(int64_t), s0));
        prof_reset(p);
        if (p->compact) {
            // PREP tasks copy each tile from A into its ring slot right before its first use
            factor_incore_f64(p, s0, true, nullptr, lda, nullptr, A);
        } else {
            {
                Prof pr(p, s0, MXP_KCLASS_OTHER, 0.0);
                launch_pack_f64(A, lda, p->n, p->pool, p->d_slot, p->Nt, p->nb, 0, p->Nt, s0, p->rank, p->nranks);
                ++p->launches;
                dbg(p, s0, "pack");
            }
            factor_incore_f64(p, s0, false);
        }
        CK(cudaEventRecord(p->ev_done, p->sU));
        CK(cudaStreamWaitEvent(s0, p->ev_done, 0));
        finish_pushes(p, s0);
        {
            Prof pr(p, s0, MXP_KCLASS_OTHER, 0.0, 3);
            if (!p->in_group || p->rank == 0) {  // (a group's ranks share A: rank 0 writes L back)
                launch_unpack_f64(A, lda, p->n, p->pool, p->d_slot, p->Nt, p->nb, 0, p->Nt, s0, decode_args(p));
                p->launches += 1;
            }
            launch_logdet_final(p->d_logdet_parts, p->Nt, p->d_logdet, s0);
            p->launches += 1;
            dbg(p, s0, "unpack");
        }
        int64_t hinfo = 0;
        double ld = 0.0;
        int herr = 0;
        CK(cudaMemcpyAsync(&hinfo, p->d_info, sizeof(int64_t), cudaMemcpyDeviceToHost, s0));
        CK(cudaMemcpyAsync(&ld, p->d_logdet, sizeof(double), cudaMemcpyDeviceToHost, s0));
        CK(cudaMemcpyAsync(&herr, p->d_flags + 1, sizeof(int), cudaMemcpyDeviceToHost, s0));
        CK(cudaStreamSynchronize(s0));
        if (herr) {
            g_last_error = "static schedule: a Ready-table wait timed out (scheduler error)" + sched_timeout_detail(p);
            throw CudaError{cudaErrorLaunchTimeout};
        }
        prof_collect(p);
        if (p->profile) {
            p->h_stats.resize(STAT_POTRF + 3 * (size_t)p->Nt);
            CK(cudaMemcpy(p->h_stats.data(), p->d_stats, sizeof(unsigned long long) * p->h_stats.size(),
                          cudaMemcpyDeviceToHost));
        }
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
    if (is_group(p)) {  // every rank streams its own tile rows; A pinned once, for every GPU
        cudaPointerAttributes attr{};
        const size_t host_bytes = sizeof(double) * ((size_t)lda * (size_t)(p->n - 1) + (size_t)p->n);
        bool reg = false;
        if (!(cudaPointerGetAttributes(&attr, A_host) == cudaSuccess && attr.type == cudaMemoryTypeHost)) {
            cudaGetLastError();
            if (cudaHostRegister(A_host, host_bytes, cudaHostRegisterPortable) != cudaSuccess) {
                cudaGetLastError();
                return MXP_EHOSTPIN;
            }
            reg = true;
        }
        const int rc = group_run(p, info, [&](mxp_plan_s* c, int64_t* inf) { return mxp_chol_factor(c, A_host, lda, inf); });
        if (reg) cudaHostUnregister(A_host);
        return rc;
    }
    // Host-resident path (Alg. 2): tiles stream host->device on a copy
    // stream in schedule order while the static schedule runs; each finished
    // tile streams back as soon as it is final (lower triangle only).
    // Several ranks: each rank reads and writes back only the tile rows it
    // owns (m mod nranks == rank); ranks sharing one host matrix (e.g. a
    // shared-memory mapping) together produce all of L.  In-core only.
    if (p->nranks > 1 && pool_slots(p) < p->T) {
        g_last_error = "out-of-core streaming with several ranks: not in this build";
        return MXP_ENOTSUP;
    }
    p->have_result = false;
    p->launches = p->h2d = p->d2h = 0;
    int cur = 0;
    cudaGetDevice(&cur);
    bool registered = false;
    try {
        CK(cudaSetDevice(p->device));
        if (!stream_memops()) {
            g_last_error = "cuStreamWriteValue32/cuStreamWaitValue32 unavailable";
            cudaSetDevice(cur);
            return MXP_ENOTSUP;
        }
        cudaPointerAttributes attr{};
        const size_t host_bytes = sizeof(double) * ((size_t)lda * (size_t)(p->n - 1) + (size_t)p->n);
        if (!(cudaPointerGetAttributes(&attr, A_host) == cudaSuccess && attr.type == cudaMemoryTypeHost)) {
            cudaGetLastError();
            if (cudaHostRegister(A_host, host_bytes, cudaHostRegisterDefault) != cudaSuccess) {
                cudaGetLastError();
                cudaSetDevice(cur);
                return MXP_EHOSTPIN;
            }
            registered = true;
        }
        ensure_streams(p);
        bind_workspace(p);
        const int64_t nb = p->nb, Nt = p->Nt;
        const size_t stage_bytes = sizeof(double) * (size_t)Nt * nb * nb;
        if (p->h_stage_bytes < stage_bytes) {
            if (p->h_stage) cudaFreeHost(p->h_stage);
            p->h_stage = nullptr;
            p->h_stage_bytes = 0;
            CK(cudaMallocHost((void**)&p->h_stage, stage_bytes));
            p->h_stage_bytes = stage_bytes;
        }
        cudaStream_t s0 = entry_stream(p);
        const int64_t C = pool_slots(p);
        if (!plan_slots(p, C)) {
            g_last_error = "HBM cap below the out-of-core working set (live tiles of two columns)";
            if (registered) cudaHostUnregister(A_host);
            cudaSetDevice(cur);
            return MXP_ENOMEM;
        }
        p->slots = C;
        CK(cudaMemcpyAsync(p->d_slot, p->slot_plan.data(), sizeof(int32_t) * p->T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemcpyAsync(p->d_prev, p->prev_owner.data(), sizeof(int32_t) * p->T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemsetAsync(p->d_info, 0, sizeof(int64_t), s0));
        prof_reset(p);
        if (p->profile) timeline_begin(p);
        factor_incore_f64(p, s0, true, A_host, lda);
        finish_pushes(p, s0);  // several ranks: drain / await the tile exchange
        // the schedule (U) and the POTRFs (P) end first; on failure the later
        // Ready flags never flip, so release the D2H stream explicitly
        CK(cudaStreamSynchronize(p->sU));
        int64_t hinfo = 0;
        int herr = 0;
        CK(cudaMemcpy(&hinfo, p->d_info, sizeof(int64_t), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&herr, p->d_flags + 1, sizeof(int), cudaMemcpyDeviceToHost));
        if (hinfo != 0 || herr) {
            // release the copy streams: Ready flags (D2H gates) and column counters (slot reuse gates)
            CK(cudaMemsetAsync(p->d_flags + 2, 0x7f, sizeof(int) * p->T, p->sAux));
            int* col_ready = p->d_flags + 2 + 6 * p->T + p->T * blocks_per_tile(p->nb) + p->Nt;
            CK(cudaMemsetAsync(col_ready, 0x7f, sizeof(int) * p->Nt, p->sAux));
            CK(cudaStreamSynchronize(p->sAux));
            p->ready_dirty = true;
        }
        CK(cudaStreamSynchronize(p->sD2H));
        CK(cudaStreamSynchronize(p->sH2D));
        CK(cudaStreamSynchronize(p->sP));
        timeline_collect(p);
        if (herr) {
            g_last_error = "static schedule: a Ready-table wait timed out (scheduler error)" + sched_timeout_detail(p);
            throw CudaError{cudaErrorLaunchTimeout};
        }
        // merge the lower triangles of the staged diagonal tiles (upper untouched)
        {
            const int64_t n = p->n;
            unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
            std::vector<std::thread> th;
            for (unsigned w = 0; w < nth; ++w)
                th.emplace_back([&, w] {
                    for (int64_t k = w; k < Nt; k += nth) {
                        if (k % p->nranks != p->rank) continue;
                        const int64_t cr = std::min(nb, n - k * nb);
                        const double* S = p->h_stage + (size_t)k * nb * nb;
                        for (int64_t c = 0; c < cr; ++c)
                            std::memcpy(A_host + (size_t)(k * nb + c) * lda + k * nb + c, S + c * nb + c,
                                        sizeof(double) * (size_t)(cr - c));
                    }
                });
            for (auto& x : th) x.join();
        }
        double ld = 0.0;
        {
            Prof pr(p, s0, MXP_KCLASS_OTHER, 0.0, 2);
            launch_logdet_final(p->d_logdet_parts, p->Nt, p->d_logdet, s0);
            p->launches += 1;
        }
        CK(cudaMemcpyAsync(&ld, p->d_logdet, sizeof(double), cudaMemcpyDeviceToHost, s0));
        CK(cudaStreamSynchronize(s0));
        prof_collect(p);
        if (p->profile) {
            p->h_stats.resize(STAT_POTRF + 3 * (size_t)p->Nt);
            CK(cudaMemcpy(p->h_stats.data(), p->d_stats, sizeof(unsigned long long) * p->h_stats.size(),
                          cudaMemcpyDeviceToHost));
        }
        *info = hinfo;
        p->have_result = (hinfo == 0);
        p->logdet = ld;
        if (registered) cudaHostUnregister(A_host);
    } catch (const CudaError& e) {
        if (registered) cudaHostUnregister(A_host);
        cudaSetDevice(cur);
        return status_from_exception(e);
    }
    cudaSetDevice(cur);
    return MXP_OK;
}

int mxp_chol_factor_tiles(mxp_plan_t p, void* const* tiles, double* scales, int64_t* info) {
    if (!p) return -1;
    if (!tiles) return -2;
    if (!scales) return -3;
    if (!info) return -4;
    if (is_group(p))
        return group_run(p, info, [&](mxp_plan_s* c, int64_t* inf) { return mxp_chol_factor_tiles(c, tiles, scales, inf); });
    // tile-packed host storage (the C5 input): tiles below FP64 travel as their codes,
    // which needs the compact pool (native engine); an all-FP64 map works on every engine
    if (p->nranks > 1) {
        g_last_error = "factor_tiles: single rank";
        return MXP_ENOTSUP;
    }
    for (int64_t t = 0; t < p->T; ++t)
        if (!tiles[t]) return -2;
    p->have_result = false;
    p->launches = p->h2d = p->d2h = 0;
    int cur = 0;
    cudaGetDevice(&cur);
    try {
        CK(cudaSetDevice(p->device));
        if (!stream_memops()) {
            g_last_error = "cuStreamWriteValue32/cuStreamWaitValue32 unavailable";
            cudaSetDevice(cur);
            return MXP_ENOTSUP;
        }
        ensure_streams(p);
        bind_workspace(p);
        if (p->mxp && !p->compact) {
            g_last_error = "factor_tiles with tiles below FP64 needs the compact pool (MXP_ATTR_TC_ENGINE 3, "
                           "MXP_ATTR_FP64_ENGINE 1, in core, MXP_ATTR_COMPACT_POOL 1)";
            cudaSetDevice(cur);
            return MXP_ENOTSUP;
        }
        cudaStream_t s0 = entry_stream(p);
        const int64_t C = pool_slots(p);
        if (!plan_slots(p, C)) {
            g_last_error = "HBM cap below the out-of-core working set (live tiles of two columns)";
            cudaSetDevice(cur);
            return MXP_ENOMEM;
        }
        p->slots = C;
        CK(cudaMemcpyAsync(p->d_slot, p->slot_plan.data(), sizeof(int32_t) * p->T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemcpyAsync(p->d_prev, p->prev_owner.data(), sizeof(int32_t) * p->T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemcpyAsync(p->d_in_scale, scales, sizeof(double) * p->T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemsetAsync(p->d_info, 0, sizeof(int64_t), s0));
        prof_reset(p);
        p->tiles_io = tiles;
        try {
            if (p->profile) timeline_begin(p);
            factor_incore_f64(p, s0, true, nullptr, p->n);
        } catch (...) {
            p->tiles_io = nullptr;
            throw;
        }
        p->tiles_io = nullptr;
        CK(cudaStreamSynchronize(p->sU));
        int64_t hinfo = 0;
        int herr = 0;
        CK(cudaMemcpy(&hinfo, p->d_info, sizeof(int64_t), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(&herr, p->d_flags + 1, sizeof(int), cudaMemcpyDeviceToHost));
        CK(cudaStreamSynchronize(p->sD2H));
        CK(cudaStreamSynchronize(p->sH2D));
        CK(cudaStreamSynchronize(p->sP));
        timeline_collect(p);
        if (herr) {
            g_last_error = "static schedule: a Ready-table wait timed out (scheduler error)" + sched_timeout_detail(p);
            throw CudaError{cudaErrorLaunchTimeout};
        }
        // output scales: the storage scale of every tile below FP64 (code = value * scale), 1 otherwise
        std::vector<double> sc(3 * (size_t)p->T, 1.0);
        if (p->mxp) CK(cudaMemcpy(sc.data(), p->d_iscale, sizeof(double) * 3 * p->T, cudaMemcpyDeviceToHost));
        for (int64_t t = 0; t < p->T; ++t) scales[t] = p->map[t] == MXP_FP64 ? 1.0 : sc[3 * t + 2];
        double ld = 0.0;
        launch_logdet_final(p->d_logdet_parts, p->Nt, p->d_logdet, s0);
        p->launches += 1;
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

int mxp_chol_logdet(mxp_plan_t p, double* logdet) {
    if (is_group(p)) return mxp_chol_logdet(p->group[0], logdet);
    if (!p) return -1;
    if (!logdet) return -2;
    if (!p->have_result) return MXP_ESTATE;
    *logdet = p->logdet;
    return MXP_OK;
}

}  // extern "C"

namespace {
// P:335 criterion (G6) from per-tile norms: F with off-diagonal tiles counted
// twice; least precise allowed p with Nt f_ij / F < eps / u_p.
int plan_from_norms(int64_t Nt, const std::vector<double>& f, double eps, uint32_t allowed, uint8_t* map_out,
                    double* norms_out) {
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
}  // namespace

extern "C" {

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
    return plan_from_norms(Nt, f, eps, allowed, map_out, norms_out);
}

int mxp_precision_map_from_matrix(int64_t n, int64_t nb, const double* A, int64_t lda, double eps,
                                  uint32_t allowed, uint8_t* map_out, double* norms_out) {
    if (n < 1) return -1;
    if (nb < 1) return -2;
    if (!A) return -3;
    if (lda < n) return -4;
    if (!(eps > 0.0 && eps < 1.0)) return -5;
    if (!(allowed & 1u) || (allowed & ~0xFu)) return -6;
    if (!map_out) return -7;
    const int64_t Nt = (n + nb - 1) / nb, T = Nt * (Nt + 1) / 2;
    double *dn = nullptr, *dp = nullptr;
    std::vector<double> f(T);
    cudaStream_t s = nullptr;
    try {
        CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        CK(cudaMalloc(&dn, sizeof(double) * T));
        // one tile column at a time: H2D of rows [j nb, n) x columns [j nb, j nb + nb) (the lower
        // triangle and the diagonal tile's upper part, which the norm mirrors), then its norms
        CK(cudaMalloc(&dp, sizeof(double) * (size_t)n * (size_t)nb));
        for (int64_t j = 0; j < Nt; ++j) {
            const int64_t r0 = j * nb, rows = n - r0, cols = std::min(nb, n - r0);
            CK(cudaMemcpy2DAsync(dp, sizeof(double) * rows, A + r0 + r0 * lda, sizeof(double) * lda,
                                 sizeof(double) * rows, cols, cudaMemcpyHostToDevice, s));
            launch_panel_norms(dp, rows, n, nb, j, dn, s);
            CK(cudaGetLastError());
        }
        CK(cudaMemcpyAsync(f.data(), dn, sizeof(double) * T, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        CK(cudaFree(dn));
        CK(cudaFree(dp));
        CK(cudaStreamDestroy(s));
    } catch (const CudaError& e) {
        if (dn) cudaFree(dn);
        if (dp) cudaFree(dp);
        if (s) cudaStreamDestroy(s);
        return status_from_exception(e);
    }
    return plan_from_norms(Nt, f, eps, allowed, map_out, norms_out);
}

int mxp_precision_map_matern_device(int64_t n, int64_t nb, const double* xy_dev, double sigma2, double range_a,
                                    double nugget, double eps, uint32_t allowed, uint8_t* map_out,
                                    double* norms_out) {
    if (n < 1) return -1;
    if (nb < 1) return -2;
    if (!xy_dev) return -3;
    if (!(sigma2 > 0.0)) return -4;
    if (!(range_a > 0.0)) return -5;
    if (!(nugget >= 0.0)) return -6;
    if (!(eps > 0.0 && eps < 1.0)) return -7;
    if (!(allowed & 1u) || (allowed & ~0xFu)) return -8;
    if (!map_out) return -9;
    int64_t Nt = (n + nb - 1) / nb, T = Nt * (Nt + 1) / 2;
    double* dn = nullptr;
    std::vector<double> f(T);
    try {
        CK(cudaMalloc(&dn, sizeof(double) * T));
        launch_matern_tile_norms(xy_dev, n, nb, sigma2, range_a, nugget, dn, 0);
        CK(cudaGetLastError());
        CK(cudaMemcpy(f.data(), dn, sizeof(double) * T, cudaMemcpyDeviceToHost));
        CK(cudaFree(dn));
    } catch (const CudaError& e) {
        if (dn) cudaFree(dn);
        return status_from_exception(e);
    }
    return plan_from_norms(Nt, f, eps, allowed, map_out, norms_out);
}

int mxp_chol_factor_matern(mxp_plan_t p, const double* xy_dev, double sigma2, double range_a, double nugget,
                           int64_t* info) {
    if (!p) return -1;
    if (!xy_dev) return -2;
    if (!(sigma2 > 0.0)) return -3;
    if (!(range_a > 0.0)) return -4;
    if (!(nugget >= 0.0)) return -5;
    if (!info) return -6;
    if (is_group(p))
        return group_run(p, info, [&](mxp_plan_s* c, int64_t* inf) {
            return mxp_chol_factor_matern(c, xy_dev, sigma2, range_a, nugget, inf);
        });
    p->have_result = false;
    p->launches = p->h2d = p->d2h = 0;
    int cur = 0;
    cudaGetDevice(&cur);
    try {
        CK(cudaSetDevice(p->device));
        ensure_streams(p);
        bind_workspace(p);
        cudaStream_t s0 = entry_stream(p);
        const int64_t C = pool_slots(p);
        if (!plan_slots(p, C)) {
            g_last_error = "HBM cap below the out-of-core working set (live tiles of two columns)";
            cudaSetDevice(cur);
            return MXP_ENOMEM;
        }
        p->slots = C;
        CK(cudaMemcpyAsync(p->d_slot, p->slot_plan.data(), sizeof(int32_t) * p->T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemcpyAsync(p->d_prev, p->prev_owner.data(), sizeof(int32_t) * p->T, cudaMemcpyHostToDevice, s0));
        CK(cudaMemsetAsync(p->d_info, 0, sizeof(int64_t), s0));
        prof_reset(p);
        GenSource g;
        g.xy = xy_dev;
        g.sigma2 = sigma2;
        g.range = range_a;
        g.nugget = nugget;
        factor_incore_f64(p, s0, true, nullptr, 0, &g);
        CK(cudaEventRecord(p->ev_done, p->sU));
        CK(cudaStreamWaitEvent(s0, p->ev_done, 0));
        finish_pushes(p, s0);
        {
            Prof pr(p, s0, MXP_KCLASS_OTHER, 0.0, 1);
            launch_logdet_final(p->d_logdet_parts, p->Nt, p->d_logdet, s0);
            p->launches += 1;
        }
        int64_t hinfo = 0;
        double ld = 0.0;
        int herr = 0;
        CK(cudaMemcpyAsync(&hinfo, p->d_info, sizeof(int64_t), cudaMemcpyDeviceToHost, s0));
        CK(cudaMemcpyAsync(&ld, p->d_logdet, sizeof(double), cudaMemcpyDeviceToHost, s0));
        CK(cudaMemcpyAsync(&herr, p->d_flags + 1, sizeof(int), cudaMemcpyDeviceToHost, s0));
        CK(cudaStreamSynchronize(s0));
        if (herr) {
            g_last_error = "static schedule: a Ready-table wait timed out (scheduler error)" + sched_timeout_detail(p);
            throw CudaError{cudaErrorLaunchTimeout};
        }
        prof_collect(p);
        if (p->profile) {
            p->h_stats.resize(STAT_POTRF + 3 * (size_t)p->Nt);
            CK(cudaMemcpy(p->h_stats.data(), p->d_stats, sizeof(unsigned long long) * p->h_stats.size(),
                          cudaMemcpyDeviceToHost));
        }
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

int mxp_chol_describe(mxp_plan_t p, int streaming, int64_t* counts) {
    if (is_group(p)) return mxp_chol_describe(p->group[0], streaming, counts);
    if (!p) return -1;
    if (!counts) return -3;
    const bool saved = p->host_mode;
    p->host_mode = streaming != 0;
    build_task_list(p);
    p->host_mode = saved;
    p->list_uploaded = false;
    for (int i = 0; i < 6; ++i) counts[i] = 0;
    for (const int4& it : p->items) counts[it.x]++;
    for (const int4& it : p->items2) counts[it.x]++;
    for (int64_t k = 0; k < p->Nt; ++k)
        for (int64_t m = k; m < p->Nt; ++m)
            if (m % p->nranks == p->rank) counts[5]++;
    return MXP_OK;
}

int mxp_chol_ipc_handle(mxp_plan_t p, void* handle_out, uint64_t* ws_bytes) {
    if (is_group(p)) {
        g_last_error = "not for a group plan (ngpus > 1): it attaches its GPUs itself";
        return MXP_ENOTSUP;
    }
    if (!p) return -1;
    if (!handle_out) return -2;
    if (!ws_bytes) return -3;
    if (p->ws && !p->ws_owned) return MXP_ESTATE;  // IPC needs the plan's own cudaMalloc'd workspace
    int cur = 0;
    cudaGetDevice(&cur);
    try {
        CK(cudaSetDevice(p->device));
        ensure_streams(p);
        bind_workspace(p);
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, p->ws));
        std::memcpy(handle_out, &h, sizeof(h));
        *ws_bytes = p->ws_bytes;
    } catch (const CudaError& e) {
        cudaSetDevice(cur);
        return status_from_exception(e);
    }
    cudaSetDevice(cur);
    return MXP_OK;
}

int mxp_chol_ipc_attach(mxp_plan_t p, int peer_rank, const void* handle, uint64_t ws_bytes) {
    if (is_group(p)) {
        g_last_error = "not for a group plan (ngpus > 1): it attaches its GPUs itself";
        return MXP_ENOTSUP;
    }
    if (!p) return -1;
    if (peer_rank < 0 || peer_rank >= p->nranks || peer_rank == p->rank) return -2;
    if (!handle) return -3;
    int cur = 0;
    cudaGetDevice(&cur);
    try {
        CK(cudaSetDevice(p->device));
        ensure_streams(p);
        bind_workspace(p);
        if (ws_bytes != p->ws_bytes) {
            cudaSetDevice(cur);
            return -4;  // peers must use identical plans (same layout)
        }
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle, sizeof(h));
        void* ptr = nullptr;
        CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
        if (p->peer_ipc[peer_rank] && p->peer_ws[peer_rank]) cudaIpcCloseMemHandle(p->peer_ws[peer_rank]);
        p->peer_ws[peer_rank] = (char*)ptr;
        p->peer_ipc[peer_rank] = true;
    } catch (const CudaError& e) {
        cudaSetDevice(cur);
        return status_from_exception(e);
    }
    cudaSetDevice(cur);
    return MXP_OK;
}

int mxp_chol_attach_peer_plan(mxp_plan_t p, int peer_rank, mxp_plan_t peer) {
    if (is_group(p) || is_group(peer)) {
        g_last_error = "not for a group plan (ngpus > 1): it attaches its GPUs itself";
        return MXP_ENOTSUP;
    }
    if (!p) return -1;
    if (peer_rank < 0 || peer_rank >= p->nranks || peer_rank == p->rank) return -2;
    if (!peer || peer == p) return -3;
    int cur = 0;
    cudaGetDevice(&cur);
    try {
        CK(cudaSetDevice(peer->device));
        ensure_streams(peer);
        bind_workspace(peer);
        CK(cudaSetDevice(p->device));
        ensure_streams(p);
        bind_workspace(p);
        if (peer->ws_bytes != p->ws_bytes) {
            cudaSetDevice(cur);
            return -3;
        }
        if (peer->device != p->device) {
            cudaError_t e = cudaDeviceEnablePeerAccess(peer->device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
            cudaGetLastError();
        }
        p->peer_ws[peer_rank] = peer->ws;
        p->peer_ipc[peer_rank] = false;
    } catch (const CudaError& e) {
        cudaSetDevice(cur);
        return status_from_exception(e);
    }
    cudaSetDevice(cur);
    return MXP_OK;
}

int mxp_chol_get_factor_device(mxp_plan_t p, double* L_dev, int64_t ldl) {
    if (is_group(p)) return mxp_chol_get_factor_device(p->group[0], L_dev, ldl);
    if (!p) return -1;
    if (!L_dev) return -2;
    if (ldl < p->n) return -3;
    if (!p->have_result) return MXP_ESTATE;
    if (!p->pool || p->slot_plan.empty() || pool_slots(p) < p->T) return MXP_ESTATE;
    int cur = 0;
    cudaGetDevice(&cur);
    try {
        CK(cudaSetDevice(p->device));
        launch_unpack_f64(L_dev, ldl, p->n, p->pool, p->d_slot, p->Nt, p->nb, 0, p->Nt, p->user_stream,
                          decode_args(p));
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(p->user_stream));
    } catch (const CudaError& e) {
        cudaSetDevice(cur);
        return status_from_exception(e);
    }
    cudaSetDevice(cur);
    return MXP_OK;
}

int mxp_chol_solve_lower(mxp_plan_t p, const double* y_dev, double* z_dev, double* sumsq) {
    if (is_group(p)) return mxp_chol_solve_lower(p->group[0], y_dev, z_dev, sumsq);
    if (!p) return -1;
    if (!y_dev) return -2;
    if (!p->have_result) return MXP_ESTATE;
    if (!p->pool || p->slot_plan.empty() || pool_slots(p) < p->T || p->nranks > 1) return MXP_ESTATE;
    int cur = 0;
    cudaGetDevice(&cur);
    try {
        CK(cudaSetDevice(p->device));
        const int64_t N = p->Nt * p->nb;
        double* r = p->d_solve;
        double* z = r + N;
        double* sc = z + N;
        cudaStream_t s = p->user_stream;
        CK(cudaMemsetAsync(r, 0, sizeof(double) * N, s));
        CK(cudaMemcpyAsync(r, y_dev, sizeof(double) * p->n, cudaMemcpyDeviceToDevice, s));
        ensure_streams(p);
        while (p->ev_solve.size() < 2 * (size_t)p->Nt) {
            cudaEvent_t e;
            CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            p->ev_solve.push_back(e);
        }
        // (s2 = the auxiliary stream, joined after the caller's pending work)
        CK(cudaEventRecord(p->ev_done, s));
        CK(cudaStreamWaitEvent(p->sAux, p->ev_done, 0));
        launch_forward_solve(p->pool, p->d_slot, p->d_wbuf, p->Nt, p->nb, r, z, s, decode_args(p),
                             reinterpret_cast<int*>(sc + 8), ++p->solve_seq, p->sAux, p->ev_solve.data());
        launch_sumsq(z, p->n, sc, s);
        CK(cudaGetLastError());
        if (z_dev) CK(cudaMemcpyAsync(z_dev, z, sizeof(double) * p->n, cudaMemcpyDeviceToDevice, s));
        double h = 0.0;
        CK(cudaMemcpyAsync(&h, sc, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (sumsq) *sumsq = h;
    } catch (const CudaError& e) {
        cudaSetDevice(cur);
        return status_from_exception(e);
    }
    cudaSetDevice(cur);
    return MXP_OK;
}

int mxp_chol_loglik(mxp_plan_t p, const double* y_dev, double* loglik) {
    if (is_group(p)) return mxp_chol_loglik(p->group[0], y_dev, loglik);
    if (!p) return -1;
    if (!loglik) return -3;
    if (!p->have_result) return MXP_ESTATE;
    double q = 0.0;
    if (y_dev) {
        const int st = mxp_chol_solve_lower(p, y_dev, nullptr, &q);
        if (st != MXP_OK) return st;
    }
    // Eq. 1: l = -n/2 log(2 pi) - 1/2 log|Sigma| - 1/2 y^T Sigma^-1 y
    *loglik = -0.5 * (double)p->n * 1.8378770664093454836 - 0.5 * p->logdet - 0.5 * q;
    return MXP_OK;
}

int mxp_chol_tile_device_ptr(mxp_plan_t p, int64_t i, int64_t j, double** ptr) {
    if (is_group(p)) return mxp_chol_tile_device_ptr(p->group[0], i, j, ptr);
    if (!p) return -1;
    if (i < 0 || i >= p->Nt) return -2;
    if (j < 0 || j > i) return -3;
    if (!ptr) return -4;
    if (!p->pool || p->slot_plan.empty() || pool_slots(p) < p->T) return MXP_ESTATE;
    if (p->compact && p->sto[tile_index(p->Nt, i, j)] >= 0) return MXP_ESTATE;  // stored as codes
    *ptr = p->pool + (size_t)p->slot_plan[tile_index(p->Nt, i, j)] * p->nb * p->nb;
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
