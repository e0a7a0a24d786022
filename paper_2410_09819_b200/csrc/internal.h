// internal.h -- shared declarations of the B200 engine (kernels <-> host runtime).
// Not part of the C ABI (see include/mxp_chol.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mxp {

// Every kernel of the library asks for the maximum shared-memory carve-out.
// An SM keeps the L1/shared split of the CTAs resident on it, and a CTA that
// fits the current split does not make the SM switch: if a small kernel (pack,
// input quantization, ...) leaves SMs at a small split and a k_sched CTA lands
// there, the tensor-core kernel k_tc (~150 KB) cannot join it until k_sched
// exits -- the two persistent kernels of the Ozaki mode must share every SM.
#define MXP_CARVEOUT_MAX(kernel)                                                                   \
    do {                                                                                           \
        static bool mxp_carveout_done_ = false;                                                    \
        if (!mxp_carveout_done_) {                                                                 \
            cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);     \
            mxp_carveout_done_ = true;                                                             \
        }                                                                                          \
    } while (0)

// Tile pool: every lower tile (i,j) of the matrix lives in a pool slot of
// nb*nb elements, column-major inside the tile (ld = nb).  slot_of[t] maps
// the column-major lower-tile index t(i,j) to its slot (in-core: identity).
__host__ __device__ inline int64_t tile_index(int64_t Nt, int64_t i, int64_t j) {
    return j * Nt - j * (j - 1) / 2 + (i - j);
}

// ---- device-resident static schedule (sched_f64.cu) ----------------------
// Task list entries (int4): {type, m, k, w}; GEMM: w = (block << 16) | chunk,
// TRSM: w = 64-row block index.
enum { ITEM_GEMM = 0, ITEM_TRSM = 1, ITEM_QUANT = 2, ITEM_PREP = 3, ITEM_POTRF = 4 };
constexpr int MAX_RANKS = 8;

struct SchedArgs {
    double* pool;
    const int32_t* slot;
    int64_t* dinfo;            // LAPACK info (global row of the failed pivot), 0 = ok
    int* err;                  // scheduler timeout flag
    int64_t Nt, nb;
    int64_t KC;                // bulk chunk, in tiles
    int64_t NB;                // 64x128 blocks per tile
    const int4* items;
    int nitems;
    int* counter;              // next task ticket
    int* ready;                // [T] Ready table: tile final and present in this rank's pool
                               //     (== epoch of the factorization; peers write it after pushing a tile)
    int epoch;                 // factorization counter (Ready entries are compared against it)
    int* gemm_done;            // [T] completed GEMM tasks of the tile
    const int* gemm_expected;  // [T]
    int* trsm_done;            // [T] completed TRSM row tasks of the tile
    int* blk_chunk;            // [T*NB] chunks applied to each output block
    double* wbuf;              // [Nt][nb/128][128*128] inverses of L_kk's diagonal blocks
    const uint8_t* prec;       // [T] storage / compute precision of each tile; NULL = all FP64
    unsigned long long* amax_x;  // [T] max |X| of the tile before quantization (atomicMax on bits)
    double* amax_s;            // [T] max |stored value| (drives down-casts of the tile as an operand)
    int* quant_done;           // [T] completed QUANT row tasks
    int tc_engine;             // 1: non-FP64 tiles on tcgen05 (128x128 blocks); 0: DMMA with casts (64x128)
    // host-streaming mode (mxp_chol_factor): tiles arrive by DMA in schedule order
    const int* loaded;         // [T] set to 1 by the copy stream after a tile's H2D; NULL = device mode
    int* prep_done;            // [T] PREP task finished (padding + input quantization)
    int64_t n;                 // real matrix order (padding of edge tiles)
    int gen_mode;              // 0: tiles come from A; 1: PREP generates Matern nu=0.5 tiles (no input copy)
    const int32_t* prev_owner; // [T] previous tile in t's slot (-1: none); generated mode waits for its death
    const double* gen_xy;      // [2n] locations (device)
    double gen_sigma2, gen_range, gen_nugget;
    int* potrf_claim;          // [Nt] POTRF(k) taken (dedicated kernel or scheduler fallback)
    int* col_ready;            // [Nt] tiles of column k that are final (== Nt-k: column complete;
                               //      out-of-core slot reuse waits on it)
    double* logdet_parts;      // [Nt] sum of log L_ii over diagonal tile k (written by its POTRF)
    // multi-GPU (row-cyclic: tile (m, n) belongs to rank m mod nranks)
    int rank, nranks;
    int sm_lo, sm_hi;          // SM partition of this rank's scheduler (co-located ranks)
    int64_t* peer_dinfo[MAX_RANKS];  // peers' info words (a failed pivot stops every rank)
    // MxP operand images (tcgen05 engine, in core): per lower tile 4 byte
    // offsets into `shadow` (-1 = absent): [0..2] = fp32 image of cast_e(L)
    // for e = FP32, FP16, FP8; [3] = the TF32 remainder (lo) of the FP32 image.
    // Each image is nb/128 row blocks x nb/16 K-chunks of 8 KB, every chunk in
    // the tcgen05 shared-memory layout (tc_tf32.cuh).
    const uint8_t* qtile;      // [T] 1 = tile has QUANT tasks (stored below FP64 or has images)
    const long long* img;      // [4T] (nullptr: no images; register-staged engine)
    uint8_t* shadow;
    int reserved_sms;          // SMs (smid < this) left to the POTRF kernels
    // FP64 tiles on the int8 tensor cores (Ozaki scheme, oz_i8.cuh; MXP_ATTR_FP64_ENGINE = 1):
    // every GEMM task goes to a second list run by the tensor-core kernel k_tc
    // (one CTA per SM, all of its TMEM); k_sched keeps TRSM / QUANT / PREP / POTRF.
    const long long* oz_img;   // [T] byte offset of the tile's int8 slice image in `shadow` (-1: none);
                               //     nullptr: the Ozaki engine is off
    int oz_slices;             // s (slices per operand, 1..8)
    // Ozaki running row scales (oz_slice_rows): oz_flag[t] = 1 when a row of tile t = (m, k) needed
    // a larger scale than in tile (m, k-1); a GEMM chunk with no flagged tile after its first
    // accumulates across its K tiles in int32 TMEM and drains once.  nullptr: per-tile scales.
    int* oz_flag;              // [T]
    int oz_prefetch;           // L2 prefetch distance of the Ozaki operand ring, in K steps (0: off)
    const int32_t* img_prev;   // Ozaki out of core: [T] previous owner of t's slice-image slot (its QUANT
                               //     waits until that tile's row died: column complete); nullptr in core
    int ring_all;              // Ozaki out of core: every tile's fp64 slot is a ring slot (diagonal tiles
                               //     die with their column, the others when final)
    const int4* items2;        // k_tc's list: the WHOLE static list (k_tc alone can finish the
    int nitems2;               //   schedule, e.g. when a profiler serializes the kernels); k_sched
    int* counter2;             //   takes the non-GEMM subsequence (items); both claim non-GEMM tasks
    int* task_claim;           //   by CAS here: TRSM [T*R] | QUANT [T*R] | PREP [T]  (R = nb/64)
    int* tdiag;                // [24] first timed-out wait: flag offset from `ready`, target, value, smid,
                               //     block, grid, column, taken (host reports it in mxp_last_error)
    // native-width operand images (tc_native.cuh; MXP_ATTR_TC_ENGINE = 3, tensor-core kernel k_tc):
    // img[4t+1] = fp16 codes of cast_FP16(L) for FP16 outputs, img[4t+2] = E4M3 codes of cast_FP8(L)
    // for FP8 outputs, iscale[3t + kind] = the power-of-two scale of those codes (code = value * scale)
    int native;
    double* iscale;            // [3T]: + [3t+2] = scale of the storage image (code = value * scale)
    // compact pool (native engine): tiles below FP64 live as storage images after their QUANT
    int compact;
    const long long* sto;      // [T] offsets of the storage images in `shadow` (-1: FP64 tile)
    const double* src_A;       // compact device path: the caller's matrix (PREP copies tiles from it)
    int64_t src_lda;
    int tile_codes;            // mxp_chol_factor_tiles: input tiles below FP64 arrive as codes in their
    const double* in_scale;    //   storage images (value = code / in_scale[t]); PREP decodes them
    int* sm_claim;             // [256] k_sched CTAs per SM in the Ozaki mode (extras leave at once,
                               //       keeping room for the k_tc CTA of every SM)
    unsigned long long* stats; // optional diagnostics (MXP_ATTR_PROFILE): see STAT_*
};
// diagnostics layout (ns from %globaltimer, summed over CTAs)
enum {
    STAT_GEMM_BUSY = 0, STAT_GEMM_WAIT = 1, STAT_TRSM_BUSY = 2, STAT_TRSM_WAIT = 3,
    STAT_GEMM_N = 4, STAT_TRSM_N = 5, STAT_T0 = 6, STAT_TEND = 7, STAT_CTAS = 8,
    // POTRF phases (ns summed over columns): block-column update, unblocked
    // factor, W_J inverse (+ write-back), in-tile TRSM
    STAT_PF_UPD = 9, STAT_PF_CHOL = 10, STAT_PF_INV = 11, STAT_PF_TRSM = 12,
    // Ozaki GEMM tasks (k_tc): the issuing thread's waits for operand stages (full) and for
    // MMA completion before refills (done), and the per-tile drains (tile MMAs end -> fp64)
    STAT_OZ_FULL = 13, STAT_OZ_DONE = 14, STAT_OZ_DRAIN = 15,
    // busy ns of the GEMM tasks by output precision (FP64, FP32, FP16, FP8) and their counts
    STAT_GEMM_P = 16, STAT_GEMM_PN = 20,
    // Ozaki GEMM loop: time of the issuing thread in MMA issue, in bulk-copy issue, and in the loop
    STAT_OZ_MMA = 24, STAT_OZ_COPY = 25, STAT_OZ_LOOP = 26,
    // native engine: issuer waits for stages (full), for refills (empty), for drained
    // accumulators (tempty); drain warps' time in drains; the final C update
    STAT_NAT_FULL = 28, STAT_NAT_EMPTY = 29, STAT_NAT_TEMPTY = 30, STAT_NAT_DRAIN = 31, STAT_NAT_FINAL = 32,
    STAT_OZ_TBAR = 33,  // Ozaki: drain warps waiting for a tile's last MMAs (the rest of STAT_OZ_DRAIN is the drain)
    STAT_POTRF = 36  // + 3k: kernel start, wait done, end
};
int sched_ctas_per_sm();
// load every kernel of the library eagerly (one call per file; see preload_sched)
void preload_sched();
void preload_layout();
void preload_solve();
void preload_generators();
// input stage of MxP (a3, O3): per-tile amax, then A^ = deq(q_p(A)) in place
void launch_input_quantize(double* pool, const int32_t* slot, const uint8_t* prec, int64_t Nt, int64_t nb,
                           unsigned long long* amax_x, double* amax_s, cudaStream_t s, int rank = 0,
                           int nranks = 1);
void launch_sched(const SchedArgs& a, const SchedArgs* a_dev, bool mxp, int grid, cudaStream_t s);  // a_dev: device copy of a
// tensor-core GEMM kernel of the Ozaki mode (one CTA per SM, beside k_sched)
void launch_tc(const SchedArgs* a_dev, int grid, cudaStream_t s, bool native);
int tc_ctas_per_sm();
void launch_potrf_tile(const SchedArgs& a, int64_t k, cudaStream_t s);

// Final tiles stored as codes (compact pool): value = code / scale[3t+2], code at prec[t]
// (FP32 float, FP16 binary16, FP8 E4M3), column-major nb x nb at shadow + sto[t];
// sto == nullptr or sto[t] < 0: the fp64 slot.
struct TileCodes {
    const long long* sto;
    const uint8_t* shadow;
    const uint8_t* prec;
    const double* scale;
};

// ---- forward solve / log-likelihood (solve.cu) -----------
// z = L^-1 r on the resident factor (r, z: Nt*nb, padded with zeros; r is consumed)
// flags: >= nb/128 ints of device memory for the parallel diagonal solves (publication tags
// seq * Nt + k + 1; seq distinct per call), or nullptr for the one-CTA diagonal solve
// s2 / ev (2 Nt events): the updates of the rows below the next tile row run on s2, overlapping
// the diagonal solves on s (bitwise the same result); s2 == nullptr: one stream
void launch_forward_solve(const double* pool, const int32_t* slot, const double* wbuf, int64_t Nt, int64_t nb,
                          double* r, double* z, cudaStream_t s, TileCodes codes = TileCodes{},
                          int* flags = nullptr, int seq = 0, cudaStream_t s2 = nullptr, cudaEvent_t* ev = nullptr);
void launch_sumsq(const double* z, int64_t n, double* out, cudaStream_t s);

// ---- layout / utility kernels --------------------------------------------
// lda matrix <-> pool tiles (padding: zeros, 1 on the padded diagonal)
void launch_pack_f64(const double* A, int64_t lda, int64_t n, double* pool, const int32_t* slot,
                     int64_t Nt, int64_t nb, int64_t col0, int64_t col1, cudaStream_t s, int rank = 0,
                     int nranks = 1);
void launch_unpack_f64(double* A, int64_t lda, int64_t n, const double* pool, const int32_t* slot,
                       int64_t Nt, int64_t nb, int64_t col0, int64_t col1, cudaStream_t s,
                       TileCodes codes = TileCodes{});
// logdet = 2 sum_k parts[k] in ascending k (parts from the POTRFs; deterministic)
void launch_logdet_final(const double* parts, int64_t Nt, double* out, cudaStream_t s);
// planner on a generated Matern covariance: per-tile Frobenius norms computed
// while generating the entries (nothing stored)
void launch_matern_tile_norms(const double* xy, int64_t n, int64_t nb, double sigma2, double range_a,
                              double nugget, double* norms, cudaStream_t s);
// planner: per-tile Frobenius norms (fp64) of the lower tiles of an lda matrix
// planner on a host matrix: norms of tile column j from its device panel copy (ld = ldp)
void launch_panel_norms(const double* P, int64_t ldp, int64_t n, int64_t nb, int64_t j, double* norms,
                        cudaStream_t s);
void launch_tile_norms(const double* A, int64_t lda, int64_t n, int64_t nb, double* norms,
                       cudaStream_t s);


}  // namespace mxp
