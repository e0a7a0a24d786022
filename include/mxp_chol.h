/*
 * mxp_chol.h -- C ABI of the B200-native mixed-precision, out-of-core,
 * left-looking tile Cholesky factorization of arxiv 2410.09819.
 *
 * Problem statement (Alg. 1): factor a symmetric
 * positive-definite n x n matrix A = L L^T, A partitioned into Nt x Nt tiles
 * of nb x nb (Nt = ceil(n/nb)); the lower tiles are traversed column by
 * column (left-looking): SYRK+POTRF on the diagonal tile, GEMM+TRSM on each
 * tile below it, every tile with its own precision.
 *
 * Conventions shared by every call:
 *  - Matrices are column-major with a leading dimension (lda >= n); only the
 *    lower triangle is referenced or written (LAPACK dpotrf('L') semantics).
 *  - "host" pointers are CPU memory (pageable or pinned); "device" pointers
 *    are CUDA global memory of the plan's device.  The caller owns every
 *    buffer it passes; the plan owns everything it allocates itself.
 *  - Precision codes: MXP_FP64 = 0, MXP_FP32 = 1, MXP_FP16 = 2, MXP_FP8 = 3
 *    (OCP E4M3 "fn", saturating).  FP16/FP8 tiles carry a per-tile power-of-two
 *    scale s: stored codes = RNE(x * s); value = code / s  (G11).
 *  - Precision maps hold Nt(Nt+1)/2 codes in column-major lower-tile order
 *    (0,0),(1,0),...,(Nt-1,0),(1,1),... ; diagonal tiles must be MXP_FP64.
 *  - Return value: MXP_OK (0); -i when the i-th argument is invalid (LAPACK
 *    style); or one of the negative MXP_E* codes below.
 *  - `info` (LAPACK / cuSOLVER devInfo): 0 on success; j > 0 when the leading
 *    minor of order j is not positive definite (global 1-based row of the
 *    failing pivot).  On failure, tile columns before the failing one hold L;
 *    later content is unspecified.
 *  - Calls on one plan are not reentrant; different plans are independent.
 */
#ifndef MXP_CHOL_H
#define MXP_CHOL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MXP_CHOL_ABI_VERSION 1

enum mxp_status {
    MXP_OK = 0,
    MXP_ECUDA = -1001,    /* a CUDA runtime call failed (see mxp_last_error) */
    MXP_ENOMEM = -1002,   /* device memory (or the HBM cap) below the working-set bound */
    MXP_EHOSTPIN = -1003, /* pinning / registering host memory failed */
    MXP_ESTATE = -1004,   /* call not valid in the plan's current state */
    MXP_ENOTSUP = -1005,  /* configuration not supported by this build */
    MXP_EZERO = -1006,    /* ||A||_F = 0 in the planner (SPEC S:296 ZeroMatrix) */
    MXP_ENCCL = -1007     /* inter-GPU exchange failed */
};

enum mxp_precision { MXP_FP64 = 0, MXP_FP32 = 1, MXP_FP16 = 2, MXP_FP8 = 3 };

typedef struct mxp_plan_s* mxp_plan_t;

/* Plan attributes (mxp_chol_plan_set / _get). */
typedef enum mxp_attr {
    MXP_ATTR_DEVICE = 0,          /* CUDA device ordinal (default: current device at plan time) */
    MXP_ATTR_STREAM = 1,          /* cudaStream_t (as int64) all work is ordered after/before; 0 = legacy default */
    MXP_ATTR_HBM_BYTES_CAP = 2,   /* cap on the tile pool; forces out-of-core when the lower triangle exceeds it */
    MXP_ATTR_SPLITK_TILES = 3,    /* K chunk of one GEMM task, in tiles (default 16); results are bitwise
                                     deterministic for a fixed value */
    MXP_ATTR_LOOKAHEAD = 4,       /* reserved (the task list always carries one column of lookahead) */
    MXP_ATTR_DEBUG_SYNC = 5,      /* 1 = synchronize and check after every kernel; 2 = GEMM-throughput
                                     probe (GEMM tasks only, Ready pre-set, no POTRF: result is garbage);
                                     3 = no dedicated POTRF kernels (the scheduler's fallback factors every
                                     diagonal tile) */
    MXP_ATTR_PROFILE = 6,         /* 1 = time every launch with CUDA events on its stream (mxp_chol_kernel_stats) */
    MXP_ATTR_TC_ENGINE = 7,       /* GEMM tasks of tiles below FP64 (G12):
                                     3 (default) = native operand width: FP16 outputs on tcgen05 kind::f16 (fp16
                                       codes), FP8 outputs on kind::f8f6f4 (E4M3 codes), per-tile power-of-two
                                       scales applied to the fp32 TMEM partial of every K tile; FP32 outputs on
                                       3xTF32 as 1.  Needs the tensor-core kernel of MXP_ATTR_FP64_ENGINE = 1 (in
                                       core, single rank); otherwise it behaves as 1 (MXP_ATTR_TC_ENGINE_USED);
                                     1 = tcgen05 kind::tf32 (3xTF32 for FP32 tiles, 1xTF32 for the exact
                                       FP16/FP8 values) fed by bulk copies of per-tile fp32 operand images written
                                       once by the QUANT tasks (in core; out of core it behaves as 2);
                                     2 = tcgen05, operands converted from the fp64 tiles in registers;
                                     0 = FP64 DMMA with the same casts (fp64 accumulation).
                                     Changing it re-sizes the workspace (images: 1, 2 or 4(+4) bytes per element
                                     and consumer precision). */
    MXP_ATTR_RANK = 8,            /* this plan's rank in a row-cyclic distribution (tile (m,n) on rank m mod nranks) */
    MXP_ATTR_NRANKS = 9,          /* ranks (GPUs) sharing the factorization, <= 8; peers attached with
                                     mxp_chol_ipc_attach / mxp_chol_attach_peer_plan.  Each rank keeps streams
                                     parked on cuStreamWaitValue32; ranks co-located in one process need
                                     CUDA_DEVICE_MAX_CONNECTIONS >= 8 * nranks (set before CUDA starts) */
    MXP_ATTR_SM_FIRST = 10,       /* first SM of this plan's scheduler partition (ranks co-located on one GPU) */
    MXP_ATTR_SM_COUNT = 11,       /* SMs in the partition (0 = all) */
    MXP_ATTR_FP64_ENGINE = 12,    /* GEMM/SYRK tasks of FP64 tiles:
                                     0 (default) = FP64 tensor pipe (DMMA, mma.sync.m8n8k4.f64);
                                     1 = Ozaki scheme I on the int8 tensor cores (tcgen05 kind::i8): every
                                       off-diagonal tile is split once, exactly, into s int8 slices with a
                                       power-of-two scale per row (8s - 2 bits + sign, balanced base-256
                                       digits; a row keeps its scale from tile to tile unless a larger
                                       entry needs more, with two binades of headroom), the s(s+1)/2 slice
                                       products of weight >= 2^-8(s-1) are accumulated exactly in int32
                                       TMEM across the K tiles that share their scales, and the levels are
                                       combined in fp64 (fp64 accumulation across those groups).  Single rank.  In core the pool keeps every fp64 tile
                                       beside the slice images.  Out of core (FP64 map, HBM cap below the
                                       lower triangle; mxp_chol_factor / _factor_tiles / _factor_matern) an
                                       fp64 tile lives in a ring slot only while it is computed and a final
                                       off-diagonal tile lives on as its slice image (s bytes per element) in
                                       an arena whose slots are recycled when the tile's row dies; ring +
                                       arena must fit under the cap (MXP_ATTR_OZ_IMAGE_SLOTS).  Otherwise it
                                       behaves as 0 -- see MXP_ATTR_FP64_ENGINE_USED.  Re-sizes the workspace. */
    MXP_ATTR_OZ_SLICES = 13,      /* s for MXP_ATTR_FP64_ENGINE = 1, 4..8 (default 7: 54 bits per operand,
                                     28 int8 products; dropped products <= 6 * 2^-52 of the row maxima) */
    MXP_ATTR_OZ_PREFETCH = 15,    /* Ozaki engine: L2 prefetch (cp.async.bulk.prefetch.L2) of the operand chunks
                                     this many 32-K steps ahead of the shared-memory ring, 0..64 (0 = off) */
    MXP_ATTR_COMPACT_POOL = 14,   /* with the native engine (MXP_ATTR_TC_ENGINE_USED = 3): 1 (default) = store every
                                     tile below FP64 at its precision (codes + a power-of-two scale: 4/2/1 bytes per
                                     element, "minimum acceptable bytes per word"); its fp64 accumulator slot
                                     is recycled once the tile is final, so only FP64 tiles keep 8-byte slots.
                                     mxp_chol_tile_device_ptr then refuses such tiles (MXP_ESTATE); unpack, the
                                     forward solve and the D2H decode them.  0 = every tile keeps an fp64 slot. */
    MXP_ATTR_GPU_LAUNCHES = 100,  /* (get only) kernels launched by the last factorization */
    MXP_ATTR_H2D_BYTES = 101,     /* (get only) host->device bytes moved by the last factorization */
    MXP_ATTR_D2H_BYTES = 102,     /* (get only) device->host bytes moved by the last factorization */
    MXP_ATTR_POOL_SLOTS = 103,    /* (get only) tile slots in the device pool */
    MXP_ATTR_NT = 104,            /* (get only) Nt = ceil(n/nb) */
    MXP_ATTR_IMAGE_BYTES = 105,   /* (get only) bytes of tcgen05 operand images in the workspace (0: none) */
    MXP_ATTR_FP64_ENGINE_USED = 106, /* (get only) FP64 engine the next factorization uses (0 DMMA, 1 Ozaki) */
    MXP_ATTR_TC_ENGINE_USED = 107, /* (get only) engine of the tiles below FP64 the next factorization uses
                                     (-1: all-FP64 map; else as MXP_ATTR_TC_ENGINE) */
    MXP_ATTR_COMPACT_USED = 108,  /* (get only) 1 if the next factorization uses the compact pool */
    MXP_ATTR_OZ_IMAGE_SLOTS = 109 /* (get only) slice-image slots of the out-of-core Ozaki mode (the peak live
                                     set of final off-diagonal tiles, ~Nt^2/4); 0 when that mode is off */
} mxp_attr_t;

/*
 * mxp_chol_plan -- describe one factorization problem (Alg. 1 P:117 "A ... of
 * size n x n, partitioned into Nt x Nt tiles"; precision map P:335).
 *   n             matrix order, n >= 1                              (arg 1)
 *   nb            tile size; nb % 128 == 0, 128 <= nb <= 2048        (arg 2)
 *   precision_map host array of Nt(Nt+1)/2 codes, copied; NULL = all FP64 (arg 3)
 *   ngpus         GPUs the plan spans, 1..8 (other values return -4)    (arg 4)
 *                 1: one plan per GPU and process; several processes cooperate through
 *                    MXP_ATTR_RANK / MXP_ATTR_NRANKS and the peer attach calls below.
 *                 > 1: a group plan in this process (SURVEY 8(e), row-cyclic P x 1):
 *                    one sub-plan per rank r on device r mod cudaGetDeviceCount(), tile row
 *                    m owned by rank m mod ngpus, finished tiles pushed to the peers over
 *                    P2P; the factor calls run every rank from its own host thread and
 *                    return when all are done.  Ranks that share a device split its SMs.
 *                    Attributes apply to every rank (MXP_ATTR_DEVICE / RANK / NRANKS /
 *                    SM_FIRST / SM_COUNT: MXP_ENOTSUP; MXP_ATTR_STREAM orders rank 0);
 *                    mxp_chol_factor_device reads A from its device (peers by P2P) and
 *                    rank 0 writes L back; results, log-det and solves come from rank 0;
 *                    the *_BYTES / GPU_LAUNCHES getters sum over ranks.  Out-of-core
 *                    streaming and mxp_chol_factor_tiles stay single-rank (MXP_ENOTSUP).
 *   out           receives the plan handle                           (arg 5)
 * No device memory is allocated here; that happens on the first factor call
 * (or mxp_chol_set_workspace).
 */
int mxp_chol_plan(int64_t n, int64_t nb, const uint8_t* precision_map, int ngpus, mxp_plan_t* out);

/* Set / get a plan attribute.  Returns -2 for an unknown key, -3 for a bad value. */
int mxp_chol_plan_set(mxp_plan_t plan, mxp_attr_t key, int64_t value);
int mxp_chol_plan_get(mxp_plan_t plan, mxp_attr_t key, int64_t* value);

/*
 * Device workspace.  mxp_chol_workspace_size reports the bytes the plan needs
 * on its device (tile pool + split-K partials + scratch) for the current
 * attributes.  mxp_chol_set_workspace hands the plan a caller-owned device
 * buffer of at least that size (e.g. a torch tensor); without it the plan
 * cudaMallocs its own on first use and frees it in mxp_chol_plan_destroy.
 */
int mxp_chol_workspace_size(mxp_plan_t plan, size_t* bytes);
int mxp_chol_set_workspace(mxp_plan_t plan, void* device_ptr, size_t bytes);

/*
 * mxp_chol_factor_device -- in-core factorization of a device-resident matrix
 * (the like-for-like comparison with cusolverDnXpotrf).
 *   A_dev  device pointer, n x n column-major, lda >= n; lower triangle is
 *          overwritten by L (values of FP16/FP8/FP32 tiles are the
 *          dequantized stored values); strict upper triangle untouched. (arg 2)
 *   lda    leading dimension                                          (arg 3)
 *   info   host pointer, receives info                                (arg 4)
 * Ordered on MXP_ATTR_STREAM; returns after the result is complete.
 */
int mxp_chol_factor_device(mxp_plan_t plan, double* A_dev, int64_t lda, int64_t* info);

/*
 * mxp_chol_factor -- factorization of a host-resident matrix (Alg. 2
 * P:240-278): tiles are streamed host->device on side streams, factored, and
 * written back device->host (lower triangle only).  When the lower
 * triangle at its storage precisions exceeds the device pool
 * (MXP_ATTR_HBM_BYTES_CAP or HBM), tiles are cached and evicted out-of-core
 * with a static plan computed ahead from the static schedule: a tile's
 * slot is recycled once the tile is dead (after its last reader; with the
 * compact pool, once the tile is final), every tile crosses the link once each
 * way, and the accumulator of a task stays in its slot for the whole GEMM
 * chain.  Re-fetching evicted live tiles (the paper's V2 regime, Alg. 3
 * P:281-301) is not implemented: an HBM cap below the live set returns
 * MXP_ENOMEM.
 *   A_host host pointer (pinned via mxp_host_alloc for full copy bandwidth;
 *          pageable memory is registered for the call), column-major, lda >= n;
 *          lower triangle overwritten by L as in mxp_chol_factor_device. (arg 2)
 *   lda, info as above.
 */
int mxp_chol_factor(mxp_plan_t plan, double* A_host, int64_t lda, int64_t* info);

/*
 * mxp_chol_factor_tiles -- factorization of a matrix held as tile-packed HOST
 * storage at each tile's precision (the only feasible input of
 * C5: a dense lda matrix would be 2.2 TB).  P:42 "transmitting the minimum
 * acceptable bytes per word": tiles below FP64 cross the host link as codes.
 *   tiles   host array of Nt(Nt+1)/2 pointers in column-major lower-tile order;
 *           tile t is nb x nb column-major at precision map[t]: FP64 doubles,
 *           FP32 floats, FP16 binary16 codes, FP8 E4M3 codes (padding beyond n
 *           ignored).  Diagonal tiles hold the full symmetric nb x nb block (only
 *           its lower triangle is read).  Pinned memory (mxp_host_alloc) gives
 *           full copy bandwidth.                                        (arg 2)
 *   scales  host array of Nt(Nt+1)/2 doubles: value = code / scales[t] for
 *           FP16/FP8 tiles (a power of two; 1 for FP64/FP32 tiles)     (arg 3)
 *   info    as mxp_chol_factor                                         (arg 4)
 * On return every tile holds L's tile at the same precision (codes), scales[t]
 * its new scale; diagonal tiles hold L_kk with zeros above the diagonal.  The
 * input is stored at its precision (O3) before use.  Host<->device traffic is
 * one pass each way at storage precision (MXP_ATTR_H2D_BYTES / _D2H_BYTES).
 * Tiles below FP64 need the compact pool (MXP_ATTR_COMPACT_USED = 1, i.e. the
 * native engine in core); otherwise MXP_ENOTSUP.  An all-FP64 map works on
 * every engine, in core or out of core.  Single rank.
 */
int mxp_chol_factor_tiles(mxp_plan_t plan, void* const* tiles, double* scales, int64_t* info);

/*
 * mxp_chol_factor_matern -- factor the Matern nu = 0.5 covariance of n
 * locations (Eq. 2, the paper's geospatial workload P:168-190)
 * WITHOUT materializing it: every tile is generated on the device by the
 * schedule's PREP task right before its first use (fused generation; SURVEY
 * N2), then stored at its precision.  L stays in the plan's pool (read it
 * with mxp_chol_get_factor_device / mxp_chol_tile_device_ptr) when the pool
 * holds every tile; under MXP_ATTR_HBM_BYTES_CAP dead tiles are recycled and
 * only the log-determinant survives.
 *   xy_dev   device array of 2n doubles (x0,y0,x1,y1,...)               (arg 2)
 *   sigma2, range_a, nugget   theta = (sigma^2, a) and a diagonal nugget  (args 3-5)
 *   info     host pointer, receives info                                 (arg 6)
 */
int mxp_chol_factor_matern(mxp_plan_t plan, const double* xy_dev, double sigma2, double range_a, double nugget,
                           int64_t* info);

/* Planner (as mxp_precision_map_from_matrix_device) for the generated Matern
 * covariance: tile norms are computed while generating the entries. */
int mxp_precision_map_matern_device(int64_t n, int64_t nb, const double* xy_dev, double sigma2, double range_a,
                                    double nugget, double eps, uint32_t allowed_mask, uint8_t* map_out,
                                    double* norms_out);

/* Copy the resident factor L (lower triangle) of the last successful
 * factorization into a caller-owned device matrix (column-major, ldl >= n);
 * MXP_ESTATE if the factor is not resident (out-of-core run). */
int mxp_chol_get_factor_device(mxp_plan_t plan, double* L_dev, int64_t ldl);

/* Device pointer to tile (i, j) of the resident factor (nb x nb, column-major,
 * ld = nb), valid until the plan's next factorization. */
int mxp_chol_tile_device_ptr(mxp_plan_t plan, int64_t i, int64_t j, double** ptr);

/*
 * mxp_chol_logdet -- log|A| = 2 sum_i log L_ii (Eq. 1) of the
 * last successful factorization of this plan, reduced in fp64 on the device.
 * Returns MXP_ESTATE if no factorization succeeded.
 */
int mxp_chol_logdet(mxp_plan_t plan, double* logdet);

/*
 * mxp_chol_solve_lower -- forward substitution L z = y on the resident factor
 * of the last successful factorization (the quadratic form of Eq. 1, P:172:
 * y^T A^-1 y = ||z||^2).  y_dev: n doubles on the plan's
 * device (read only); z_dev: n doubles (device, may be NULL); sumsq: ||z||^2
 * on return (host, may be NULL).  For tiles stored below FP64 the solve uses
 * their stored (dequantized) values.  Every lower tile is read once (HBM
 * bound); sums run in a fixed order (bitwise reproducible).  Ordered on
 * MXP_ATTR_STREAM; returns after the result is complete.  MXP_ESTATE if no
 * factorization succeeded or the factor is not resident (out of core, several
 * ranks).
 */
int mxp_chol_solve_lower(mxp_plan_t plan, const double* y_dev, double* z_dev, double* sumsq);

/*
 * mxp_chol_loglik -- Gaussian log-likelihood of Eq. 1,
 *   l = -n/2 log(2 pi) - 1/2 log|A| - 1/2 y^T A^-1 y,
 * with A the last factorized matrix (covariance) and y_dev n observations on
 * the device (NULL: y = 0, the convention of the paper's Eq. 3 KL check).
 * loglik: host double.  Errors as mxp_chol_solve_lower.
 */
int mxp_chol_loglik(mxp_plan_t plan, const double* y_dev, double* loglik);

/*
 * mxp_precision_map_from_matrix_device -- the MxP planner: per-tile
 * Frobenius norms f_ij (fp64), F = ||A||_F with off-diagonal tiles counted
 * twice, and for each off-diagonal tile the least precise allowed p with
 *     Nt * f_ij / F < eps / u_p      (u_p the unit roundoff, G6);
 * diagonal tiles and tiles where none qualifies get FP64.
 *   n, nb        as in mxp_chol_plan                                (args 1-2)
 *   A_dev        device pointer, column-major, lower triangle read   (arg 3)
 *   lda          leading dimension                                   (arg 4)
 *   eps          target accuracy, 0 < eps < 1                        (arg 5)
 *   allowed_mask bit p set => precision p may be chosen; must include FP64 (arg 6)
 *   map_out      host array of Nt(Nt+1)/2 codes                      (arg 7)
 *   norms_out    optional host array of Nt(Nt+1)/2 tile norms, or NULL (arg 8)
 * Runs on the current device and the legacy default stream.  Returns
 * MXP_EZERO when ||A||_F = 0.
 */
int mxp_precision_map_from_matrix_device(int64_t n, int64_t nb, const double* A_dev, int64_t lda,
                                         double eps, uint32_t allowed_mask, uint8_t* map_out,
                                         double* norms_out);

/*
 * mxp_precision_map_from_matrix -- the same planner (G6) for a HOST matrix
 * (SURVEY 8(b)): A is streamed to the device one tile column panel at a time
 * (rows j*nb..n-1 of columns j*nb..j*nb+nb-1; one panel of n x nb doubles of
 * device memory) and the tile norms are reduced there.  Arguments and errors as
 * mxp_precision_map_from_matrix_device, with A a host pointer (pageable or
 * pinned, lower triangle and the diagonal tiles read).  Synchronous; uses the
 * current device and a private stream.
 */
int mxp_precision_map_from_matrix(int64_t n, int64_t nb, const double* A, int64_t lda, double eps,
                                  uint32_t allowed_mask, uint8_t* map_out, double* norms_out);

/*
 * Synthetic input generators, bit-identical to the host
 * generators in workloads/ (same counter hash), writing the full symmetric
 * matrix (both triangles) into a device buffer on `stream` (cudaStream_t, may
 * be NULL for the legacy default stream).  AUX: they are not part of the
 * factorization; they exist so bench-sized inputs need no host copy.
 *  plgsy: A_ij = A_ji = u(seed, max(i,j), min(i,j)) - 0.5, A_ii += n, where
 *         u = (mix64(((i << 32) | j) ^ mix64(seed + 0x9E3779B97F4A7C15)) >> 11) * 2^-53
 *         and mix64 is the splitmix64 finaliser.
 *  kms:   A_ij = rho^|i-j|  (Kac-Murdock-Szego, config C1).
 */
int mxp_generate_plgsy_device(int64_t n, uint64_t seed, double* A_dev, int64_t lda, void* stream);
int mxp_generate_kms_device(int64_t n, double rho, double* A_dev, int64_t lda, void* stream);
/* Matern nu = 0.5 covariance (Eq. 2 closed form): A_ij = sigma2 exp(-|s_i - s_j| / range_a)
 * (+ nugget on the diagonal) from n locations xy_dev (device, interleaved x,y); see workloads.matern_*. */
int mxp_generate_matern_device(int64_t n, const double* xy_dev, double sigma2, double range_a, double nugget,
                               double* A_dev, int64_t lda, void* stream);

/*
 * Per-kernel-class statistics of the last factorization when MXP_ATTR_PROFILE
 * is 1: launches, summed CUDA-event durations (ms, each measured on the
 * launching stream), and algorithmic flops (the n^3/3 decomposition: 2 nb^3
 * per GEMM update, nb^3 per SYRK update and per TRSM, nb^3/3 per POTRF).
 *   kernel_class  MXP_KCLASS_CHAIN (GEMM/SYRK chains + split-K reduction),
 *                 MXP_KCLASS_POTRF (diagonal tile), MXP_KCLASS_TRSM,
 *                 MXP_KCLASS_OTHER (pack/unpack/log-det/conversion)   (arg 2)
 *   launches, milliseconds, flops   host outputs (any may be NULL)     (args 3-5)
 */
enum mxp_kclass { MXP_KCLASS_CHAIN = 0, MXP_KCLASS_POTRF = 1, MXP_KCLASS_TRSM = 2, MXP_KCLASS_OTHER = 3 };
int mxp_chol_kernel_stats(mxp_plan_t plan, int kernel_class, int64_t* launches, double* milliseconds,
                          double* flops);

/*
 * Copy/compute timeline of the last host-streaming factorization (mxp_chol_factor /
 * mxp_chol_factor_tiles) run with MXP_ATTR_PROFILE = 1 -- the paper's C2G / G2C / Work rows
 * (Fig. 7): for each tile column k, three times in milliseconds since the start of
 * the factorization (CUDA events): [3k] the H2D loads of column k are complete, [3k+1] its D2H
 * write-backs are complete, [3k+2] its POTRF has finished; -1 where none was recorded.
 *   ms       host array of `count` doubles (may be NULL when count = 0)  (arg 2)
 *   count    capacity of ms                                            (arg 3)
 *   written  receives the number of entries available (3 Nt)            (arg 4)
 * Returns MXP_ESTATE when no such run exists.
 */
int mxp_chol_timeline(mxp_plan_t plan, double* ms, int64_t count, int64_t* written);

/*
 * Host-link byte ledger of the paper's out-of-core variants (P:202-206 sync /
 * async, P:235 V1, Alg. 3 P:281-303 V2, P:303 V3, volumes P:496-508) replayed over the static
 * left-looking task sequence of Alg. 2 (tasks (m, k) column by column, dealt 1-D cyclically to
 * `streams` streams that advance in lockstep) with a tile cache of hbm_bytes / (8 nb^2) FP64
 * tiles.  Pure host computation (no GPU); the engine itself runs variant 5.
 *   n, nb      problem size and tile size                                  (args 1, 2)
 *   variant    0 sync, 1 async (no cache: every update loads its accumulator and operands and
 *              writes the accumulator back), 2 V1 (accumulator resident per task), 3 V2 (+ LRU
 *              cache table of operands and final tiles), 4 V3 (V2 + L_kk pinned until the last
 *              TRSM of its column), 5 static dead-tile plan (each tile once each way; needs the
 *              live set), 6 MIN (Belady's optimal eviction for this sequence)      (arg 3)
 *   streams    1..64 concurrent task streams (the paper's multi-stream async)  (arg 4)
 *   hbm_bytes  device memory for tiles; 0 = unlimited                          (arg 5)
 *   out        [4]: host->device bytes, device->host bytes, tile loads, peak resident tiles
 * Returns MXP_ENOMEM when the capacity cannot hold the variant's minimum working set.
 */
int mxp_ooc_variant_volume(int64_t n, int64_t nb, int variant, int streams, int64_t hbm_bytes, int64_t* out);

/*
 * Scheduler diagnostics of the last factorization when MXP_ATTR_PROFILE is 1
 * (%globaltimer nanoseconds, summed over CTAs): [0] GEMM busy, [1] GEMM wait,
 * [2] TRSM busy, [3] TRSM wait, [4] #GEMM tasks, [5] #TRSM tasks, [6] first
 * CTA start, [7] last CTA end, [8] #CTAs that ran tasks, [9..12] POTRF phases, [13..15]
 * Ozaki GEMM loop (stage waits, MMA-completion waits, per-tile drains), [16..19] GEMM busy
 * by output precision (FP64, FP32, FP16, FP8), [20..23] their task counts, [24..26] Ozaki
 * issuing thread in MMA issue, bulk-copy issue, whole K loop, [28..32] native engine
 * (issuer waits for stages / refills / drained accumulators, drain time of warp 0, final
 * C update); then for each column k at [36+3k]: POTRF kernel start, Ready-wait done, end.
 *   out      host array of `count` entries (may be NULL when count = 0) (arg 2)
 *   count    capacity of out                                           (arg 3)
 *   written  receives the number of entries available (36 + 3 Nt)       (arg 4)
 */
int mxp_chol_sched_diagnostics(mxp_plan_t plan, uint64_t* out, int64_t count, int64_t* written);

/*
 * Multi-GPU (SURVEY 8(e), row-cyclic P x 1; P:343-363 distributes 1D
 * block-cyclic as well).  Every rank builds an identical plan (same n, nb, map,
 * attributes) with its own MXP_ATTR_RANK / MXP_ATTR_NRANKS, maps its peers'
 * workspaces, and then all ranks call the same factorization entry point
 * (mxp_chol_factor_device with a replicated input, or mxp_chol_factor_matern).
 * Each rank runs the tasks of its rows; every finished tile is pushed by the
 * copy engines into each peer's pool (NVLink P2P), so every rank ends with
 * the whole factor.  Ranks must not start factorization i+1 before every rank
 * returned from factorization i (a barrier between calls).
 *   mxp_chol_ipc_handle   exports this plan's workspace: handle_out receives
 *                         a 64-byte cudaIpcMemHandle, ws_bytes its size.
 *   mxp_chol_ipc_attach   maps peer `peer_rank`'s exported workspace (other
 *                         process); -4 if the layouts differ.
 *   mxp_chol_attach_peer_plan  same, for a peer plan in this process.
 */
int mxp_chol_ipc_handle(mxp_plan_t plan, void* handle_out, uint64_t* ws_bytes);
/* Host-only description of this rank's static task list (no GPU work):
 * counts[0..4] = GEMM, TRSM, QUANT, PREP, POTRF tasks; counts[5] = tiles this
 * rank owns.  streaming != 0 describes the host/generated-input list. */
int mxp_chol_describe(mxp_plan_t plan, int streaming, int64_t* counts);
int mxp_chol_ipc_attach(mxp_plan_t plan, int peer_rank, const void* handle, uint64_t ws_bytes);
int mxp_chol_attach_peer_plan(mxp_plan_t plan, int peer_rank, mxp_plan_t peer);

/* Destroy a plan and every device resource it owns. NULL is a no-op. */
void mxp_chol_plan_destroy(mxp_plan_t plan);

/* Page-locked host buffers for full-bandwidth H2D/D2H. */
int mxp_host_alloc(size_t bytes, void** ptr);
int mxp_host_free(void* ptr);

/* Human-readable text for a status code; detail of the last CUDA error. */
const char* mxp_strerror(int status);
const char* mxp_last_error(void);

/* ABI version of the loaded library (MXP_CHOL_ABI_VERSION). */
int mxp_chol_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MXP_CHOL_H */
