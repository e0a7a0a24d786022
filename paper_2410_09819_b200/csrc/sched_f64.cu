// sched_f64.cu -- the FP64 left-looking tile Cholesky as a device-resident
// static schedule (Alg. 1, Alg. 2).
//
// The paper's static scheduler gives every host thread a fixed, cyclic list of
// tasks and resolves dependencies by busy-waiting on a write-once progress
// table `Ready`.  On B200 the "threads" are persistent CTAs of
// one kernel (k_sched): they walk ONE fixed task list in order (each CTA takes
// the next task with an atomic ticket), and `Ready` lives in global memory
// (acquire/release flags).  Tasks are the paper's GEMM/SYRK updates and TRSMs
// at 64x128-block x K-chunk granularity; the POTRF of each diagonal tile runs
// in its own kernel (k_potrf_tile) on a reserved SM on a high-priority
// stream, spinning on the same table, so it never waits behind GEMM CTAs.
//
// Determinism: the accumulation order of every output block is fixed (chunks
// are applied in chunk order, guarded by a per-block chunk counter; the
// chunking is a function of (k, KC) only), so results are bitwise identical
// run to run, whatever CTA executes what.
//
// Deadlock freedom: a task only waits on tasks that precede it in the list;
// tasks are taken in list order by resident CTAs, so every awaited task is
// done or running.  Every wait has a 20 s timeout (error flag, no hang).
#include <math.h>

#include "dmma_gemm.cuh"
#include "quant.cuh"
#include "tc_block.cuh"
#include "oz_i8.cuh"
#include "tc_native.cuh"

namespace mxp {

namespace {

constexpr uint64_t WAIT_TIMEOUT_NS = 20ull * 1000 * 1000 * 1000;

// Thread 0 waits until *flag >= target.  Returns false to abort (failure in an
// earlier column at or before `col`, or timeout).
__device__ bool wait_flag(const int* flag, int target, const SchedArgs& a, int64_t col) {
    if (ld_acquire(flag) >= target) return true;
    uint64_t t0 = globaltimer();
    unsigned ns = 32;
    while (ld_acquire(flag) < target) {
        int64_t info = *(volatile int64_t*)a.dinfo;
        if (info != 0 && col >= (info - 1) / a.nb) return false;
        if (*(volatile int*)a.err) return false;
        if (globaltimer() - t0 > WAIT_TIMEOUT_NS) {
            if (a.tdiag && atomicCAS(a.tdiag + 7, 0, 1) == 0) {
                a.tdiag[0] = (int)(flag - a.ready);
                a.tdiag[1] = target;
                a.tdiag[2] = ld_acquire(flag);
                a.tdiag[3] = (int)smid();
                a.tdiag[4] = (int)blockIdx.x;
                a.tdiag[5] = (int)gridDim.x;
                a.tdiag[6] = (int)col;
                __threadfence();
            }
            atomicExch(a.err, 1);
            return false;
        }
        __nanosleep(ns);
        if (ns < 1024) ns *= 2;
    }
    return true;
}

__device__ __forceinline__ bool skip_column(const SchedArgs& a, int64_t col) {
    int64_t info = *(volatile int64_t*)a.dinfo;
    return (info != 0 && col >= (info - 1) / a.nb) || *(volatile int*)a.err;
}

// streaming modes (host input or generated tiles): tile t has been prepared
__device__ __forceinline__ bool wait_input(const SchedArgs& a, int64_t t, int64_t col) {
    return !(a.loaded || a.gen_mode || a.src_A) || wait_flag(a.prep_done + t, 1, a, col);
}

// Matern nu = 0.5 covariance entry (Eq. 2 closed form)
__device__ __forceinline__ double matern_entry(const SchedArgs& a, int64_t i, int64_t j) {
    const double dx = a.gen_xy[2 * i] - a.gen_xy[2 * j], dy = a.gen_xy[2 * i + 1] - a.gen_xy[2 * j + 1];
    double v = a.gen_sigma2 * exp(-sqrt(dx * dx + dy * dy) / a.gen_range);
    return i == j ? v + a.gen_nugget : v;
}

// chunk c of column k: fixed-size chunks over [0, k-1), then the singleton {k-1}
__device__ __forceinline__ void chunk_range(int64_t k, int64_t c, int64_t KC, int64_t& n0, int64_t& n1) {
    int64_t nfull = k >= 2 ? (k - 1 + KC - 1) / KC : 0;
    if (c < nfull) {
        n0 = c * KC;
        n1 = n0 + KC < k - 1 ? n0 + KC : k - 1;
    } else {
        n0 = k - 1;
        n1 = k;
    }
}

template <class C>
__device__ __forceinline__ void zero_acc(double (&acc)[C::MI][C::NI][2]) {
#pragma unroll
    for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < C::NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
}

// Stage transform of the non-FP64 GEMM path: cast_c(L) = deq(q_c(L)) of the
// operands stored finer than the compute precision c (P:42 down-casting).
struct CastPost {
    static constexpr bool active = true;
    const SchedArgs* a;
    int64_t m, k, n0, kper;
    int c;
    __device__ void operator()(int it, double* sA, double* sB) const {
        const int64_t n = n0 + it / kper;
        const int64_t ta = tile_index(a->Nt, m, n), tb = tile_index(a->Nt, k, n);
        const Cast ca = make_cast(a->prec[ta], c, a->amax_s[ta]);
        const Cast cb = make_cast(a->prec[tb], c, a->amax_s[tb]);
        if (ca.mode != P_FP64)
            for (int idx = threadIdx.x; idx < BK * CC::BM; idx += CC::NT) {
                double* p = sA + (idx / CC::BM) * CC::LDA_S + idx % CC::BM;
                *p = apply_cast(ca, *p);
            }
        if (cb.mode != P_FP64)
            for (int idx = threadIdx.x; idx < BK * CC::BN; idx += CC::NT) {
                double* p = sB + (idx / CC::BN) * CC::LDB_S + idx % CC::BN;
                *p = apply_cast(cb, *p);
            }
    }
};

// ---------------------------------------------------------------- GEMM task
// C(m,k)[block b] -= sum_{n in chunk c} A(m,n)[rows] A(k,n)[cols]^T
// GEMM task busy time, in total and by the output tile's precision (MXP_ATTR_PROFILE)
__device__ __forceinline__ void gemm_busy(const SchedArgs& a, int64_t t, uint64_t tw0) {
    const unsigned long long dt = globaltimer() - tw0;
    atomicAdd(a.stats + STAT_GEMM_BUSY, dt);
    const int p = a.prec ? a.prec[t] : P_FP64;
    atomicAdd(a.stats + STAT_GEMM_P + p, dt);
    atomicAdd(a.stats + STAT_GEMM_PN + p, 1ull);
}

template <bool CAST>
__device__ __forceinline__ bool task_gemm(const SchedArgs& a, int64_t m, int64_t k, int64_t b, int64_t c, double* smem,
                          int* s_flag) {
    const int64_t Nt = a.Nt, nb = a.nb;
    const int64_t SR = nb / CC::BM;
    const int64_t bi = b % SR, bj = b / SR;
    const int64_t t = tile_index(Nt, m, k);
    int64_t n0, n1;
    chunk_range(k, c, a.KC, n0, n1);
    int* chunk_flag = a.blk_chunk + t * a.NB + b;
    uint64_t tw0 = 0;
    if (threadIdx.x == 0) {
        if (a.stats) tw0 = globaltimer();
        bool ok = wait_input(a, t, k);
        for (int64_t n = n0; n < n1 && ok; ++n) {
            ok = wait_flag(a.ready + tile_index(Nt, m, n), a.epoch, a, k) &&
                 wait_flag(a.ready + tile_index(Nt, k, n), a.epoch, a, k);
        }
        if (ok) ok = wait_flag(chunk_flag, (int)c, a, k);
        *s_flag = ok;
        if (a.stats) {
            uint64_t tw1 = globaltimer();
            atomicAdd(a.stats + STAT_GEMM_WAIT, tw1 - tw0);
            tw0 = tw1;
        }
    }
    __syncthreads();
    if (!*s_flag) return false;

    const int64_t kper = nb / BK;
    const int nk = (int)((n1 - n0) * kper);
    const int64_t roff = bi * CC::BM, coff = bj * CC::BN;
    double* pool = a.pool;
    const int32_t* slot = a.slot;
    // Stateful operand walk: the mainloop asks for K-chunks in increasing
    // order, so tile pointers are looked up only when the walk enters the next
    // tile n (once per nb/BK stages) -- no slot loads or divisions per stage.
    int64_t cur_n = n0, kcol = 0;
    const double* ta = tile_ptr(pool, slot, Nt, nb, m, n0) + roff;
    const double* tb = tile_ptr(pool, slot, Nt, nb, k, n0) + coff;
    auto src = [&](int, const double*& pa, const double*& pb) {
        if (kcol == nb) {
            kcol = 0;
            ++cur_n;
            ta = tile_ptr(pool, slot, Nt, nb, m, cur_n) + roff;
            tb = tile_ptr(pool, slot, Nt, nb, k, cur_n) + coff;
        }
        pa = ta + kcol * nb;
        pb = tb + kcol * nb;
        kcol += BK;
    };
    double acc[CC::MI][CC::NI][2];
    zero_acc<CC>(acc);
    const int cprec = a.prec ? a.prec[t] : P_FP64;  // compute precision = the output tile's (G12)
    if constexpr (!CAST) {
        // FP64 compute: every stored operand is exactly representable (up-casts
        // are the identity), so the raw cp.async pipeline is already exact.
        gemm_mainloop<CC>(acc, src, nb, nb, nk, smem);
    } else {
        // operands stored finer than c are cast in shared memory, stage by stage
        CastPost post{&a, m, k, n0, kper, cprec};
        gemm_mainloop<CC>(acc, src, nb, nb, nk, smem, post);
    }
    double* Ct = tile_ptr(pool, slot, Nt, nb, m, k) + roff + coff * nb;
    // (loads of a fragment row first, then the stores: an interleaved
    // load-subtract-store per element is serialized by possible aliasing)
#pragma unroll
    for (int mi = 0; mi < CC::MI; ++mi) {
        double cv[CC::NI][2];
#pragma unroll
        for (int ni = 0; ni < CC::NI; ++ni)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                int r, cc;
                frag_pos<CC>(mi, ni, i, r, cc);
                cv[ni][i] = __ldcg(Ct + r + (int64_t)cc * nb);
            }
#pragma unroll
        for (int ni = 0; ni < CC::NI; ++ni)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                int r, cc;
                frag_pos<CC>(mi, ni, i, r, cc);
                __stcg(Ct + r + (int64_t)cc * nb, cv[ni][i] - acc[mi][ni][i]);
            }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        st_release(chunk_flag, (int)c + 1);
        atom_add_release(a.gemm_done + t, 1);
        if (a.stats) {
            gemm_busy(a, t, tw0);
            atomicAdd(a.stats + STAT_GEMM_N, 1ull);
        }
    }
    return true;
}

__device__ __noinline__ bool task_gemm_cast(const SchedArgs& a, int64_t m, int64_t k, int64_t b, int64_t c,
                                           double* smem, int* s_flag) {
    return task_gemm<true>(a, m, k, b, c, smem, s_flag);
}

// ---------------------------------------------------------------- TRSM task
// X L_kk^T = C on rows [64r, 64r+64) of tile (m,k), in place (Alg. 2
// P:269, G3).  Blocked by 128 columns J with the inverses W_J = L_JJ^-1 from
// the POTRF kernel (MAGMA-style):  X[:,J] = (C[:,J] - X[:,<J] L[J,<J]^T) W_J^T.
__device__ __forceinline__ bool task_trsm(const SchedArgs& a, int64_t m, int64_t k, int64_t r, double* smem, int* s_flag) {
    const int64_t Nt = a.Nt, nb = a.nb, S = nb / 128;
    const int64_t t = tile_index(Nt, m, k);
    uint64_t tw0 = 0;
    if (threadIdx.x == 0) {
        if (a.stats) tw0 = globaltimer();
        bool ok = wait_input(a, t, k) && wait_flag(a.ready + tile_index(Nt, k, k), a.epoch, a, k) &&
                  wait_flag(a.gemm_done + t, a.gemm_expected[t], a, k);
        *s_flag = ok;
        if (a.stats) {
            uint64_t tw1 = globaltimer();
            atomicAdd(a.stats + STAT_TRSM_WAIT, tw1 - tw0);
            tw0 = tw1;
        }
    }
    sync_workers();
    if (!*s_flag) return false;
    double* X = tile_ptr(a.pool, a.slot, Nt, nb, m, k) + r * 64;
    const double* L = tile_ptr(a.pool, a.slot, Nt, nb, k, k);
    const double* Wk = a.wbuf + k * S * (128 * 128);
    double xmax = 0.0;  // max |X| over this task's rows (tile amax for quantization, G11)
    for (int64_t J = 0; J < S; ++J) {
        double acc[CC::MI][CC::NI][2];
        zero_acc<CC>(acc);
        if (J > 0) {
            auto src = [&](int it, const double*& pa, const double*& pb) {
                int64_t kcol = (int64_t)it * BK;
                pa = X + kcol * nb;
                pb = L + J * 128 + kcol * nb;
            };
            gemm_mainloop<CC>(acc, src, nb, nb, (int)(J * 128 / BK), smem);
        }
        double* XJ = X + J * 128 * nb;
#pragma unroll
        for (int mi = 0; mi < CC::MI; ++mi) {  // (loads first, then stores: see task_gemm)
            double cv[CC::NI][2];
#pragma unroll
            for (int ni = 0; ni < CC::NI; ++ni)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    int rr, cc;
                    frag_pos<CC>(mi, ni, i, rr, cc);
                    cv[ni][i] = __ldcg(XJ + rr + (int64_t)cc * nb);
                }
#pragma unroll
            for (int ni = 0; ni < CC::NI; ++ni)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    int rr, cc;
                    frag_pos<CC>(mi, ni, i, rr, cc);
                    __stcg(XJ + rr + (int64_t)cc * nb, cv[ni][i] - acc[mi][ni][i]);
                }
        }
        __threadfence_block();
        sync_workers();
        zero_acc<CC>(acc);
        const double* W = Wk + J * (128 * 128);
        auto src2 = [&](int it, const double*& pa, const double*& pb) {
            int64_t kcol = (int64_t)it * BK;
            pa = XJ + kcol * nb;
            pb = W + kcol * 128;
        };
        gemm_mainloop<CC>(acc, src2, nb, 128, 128 / BK, smem);
#pragma unroll
        for (int mi = 0; mi < CC::MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < CC::NI; ++ni)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    int rr, cc;
                    frag_pos<CC>(mi, ni, i, rr, cc);
                    __stcg(XJ + rr + (int64_t)cc * nb, acc[mi][ni][i]);
                    xmax = fmax(xmax, fabs(acc[mi][ni][i]));
                }
        __threadfence_block();
        sync_workers();
    }
    for (int o = 16; o > 0; o >>= 1) xmax = fmax(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
    if ((threadIdx.x & 31) == 0) atomic_max_abs(a.amax_x + t, xmax);
    __threadfence();
    sync_workers();
    if (threadIdx.x == 0) {
        int old = atom_add_release(a.trsm_done + t, 1);
        const bool fp64 = !a.prec || !a.qtile[t];  // no QUANT task follows
        if (old + 1 == (int)(nb / 64) && fp64) {
            // FP64 tile: stored values are the TRSM result; amax_s drives later down-casts
            a.amax_s[t] = amax_of(a.amax_x + t);
            __threadfence();
            st_release(a.ready + t, a.epoch);
            atom_add_release(a.col_ready + k, 1);
        }
        if (a.stats) {
            atomicAdd(a.stats + STAT_TRSM_BUSY, globaltimer() - tw0);
            atomicAdd(a.stats + STAT_TRSM_N, 1ull);
        }
    }
    return true;
}

__device__ __noinline__ bool task_trsm_ool(const SchedArgs& a, int64_t m, int64_t k, int64_t r, double* smem,
                                          int* s_flag) {
    return task_trsm(a, m, k, r, smem, s_flag);
}

// ------------------------------------------------------ tcgen05 GEMM task
// Tiles stored below FP64 (G12): C(m,k)[128x128 block b] -= sum over the
// chunk of cast_c(A(m,n)) cast_c(A(k,n))^T on the 5th-gen tensor cores
// (kind::tf32; 3xTF32 when c = FP32, else 1xTF32 on exact FP16/E4M3 values),
// fp32 accumulator in TMEM, added into the fp64 container.
template <bool THREE>
__device__ __noinline__ bool task_gemm_tc(const SchedArgs& a, int64_t m, int64_t k, int64_t b, int64_t c, int cprec,
                             uint8_t* smem, uint64_t* mbar, uint32_t tmem, int* s_flag) {
    const int64_t Nt = a.Nt, nb = a.nb, S = nb / 128;
    const int64_t bi = b % S, bj = b / S;
    const int64_t t = tile_index(Nt, m, k);
    int64_t n0, n1;
    chunk_range(k, c, a.KC, n0, n1);
    int* chunk_flag = a.blk_chunk + t * a.NB + b;
    uint64_t tw0 = 0;
    if (threadIdx.x == 0) {
        if (a.stats) tw0 = globaltimer();
        bool ok = wait_input(a, t, k);
        for (int64_t n = n0; n < n1 && ok; ++n)
            ok = wait_flag(a.ready + tile_index(Nt, m, n), a.epoch, a, k) &&
                 wait_flag(a.ready + tile_index(Nt, k, n), a.epoch, a, k);
        if (ok) ok = wait_flag(chunk_flag, (int)c, a, k);
        *s_flag = ok;
        if (a.stats) {
            uint64_t tw1 = globaltimer();
            atomicAdd(a.stats + STAT_GEMM_WAIT, tw1 - tw0);
            tw0 = tw1;
        }
    }
    __syncthreads();
    if (!*s_flag) return false;
    const int64_t kper = nb / tc::KS;
    const int nsteps = (int)((n1 - n0) * kper);
    const int64_t roff = bi * 128, coff = bj * 128;
    // stateful K walk: tile pointers and casts change only at tile boundaries
    int64_t cur_n = n0 - 1, kcol = nb;
    tc::Chunk cur{};
    auto src = [&](int) {
        if (kcol == nb) {
            kcol = 0;
            ++cur_n;
            const int64_t ta = tile_index(Nt, m, cur_n), tb = tile_index(Nt, k, cur_n);
            cur.a = tile_ptr(a.pool, a.slot, Nt, nb, m, cur_n) + roff;
            cur.b = tile_ptr(a.pool, a.slot, Nt, nb, k, cur_n) + coff;
            cur.ca = make_cast(a.prec[ta], cprec, a.amax_s[ta]);
            cur.cb = make_cast(a.prec[tb], cprec, a.amax_s[tb]);
        }
        tc::Chunk ch = cur;
        ch.a += kcol * nb;
        ch.b += kcol * nb;
        kcol += tc::KS;
        return ch;
    };
    double* Ct = tile_ptr(a.pool, a.slot, Nt, nb, m, k) + roff + coff * nb;
    tc::block_gemm<THREE>(Ct, nb, src, nsteps, nb, nb, smem, mbar, tmem);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        st_release(chunk_flag, (int)c + 1);
        atom_add_release(a.gemm_done + t, 1);
        if (a.stats) {
            gemm_busy(a, t, tw0);
            atomicAdd(a.stats + STAT_GEMM_N, 1ull);
        }
    }
    return true;
}

// tcgen05 GEMM task on operand images: the same contraction as task_gemm_tc,
// operands bulk-copied from the per-tile fp32 images of cast_c(L) (written
// once by the QUANT task of each operand tile), image e = max(c, p_operand)
// (an operand stored at or below c is used as stored).
template <bool THREE, int NST>
__device__ __noinline__ bool task_gemm_img(const SchedArgs& a, int64_t m, int64_t k, int64_t b, int64_t c,
                                           int cprec, uint8_t* smem, uint32_t tmem, int* s_flag) {
    const int64_t Nt = a.Nt, nb = a.nb, S = nb / 128;
    const int64_t bi = b % S, bj = b / S;
    const int64_t t = tile_index(Nt, m, k);
    int64_t n0, n1;
    chunk_range(k, c, a.KC, n0, n1);
    int* chunk_flag = a.blk_chunk + t * a.NB + b;
    uint64_t tw0 = 0;
    if (threadIdx.x == 0) {
        if (a.stats) tw0 = globaltimer();
        bool ok = wait_input(a, t, k);
        for (int64_t n = n0; n < n1 && ok; ++n)
            ok = wait_flag(a.ready + tile_index(Nt, m, n), a.epoch, a, k) &&
                 wait_flag(a.ready + tile_index(Nt, k, n), a.epoch, a, k);
        if (ok) ok = wait_flag(chunk_flag, (int)c, a, k);
        *s_flag = ok;
        if (a.stats) {
            uint64_t tw1 = globaltimer();
            atomicAdd(a.stats + STAT_GEMM_WAIT, tw1 - tw0);
            tw0 = tw1;
        }
    }
    __syncthreads();
    if (!*s_flag) return false;
    const int64_t kper = nb / tc::KS;
    const int nsteps = (int)((n1 - n0) * kper);
    const int64_t aoff = bi * kper * tc::SUB_BYTES, boff = bj * kper * tc::SUB_BYTES;
    int64_t cur_n = n0 - 1, kc = kper;
    const uint8_t *ahi = nullptr, *alo = nullptr, *bhi = nullptr, *blo = nullptr;
    auto src = [&](int) {
        if (kc == kper) {
            kc = 0;
            ++cur_n;
            const int64_t ta = tile_index(Nt, m, cur_n), tb = tile_index(Nt, k, cur_n);
            const int ea = a.prec[ta] > cprec ? a.prec[ta] : cprec;
            const int eb = a.prec[tb] > cprec ? a.prec[tb] : cprec;
            // tf32 images: slot e - 1 of e = max(c, p); native mode: the FP32 consumers' slot 0
            // (values of cast_max(FP32, p)), remainder slot 3 only for operands stored at FP32 or finer
            ahi = a.shadow + a.img[4 * ta + (a.native ? 0 : ea - 1)] + aoff;
            bhi = a.shadow + a.img[4 * tb + (a.native ? 0 : eb - 1)] + boff;
            const bool la = THREE && (a.native ? a.img[4 * ta + 3] >= 0 : ea == P_FP32);
            const bool lb = THREE && (a.native ? a.img[4 * tb + 3] >= 0 : eb == P_FP32);
            alo = la ? a.shadow + a.img[4 * ta + 3] + aoff : nullptr;
            blo = lb ? a.shadow + a.img[4 * tb + 3] + boff : nullptr;
        }
        const int64_t o = kc * tc::SUB_BYTES;
        ++kc;
        return tc::ImgStep{ahi + o, alo ? alo + o : nullptr, bhi + o, blo ? blo + o : nullptr};
    };
    double* Ct = tile_ptr(a.pool, a.slot, Nt, nb, m, k) + bi * 128 + bj * 128 * nb;
    tc::block_gemm_img<THREE, NST>(Ct, nb, src, nsteps, smem, tmem);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        st_release(chunk_flag, (int)c + 1);
        atom_add_release(a.gemm_done + t, 1);
        if (a.stats) {
            gemm_busy(a, t, tw0);
            atomicAdd(a.stats + STAT_GEMM_N, 1ull);
        }
    }
    return true;
}

// GEMM task of an FP16 / FP8 output tile at native operand width (tc_native.cuh):
// C(m,k)[128x128 block b] -= sum over the chunk of cast_c(L(m,n)) cast_c(L(k,n))^T
// as fp16 (kind::f16) or E4M3 (kind::f8f6f4) code products, rescaled per K tile.
template <int KIND>
__device__ __noinline__ bool task_gemm_nat(const SchedArgs& a, int64_t m, int64_t k, int64_t b, int64_t c,
                                           uint8_t* smem, uint32_t tmem, int* s_flag) {
    const int64_t Nt = a.Nt, nb = a.nb, S = nb / 128;
    const int64_t bi = b % S, bj = b / S;
    const int64_t t = tile_index(Nt, m, k);
    int64_t n0, n1;
    chunk_range(k, c, a.KC, n0, n1);
    int* chunk_flag = a.blk_chunk + t * a.NB + b;
    uint64_t tw0 = 0;
    if (threadIdx.x == 0) {
        if (a.stats) tw0 = globaltimer();
        bool ok = wait_input(a, t, k);
        for (int64_t n = n0; n < n1 && ok; ++n)
            ok = wait_flag(a.ready + tile_index(Nt, m, n), a.epoch, a, k) &&
                 wait_flag(a.ready + tile_index(Nt, k, n), a.epoch, a, k);
        if (ok) ok = wait_flag(chunk_flag, (int)c, a, k);
        *s_flag = ok;
        if (a.stats) {
            uint64_t tw1 = globaltimer();
            atomicAdd(a.stats + STAT_GEMM_WAIT, tw1 - tw0);
            tw0 = tw1;
        }
    }
    __syncthreads();
    if (!*s_flag) return false;
    // img[4t+1]: fp16 codes (FP16 and FP32 outputs), img[4t+2]: E4M3 codes, img[4t+3]: fp16 remainders
    constexpr int slot = KIND == nat::K_F8 ? 2 : 1, sk = KIND == nat::K_F8 ? 1 : 0;
    auto src = [&](int i) {
        const int64_t n = n0 + i;
        const int64_t ta = tile_index(Nt, m, n), tb = tile_index(Nt, k, n);
        nat::NatTile o;
        o.a = a.shadow + a.img[4 * ta + slot] + nat::chunk_offset(KIND, nb, bi, 0);
        o.b = a.shadow + a.img[4 * tb + slot] + nat::chunk_offset(KIND, nb, bj, 0);
        o.al = o.bl = nullptr;
        if (KIND == nat::K_F32X2) {
            const long long ra = a.img[4 * ta + 3], rb = a.img[4 * tb + 3];
            if (ra >= 0) o.al = a.shadow + ra + nat::chunk_offset(KIND, nb, bi, 0);
            if (rb >= 0) o.bl = a.shadow + rb + nat::chunk_offset(KIND, nb, bj, 0);
        }
        nat::inv_scales(__ldcg(a.iscale + 3 * ta + sk), __ldcg(a.iscale + 3 * tb + sk), o.inv0, o.inv1);
        return o;
    };
    double* Ct = tile_ptr(a.pool, a.slot, Nt, nb, m, k) + bi * 128 + bj * 128 * nb;
    nat::block_gemm<KIND>(Ct, nb, src, (int)(n1 - n0), (int)(nb / nat::ke(KIND)), smem, tmem, a.stats,
                          a.oz_prefetch);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        st_release(chunk_flag, (int)c + 1);
        atom_add_release(a.gemm_done + t, 1);
        if (a.stats) {
            gemm_busy(a, t, tw0);
            atomicAdd(a.stats + STAT_GEMM_N, 1ull);
        }
    }
    return true;
}

// FP64 GEMM task on the int8 tensor cores (Ozaki scheme, oz_i8.cuh; SURVEY
// §8(f) N4): C(m,k)[128x64 block b] -= sum over the chunk of L(m,n) L(k,n)^T,
// operands from the int8 slice images written by the QUANT tasks, levels
// drained to fp64 after every tile of K.
template <bool RACC>
__device__ __noinline__ bool task_gemm_oz(const SchedArgs& a, int64_t m, int64_t k, int64_t b, int64_t c,
                                          uint8_t* smem, uint32_t tmem, int* s_flag) {
    __shared__ int s_uni;
    const int64_t Nt = a.Nt, nb = a.nb, SR = nb / 128;
    const int64_t bi = b % SR, bj = b / SR;  // 128-row block bi, 64-column block bj
    const int64_t t = tile_index(Nt, m, k);
    int64_t n0, n1;
    chunk_range(k, c, a.KC, n0, n1);
    int* chunk_flag = a.blk_chunk + t * a.NB + b;
    uint64_t tw0 = 0;
    if (threadIdx.x == 0) {
        if (a.stats) tw0 = globaltimer();
        bool ok = wait_input(a, t, k);
        for (int64_t n = n0; n < n1 && ok; ++n)
            ok = wait_flag(a.ready + tile_index(Nt, m, n), a.epoch, a, k) &&
                 wait_flag(a.ready + tile_index(Nt, k, n), a.epoch, a, k);
        if (ok) ok = wait_flag(chunk_flag, (int)c, a, k);
        // one drain for the chunk when no row scale changes inside it (oz_flag of the tiles after
        // the first, set by their QUANTs before the Ready words just acquired)
        int uni = (ok && a.oz_flag) ? 1 : 0;
        for (int64_t n = n0 + 1; n < n1 && uni; ++n)
            if (__ldcg(a.oz_flag + tile_index(Nt, m, n)) | __ldcg(a.oz_flag + tile_index(Nt, k, n))) uni = 0;
        s_uni = uni;
        *s_flag = ok;
        if (a.stats) {
            uint64_t tw1 = globaltimer();
            atomicAdd(a.stats + STAT_GEMM_WAIT, tw1 - tw0);
            tw0 = tw1;
        }
    }
    __syncthreads();
    if (!*s_flag) return false;
    const bool uniform = s_uni != 0;
    const int s = a.oz_slices;
    const int64_t sc_off = (int64_t)s * nb * nb;
    auto src = [&](int i) {
        const int64_t n = n0 + i;
        const uint8_t* ia = a.shadow + a.oz_img[tile_index(Nt, m, n)];
        const uint8_t* ib = a.shadow + a.oz_img[tile_index(Nt, k, n)];
        oz::OzTile o;
        o.a = ia + oz::chunk_offset(nb, 0, bi, 0);
        o.b = ib + oz::chunk_offset(nb, 0, bj >> 1, 0) + 2048 * (bj & 1);
        o.sa = reinterpret_cast<const double*>(ia + sc_off) + bi * 128;
        o.sb = reinterpret_cast<const double*>(ib + sc_off) + bj * 64;
        return o;
    };
    double* Ct = tile_ptr(a.pool, a.slot, Nt, nb, m, k) + bi * 128 + bj * 64 * nb;
    oz::block_gemm<RACC>(Ct, nb, src, (int)(n1 - n0), s, (int)(nb / 32), nb, smem, tmem, a.oz_prefetch, a.stats,
                         uniform);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        st_release(chunk_flag, (int)c + 1);
        atom_add_release(a.gemm_done + t, 1);
        if (a.stats) {
            gemm_busy(a, t, tw0);
            atomicAdd(a.stats + STAT_GEMM_N, 1ull);
        }
    }
    return true;
}

// Int8 slice image of rows [64r, 64r+64) of a final tile (Ozaki operands):
// per-row scale 2^(E-6) from the row max, then s digits per element.  Thread
// (row = tid & 63, half = tid >> 6) covers half of the row's columns.
__device__ void oz_slice_rows(const SchedArgs& a, const double* X, int64_t m, int64_t k, int64_t r, uint8_t* img,
                              double* red) {
    const int64_t nb = a.nb;
    const int s = a.oz_slices;
    const int tid = threadIdx.x, row = tid & 63, half = tid >> 6;
    const int64_t c0 = half * (nb / 2), c1 = c0 + nb / 2;
    double mx = 0.0;
    for (int64_t cc = c0; cc < c1; ++cc) mx = fmax(mx, fabs(__ldcg(X + row + cc * nb)));
    red[tid] = mx;
    sync_workers();
    double inv;
    const double rmax = fmax(red[row], red[row + 64]);
    double sc = oz::row_scale(rmax, inv);
    if (a.oz_flag && !(rmax > 0.0)) {  // a zero row: the smallest scale, replaced by any later one
        sc = 0x1p-1000;
        inv = 0x1p994;
    } else if (a.oz_flag) {  // two binades of headroom, so the running scale rarely has to grow
        sc *= 4.0;
        inv *= 0.25;
    }
    if (a.oz_flag && k > 0) {
        // Running row scales: a row keeps the scale it had in tile (m, k-1) unless this tile holds
        // a larger entry, so consecutive tiles of a row usually share their scales and a GEMM
        // chunk over them can accumulate in int32 TMEM across its K tiles (one drain); a tile
        // whose scales changed is flagged (oz_flag) and its chunk drains per tile.  A scale is
        // then >= the tile's own row max (as precise, or one binade coarser for the smaller rows
        // of a tile), and exactly the row max where the row max grew.
        const uint8_t* pimg = a.shadow + a.oz_img[tile_index(a.Nt, m, k - 1)];
        const double ps = __ldcg(reinterpret_cast<const double*>(pimg + (int64_t)s * nb * nb) + r * 64 + row);
        if (ps >= 0.25 * sc) {  // (the previous scale still covers this row's max)
            sc = ps;
            inv = 1.0 / (64.0 * ps);  // ps = 2^(E-6): inv = 2^-E, exact
        } else if (half == 0) {
            atomicOr(a.oz_flag + tile_index(a.Nt, m, k), 1);
        }
    }
    if (half == 0) reinterpret_cast<double*>(img + (int64_t)s * nb * nb)[r * 64 + row] = sc;
    for (int64_t k0 = c0; k0 < c1; k0 += 16) {
        double x[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) x[e] = __ldcg(X + row + (k0 + e) * nb);
        oz::write_slices16(img, nb, s, (int)(r * 64 + row), (int)k0, x, inv);
    }
}

// --------------------------------------------------------------- QUANT task
// L_mk = deq(q_p(X)) on rows [64r, 64r+64) once every TRSM row task of the
// tile has contributed to its amax (quantize once per task, after TRSM; O4).
__device__ __noinline__ bool task_quant(const SchedArgs& a, int64_t m, int64_t k, int64_t r, double* red,
                                        int* s_flag) {
    const int64_t Nt = a.Nt, nb = a.nb;
    const int64_t t = tile_index(Nt, m, k);
    if (threadIdx.x == 0) *s_flag = wait_flag(a.trsm_done + t, (int)(nb / 64), a, k);
    sync_workers();
    if (!*s_flag) return false;
    const int p = a.prec ? a.prec[t] : P_FP64;
    const double amax = amax_of(a.amax_x + t);
    const double sc = tile_scale(p, amax), isc = 1.0 / sc;
    const double amax_st = quantize_value(p, amax, sc, isc);  // q is monotone: max|q(x)| = q(max|x|)
    double* X = tile_ptr(a.pool, a.slot, Nt, nb, m, k) + r * 64;
    // operand images of this tile (rows [64r, 64r+64)): fp32 values of
    // cast_e(L) = deq(q_e(L)) with the stored amax (identity when e <= p),
    // FP32 image split into TF32 hi + lo (3xTF32)
    uint8_t* im[4] = {nullptr, nullptr, nullptr, nullptr};
    Cast ce[3];
    bool any = false;
    if (a.img) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const long long o = a.img[4 * t + e];
            if (o >= 0) im[e] = a.shadow + o, any = true;
        }
#pragma unroll
        for (int e = 0; e < 3; ++e) ce[e] = make_cast(p, e + 1, amax_st);
    }
    if (p != P_FP64 || any) {
        const int64_t kper = nb / tc::KS;
        for (int64_t idx = threadIdx.x; idx < 16 * nb; idx += CC::NT) {
            const int q4 = (int)(idx & 15), col = (int)(idx >> 4);
            double* q = X + 4 * q4 + (int64_t)col * nb;
            double2 v01 = __ldcg(reinterpret_cast<const double2*>(q));
            double2 v23 = __ldcg(reinterpret_cast<const double2*>(q + 2));
            double x[4] = {v01.x, v01.y, v23.x, v23.y};
            if (p != P_FP64) {
#pragma unroll
                for (int i = 0; i < 4; ++i) x[i] = quantize_value(p, x[i], sc, isc);
                __stcg(reinterpret_cast<double2*>(q), make_double2(x[0], x[1]));
                __stcg(reinterpret_cast<double2*>(q + 2), make_double2(x[2], x[3]));
            }
            if (!any) continue;
            const int row = (int)(r * 64) + 4 * q4;
            const int64_t chunk = (int64_t)(row >> 7) * kper + (col >> 4);
            const uint32_t off = tc::sw_offset(row & 127, col & 15);
#pragma unroll
            for (int e = 0; e < 3; ++e) {
                if (!im[e] || a.native) continue;
                float f[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) f[i] = (float)apply_cast(ce[e], x[i]);
                uint8_t* dst = im[e] + chunk * tc::SUB_BYTES + off;
                if (e == 0 && im[3]) {  // FP32: hi = RNE_tf32(v), lo = RNE_tf32(v - hi)
                    float h[4], l[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) h[i] = tc::rne_tf32(f[i]), l[i] = tc::rne_tf32(f[i] - h[i]);
                    __stcg(reinterpret_cast<float4*>(dst), make_float4(h[0], h[1], h[2], h[3]));
                    __stcg(reinterpret_cast<float4*>(im[3] + chunk * tc::SUB_BYTES + off),
                           make_float4(l[0], l[1], l[2], l[3]));
                } else {  // (native FP32 image of an FP16 / E4M3 operand: its values are exact in TF32)
                    __stcg(reinterpret_cast<float4*>(dst), make_float4(f[0], f[1], f[2], f[3]));
                }
            }
        }
    }
    if (a.native && (im[1] || im[2] || im[3])) {  // native-width code images (tc_native.cuh)
        sync_workers();
        // scale of the codes: the stored scale when the tile is stored at or below the image's
        // precision (up-cast: the stored codes themselves, exact in fp16 / E4M3), else the
        // down-cast's own scale from the stored amax (G11)
        const double s16 = p >= P_FP16 ? sc : tile_scale(P_FP16, amax_st);
        const double s8 = p == P_FP8 ? sc : tile_scale(P_FP8, amax_st);
        const Cast c16 = make_cast(p, P_FP16, amax_st), c8 = make_cast(p, P_FP8, amax_st);
        const int tid = threadIdx.x, row = (int)(r * 64) + (tid & 63), half = tid >> 6;
        const int64_t c0 = half * (nb / 2), c1 = c0 + nb / 2;
        for (int64_t k0 = c0; k0 < c1; k0 += 16) {
            double x[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) x[e] = __ldcg(X + (tid & 63) + (k0 + e) * nb);
            if (im[1]) {
                double y[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) y[e] = apply_cast(c16, x[e]);
                nat::write_f16_16(im[1], nb, row, (int)k0, y, s16);
            }
            if (im[3]) nat::write_f16rem_16(im[3], nb, row, (int)k0, x, s16);  // (x stored at FP32 or finer)
            if (im[2]) {
                double y[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) y[e] = apply_cast(c8, x[e]);
                nat::write_f8_16(im[2], nb, row, (int)k0, y, s8);
            }
        }
        if (tid == 0) {
            a.iscale[3 * t + 0] = s16;
            a.iscale[3 * t + 1] = s8;
        }
    }
    if (a.sto && a.sto[t] >= 0) {  // compact pool: the tile's storage image (codes, column-major)
        sync_workers();
        uint8_t* dst = a.shadow + a.sto[t];
        for (int64_t idx = threadIdx.x; idx < 16 * nb; idx += CC::NT) {
            const int q4 = (int)(idx & 15), col = (int)(idx >> 4);
            const double* q = X + 4 * q4 + (int64_t)col * nb;
            const double2 v01 = __ldcg(reinterpret_cast<const double2*>(q));
            const double2 v23 = __ldcg(reinterpret_cast<const double2*>(q + 2));
            const int64_t e = (int64_t)col * nb + r * 64 + 4 * q4;  // element index in the tile
            if (p == P_FP32) {
                __stcg(reinterpret_cast<float4*>(dst + 4 * e),
                       make_float4((float)v01.x, (float)v01.y, (float)v23.x, (float)v23.y));
            } else if (p == P_FP16) {
                const unsigned short h0 = __half_as_ushort(__double2half(v01.x * sc));
                const unsigned short h1 = __half_as_ushort(__double2half(v01.y * sc));
                const unsigned short h2 = __half_as_ushort(__double2half(v23.x * sc));
                const unsigned short h3 = __half_as_ushort(__double2half(v23.y * sc));
                __stcg(reinterpret_cast<uint2*>(dst + 2 * e),
                       make_uint2((uint32_t)h0 | ((uint32_t)h1 << 16), (uint32_t)h2 | ((uint32_t)h3 << 16)));
            } else {
                unsigned short lo, hi;
                asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(lo) : "f"((float)(v01.y * sc)), "f"((float)(v01.x * sc)));
                asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(hi) : "f"((float)(v23.y * sc)), "f"((float)(v23.x * sc)));
                __stcg(reinterpret_cast<uint32_t*>(dst + e), (uint32_t)lo | ((uint32_t)hi << 16));
            }
        }
        if (threadIdx.x == 0) a.iscale[3 * t + 2] = sc;
    }
    if (a.oz_img && a.oz_img[t] >= 0) {  // int8 slices of the stored values (FP64 GEMM operands)
        if (a.img_prev && threadIdx.x == 0) {  // out of core: the image slot's previous tile (pm, .) has died
            const int32_t prev = a.img_prev[t];
            bool ok = true;
            if (prev >= 0) {
                int64_t pc = 0, r = prev;
                while (r >= Nt - pc) { r -= Nt - pc; ++pc; }
                const int64_t pm = pc + r;
                ok = wait_flag(a.col_ready + pm, (int)(Nt - pm), a, k);
            }
            *s_flag = ok;
        }
        __threadfence_block();
        sync_workers();
        if (!*s_flag) return false;
        oz_slice_rows(a, X, m, k, r, a.shadow + a.oz_img[t], red);
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");  // images are read by bulk copies
    __threadfence();
    sync_workers();
    if (threadIdx.x == 0) {
        a.amax_s[t] = amax_st;
        __threadfence();
        int old = atom_add_release(a.quant_done + t, 1);
        if (old + 1 == (int)(nb / 64)) {
            st_release(a.ready + t, a.epoch);
            atom_add_release(a.col_ready + k, 1);
        }
    }
    return true;
}

// ---------------------------------------------------------------- PREP task
// Host-streaming mode: once the DMA of tile (m,k) has landed, set its padding
// (0, and 1 on the padded diagonal) and store it at its precision
// (O3: A^ = deq(q_p(A)), tile amax reduced inside this CTA).
__device__ __noinline__ bool task_prep(const SchedArgs& a, int64_t m, int64_t k, double* red, int* s_flag) {
    const int64_t Nt = a.Nt, nb = a.nb, n = a.n;
    const int64_t t = tile_index(Nt, m, k);
    if (threadIdx.x == 0) {
        bool ok;
        if (a.gen_mode || a.src_A) {
            ok = !skip_column(a, k);
            const int32_t prev = a.prev_owner[t];
            int64_t pm = 0, pc = 0;
            if (prev >= 0) {
                int64_t r = prev;
                while (r >= Nt - pc) { r -= Nt - pc; ++pc; }
                pm = pc + r;
            }
            if (ok && prev >= 0 && (a.compact || a.ring_all) && pm != pc) {
                // compact / Ozaki ring: an off-diagonal tile's slot is free once the tile is final
                ok = wait_flag(a.ready + prev, a.epoch, a, k);
            } else if (ok && prev >= 0) {
                // out of core: the slot's previous tile (pm, .) dies with column pm; a diagonal
                // tile of the Ozaki ring with its own column (pm = pc)
                ok = wait_flag(a.col_ready + pm, (int)(Nt - pm), a, k);
            }
        } else {
            ok = wait_flag(a.loaded + t, 1, a, k);
            const int32_t prev = a.prev_owner[t];
            if (ok && a.tile_codes && a.sto && a.sto[t] >= 0 && prev >= 0)  // codes staged aside: the slot must be free
                ok = wait_flag(a.ready + prev, a.epoch, a, k);
        }
        *s_flag = ok;
    }
    sync_workers();
    if (!*s_flag) return false;
    double* T = tile_ptr(a.pool, a.slot, Nt, nb, m, k);
    if (a.tile_codes && a.sto && a.sto[t] >= 0) {  // factor_tiles: decode the input codes into the fp64 slot
        const int pc = a.prec[t];
        const uint8_t* cp = a.shadow + a.sto[t];
        const double inv = 1.0 / __ldcg(a.in_scale + t);
        for (int64_t e = threadIdx.x; e < nb * nb; e += CC::NT) __stcg(T + e, decode_code(pc, cp, e, inv));
        sync_workers();
    }
    const int64_t rr = n - m * nb, cr = n - k * nb;  // real rows / columns of this tile
    if (a.gen_mode) {  // N2: generate the tile in place (fused generation, no input copy)
        for (int64_t e = threadIdx.x; e < nb * nb; e += CC::NT) {
            const int64_t r = e % nb, c = e / nb;
            double v;
            if (r < rr && c < cr) v = matern_entry(a, m * nb + r, k * nb + c);
            else v = (m == k && r == c) ? 1.0 : 0.0;
            __stcg(T + e, v);
        }
        sync_workers();
    } else if (a.src_A) {  // compact device path: the tile from the caller's matrix (lower part), padded
        for (int64_t e = threadIdx.x; e < nb * nb; e += CC::NT) {
            const int64_t r = e % nb, c = e / nb, gi = m * nb + r, gj = k * nb + c;
            double v;
            if (r < rr && c < cr) v = gi >= gj ? __ldcg(a.src_A + gi + gj * a.src_lda) : 0.0;
            else v = (m == k && r == c) ? 1.0 : 0.0;
            __stcg(T + e, v);
        }
        sync_workers();
    } else if (rr < nb || cr < nb) {
        for (int64_t e = threadIdx.x; e < nb * nb; e += CC::NT) {
            const int64_t r = e % nb, c = e / nb;
            if (r >= rr || c >= cr) __stcg(T + e, (m == k && r == c) ? 1.0 : 0.0);
        }
        sync_workers();
    }
    const int p = a.prec ? a.prec[t] : P_FP64;
    // (factor_tiles: a tile given as codes already IS the stored input -- re-quantizing it with a
    // scale recomputed from its amax would not be the identity when that amax rounded up into
    // the next binade, the up-cast reading of O4.2.3)
    if (p != P_FP64 && !(a.tile_codes && a.sto && a.sto[t] >= 0)) {
        double v = 0.0;
        for (int64_t e = threadIdx.x; e < nb * nb; e += CC::NT) v = fmax(v, fabs(__ldcg(T + e)));
        for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
        sync_workers();
        double amax = 0.0;
        for (int w = 0; w < (CC::NT >> 5); ++w) amax = fmax(amax, red[w]);
        const double sc = tile_scale(p, amax), isc = 1.0 / sc;
        for (int64_t e = threadIdx.x; e < nb * nb; e += CC::NT) __stcg(T + e, quantize_value(p, __ldcg(T + e), sc, isc));
    }
    __threadfence();
    sync_workers();
    if (threadIdx.x == 0) st_release(a.prep_done + t, 1);
    return true;
}

}  // namespace

namespace {
constexpr int PK = 128 * 129 / 2;  // packed lower-triangle length
__device__ __forceinline__ int pidx_c(int i, int j) { return j * 128 - j * (j - 1) / 2 + (i - j); }  // col-major
__device__ __forceinline__ int pidx_r(int i, int j) { return i * (i + 1) / 2 + j; }                  // row-major

template <class C>
__device__ void store_acc(double (&acc)[C::MI][C::NI][2], double* Ct, int64_t ld, bool subtract) {
#pragma unroll
    for (int mi = 0; mi < C::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < C::NI; ++ni)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                int r, c;
                frag_pos<C>(mi, ni, i, r, c);
                double* p = Ct + r + (int64_t)c * ld;
                __stcg(p, subtract ? __ldcg(p) - acc[mi][ni][i] : acc[mi][ni][i]);
            }
}
}  // namespace

// Factor the diagonal tile (the claim for column k is already held),
// left-looking over its 128-column blocks J: update block column J with the
// finished columns (one GEMM of K = 128 J per block), factor D_JJ unblocked,
// form W_J = L_JJ^-1, then D[I,J] = D[I,J] W_J^T for I > J.
// NT = 256: the dedicated kernel (W_J in shared memory, 128x128 DMMA blocks);
// NT = 128: the scheduler-CTA fallback (77 KB budget: W_J through global
// memory, 64x128 DMMA blocks in two row halves).  Returns false on a non-PD
// pivot (info set) -- the caller must not publish Ready.
template <int NT>
__device__ bool potrf_tile_body(const SchedArgs& a, int64_t k, double* smem, int* s_flag) {
    const int t = threadIdx.x;
    const int64_t Nt = a.Nt, nb = a.nb;
    const int S = (int)(nb / 128);
    double* D = tile_ptr(a.pool, a.slot, Nt, nb, k, k);
    double* Wk = a.wbuf + k * S * (128 * 128);
    // packed L_JJ (column-major lower); the fallback keeps the first 128
    // doubles free (scheduler scratch lives in that stage padding)
    double* P = smem + (NT == 256 ? 0 : 128);
    double* R = P + PK;      // packed W_J, row-major lower (NT = 256 only)
    using G = typename std::conditional<NT == 256, PC, CC>::type;
    uint64_t tp = (a.stats && t == 0) ? globaltimer() : 0;
    auto phase = [&](int slot) {  // diagnostics: time since the last mark into stats[slot]
        if (a.stats && t == 0) {
            const uint64_t now = globaltimer();
            atomicAdd(a.stats + slot, now - tp);
            tp = now;
        }
    };
    for (int J = 0; J < S; ++J) {
        double* DJJ = D + (int64_t)J * 128 * (1 + nb);
        // ---- left-looking update of block column J (one long-K GEMM per
        //      block instead of J short trailing updates):
        //      D[I,J] -= D[I,0:J] D[J,0:J]^T for I >= J
        if (J > 0) {
            for (int I = J; I < S; ++I)
                for (int h = 0; h < 128 / G::BM; ++h) {
                    double acc[G::MI][G::NI][2];
                    zero_acc<G>(acc);
                    const double* Ab = D + (int64_t)I * 128 + h * G::BM;
                    const double* Bb = D + (int64_t)J * 128;
                    auto src = [&](int it, const double*& pa, const double*& pb) {
                        pa = Ab + (int64_t)it * BK * nb;
                        pb = Bb + (int64_t)it * BK * nb;
                    };
                    gemm_mainloop<G>(acc, src, nb, nb, J * 128 / BK, smem);
                    store_acc<G>(acc, D + (int64_t)I * 128 + h * G::BM + (int64_t)J * 128 * nb, nb, true);
                    __threadfence_block();
                    sync_nt<NT>();
                }
        }
        phase(STAT_PF_UPD);
        double* W = Wk + J * (128 * 128);
        for (int idx = t; idx < 128 * 128; idx += NT) {
            int c = idx >> 7, r = idx & 127;
            if (r >= c) P[pidx_c(r, c)] = __ldcg(DJJ + r + (int64_t)c * nb);
        }
        if (t == 0) *s_flag = 0;
        sync_nt<NT>();
        // ---- unblocked left-looking (column) Cholesky of the packed block:
        //      thread i computes L[i,j] = (D[i,j] - sum_{q<j} L[i,q] L[j,q]) / L[j,j]
        //      (S:144 up to summation order); 2 barriers per column.
        //      pidx_c(x, q) = off(q) + x with off(q+1) = off(q) + 127 - q.
        for (int j = 0; j < 128; ++j) {
            double sv = 0.0;
            if (t >= j && t < 128) {
                double s0 = P[pidx_c(t, j)], s1 = 0.0, s2 = 0.0, s3 = 0.0;
                int off = 0, q = 0;
                for (; q + 3 < j; q += 4) {
                    const int o1 = off + 127 - q, o2 = o1 + 126 - q, o3 = o2 + 125 - q;
                    s0 -= P[off + t] * P[off + j];
                    s1 -= P[o1 + t] * P[o1 + j];
                    s2 -= P[o2 + t] * P[o2 + j];
                    s3 -= P[o3 + t] * P[o3 + j];
                    off = o3 + 124 - q;
                }
                for (; q < j; ++q) {
                    s0 -= P[off + t] * P[off + j];
                    off += 127 - q;
                }
                sv = (s0 + s1) + (s2 + s3);
            }
            if (t == j) {
                if (!(sv > 0.0)) {
                    *s_flag = 1;
                    const int64_t info = k * nb + (int64_t)J * 128 + j + 1;
                    *(volatile int64_t*)a.dinfo = info;
                    for (int q = 0; q < MAX_RANKS; ++q)  // other ranks stop at this column too
                        if (a.peer_dinfo[q]) *(volatile int64_t*)a.peer_dinfo[q] = info;
                    __threadfence_system();
                } else {
                    P[pidx_c(j, j)] = sqrt(sv);
                }
            }
            sync_nt<NT>();
            if (*s_flag) return false;
            if (t > j && t < 128) P[pidx_c(t, j)] = sv / P[pidx_c(j, j)];
            sync_nt<NT>();
        }
        phase(STAT_PF_CHOL);
        // ---- W = L^-1 row by row: W[r,c] = (delta_rc - sum_{q<r} L[r,q] W[q,c]) / L[r,r]
        //      (thread = column c, independent of the others; L[r,q] is a
        //      broadcast, W[q,c] consecutive in c).
        //      Dedicated kernel: W row-major packed in smem (R); fallback: row-major
        //      in the global W block, transposed in place afterwards.
        for (int r = 0; r < 128; ++r) {
            if (t <= r) {
                const int c = t;
                double s0 = (r == c) ? 1.0 : 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                int off = 0, q = 0;
                auto wqc = [&](int qq) -> double {
                    if (c > qq) return 0.0;
                    if (NT == 256) return R[pidx_r(qq, c)];
                    return __ldcg(W + qq * 128 + c);
                };
                for (; q + 3 < r; q += 4) {
                    const int o1 = off + 127 - q, o2 = o1 + 126 - q, o3 = o2 + 125 - q;
                    s0 -= P[off + r] * wqc(q);
                    s1 -= P[o1 + r] * wqc(q + 1);
                    s2 -= P[o2 + r] * wqc(q + 2);
                    s3 -= P[o3 + r] * wqc(q + 3);
                    off = o3 + 124 - q;
                }
                for (; q < r; ++q) {
                    s0 -= P[off + r] * wqc(q);
                    off += 127 - q;
                }
                const double v = ((s0 + s1) + (s2 + s3)) / P[pidx_c(r, r)];
                if (NT == 256) R[pidx_r(r, c)] = v;
                else __stcg(W + r * 128 + c, v);
            } else if (NT != 256 && t < 128) {
                __stcg(W + r * 128 + t, 0.0);  // strictly upper part of row r
            }
            // (no barrier: column c of W is read and written by thread c only)
        }
        sync_nt<NT>();
        if (NT != 256) {  // row-major -> column-major in place
            for (int idx = t; idx < 128 * 128; idx += NT) {
                const int r = idx >> 7, c = idx & 127;
                if (r < c) {
                    const double x = __ldcg(W + r * 128 + c), y = __ldcg(W + c * 128 + r);
                    __stcg(W + r * 128 + c, y);
                    __stcg(W + c * 128 + r, x);
                }
            }
            __threadfence_block();
        }
        sync_nt<NT>();
        // ---- write L_JJ (zero upper) [and W_J, col-major, zero upper]
        for (int idx = t; idx < 128 * 128; idx += NT) {
            int c = idx >> 7, r = idx & 127;
            __stcg(DJJ + r + (int64_t)c * nb, r >= c ? P[pidx_c(r, c)] : 0.0);
            if (NT == 256) __stcg(W + r + c * 128, r >= c ? R[pidx_r(r, c)] : 0.0);
        }
        __threadfence_block();
        sync_nt<NT>();
        phase(STAT_PF_INV);
        // ---- TRSM of the blocks below: D[I,J] = D[I,J] W^T (the mainloop
        //      consumes all of D[I,J] before the epilogue overwrites it)
        for (int I = J + 1; I < S; ++I)
            for (int h = 0; h < 128 / G::BM; ++h) {
                double acc[G::MI][G::NI][2];
                zero_acc<G>(acc);
                double* DIJ = D + (int64_t)I * 128 + h * G::BM + (int64_t)J * 128 * nb;
                auto src = [&](int it, const double*& pa, const double*& pb) {
                    pa = DIJ + (int64_t)it * BK * nb;
                    pb = W + it * BK * 128;
                };
                gemm_mainloop<G>(acc, src, nb, 128, 128 / BK, smem);
                store_acc<G>(acc, DIJ, nb, false);
                __threadfence_block();
                sync_nt<NT>();
            }
        phase(STAT_PF_TRSM);
    }
    return true;
}

// Thread 0: wait until tile (k,k) is fully updated, then try to take the
// claim for POTRF(k).  `grace_ns` > 0: give the dedicated kernel that long to
// take it first (the scheduler-CTA fallback).  Sets *s_flag = 1 iff claimed.
__device__ void claim_potrf(const SchedArgs& a, int64_t k, uint64_t grace_ns, int* s_flag) {
    const int64_t tk = tile_index(a.Nt, k, k);
    bool ok = !skip_column(a, k) && k % a.nranks == a.rank;  // only the owner of row k factors (k,k)
    if (ok) ok = wait_input(a, tk, k);
    if (ok && k > 0) ok = wait_flag(a.gemm_done + tk, a.gemm_expected[tk], a, k);
    if (ok && grace_ns) {
        uint64_t t0 = globaltimer();
        while (*(volatile int*)(a.potrf_claim + k) == 0 && globaltimer() - t0 < grace_ns) __nanosleep(1000);
    }
    *s_flag = ok && atomicCAS(a.potrf_claim + k, 0, 1) == 0;
}

template <int NT>
__device__ void publish_potrf(const SchedArgs& a, int64_t k, double* red) {
    // this tile's share of log|A| = 2 sum log L_ii: fixed-order tree
    // reduction over the real diagonal entries (deterministic)
    const int64_t nb = a.nb;
    const double* D = tile_ptr(a.pool, a.slot, a.Nt, nb, k, k);
    const int64_t real = a.n - k * nb < nb ? a.n - k * nb : nb;
    double v = 0.0;
    for (int64_t r = threadIdx.x; r < real; r += NT) v += log(__ldcg(D + r + r * nb));
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    sync_nt<NT>();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    sync_nt<NT>();
    if (threadIdx.x == 0) {
        double sum = 0.0;
        for (int w = 0; w < (NT >> 5); ++w) sum += red[w];
        a.logdet_parts[k] = sum;
    }
    __threadfence();
    sync_nt<NT>();
    if (threadIdx.x == 0) {
        st_release(a.ready + tile_index(a.Nt, k, k), a.epoch);
        atom_add_release(a.col_ready + k, 1);
        if (a.stats) a.stats[STAT_POTRF + 3 * k + 2] = globaltimer();
    }
}

// POTRF(k) in the task list: normally taken by the dedicated kernel; if it has
// not claimed it 200 us after the tile is ready (e.g. kernels serialized by a
// profiler, or the reserved SM busy) a scheduler CTA factors the tile itself.
__device__ __noinline__ void task_potrf_fallback(const SchedArgs& a, int64_t k, double* smem, int* s_flag) {
    if (threadIdx.x == 0) claim_potrf(a, k, 200000, s_flag);
    sync_workers();
    if (!*s_flag) return;
    if (potrf_tile_body<CC::NT>(a, k, smem, s_flag)) publish_potrf<CC::NT>(a, k, smem + CC::LDA_S + CC::BM);
}

// Ozaki mode: a non-GEMM task is listed for both kernels and run by whichever
// claims it first (POTRF has its own claim word, shared with k_potrf_tile).
__device__ __forceinline__ bool claim_task(const SchedArgs& a, const int4& it) {
    if (!a.oz_img || it.x == ITEM_GEMM || it.x == ITEM_POTRF) return true;
    const int64_t R = a.nb / 64, T = a.Nt * (a.Nt + 1) / 2, t = tile_index(a.Nt, it.y, it.z);
    int* c = it.x == ITEM_TRSM ? a.task_claim + t * R + it.w
           : it.x == ITEM_QUANT ? a.task_claim + T * R + t * R + it.w
                                : a.task_claim + 2 * T * R + t;
    return atomicCAS(c, 0, 1) == 0;
}

// ------------------------------------------------------ the static schedule
// The arguments live in global memory (copied once per factorization) so the
// out-of-line task functions can take them by reference without a local copy.
// MXP = false: FP64-only task list (DMMA GEMM + TRSM, fully inlined, no
// spills); MXP = true adds tcgen05 / cast / QUANT tasks, kept out of line.
// (FP64: arguments by value in the constant bank -- operands read straight
// from it keep register pressure at the no-spill level; MxP: through `ap`.)
template <bool MXP>
__global__ void __launch_bounds__(CC::NT, 3) k_sched(const SchedArgs a_param, const SchedArgs* __restrict__ ap) {
    const SchedArgs& a = MXP ? *ap : a_param;
    // this rank's SM partition [sm_lo, sm_hi) (all SMs unless ranks share a GPU);
    // its first `reserved_sms` SMs are left to the POTRF kernels
    const int id = (int)smid();
    if (id < a.sm_lo + a.reserved_sms || id >= a.sm_hi) return;
    extern __shared__ __align__(16) double smem[];
    // The task ticket and wait verdict live in the padding columns of the A
    // stage buffer (doubles BM..BM+PAD-1 of row 0 are never read or written by
    // the pipeline): any static __shared__ byte would push 3 x (76.8 KB + 1 KB
    // reserve) over the SM's 228 KB and drop occupancy from 3 CTAs/SM to 2.
    static_assert(PAD * 8 >= 2 * sizeof(int), "scratch must fit in the padding");
    int& s_idx = *reinterpret_cast<int*>(smem + CC::BM);
    int& s_flag = *(reinterpret_cast<int*>(smem + CC::BM) + 1);
    if (MXP && a.oz_img) {  // Ozaki mode: one k_sched CTA per SM (the k_tc CTA needs the rest of the SM)
        if (threadIdx.x == 0) s_idx = atomicAdd(a.sm_claim + (id & 255), 1);
        __syncthreads();
        if (s_idx > 0) return;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        atomicAdd(a.tdiag + 10, 1);
        atomicCAS(a.tdiag + 15, 0, (int)((globaltimer() >> 10) & 0x3FFFFFFF) | 1);
    }
    // tcgen05 state in the last 32 bytes (padding of the last B row of the DMMA
    // pipeline, never touched by it): two mbarriers + the TMEM base address.
    uint8_t* smem_b = reinterpret_cast<uint8_t*>(smem);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem_b + CC::SMEM_BYTES - 32);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_b + CC::SMEM_BYTES - 16);
    uint32_t tmem = 0;
    if (MXP && a.tc_engine && !a.oz_img) {  // MxP: this CTA owns 128 TMEM columns (3 CTAs x 128 <= 512 per SM)
        if (threadIdx.x < 32) tc::tmem_alloc(tmem_slot, tc::TMEM_COLS);
        tc::fence_before();
        __syncthreads();
        tc::fence_after();
        tmem = *tmem_slot;
        __syncthreads();
    }
    if (a.stats && threadIdx.x == 0) {
        atomicMin(a.stats + STAT_T0, globaltimer());
        atomicAdd(a.stats + STAT_CTAS, 1ull);
    }
    while (true) {
        if (threadIdx.x == 0) {
            int i = atomicAdd(a.counter, 1);
            // -1: list exhausted; -2: task of a failed column (skip)
            if (i >= a.nitems) i = -1;
            else if (skip_column(a, a.items[i].z)) i = -2;
            s_idx = i;
        }
        __syncthreads();
        const int idx = s_idx;
        __syncthreads();
        if (idx == -1) break;
        if (idx == -2) continue;
        const int4 it = a.items[idx];
        const int64_t m = it.y, k = it.z;
        if (MXP && a.oz_img) {  // Ozaki mode: k_tc may have run it already
            if (threadIdx.x == 0) s_flag = claim_task(*ap, it);
            __syncthreads();
            const bool mine = s_flag;
            __syncthreads();
            if (!mine) continue;
        }
        // out-of-line tasks take the global copy of the arguments (*ap): a
        // reference to the by-value kernel parameter would force a local copy
        if (it.x == ITEM_POTRF) {
            task_potrf_fallback(*ap, k, smem, &s_flag);
        } else if (it.x == ITEM_PREP) {
            // (scratch for the block reduction: the A-stage padding doubles of rows 1..4)
            task_prep(*ap, m, k, reinterpret_cast<double*>(smem) + CC::LDA_S + CC::BM, &s_flag);
        } else if constexpr (!MXP) {
            if (it.x == ITEM_GEMM) task_gemm<false>(a, m, k, it.w >> 16, it.w & 0xFFFF, smem, &s_flag);
            else task_trsm(a, m, k, it.w, smem, &s_flag);
        } else {
            if (it.x == ITEM_GEMM) {
                const int cp = a.prec[tile_index(a.Nt, m, k)];
                if (cp == P_FP64)
                    task_gemm<false>(a, m, k, it.w >> 16, it.w & 0xFFFF, smem, &s_flag);
                else if (!a.tc_engine)
                    task_gemm_cast(*ap, m, k, it.w >> 16, it.w & 0xFFFF, smem, &s_flag);
                else if (a.img && cp == P_FP32)
                    task_gemm_img<true, 2>(*ap, m, k, it.w >> 16, it.w & 0xFFFF, cp, smem_b, tmem, &s_flag);
                else if (a.img)
                    task_gemm_img<false, 2>(*ap, m, k, it.w >> 16, it.w & 0xFFFF, cp, smem_b, tmem, &s_flag);
                else if (cp == P_FP32)
                    task_gemm_tc<true>(*ap, m, k, it.w >> 16, it.w & 0xFFFF, cp, smem_b, mbar, tmem, &s_flag);
                else
                    task_gemm_tc<false>(*ap, m, k, it.w >> 16, it.w & 0xFFFF, cp, smem_b, mbar, tmem, &s_flag);
            } else if (it.x == ITEM_TRSM) {
                task_trsm_ool(*ap, m, k, it.w, smem, &s_flag);
            } else {
                task_quant(*ap, m, k, it.w, reinterpret_cast<double*>(smem) + 2048, &s_flag);
            }
        }
        __syncthreads();
    }
    if (MXP && a.tc_engine && !a.oz_img) {
        tc::fence_before();
        __syncthreads();
        if (threadIdx.x < 32) tc::tmem_dealloc(tmem, tc::TMEM_COLS);
    }
    if (threadIdx.x == 0) atomicAdd(a.tdiag + 11, 1);
    if (a.stats && threadIdx.x == 0) atomicMax(a.stats + STAT_TEND, globaltimer());
}

// ------------------------------------------- tensor-core GEMM kernel (Ozaki mode)
// MXP_ATTR_FP64_ENGINE = 1: every GEMM task of the schedule runs here -- FP64
// outputs on the int8 tensor cores (task_gemm_oz), outputs below FP64 on the
// tf32 operand-image engine -- one persistent CTA per SM owning all 512 TMEM
// columns, co-resident with one k_sched CTA per SM that takes the non-GEMM
// subsequence (TRSM / QUANT / PREP / POTRF fallback).  k_tc walks the WHOLE
// list in order and runs a non-GEMM task itself when k_sched has not claimed
// it yet: so k_tc alone is a complete static schedule (the ticket argument of
// k_sched holds for it), and k_sched only takes work off it -- a task claimed
// by k_sched depends on earlier tasks only, which k_tc or k_sched finish.
// (Profilers that serialize kernels run k_tc alone: still correct.)
// (5 warps at <= 168 registers: with one k_sched CTA (4 warps, 168 registers)
// beside it, SM sub-partition 0 holds k_tc's warps 0 and 4 and one k_sched warp,
// 3 x 168 x 32 <= 16K registers.  Warps 0-3 are the TMEM lanes 0-127; warp 4
// issues the native engine's copies and MMAs and otherwise joins the barriers.)
template <int NW>
__device__ __forceinline__ void k_tc_body(const SchedArgs* __restrict__ ap) {
    const SchedArgs& a = *ap;
    const int id = (int)smid();
    if (id < a.sm_lo + a.reserved_sms || id >= a.sm_hi) return;
    extern __shared__ __align__(1024) uint8_t smem_t[];
    __shared__ int s_idx, s_flag;
    __shared__ uint32_t tmem_slot;
    if (threadIdx.x == 0) {
        atomicAdd(a.tdiag + 16, 1);
        atomicCAS(a.tdiag + 17, 0, (int)((globaltimer() >> 10) & 0x3FFFFFFF) | 1);
    }
    if (threadIdx.x < 32) tc::tmem_alloc(&tmem_slot, oz::TMEM_COLS);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {  // (diagnostics: CTAs started / ended, first start in us)
        atomicAdd(a.tdiag + 8, 1);
        atomicCAS(a.tdiag + 14, 0, (int)((globaltimer() >> 10) & 0x3FFFFFFF) | 1);
    }
    if (a.stats && threadIdx.x == 0) atomicMin(a.stats + STAT_T0, globaltimer());
    while (true) {
        if (threadIdx.x == 0) {
            int i = atomicAdd(a.counter2, 1);
            if (i >= a.nitems2) i = -1;
            else if (skip_column(a, a.items2[i].z)) i = -2;
            s_idx = i;
        }
        __syncthreads();
        const int idx = s_idx;
        __syncthreads();
        if (idx == -1) break;
        if (idx == -2) continue;
        const int4 it = a.items2[idx];
        const int64_t m = it.y, k = it.z;
        double* smem_d = reinterpret_cast<double*>(smem_t);
        if (it.x == ITEM_GEMM) {
            const int cp = a.prec[tile_index(a.Nt, m, k)];
            if (threadIdx.x == 0) atomicAdd(a.tdiag + 12, 1);
            if (cp == P_FP64)
                task_gemm_oz<NW == 4>(a, m, k, it.w >> 16, it.w & 0xFFFF, smem_t, tmem, &s_flag);
            else if (cp == P_FP32 && a.native)
                { if constexpr (NW == 5) task_gemm_nat<nat::K_F32X2>(a, m, k, it.w >> 16, it.w & 0xFFFF, smem_t, tmem, &s_flag); else if (threadIdx.x == 0) atomicExch(a.err, 1); }
            else if (cp == P_FP32)
                task_gemm_img<true, 4>(a, m, k, it.w >> 16, it.w & 0xFFFF, cp, smem_t, tmem, &s_flag);
            else if (a.native && cp == P_FP16)
                { if constexpr (NW == 5) task_gemm_nat<nat::K_F16>(a, m, k, it.w >> 16, it.w & 0xFFFF, smem_t, tmem, &s_flag); else if (threadIdx.x == 0) atomicExch(a.err, 1); }
            else if (a.native)
                { if constexpr (NW == 5) task_gemm_nat<nat::K_F8>(a, m, k, it.w >> 16, it.w & 0xFFFF, smem_t, tmem, &s_flag); else if (threadIdx.x == 0) atomicExch(a.err, 1); }
            else
                task_gemm_img<false, 4>(a, m, k, it.w >> 16, it.w & 0xFFFF, cp, smem_t, tmem, &s_flag);
            if (threadIdx.x == 0) atomicAdd(a.tdiag + 13, 1);
        } else {
            if (threadIdx.x == 0) s_flag = claim_task(a, it);
            __syncthreads();
            const bool mine = s_flag;
            __syncthreads();
            if (mine && threadIdx.x < 128) {  // the 128 workers (named barrier 1); warp 4 waits below
                if (it.x == ITEM_POTRF) task_potrf_fallback(a, k, smem_d, &s_flag);
                else if (it.x == ITEM_PREP) task_prep(a, m, k, smem_d + CC::LDA_S + CC::BM, &s_flag);
                else if (it.x == ITEM_TRSM) task_trsm_ool(a, m, k, it.w, smem_d, &s_flag);
                else task_quant(a, m, k, it.w, smem_d + 2048, &s_flag);
            }
        }
        __syncthreads();
    }
    tc::fence_before();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(a.tdiag + 9, 1);
    if (threadIdx.x < 32) tc::tmem_dealloc(tmem, oz::TMEM_COLS);
    if (a.stats && threadIdx.x == 0) atomicMax(a.stats + STAT_TEND, globaltimer());
}
// the 4-warp variant (255 registers, register accumulators in the Ozaki
// engine) for maps without native-width tiles; the 5-warp variant for the rest
__global__ void __launch_bounds__(128, 1) k_tc4(const SchedArgs* __restrict__ ap) { k_tc_body<4>(ap); }
__global__ void __maxnreg__(168) k_tc5(const SchedArgs* __restrict__ ap) { k_tc_body<5>(ap); }

// ------------------------------------------------- POTRF of a diagonal tile
// One CTA (256 threads) on a reserved SM: waits until every GEMM/SYRK task of
// tile (k,k) is done, then factors it right-looking in 128 blocks:
//   L_JJ = chol(D_JJ) (packed in smem, kij order) and W_J = L_JJ^-1,
//   D[I,J] = D[I,J] W_J^T (I > J),  D[I,J'] -= D[I,J] D[J',J]^T (J < J' <= I).
// Writes L_kk in place, W_J to wbuf (for the TRSM tasks), sets Ready(k,k).
// The dedicated POTRF kernel: one CTA (256 threads) on a reserved SM.
__global__ void __launch_bounds__(256, 1) k_potrf_tile(SchedArgs a, int64_t k) {
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_flag;
    if (threadIdx.x == 0) {
        if (a.stats) a.stats[STAT_POTRF + 3 * k] = globaltimer();
        claim_potrf(a, k, 0, &s_flag);
        if (a.stats && s_flag) a.stats[STAT_POTRF + 3 * k + 1] = globaltimer();
    }
    __syncthreads();
    if (!s_flag) return;
    if (potrf_tile_body<256>(a, k, smem, &s_flag)) publish_potrf<256>(a, k, smem);
}

// ------------------------------------------------- generated-matrix planner
__global__ void k_matern_tile_norms(const double* __restrict__ xy, int64_t n, int64_t nb, int64_t Nt, double sigma2,
                                    double range_a, double nugget, double* norms) {
    __shared__ double red[256];
    const int64_t j = blockIdx.y, i = j + blockIdx.x;
    if (i >= Nt) return;
    double s = 0.0;
    for (int64_t c = j * nb; c < (j + 1) * nb && c < n; ++c)
        for (int64_t r = i * nb + threadIdx.x; r < (i + 1) * nb && r < n; r += blockDim.x) {
            const double dx = xy[2 * r] - xy[2 * c], dy = xy[2 * r + 1] - xy[2 * c + 1];
            double v = sigma2 * exp(-sqrt(dx * dx + dy * dy) / range_a);
            if (r == c) v += nugget;
            s += v * v;
        }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) norms[tile_index(Nt, i, j)] = sqrt(red[0]);
}
void launch_matern_tile_norms(const double* xy, int64_t n, int64_t nb, double sigma2, double range_a,
                              double nugget, double* norms, cudaStream_t s) {
    int64_t Nt = (n + nb - 1) / nb;
    dim3 grid((unsigned)Nt, (unsigned)Nt, 1);
    MXP_CARVEOUT_MAX(k_matern_tile_norms);
    k_matern_tile_norms<<<grid, 256, 0, s>>>(xy, n, nb, Nt, sigma2, range_a, nugget, norms);
}

// ------------------------------------------------------ input quantization
// (O3, G14): the accumulator of every task starts from A^ = deq(q_p(A)).
__global__ void k_tile_amax(const double* pool, const int32_t* slot, int64_t Nt, int64_t nb,
                            unsigned long long* amax_x, int rank, int nranks) {
    const int64_t j = blockIdx.y, i = j + blockIdx.x;
    if (i >= Nt || i % nranks != rank) return;
    const int64_t t = tile_index(Nt, i, j);
    const double* T = pool + (int64_t)slot[t] * nb * nb;
    double v = 0.0;
    for (int64_t e = (int64_t)blockIdx.z * blockDim.x + threadIdx.x; e < nb * nb; e += (int64_t)gridDim.z * blockDim.x)
        v = fmax(v, fabs(T[e]));
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) atomic_max_abs(amax_x + t, v);
}
__global__ void k_tile_quantize(double* pool, const int32_t* slot, const uint8_t* prec, int64_t Nt, int64_t nb,
                                const unsigned long long* amax_x, double* amax_s, int rank, int nranks) {
    const int64_t j = blockIdx.y, i = j + blockIdx.x;
    if (i >= Nt || i % nranks != rank) return;
    const int64_t t = tile_index(Nt, i, j);
    const int p = prec[t];
    const double amax = amax_of(amax_x + t);
    const double sc = tile_scale(p, amax);
    if (blockIdx.z == 0 && threadIdx.x == 0) amax_s[t] = quantize_value(p, amax, sc);
    if (p == P_FP64) return;
    double* T = pool + (int64_t)slot[t] * nb * nb;
    for (int64_t e = (int64_t)blockIdx.z * blockDim.x + threadIdx.x; e < nb * nb; e += (int64_t)gridDim.z * blockDim.x)
        T[e] = quantize_value(p, T[e], sc);
}
void launch_input_quantize(double* pool, const int32_t* slot, const uint8_t* prec, int64_t Nt, int64_t nb,
                           unsigned long long* amax_x, double* amax_s, cudaStream_t s, int rank, int nranks) {
    dim3 grid((unsigned)Nt, (unsigned)Nt, 8);
    MXP_CARVEOUT_MAX(k_tile_amax);
    k_tile_amax<<<grid, 256, 0, s>>>(pool, slot, Nt, nb, amax_x, rank, nranks);
    MXP_CARVEOUT_MAX(k_tile_quantize);
    k_tile_quantize<<<grid, 256, 0, s>>>(pool, slot, prec, Nt, nb, amax_x, amax_s, rank, nranks);
}

constexpr int POTRF_SMEM = (2 * PK * 8 > PC::SMEM_BYTES) ? 2 * PK * 8 : PC::SMEM_BYTES;
constexpr int TC_SMEM = oz::SMEM_BYTES > nat::SMEM_BYTES ? oz::SMEM_BYTES : nat::SMEM_BYTES;

void configure_sched() {
    static bool done = false;
    if (done) return;
    cudaFuncSetAttribute(k_sched<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM_BYTES);
    cudaFuncSetAttribute(k_sched<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, CC::SMEM_BYTES);
    cudaFuncSetAttribute(k_potrf_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, POTRF_SMEM);
    cudaFuncSetAttribute(k_tc4, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
    cudaFuncSetAttribute(k_tc5, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
    // every SM configured for the full 228 KB of shared memory: the Ozaki mode
    // co-schedules one k_tc CTA (~150 KB) and one k_sched CTA (~78 KB) per SM,
    // which a smaller carve-out picked for whichever kernel lands first would
    // forbid (the second kernel's CTAs would then wait for the first to exit)
    cudaFuncSetAttribute(k_tc4, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_tc5, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_sched<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_sched<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_potrf_tile, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    done = true;
}

int sched_ctas_per_sm() {
    int occ = 0;
    configure_sched();
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sched<false>, CC::NT, CC::SMEM_BYTES);
    return occ;
}

void launch_sched(const SchedArgs& a, const SchedArgs* a_dev, bool mxp, int grid, cudaStream_t s) {
    configure_sched();
    if (mxp) k_sched<true><<<grid, CC::NT, CC::SMEM_BYTES, s>>>(a, a_dev);
    else k_sched<false><<<grid, CC::NT, CC::SMEM_BYTES, s>>>(a, a_dev);
}

int tc_ctas_per_sm() {
    int occ = 0;
    configure_sched();
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tc5, 160, TC_SMEM);
    return occ;
}

void launch_tc(const SchedArgs* a_dev, int grid, cudaStream_t s, bool native) {
    configure_sched();
    if (native) k_tc5<<<grid, 160, TC_SMEM, s>>>(a_dev);
    else k_tc4<<<grid, 128, TC_SMEM, s>>>(a_dev);
}

void launch_potrf_tile(const SchedArgs& a, int64_t k, cudaStream_t s) {
    configure_sched();
    k_potrf_tile<<<1, 256, POTRF_SMEM, s>>>(a, k);
}


// Load every kernel of this file now (CUDA lazy loading would otherwise load a
// kernel at its first launch, which can wait for running kernels -- with ranks
// co-located on one GPU those spin on each other: a deadlock).
void preload_sched() {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, (const void*)k_sched<true>);
    cudaFuncGetAttributes(&fa, (const void*)k_sched<false>);
    cudaFuncGetAttributes(&fa, (const void*)k_tc4);
    cudaFuncGetAttributes(&fa, (const void*)k_tc5);
    cudaFuncGetAttributes(&fa, (const void*)k_potrf_tile);
    cudaFuncGetAttributes(&fa, (const void*)k_matern_tile_norms);
    cudaFuncGetAttributes(&fa, (const void*)k_tile_amax);
    cudaFuncGetAttributes(&fa, (const void*)k_tile_quantize);
    cudaGetLastError();
}

}  // namespace mxp
