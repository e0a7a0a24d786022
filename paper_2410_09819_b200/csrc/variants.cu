// variants.cu -- host-to-device byte ledgers of the paper's out-of-core
// variants over the static left-looking schedule (PAPER.md
// P:202-206 sync/async, P:235-238 V1, Alg. 2, Alg. 3 V2,
// P:303 V3, P:456-508 data-movement volumes).
//
// The engine executes one policy: every tile crosses the host link once each
// way (static dead-tile slot plan, engine.cu), which needs the live set in
// HBM.  The paper's variants are cache policies over the same task sequence;
// this file replays that sequence (Alg. 2, tasks (m, k) column by column, one
// stream) against a tile cache of the given capacity and counts the transfers
// each policy issues -- the "data movement volume" the paper plots
// -- so the engine's ledger can be set beside them at the same n, nb and HBM
// size.  Tile units are converted to bytes at 8 nb^2 (FP64 tiles).
//
//   sync / async: no cache; every update kernel loads its
//       accumulator and operands and writes the accumulator back (sync: one
//       stream, the same volume at equal nb -- the paper's sync volume differs
//       only through its larger tuned tile)
//   V1: the accumulator stays resident for its whole task
//   V2 (Alg. 3): + a cache table: operands (and final tiles) stay
//       until the capacity is reached, then the least recently used one is
//       repurposed ("remove_steal")
//   V3: + the diagonal tile L_kk is not evicted before the last TRSM of
//       its column
//   static dead-tile (this engine): each tile loaded once, evicted only when
//       dead (needs the live set max_k (Nt-k) k + the column's tiles in HBM)
//   MIN (Belady): the optimal offline eviction for this access sequence --
//       known ahead because the schedule is static; a lower bound for
//       every policy with this task order
#include <cstdint>
#include <list>
#include <queue>
#include <unordered_map>
#include <vector>

#include "../../include/mxp_chol.h"

namespace {

enum { V_SYNC = 0, V_ASYNC = 1, V_V1 = 2, V_V2 = 3, V_V3 = 4, V_STATIC = 5, V_MIN = 6 };

inline int64_t tidx(int64_t Nt, int64_t m, int64_t k) { return k * Nt - k * (k - 1) / 2 + (m - k); }

// One access of the cached variants: tile t read by a task of stream `s`;
// kind 1 = the task's accumulator (its first access: in use until the task
// ends), `task_end` marks a task's last access.
struct Access {
    int32_t t;
    int8_t kind;  // 0 operand, 1 accumulator (task start), 2 diagonal for TRSM
    int8_t task_end;
    int16_t s;
};

// Alg. 2's tasks (m, k), column by column, dealt to `streams` streams in a 1-D
// cyclic manner ("assigned to threads in a 1D cyclic manner"); the
// streams advance in lockstep, one tile access each per round (the cache sees
// their interleaving; waits on Ready are not modelled).
std::vector<Access> access_sequence(int64_t Nt, int streams) {
    std::vector<std::vector<Access>> per(streams);
    int64_t task = 0;
    for (int64_t k = 0; k < Nt; ++k)
        for (int64_t m = k; m < Nt; ++m, ++task) {
            const int s = (int)(task % streams);
            auto& a = per[s];
            a.push_back({(int32_t)tidx(Nt, m, k), 1, 0, (int16_t)s});
            for (int64_t n = 0; n < k; ++n) {
                a.push_back({(int32_t)tidx(Nt, m, n), 0, 0, (int16_t)s});
                if (m != k) a.push_back({(int32_t)tidx(Nt, k, n), 0, 0, (int16_t)s});
            }
            if (m != k) a.push_back({(int32_t)tidx(Nt, k, k), 2, 0, (int16_t)s});
            a.back().task_end = 1;
        }
    std::vector<Access> out;
    size_t total = 0;
    for (auto& a : per) total += a.size();
    out.reserve(total);
    for (size_t i = 0; out.size() < total; ++i)
        for (int s = 0; s < streams; ++s)
            if (i < per[s].size()) out.push_back(per[s][i]);
    return out;
}

// LRU cache replay (V2; V3 pins L_kk until its column's last TRSM).  Returns
// loads, or -1 when the capacity cannot hold one task's working set.
int64_t replay_lru(int64_t Nt, int streams, int64_t cap, bool pin_diag, int64_t& peak) {
    const std::vector<Access> seq = access_sequence(Nt, streams);
    std::list<int32_t> lru;  // front = most recent
    std::unordered_map<int32_t, std::list<int32_t>::iterator> where;
    std::vector<int32_t> acc(streams, -1);  // accumulators in use (one per stream)
    std::vector<int32_t> prev(streams, -1); // each stream's previous operand (an update reads A and B together)
    std::vector<int64_t> trsm_left(Nt, 0);  // V3: TRSMs of column k still to run
    for (int64_t k = 0; k < Nt; ++k) trsm_left[k] = Nt - 1 - k;
    std::vector<int32_t> pinned;            // V3: diagonal tiles with TRSMs pending
    int64_t loads = 0;
    peak = 0;
    auto busy = [&](int32_t t) {
        for (int32_t a : acc) if (a == t) return true;
        for (int32_t a : prev) if (a == t) return true;
        for (int32_t d : pinned) if (d == t) return true;
        return false;
    };
    for (size_t i = 0; i < seq.size(); ++i) {
        const Access& x = seq[i];
        if (x.kind == 1) acc[x.s] = x.t;
        auto it = where.find(x.t);
        if (it != where.end()) {
            lru.splice(lru.begin(), lru, it->second);
        } else {
            ++loads;
            if ((int64_t)lru.size() >= cap) {  // remove_steal: least recently used, not in use now
                auto victim = lru.end();
                for (auto r = lru.rbegin(); r != lru.rend(); ++r)
                    if (*r != x.t && !busy(*r)) {
                        victim = std::next(r).base();
                        break;
                    }
                if (victim == lru.end()) return -1;
                where.erase(*victim);
                lru.erase(victim);
            }
            lru.push_front(x.t);
            where[x.t] = lru.begin();
        }
        peak = std::max<int64_t>(peak, (int64_t)lru.size());
        int64_t k = 0, r = x.t;  // tile coordinates (column k, row k + r)
        while (r >= Nt - k) r -= Nt - k, ++k;
        if (pin_diag && x.kind == 1 && r == 0 && trsm_left[k] > 0) pinned.push_back(x.t);  // POTRF(k) task
        if (x.kind == 2 && --trsm_left[k] == 0)  // last TRSM of column k: L_kk may go
            for (size_t q = 0; q < pinned.size(); ++q)
                if (pinned[q] == x.t) {
                    pinned.erase(pinned.begin() + (int64_t)q);
                    break;
                }
        prev[x.s] = x.task_end ? -1 : x.t;
        if (x.task_end) acc[x.s] = -1;
    }
    return loads;
}

// Belady MIN over the same sequence (evict the resident tile whose next use is
// farthest away; the current accumulator is in use until its task ends).
int64_t replay_min(int64_t Nt, int streams, int64_t cap, int64_t& peak) {
    const std::vector<Access> seq = access_sequence(Nt, streams);
    const size_t N = seq.size();
    const int64_t T = Nt * (Nt + 1) / 2;
    std::vector<int64_t> next(N), last(T, (int64_t)1 << 60);
    for (size_t i = N; i-- > 0;) {
        next[i] = last[seq[i].t];
        last[seq[i].t] = (int64_t)i;
    }
    std::vector<int64_t> nxt(T, -1);  // next use of each resident tile (-1: not resident)
    std::priority_queue<std::pair<int64_t, int32_t>> heap;  // (next use, tile), lazy deletion
    int64_t loads = 0, resident = 0;
    std::vector<int32_t> acc(streams, -1), prev(streams, -1);
    peak = 0;
    auto in_use = [&](int32_t t) {
        for (int32_t a : acc) if (a == t) return true;
        for (int32_t a : prev) if (a == t) return true;
        return false;
    };
    for (size_t i = 0; i < N; ++i) {
        const Access& x = seq[i];
        if (x.kind == 1) acc[x.s] = x.t;
        if (nxt[x.t] < 0) {
            ++loads;
            if (resident >= cap) {
                std::vector<std::pair<int64_t, int32_t>> keep;
                bool done = false;
                while (!heap.empty()) {
                    auto top = heap.top();
                    heap.pop();
                    if (nxt[top.second] != top.first) continue;  // stale
                    if (top.second == x.t || in_use(top.second)) {
                        keep.push_back(top);
                        continue;
                    }
                    nxt[top.second] = -1;
                    --resident;
                    done = true;
                    break;
                }
                for (auto& k : keep) heap.push(k);
                if (!done) return -1;
            }
            ++resident;
        }
        nxt[x.t] = next[i];
        heap.push({next[i], x.t});
        peak = std::max(peak, resident);
        prev[x.s] = x.task_end ? -1 : x.t;
        if (x.task_end) acc[x.s] = -1;
    }
    return loads;
}

}  // namespace

extern "C" int mxp_ooc_variant_volume(int64_t n, int64_t nb, int variant, int streams, int64_t hbm_bytes,
                                      int64_t* out) {
    if (n < 1) return -1;
    if (nb < 1) return -2;
    if (variant < V_SYNC || variant > V_MIN) return -3;
    if (streams < 1 || streams > 64) return -4;
    if (hbm_bytes < 0) return -5;
    if (!out) return -6;
    const int64_t Nt = (n + nb - 1) / nb, T = Nt * (Nt + 1) / 2, tile = 8 * nb * nb;
    const int64_t cap = hbm_bytes > 0 ? hbm_bytes / tile : T;
    int64_t loads = 0, stores = T, peak = 0;
    switch (variant) {
    case V_SYNC:
    case V_ASYNC:  // per update: accumulator in + operands in + accumulator out; POTRF / TRSM likewise
        loads = stores = 0;
        for (int64_t k = 0; k < Nt; ++k)
            for (int64_t m = k; m < Nt; ++m) {
                const bool diag = m == k;
                loads += k * (diag ? 2 : 3) + (diag ? 1 : 2);
                stores += k + 1;
            }
        peak = 4 * streams;
        break;
    case V_V1:  // accumulator in once, operands per update, L_kk per TRSM, result out once
        for (int64_t k = 0; k < Nt; ++k)
            for (int64_t m = k; m < Nt; ++m) loads += m == k ? 1 + k : 2 + 2 * k;
        peak = 4 * streams;
        break;
    case V_V2:
    case V_V3:
        loads = replay_lru(Nt, streams, cap, variant == V_V3, peak);
        if (loads < 0) return MXP_ENOMEM;
        break;
    case V_STATIC: {  // each tile once; the live set + one column must fit
        int64_t live = 0;
        for (int64_t k = 0; k < Nt; ++k) live = std::max(live, (Nt - k) * k + (Nt - k));
        if (live > cap) return MXP_ENOMEM;
        loads = T;
        peak = live;
        break;
    }
    case V_MIN:
        loads = replay_min(Nt, streams, cap, peak);
        if (loads < 0) return MXP_ENOMEM;
        break;
    }
    out[0] = loads * tile;
    out[1] = stores * tile;
    out[2] = loads;
    out[3] = peak;
    return MXP_OK;
}
