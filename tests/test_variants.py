"""Host-link ledgers of the paper's out-of-core variants (mxp_ooc_variant_volume;
SURVEY §8(f) N3, Alg. 3).
CPU only: closed forms for the cache-less variants, an independent Python replay of
Alg. 2's access sequence for LRU (V2) and Belady MIN on small problems, and the
paper's volume ordering V3 <= V2 < V1 < async."""
import pytest

import paper_2410_09819_b200 as m


def _tiles(Nt):
    return Nt * (Nt + 1) // 2


def _vol(n, nb, v, frac=0.0, streams=1):
    Nt = -(-n // nb)
    cap = int(frac * _tiles(Nt) * 8 * nb * nb) if frac else 0
    return m.ooc_variant_volume(n, nb, v, cap, streams)


@pytest.mark.parametrize("Nt", [1, 2, 5, 16])
def test_cacheless_closed_forms(Nt):
    nb = 128
    n = Nt * nb
    tb = 8 * nb * nb
    # async: per update the accumulator and its operands in, the accumulator out; POTRF (in, out)
    # and TRSM (accumulator + L_kk in, out) likewise
    a_in = sum((2 * k + 1) + (Nt - k - 1) * (3 * k + 2) for k in range(Nt))
    a_out = sum((Nt - k) * (k + 1) for k in range(Nt))
    r = _vol(n, nb, "async")
    assert r["h2d_bytes"] == a_in * tb and r["d2h_bytes"] == a_out * tb
    assert _vol(n, nb, "sync") == r
    # V1: the accumulator in once per task, operands per update, L_kk per TRSM, result out once
    v1_in = sum((1 + k) + (Nt - k - 1) * (2 + 2 * k) for k in range(Nt))
    r = _vol(n, nb, "V1")
    assert r["h2d_bytes"] == v1_in * tb and r["d2h_bytes"] == _tiles(Nt) * tb


def test_unlimited_memory_every_tile_once():
    n, nb = 32 * 256, 256
    T = _tiles(32)
    for v in ("V2", "V3", "static", "MIN"):
        r = _vol(n, nb, v)
        assert r["loads"] == T and r["d2h_bytes"] == T * 8 * nb * nb


def _alg2_accesses(Nt, streams):
    """Alg. 2 written out: per task (m, k) the accumulator, then per n the
    operands L(m,n) [and L(k,n)], then L_kk for the TRSM; tasks dealt cyclically to
    streams that advance one access per round."""
    idx = {}
    for k in range(Nt):
        for mm in range(k, Nt):
            idx[(mm, k)] = len(idx)
    per = [[] for _ in range(streams)]
    task = 0
    for k in range(Nt):
        for mm in range(k, Nt):
            s = task % streams
            task += 1
            acc = idx[(mm, k)]
            seq = [(acc, acc)]
            for nn in range(k):
                seq.append((idx[(mm, nn)], acc))
                if mm != k:
                    seq.append((idx[(k, nn)], acc))
            if mm != k:
                seq.append((idx[(k, k)], acc))
            per[s] += [(t, a, s, i == len(seq) - 1) for i, (t, a) in enumerate(seq)]
    out = []
    for i in range(max(len(p) for p in per)):
        for s in range(streams):
            if i < len(per[s]):
                out.append(per[s][i])
    return out


def _py_lru(Nt, cap, streams):
    seq = _alg2_accesses(Nt, streams)
    cache = []  # most recent last
    acc = [None] * streams
    prev = [None] * streams  # an update holds its two operands together
    loads = 0
    for t, a, s, end in seq:
        acc[s] = a
        if t in cache:
            cache.remove(t)
        else:
            loads += 1
            if len(cache) >= cap:
                victim = next(x for x in cache if x not in acc and x not in prev and x != t)
                cache.remove(victim)
        cache.append(t)
        prev[s] = None if end else t
        if end:
            acc[s] = None
    return loads


def _py_min(Nt, cap, streams):
    seq = _alg2_accesses(Nt, streams)
    acc = [None] * streams
    prev = [None] * streams
    res = set()
    loads = 0
    for i, (t, a, s, end) in enumerate(seq):
        acc[s] = a
        if t not in res:
            loads += 1
            if len(res) >= cap:
                def nxt(x):
                    for j in range(i + 1, len(seq)):
                        if seq[j][0] == x:
                            return j
                    return 1 << 60
                cand = [x for x in res if x not in acc and x not in prev]
                res.remove(max(cand, key=lambda x: (nxt(x), x)))
            res.add(t)
        prev[s] = None if end else t
        if end:
            acc[s] = None
    return loads


@pytest.mark.parametrize("cap,streams", [(3, 1), (4, 1), (6, 1), (9, 1), (14, 1), (6, 2), (9, 2), (14, 2), (9, 3)])
def test_lru_and_min_match_independent_replay(cap, streams):
    Nt, nb = 6, 128
    tb = 8 * nb * nb
    r2 = m.ooc_variant_volume(Nt * nb, nb, "V2", cap * tb, streams)
    rmin = m.ooc_variant_volume(Nt * nb, nb, "MIN", cap * tb, streams)
    assert r2["loads"] == _py_lru(Nt, cap, streams)
    assert rmin["loads"] == _py_min(Nt, cap, streams)


@pytest.mark.parametrize("frac", [0.65, 0.35, 0.2])
def test_paper_volume_ordering(frac):
    """V3 <= V2 < V1 < async; MIN bounds every cache policy from below; the
    engine's static dead-tile plan moves each tile once when the live set fits."""
    n, nb = 48 * 512, 512
    v = {k: _vol(n, nb, k, frac, streams=4) for k in ("async", "V1", "V2", "V3", "static", "MIN")}
    h = {k: (x["h2d_bytes"] if x else None) for k, x in v.items()}
    assert h["MIN"] <= h["V3"] <= h["V2"] < h["V1"] < h["async"]
    if h["static"] is not None:
        assert h["static"] == h["MIN"] == v["static"]["loads"] * 8 * nb * nb
        assert v["static"]["loads"] == _tiles(48)
    else:
        assert h["MIN"] > _tiles(48) * 8 * nb * nb  # below the live set every policy re-fetches


def test_lru_and_min_monotone_in_memory():
    n, nb = 24 * 256, 256
    prev2 = prevm = None
    for frac in (0.15, 0.25, 0.35, 0.5, 0.7):
        r2, rm = _vol(n, nb, "V2", frac), _vol(n, nb, "MIN", frac)
        if prev2 is not None:
            assert r2["loads"] <= prev2 and rm["loads"] <= prevm
        prev2, prevm = r2["loads"], rm["loads"]


def test_capacity_below_working_set():
    assert m.ooc_variant_volume(4096, 256, "V2", 2 * 8 * 256 * 256) is None
    assert m.ooc_variant_volume(4096, 256, "static", 20 * 8 * 256 * 256) is None
