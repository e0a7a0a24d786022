"""-m gpu: the compact pool (tiles below FP64 stored at their precision, P:42
"minimum acceptable bytes per word").

With the native engine the fp64 slot of a tile stored below FP64 is only an
accumulator: it is recycled once the tile is final, and the tile lives on as
its codes (4/2/1 B per element) + a power-of-two scale.  Every value is the
same as with a full fp64 pool (decoding is exact), so the compact runs must be
bitwise equal to the full-pool runs of the same engine, on every path (device,
host streaming, generated), for the factor, the log-det and the forward solve.
"""
import ctypes

import numpy as np
import pytest

import oracle
import workloads as w
from gpu_util import gpu_factor

pytestmark = pytest.mark.gpu

NAT = {"fp64_engine": 1, "tc_engine": 3}


def _matern(n, a=0.02627):
    xy = w.matern_locations(n, seed=1)
    return xy, w.matern_cov(xy, 1.0, a)


@pytest.mark.parametrize("eps", [1e-5, 1e-8])
@pytest.mark.parametrize("n,nb", [(4096, 256), (1900, 256), (3072, 1024)])
def test_compact_equals_full_pool_device_path(n, nb, eps):
    import torch
    xy, S = _matern(n)
    pmap = oracle.plan(S, nb, eps)
    Lc, ic, ldc, pc = gpu_factor(S, nb, pmap, attrs=NAT)
    Lf, if_, ldf, pf = gpu_factor(S, nb, pmap, attrs=dict(NAT, compact_pool=0))
    assert ic == if_ == 0
    assert pc.get("compact_used") == 1 and pf.get("compact_used") == 0
    assert pc.get("tc_engine_used") == 3 and pf.get("tc_engine_used") == 3
    assert np.array_equal(Lc, Lf) and ldc == ldf
    assert pc.get("pool_slots") < pf.get("pool_slots")
    if n // nb >= 8:  # (few tiles: the storage images outweigh the recycled slots)
        assert pc.workspace_size() < pf.workspace_size()
    # the resident factor decodes to the same values; the forward solve reads the codes
    assert np.array_equal(np.tril(pc.get_factor().cpu().numpy()), Lc)
    y = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    zc = torch.empty_like(y)
    zf = torch.empty_like(y)
    qc = pc.solve_lower(y, zc)
    qf = pf.solve_lower(y, zf)
    assert qc == qf and torch.equal(zc, zf)
    assert pc.loglik(y) == pf.loglik(y)
    # vs the oracle (G15 normwise, fp32-accumulation bar)
    Lo, _ = oracle.factor(S, nb, pmap)
    assert np.max(np.abs(Lc - Lo)) <= 1e-4 * np.max(np.abs(Lo))


def test_compact_tile_pointer_refused_for_coded_tiles():
    import paper_2410_09819_b200 as m
    n, nb = 2048, 256
    xy, S = _matern(n)
    pmap = oracle.plan(S, nb, 1e-5)
    L, info, _, plan = gpu_factor(S, nb, pmap, attrs=NAT)
    assert info == 0 and plan.get("compact_used") == 1
    Nt = n // nb
    ptr = ctypes.c_void_p()
    lib = m.lib()
    lib.mxp_chol_tile_device_ptr.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
    for i in range(Nt):
        for j in range(i + 1):
            rc = lib.mxp_chol_tile_device_ptr(plan._h, i, j, ctypes.byref(ptr))
            coded = i != j and pmap[oracle.tile_index(Nt, i, j)] != oracle.FP64
            assert rc == (-1004 if coded else 0), (i, j, rc)


@pytest.mark.parametrize("eps", [1e-5, 1e-8])
def test_compact_host_path(eps):
    """mxp_chol_factor (host streaming) with the compact ring: the H2D of a tile
    waits for the previous owner of its slot to be final and written back."""
    n, nb = 4096, 256
    xy, S = _matern(n)
    pmap = oracle.plan(S, nb, eps)
    Ld, _, ldd, _ = gpu_factor(S, nb, pmap, attrs=NAT)
    M = np.tril(S) + np.triu(np.full((n, n), 7.0), 1)
    Lh, info, ldh, plan = gpu_factor(M, nb, pmap, attrs=NAT, host=True)
    assert info == 0 and plan.get("compact_used") == 1
    assert np.array_equal(np.tril(Lh), Ld) and ldh == ldd


def test_compact_generated_path_and_loglik():
    import torch

    import paper_2410_09819_b200 as m
    n, nb = 4096, 256
    xy = w.matern_locations(n, seed=1)
    pmap, _ = m.precision_map_matern_device(xy, nb, 1e-6)
    out = {}
    y = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(9))
    for cp in (1, 0):
        pl = m.Plan(n, nb, pmap)
        for k, v in dict(NAT, compact_pool=cp).items():
            pl.set(k, v)
        assert pl.factor_matern(xy, 1.0, 0.02627) == 0
        assert pl.get("compact_used") == cp
        out[cp] = (pl.get_factor().cpu().numpy(), pl.logdet(), pl.loglik(y))
        pl.close()
    assert np.array_equal(out[1][0], out[0][0])
    assert out[1][1] == out[0][1] and out[1][2] == out[0][2]


def test_compact_not_pd():
    n, nb = 2048, 256
    xy, S = _matern(n, 0.078809)
    pmap = oracle.plan(S, nb, 1e-5)
    B = S.copy()
    B[1500, 1500] = -1.0
    L, info, _, plan = gpu_factor(B, nb, pmap, attrs=NAT)
    assert plan.get("compact_used") == 1
    _, oinfo = oracle.factor(B, nb, pmap)
    assert info == oinfo == 1501
