"""-m gpu: mxp_chol_factor_tiles -- tile-packed host storage at each tile's precision
(the C5 input; P:42 minimum bytes per word).  The codes of the stored
input (O3) go in; L's codes come out; host<->device bytes are one pass each way at
storage precision; the values equal the device path's bit for bit."""
import numpy as np
import pytest

import oracle
import workloads as w
from gpu_util import gpu_factor

pytestmark = pytest.mark.gpu

NAT = {"fp64_engine": 1, "tc_engine": 3}
DT = {0: np.float64, 1: np.float32, 2: np.float16, 3: np.uint8}
ESZ = {0: 8, 1: 4, 2: 2, 3: 1}


def e4m3_encode(v):
    """exactly representable E4M3 values -> OCP fn bytes (sign, 4-bit exponent bias 7, 3-bit mantissa)"""
    v = np.asarray(v, np.float64)
    out = np.zeros(v.shape, np.uint8)
    a = np.abs(v)
    nz = a > 0
    e = np.floor(np.log2(np.where(nz, a, 1.0)))
    sub = nz & (e < -6)
    norm = nz & ~sub
    mant_n = (a / 2.0 ** e - 1.0) * 8.0
    out[norm] = ((e[norm] + 7).astype(np.int64) << 3 | mant_n[norm].astype(np.int64)).astype(np.uint8)
    out[sub] = (a[sub] / 2.0 ** -9).astype(np.uint8)
    assert np.all(np.where(norm, mant_n, 0) == np.floor(np.where(norm, mant_n, 0)))
    out[v < 0] |= 0x80
    return out


def e4m3_decode(b):
    b = np.asarray(b, np.uint8)
    s = np.where(b & 0x80, -1.0, 1.0)
    ef = (b >> 3) & 0xF
    mf = (b & 7).astype(np.float64)
    return s * np.where(ef == 0, mf * 2.0 ** -9, (1.0 + mf / 8.0) * 2.0 ** (ef.astype(np.float64) - 7))


def pack(A, nb, pmap):
    n = A.shape[0]
    Nt = n // nb
    tiles, scales = [], np.ones(Nt * (Nt + 1) // 2)
    for j in range(Nt):
        for i in range(j, Nt):
            t = oracle.tile_index(Nt, i, j)
            p = int(pmap[t]) if i != j else 0
            T = np.asfortranarray(A[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb])
            if p == 0:
                tiles.append(np.ascontiguousarray(T.T.ravel()))  # column-major bytes
                continue
            q, s = oracle.quantize_tile(p, T.T.ravel())        # column-major element order
            code = q * s
            if p == 3:
                tiles.append(e4m3_encode(code))
            else:
                tiles.append(code.astype(DT[p]))
                assert np.array_equal(tiles[-1].astype(np.float64), code)
            scales[t] = s if p >= 2 else 1.0
    return tiles, scales


def unpack(tiles, scales, n, nb, pmap):
    Nt = n // nb
    L = np.zeros((n, n))
    for j in range(Nt):
        for i in range(j, Nt):
            t = oracle.tile_index(Nt, i, j)
            p = int(pmap[t]) if i != j else 0
            c = e4m3_decode(tiles[t]) if p == 3 else tiles[t].astype(np.float64)
            L[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb] = (c / scales[t]).reshape(nb, nb).T
    return np.tril(L)


@pytest.mark.parametrize("eps", [1e-5, 1e-8])
def test_factor_tiles_mxp_equals_device_path(eps):
    import paper_2410_09819_b200 as m
    n, nb = 4096, 256
    xy = w.matern_locations(n, seed=1)
    S = w.matern_cov(xy, 1.0, 0.02627)
    pmap = oracle.plan(S, nb, eps)
    Ld, info, ld, _ = gpu_factor(S, nb, pmap, attrs=NAT)
    assert info == 0
    tiles, scales = pack(S, nb, pmap)
    plan = m.Plan(n, nb, pmap)
    for k, v in NAT.items():
        plan.set(k, v)
    assert plan.get("compact_used") == 1
    assert plan.factor_tiles(tiles, scales) == 0
    Lt = unpack(tiles, scales, n, nb, pmap)
    assert np.array_equal(Lt, Ld) and plan.logdet() == ld
    Nt = n // nb
    want = sum(nb * nb * ESZ[int(pmap[oracle.tile_index(Nt, i, j)]) if i != j else 0]
               for j in range(Nt) for i in range(j, Nt))
    assert plan.get("h2d_bytes") == want and plan.get("d2h_bytes") == want
    # the scales returned are the oracle quantizer's (powers of two)
    for t in range(len(scales)):
        assert scales[t] > 0 and np.log2(scales[t]) == np.round(np.log2(scales[t]))


@pytest.mark.parametrize("cap", [0, 0.8])
def test_factor_tiles_fp64_any_engine_and_out_of_core(cap):
    import paper_2410_09819_b200 as m
    n, nb = 2048, 256
    A = w.plgsy(n, seed=12)
    Ld, info, ld, _ = gpu_factor(A, nb)
    Nt = n // nb
    tiles, scales = pack(A, nb, np.zeros(Nt * (Nt + 1) // 2, np.uint8))
    plan = m.Plan(n, nb)
    if cap:
        plan.set("hbm_bytes_cap", int(cap * 8 * nb * nb * Nt * (Nt + 1) // 2))
    assert plan.factor_tiles(tiles, scales) == 0
    Lt = unpack(tiles, scales, n, nb, np.zeros(Nt * (Nt + 1) // 2, np.uint8))
    assert np.array_equal(Lt, Ld) and plan.logdet() == ld
