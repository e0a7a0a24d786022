"""-m gpu parity of the mixed-precision (MxP) path vs the CPU oracle.

Tolerance (BASELINE north_star, reading G15): normwise
max|L_gpu - L_oracle| <= 5e-3 * max|L_oracle|; bitwise on the exact banded
integer-L0 case and for the all-FP64 map; log-det close to the oracle's.
"""
import math

import numpy as np
import pytest

import oracle
import workloads as w
from gpu_util import gpu_factor

pytestmark = pytest.mark.gpu


def _matern(n, a=0.02627):
    xy = w.matern_locations(n, seed=1)
    return w.matern_cov(xy, 1.0, a)


@pytest.mark.parametrize("tc", [1, 2, 0])
@pytest.mark.parametrize("eps", [1e-5, 1e-8])
@pytest.mark.parametrize("n,nb", [(2048, 128), (4096, 256), (1900, 256)])
def test_mxp_matern_against_oracle(n, nb, eps, tc):
    """tc=1: tiles below FP64 on tcgen05 fed by per-tile operand images
    (3xTF32 / 1xTF32, fp32 accumulation); tc=2: tcgen05 with operands
    converted in registers; tc=0: the same casts on FP64 DMMA (fp64
    accumulation, like the oracle)."""
    S = _matern(n)
    pmap = oracle.plan(S, nb, eps)
    assert np.any(pmap != oracle.FP64)
    L, info, ld, _ = gpu_factor(S, nb, pmap, attrs={"tc_engine": tc})
    Lo, oinfo = oracle.factor(S, nb, pmap)
    assert info == oinfo == 0
    err = np.max(np.abs(L - Lo))
    assert err <= 5e-3 * np.max(np.abs(Lo)), err
    if tc == 0:  # same casts, fp64 accumulation: far inside the tolerance
        assert err <= 1e-6 * np.max(np.abs(Lo)), err
    else:        # fp32 accumulation of the non-FP64 tiles (G12)
        assert err <= 1e-4 * np.max(np.abs(Lo)), err
    assert abs(ld - oracle.logdet(Lo)) <= 1e-6 * abs(oracle.logdet(Lo))


def test_mxp_stored_values_are_quantized():
    """Every stored tile of L holds values of its precision: re-quantizing the
    GPU's tile with the oracle's quantizer is the identity (idempotence)."""
    n, nb = 2048, 256
    S = _matern(n)
    pmap = oracle.plan(S, nb, 1e-5)
    L, info, _, _ = gpu_factor(S, nb, pmap)
    assert info == 0
    Nt = n // nb
    seen = set()
    for j in range(Nt):
        for i in range(j + 1, Nt):
            p = int(pmap[oracle.tile_index(Nt, i, j)])
            T = np.ascontiguousarray(L[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb])
            q, _ = oracle.quantize_tile(p, T)
            assert np.array_equal(q, T), (i, j, p)
            seen.add(p)
    assert len(seen) >= 2


def test_all_fp64_map_is_the_fp64_path():
    A = w.plgsy(1536, seed=6)
    Nt = 6
    L1, _, _, _ = gpu_factor(A, 256)
    L2, _, _, _ = gpu_factor(A, 256, np.zeros(Nt * (Nt + 1) // 2, np.uint8))
    assert np.array_equal(L1, L2)


def test_banded_integer_l0_mxp_bitwise():
    """Bandwidth < nb: far tiles are zero -> planned FP8 (s = 1); near tiles hold
    small integers -> the MxP plumbing must return L0 bit for bit."""
    n, nb = 2048, 256
    L0 = w.integer_l0(n, seed=11, band=100)
    A = w.spd_from_l0(L0)
    pmap = oracle.plan(A, nb, 1e-3)
    assert np.sum(pmap == oracle.FP8) > 0
    L, info, _, _ = gpu_factor(A, nb, pmap)
    assert info == 0 and np.array_equal(L, L0)
    Lo, _ = oracle.factor(A, nb, pmap)
    assert np.array_equal(Lo, L0)


def test_mxp_loglik_close_to_fp64():
    """Not parity (no closed form for the MxP factor): the MxP log-likelihood at
    y = 0 stays near the FP64 one and tightens with eps."""
    n, nb = 4096, 256
    S = _matern(n)
    L64, _, ld64, _ = gpu_factor(S, nb)
    errs = []
    for eps in (1e-5, 1e-8):
        pmap = oracle.plan(S, nb, eps)
        _, info, ld, _ = gpu_factor(S, nb, pmap)
        assert info == 0
        l64 = -0.5 * n * math.log(2 * math.pi) - 0.5 * ld64
        lm = -0.5 * n * math.log(2 * math.pi) - 0.5 * ld
        errs.append(abs(lm - l64) / abs(l64))
    assert errs[1] <= errs[0] + 1e-12
    assert errs[1] <= 1e-6


def test_mxp_host_path_equals_device_path():
    """Host streaming (PREP tasks quantize the input in-kernel) and device path
    (input-quantization kernels) give the same bits."""
    n, nb = 2048, 256
    S = _matern(n)
    pmap = oracle.plan(S, nb, 1e-5)
    Ld, info_d, ld_d, _ = gpu_factor(S, nb, pmap)
    Lh, info_h, ld_h, _ = gpu_factor(S, nb, pmap, host=True)
    assert info_d == info_h == 0
    assert np.array_equal(Ld, Lh)
    assert ld_d == ld_h


@pytest.mark.parametrize("eps", [None, 1e-5, 1e-8])
def test_generated_matern_against_oracle(eps):
    """mxp_chol_factor_matern: tiles generated on the device inside the
    schedule (N2).  The oracle factors the host-built matrix of the same
    locations (device and host exp may differ in the last ulp)."""
    import paper_2410_09819_b200 as m
    n, nb = 2048, 256
    xy = w.matern_locations(n, seed=1)
    S = w.matern_cov(xy, 1.0, 0.02627)
    pmap = None
    if eps is not None:
        pmap, f = m.precision_map_matern_device(xy, nb, eps)
        mo = oracle.plan(S, nb, eps)
        assert np.mean(pmap == mo) >= 0.999
        fo = oracle.tile_norms(S, nb)
        assert np.max(np.abs(f - fo) / fo) <= 1e-12
    plan = m.Plan(n, nb, pmap)
    info = plan.factor_matern(xy, 1.0, 0.02627)
    assert info == 0
    L = np.tril(plan.get_factor().cpu().numpy())
    Lo, _ = oracle.factor(S, nb, pmap)
    tol = 1e-10 if eps is None else 1e-4
    assert np.max(np.abs(L - Lo)) <= tol * np.max(np.abs(Lo))
    assert abs(plan.logdet() - oracle.logdet(Lo)) <= 1e-8 * abs(oracle.logdet(Lo))


def test_generated_matern_out_of_core_logdet():
    import paper_2410_09819_b200 as m
    n, nb = 4096, 256
    xy = w.matern_locations(n, seed=1)
    p1 = m.Plan(n, nb)
    assert p1.factor_matern(xy, 1.0, 0.078809) == 0
    p2 = m.Plan(n, nb)
    p2.set("hbm_bytes_cap", 80 * nb * nb * 8)
    assert p2.factor_matern(xy, 1.0, 0.078809) == 0
    assert p2.logdet() == p1.logdet()
