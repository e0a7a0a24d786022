"""-m gpu parity of the FP64 tiles on the int8 tensor cores (Ozaki scheme I,
MXP_ATTR_FP64_ENGINE = 1) vs the CPU oracle.

The FP64 bar of BASELINE north_star applies unchanged: per-entry
|L_gpu - L_oracle| <= 1e-10 ||L||_max, backward error <= 1e-13; bitwise on the
integer-L0 inputs (small integers split exactly into slices and every product
and sum is exact); MxP maps within G15 and as close as the tf32 engine."""
import math

import numpy as np
import pytest

import oracle
import workloads as w
from gpu_util import gpu_factor

pytestmark = pytest.mark.gpu

OZ = {"fp64_engine": 1}


def _close(L, Lo, tol=1e-10):
    err = np.max(np.abs(L - Lo))
    assert err <= tol * np.max(np.abs(Lo)), err
    return err


def _check_used(plan):
    assert plan.get("fp64_engine_used") == 1


def test_ozaki_kms_closed_form():
    n, nb, rho = 1024, 256, 0.5
    A = w.kms(n, rho)
    L, info, ld, plan = gpu_factor(A, nb, attrs=OZ)
    _check_used(plan)
    assert info == 0
    Lo, _ = oracle.factor(A, nb)
    _close(L, Lo)
    closed = (n - 1) * math.log(1 - rho * rho)
    assert abs(ld - closed) <= 1e-12 * abs(closed)
    assert np.linalg.norm(A - L @ L.T) / np.linalg.norm(A) <= 1e-13


@pytest.mark.parametrize("n,nb", [(2048, 256), (1536, 512), (1100, 128), (3072, 1024), (2900, 256)])
def test_ozaki_plgsy_against_oracle(n, nb):
    A = w.plgsy(n, seed=42)
    L, info, ld, plan = gpu_factor(A, nb, attrs=OZ)
    _check_used(plan)
    assert info == 0
    Lo, _ = oracle.factor(A, nb)
    _close(L, Lo)
    assert abs(ld - oracle.logdet(Lo)) <= 1e-12 * abs(ld)
    assert np.linalg.norm(A - L @ L.T) / np.linalg.norm(A) <= 1e-13


@pytest.mark.parametrize("rho", [0.9, 0.99])
def test_ozaki_kms_ill_conditioned(rho):
    n, nb = 2048, 256
    A = w.kms(n, rho)
    L, info, ld, _ = gpu_factor(A, nb, attrs=OZ)
    Lo, _ = oracle.factor(A, nb)
    assert info == 0
    _close(L, Lo)
    assert np.linalg.norm(A - L @ L.T) / np.linalg.norm(A) <= 1e-13


def test_ozaki_matern_strong_correlation_fp64():
    xy = w.matern_locations(2048, seed=1)
    S = w.matern_cov(xy, 1.0, 0.210158)
    L, info, ld, _ = gpu_factor(S, 256, attrs=OZ)
    Lo, oinfo = oracle.factor(S, 256)
    assert info == oinfo == 0
    _close(L, Lo, 1e-9)  # the DMMA path's bar for this kappa ~ 1e5 input
    assert abs(ld - oracle.logdet(Lo)) <= 1e-9 * abs(ld)
    assert np.linalg.norm(S - L @ L.T) / np.linalg.norm(S) <= 1e-13


@pytest.mark.parametrize("n,nb", [(1024, 128), (1024, 256), (2048, 512), (1000, 256)])
def test_ozaki_integer_l0_bitwise(n, nb):
    L0 = w.integer_l0(n, seed=n + nb)
    A = w.spd_from_l0(L0)
    L, info, ld, _ = gpu_factor(A, nb, attrs=OZ)
    assert info == 0
    assert np.array_equal(L, L0)


@pytest.mark.parametrize("n,nb,j", [(1024, 256, 700), (1024, 128, 0), (1024, 256, 300)])
def test_ozaki_not_pd_info(n, nb, j):
    L0 = w.integer_l0(n, seed=5)
    A = w.spd_from_l0(L0)
    A[j, j] = -1.0 + np.sum(L0[j, :j] ** 2)
    L, info, ld, _ = gpu_factor(A, nb, attrs=OZ)
    _, oinfo = oracle.factor(A, nb)
    assert info == oinfo == j + 1
    kfail = j // nb
    assert np.array_equal(L[:, : kfail * nb], L0[:, : kfail * nb])


def test_ozaki_determinism_and_repeat():
    A = w.plgsy(2048, seed=3)
    L1, i1, ld1, plan = gpu_factor(A, 256, attrs=OZ)
    L2, i2, ld2, _ = gpu_factor(A, 256, plan=plan)
    assert i1 == i2 == 0
    assert np.array_equal(L1, L2) and ld1 == ld2
    L3, _, _, _ = gpu_factor(A, 256, attrs=dict(OZ, splitk_tiles=2))
    _close(L3, L1, 1e-13)


def test_ozaki_host_path_equals_device_path():
    A = w.plgsy(2048, seed=9)
    Ld, _, ldd, _ = gpu_factor(A, 256, attrs=OZ)
    Lh, info, ldh, plan = gpu_factor(A, 256, attrs=OZ, host=True)
    assert info == 0
    assert np.array_equal(Ld, Lh) and ldd == ldh


@pytest.mark.parametrize("s", [5, 6])
def test_ozaki_fewer_slices_accuracy(s):
    """s slices carry 8s-2 bits; the error scales accordingly (s=6: ~1e-12)."""
    A = w.plgsy(2048, seed=42)
    L, info, _, _ = gpu_factor(A, 256, attrs=dict(OZ, oz_slices=s))
    assert info == 0
    Lo, _ = oracle.factor(A, 256)
    err = np.max(np.abs(L - Lo)) / np.max(np.abs(Lo))
    assert err <= 2.0 ** (-8 * s + 12), err
    assert np.linalg.norm(A - L @ L.T) / np.linalg.norm(A) <= 2.0 ** (-8 * s + 10)


@pytest.mark.parametrize("tc", [1, 3])
@pytest.mark.parametrize("eps", [1e-5, 1e-8])
@pytest.mark.parametrize("n,nb", [(2048, 128), (1900, 256)])
def test_ozaki_mxp_matern_against_oracle(n, nb, eps, tc):
    """MxP map with the FP64 tiles on the int8 tensor cores and the others on
    the tf32 image engine (tc=1) or at native width (tc=3: fp16 codes on
    kind::f16, E4M3 codes on kind::f8f6f4, 3xTF32 for FP32), all in k_tc."""
    xy = w.matern_locations(n, seed=1)
    S = w.matern_cov(xy, 1.0, 0.02627)
    pmap = oracle.plan(S, nb, eps)
    assert np.any(pmap != oracle.FP64)
    L, info, ld, plan = gpu_factor(S, nb, pmap, attrs=dict(OZ, tc_engine=tc))
    _check_used(plan)
    assert plan.get("tc_engine_used") == tc
    Lo, oinfo = oracle.factor(S, nb, pmap)
    assert info == oinfo == 0
    err = np.max(np.abs(L - Lo))
    assert err <= 1e-4 * np.max(np.abs(Lo)), err  # the tf32 engine's bar (fp32 accumulation)
    Lt, _, ldt, _ = gpu_factor(S, nb, pmap, attrs={"tc_engine": 1})  # DMMA FP64 tiles, tf32 images
    # tc=1: the same tf32 arithmetic as the DMMA run; tc=3: FP32 tiles as fp16 h + l pairs
    # (22 bits, like 3xTF32) -- both within FP32-class rounding of each other and of the oracle
    assert abs(ld - ldt) <= (1e-9 if tc == 1 else 1e-7) * abs(ldt)
    ldo = oracle.logdet(Lo)
    assert abs(ld - ldo) <= 1e-6 * abs(ldo)


def test_ozaki_tc_kernel_alone_completes_the_schedule():
    """debug_sync=1 synchronizes after every launch, so k_tc runs before k_sched
    and the POTRF kernels exist (as under a profiler that serializes kernels):
    it must finish the whole static schedule by itself, with the same bits."""
    A = w.plgsy(2048, seed=8)
    L1, i1, ld1, _ = gpu_factor(A, 256, attrs=OZ)
    L2, i2, ld2, _ = gpu_factor(A, 256, attrs=dict(OZ, debug_sync=1))
    assert i1 == i2 == 0
    assert np.array_equal(L1, L2) and ld1 == ld2


# ---------------------------------------------------------------- out of core
def _oz_ooc_cap(n, nb, frac, s=7):
    """A cap of `frac` x the fp64 lower triangle (the Ozaki out-of-core mode needs
    the fp64 ring + the slice images of the live set under it)."""
    Nt = -(-n // nb)
    return int(frac * Nt * (Nt + 1) // 2 * nb * nb * 8)


@pytest.mark.parametrize("n,nb,frac", [(4096, 256, 0.9), (3000, 256, 0.97), (8192, 512, 0.9), (12288, 256, 0.62)])
def test_ozaki_out_of_core_bitwise_equals_in_core(n, nb, frac):
    """HBM cap below the lower triangle with the Ozaki engine: fp64 tiles live in a
    ring only while computed, final tiles as slice images whose slots are recycled
    when their row dies (DESIGN 5.4).  Same slices, same sums: the same bits as the
    in-core Ozaki run, each tile H2D once and D2H once."""
    import paper_2410_09819_b200 as m
    A = w.plgsy(n, seed=21)
    Lin, info, ld_in, pin = gpu_factor(A, nb, attrs=OZ, host=True)
    assert info == 0 and pin.get("fp64_engine_used") == 1
    Nt = -(-n // nb)
    T = Nt * (Nt + 1) // 2
    plan = m.Plan(n, nb)
    plan.set("fp64_engine", 1)
    plan.set("hbm_bytes_cap", _oz_ooc_cap(n, nb, frac))
    assert plan.get("fp64_engine_used") == 1
    assert 0 < plan.get("oz_image_slots") < T - Nt
    assert plan.get("pool_slots") < T
    Lo, info, ld_o, plan = gpu_factor(A, nb, host=True, plan=plan)
    assert info == 0
    assert np.array_equal(Lo, Lin)
    assert ld_o == ld_in
    assert plan.get("h2d_bytes") == 8 * sum(min(nb, n - i * nb) * min(nb, n - j * nb)
                                            for j in range(Nt) for i in range(j, Nt))
    Lor, _ = oracle.factor(A, nb)
    _close(Lo, Lor)


def test_ozaki_out_of_core_repeat_and_kms():
    """Repeat runs on one plan (Ready epochs, recycled slots) and the KMS closed form."""
    import paper_2410_09819_b200 as m
    n, nb, rho = 4096, 256, 0.9
    A = w.kms(n, rho)
    plan = m.Plan(n, nb)
    plan.set("fp64_engine", 1)
    plan.set("hbm_bytes_cap", _oz_ooc_cap(n, nb, 0.9))
    assert plan.get("oz_image_slots") > 0
    L1, i1, ld1, _ = gpu_factor(A, nb, host=True, plan=plan)
    L2, i2, ld2, _ = gpu_factor(A, nb, host=True, plan=plan)
    assert i1 == i2 == 0 and np.array_equal(L1, L2) and ld1 == ld2
    closed = (n - 1) * math.log(1 - rho * rho)
    assert abs(ld1 - closed) <= 1e-12 * abs(closed)
    assert np.linalg.norm(A - L1 @ L1.T) / np.linalg.norm(A) <= 1e-13


def test_ozaki_out_of_core_cap_below_live_set_falls_back():
    """A cap below ring + live slice images: the plan falls back to the DMMA
    out-of-core path (or refuses with MXP_ENOMEM below its live set)."""
    import paper_2410_09819_b200 as m
    n, nb = 4096, 256
    plan = m.Plan(n, nb)
    plan.set("fp64_engine", 1)
    plan.set("hbm_bytes_cap", _oz_ooc_cap(n, nb, 0.62))
    assert plan.get("fp64_engine_used") == 0 and plan.get("oz_image_slots") == 0
    A = w.plgsy(n, seed=5)
    L, info, _, _ = gpu_factor(A, nb, host=True, plan=plan)
    assert info == 0
    Lo, _ = oracle.factor(A, nb)
    _close(L, Lo)


@pytest.mark.parametrize("j", [0, 5000])
def test_ozaki_out_of_core_not_pd_does_not_hang(j):
    """A failed pivot out of core (Nt = 48): info is returned, no parked stream or
    image-slot wait hangs."""
    import torch

    import paper_2410_09819_b200 as m
    n, nb = 12288, 256
    Ad = torch.empty((n, n), dtype=torch.float64, device="cuda").T
    m.generate_plgsy_device(Ad, seed=3)
    Ad[j, j] = -1.0
    Ah = Ad.T.cpu().pin_memory()
    del Ad
    plan = m.Plan(n, nb)
    plan.set("fp64_engine", 1)
    plan.set("hbm_bytes_cap", _oz_ooc_cap(n, nb, 0.62))
    assert plan.get("oz_image_slots") > 0
    assert plan.factor(Ah.T) == j + 1


def test_ozaki_out_of_core_generated_matern_fp64():
    """Generated tiles (N2) out of core with the Ozaki engine: the log-determinant
    equals the in-core run's (the factor itself is not kept out of core)."""
    import torch

    import paper_2410_09819_b200 as m
    n, nb = 4096, 256
    xy = torch.tensor(w.matern_locations(n, seed=1), device="cuda")
    pin = m.Plan(n, nb)
    pin.set("fp64_engine", 1)
    assert pin.factor_matern(xy, 1.0, 0.078809) == 0
    pl = m.Plan(n, nb)
    pl.set("fp64_engine", 1)
    pl.set("hbm_bytes_cap", _oz_ooc_cap(n, nb, 0.9))
    assert pl.get("oz_image_slots") > 0
    assert pl.factor_matern(xy, 1.0, 0.078809) == 0
    assert pl.logdet() == pin.logdet()


def test_out_of_core_timeline():
    """mxp_chol_timeline (profile=1): per column, the loads complete in column order and
    before the column's write-backs; its POTRF completes before its last write-back."""
    import paper_2410_09819_b200 as m
    n, nb = 4096, 256
    A = w.plgsy(n, seed=8)
    for eng, frac in ((1, 0.9), (0, 0.62)):
        plan = m.Plan(n, nb)
        plan.set("fp64_engine", eng)
        plan.set("hbm_bytes_cap", _oz_ooc_cap(n, nb, frac))
        plan.set("profile", 1)
        L, info, _, _ = gpu_factor(A, nb, host=True, plan=plan)
        assert info == 0 and plan.get("fp64_engine_used") == eng
        tl = plan.timeline()
        Nt = n // nb
        assert len(tl["h2d"]) == len(tl["d2h"]) == len(tl["work"]) == Nt
        for k in range(Nt):
            assert 0 <= tl["h2d"][k] <= tl["d2h"][k] and 0 <= tl["work"][k] <= tl["d2h"][k] + 1e-3, (k, tl)
            assert k == 0 or tl["h2d"][k - 1] <= tl["h2d"][k] + 1e-3
