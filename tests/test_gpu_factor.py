"""-m gpu parity tests: the CUDA path (through the C ABI) vs the CPU oracle on
the same seeded inputs.  Tolerances from BASELINE north_star:
FP64 per-entry |L_gpu - L_oracle| <= 1e-10 ||L||_max, backward error <= 1e-13,
bit-exact on the integer-L0 exact-recovery inputs."""
import math

import numpy as np
import pytest

import oracle
import workloads as w
from gpu_util import gpu_factor

pytestmark = pytest.mark.gpu


def _close(L, Lo, tol=1e-10):
    err = np.max(np.abs(L - Lo))
    assert err <= tol * np.max(np.abs(Lo)), err


def test_c1_kms_against_oracle_and_closed_form():
    n, nb, rho = 1024, 256, 0.5
    A = w.kms(n, rho)
    L, info, ld, plan = gpu_factor(A, nb)
    assert info == 0
    Lo, _ = oracle.factor(A, nb)
    _close(L, Lo)
    closed = (n - 1) * math.log(1 - rho * rho)
    assert abs(ld - closed) <= 1e-12 * abs(closed)
    be = np.linalg.norm(A - L @ L.T) / np.linalg.norm(A)
    assert be <= 1e-13
    assert plan.get("gpu_launches") > 0


@pytest.mark.parametrize("n,nb", [(1024, 128), (1024, 256), (2048, 512), (1280, 256), (1000, 256), (700, 128)])
def test_integer_l0_bitwise(n, nb):
    L0 = w.integer_l0(n, seed=n + nb)
    A = w.spd_from_l0(L0)
    L, info, ld, _ = gpu_factor(A, nb)
    assert info == 0
    assert np.array_equal(L, L0)


@pytest.mark.parametrize("n,nb", [(2048, 256), (1536, 512), (1100, 128), (3072, 1024)])
def test_plgsy_against_oracle(n, nb):
    A = w.plgsy(n, seed=42)
    L, info, ld, _ = gpu_factor(A, nb)
    assert info == 0
    Lo, _ = oracle.factor(A, nb)
    _close(L, Lo)
    assert abs(ld - oracle.logdet(Lo)) <= 1e-12 * abs(ld)
    be = np.linalg.norm(A - L @ L.T) / np.linalg.norm(A)
    assert be <= 1e-13


def test_matern_strong_correlation_fp64():
    xy = w.matern_locations(2048, seed=1)
    S = w.matern_cov(xy, 1.0, 0.210158)
    L, info, ld, _ = gpu_factor(S, 256)
    Lo, oinfo = oracle.factor(S, 256)
    assert info == oinfo == 0
    _close(L, Lo, 1e-9)
    assert abs(ld - oracle.logdet(Lo)) <= 1e-9 * abs(ld)


@pytest.mark.parametrize("n,nb,j", [(1024, 256, 700), (1024, 128, 0), (768, 256, 767), (1024, 256, 300)])
def test_not_pd_info(n, nb, j):
    L0 = w.integer_l0(n, seed=5)
    A = w.spd_from_l0(L0)
    A[j, j] = -1.0 + np.sum(L0[j, :j] ** 2)
    L, info, ld, _ = gpu_factor(A, nb)
    _, oinfo = oracle.factor(A, nb)
    assert info == oinfo == j + 1
    kfail = j // nb
    assert np.array_equal(L[:, : kfail * nb], L0[:, : kfail * nb])


def test_determinism_and_lookahead_invariance():
    A = w.plgsy(2048, seed=3)
    L1, _, _, _ = gpu_factor(A, 256)
    L2, _, _, _ = gpu_factor(A, 256)
    L3, _, _, _ = gpu_factor(A, 256, attrs={"lookahead": 0})
    assert np.array_equal(L1, L2)
    assert np.array_equal(L1, L3)


def test_splitk_chunks_within_tolerance():
    A = w.plgsy(4096, seed=5)
    L1, _, _, _ = gpu_factor(A, 128)
    L2, _, _, _ = gpu_factor(A, 128, attrs={"splitk_tiles": 1})
    _close(L1, L2, 1e-13)


def test_host_path_equals_device_path():
    A = w.plgsy(1536, seed=11)
    Ld, info_d, ld_d, _ = gpu_factor(A, 256)
    Lh, info_h, ld_h, plan = gpu_factor(A, 256, host=True)
    assert info_d == info_h == 0
    assert np.array_equal(Ld, Lh)
    assert ld_d == ld_h
    assert plan.get("h2d_bytes") > 0 and plan.get("d2h_bytes") > 0


def test_upper_triangle_untouched_and_lda():
    import torch

    import paper_2410_09819_b200 as m
    n, nb, lda = 1024, 256, 1100
    A = w.plgsy(n, seed=2)
    M = np.full((lda, n), 7.0)
    M[:n, :] = np.tril(A) + np.triu(np.full((n, n), 3.0), 1)
    Md = torch.tensor(np.ascontiguousarray(M.T), device="cuda")  # (n, lda) row-major == M column-major
    view = Md.T[:n, :]  # stride (1, lda)
    plan = m.Plan(n, nb)
    info = plan.factor_device(view)
    torch.cuda.synchronize()
    R = Md.T.cpu().numpy()
    assert info == 0
    assert np.all(np.triu(R[:n, :], 1) == np.triu(np.full((n, n), 3.0), 1))
    assert np.all(R[n:, :] == 7.0)
    Lo, _ = oracle.factor(A, nb)
    _close(np.tril(R[:n, :]), Lo)


def test_device_generators_match_host():
    import torch

    import paper_2410_09819_b200 as m
    n = 777
    Ad = torch.empty((n, n), dtype=torch.float64, device="cuda").T
    m.generate_plgsy_device(Ad, seed=42)
    torch.cuda.synchronize()
    assert np.array_equal(Ad.cpu().numpy(), w.plgsy(n, 42))
    m.generate_kms_device(Ad, 0.5)
    torch.cuda.synchronize()
    assert np.array_equal(Ad.cpu().numpy(), w.kms(n, 0.5))


def test_planner_device_matches_oracle():
    import torch

    import paper_2410_09819_b200 as m
    xy = w.matern_locations(2048, seed=1)
    S = w.matern_cov(xy, 1.0, 0.02627)
    Sd = torch.tensor(S, device="cuda").T
    for eps in (1e-5, 1e-8):
        mp, f = m.precision_map_from_matrix_device(Sd, 128, eps)
        fo = oracle.tile_norms(S, 128)
        assert np.max(np.abs(f - fo) / np.maximum(fo, 1e-300)) <= 1e-13
        mo = oracle.plan(S, 128, eps)
        # identical except where a norm sits within rounding of a threshold
        assert np.mean(mp == mo) >= 0.999


@pytest.mark.parametrize("n,nb", [(2048, 128), (1900, 256), (3000, 1024)])
def test_planner_host_matches_device_and_oracle(n, nb):
    """mxp_precision_map_from_matrix (host A streamed by tile-column panels) gives the device
    planner's norms bit for bit (same kernel arithmetic) and the oracle's within rounding."""
    import torch

    import paper_2410_09819_b200 as m
    xy = w.matern_locations(n, seed=1)
    S = w.matern_cov(xy, 1.0, 0.02627)
    M = np.tril(S) + np.triu(np.full((n, n), 5.0), 1)  # the strict upper triangle is not read ...
    Nt = -(-n // nb)
    for i in range(Nt):  # ... except inside diagonal tiles (mirrored there): keep it symmetric
        r = slice(i * nb, min(n, (i + 1) * nb))
        M[r, r] = S[r, r]
    Sd = torch.tensor(S, device="cuda").T
    for eps in (1e-5, 1e-8):
        mh, fh = m.precision_map_from_matrix(M, nb, eps)
        md, fd = m.precision_map_from_matrix_device(Sd, nb, eps)
        assert np.array_equal(fh, fd) and np.array_equal(mh, md)
        fo = oracle.tile_norms(S, nb)
        assert np.max(np.abs(fh - fo) / np.maximum(fo, 1e-300)) <= 1e-12  # (nb^2-term sums, other order)
        assert np.mean(mh == oracle.plan(S, nb, eps)) >= 0.999


@pytest.mark.parametrize("n,nb", [(1000, 256), (2048, 512), (1300, 128)])
def test_host_streaming_path_against_oracle(n, nb):
    """mxp_chol_factor: tiles stream H2D/D2H around the static schedule."""
    A = w.plgsy(n, seed=13)
    M = A + np.triu(np.full((n, n), 5.0), 1)  # distinctive strict upper triangle
    L, info, ld, plan = gpu_factor(M, nb, host=True)
    assert info == 0
    Lo, _ = oracle.factor(A, nb)
    _close(L, Lo)
    assert plan.get("h2d_bytes") == 8 * n * (n + nb) // 2 or plan.get("h2d_bytes") > 0


def test_host_path_upper_untouched_and_not_pd():
    import torch

    import paper_2410_09819_b200 as m
    n, nb = 1024, 256
    L0 = w.integer_l0(n, seed=5)
    A = w.spd_from_l0(L0)
    M = np.tril(A) + np.triu(np.full((n, n), 9.0), 1)
    Ah = torch.tensor(np.ascontiguousarray(M.T))  # row-major (n,n) == column-major M
    plan = m.Plan(n, nb)
    info = plan.factor(Ah.T)
    R = Ah.T.numpy()
    assert info == 0
    assert np.array_equal(np.tril(R), L0)
    assert np.all(R[np.triu_indices(n, 1)] == 9.0)
    # non-PD: the copy stream must not wait forever on Ready flags that never flip
    j = 600
    B = A.copy()
    B[j, j] = -1.0 + np.sum(L0[j, :j] ** 2)
    Bh = torch.tensor(np.ascontiguousarray(B.T))
    info = plan.factor(Bh.T)
    assert info == j + 1
    kfail = j // nb
    assert np.array_equal(np.tril(Bh.T.numpy())[:, : kfail * nb], L0[:, : kfail * nb])


@pytest.mark.parametrize("host", [False, True])
def test_potrf_fallback_inside_the_schedule(host):
    """debug_sync=3: no dedicated POTRF kernels; the scheduler CTAs claim and
    factor every diagonal tile themselves (the path a kernel-serializing
    profiler exercises).  Same parity bar."""
    A = w.kms(1024, 0.5)
    L, info, ld, _ = gpu_factor(A, 256, attrs={"debug_sync": 3}, host=host)
    assert info == 0
    Lo, _ = oracle.factor(A, 256)
    _close(L, Lo)
    L0 = w.integer_l0(1024, seed=3)
    L, info, _, _ = gpu_factor(w.spd_from_l0(L0), 256, attrs={"debug_sync": 3}, host=host)
    assert info == 0 and np.array_equal(L, L0)
    B = w.spd_from_l0(L0)
    B[700, 700] = -1.0 + np.sum(L0[700, :700] ** 2)
    _, info, _, _ = gpu_factor(B, 256, attrs={"debug_sync": 3}, host=host)
    assert info == 701


# (12288, 256): Nt = 48 -> ~3.5k parked stream ops per copy stream, more than a
# stream's command queue holds (the host feeders must not block each other)
@pytest.mark.parametrize("n,nb,frac", [(4096, 256, 0.6), (3000, 256, 0.65), (4096, 512, 0.7), (12288, 256, 0.62)])
def test_out_of_core_bitwise_equals_in_core(n, nb, frac):
    """HBM cap below the lower triangle: the streaming path recycles the slots
    of dead tiles (each tile H2D once, D2H once); same bits as in core."""
    import torch

    import paper_2410_09819_b200 as m
    A = w.plgsy(n, seed=21)
    Lin, info, ld_in, _ = gpu_factor(A, nb, host=True)
    assert info == 0
    Nt = -(-n // nb)
    T = Nt * (Nt + 1) // 2
    cap = int(frac * T) * nb * nb * 8
    plan = m.Plan(n, nb)
    plan.set("hbm_bytes_cap", cap)
    assert plan.get("pool_slots") < T
    Lo, info, ld_o, plan = gpu_factor(A, nb, host=True, plan=plan)
    assert info == 0
    assert np.array_equal(Lo, Lin)
    assert ld_o == ld_in
    assert plan.get("h2d_bytes") == 8 * sum(min(nb, n - i * nb) * min(nb, n - j * nb)
                                            for j in range(Nt) for i in range(j, Nt))


def test_out_of_core_cap_too_small():
    import paper_2410_09819_b200 as m
    n, nb = 4096, 256
    plan = m.Plan(n, nb)
    plan.set("hbm_bytes_cap", 20 * nb * nb * 8)  # 20 slots < the live set
    with pytest.raises(m.MxpError) as e:
        gpu_factor(w.plgsy(n, 1), nb, host=True, plan=plan)
    assert e.value.status == -1002
    Ad = __import__("torch").zeros((n, n), dtype=__import__("torch").float64, device="cuda").T
    with pytest.raises(m.MxpError):
        plan.factor_device(Ad)  # device-resident input needs every tile in the pool


def test_out_of_core_mxp():
    import paper_2410_09819_b200 as m
    n, nb = 4096, 256
    xy = w.matern_locations(n, seed=1)
    S = w.matern_cov(xy, 1.0, 0.02627)
    pmap = oracle.plan(S, nb, 1e-8)
    Lin, info, _, _ = gpu_factor(S, nb, pmap, host=True)
    plan = m.Plan(n, nb, pmap)
    plan.set("hbm_bytes_cap", 80 * nb * nb * 8)
    Lo, info2, _, _ = gpu_factor(S, nb, pmap, host=True, plan=plan)
    assert info == info2 == 0
    assert np.array_equal(Lo, Lin)


@pytest.mark.parametrize("j,cap_frac", [(0, 0.0), (5000, 0.0), (5000, 0.6)])
def test_host_path_not_pd_large_nt_does_not_hang(j, cap_frac):
    """with Nt = 48 the copy-stream queues fill up behind
    parked waits; a failed column must still release every parked stream (the
    failure watcher in factor_incore_f64), in core and out of core."""
    import torch

    import paper_2410_09819_b200 as m
    n, nb = 12288, 256
    Ad = torch.empty((n, n), dtype=torch.float64, device="cuda").T
    m.generate_plgsy_device(Ad, seed=3)
    Ad[j, j] = -1.0
    Ah = Ad.T.cpu().pin_memory()  # row-major (n,n) of a symmetric matrix == column-major A
    Ad[j, j] = float(n)
    Agood = Ad.T.cpu().pin_memory()
    del Ad
    plan = m.Plan(n, nb)
    if cap_frac:
        plan.set("hbm_bytes_cap", int(cap_frac * 8 * nb * nb * 48 * 49 // 2))
    info = plan.factor(Ah.T)
    assert info == j + 1
    # the plan is reusable afterwards: a good matrix factors
    assert plan.factor(Agood.T) == 0
    plan.close()
