"""-m gpu parity of the forward solve L z = y and the Eq. 1 log-likelihood
(Eq. 1) on the resident factor vs the CPU
oracle (oracle.forward_solve / oracle.loglik on the oracle's own factor).

Bars: FP64 maps -- z within 1e-10 relative (the factor itself matches the
oracle to 1e-10 ||L||_max), log-likelihood within 1e-12 relative; MxP maps --
vs the oracle's MxP factor within the G15 regime, and the log-likelihood
error vs FP64 shrinking with eps (G16: <= 1e-6 relative at eps = 1e-8)."""
import numpy as np
import pytest

import oracle
import workloads as w
from gpu_util import gpu_factor

pytestmark = pytest.mark.gpu


def _y(n, seed=11):
    return np.random.default_rng(seed).standard_normal(n)


@pytest.mark.parametrize("n,nb", [(2048, 256), (1900, 256), (3072, 1024), (1100, 128)])
def test_forward_solve_and_loglik_fp64(n, nb):
    import torch
    xy = w.matern_locations(n, seed=1)
    S = w.matern_cov(xy, 1.0, 0.078809)
    L, info, ld, plan = gpu_factor(S, nb)
    assert info == 0
    Lo, _ = oracle.factor(S, nb)
    y = _y(n)
    yd = torch.tensor(y, device="cuda")
    zd = torch.empty_like(yd)
    q = plan.solve_lower(yd, zd)
    zo = oracle.forward_solve(Lo, y)
    z = zd.cpu().numpy()
    assert np.max(np.abs(z - zo)) <= 1e-10 * np.max(np.abs(zo))
    assert abs(q - float(zo @ zo)) <= 1e-10 * float(zo @ zo)
    ll = plan.loglik(yd)
    llo = oracle.loglik(Lo, y)
    assert abs(ll - llo) <= 1e-12 * abs(llo)
    assert abs(plan.loglik() - oracle.loglik(Lo)) <= 1e-12 * abs(llo)  # y = 0
    # bitwise reproducible
    z2 = torch.empty_like(yd)
    plan.solve_lower(yd, z2)
    assert torch.equal(zd, z2)


def test_forward_solve_identity_and_scaled():
    """Closed forms: A = I -> z = y; A = 4 I -> z = y / 2, ||z||^2 = ||y||^2 / 4."""
    import torch
    n, nb = 1024, 256
    y = _y(n, 3)
    yd = torch.tensor(y, device="cuda")
    for c, f in ((1.0, 1.0), (4.0, 0.5)):
        A = c * np.eye(n)
        _, info, _, plan = gpu_factor(A, nb)
        assert info == 0
        zd = torch.empty_like(yd)
        q = plan.solve_lower(yd, zd)
        assert np.array_equal(zd.cpu().numpy(), y * f)
        assert abs(q - float(y @ y) * f * f) <= 1e-13 * float(y @ y)


@pytest.mark.parametrize("eps", [1e-5, 1e-8])
def test_loglik_mxp_against_oracle(eps):
    import torch
    n, nb = 2048, 128
    xy = w.matern_locations(n, seed=1)
    S = w.matern_cov(xy, 1.0, 0.02627)
    pmap = oracle.plan(S, nb, eps)
    L, info, _, plan = gpu_factor(S, nb, pmap)
    assert info == 0
    Lo, _ = oracle.factor(S, nb, pmap)
    y = _y(n, 5)
    yd = torch.tensor(y, device="cuda")
    ll = plan.loglik(yd)
    llo = oracle.loglik(Lo, y)
    assert abs(ll - llo) <= 1e-6 * abs(llo)
    L64, _ = oracle.factor(S, nb)
    ll64 = oracle.loglik(L64, y)
    if eps <= 1e-8:
        assert abs(ll - ll64) <= 1e-6 * abs(ll64)  # G16


def test_solve_needs_a_result():
    import torch
    import paper_2410_09819_b200 as m
    plan = m.Plan(1024, 256)
    with pytest.raises(m.MxpError):
        plan.solve_lower(torch.zeros(1024, dtype=torch.float64, device="cuda"))
