"""GPU parity on the hand-derived MxP rounding-point pins (tests/golden/mxp_rounding_points.json).

Each scalar case is embedded as tile (i,j) = A_ij * I_nb: every tile stays
diagonal and its amax is |A_ij|, so the GPU factor must be L_ij * I_nb bit for
bit -- the hand-derived values, not the oracle's output -- on every GEMM engine
of the tiles below FP64 and both FP64 engines.
"""
import numpy as np
import pytest

from gpu_util import gpu_factor
from mxp_pins import cases, embed, scalar_case

pytestmark = pytest.mark.gpu

ENGINES = {"dmma_cast": {"tc_engine": 0}, "tc_images": {"tc_engine": 1}, "tc_regs": {"tc_engine": 2},
           "ozaki_images": {"tc_engine": 1, "fp64_engine": 1},
           "ozaki_native": {"tc_engine": 3, "fp64_engine": 1}}


@pytest.mark.parametrize("case", cases(), ids=lambda c: c["name"])
@pytest.mark.parametrize("nb", [128, 256])
@pytest.mark.parametrize("engine", list(ENGINES))
def test_gpu_hand_derived_pins(case, nb, engine):
    A, Lexp, pmap = scalar_case(case)
    L, info, _, plan = gpu_factor(embed(A, nb), nb, pmap, attrs=ENGINES[engine])
    plan.close()
    assert info == 0
    assert np.array_equal(L, embed(Lexp, nb)), (case["name"], engine,
                                                np.max(np.abs(L - embed(Lexp, nb))))


@pytest.mark.parametrize("case", cases(), ids=lambda c: c["name"])
def test_gpu_hand_derived_pins_host_path(case):
    A, Lexp, pmap = scalar_case(case)
    L, info, _, plan = gpu_factor(embed(A, 128), 128, pmap, host=True)
    plan.close()
    assert info == 0
    assert np.array_equal(L, embed(Lexp, 128))
