"""CPU-side checks of the C ABI boundary: the library loads, exports every
symbol include/*.h declares, and validates arguments without touching a GPU."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mxp():
    import __graft_entry__
    __graft_entry__.build()
    import paper_2410_09819_b200 as m
    return m


def declared_symbols():
    syms = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        for m in re.finditer(r"^\s*(?:int|void|const char\s*\*)\s+(mxp_\w+)\s*\(", text, re.M):
            syms.add(m.group(1))
    return syms


def test_header_declares_boundary():
    syms = declared_symbols()
    for s in ("mxp_chol_plan", "mxp_chol_factor", "mxp_chol_factor_device", "mxp_chol_logdet",
              "mxp_precision_map_from_matrix_device", "mxp_chol_plan_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol(mxp):
    lib = mxp.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing
    assert set(mxp.binding.EXPORTS) == declared_symbols()
    assert mxp.abi_version() == 1


def test_library_is_sm100a(mxp):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {mxp.lib_path()}").read()
    assert "sm_100a" in out
    sass = os.popen(f"/usr/local/cuda/bin/cuobjdump -sass {mxp.lib_path()}").read()
    assert "DMMA.8x8x4" in sass  # FP64 tensor-pipe contraction in the chain kernels
    assert "LDGSTS" in sass     # cp.async operand staging
    assert "UTCIMMA" in sass    # int8 tcgen05 MMA (Ozaki FP64 engine)
    assert "UTCHMMA" in sass    # tf32 tcgen05 MMA (tiles below FP64)


def test_argument_validation_without_gpu(mxp):
    lib = mxp.lib()
    h = ctypes.c_void_p()
    assert lib.mxp_chol_plan(0, 256, None, 1, ctypes.byref(h)) == -1
    assert lib.mxp_chol_plan(1024, 100, None, 1, ctypes.byref(h)) == -2
    assert lib.mxp_chol_plan(1024, 256, None, 0, ctypes.byref(h)) == -4
    assert lib.mxp_chol_plan(1024, 256, None, 9, ctypes.byref(h)) == -4  # ngpus <= 8
    import torch
    g = ctypes.c_void_p()  # a group plan (ngpus > 1) needs a CUDA device to place its ranks
    rc = lib.mxp_chol_plan(1024, 256, None, 2, ctypes.byref(g))
    assert rc == (0 if torch.cuda.is_available() else -1001)
    if rc == 0:
        assert lib.mxp_chol_plan_set(g, 8, 1) == -1005  # MXP_ATTR_RANK: the group places its ranks
        lib.mxp_chol_plan_destroy(g)
    bad = (ctypes.c_uint8 * 10)(*([1] + [0] * 9))  # FP32 diagonal tile -> invalid map
    assert lib.mxp_chol_plan(1024, 256, bad, 1, ctypes.byref(h)) == -3
    assert lib.mxp_chol_plan(1024, 256, None, 1, ctypes.byref(h)) == 0
    v = ctypes.c_int64()
    assert lib.mxp_chol_plan_get(h, 104, ctypes.byref(v)) == 0 and v.value == 4
    assert lib.mxp_chol_plan_set(h, 999, 1) == -2
    assert lib.mxp_chol_plan_set(h, 3, 0) == -3
    sz = ctypes.c_size_t()
    assert lib.mxp_chol_workspace_size(h, ctypes.byref(sz)) == 0
    assert sz.value >= 10 * 256 * 256 * 8
    info = ctypes.c_int64()
    assert lib.mxp_chol_factor_device(h, None, 1024, ctypes.byref(info)) == -2
    assert lib.mxp_chol_factor_device(h, ctypes.c_void_p(16), 1000, ctypes.byref(info)) == -3
    d = ctypes.c_double()
    assert lib.mxp_chol_logdet(h, ctypes.byref(d)) == -1004  # MXP_ESTATE: nothing factored
    assert lib.mxp_strerror(-1004) == b"invalid plan state"
    lib.mxp_chol_plan_destroy(h)
    lib.mxp_chol_plan_destroy(None)


def test_product_package_does_not_touch_oracle():
    """The product path never imports / links the oracle."""
    pkg = os.path.join(ROOT, "paper_2410_09819_b200")
    for path in glob.glob(os.path.join(pkg, "**", "*.*"), recursive=True):
        if path.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
            text = open(path).read()
            assert "oracle" not in re.sub(r"#.*|//.*", "", text).lower().replace("oracle_", ""), path
