"""ctypes marshalling for libmxpchol.so (include/mxp_chol.h).  No arithmetic."""
from __future__ import annotations

import ctypes
import os
import threading

FP64, FP32, FP16, FP8 = 0, 1, 2, 3

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libmxpchol.so")
_lib = None
_lock = threading.Lock()

ATTR = {
    "device": 0, "stream": 1, "hbm_bytes_cap": 2, "splitk_tiles": 3, "lookahead": 4,
    "debug_sync": 5, "profile": 6, "tc_engine": 7, "rank": 8, "nranks": 9, "sm_first": 10,
    "sm_count": 11, "fp64_engine": 12, "oz_slices": 13, "oz_prefetch": 15, "gpu_launches": 100, "h2d_bytes": 101, "d2h_bytes": 102,
    "pool_slots": 103, "nt": 104, "image_bytes": 105, "fp64_engine_used": 106, "tc_engine_used": 107, "compact_pool": 14,
    "compact_used": 108, "oz_image_slots": 109,
}

# every symbol include/mxp_chol.h declares (tests check the library exports them)
EXPORTS = [
    "mxp_chol_plan", "mxp_chol_plan_set", "mxp_chol_plan_get", "mxp_chol_workspace_size",
    "mxp_chol_set_workspace", "mxp_chol_factor_device", "mxp_chol_factor", "mxp_chol_factor_tiles", "mxp_chol_logdet",
    "mxp_precision_map_from_matrix_device", "mxp_precision_map_from_matrix", "mxp_generate_plgsy_device", "mxp_generate_kms_device",
    "mxp_generate_matern_device", "mxp_chol_factor_matern", "mxp_precision_map_matern_device",
    "mxp_chol_get_factor_device", "mxp_chol_tile_device_ptr", "mxp_chol_ipc_handle", "mxp_chol_ipc_attach",
    "mxp_chol_attach_peer_plan", "mxp_chol_describe", "mxp_chol_solve_lower", "mxp_chol_loglik",
    "mxp_chol_plan_destroy", "mxp_host_alloc", "mxp_host_free", "mxp_strerror", "mxp_last_error",
    "mxp_chol_abi_version", "mxp_chol_kernel_stats", "mxp_chol_timeline", "mxp_ooc_variant_volume", "mxp_chol_sched_diagnostics",
]
KCLASS = {"chain": 0, "potrf": 1, "trsm": 2, "other": 3}


class MxpError(RuntimeError):
    def __init__(self, call: str, status: int):
        msg = lib().mxp_strerror(status).decode()
        detail = lib().mxp_last_error().decode()
        super().__init__(f"{call} -> {status} ({msg}){': ' + detail if detail else ''}")
        self.status = status


def lib_path() -> str:
    return _LIB_PATH


def lib():
    """Load the in-tree CUDA library.  Raises if it is missing: no fallback."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} not built; run __graft_entry__.build() "
                              "(python paper_2410_09819_b200/build.py)")
        L = ctypes.CDLL(_LIB_PATH)
        i64, u64, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        vp, pi64, psz = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_size_t)
        pd = ctypes.POINTER(ctypes.c_double)
        L.mxp_chol_plan.argtypes = [i64, i64, vp, i32, ctypes.POINTER(vp)]
        L.mxp_chol_plan_set.argtypes = [vp, i32, i64]
        L.mxp_chol_plan_get.argtypes = [vp, i32, pi64]
        L.mxp_chol_workspace_size.argtypes = [vp, psz]
        L.mxp_chol_set_workspace.argtypes = [vp, vp, ctypes.c_size_t]
        L.mxp_chol_factor_device.argtypes = [vp, vp, i64, pi64]
        L.mxp_chol_factor.argtypes = [vp, vp, i64, pi64]
        L.mxp_chol_factor_tiles.argtypes = [vp, vp, vp, pi64]
        L.mxp_chol_logdet.argtypes = [vp, pd]
        L.mxp_precision_map_from_matrix_device.argtypes = [i64, i64, vp, i64, ctypes.c_double,
                                                            ctypes.c_uint32, vp, vp]
        L.mxp_precision_map_from_matrix.argtypes = [i64, i64, vp, i64, ctypes.c_double, ctypes.c_uint32, vp, vp]
        L.mxp_generate_plgsy_device.argtypes = [i64, u64, vp, i64, vp]
        L.mxp_generate_kms_device.argtypes = [i64, ctypes.c_double, vp, i64, vp]
        L.mxp_generate_matern_device.argtypes = [i64, vp, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                                 vp, i64, vp]
        L.mxp_chol_plan_destroy.argtypes = [vp]
        L.mxp_chol_plan_destroy.restype = None
        L.mxp_host_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(vp)]
        L.mxp_host_free.argtypes = [vp]
        L.mxp_strerror.argtypes = [i32]
        L.mxp_strerror.restype = ctypes.c_char_p
        L.mxp_last_error.argtypes = []
        L.mxp_last_error.restype = ctypes.c_char_p
        L.mxp_chol_abi_version.argtypes = []
        L.mxp_chol_kernel_stats.argtypes = [vp, i32, pi64, pd, pd]
        L.mxp_chol_timeline.argtypes = [vp, pd, i64, pi64]
        L.mxp_ooc_variant_volume.argtypes = [i64, i64, i32, i32, i64, pi64]
        L.mxp_chol_factor_matern.argtypes = [vp, vp, ctypes.c_double, ctypes.c_double, ctypes.c_double, pi64]
        L.mxp_precision_map_matern_device.argtypes = [i64, i64, vp, ctypes.c_double, ctypes.c_double,
                                                      ctypes.c_double, ctypes.c_double, ctypes.c_uint32, vp, vp]
        L.mxp_chol_get_factor_device.argtypes = [vp, vp, i64]
        L.mxp_chol_ipc_handle.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_uint64)]
        L.mxp_chol_ipc_attach.argtypes = [vp, i32, vp, ctypes.c_uint64]
        L.mxp_chol_attach_peer_plan.argtypes = [vp, i32, vp]
        L.mxp_chol_describe.argtypes = [vp, i32, pi64]
        L.mxp_chol_tile_device_ptr.argtypes = [vp, i64, i64, ctypes.POINTER(vp)]
        L.mxp_chol_sched_diagnostics.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64), i64, pi64]
        L.mxp_chol_solve_lower.argtypes = [vp, vp, vp, pd]
        L.mxp_chol_loglik.argtypes = [vp, vp, pd]
        _lib = L
        return L


def _check(call: str, rc: int):
    if rc != 0:
        raise MxpError(call, rc)


def abi_version() -> int:
    return lib().mxp_chol_abi_version()


def _colmajor_ptr(A, n: int):
    """(pointer, lda) of a Fortran-strided 2-D tensor/array with >= n rows."""
    try:  # torch
        import torch
        if isinstance(A, torch.Tensor):
            if A.dtype != torch.float64:
                raise TypeError("A must be float64")
            if A.dim() != 2 or A.shape[0] != n or A.shape[1] != n:
                raise ValueError("A must be n x n")
            if A.stride(0) != 1:
                raise ValueError("A must be column-major (stride(0) == 1); pass S.T for a "
                                 "row-major symmetric S")
            return A.data_ptr(), max(A.stride(1), n), A.is_cuda
    except ImportError:
        pass
    import numpy as np
    if isinstance(A, np.ndarray):
        if A.dtype != np.float64 or A.shape != (n, n) or not A.flags.f_contiguous:
            raise ValueError("A must be an n x n Fortran-ordered float64 array")
        return A.ctypes.data, n, False
    raise TypeError("A must be a torch tensor or numpy array")


class Plan:
    """Owns an ``mxp_plan_t``.  ``Plan(n, nb, precision_map=None)``."""

    def __init__(self, n: int, nb: int, precision_map=None, ngpus: int = 1):
        self._h = ctypes.c_void_p()
        self.n, self.nb = int(n), int(nb)
        self._map = None
        mp = None
        if precision_map is not None:
            import numpy as np
            self._map = np.ascontiguousarray(precision_map, dtype=np.uint8)
            mp = self._map.ctypes.data
        _check("mxp_chol_plan", lib().mxp_chol_plan(self.n, self.nb, mp, ngpus, ctypes.byref(self._h)))
        self._ws = None

    def __del__(self):
        self.close()

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().mxp_chol_plan_destroy(self._h)
            self._h = ctypes.c_void_p()
        self._ws = self._ws_keep = None  # release a torch-provided workspace with the plan

    def set(self, key: str, value: int):
        _check(f"mxp_chol_plan_set({key})", lib().mxp_chol_plan_set(self._h, ATTR[key], int(value)))

    def get(self, key: str) -> int:
        v = ctypes.c_int64()
        _check(f"mxp_chol_plan_get({key})", lib().mxp_chol_plan_get(self._h, ATTR[key], ctypes.byref(v)))
        return v.value

    def workspace_size(self) -> int:
        v = ctypes.c_size_t()
        _check("mxp_chol_workspace_size", lib().mxp_chol_workspace_size(self._h, ctypes.byref(v)))
        return v.value

    def set_workspace(self, tensor):
        """Hand the plan a caller-owned device buffer (a torch uint8 CUDA tensor)."""
        _check("mxp_chol_set_workspace",
               lib().mxp_chol_set_workspace(self._h, tensor.data_ptr(), tensor.numel() * tensor.element_size()))
        self._ws = tensor

    def use_torch_workspace(self, device=None):
        import torch
        nbytes = self.workspace_size()
        t = torch.empty(nbytes + 256, dtype=torch.uint8, device=device or "cuda")
        off = (-t.data_ptr()) % 256
        self.set_workspace(t[off:off + nbytes])
        self._ws_keep = t
        return t

    def _stream_from_torch(self):
        import torch
        self.set("stream", torch.cuda.current_stream().cuda_stream)

    def factor_device(self, A, stream_from_torch: bool = True) -> int:
        """In-place factorization of a device-resident column-major fp64 matrix.
        Returns info (0 = success, j > 0 = leading minor j not PD)."""
        ptr, lda, is_cuda = _colmajor_ptr(A, self.n)
        if not is_cuda:
            raise ValueError("factor_device needs a CUDA tensor")
        if stream_from_torch:
            self._stream_from_torch()
        info = ctypes.c_int64()
        _check("mxp_chol_factor_device", lib().mxp_chol_factor_device(self._h, ptr, lda, ctypes.byref(info)))
        return info.value

    def factor(self, A_host, stream_from_torch: bool = True) -> int:
        """In-place factorization of a host-resident column-major fp64 matrix
        (torch CPU tensor, ideally pinned, or numpy Fortran array)."""
        ptr, lda, is_cuda = _colmajor_ptr(A_host, self.n)
        if is_cuda:
            raise ValueError("factor needs a host buffer; use factor_device")
        if stream_from_torch:
            self._stream_from_torch()
        info = ctypes.c_int64()
        _check("mxp_chol_factor", lib().mxp_chol_factor(self._h, ptr, lda, ctypes.byref(info)))
        return info.value

    def factor_tiles(self, tiles, scales, stream_from_torch: bool = True) -> int:
        """Tile-packed host storage at storage precision (mxp_chol_factor_tiles): `tiles` is a
        list of Nt(Nt+1)/2 C-contiguous host buffers (numpy arrays or CPU tensors) in column-major
        lower-tile order, each the nb x nb column-major tile at its precision (float64, float32,
        float16 codes, uint8 E4M3 codes); `scales` a float64 array (value = code / scale).
        Both are overwritten with L.  Returns info."""
        import numpy as np
        ptrs = (ctypes.c_void_p * len(tiles))()
        for t, x in enumerate(tiles):
            ptrs[t] = x.ctypes.data if hasattr(x, "ctypes") else x.data_ptr()
        assert isinstance(scales, np.ndarray) and scales.dtype == np.float64 and scales.flags.c_contiguous
        if stream_from_torch:
            self._stream_from_torch()
        info = ctypes.c_int64()
        _check("mxp_chol_factor_tiles", lib().mxp_chol_factor_tiles(self._h, ptrs, scales.ctypes.data,
                                                                    ctypes.byref(info)))
        return info.value

    def factor_matern(self, xy, sigma2: float = 1.0, range_a: float = 0.02627, nugget: float = 0.0,
                      stream_from_torch: bool = True) -> int:
        """Factor the Matern covariance of locations xy (n x 2), generated tile by
        tile on the device (never stored densely).  Returns info."""
        import torch
        xyd = torch.as_tensor(xy, dtype=torch.float64).to("cuda").contiguous()
        if stream_from_torch:
            self._stream_from_torch()
        info = ctypes.c_int64()
        _check("mxp_chol_factor_matern", lib().mxp_chol_factor_matern(
            self._h, xyd.data_ptr(), float(sigma2), float(range_a), float(nugget), ctypes.byref(info)))
        self._xy = xyd
        return info.value

    def get_factor(self, L=None):
        """Resident factor as a (column-major view of a) device tensor."""
        import torch
        if L is None:
            L = torch.zeros((self.n, self.n), dtype=torch.float64, device="cuda").T
        ptr, ld, _ = _colmajor_ptr(L, self.n)
        _check("mxp_chol_get_factor_device", lib().mxp_chol_get_factor_device(self._h, ptr, ld))
        return L

    def describe(self, streaming: bool = False) -> dict:
        """Host-only task-list census of this rank (no GPU needed)."""
        c = (ctypes.c_int64 * 6)()
        _check("mxp_chol_describe", lib().mxp_chol_describe(self._h, int(streaming), c))
        return dict(zip(["gemm", "trsm", "quant", "prep", "potrf", "owned_tiles"], list(c)))

    def ipc_handle(self) -> tuple[bytes, int]:
        """(64-byte cudaIpcMemHandle of this plan's workspace, workspace bytes)."""
        buf = (ctypes.c_uint8 * 64)()
        nbytes = ctypes.c_uint64()
        _check("mxp_chol_ipc_handle", lib().mxp_chol_ipc_handle(self._h, buf, ctypes.byref(nbytes)))
        return bytes(buf), nbytes.value

    def ipc_attach(self, peer_rank: int, handle: bytes, ws_bytes: int):
        buf = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
        _check("mxp_chol_ipc_attach", lib().mxp_chol_ipc_attach(self._h, peer_rank, buf, ws_bytes))

    def connect(self, rank: int, world: int, group=None, sm_partition: bool = False):
        """Join a row-cyclic multi-GPU factorization, one process per rank:
        sets rank/nranks, exchanges the workspaces' IPC handles over the
        torch.distributed ``group`` (object all-gather; plumbing only) and maps
        every peer's workspace.  ``sm_partition``: ranks share one GPU (tests)
        and split its SMs evenly.  Collective: every rank must call it."""
        import torch.distributed as dist
        self.set("rank", rank)
        self.set("nranks", world)
        if sm_partition:
            import torch
            nsm = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
            share = nsm // world
            self.set("sm_first", rank * share)
            self.set("sm_count", share)
        mine = self.ipc_handle()
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        for q, (h, nbytes) in enumerate(allh):
            if q != rank:
                self.ipc_attach(q, h, nbytes)

    def attach_peer(self, peer_rank: int, peer: "Plan"):
        _check("mxp_chol_attach_peer_plan", lib().mxp_chol_attach_peer_plan(self._h, peer_rank, peer._h))

    def kernel_stats(self) -> dict:
        """{class: (launches, ms, flops)} of the last factorization (profile=1)."""
        out = {}
        for name, c in KCLASS.items():
            n, ms, fl = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
            _check("mxp_chol_kernel_stats", lib().mxp_chol_kernel_stats(
                self._h, c, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(fl)))
            out[name] = (n.value, ms.value, fl.value)
        return out

    def timeline(self) -> dict:
        """Per-column copy/compute timeline of the last host-streaming factorization with
        profile=1 (ms since its start): {"h2d": [...], "d2h": [...], "work": [...]}, -1 = none."""
        n = ctypes.c_int64()
        _check("mxp_chol_timeline", lib().mxp_chol_timeline(self._h, None, 0, ctypes.byref(n)))
        buf = (ctypes.c_double * n.value)()
        _check("mxp_chol_timeline", lib().mxp_chol_timeline(self._h, buf, n.value, ctypes.byref(n)))
        v = list(buf)
        return {"h2d": v[0::3], "d2h": v[1::3], "work": v[2::3]}

    def sched_diagnostics(self) -> dict:
        """Device-side scheduler timing of the last factorization (profile=1)."""
        n = ctypes.c_int64()
        _check("mxp_chol_sched_diagnostics", lib().mxp_chol_sched_diagnostics(self._h, None, 0, ctypes.byref(n)))
        if n.value == 0:
            return {}
        buf = (ctypes.c_uint64 * n.value)()
        _check("mxp_chol_sched_diagnostics", lib().mxp_chol_sched_diagnostics(self._h, buf, n.value, ctypes.byref(n)))
        v = list(buf)
        nt = (len(v) - 36) // 3
        span = (v[7] - v[6]) / 1e6 if v[7] > v[6] else 0.0
        pot = [((v[36 + 3 * k] - v[6]) / 1e6, (v[37 + 3 * k] - v[6]) / 1e6, (v[38 + 3 * k] - v[6]) / 1e6)
               for k in range(nt)]
        return {"gemm_busy_ms": v[0] / 1e6, "gemm_wait_ms": v[1] / 1e6, "trsm_busy_ms": v[2] / 1e6,
                "trsm_wait_ms": v[3] / 1e6, "gemm_tasks": v[4], "trsm_tasks": v[5], "span_ms": span,
                "ctas": v[8], "potrf_phase_ms": {"update": v[9] / 1e6, "chol": v[10] / 1e6, "inverse": v[11] / 1e6,
                                                  "trsm": v[12] / 1e6},
                "ozaki_ms": {"stage_wait": v[13] / 1e6, "mma_done_wait": v[14] / 1e6, "drain": v[15] / 1e6,
                             "mma_issue": v[24] / 1e6, "copy_issue": v[25] / 1e6, "k_loop": v[26] / 1e6,
                             "drain_tile_wait": v[33] / 1e6},
                "native_ms": {"stage_wait": v[28] / 1e6, "refill_wait": v[29] / 1e6, "drained_wait": v[30] / 1e6,
                              "drain": v[31] / 1e6, "final_c": v[32] / 1e6},
                "gemm_busy_ms_by_precision": {p: v[16 + i] / 1e6 for i, p in enumerate(("fp64", "fp32", "fp16", "fp8"))},
                "gemm_tasks_by_precision": {p: v[20 + i] for i, p in enumerate(("fp64", "fp32", "fp16", "fp8"))},
                "potrf_timeline_ms": pot}

    def logdet(self) -> float:
        v = ctypes.c_double()
        _check("mxp_chol_logdet", lib().mxp_chol_logdet(self._h, ctypes.byref(v)))
        return v.value

    @staticmethod
    def _dev_vec(y, n):
        import torch
        if not (isinstance(y, torch.Tensor) and y.is_cuda and y.dtype == torch.float64 and y.numel() == n
                and y.is_contiguous()):
            raise ValueError("y must be a contiguous float64 CUDA tensor of n elements")
        return y.data_ptr()

    def solve_lower(self, y, z=None) -> float:
        """z = L^-1 y on the resident factor (device tensors); returns ||z||^2."""
        q = ctypes.c_double()
        zp = self._dev_vec(z, self.n) if z is not None else None
        _check("mxp_chol_solve_lower",
               lib().mxp_chol_solve_lower(self._h, self._dev_vec(y, self.n), zp, ctypes.byref(q)))
        return q.value

    def loglik(self, y=None) -> float:
        """Eq. 1 log-likelihood of the last factorized covariance at y (device; None: y = 0)."""
        v = ctypes.c_double()
        yp = self._dev_vec(y, self.n) if y is not None else None
        _check("mxp_chol_loglik", lib().mxp_chol_loglik(self._h, yp, ctypes.byref(v)))
        return v.value


def precision_map_from_matrix(A, nb: int, eps: float, allowed: int = 0xF):
    """Planner on a HOST matrix (numpy array or CPU tensor; streamed to the device one
    tile column at a time) -> (uint8 map, float64 tile norms)."""
    import numpy as np
    Af = np.asfortranarray(np.asarray(A, dtype=np.float64))
    n = Af.shape[0]
    Nt = -(-n // nb)
    m = np.empty(Nt * (Nt + 1) // 2, np.uint8)
    f = np.empty(Nt * (Nt + 1) // 2, np.float64)
    _check("mxp_precision_map_from_matrix",
           lib().mxp_precision_map_from_matrix(n, nb, Af.ctypes.data, n, float(eps), allowed,
                                               m.ctypes.data, f.ctypes.data))
    return m, f


def precision_map_from_matrix_device(A, nb: int, eps: float, allowed: int = 0xF):
    """Planner on a device matrix -> (uint8 map, float64 tile norms)."""
    import numpy as np
    n = A.shape[0]
    ptr, lda, is_cuda = _colmajor_ptr(A, n)
    if not is_cuda:
        raise ValueError("needs a CUDA tensor")
    Nt = -(-n // nb)
    m = np.empty(Nt * (Nt + 1) // 2, np.uint8)
    f = np.empty(Nt * (Nt + 1) // 2, np.float64)
    _check("mxp_precision_map_from_matrix_device",
           lib().mxp_precision_map_from_matrix_device(n, nb, ptr, lda, float(eps), allowed,
                                                      m.ctypes.data, f.ctypes.data))
    return m, f


OOC_VARIANTS = {"sync": 0, "async": 1, "V1": 2, "V2": 3, "V3": 4, "static": 5, "MIN": 6}


def ooc_variant_volume(n: int, nb: int, variant: str, hbm_bytes: int = 0, streams: int = 1):
    """Host-link ledger of one of the paper's OOC variants over the static schedule
    (mxp_ooc_variant_volume): {"h2d_bytes", "d2h_bytes", "loads", "peak_tiles"}, or None
    when the capacity cannot hold the variant's working set."""
    out = (ctypes.c_int64 * 4)()
    rc = lib().mxp_ooc_variant_volume(int(n), int(nb), OOC_VARIANTS[variant], int(streams), int(hbm_bytes), out)
    if rc == -1002:
        return None
    _check("mxp_ooc_variant_volume", rc)
    return {"h2d_bytes": out[0], "d2h_bytes": out[1], "loads": out[2], "peak_tiles": out[3]}


def precision_map_matern_device(xy, nb: int, eps: float, sigma2: float = 1.0, range_a: float = 0.02627,
                                nugget: float = 0.0, allowed: int = 0xF):
    """Planner on the generated Matern covariance -> (uint8 map, tile norms)."""
    import numpy as np
    import torch
    xyd = torch.as_tensor(xy, dtype=torch.float64).to("cuda").contiguous()
    n = xyd.shape[0]
    Nt = -(-n // nb)
    m = np.empty(Nt * (Nt + 1) // 2, np.uint8)
    f = np.empty(Nt * (Nt + 1) // 2, np.float64)
    _check("mxp_precision_map_matern_device",
           lib().mxp_precision_map_matern_device(n, nb, xyd.data_ptr(), float(sigma2), float(range_a),
                                                 float(nugget), float(eps), allowed, m.ctypes.data, f.ctypes.data))
    return m, f


def generate_plgsy_device(A, seed: int = 42, stream=None):
    n = A.shape[0]
    ptr, lda, is_cuda = _colmajor_ptr(A, n)
    _check("mxp_generate_plgsy_device", lib().mxp_generate_plgsy_device(n, seed, ptr, lda, stream))


def generate_kms_device(A, rho: float, stream=None):
    n = A.shape[0]
    ptr, lda, is_cuda = _colmajor_ptr(A, n)
    _check("mxp_generate_kms_device", lib().mxp_generate_kms_device(n, float(rho), ptr, lda, stream))


def generate_matern_device(A, xy, sigma2: float = 1.0, range_a: float = 0.02627, nugget: float = 0.0,
                           stream=None):
    """A (column-major device view) <- Matern nu=0.5 covariance of the n x 2
    locations xy (numpy or torch; copied to the device)."""
    import torch
    n = A.shape[0]
    ptr, lda, is_cuda = _colmajor_ptr(A, n)
    xyd = torch.as_tensor(xy, dtype=torch.float64).to(A.device).contiguous()
    _check("mxp_generate_matern_device",
           lib().mxp_generate_matern_device(n, xyd.data_ptr(), float(sigma2), float(range_a), float(nugget),
                                            ptr, lda, stream))
    return xyd


def host_alloc(nbytes: int) -> int:
    p = ctypes.c_void_p()
    _check("mxp_host_alloc", lib().mxp_host_alloc(nbytes, ctypes.byref(p)))
    return p.value


def host_free(ptr: int):
    _check("mxp_host_free", lib().mxp_host_free(ptr))
