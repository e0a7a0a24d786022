"""cuSOLVER potrf baseline (cusolverDnXpotrf, 64-bit API) through ctypes.

Library baseline only: it never touches our kernels.
"""
import ctypes
import glob
import os

_lib = None


def _load():
    global _lib
    if _lib is None:
        import nvidia
        cands = sorted(glob.glob(os.path.join(nvidia.__path__[0], "cusolver", "lib", "libcusolver.so*")))
        cands += ["/usr/local/cuda/lib64/libcusolver.so.11"]
        last = None
        for c in cands:
            try:
                _lib = ctypes.CDLL(c)
                break
            except OSError as e:
                last = e
        if _lib is None:
            raise OSError(f"libcusolver not found: {last}")
    return _lib


class Potrf:
    def __init__(self, n: int, lda: int, A_ptr: int, stream: int, uplo: int = 0):
        self.uplo = uplo
        L = _load()
        self.L = L
        self.h = ctypes.c_void_p()
        self.p = ctypes.c_void_p()
        assert L.cusolverDnCreate(ctypes.byref(self.h)) == 0
        assert L.cusolverDnSetStream(self.h, ctypes.c_void_p(stream)) == 0
        assert L.cusolverDnCreateParams(ctypes.byref(self.p)) == 0
        self.n, self.lda = n, lda
        dws, hws = ctypes.c_size_t(), ctypes.c_size_t()
        L.cusolverDnXpotrf_bufferSize.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                                  ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int,
                                                  ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]
        rc = L.cusolverDnXpotrf_bufferSize(self.h, self.p, uplo, n, 1, ctypes.c_void_p(A_ptr), lda, 1,
                                           ctypes.byref(dws), ctypes.byref(hws))
        assert rc == 0, rc
        self.dws, self.hws = dws.value, hws.value
        import torch
        self.dbuf = torch.empty(max(self.dws, 1), dtype=torch.uint8, device="cuda")
        self.hbuf = (ctypes.c_uint8 * max(self.hws, 1))()
        self.info = torch.zeros(1, dtype=torch.int32, device="cuda")
        L.cusolverDnXpotrf.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int,
                                       ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                       ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]

    def __call__(self, A_ptr: int) -> int:
        rc = self.L.cusolverDnXpotrf(self.h, self.p, self.uplo, self.n, 1, ctypes.c_void_p(A_ptr), self.lda, 1,
                                     ctypes.c_void_p(self.dbuf.data_ptr()), self.dws,
                                     ctypes.cast(self.hbuf, ctypes.c_void_p), self.hws,
                                     ctypes.c_void_p(self.info.data_ptr()))
        assert rc == 0, rc
        return rc

    def close(self):
        self.L.cusolverDnDestroyParams(self.p)
        self.L.cusolverDnDestroy(self.h)


def potrs(h_potrf: "Potrf", A_ptr: int, B_ptr: int, nrhs: int = 1) -> None:
    """cusolverDnXpotrs on the factor left in A by Potrf (same uplo): B <- A^-1 B."""
    L = h_potrf.L
    L.cusolverDnXpotrs.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                   ctypes.c_int64, ctypes.c_void_p]
    rc = L.cusolverDnXpotrs(h_potrf.h, h_potrf.p, h_potrf.uplo, h_potrf.n, nrhs, 1, ctypes.c_void_p(A_ptr),
                            h_potrf.lda, 1, ctypes.c_void_p(B_ptr), h_potrf.n, ctypes.c_void_p(h_potrf.info.data_ptr()))
    assert rc == 0, rc
