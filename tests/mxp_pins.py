"""Shared loader for tests/golden/mxp_rounding_points.json (hand-derived MxP pins).

Only parses the golden file into numpy arrays; holds none of the method's
arithmetic (the expected values are the file's, derived by hand).
"""
import json
import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mxp_rounding_points.json")


def num(s: str) -> float:
    return float.fromhex(s) if s.lower().startswith(("0x", "-0x")) else float(s)


def ij(key: str):
    i, j = key.split(",")
    return int(i), int(j)


def tile_index(Nt, i, j):  # column-major lower-tile order
    return j * Nt - j * (j - 1) // 2 + (i - j)


def cases():
    with open(PATH) as f:
        return json.load(f)["cases"]


def scalar_case(c):
    """(A, L_expected, map) of a case at nb = 1 (dense symmetric A, lower L)."""
    n = c["n"]
    A = np.zeros((n, n))
    L = np.zeros((n, n))
    for k, v in c["A_lower"].items():
        i, j = ij(k)
        A[i, j] = A[j, i] = num(v)
    for k, v in c["L_lower"].items():
        i, j = ij(k)
        L[i, j] = num(v)
    pmap = np.zeros(n * (n + 1) // 2, np.uint8)
    for k, p in c["map"].items():
        i, j = ij(k)
        pmap[tile_index(n, i, j)] = p
    return A, L, pmap


def embed(M: np.ndarray, nb: int) -> np.ndarray:
    """Tile (i, j) = M[i, j] * I_nb (the GPU embedding of a scalar case)."""
    return np.kron(M, np.eye(nb))
