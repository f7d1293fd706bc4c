"""Barycentric multi-index space of the degree-N simplex (host side).

Degrees of freedom are addressed by exponent tuples ``alpha`` with
``|alpha| = N``.  The enumeration is the reference's frozen canonical order
(first exponent slowest, ascending; the last exponent implied) --
``/root/reference/pkg/src/bbdg/multiindex.py:1-12,48-61``.  Unlike the reference,
which enumerates tuples recursively and inverts them through a dict, the
position of a tuple is given here by a closed form, which is the same formula
the CUDA kernels evaluate in registers:

    pos3(a0,a1,a2)   = sum_{a<a0} C(N-a+2,2) + sum_{b<a1} (N-a0-b+1) + a2
    pos2(b0,b1)      = sum_{a<b0} (N-a+1) + b1

Face ``f`` is ``{alpha_f = 0}`` and layer ``j`` of face ``f`` is
``{alpha_f = j}`` (``multiindex.py:81-120`` of the reference).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

MAX_DEGREE = 20

# bi-unit reference tetrahedron; lambda_0 vanishes on r+s+t=-1 and
# lambda_{1,2,3} on r=-1, s=-1, t=-1 (reference multiindex.py:123-133)
TET_VERTICES = np.array(
    [[-1.0, -1.0, -1.0], [1.0, -1.0, -1.0], [-1.0, 1.0, -1.0], [-1.0, -1.0, 1.0]]
)
TRI_VERTICES = np.array([[-1.0, -1.0], [1.0, -1.0], [-1.0, 1.0]])
FACE_VERTICES = ((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2))
REFERENCE_TET_VOLUME = 4.0 / 3.0


def simplex_dim(N: int, d: int) -> int:
    return math.comb(N + d, d) if N >= 0 else 0


def tet_dim(N: int) -> int:
    return simplex_dim(N, 3)


def face_dim(N: int) -> int:
    return simplex_dim(N, 2)


def check_degree(N, lowest=0):
    if not isinstance(N, (int, np.integer)) or not lowest <= N <= MAX_DEGREE:
        raise ValueError(f"degree must be an integer in {lowest}..{MAX_DEGREE}, got {N!r}")


def check_face(f):
    if f not in (0, 1, 2, 3):
        raise ValueError(f"face id must be one of 0..3, got {f!r}")


@lru_cache(maxsize=None)
def simplex_indices(N: int, d: int = 3) -> np.ndarray:
    """(simplex_dim, d+1) int array of exponents in canonical order."""
    check_degree(N)
    if d == 0:
        return np.array([[N]], dtype=np.int64)
    rows = []
    for a in range(N + 1):
        rest = simplex_indices(N - a, d - 1)
        rows.append(np.concatenate([np.full((len(rest), 1), a, dtype=np.int64), rest], axis=1))
    out = np.concatenate(rows, axis=0)
    out.setflags(write=False)
    return out


def tet_indices(N: int) -> np.ndarray:
    check_degree(N, lowest=1)
    return simplex_indices(N, 3)


def pos2(N, b0, b1):
    """Closed-form canonical position of (b0, b1, N-b0-b1) in the triangle space."""
    b0 = np.asarray(b0, dtype=np.int64)
    b1 = np.asarray(b1, dtype=np.int64)
    return b0 * (N + 1) - (b0 * (b0 - 1)) // 2 + b1


def pos3(N, a0, a1, a2):
    """Closed-form canonical position of (a0, a1, a2, N-a0-a1-a2) in the tet space."""
    a0 = np.asarray(a0, dtype=np.int64)
    a1 = np.asarray(a1, dtype=np.int64)
    a2 = np.asarray(a2, dtype=np.int64)
    # sum_{a<a0} C(N-a+2, 2) = C(N+3,3) - C(N-a0+3,3)
    head = math.comb(N + 3, 3) - _c3(N - a0 + 3)
    M = N - a0
    return head + a1 * (M + 1) - (a1 * (a1 - 1)) // 2 + a2


def _c3(n):
    n = np.asarray(n, dtype=np.int64)
    return n * (n - 1) * (n - 2) // 6


def index_positions(N: int, d: int = 3) -> dict:
    """tuple -> position map (compatibility with the reference API)."""
    return {tuple(int(x) for x in a): k for k, a in enumerate(simplex_indices(N, d))}


@lru_cache(maxsize=None)
def face_trace_positions(N: int, f: int) -> np.ndarray:
    """Volume positions of face f's coefficients, in 2-D canonical order."""
    check_degree(N, lowest=1)
    check_face(f)
    b = simplex_indices(N, 2)
    alpha = np.insert(b, f, 0, axis=1)
    out = pos3(N, alpha[:, 0], alpha[:, 1], alpha[:, 2])
    out.setflags(write=False)
    return out


@dataclass(frozen=True)
class FaceLayers:
    face: int
    layers: tuple

    @property
    def sizes(self):
        return tuple(len(x) for x in self.layers)


@lru_cache(maxsize=None)
def face_layers(N: int, f: int) -> FaceLayers:
    """layers[j] = positions with alpha_f = j, 2-D canonical order of the rest."""
    check_degree(N, lowest=1)
    check_face(f)
    out = []
    for j in range(N + 1):
        b = simplex_indices(N - j, 2)
        alpha = np.insert(b, f, j, axis=1)
        out.append(pos3(N, alpha[:, 0], alpha[:, 1], alpha[:, 2]))
    return FaceLayers(face=f, layers=tuple(out))


def barycentric_from_rst(rst) -> np.ndarray:
    rst = np.asarray(rst, dtype=float)
    r, s, t = rst[..., 0], rst[..., 1], rst[..., 2]
    return np.stack([-(1.0 + r + s + t) / 2.0, (1.0 + r) / 2.0, (1.0 + s) / 2.0, (1.0 + t) / 2.0], -1)


def tri_barycentric_from_rs(rs) -> np.ndarray:
    rs = np.asarray(rs, dtype=float)
    r, s = rs[..., 0], rs[..., 1]
    return np.stack([-(r + s) / 2.0, (1.0 + r) / 2.0, (1.0 + s) / 2.0], -1)


def lattice_barycentric(N: int, d: int = 3) -> np.ndarray:
    return simplex_indices(N, d).astype(float) / N


def tet_lattice_rst(N: int) -> np.ndarray:
    return lattice_barycentric(N, 3) @ TET_VERTICES


def face_lattice_rst(N: int, f: int) -> np.ndarray:
    """Face f lattice points in volume (r,s,t), in trace order."""
    check_face(f)
    lam = np.insert(lattice_barycentric(N, 2), f, 0.0, axis=1)
    return lam @ TET_VERTICES


@lru_cache(maxsize=None)
def face_permutation_table(N: int) -> np.ndarray:
    """(6, Nfp) face-point permutations, one per ordering of the face's vertices.

    Row ``s`` maps local face point ``m`` (2-D barycentric exponents b) to the
    neighbour's face point whose exponents are ``b`` re-ordered by the vertex
    permutation ``PERMS3[s]`` (neighbour slot ``PERMS3[s][k]`` holds local
    vertex ``k``).  This replaces the reference's per-node coordinate matching
    (``mesh.py:158-188``) for conforming meshes.
    """
    b = simplex_indices(N, 2)
    out = np.empty((6, len(b)), dtype=np.int64)
    for s, sig in enumerate(PERMS3):
        nb = np.empty_like(b)
        for k in range(3):
            nb[:, sig[k]] = b[:, k]
        out[s] = pos2(N, nb[:, 0], nb[:, 1])
    return out


PERMS3 = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))
