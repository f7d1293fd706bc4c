"""Bernstein-Bezier reference operators: host tables for the sm_100a kernels.

The reference builds every operator as a fixed-width sparse-row table and
applies it through a numpy gather + einsum (``/root/reference/pkg/src/bbdg/
bernstein.py:182-347``, ``sparse.py:29-38``).  Here the derivative operators,
L0 and the one-degree reductions are never stored: the CUDA kernels evaluate
their entries by index arithmetic (closed forms below).  The host only builds
what has no cheap closed form on the device:

* ``el_cols/el_vals`` -- E_L as a fixed-width ELL table for the paper's
  non-optimal "factorized" surface kernel (Alg. 3),
* ``dense_L`` -- the classical ``M^{-1} M^f`` lift for the "dense" mode,
* ``mass`` -- for the energy functional.

Closed forms (each checked against the reference's stored tables in
``tests/test_host_tables.py``):

* D^i row alpha: value alpha_j at column alpha + e_i - e_j   (bernstein.py:182-218)
* L0[a,a] = 1/2 sum_j (a_j+1)^2, L0[a, a+e_j-e_k] = 1/2 (a_j+1) a_k   (bernstein.py:221-229)
* one-degree reduction (E^m_{m-1})^T: out[b] = sum_j (b_j+1)/m w[b+e_j]   (bernstein.py:290-295)
* ell_j = (-1)^j C(N,j)/(1+j)                                            (bernstein.py:232-236)
* E_L face f, layer j: ell_j * prod_k C(g_k, d_k) / C(N, j) at g = b + d   (bernstein.py:273-298)
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from .multiindex import (
    TET_VERTICES,
    barycentric_from_rst,
    face_dim,
    face_lattice_rst,
    face_layers,
    face_trace_positions,
    pos2,
    pos3,
    simplex_dim,
    simplex_indices,
    tet_dim,
)

REF_MEASURE = {1: 2.0, 2: 2.0, 3: 4.0 / 3.0}


def _multinomial(n: int, alpha) -> int:
    out = math.factorial(n)
    for a in alpha:
        out //= math.factorial(int(a))
    return out


def basis_matrix(N: int, d: int, bary) -> np.ndarray:
    """Degree-N Bernstein values C(N,alpha) lambda^alpha at (npts, d+1) points."""
    bary = np.atleast_2d(np.asarray(bary, dtype=float))
    idx = simplex_indices(N, d)
    coef = np.array([float(_multinomial(N, a)) for a in idx])
    out = np.ones((bary.shape[0], len(idx)))
    for m in range(d + 1):
        out *= bary[:, m : m + 1] ** idx[None, :, m]
    return out * coef[None, :]


@lru_cache(maxsize=None)
def mass_matrix(N: int, d: int = 3) -> np.ndarray:
    """Mass matrix |T| C(N,a)C(N,b) / (C(2N,a+b) C(2N+d,d)), evaluated in float64
    in the reference's operation order (bernstein.py:115-133) so the dense lift
    built from it reproduces the reference's to the last bit."""
    idx = simplex_indices(N, d)
    n = len(idx)
    mult = [_multinomial(N, a) for a in idx]
    den = math.comb(2 * N + d, d)
    meas = REF_MEASURE[d]
    M = np.empty((n, n))
    for r in range(n):
        for c in range(r, n):
            M[r, c] = M[c, r] = meas * mult[r] * mult[c] / (_multinomial(2 * N, idx[r] + idx[c]) * den)
    M.setflags(write=False)
    return M


def elevation_dense(m: int, d: int) -> np.ndarray:
    """One-degree elevation E^m_{m-1}: entry (b, a) = b_j/m for b = a + e_j."""
    rows = simplex_indices(m, d)
    E = np.zeros((len(rows), simplex_dim(m - 1, d)))
    lo = {tuple(a): k for k, a in enumerate(simplex_indices(m - 1, d))}
    for r, b in enumerate(rows):
        for j in range(d + 1):
            if b[j] >= 1:
                a = b.copy()
                a[j] -= 1
                E[r, lo[tuple(a)]] = b[j] / m
    return E


def lift_scalings(N: int) -> np.ndarray:
    return np.array([1.0] + [(-1.0) ** j * math.comb(N, j) / (1.0 + j) for j in range(1, N + 1)])


def L0_dense(N: int) -> np.ndarray:
    """L0 from its closed form (equals (N+1)^2/2 E^T E, reference bernstein.py:221-229)."""
    b = simplex_indices(N, 2)
    n = len(b)
    L = np.zeros((n, n))
    for r in range(n):
        a = b[r]
        L[r, r] = 0.5 * float(((a + 1) ** 2).sum())
        for j in range(3):
            for k in range(3):
                if j != k and a[k] >= 1:
                    g = a.copy()
                    g[j] += 1
                    g[k] -= 1
                    L[r, int(pos2(N, g[0], g[1]))] = 0.5 * (a[j] + 1) * a[k]
    return L


def reduction_dense(N: int, j: int) -> np.ndarray:
    """(E^N_{N-j})^T in closed form: entry (b, b+d) = prod_k C(b_k+d_k, d_k) / C(N, j)."""
    lo = simplex_indices(N - j, 2)
    dd = simplex_indices(j, 2) if j > 0 else np.zeros((1, 3), dtype=np.int64)
    R = np.zeros((len(lo), face_dim(N)))
    cnj = math.comb(N, j)
    for r, b in enumerate(lo):
        for d in dd:
            g = b + d
            c = math.comb(int(g[0]), int(d[0])) * math.comb(int(g[1]), int(d[1])) * math.comb(int(g[2]), int(d[2]))
            R[r, int(pos2(N, g[0], g[1]))] = c / cnj
    return R


@lru_cache(maxsize=None)
def el_dense(N: int) -> np.ndarray:
    """E_L (Np, 4 Nfp): face f, layer j rows carry ell_j (E^N_{N-j})^T."""
    Np, Nfp = tet_dim(N), face_dim(N)
    ell = lift_scalings(N)
    EL = np.zeros((Np, 4 * Nfp))
    for f in range(4):
        lay = face_layers(N, f).layers
        for j in range(N + 1):
            EL[np.ix_(lay[j], np.arange(f * Nfp, (f + 1) * Nfp))] = ell[j] * reduction_dense(N, j)
    EL.setflags(write=False)
    return EL


def ell_table(A: np.ndarray, width: int | None = None):
    """Dense -> fixed-width ELL (cols int32, vals float64), ascending columns,
    padding lanes at column 0 with value 0 (reference sparse.py:56-77)."""
    nz = [np.nonzero(A[r])[0] for r in range(A.shape[0])]
    w = max(1, max(len(c) for c in nz)) if width is None else width
    cols = np.zeros((A.shape[0], w), dtype=np.int32)
    vals = np.zeros((A.shape[0], w))
    for r, c in enumerate(nz):
        cols[r, : len(c)] = c
        vals[r, : len(c)] = A[r, c]
    return cols, vals


@lru_cache(maxsize=None)
def dense_lift(N: int) -> np.ndarray:
    """Classical lift M^{-1} [M^f embedded at face f's trace] (Np, 4 Nfp)."""
    Np, Nfp = tet_dim(N), face_dim(N)
    M = mass_matrix(N, 3)
    Mf = mass_matrix(N, 2)
    L = np.empty((Np, 4 * Nfp))
    for f in range(4):
        emb = np.zeros((Np, Nfp))
        emb[face_trace_positions(N, f), :] = Mf
        L[:, f * Nfp : (f + 1) * Nfp] = np.linalg.solve(M, emb)
    L.setflags(write=False)
    return L


def derivative_tables(N: int):
    """Reference-layout derivative tables (values (Np,4), cols (4,Np,4)) -- for
    parity tests of the index arithmetic only; kernels never read them."""
    idx = simplex_indices(N, 3)
    Np = len(idx)
    cols = np.zeros((4, Np, 4), dtype=np.int64)
    for i in range(4):
        for j in range(4):
            beta = idx.copy()
            beta[:, i] += 1
            beta[:, j] -= 1
            ok = beta[:, j] >= 0
            p = pos3(N, beta[:, 0], beta[:, 1], beta[:, 2])
            cols[i, :, j] = np.where(ok, p, 0)
    return idx.astype(float), cols


@dataclass(frozen=True, eq=False)
class BernsteinRefOps:
    """Degree-N Bernstein bundle (duck type of reference bernstein.py:387-466).

    Holds host tables only; the hot-path operators live in the CUDA library
    and are bound to a mesh through ``WaveSystem``.
    """

    N: int
    Np: int
    Nfp: int
    trace: np.ndarray
    dtype: object = np.float64
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    basis = "bernstein"

    @classmethod
    def build(cls, N: int) -> "BernsteinRefOps":
        if not isinstance(N, (int, np.integer)) or not 1 <= N <= 20:
            raise ValueError(f"degree must be an integer in 1..20, got {N!r}")
        trace = np.stack([face_trace_positions(N, f) for f in range(4)])
        return cls(N=int(N), Np=tet_dim(N), Nfp=face_dim(N), trace=trace)

    def astype(self, dtype) -> "BernsteinRefOps":
        if np.dtype(dtype) == np.dtype(self.dtype):
            return self
        return BernsteinRefOps(self.N, self.Np, self.Nfp, self.trace, np.dtype(dtype).type, self._cache)

    @property
    def mass(self) -> np.ndarray:
        return mass_matrix(self.N, 3)

    @property
    def dense_L(self) -> np.ndarray:
        return dense_lift(self.N)

    @property
    def ell(self) -> np.ndarray:
        return lift_scalings(self.N)

    def el_ell(self):
        """E_L as ELL (cols, vals), width <= Nfp + 3 (reference bernstein.py:286-289)."""
        if "el" not in self._cache:
            self._cache["el"] = ell_table(el_dense(self.N))
        return self._cache["el"]

    def face_trace(self, q):
        return q[..., self.trace]

    def face_ref_points(self, f):
        return face_lattice_rst(self.N, f)

    def eval_matrix(self, rst):
        return basis_matrix(self.N, 3, barycentric_from_rst(rst))
