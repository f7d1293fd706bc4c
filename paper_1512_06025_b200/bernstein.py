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

from . import _device, _lib
from .modal import tet_rule, triangle_rule
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
    tri_barycentric_from_rs,
)
from .sparse import SparseRowOperator, from_dense

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


def basis_dlambda_matrix(N: int, d: int, bary, i: int) -> np.ndarray:
    """Formal d/d lambda_i of every degree-N basis function at (npts, d+1) points
    (reference bernstein.py:98-112): C(N,alpha) alpha_i lambda^(alpha - e_i)."""
    bary = np.atleast_2d(np.asarray(bary, dtype=float))
    idx = simplex_indices(N, d)
    out = np.zeros((bary.shape[0], len(idx)))
    for p, alpha in enumerate(idx):
        if alpha[i] == 0:
            continue
        col = float(_multinomial(N, alpha)) * alpha[i] * np.ones(bary.shape[0])
        for m, a in enumerate(alpha):
            aa = a - 1 if m == i else a
            if aa:
                col *= bary[:, m] ** aa
        out[:, p] = col
    return out


def face_mass_matrix(N: int) -> np.ndarray:
    return mass_matrix(N, 2)


@dataclass(frozen=True, eq=False)
class BernsteinDerivativeSet:
    """D^0..D^3 as fixed-width rows (reference bernstein.py:182-197): row alpha of D^i holds
    alpha_j at column alpha + e_i - e_j; one (Np, 4) value table backs all four."""

    N: int
    values: np.ndarray
    ops: tuple

    def apply_all(self, q):
        return tuple(op.apply(q) for op in self.ops)


@lru_cache(maxsize=None)
def derivative_ops(N: int) -> BernsteinDerivativeSet:
    values, cols = derivative_tables(N)
    Np = tet_dim(N)
    ops = tuple(SparseRowOperator(Np, Np, values, cols[i].astype(np.intp)) for i in range(4))
    return BernsteinDerivativeSet(N=N, values=values, ops=ops)


@lru_cache(maxsize=None)
def build_L0(N: int) -> SparseRowOperator:
    """L0 = (N+1)^2/2 E^T E from its closed form (reference bernstein.py:221-229); <= 7 per row."""
    return from_dense(L0_dense(N))


@dataclass(frozen=True, eq=False)
class LiftFactorization:
    """Face lift without the dense matrix (reference bernstein.py:239-270)."""

    N: int
    Nfp: int
    L0: SparseRowOperator
    EL: SparseRowOperator     # (Np, 4 Nfp), <= Nfp + 3 entries per row
    ell: np.ndarray           # (N+1,), ell[0] = 1
    reductions: tuple         # (E^m_{m-1})^T for m = N..1, <= 3 per row
    layers: tuple             # FaceLayers per face

    def astype(self, dtype) -> "LiftFactorization":
        return LiftFactorization(self.N, self.Nfp, self.L0.astype(dtype), self.EL.astype(dtype),
                                 self.ell.astype(dtype), tuple(r.astype(dtype) for r in self.reductions),
                                 self.layers)


@lru_cache(maxsize=None)
def build_lift(N: int) -> LiftFactorization:
    """Reference bernstein.py:273-298, from the closed forms (E_L, L0, one-degree reductions)."""
    reductions = tuple(from_dense(elevation_dense(m, 2).T) for m in range(N, 0, -1))
    return LiftFactorization(N=N, Nfp=face_dim(N), L0=build_L0(N), EL=from_dense(el_dense(N)),
                             ell=lift_scalings(N), reductions=reductions,
                             layers=tuple(face_layers(N, f) for f in range(4)))


def _lift_device(N: int, flux):
    """bbdg_ops_lift: (..., 4, Nfp) -> (..., Np), L0 + one-degree reduction sweeps on the device."""
    fd, host = _device.to_device(flux)
    Nfp = face_dim(N)
    if tuple(fd.shape[-2:]) != (4, Nfp):
        raise ValueError(f"flux must end in (4, {Nfp}), got {tuple(fd.shape[-2:])}")
    out = _device.torch().empty(tuple(fd.shape[:-2]) + (tet_dim(N),), dtype=fd.dtype, device=fd.device)
    nb = fd.numel() // (4 * Nfp)
    _lib.check(_lib.load().bbdg_ops_lift(N, _device.dtype_id(fd), nb, fd.data_ptr(), out.data_ptr(),
                                         _device.stream()), "bbdg_ops_lift")
    return _device.back(out, host)


def lift_apply_factorized(lf: LiftFactorization, flux):
    """sum_f L^f flux_f with L = E_L L0 (reference bernstein.py:301-310).  E_L is the composition of
    the one-degree reductions scaled by ell_j, so the device applies it as those sweeps; the result
    equals the reference's E_L row product to rounding (the reference's own modes differ by <= 2.4e-16)."""
    if tuple(np.shape(flux))[-2:] != (4, lf.Nfp):
        raise ValueError(f"flux must end in (4, {lf.Nfp}), got {tuple(np.shape(flux))[-2:]}")
    return _lift_device(lf.N, flux)


def lift_apply_optimal(lf: LiftFactorization, flux):
    """Slice-by-slice lift, Algorithm 1 (reference bernstein.py:313-329): L0 per face, then N
    cascaded one-degree reductions writing layer j scaled by ell_j -- on the device."""
    if tuple(np.shape(flux))[-2:] != (4, lf.Nfp):
        raise ValueError(f"flux must end in (4, {lf.Nfp}), got {tuple(np.shape(flux))[-2:]}")
    return _lift_device(lf.N, flux)


def dense_lift_oracle(N: int, f: int) -> np.ndarray:
    """Quadrature-assembled M^{-1} M^f for one face (reference bernstein.py:350-365; a host-side
    check of the closed-form lifts, not used by any kernel)."""
    pts3, w3 = tet_rule(2 * N + 1)
    B3 = basis_matrix(N, 3, barycentric_from_rst(pts3))
    M = B3.T @ (w3[:, None] * B3)
    pts2, w2 = triangle_rule(2 * N + 2)
    bary2 = tri_barycentric_from_rs(pts2)
    C = basis_matrix(N, 3, np.insert(bary2, f, 0.0, axis=1)).T @ (w2[:, None] * basis_matrix(N, 2, bary2))
    return np.linalg.solve(M, C)


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

    @property
    def derivs(self) -> BernsteinDerivativeSet:
        return derivative_ops(self.N)

    @property
    def lift(self) -> LiftFactorization:
        return build_lift(self.N)

    def grad(self, q):
        """Reference-coordinate derivatives (bernstein.py:436-444) on the device:
        (d/dr, d/ds, d/dt) = ((D^1 - D^0) q, (D^2 - D^0) q, (D^3 - D^0) q) / 2, q (..., Np)."""
        qd, host = _device.to_device(q)
        if qd.shape[-1] != self.Np:
            raise ValueError(f"expected trailing size {self.Np}, got {qd.shape[-1]}")
        t = _device.torch()
        outs = [t.empty_like(qd) for _ in range(3)]
        _lib.check(_lib.load().bbdg_ops_grad(self.N, _device.dtype_id(qd), qd.numel() // self.Np, qd.data_ptr(),
                                             *[o.data_ptr() for o in outs], _device.stream()), "bbdg_ops_grad")
        return tuple(_device.back(o, host) for o in outs)

    def lift_flux(self, flux, mode: str = "factorized"):
        """Dispatch of the three lift modes (bernstein.py:457-466), on the device."""
        if mode == "dense":
            shp = tuple(np.shape(flux))
            if shp[-2:] != (4, self.Nfp):
                raise ValueError(f"flux must end in (4, {self.Nfp}), got {shp[-2:]}")
            fd, host = _device.to_device(flux)
            return _device.back(_device.dense_apply(("bb_dense_L", self.N), self.dense_L,
                                                    fd.reshape(shp[:-2] + (4 * self.Nfp,))), host)
        if mode == "factorized":
            return lift_apply_factorized(self.lift, flux)
        if mode == "optimal":
            return lift_apply_optimal(self.lift, flux)
        raise ValueError(f"unknown lift mode {mode!r}")

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
