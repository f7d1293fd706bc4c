"""CPU ORACLE for the BB-DG hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module, and only
as the checker / the reference CPU arm.  The product (``paper_1512_06025_b200``)
never imports it and has no CPU fallback.

A plain numpy restatement of the reference package's per-timestep RHS and
LSRK4 update (``/root/reference/pkg/src/bbdg``), following its algorithm
line by line: fixed-width sparse rows applied by gather + einsum
(``sparse.py:29-38``), the four barycentric derivative operators
(``bernstein.py:200-218``), ``L0 = (N+1)^2/2 E^T E`` (``:221-229``), E_L from the
composed reduction stack (``:263-298``), the three lift modes (``:301-347,
457-466``), coordinate-matched trace gathers (``mesh.py:158-188``),
``volume_rhs`` / ``surface_rhs`` / ``rhs`` (``solver.py:139-193``) and the
five-stage LSRK4 step (``solver.py:196-214``).  The operator tables are built
here from the reference's definitions, independently of the product's
closed forms.

Parity is pinned: ``tests/test_oracle_golden.py`` checks this module against
vectors produced by running the reference itself
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import math
from functools import lru_cache

import numpy as np

RK4A = np.array([0.0, -567301805773.0 / 1357537059087.0, -2404267990393.0 / 2016746695238.0,
                 -3550918686646.0 / 2091501179385.0, -1275806237668.0 / 842570457699.0])
RK4B = np.array([1432997174477.0 / 9575080441755.0, 5161836677717.0 / 13612068292357.0,
                 1720146321549.0 / 2090206949498.0, 3134564353537.0 / 4481467310338.0,
                 2277821191437.0 / 14882151754819.0])
TET_VERTICES = np.array([[-1.0, -1.0, -1.0], [1.0, -1.0, -1.0], [-1.0, 1.0, -1.0], [-1.0, -1.0, 1.0]])


# ----------------------------------------------------------------- index space (multiindex.py:48-120)
@lru_cache(maxsize=None)
def indices(N: int, d: int):
    def rec(total, slots):
        if slots == 1:
            yield (total,)
            return
        for a in range(total + 1):
            for rest in rec(total - a, slots - 1):
                yield (a,) + rest
    return tuple(rec(N, d + 1))


@lru_cache(maxsize=None)
def positions(N: int, d: int):
    return {a: k for k, a in enumerate(indices(N, d))}


def face_trace(N, f):
    pos = positions(N, 3)
    return np.array([pos[b[:f] + (0,) + b[f:]] for b in indices(N, 2)])


def face_layers(N, f):
    pos = positions(N, 3)
    return [np.array([pos[b[:f] + (j,) + b[f:]] for b in indices(N - j, 2)]) for j in range(N + 1)]


# ----------------------------------------------------------------- fixed-width sparse rows (sparse.py)
class Ell:
    def __init__(self, n_rows, n_cols, values, cols):
        self.n_rows, self.n_cols, self.values, self.cols = n_rows, n_cols, values, cols

    def apply(self, x):
        flat = x.reshape(-1, self.n_cols)
        out = np.einsum("brw,rw->br", flat[:, self.cols], self.values.astype(x.dtype, copy=False))
        return out.reshape(x.shape[:-1] + (self.n_rows,))

    def astype(self, dt):
        return Ell(self.n_rows, self.n_cols, self.values.astype(dt), self.cols)

    def dense(self):
        A = np.zeros((self.n_rows, self.n_cols))
        for r in range(self.n_rows):
            for v, c in zip(self.values[r], self.cols[r]):
                A[r, c] += v
        return A


def ell_from_rows(n_rows, n_cols, rows, width=None):
    width = max(1, width or max((len(r) for r in rows), default=1))
    vals = np.zeros((n_rows, width))
    cols = np.zeros((n_rows, width), dtype=np.intp)
    for r, ent in enumerate(rows):
        for k, (c, v) in enumerate(ent):
            cols[r, k], vals[r, k] = c, v
    return Ell(n_rows, n_cols, vals, cols)


def ell_from_dense(A):
    return ell_from_rows(A.shape[0], A.shape[1], [[(c, A[r, c]) for c in np.nonzero(A[r])[0]] for r in range(A.shape[0])])


# ----------------------------------------------------------------- Bernstein operators (bernstein.py)
def elevation(m, d):
    lo = positions(m - 1, d)
    rows = []
    for beta in indices(m, d):
        ent = []
        for j in range(d + 1):
            if beta[j] >= 1:
                a = tuple(b - (1 if k == j else 0) for k, b in enumerate(beta))
                ent.append((lo[a], beta[j] / m))
        rows.append(ent)
    return ell_from_rows(len(rows), len(lo), rows, width=d + 1)


def multinomial(n, alpha):
    out, rem = 1, n
    for a in alpha:
        out *= math.comb(rem, a)
        rem -= a
    return out


def mass(N, d):
    idx = indices(N, d)
    meas = {2: 2.0, 3: 4.0 / 3.0}[d]
    M = np.empty((len(idx), len(idx)))
    mult = [multinomial(N, a) for a in idx]
    den = math.comb(2 * N + d, d)
    for r, a in enumerate(idx):
        for c in range(r, len(idx)):
            ab = tuple(x + y for x, y in zip(a, idx[c]))
            M[r, c] = M[c, r] = meas * mult[r] * mult[c] / (multinomial(2 * N, ab) * den)
    return M


class BernsteinTables:
    """Reference operator tables for degree N (float64, cast on use)."""

    def __init__(self, N):
        self.N = N
        idx = indices(N, 3)
        pos = positions(N, 3)
        self.Np, self.Nfp = len(idx), len(indices(N, 2))
        self.dvals = np.array(idx, dtype=float)
        self.dcols = []
        for i in range(4):
            cols = np.zeros((self.Np, 4), dtype=np.intp)
            for r, a in enumerate(idx):
                for j in range(4):
                    b = list(a)
                    b[i] += 1
                    b[j] -= 1
                    if b[j] >= 0:
                        cols[r, j] = pos[tuple(b)]
            self.dcols.append(cols)
        E = elevation(N + 1, 2).dense()
        self.L0 = ell_from_dense(0.5 * (N + 1) ** 2 * (E.T @ E))
        stack = [np.eye(self.Nfp)]
        for j in range(1, N + 1):
            stack.append(elevation(N - j + 1, 2).dense().T @ stack[-1])
        self.ell = np.array([1.0] + [(-1.0) ** j * math.comb(N, j) / (1.0 + j) for j in range(1, N + 1)])
        self.layers = [face_layers(N, f) for f in range(4)]
        EL = np.zeros((self.Np, 4 * self.Nfp))
        for f in range(4):
            for j in range(N + 1):
                EL[np.ix_(self.layers[f][j], np.arange(f * self.Nfp, (f + 1) * self.Nfp))] = self.ell[j] * stack[j]
        self.EL = ell_from_dense(EL)
        self.reductions = [ell_from_dense(elevation(m, 2).dense().T) for m in range(N, 0, -1)]
        M, Mf = mass(N, 3), mass(N, 2)
        self.mass = M
        self.dense_L = np.empty((self.Np, 4 * self.Nfp))
        for f in range(4):
            emb = np.zeros((self.Np, self.Nfp))
            emb[face_trace(N, f), :] = Mf
            self.dense_L[:, f * self.Nfp : (f + 1) * self.Nfp] = np.linalg.solve(M, emb)
        self.trace = np.stack([face_trace(N, f) for f in range(4)])
        self.face_pts = np.stack([np.insert(np.array(indices(N, 2), dtype=float) / N, f, 0.0, axis=1) @ TET_VERTICES
                                  for f in range(4)])

    def grad(self, q):
        vals = self.dvals.astype(q.dtype)
        d = [np.einsum("brw,rw->br", q[:, c], vals) for c in self.dcols]
        h = q.dtype.type(0.5)
        return h * (d[1] - d[0]), h * (d[2] - d[0]), h * (d[3] - d[0])

    def lift(self, flux, mode, dtype):
        Nfp = self.Nfp
        if mode == "dense":
            return flux.reshape(flux.shape[:-2] + (4 * Nfp,)) @ self.dense_L.astype(dtype).T
        L0 = self.L0.astype(dtype)
        if mode == "factorized":
            v = L0.apply(flux)
            return self.EL.astype(dtype).apply(v.reshape(flux.shape[:-2] + (4 * Nfp,)))
        if mode == "optimal":
            out = np.zeros(flux.shape[:-2] + (self.Np,), dtype=flux.dtype)
            ell = self.ell.astype(dtype)
            for f in range(4):
                lay = self.layers[f]
                w = L0.apply(flux[..., f, :])
                out[..., lay[0]] += w
                for j in range(1, self.N + 1):
                    w = self.reductions[j - 1].astype(dtype).apply(w)
                    out[..., lay[j]] += ell[j] * w
            return out
        raise ValueError(f"unknown lift mode {mode!r}")


@lru_cache(maxsize=None)
def bernstein_tables(N):
    return BernsteinTables(N)


class NodalTables:
    """Nodal operators supplied by the caller (Dr, Ds, Dt, dense_L, trace, nodes)."""

    def __init__(self, N, Dr, Ds, Dt, dense_L, trace, nodes):
        self.N, self.Dr, self.Ds, self.Dt, self.dense_L = N, Dr, Ds, Dt, dense_L
        self.trace = np.asarray(trace)
        self.Np, self.Nfp = Dr.shape[0], self.trace.shape[1]
        self.face_pts = np.stack([nodes[self.trace[f]] for f in range(4)])

    def grad(self, q):
        dt = q.dtype
        return q @ self.Dr.astype(dt).T, q @ self.Ds.astype(dt).T, q @ self.Dt.astype(dt).T

    def lift(self, flux, mode, dtype):
        return flux.reshape(flux.shape[:-2] + (4 * self.Nfp,)) @ self.dense_L.astype(dtype).T


# ----------------------------------------------------------------- trace maps (mesh.py:158-188)
def trace_maps(vertices, tets, etoe, etof, face_pts, trace, Np, h_elem, rows=None):
    """Coordinate-matched flat gather (K,4,Nfp) + boundary mask (vectorised, bounded chunks).

    ``rows``: optional list of element ranges (k0, k1); only their gather rows are built (the
    others stay -1), for spot checks of meshes too large for the full map."""
    K, Nfp = len(tets), face_pts.shape[1]
    lam = np.stack([-(1.0 + face_pts[..., 0] + face_pts[..., 1] + face_pts[..., 2]) / 2.0,
                    (1.0 + face_pts[..., 0]) / 2.0, (1.0 + face_pts[..., 1]) / 2.0,
                    (1.0 + face_pts[..., 2]) / 2.0], -1)                    # (4,Nfp,4)

    def phys(ks):                                                          # (..., 4, Nfp, 3)
        return np.einsum("fnl,...lx->...fnx", lam, vertices[tets[ks]])

    kk = np.arange(K)[:, None]
    bnd = (etoe == kk) & (etof == np.arange(4)[None, :])
    gather = np.full((K, 4, Nfp), -1, dtype=np.int64)
    tol = 1e-8 * np.maximum(h_elem, 1.0)
    step = max(1, (1 << 22) // (4 * Nfp * Nfp))                             # bounded (n,4,Nfp,Nfp) chunks
    for r0, r1 in (rows if rows is not None else [(0, K)]):
        for k0 in range(r0, r1, step):
            k1 = min(r1, k0 + step)
            mine = phys(np.arange(k0, k1))                                  # (n,4,Nfp,3)
            theirs = np.einsum("kfnl,kflx->kfnx", lam[etof[k0:k1]], vertices[tets[etoe[k0:k1]]])
            d = np.linalg.norm(mine[:, :, :, None, :] - theirs[:, :, None, :, :], axis=-1)
            perm = np.argmin(d, axis=-1)                                    # (n,4,Nfp)
            dmin = np.take_along_axis(d, perm[..., None], -1)[..., 0]
            b = bnd[k0:k1]
            if np.any((dmin.max(axis=2) > tol[k0:k1, None]) & ~b):
                raise ValueError("non-conforming mesh")
            ef = etof[k0:k1]
            g = etoe[k0:k1, :, None] * Np + trace[ef][np.arange(k1 - k0)[:, None, None], np.arange(4)[None, :, None],
                                                      perm]
            own = np.arange(k0, k1)[:, None, None] * Np + trace[None, :, :]
            gather[k0:k1] = np.where(b[..., None], own, g)
    return gather, bnd


# ----------------------------------------------------------------- the solver (solver.py:99-214)
class OracleSystem:
    def __init__(self, mesh_arrays: dict, tables, kappa, rho, dtype=np.float64, rows=None, maps=None):
        m = mesh_arrays
        self.t = tables
        self.dtype = np.dtype(dtype).type
        self.K = len(m["tets"])
        if maps is None:
            maps = trace_maps(m["vertices"], m["tets"], m["etoe"], m["etof"], tables.face_pts, tables.trace,
                              tables.Np, m["h_elem"], rows)
        self.gather, self.boundary = maps
        rc = rho * np.sqrt(kappa / rho)
        mean_rc = 0.5 * (rc[:, None] + rc[m["etoe"]])
        d = self.dtype
        self.tau_p = (1.0 / mean_rc).astype(d)[:, :, None]
        self.tau_u = mean_rc.astype(d)[:, :, None]
        self.face_scale = (m["jf"] / m["jac"][:, None]).astype(d)[:, :, None]
        self.normals = m["normals"].astype(d)
        self.rst_dx = m["rst_dx"].astype(d)
        self.kappa = kappa.astype(d)[:, None]
        self.inv_rho = (1.0 / rho).astype(d)[:, None]

    # `sl` (a slice of elements) evaluates the rows of those elements only -- the same arithmetic per
    # element, so config-2 / bench-size meshes are checked in bounded-memory chunks (rhs_chunked)
    def volume_rhs(self, q, sl=slice(None)):
        qs = q[:, sl]
        dq = np.empty_like(qs)
        B = self.rst_dx[sl]
        gr, gs, gt = (g.reshape(qs.shape) for g in self.t.grad(qs.reshape(4 * qs.shape[1], -1)))
        for i in range(3):
            dq[1 + i] = -self.inv_rho[sl] * (B[:, 0, i, None] * gr[0] + B[:, 1, i, None] * gs[0]
                                             + B[:, 2, i, None] * gt[0])
        div = sum(B[:, 0, i, None] * gr[1 + i] + B[:, 1, i, None] * gs[1 + i] + B[:, 2, i, None] * gt[1 + i]
                  for i in range(3))
        dq[0] = -self.kappa[sl] * div
        return dq

    def surface_rhs(self, q, lift_mode="factorized", sl=slice(None)):
        loc = q[:, sl][..., self.t.trace]
        nbr = q.reshape(4, -1)[:, self.gather[sl]]
        jump = nbr - loc
        jp = np.where(self.boundary[sl][:, :, None], -2.0 * loc[0], jump[0])
        n = self.normals[sl]
        jun = n[:, :, 0, None] * jump[1] + n[:, :, 1, None] * jump[2] + n[:, :, 2, None] * jump[3]
        half = q.dtype.type(0.5)
        Fp = half * (self.tau_p[sl] * jp - jun) * self.face_scale[sl]
        Fu = half * (self.tau_u[sl] * jun - jp) * self.face_scale[sl]
        flux = np.stack([Fp] + [n[:, :, i, None] * Fu for i in range(3)])
        lifted = self.t.lift(flux, lift_mode, q.dtype)
        dq = np.empty((4,) + lifted.shape[1:], dtype=q.dtype)
        dq[0] = self.kappa[sl] * lifted[0]
        for i in range(3):
            dq[1 + i] = self.inv_rho[sl] * lifted[1 + i]
        return dq

    def rhs(self, q, lift_mode="factorized", sl=slice(None)):
        return self.volume_rhs(q, sl) + self.surface_rhs(q, lift_mode, sl)

    def rhs_chunked(self, q, lift_mode="factorized", k0=0, k1=None, chunk=2048):
        """rhs rows of elements [k0, k1) (all of them by default), evaluated chunk by chunk."""
        k1 = self.K if k1 is None else k1
        out = np.empty((4, k1 - k0, q.shape[2]), dtype=q.dtype)
        for a in range(k0, k1, chunk):
            b = min(k1, a + chunk)
            out[:, a - k0 : b - k0] = self.rhs(q, lift_mode, slice(a, b))
        return out

    def stage(self, q, res, rk_a, rk_b, dt, lift_mode="factorized", k0=0, k1=None, chunk=2048):
        """One LSRK stage for elements [k0, k1): (q_out, res_out) rows (solver.py:208-213)."""
        k1 = self.K if k1 is None else k1
        t = q.dtype.type
        k = self.rhs_chunked(q, lift_mode, k0, k1, chunk)
        r = res[:, k0:k1] * t(rk_a)
        r += t(dt) * k
        return q[:, k0:k1] + t(rk_b) * r, r

    def lsrk4_step(self, q, dt, lift_mode="factorized", res=None):
        if res is None:
            res = np.zeros_like(q)
        else:
            res[...] = 0.0
        for s in range(5):
            k = self.rhs(q, lift_mode)
            res *= q.dtype.type(RK4A[s])
            res += q.dtype.type(dt) * k
            q += q.dtype.type(RK4B[s]) * res
        return q


def mesh_arrays(mesh) -> dict:
    """The reference Mesh fields the oracle consumes, as plain arrays."""
    return {k: np.asarray(getattr(mesh, k)) for k in
            ("vertices", "tets", "jac", "rst_dx", "normals", "jf", "etoe", "etof", "h_elem")}
