"""Orthonormal (PKDO / Dubiner) simplex bases and collapsed-coordinate quadrature.

Host-side setup only: the nodal comparison operators (Vandermonde, Dr/Ds/Dt,
dense lift) and the error functional's quadrature are built once in float64
and uploaded.  Same bases and normalisations as the reference
(``/root/reference/pkg/src/bbdg/modal.py:87-175``, ``quadrature.py:205-231``),
written from the Hesthaven-Warburton formulas.
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import eval_jacobi, roots_jacobi

_EPS = 1.0e-12


def jacobi_p(x, n: int, a: float, b: float) -> np.ndarray:
    """Jacobi polynomial normalised to unit weighted L2 norm on [-1, 1]."""
    lognorm = ((a + b + 1.0) * math.log(2.0) + math.lgamma(n + a + 1.0) + math.lgamma(n + b + 1.0)
               - math.log(2.0 * n + a + b + 1.0) - math.lgamma(n + a + b + 1.0) - math.lgamma(n + 1.0))
    return eval_jacobi(n, a, b, np.asarray(x, dtype=float)) * math.exp(-0.5 * lognorm)


def jacobi_dp(x, n: int, a: float, b: float) -> np.ndarray:
    if n == 0:
        return np.zeros_like(np.asarray(x, dtype=float))
    return math.sqrt(n * (n + a + b + 1.0)) * jacobi_p(x, n - 1, a + 1.0, b + 1.0)


def mode_tuples(N: int, d: int):
    if d == 1:
        return [(i,) for i in range(N + 1)]
    if d == 2:
        return [(i, j) for i in range(N + 1) for j in range(N + 1 - i)]
    if d == 3:
        return [(i, j, k) for i in range(N + 1) for j in range(N + 1 - i) for k in range(N + 1 - i - j)]
    raise ValueError(f"unsupported dimension {d}")


def _collapse3(rst):
    r, s, t = rst[:, 0], rst[:, 1], rst[:, 2]
    st = -s - t
    a = np.where(np.abs(s + t) > _EPS, 2.0 * (1.0 + r) / np.where(np.abs(st) > _EPS, st, 1.0) - 1.0, -1.0)
    omt = 1.0 - t
    b = np.where(np.abs(omt) > _EPS, 2.0 * (1.0 + s) / np.where(np.abs(omt) > _EPS, omt, 1.0) - 1.0, -1.0)
    return a, b, t.copy()


def _collapse2(rs):
    r, s = rs[:, 0], rs[:, 1]
    oms = 1.0 - s
    a = np.where(np.abs(oms) > _EPS, 2.0 * (1.0 + r) / np.where(np.abs(oms) > _EPS, oms, 1.0) - 1.0, -1.0)
    return a, s.copy()


def ortho_basis(N: int, d: int, pts) -> np.ndarray:
    """(npts, dim) values of the orthonormal basis on the bi-unit simplex."""
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    modes = mode_tuples(N, d)
    V = np.empty((pts.shape[0], len(modes)))
    if d == 1:
        for m, (i,) in enumerate(modes):
            V[:, m] = jacobi_p(pts[:, 0], i, 0.0, 0.0)
    elif d == 2:
        a, b = _collapse2(pts)
        for m, (i, j) in enumerate(modes):
            V[:, m] = math.sqrt(2.0) * jacobi_p(a, i, 0, 0) * jacobi_p(b, j, 2 * i + 1, 0) * (1.0 - b) ** i
    else:
        a, b, c = _collapse3(pts)
        for m, (i, j, k) in enumerate(modes):
            V[:, m] = (2.0 * math.sqrt(2.0) * jacobi_p(a, i, 0, 0) * jacobi_p(b, j, 2 * i + 1, 0)
                       * (1.0 - b) ** i * jacobi_p(c, k, 2 * (i + j) + 2, 0) * (1.0 - c) ** (i + j))
    return V


def ortho_basis_grad(N: int, pts):
    """(Vr, Vs, Vt) gradients of the tet basis; negative powers cancelled analytically."""
    pts = np.atleast_2d(np.asarray(pts, dtype=float))
    a, b, c = _collapse3(pts)
    modes = mode_tuples(N, 3)
    out = [np.empty((pts.shape[0], len(modes))) for _ in range(3)]
    hb, hc = 0.5 * (1.0 - b), 0.5 * (1.0 - c)
    for m, (i, j, k) in enumerate(modes):
        fa, dfa = jacobi_p(a, i, 0, 0), jacobi_dp(a, i, 0, 0)
        gb, dgb = jacobi_p(b, j, 2 * i + 1, 0), jacobi_dp(b, j, 2 * i + 1, 0)
        gc, dgc = jacobi_p(c, k, 2 * (i + j) + 2, 0), jacobi_dp(c, k, 2 * (i + j) + 2, 0)
        vr = dfa * gb * gc
        if i > 0:
            vr = vr * hb ** (i - 1)
        if i + j > 0:
            vr = vr * hc ** (i + j - 1)
        tb = dgb * hb ** i
        if i > 0:
            tb = tb - 0.5 * i * gb * hb ** (i - 1)
        if i + j > 0:
            tb = tb * hc ** (i + j - 1)
        tb = fa * tb * gc
        vs = 0.5 * (1.0 + a) * vr + tb
        tc = dgc * hc ** (i + j)
        if i + j > 0:
            tc = tc - 0.5 * (i + j) * gc * hc ** (i + j - 1)
        vt = 0.5 * (1.0 + a) * vr + 0.5 * (1.0 + b) * tb + fa * gb * tc * hb ** i
        scale = 2.0 ** (2 * i + j + 1.5)
        out[0][:, m], out[1][:, m], out[2][:, m] = scale * vr, scale * vs, scale * vt
    return tuple(out)


def _npts(order: int) -> int:
    return order // 2 + 2


def triangle_rule(order: int):
    """Collapsed Gauss rule on the bi-unit triangle (area 2)."""
    n = _npts(order)
    xa, wa = roots_jacobi(n, 0.0, 0.0)
    xb, wb = roots_jacobi(n, 1.0, 0.0)
    A, B = np.meshgrid(xa, xb, indexing="ij")
    W = np.outer(wa, wb) / 2.0
    r = (1.0 + A) * (1.0 - B) / 2.0 - 1.0
    return np.stack([r.ravel(), B.ravel()], axis=1), W.ravel()


def tet_rule(order: int):
    """Collapsed Gauss rule on the bi-unit tetrahedron (volume 4/3)."""
    n = _npts(order)
    xa, wa = roots_jacobi(n, 0.0, 0.0)
    xb, wb = roots_jacobi(n, 1.0, 0.0)
    xc, wc = roots_jacobi(n, 2.0, 0.0)
    A, B, C = np.meshgrid(xa, xb, xc, indexing="ij")
    W = wa[:, None, None] * wb[None, :, None] * wc[None, None, :] / 8.0
    r = (1.0 + A) * (1.0 - B) * (1.0 - C) / 4.0 - 1.0
    s = (1.0 + B) * (1.0 - C) / 2.0 - 1.0
    return np.stack([r.ravel(), s.ravel(), C.ravel()], axis=1), W.ravel()
