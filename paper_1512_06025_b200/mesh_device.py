"""Box meshes built on the GPU: HBM-filling meshes in seconds.

``box_mesh_device`` produces exactly the mesh of ``mesh.box_mesh`` (same
vertices, tets, element order, connectivity and vertex-permutation codes;
geometry equal to rounding) with every per-element array computed by
vectorised device code, then hands the reference ``Mesh`` data contract back
as host arrays (``WaveSystem`` and the C ABI take host geometry).  The
reference builds 105k tets in 66 s and the vectorised host builder 1.3 M in
7 s; here 13 M tets take a few seconds.  Setup only -- not on the per-step
hot path.
"""

from __future__ import annotations

import numpy as np

from .mesh import Mesh, _AXIS_PERMS, _FV, _PERM_CODE
from .multiindex import REFERENCE_TET_VOLUME


def _lexsort_rows(torch, key):
    """Indices sorting the rows of key (n, 3) lexicographically (stable sorts, last column first)."""
    order = torch.argsort(key[:, 2], stable=True)
    order = order[torch.argsort(key[order, 1], stable=True)]
    return order[torch.argsort(key[order, 0], stable=True)]


def box_mesh_device(nx: int, ny: int, nz: int, lo=(-0.5, -0.5, -0.5), hi=(0.5, 0.5, 0.5), device="cuda") -> Mesh:
    """6 nx ny nz Kuhn tetrahedra, x-slab-major (as mesh.box_mesh), built on `device`."""
    import torch

    if min(nx, ny, nz) < 1:
        raise ValueError("need at least one cell per axis")
    f64 = dict(dtype=torch.float64, device=device)
    i64 = dict(dtype=torch.int64, device=device)
    lo_, hi_ = np.asarray(lo, dtype=float), np.asarray(hi, dtype=float)
    # the axis coordinates come from numpy.linspace so vertices match mesh.box_mesh bit for bit
    axes = [torch.as_tensor(np.linspace(lo_[i], hi_[i], d + 1), **f64) for i, d in enumerate((nx, ny, nz))]
    X, Y, Z = torch.meshgrid(*axes, indexing="ij")
    vertices = torch.stack([X.reshape(-1), Y.reshape(-1), Z.reshape(-1)], dim=1)
    ci, cj, ck = torch.meshgrid(torch.arange(nx, **i64), torch.arange(ny, **i64), torch.arange(nz, **i64),
                                indexing="ij")
    corner = torch.stack([ci.reshape(-1), cj.reshape(-1), ck.reshape(-1)], dim=1)
    paths = []
    for perm in _AXIS_PERMS:
        cur, pts = [0, 0, 0], [[0, 0, 0]]
        for ax in perm:
            cur = list(cur)
            cur[ax] = 1
            pts.append(cur)
        paths.append(pts)
    paths = torch.tensor(paths, **i64)                                   # (6, 4, 3)
    p = corner[:, None, None, :] + paths[None]                          # (n^3, 6, 4, 3)
    tets = ((p[..., 0] * (ny + 1) + p[..., 1]) * (nz + 1) + p[..., 2]).reshape(-1, 4)
    del p, corner
    # orientation (mesh._orient)
    v = vertices[tets]
    neg = torch.linalg.det(v[:, 1:] - v[:, :1]) < 0
    t1, t2 = tets[:, 1].clone(), tets[:, 2].clone()
    tets[:, 1] = torch.where(neg, t2, t1)
    tets[:, 2] = torch.where(neg, t1, t2)
    # geometry (mesh._geometry)
    v = vertices[tets]                                                  # (K, 4, 3)
    dxdr = 0.5 * (v[:, 1:] - v[:, :1]).transpose(1, 2)
    jac = torch.linalg.det(dxdr)
    if bool((jac <= 1.0e-14).any()):
        raise ValueError("degenerate or negatively oriented tetrahedron")
    rst_dx = torch.linalg.inv(dxdr)
    centroid = v.mean(dim=1)
    FV = torch.as_tensor(_FV, **i64)
    fv = v[:, FV]                                                       # (K, 4, 3, 3)
    avec = 0.5 * torch.linalg.cross(fv[:, :, 1] - fv[:, :, 0], fv[:, :, 2] - fv[:, :, 0], dim=-1)
    area = torch.linalg.norm(avec, dim=2)
    n = avec / area[..., None]
    outward = ((n * (fv.mean(dim=2) - centroid[:, None])).sum(-1)) > 0
    n = torch.where(outward[..., None], n, -n)
    jf = area / 2.0
    h = 6.0 * jac * REFERENCE_TET_VOLUME / (2.0 * jf.sum(dim=1))
    del v, fv, avec, dxdr
    # connectivity (mesh._connectivity): match faces by sorted vertex triples
    K = tets.shape[0]
    fverts = tets[:, FV].reshape(K * 4, 3)
    key = torch.sort(fverts, dim=1).values
    order = _lexsort_rows(torch, key)
    ks = key[order]
    same = (ks[1:] == ks[:-1]).all(dim=1)
    if bool((same[1:] & same[:-1]).any()):
        raise ValueError("non-manifold mesh: a face is shared by more than two tets")
    a, b = order[:-1][same], order[1:][same]
    nbr = torch.arange(K * 4, **i64)
    nbr[a] = b
    nbr[b] = a
    del key, ks, order, same, a, b
    etoe, etof = (nbr // 4).reshape(K, 4), (nbr % 4).reshape(K, 4)
    w = fverts[nbr]
    sig = torch.argmax((fverts[:, :, None] == w[:, None, :]).to(torch.int32), dim=2)
    code = torch.zeros(K * 4, dtype=torch.int8, device=device)
    for perm, s in _PERM_CODE.items():
        code[(sig == torch.as_tensor(perm, **i64)).all(dim=1)] = s
    del w, sig, fverts, nbr

    def host(x):
        return x.cpu().numpy()

    return Mesh(host(vertices), host(tets), host(jac), host(rst_dx), host(n), host(jf), host(etoe), host(etof),
                host(h), host(code.reshape(K, 4)))


def cube_mesh_device(n: int, lo=(-0.5, -0.5, -0.5), hi=(0.5, 0.5, 0.5), device="cuda") -> Mesh:
    return box_mesh_device(n, n, n, lo, hi, device)


class BoxMesh:
    """A box of nx x ny x nz cells, 6 Kuhn tets each, that is never materialised on the host:
    ``WaveSystem`` expands it on the device with ``bbdg_ctx_set_box_mesh`` (closed-form index
    arithmetic, one thread per element).  Same elements, order, connectivity and geometry as
    ``mesh.box_mesh`` / ``cube_mesh`` (reference mesh.py:127-155).  ``slab(rank, world)`` is the
    rank's contiguous range of x cell layers (x-slab-major element order), so every rank of a
    partitioned run builds only its own elements.

    Exposes the ``Mesh`` attributes the time stepper needs (``K``, ``h_min``, ``h_max``,
    ``volume``); ``to_mesh()`` materialises the full host mesh (small boxes: tests, functionals).
    """

    def __init__(self, nx: int, ny: int, nz: int, lo=(-0.5, -0.5, -0.5), hi=(0.5, 0.5, 0.5), cx0: int = 0,
                 cx1: int | None = None, xblock: int = 1):
        if min(nx, ny, nz) < 1 or xblock < 1:
            raise ValueError("need at least one cell per axis")
        self.nx, self.ny, self.nz = int(nx), int(ny), int(nz)
        self.xblock = int(xblock)   # element order: slabs of xblock x-layers (1 = reference cube_mesh order)
        self.lo = tuple(float(x) for x in lo)
        self.hi = tuple(float(x) for x in hi)
        self.cx0 = int(cx0)
        self.cx1 = self.nx if cx1 is None else int(cx1)
        if not 0 <= self.cx0 < self.cx1 <= self.nx:
            raise ValueError("slab layers must satisfy 0 <= cx0 < cx1 <= nx")
        if self.cx0 % self.xblock or (self.cx1 % self.xblock and self.cx1 != self.nx):
            raise ValueError("slab layers must be multiples of the x-blocking")
        # every cell is the same box: the 6 tets of one cell give the exact h range
        from .mesh import box_mesh

        step = [(h - l) / n for l, h, n in zip(self.lo, self.hi, (self.nx, self.ny, self.nz))]
        cell = box_mesh(1, 1, 1, lo=(0.0, 0.0, 0.0), hi=tuple(step))
        self.h_min, self.h_max = cell.h_min, cell.h_max
        self.cell_jac = float(cell.jac[0])   # every Kuhn tet of a box has the same volume

    @classmethod
    def cube(cls, n: int, lo=(-0.5, -0.5, -0.5), hi=(0.5, 0.5, 0.5)) -> "BoxMesh":
        return cls(n, n, n, lo, hi)

    @property
    def K(self) -> int:
        """Elements of this slab (the whole box unless sliced)."""
        return 6 * (self.cx1 - self.cx0) * self.ny * self.nz

    @property
    def K_total(self) -> int:
        return 6 * self.nx * self.ny * self.nz

    @property
    def k0(self) -> int:
        return 6 * self.cx0 * self.ny * self.nz

    @property
    def volume(self) -> float:
        return float(np.prod(np.subtract(self.hi, self.lo)))

    def slab_layers(self, rank: int, world: int) -> tuple[int, int]:
        """Cell layers [a, b) of `rank`: near-equal shares, cut at multiples of the x-blocking."""
        nblk = -(-self.nx // self.xblock)
        if not 1 <= world <= nblk:
            raise ValueError("need 1 <= world <= number of x-blocks")
        a, b = (nblk * rank) // world * self.xblock, (nblk * (rank + 1)) // world * self.xblock
        return a, min(b, self.nx)

    def slab(self, rank: int, world: int) -> "BoxMesh":
        a, b = self.slab_layers(rank, world)
        return BoxMesh(self.nx, self.ny, self.nz, self.lo, self.hi, a, b, self.xblock)

    def local_element(self, cx, cy, cz, t, cx0: int | None = None):
        """Element index (counted from layer cx0, default this slab's) of tet t of cell (cx, cy, cz)."""
        cx, cy, cz = (np.asarray(v, dtype=np.int64) for v in (cx, cy, cz))
        xb = self.xblock
        s = cx // xb
        ts = np.minimum(xb, self.nx - s * xb)
        lin = s * xb * self.ny * self.nz + (cy * self.nz + cz) * ts + (cx - s * xb)
        base = (self.cx0 if cx0 is None else cx0) * self.ny * self.nz
        return (lin - base) * 6 + t

    def to_mesh(self) -> Mesh:
        from .mesh import box_mesh

        return box_mesh(self.nx, self.ny, self.nz, self.lo, self.hi, self.xblock)

    def __repr__(self):
        return (f"BoxMesh({self.nx}x{self.ny}x{self.nz} cells, layers [{self.cx0}, {self.cx1}), xblock={self.xblock}, "
                f"K={self.K})")
