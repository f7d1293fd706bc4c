"""Element partitioning and face-trace halo exchange.

The reference is single-process (no domain decomposition).  Here a mesh is
split into contiguous element slabs -- ``cube_mesh`` numbers elements
x-slab-major (reference ``mesh.py:143-154``), so contiguous ranges are
geometric slabs with <= 2 neighbouring ranks.  Once per RK stage each rank
sends, for every face it shares with another rank, the four field traces of
its own face (in that face's canonical point order) and receives the remote
traces into a ``(4, nhalo, Nfp)`` halo buffer.  Faces flagged with the halo
bit read that buffer through the same vertex-permutation table as local
neighbours, so the arithmetic per element is unchanged and the partitioned
result is bitwise equal to the single-domain one.

Both sides derive the same ordering independently: the cut faces between a
receiver r and a sender s are sorted by (receiver element, receiver face);
the receiver's halo slots follow that order (peers in ascending rank) and the
sender packs its matching faces in the same order.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def slab_ranges(K: int, P: int, align: int = 1) -> list[tuple[int, int]]:
    """P contiguous element ranges of (nearly) equal size, cut at multiples of `align`."""
    if P < 1 or K < P:
        raise ValueError("need 1 <= P <= K")
    cuts = [0]
    for r in range(1, P):
        c = (K * r) // P
        c = min(K, max(cuts[-1] + 1, (c // align) * align if align > 1 else c))
        cuts.append(c)
    cuts.append(K)
    return [(cuts[r], cuts[r + 1]) for r in range(P)]


@dataclass
class HaloPlan:
    rank: int
    world: int
    k0: int
    k1: int
    nbr: np.ndarray                    # (n_loc, 4) int32: local element, or halo slot
    code: np.ndarray                   # (n_loc, 4) int8: f2 | perm<<2 | boundary<<5 | halo<<6
    send: dict = field(default_factory=dict)        # peer -> (n, 2) int32 (local elem, face)
    recv_count: dict = field(default_factory=dict)  # peer -> n
    recv_offset: dict = field(default_factory=dict)  # peer -> first halo slot
    nhalo: int = 0
    halo_elems: np.ndarray = None      # local elements with at least one halo face

    @property
    def n_local(self) -> int:
        return self.k1 - self.k0

    def launch_ranges(self):
        """(interior range or None, halo ranges): the interior is the largest run of local
        elements without halo faces, launched while the exchange is in flight."""
        n = self.n_local
        if self.nhalo == 0:
            return (0, n), []
        idx = np.asarray(self.halo_elems)
        bounds = np.concatenate([[-1], idx, [n]])
        gaps = bounds[1:] - bounds[:-1] - 1
        j = int(np.argmax(gaps))
        if gaps[j] <= 0:
            return None, [(0, n)]
        a, b = int(bounds[j] + 1), int(bounds[j + 1])
        rng = [r for r in ((0, a), (b, n)) if r[1] > r[0]]
        return (a, b), rng


def build_halo_plan(mesh, world: int, rank: int, ranges=None) -> HaloPlan:
    """Local connectivity + send/recv lists of `rank` for a slab partition of `mesh`."""
    K = mesh.K
    ranges = ranges or slab_ranges(K, world)
    starts = np.array([r[0] for r in ranges])
    k0, k1 = ranges[rank]
    owner = np.searchsorted(starts, np.arange(K), side="right") - 1
    etoe, etof = mesh.etoe, mesh.etof
    perm = mesh.face_perm.astype(np.int32)
    bnd = mesh.boundary
    loc = np.arange(k0, k1)
    nbr_g = etoe[loc]
    cut = (~bnd[loc]) & (owner[nbr_g] != rank)                      # (n_loc, 4)
    code = (etof[loc].astype(np.int32) | (perm[loc] << 2) | (bnd[loc].astype(np.int32) << 5)
            | (cut.astype(np.int32) << 6))
    nbr = np.where(bnd[loc], loc[:, None], nbr_g) - k0
    plan = HaloPlan(rank, world, k0, k1, nbr.astype(np.int32), code.astype(np.int8))
    # receive side: my cut faces grouped by the owner of the neighbour, sorted by (my elem, face)
    ke, fe = np.nonzero(cut)
    peers = owner[nbr_g[ke, fe]]
    slot = 0
    for s in sorted(set(peers.tolist())):
        sel = peers == s
        order = np.lexsort((fe[sel], ke[sel]))
        kk, ff = ke[sel][order], fe[sel][order]
        plan.recv_offset[s] = slot
        plan.recv_count[s] = len(kk)
        plan.nbr[kk, ff] = slot + np.arange(len(kk), dtype=np.int32)
        slot += len(kk)
    plan.nhalo = slot
    plan.halo_elems = np.unique(ke)
    # send side: for each peer r, the faces r receives from me, in r's order
    for r in range(world):
        if r == rank:
            continue
        a, b = ranges[r]
        rl = np.arange(a, b)
        nb = etoe[rl]
        rc = (~bnd[rl]) & (owner[nb] == rank)
        re_, rf = np.nonzero(rc)
        if len(re_) == 0:
            continue
        order = np.lexsort((rf, re_))
        re_, rf = re_[order], rf[order]
        mine_e = etoe[rl[re_], rf] - k0
        mine_f = etof[rl[re_], rf]
        plan.send[r] = np.stack([mine_e, mine_f], axis=1).astype(np.int32)
    return plan


def pack_traces_reference(q: np.ndarray, faces: np.ndarray, trace: np.ndarray) -> np.ndarray:
    """Host restatement of bbdg_halo_pack for tests: (4, K, Np) x (n,2) -> (4, n, Nfp)."""
    return q[:, faces[:, 0][:, None], trace[faces[:, 1]]]


class HaloExchanger:
    """Posts one stage's face-trace exchange through torch.distributed (NCCL on the GPU path,
    gloo in the CPU tests): ONE send and ONE receive per peer and direction -- the packed
    (4, n, Nfp) trace block -- grouped in a single batch_isend_irecv.  `packer(q, faces, out)`
    fills a send buffer; `wait` completes the receives and scatters each peer's block into its
    slots of the (4, nhalo, Nfp) halo array the kernels read.  All four fields travel so the
    receiver's flux arithmetic is exactly the single-domain one (bitwise partition invariance)."""

    def __init__(self, plan: HaloPlan, Nfp: int, dtype, device, packer, dist=None):
        import torch

        self.plan = plan
        self.torch = torch
        self.dist = dist or torch.distributed
        self.packer = packer
        self.recv = torch.zeros((4, max(plan.nhalo, 1), Nfp), dtype=dtype, device=device)
        self.send_faces = {r: torch.as_tensor(f, device=device) for r, f in plan.send.items()}
        self.send_bufs = {r: torch.empty((4, len(f), Nfp), dtype=dtype, device=device)
                          for r, f in plan.send.items()}
        self.recv_bufs = {r: torch.empty((4, n, Nfp), dtype=dtype, device=device)
                          for r, n in plan.recv_count.items()}

    def post(self, q):
        """Pack and post all sends/receives; returns the requests (wait() before use)."""
        P2POp = self.dist.P2POp
        ops = []
        for r, faces in self.send_faces.items():
            self.packer(q, faces, self.send_bufs[r])
        for r in sorted(set(self.plan.recv_count) | set(self.send_faces)):
            if r in self.send_faces:
                ops.append(P2POp(self.dist.isend, self.send_bufs[r], r))
            if r in self.recv_bufs:
                ops.append(P2POp(self.dist.irecv, self.recv_bufs[r], r))
        if not ops:
            return []
        return self.dist.batch_isend_irecv(ops)

    def wait(self, reqs):
        for r in reqs:
            r.wait()
        for r, buf in self.recv_bufs.items():
            o, n = self.plan.recv_offset[r], self.plan.recv_count[r]
            self.recv[:, o:o + n].copy_(buf)


def box_halo_plan(box, world: int, rank: int) -> HaloPlan:
    """The HaloPlan of `rank` for the x-layer slab partition of a device-built box (mesh_device.
    BoxMesh), in closed form -- the same slots and send lists build_halo_plan derives from a host
    mesh, without one.  Per interface of ny nz cells, the cut faces are the face opposite path
    vertex 3 of tets 3 and 5 of the slab's first layer (neighbour: layer - 1) and the face opposite
    path vertex 0 of tets 0 and 1 of its last layer (neighbour: layer + 1); each such tet has one
    cut face, so (receiver element, face) order is cell order, then tet.  ``nbr`` / ``code`` stay
    None: bbdg_ctx_set_box_mesh computes the local connectivity on the device."""
    a, b = box.slab_layers(rank, world)
    plane = box.ny * box.nz
    jk = np.arange(plane, dtype=np.int64)
    cy, cz = jk // box.nz, jk % box.nz
    owner = [box.slab_layers(r, world) for r in range(world)]

    def owner_of(layer):
        return next(r for r, (x0, x1) in enumerate(owner) if x0 <= layer < x1)

    plan = HaloPlan(rank, world, 6 * a * plane, 6 * b * plane, None, None)
    first = box.local_element(np.full(plane, a), cy, cz, 0, a)       # tet 0 of the first layer's cells
    last = box.local_element(np.full(plane, b - 1), cy, cz, 0, a)    # ... of the last layer's cells
    slot, halo = 0, []
    if a > 0:
        left = owner_of(a - 1)
        plan.recv_offset[left], plan.recv_count[left] = slot, 2 * plane
        slot += 2 * plane
        halo.append(np.stack([first + 3, first + 5], 1).ravel())
        # the left peer receives (its last layer, tets 0 and 1, face 0) <- mine (tets 3 and 5, face 3)
        plan.send[left] = np.stack([np.stack([first + 3, first + 5], 1).ravel(),
                                    np.full(2 * plane, 3)], 1).astype(np.int32)
    if b < box.nx:
        right = owner_of(b)
        plan.recv_offset[right], plan.recv_count[right] = slot, 2 * plane
        slot += 2 * plane
        halo.append(np.stack([last, last + 1], 1).ravel())
        plan.send[right] = np.stack([np.stack([last, last + 1], 1).ravel(), np.zeros(2 * plane, dtype=np.int64)],
                                    1).astype(np.int32)
    plan.nhalo = slot
    plan.halo_elems = np.unique(np.concatenate(halo)) if halo else np.zeros(0, dtype=np.int64)
    return plan
