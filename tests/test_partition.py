"""Element partition + face-trace halo: host logic on CPU (plans, a real
2-process gloo exchange) and bitwise partition invariance of the kernels on one GPU."""

import os

import numpy as np
import pytest

from paper_1512_06025_b200 import mesh as msh
from paper_1512_06025_b200.bernstein import BernsteinRefOps
from paper_1512_06025_b200.multiindex import face_permutation_table
from paper_1512_06025_b200.partition import HaloExchanger, build_halo_plan, pack_traces_reference, slab_ranges


def expected_neighbour_reads(m, q, N, k, f):
    """What the single-domain kernel reads for face (k, f): the neighbour's trace,
    permuted into k's face-point order (reference gather, mesh.py:158-188)."""
    ops = BernsteinRefOps.build(N)
    g, _ = msh.build_trace_maps(m, ops.trace, ops.Np)
    return q.reshape(4, -1)[:, g[k, f]]


def halo_reads(plan, recv, N, k_loc, f):
    """What the partitioned kernel reads: recv[:, slot, ptab[perm][m]]."""
    code = int(plan.code[k_loc, f]) & 0xFF
    s = (code >> 2) & 7
    slot = int(plan.nbr[k_loc, f])
    return recv[:, slot, face_permutation_table(N)[s]]


@pytest.mark.parametrize("P", [2, 3, 4])
def test_plan_roundtrip_matches_single_domain_gather(P):
    m = msh.cube_mesh(3)
    N = 3
    ops = BernsteinRefOps.build(N)
    q = np.random.default_rng(1).standard_normal((4, m.K, ops.Np))
    ranges = slab_ranges(m.K, P, align=6 * 9)
    plans = [build_halo_plan(m, P, r, ranges) for r in range(P)]
    # every face is owned exactly once; local neighbour ids stay inside the slab
    assert sum(p.n_local for p in plans) == m.K
    for p in plans:
        loc = ((p.code.astype(np.int32) >> 6) & 1) == 0
        assert np.all((p.nbr[loc] >= 0) & (p.nbr[loc] < p.n_local))
    # simulated exchange with the host packer
    for p in plans:
        recv = np.zeros((4, max(p.nhalo, 1), ops.Nfp))
        for s, cnt in p.recv_count.items():
            sender = plans[s]
            faces = sender.send[p.rank]
            assert len(faces) == cnt
            qs = q[:, sender.k0:sender.k1]
            recv[:, p.recv_offset[s]:p.recv_offset[s] + cnt] = pack_traces_reference(qs, faces, ops.trace)
        kk, ff = np.nonzero(((p.code.astype(np.int32) >> 6) & 1) == 1)
        assert len(kk) == p.nhalo
        for k_loc, f in zip(kk, ff):
            got = halo_reads(p, recv, N, k_loc, f)
            want = expected_neighbour_reads(m, q, N, p.k0 + k_loc, f)
            assert np.array_equal(got, want)


def test_launch_ranges_cover_slab():
    m = msh.cube_mesh(12)                      # 3 x-slabs of cells per rank
    ranges = slab_ranges(m.K, 4, align=6 * 144)
    for r in range(4):
        p = build_halo_plan(m, 4, r, ranges)
        inner, outer = p.launch_ranges()
        cover = np.zeros(p.n_local, dtype=int)
        for a, b in ([inner] if inner else []) + outer:
            cover[a:b] += 1
        assert np.all(cover == 1)
        if inner:
            assert not np.isin(np.arange(*inner), p.halo_elems).any()
            assert inner[1] - inner[0] >= p.n_local // 4    # the middle slab overlaps the exchange


@pytest.mark.parametrize("dims,world,xblock", [((4, 2, 3), 2, 1), ((6, 3, 2), 3, 1), ((5, 2, 2), 4, 1),
                                               ((3, 1, 1), 3, 1), ((8, 2, 3), 2, 2), ((6, 3, 2), 2, 3),
                                               ((9, 2, 2), 2, 4)])
def test_box_halo_plan_matches_host_plan(dims, world, xblock):
    """The closed-form plan of a device-built box slab (no host mesh) equals build_halo_plan's, in the
    reference element order and in the x-blocked order."""
    from paper_1512_06025_b200.mesh_device import BoxMesh
    from paper_1512_06025_b200.partition import box_halo_plan

    box = BoxMesh(*dims, xblock=xblock)
    m = box.to_mesh()
    plane = dims[1] * dims[2]
    ranges = [tuple(6 * x * plane for x in box.slab_layers(r, world)) for r in range(world)]
    for r in range(world):
        h, c = build_halo_plan(m, world, r, ranges), box_halo_plan(box, world, r)
        assert (h.k0, h.k1, h.nhalo) == (c.k0, c.k1, c.nhalo)
        assert h.recv_count == c.recv_count and h.recv_offset == c.recv_offset
        assert set(h.send) == set(c.send) and all(np.array_equal(h.send[p], c.send[p]) for p in h.send)
        assert np.array_equal(h.halo_elems, c.halo_elems)
        assert c.launch_ranges() == h.launch_ranges()


def _gloo_worker(rank, world, port, out, box_dims=None):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = 2
        ops = BernsteinRefOps.build(N)
        if box_dims is None:
            m = msh.cube_mesh(3)
            plan = build_halo_plan(m, world, rank)
            ex_plan = plan
        else:   # exchange with the closed-form box plan, verify with the host mesh's plan
            from paper_1512_06025_b200.mesh_device import BoxMesh
            from paper_1512_06025_b200.partition import box_halo_plan

            box = BoxMesh(*box_dims)
            m = box.to_mesh()
            plane = box.ny * box.nz
            ranges = [tuple(6 * x * plane for x in box.slab_layers(r, world)) for r in range(world)]
            plan = build_halo_plan(m, world, rank, ranges)
            ex_plan = box_halo_plan(box, world, rank)
        q = np.random.default_rng(7).standard_normal((4, m.K, ops.Np))
        trace = torch.as_tensor(ops.trace)

        def packer(qt, faces, outb):
            outb.copy_(qt[:, faces[:, 0].long()[:, None], trace[faces[:, 1].long()]])

        ex = HaloExchanger(ex_plan, ops.Nfp, torch.float64, "cpu", packer)
        ql = torch.as_tensor(q[:, plan.k0:plan.k1].copy())
        ex.wait(ex.post(ql))
        recv = ex.recv.numpy()
        kk, ff = np.nonzero(((plan.code.astype(np.int32) >> 6) & 1) == 1)
        ok = all(np.array_equal(halo_reads(plan, recv, N, k, f),
                                expected_neighbour_reads(m, q, N, plan.k0 + k, f)) for k, f in zip(kk, ff))
        out[rank] = int(ok and len(kk) > 0)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,box_dims", [(2, None), (2, (4, 3, 2)), (3, (5, 2, 3))])
def test_gloo_halo_exchange(world, box_dims):
    """world-size 2/3 gloo runs of the one-message-per-peer exchange (host-mesh plan, and the
    closed-form plan of a device-built box slab; the middle rank of 3 has two peers)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = 29500 + (os.getpid() % 1000) + 7 * world + (0 if box_dims is None else 3)
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, out, box_dims)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert dict(out) == {r: 1 for r in range(world)}


# ---------------------------------------------------------------------------- GPU
class _FakeWorld:
    """In-process communicator: P ranks on one GPU exchange by device copies."""

    def __init__(self):
        self.sends, self.recvs = {}, {}

    def flush(self):
        for key, rs in self.recvs.items():
            for s, r in zip(self.sends.get(key, []), rs):
                r.copy_(s)
        self.sends, self.recvs = {}, {}


class _FakeDist:
    def __init__(self, world, rank):
        self.world, self.rank = world, rank

    @staticmethod
    def P2POp(op, t, peer):
        return (op, t, peer)

    def isend(self, *a):
        raise AssertionError("not called directly")

    def irecv(self, *a):
        raise AssertionError("not called directly")

    def batch_isend_irecv(self, ops):
        for op, t, peer in ops:
            if op == self.isend:
                self.world.sends.setdefault((self.rank, peer), []).append(t)
            else:
                self.world.recvs.setdefault((peer, self.rank), []).append(t)
        world = self.world

        class _Req:
            def wait(self):
                world.flush()

        return [_Req()]


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3])
@pytest.mark.parametrize("dname", ["f64", "f32"])
@pytest.mark.parametrize("N", [4, 9])
def test_partitioned_step_bitwise_equals_single_domain(P, dname, N):
    import torch

    from paper_1512_06025_b200 import Materials, WaveSystem, stable_dt
    from paper_1512_06025_b200.dist import DistWaveSystem
    from paper_1512_06025_b200.solver import RK4A, RK4B

    dtype = np.float64 if dname == "f64" else np.float32
    m = msh.cube_mesh(6)
    ops = BernsteinRefOps.build(N)
    mat = Materials.homogeneous(m.K)
    single = WaveSystem(m, ops, mat, dtype)
    g = torch.Generator(device="cuda").manual_seed(3)
    q = torch.randn((4, m.K, single.Np), dtype=single.torch_dtype, device="cuda", generator=g)
    res0 = torch.randn_like(q)
    dt = stable_dt(m, N, 1.0)
    q_ref, res_ref = torch.empty_like(q), res0.clone()
    single.stage_into(q, q_ref, res_ref, RK4A[2], RK4B[2], dt, "optimal")

    world = _FakeWorld()
    parts = [DistWaveSystem(m, ops, mat, dtype, r, P, dist=_FakeDist(world, r), align=6 * 36) for r in range(P)]
    qs = [q[:, p.plan.k0:p.plan.k1].contiguous() for p in parts]
    rs = [res0[:, p.plan.k0:p.plan.k1].contiguous() for p in parts]
    outs = [torch.empty_like(x) for x in qs]
    reqs = [p.post(x) for p, x in zip(parts, qs)]
    for p, x, o, r, rq in zip(parts, qs, outs, rs, reqs):
        p.stage_into(x, o, r, RK4A[2], RK4B[2], dt, "optimal", reqs=rq)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs, dim=1), q_ref)
    assert torch.equal(torch.cat(rs, dim=1), res_ref)
