"""Device-built box meshes (bbdg_ctx_set_box_mesh): the records the closed-form kernel writes
equal those uploaded from the host mesh (connectivity bit-exact, geometry to rounding), slab
contexts reproduce build_halo_plan's halo slots, and stages on them match the oracle and the
single-domain run bitwise."""

import ctypes as C

import numpy as np
import pytest

import bbdg_oracle as orc
from conftest import TOL, rel_l2
from paper_1512_06025_b200 import BernsteinRefOps, Materials, WaveSystem, _lib, stable_dt
from paper_1512_06025_b200.mesh_device import BoxMesh
from paper_1512_06025_b200.partition import build_halo_plan

pytestmark = pytest.mark.gpu
DT = {"f64": np.float64, "f32": np.float32}


def records(sy):
    K = sy.K
    geo = np.empty((K, 36), dtype=sy.dtype)
    nbr = np.empty((K, 4), dtype=np.int32)
    code = np.empty(K, dtype=np.int32)
    _lib.check(_lib.load().bbdg_ctx_read_records(sy._ctx, geo.ctypes.data, nbr.ctypes.data, code.ctypes.data),
               "read records")
    return geo, nbr, code


@pytest.mark.parametrize("dims,xblock", [((1, 1, 1), 1), ((3, 2, 4), 1), ((5, 3, 2), 1), ((5, 3, 2), 2),
                                         ((7, 2, 3), 4)])
@pytest.mark.parametrize("dname", ["f64", "f32"])
def test_box_records_match_host_upload(dims, xblock, dname):
    box = BoxMesh(*dims, lo=(-1.0, 0.0, 0.5), hi=(2.0, 1.0, 3.0), xblock=xblock)
    m = box.to_mesh()
    ops = BernsteinRefOps.build(2)
    a = WaveSystem(m, ops, Materials.homogeneous(m.K, 2.0, 0.5), dtype=DT[dname])
    b = WaveSystem(box, ops, Materials.homogeneous(m.K, 2.0, 0.5), dtype=DT[dname])
    ga, na, ca = records(a)
    gb, nb, cb = records(b)
    assert np.array_equal(na, nb) and np.array_equal(ca, cb)
    scale = np.abs(ga).max(axis=0) + 1e-30
    assert (np.abs(ga - gb) / scale).max() < (4e-15 if dname == "f64" else 4e-7)
    assert box.h_min == pytest.approx(m.h_min, rel=1e-14) and box.K == m.K


@pytest.mark.parametrize("world,xblock", [(2, 1), (3, 1), (3, 2)])
def test_box_slab_connectivity_matches_host_plan(world, xblock):
    box = BoxMesh(6, 3, 2, xblock=xblock)
    m = box.to_mesh()
    plane = box.ny * box.nz
    ranges = [tuple(6 * x * plane for x in box.slab_layers(r, world)) for r in range(world)]
    ops = BernsteinRefOps.build(3)
    for r in range(world):
        plan = build_halo_plan(m, world, r, ranges)
        sy = WaveSystem(box.slab(r, world), ops, Materials.homogeneous(box.K_total), dtype=np.float64)
        _, nbr, code = records(sy)
        packed = (plan.code.astype(np.int32) & 0xFF)
        want = packed[:, 0] | (packed[:, 1] << 8) | (packed[:, 2] << 16) | (packed[:, 3] << 24)
        assert np.array_equal(nbr, plan.nbr) and np.array_equal(code, want.astype(np.int32)), r


@pytest.mark.parametrize("N", [1, 4, 9])
@pytest.mark.parametrize("dname", ["f64", "f32"])
def test_box_stage_matches_oracle(N, dname):
    from test_gpu_parity import stage_vs_oracle

    box = BoxMesh(4, 3, 3, xblock=2)
    dtype = DT[dname]
    sy = WaveSystem(box, BernsteinRefOps.build(N), Materials.homogeneous(box.K), dtype=dtype, legacy_records=False)
    m = box.to_mesh()
    ref = orc.OracleSystem(orc.mesh_arrays(m), orc.bernstein_tables(N), np.ones(m.K), np.ones(m.K), dtype)
    rng = np.random.default_rng(N)
    q = rng.standard_normal((4, m.K, sy.Np)).astype(dtype)
    stage_vs_oracle(sy, ref, q, rng.standard_normal(q.shape).astype(dtype), stable_dt(m, N, 1.0), "optimal")
    with pytest.raises(_lib.BBDGError):   # fused record only: the ELL kernel has no legacy records
        sy.surface_rhs(__import__("paper_1512_06025_b200").FieldState(q, "bernstein"), "ell")


@pytest.mark.parametrize("P,xblock", [(2, 1), (3, 1), (2, 3)])
def test_box_partitioned_stage_bitwise(P, xblock):
    import torch

    from paper_1512_06025_b200.dist import DistWaveSystem
    from paper_1512_06025_b200.solver import RK4A, RK4B
    from test_partition import _FakeDist, _FakeWorld

    box = BoxMesh(6, 4, 3, xblock=xblock)
    N = 5
    ops = BernsteinRefOps.build(N)
    mat = Materials.homogeneous(box.K_total)
    single = WaveSystem(box, ops, mat, np.float32)
    g = torch.Generator(device="cuda").manual_seed(5)
    q = torch.randn((4, box.K, single.Np), dtype=torch.float32, device="cuda", generator=g)
    res0 = torch.randn_like(q)
    dt = stable_dt(box, N, 1.0)
    q_ref, res_ref = torch.empty_like(q), res0.clone()
    single.stage_into(q, q_ref, res_ref, RK4A[3], RK4B[3], dt, "optimal")
    world = _FakeWorld()
    parts = [DistWaveSystem(box, ops, mat, np.float32, r, P, dist=_FakeDist(world, r)) for r in range(P)]
    qs = [q[:, p.plan.k0:p.plan.k1].contiguous() for p in parts]
    rs = [res0[:, p.plan.k0:p.plan.k1].contiguous() for p in parts]
    outs = [torch.empty_like(x) for x in qs]
    reqs = [p.post(x) for p, x in zip(parts, qs)]
    for p, x, o, r, rq in zip(parts, qs, outs, rs, reqs):
        p.stage_into(x, o, r, RK4A[3], RK4B[3], dt, "optimal", reqs=rq)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(outs, dim=1), q_ref)
    assert torch.equal(torch.cat(rs, dim=1), res_ref)
