"""Host-pipelined lsrk4_step (bbdg_step_host): a pinned numpy state is copied in,
stepped and copied back chunk by chunk, so the copies overlap the stages.

CPU: the chunk plan (bounds cover [0, K), reach is exact, unbanded numberings
are refused).  GPU: the pipelined step is bitwise equal to the device-resident
step (bbdg_step) -- same kernels, same per-element arithmetic -- for reach 1 and
reach 2 chunkings, and it is actually taken for pinned states.
"""

import numpy as np
import pytest

from paper_1512_06025_b200 import BernsteinRefOps, FieldState, Materials, WaveSystem, cube_mesh, lsrk4_step, stable_dt
from paper_1512_06025_b200.solver import host_chunk_plan


def _check_plan(etoe, bounds, reach):
    K = etoe.shape[0]
    assert bounds[0] == 0 and bounds[-1] == K and np.all(np.diff(bounds) > 0)
    cid = np.searchsorted(bounds, np.arange(K), side="right") - 1
    d = np.abs(cid[etoe] - cid[:, None])
    assert d.max() == reach


def test_chunk_plan_cube_mesh_reach_one():
    m = cube_mesh(40)
    plan = host_chunk_plan(m.etoe, 220, 4)
    assert plan is not None
    bounds, reach = plan
    assert reach == 1 and 30 <= len(bounds) - 1 <= 48
    _check_plan(m.etoe, bounds, reach)


def test_chunk_plan_forced_chunk_and_small_states():
    m = cube_mesh(12)
    assert host_chunk_plan(m.etoe, 20, 8) is None                 # 6.6 MB state: not worth chunking
    bounds, reach = host_chunk_plan(m.etoe, 20, 8, min_state_bytes=0)
    _check_plan(m.etoe, bounds, reach)
    band = int(np.abs(m.etoe - np.arange(m.K)[:, None]).max())
    b2, r2 = host_chunk_plan(m.etoe, 20, 8, min_state_bytes=0, chunk=band // 2 + 1)
    assert r2 == 2
    _check_plan(m.etoe, b2, r2)


def test_chunk_plan_refuses_unbanded_numbering():
    m = cube_mesh(12)
    perm = np.random.default_rng(0).permutation(m.K)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(m.K)
    etoe = inv[m.etoe[perm]]      # elements renumbered at random: neighbours anywhere
    assert host_chunk_plan(etoe, 20, 8, min_state_bytes=0) is None


def test_capi_declares_step_host():
    from pathlib import Path

    h = (Path(__file__).resolve().parents[1] / "include" / "bbdg.h").read_text()
    assert "int bbdg_step_host(" in h


@pytest.mark.gpu
@pytest.mark.parametrize("N,dname,halve", [(3, "f64", False), (5, "f32", False), (5, "f32", True), (9, "f32", False)])
def test_pipelined_step_bitwise_equals_device_step(N, dname, halve):
    import torch

    dtype = np.float64 if dname == "f64" else np.float32
    m = cube_mesh(12)
    sy = WaveSystem(m, BernsteinRefOps.build(N), Materials.homogeneous(m.K), dtype=dtype)
    band = int(np.abs(m.etoe - np.arange(m.K)[:, None]).max())
    sy._chunks = host_chunk_plan(m.etoe, sy.Np, np.dtype(dtype).itemsize, min_state_bytes=0,
                                 chunk=(band // 2 + 1) if halve else None)
    assert sy._chunks is not None and sy._chunks[1] == (2 if halve else 1)
    q0 = np.random.default_rng(11).standard_normal((4, m.K, sy.Np)).astype(dtype)
    dt = stable_dt(m, N, 1.0)
    host = torch.empty(q0.shape, dtype=sy.torch_dtype, pin_memory=True)
    host.numpy()[...] = q0
    a = FieldState(host.numpy(), "bernstein")
    b = FieldState(torch.from_numpy(q0.copy()).cuda(), "bernstein")
    calls = []
    lib = sy._lib

    class Spy:
        def __getattr__(self, k):
            if k == "bbdg_step_host":
                calls.append(1)
            return getattr(lib, k)

    sy._lib = Spy()
    try:
        for _ in range(2):
            a = lsrk4_step(sy, a, dt, "optimal")
    finally:
        sy._lib = lib
    for _ in range(2):
        b = lsrk4_step(sy, b, dt, "optimal")
    assert len(calls) == 2                            # the pipelined path ran
    assert np.array_equal(a.q, b.q.cpu().numpy())     # bitwise
    assert a.time == pytest.approx(2 * dt)


@pytest.mark.gpu
@pytest.mark.parametrize("N,dname,halve,threads", [(4, "f32", False, 1), (4, "f32", True, 4), (7, "f64", True, 3)])
def test_pageable_state_staged_pipeline_bitwise(N, dname, halve, threads, monkeypatch):
    """An ordinary numpy state goes through the pinned staging rings (bbdg_step_pageable): more
    chunks than ring slots, several copy threads, bitwise equal to the device-tensor step."""
    import torch

    monkeypatch.setenv("BBDG_COPY_THREADS", str(threads))
    dtype = np.float64 if dname == "f64" else np.float32
    m = cube_mesh(12)
    sy = WaveSystem(m, BernsteinRefOps.build(N), Materials.homogeneous(m.K), dtype=dtype)
    band = int(np.abs(m.etoe - np.arange(m.K)[:, None]).max())
    sy._chunks = host_chunk_plan(m.etoe, sy.Np, np.dtype(dtype).itemsize, min_state_bytes=0,
                                 chunk=(band // 2 + 1) if halve else None)
    assert len(sy._chunks[0]) - 1 > 3              # more chunks than the 3 ring slots
    q0 = np.random.default_rng(3).standard_normal((4, m.K, sy.Np)).astype(dtype)
    assert q0.nbytes >= 4 << 20
    dt = stable_dt(m, N, 1.0)
    calls = []
    lib = sy._lib

    class Spy:
        def __getattr__(self, k):
            if k == "bbdg_step_pageable":
                calls.append(1)
            return getattr(lib, k)

    sy._lib = Spy()
    a = FieldState(q0.copy(), "bernstein")
    try:
        for _ in range(2):
            a = lsrk4_step(sy, a, dt, "optimal")
    finally:
        sy._lib = lib
    b = FieldState(torch.from_numpy(q0.copy()).cuda(), "bernstein")
    for _ in range(2):
        b = lsrk4_step(sy, b, dt, "optimal")
    assert len(calls) == 2
    assert np.array_equal(a.q, b.q.cpu().numpy())


@pytest.mark.gpu
def test_small_pageable_state_uses_plain_path_and_matches():
    import torch

    m = cube_mesh(6)
    sy = WaveSystem(m, BernsteinRefOps.build(4), Materials.homogeneous(m.K), dtype=np.float32)
    sy._chunks = host_chunk_plan(m.etoe, sy.Np, 4, min_state_bytes=0)
    q0 = np.random.default_rng(3).standard_normal((4, m.K, sy.Np)).astype(np.float32)
    assert q0.nbytes < 4 << 20
    dt = stable_dt(m, 4, 1.0)
    a = lsrk4_step(sy, FieldState(q0.copy(), "bernstein"), dt, "optimal")       # pageable numpy
    b = lsrk4_step(sy, FieldState(torch.from_numpy(q0.copy()).cuda(), "bernstein"), dt, "optimal")
    assert np.array_equal(a.q, b.q.cpu().numpy())
