"""GPU parity: the sm_100a kernels (through the C ABI) vs the reference.

Three anchors: golden vectors produced by the reference itself
(tests/golden), the pinned CPU oracle on fresh seeded inputs, and
size-independent properties at the full config-2 size (K = 105,456).
Tolerances (relative L2): 1e-12 float64, 1e-5 float32 (north star).
"""

import numpy as np
import pytest

import bbdg_oracle as orc
from conftest import TOL, rel_l2
from paper_1512_06025_b200 import (BernsteinRefOps, FieldState, Materials, NodalRefOps, WaveSystem, cube_mesh,
                                   discrete_energy, from_arrays, initial_state, integrate, lsrk4_step,
                                   nodal_to_bernstein, stable_dt)
from paper_1512_06025_b200.multiindex import TET_VERTICES

pytestmark = pytest.mark.gpu
MODES = ("factorized", "optimal", "dense")
DT = {"f64": np.float64, "f32": np.float32}

_systems = {}


def mode_tol(g, N, dname, mode):
    """The dense lift M^-1 M^f is ill-conditioned at high N (entries up to 1386 at
    N=9): any summation order other than the reference's BLAS call differs by the
    reference's own rounding noise, which we measure from the golden vectors as
    the reference's dense-vs-factorized gap (2.6e-12 at N=9).  The
    tolerance is max(north-star tol, 2 x that gap); for the sparse modes it is the
    north-star tolerance itself."""
    tol = TOL[dname]
    if mode != "dense":
        return tol
    gap = rel_l2(g[f"N{N}_{dname}_surf_dense"], g[f"N{N}_{dname}_surf_factorized"])
    return max(tol, 2.0 * gap)


def bern_system(n, N, dname="f64", mat=None):
    key = (n, N, dname, id(mat))
    if key not in _systems:
        m = cube_mesh(n)
        _systems[key] = WaveSystem(m, BernsteinRefOps.build(N), mat or Materials.homogeneous(m.K), dtype=DT[dname])
    return _systems[key]


@pytest.mark.parametrize("N", range(1, 10))
@pytest.mark.parametrize("dname", ["f64", "f32"])
def test_bb_parity_with_reference_golden(golden_bb, N, dname):
    g = golden_bb
    sy = bern_system(int(g[f"N{N}_n"]), N, dname)
    q = g[f"N{N}_q"].astype(DT[dname])
    st = FieldState(q.copy(), "bernstein")
    tol = TOL[dname]
    vol = sy.volume_rhs(st)
    assert vol.dtype == DT[dname]
    assert rel_l2(vol, g[f"N{N}_{dname}_vol"]) < tol
    for mode in MODES:
        assert rel_l2(sy.surface_rhs(st, mode), g[f"N{N}_{dname}_surf_{mode}"]) < mode_tol(g, N, dname, mode), mode
    assert rel_l2(sy.rhs(st), g[f"N{N}_{dname}_rhs"]) < tol
    out = lsrk4_step(sy, st, float(g[f"N{N}_dt"]), "factorized")
    assert out.q is st.q                                   # in place, like the reference
    assert rel_l2(st.q, g[f"N{N}_{dname}_step"]) < tol


@pytest.mark.parametrize("N", range(1, 10))
def test_nodal_parity_with_reference_golden(golden_nodal, N):
    """Node-per-thread nodal kernels vs the reference (cube_mesh(2) for N <= 6, cube_mesh(1) above)."""
    g = golden_nodal
    m = cube_mesh(2 if N <= 6 else 1)
    sy = WaveSystem(m, NodalRefOps.build(N), Materials.homogeneous(m.K))
    q = g[f"N{N}_q"]
    assert rel_l2(sy.volume_rhs(FieldState(q.copy(), "nodal")), g[f"N{N}_vol"]) < TOL["f64"]
    assert rel_l2(sy.rhs(FieldState(q.copy(), "nodal")), g[f"N{N}_rhs"]) < TOL["f64"]
    st = lsrk4_step(sy, FieldState(q.copy(), "nodal"), float(g[f"N{N}_dt"]))
    assert rel_l2(st.q, g[f"N{N}_step"]) < TOL["f64"]


@pytest.mark.parametrize("N", range(1, 10))
@pytest.mark.parametrize("dname", ["f64", "f32"])
def test_nodal_blocked_parity_with_reference_golden(golden_nodal, N, dname):
    """Block-partitioned tensor-core nodal kernels (fp64 DMMA, fp32 3xTF32) vs the reference."""
    g = golden_nodal
    m = cube_mesh(2 if N <= 6 else 1)
    sy = WaveSystem(m, NodalRefOps.build(N), Materials.homogeneous(m.K), dtype=DT[dname])
    q = g[f"N{N}_q"].astype(DT[dname])
    assert rel_l2(sy.rhs(FieldState(q.copy(), "nodal"), "blocked"), g[f"N{N}_rhs"]) < TOL[dname]
    st = lsrk4_step(sy, FieldState(q.copy(), "nodal"), float(g[f"N{N}_dt"]), "blocked")
    assert rel_l2(st.q, g[f"N{N}_step"]) < TOL[dname]


@pytest.mark.parametrize("N", [2, 7, 9])
@pytest.mark.parametrize("dname", ["f64", "f32"])
def test_nodal_blocked_matches_dense_fresh_inputs(N, dname):
    """K = 162 (partial element tiles), heterogeneous materials: blocked vs the NPT dense kernels
    (which are pinned to the reference golden vectors above)."""
    m = cube_mesh(3)
    rng = np.random.default_rng(7 + N)
    mat = Materials(rng.uniform(0.5, 2.0, m.K), rng.uniform(0.5, 2.0, m.K))
    sd = WaveSystem(m, NodalRefOps.build(N), mat, dtype=np.float64)
    sb = WaveSystem(m, NodalRefOps.build(N), mat, dtype=DT[dname])
    q = rng.standard_normal((4, m.K, sd.Np))
    want = sd.rhs(FieldState(q.copy(), "nodal"))
    got = sb.rhs(FieldState(q.astype(DT[dname]), "nodal"), "blocked")
    assert rel_l2(got, want) < TOL[dname]


@pytest.mark.parametrize("N", [2, 5, 9])
@pytest.mark.parametrize("dname", ["f64", "f32"])
def test_nodal_blocked_stage_ranges_bitwise(N, dname):
    """Element ranges that start and end inside the tensor-core tiles (kbeg != 0 mod 32): the
    ranged stages reproduce the whole-mesh stage bitwise (row-independent GEMM, fixed K order)."""
    import torch

    from paper_1512_06025_b200.solver import RK4A, RK4B

    m = cube_mesh(3)
    sy = WaveSystem(m, NodalRefOps.build(N), Materials.homogeneous(m.K), dtype=DT[dname])
    g = torch.Generator(device="cuda").manual_seed(N)
    q = torch.randn((4, m.K, sy.Np), dtype=sy.torch_dtype, device="cuda", generator=g)
    r0 = torch.randn_like(q)
    dt = stable_dt(m, N, 1.0)
    qa, ra = torch.empty_like(q), r0.clone()
    sy.stage_into(q, qa, ra, RK4A[2], RK4B[2], dt, "blocked")
    qb, rb = torch.empty_like(q), r0.clone()
    for k0, k1 in ((0, 45), (45, 101), (101, m.K)):
        sy.stage_range_into(q, qb, rb, RK4A[2], RK4B[2], dt, "blocked", k0, k1)
    torch.cuda.synchronize()
    assert torch.equal(qa, qb) and torch.equal(ra, rb)


def stage_vs_oracle(sy, ref, q, res, dt, mode, rows=None, tol=None):
    """One fused LSRK stage (bbdg_lsrk_stage: the bench's timed kernel) against the oracle's
    res = A res + dt rhs; q_out = q + B res, element-wise over `rows` (all elements by default)."""
    import torch

    from paper_1512_06025_b200.solver import RK4A, RK4B

    qd, rd = torch.from_numpy(q).cuda(), torch.from_numpy(res.copy()).cuda()
    qo = torch.empty_like(qd)
    sy.stage_into(qd, qo, rd, RK4A[1], RK4B[1], dt, mode)
    qo, rd = qo.cpu().numpy(), rd.cpu().numpy()
    tol = tol or TOL["f64" if q.dtype == np.float64 else "f32"]
    for k0, k1 in rows or [(0, sy.K)]:
        want_q, want_r = ref.stage(q, res, RK4A[1], RK4B[1], dt, mode, k0, k1)
        assert rel_l2(qo[:, k0:k1], want_q) < tol, (mode, k0, k1)
        assert rel_l2(rd[:, k0:k1], want_r) < tol, (mode, k0, k1)


@pytest.mark.parametrize("N", range(1, 10))
@pytest.mark.parametrize("dname", ["f64", "f32"])
def test_bb_parity_with_oracle_fresh_inputs(N, dname):
    """cube_mesh(4) (K=384, so K Np = 0 mod 4: the field-stride residue FSR 0 that the bench's
    K=384,000 and the HBM-filling meshes select), heterogeneous materials, a fresh seed: every
    fused-kernel instantiation the bench times (stage; rhs / volume / surface) vs the oracle."""
    m = cube_mesh(4)
    rng = np.random.default_rng(100 + N)
    kap, rho = rng.uniform(0.5, 2.0, m.K), rng.uniform(0.5, 2.0, m.K)
    dtype = DT[dname]
    sy = WaveSystem(m, BernsteinRefOps.build(N), Materials(kap, rho), dtype=dtype)
    assert (m.K * sy.Np) % 4 == 0
    ref = orc.OracleSystem(orc.mesh_arrays(m), orc.bernstein_tables(N), kap, rho, dtype)
    q = rng.standard_normal((4, m.K, sy.Np)).astype(dtype)
    for mode in MODES:
        assert rel_l2(sy.rhs(FieldState(q.copy(), "bernstein"), mode), ref.rhs(q.copy(), mode)) < TOL[dname], mode
    assert rel_l2(sy.volume_rhs(FieldState(q.copy(), "bernstein")), ref.volume_rhs(q.copy())) < TOL[dname]
    for mode in ("optimal", "factorized", "ell"):
        want = ref.surface_rhs(q.copy(), "factorized" if mode == "ell" else mode)
        assert rel_l2(sy.surface_rhs(FieldState(q.copy(), "bernstein"), mode), want) < TOL[dname], mode
    dt = stable_dt(m, N, float(np.sqrt(kap / rho).max()))
    res = rng.standard_normal(q.shape).astype(dtype)
    for mode in ("optimal", "factorized"):
        stage_vs_oracle(sy, ref, q, res, dt, mode)
    st = lsrk4_step(sy, FieldState(q.copy(), "bernstein"), dt, "optimal")
    assert rel_l2(st.q, ref.lsrk4_step(q.copy(), dt, "optimal")) < TOL[dname]


def test_constant_state_volume_exactly_zero():
    sy = bern_system(2, 3)
    st = FieldState(np.ones((4, sy.K, sy.Np)), "bernstein")
    assert np.abs(sy.volume_rhs(st)).max() == 0.0                  # reference test_solver.py:26-33
    ds = sy.surface_rhs(st)
    interior = ~sy.boundary.any(axis=1)
    assert np.abs(ds[:, interior]).max() < 1e-13


def test_linear_pressure_gradient_exact():
    from paper_1512_06025_b200.nodal import NodalRefOps as NR

    m = from_arrays(TET_VERTICES, [(0, 1, 2, 3)])
    sy = WaveSystem(m, BernsteinRefOps.build(3), Materials.homogeneous(1, kappa=1.0, rho=2.0))
    nops = NR.build(3)
    q = np.zeros((4, 1, sy.Np))
    q[0] = nodal_to_bernstein(nops, m.map_reference_points(nops.nodes)[..., 0])
    dv = sy.volume_rhs(FieldState(q, "bernstein"))
    assert np.abs(dv[1] + 0.5).max() < 1e-12
    assert np.abs(dv[2]).max() < 1e-12 and np.abs(dv[3]).max() < 1e-12 and np.abs(dv[0]).max() < 1e-12


def test_exact_initial_state_has_zero_jumps():
    m = cube_mesh(2)
    sy = bern_system(2, 4)
    assert np.abs(sy.surface_rhs(initial_state(m, 4, "bernstein"))).max() < 1e-9


class _ScalarDecay:
    def rhs(self, state, lift_mode=None):
        return -state.q


class _Zero:
    def rhs(self, state, lift_mode=None):
        return np.zeros_like(state.q)


def test_lsrk4_scalar_ode_duck_typed():
    """Reference test_solver.py:76-84: the update kernel on a duck-typed system."""
    st = FieldState(np.ones((4, 1, 1)), "bernstein")
    for _ in range(10):
        st = lsrk4_step(_ScalarDecay(), st, 0.1)
    assert abs(st.q[0, 0, 0] - np.exp(-1.0)) == pytest.approx(1.2995611e-07, rel=1e-5)
    assert st.time == pytest.approx(1.0)
    q0 = np.random.default_rng(0).standard_normal((4, 2, 3))
    st = lsrk4_step(_Zero(), FieldState(q0.copy(), "bernstein"), 0.3)
    assert np.array_equal(st.q, q0)
    with pytest.raises(ValueError):
        lsrk4_step(_Zero(), FieldState(q0.copy(), "bernstein"), 0.0)


@pytest.mark.parametrize("dname", ["f64", "f32"])
@pytest.mark.parametrize("mode", MODES)
def test_config1_ten_steps_vs_reference(golden_c1, dname, mode):
    """Config 1: cube_mesh(6), N=3, 10 LSRK4 steps from the exact IC: the full final state vs the
    reference's own run, every lift mode and precision (element-wise relative L2)."""
    m = cube_mesh(6)
    dt = float(golden_c1["dt"])
    sy = bern_system(6, 3, dname)
    st = integrate(sy, initial_state(m, 3, "bernstein", dtype=DT[dname]), dt, 10, lift_mode=mode, energy_guard=None)
    assert st.q.dtype == DT[dname]
    assert rel_l2(st.q, golden_c1[f"q_final_{dname}_{mode}"]) < TOL[dname], (dname, mode)
    nrm = float(np.linalg.norm(st.q.astype(np.float64)))
    assert abs(nrm - float(golden_c1[f"norm_{dname}_{mode}"])) / nrm < TOL[dname], (dname, mode)


def test_single_precision_rhs_close_to_double():
    m = cube_mesh(2)
    st = initial_state(m, 3, "bernstein", dtype=np.float32)
    r = bern_system(2, 3, "f32").rhs(st)
    assert r.dtype == np.float32
    ref = bern_system(2, 3, "f64").rhs(FieldState(st.q.astype(np.float64), "bernstein"))
    assert np.abs(r - ref).max() / np.abs(ref).max() < 1e-5


@pytest.mark.parametrize("basis", ["bernstein", "nodal"])
def test_energy_decays(basis):
    m = cube_mesh(2)
    ops = BernsteinRefOps.build(2) if basis == "bernstein" else NodalRefOps.build(2)
    sy = WaveSystem(m, ops, Materials.homogeneous(m.K))
    energies = []
    integrate(sy, initial_state(m, 2, basis), stable_dt(m, 2, 1.0), 40,
              callback=lambda s, x: energies.append(discrete_energy(sy, x)))
    e = np.array(energies)
    assert (np.diff(e) <= 1e-10 * e[0]).all()


def test_unstable_run_aborts():
    m = cube_mesh(2)
    sy = bern_system(2, 3)
    with pytest.raises(RuntimeError):
        integrate(sy, initial_state(m, 3, "bernstein"), 50.0 * stable_dt(m, 3, 1.0), 2000)


def test_device_tensor_path_and_integrate_equivalence():
    import torch

    m = cube_mesh(3)
    sy = bern_system(3, 4)
    st = initial_state(m, 4, "bernstein")
    dt = stable_dt(m, 4, 1.0)
    qd = torch.from_numpy(st.q.copy()).cuda()
    r = sy.rhs(FieldState(qd, "bernstein"), "optimal")
    assert r.is_cuda
    assert rel_l2(r.cpu().numpy(), sy.rhs(FieldState(st.q.copy(), "bernstein"), "optimal")) == 0.0
    a = FieldState(qd.clone(), "bernstein")
    for _ in range(3):
        a = lsrk4_step(sy, a, dt, "optimal")
    b = integrate(sy, FieldState(qd.clone(), "bernstein"), dt, 3, lift_mode="optimal", energy_guard=None)
    assert torch.equal(a.q, b.q)                     # same kernels, same order: bitwise


# ------------------------------------------------------------------ full config-2 size (K = 105,456)
@pytest.fixture(scope="module")
def c2_mesh():
    return cube_mesh(26)


@pytest.mark.parametrize("N", [1, 5, 9])
def test_full_size_properties(c2_mesh, N):
    import torch

    m = c2_mesh
    for dname in ("f32", "f64"):
        sy = WaveSystem(m, BernsteinRefOps.build(N), Materials.homogeneous(m.K), dtype=DT[dname])
        tdt = sy.torch_dtype
        # constant state: the volume term vanishes exactly at every element
        ones = torch.ones((4, m.K, sy.Np), dtype=tdt, device="cuda")
        out = torch.empty_like(ones)
        sy.volume_into(ones, out)
        assert torch.count_nonzero(out).item() == 0
        g = torch.Generator(device="cuda").manual_seed(7)
        q1 = torch.randn((4, m.K, sy.Np), dtype=tdt, device="cuda", generator=g)
        q2 = torch.randn((4, m.K, sy.Np), dtype=tdt, device="cuda", generator=g)
        for mode in MODES if N < 9 else ("optimal", "factorized"):
            r1, r2, r12 = torch.empty_like(q1), torch.empty_like(q1), torch.empty_like(q1)
            sy.rhs_into(q1, r1, mode)
            sy.rhs_into(q2, r2, mode)
            sy.rhs_into(2.0 * q1 - 3.0 * q2, r12, mode)
            lin = (r12 - (2.0 * r1 - 3.0 * r2)).norm() / r12.norm()
            assert lin.item() < (1e-13 if dname == "f64" else 1e-5), mode
            # determinism: owner-computes, no atomics -> bitwise reproducible
            again = torch.empty_like(q1)
            sy.rhs_into(q1, again, mode)
            assert torch.equal(again, r1)
            # split volume + surface(accumulate) == fused rhs
            split = torch.empty_like(q1)
            sy.volume_into(q1, split)
            sy.surface_into(q1, split, mode, accumulate=True)
            assert ((split - r1).norm() / r1.norm()).item() < (1e-14 if dname == "f64" else 1e-6)
        # energy is non-increasing over a few steps from the smooth IC
        st = initial_state(m, N, "bernstein", dtype=DT[dname]) if N <= 5 else None
        if st is not None:
            dt = stable_dt(m, N, 1.0)
            e = [discrete_energy(sy, st)]
            qd = FieldState(torch.from_numpy(st.q).cuda(), "bernstein")
            for _ in range(3):
                qd = lsrk4_step(sy, qd, dt, "optimal")
                e.append(discrete_energy(sy, qd))
            assert (np.diff(e) <= 1e-6 * e[0]).all()
        del sy


@pytest.mark.parametrize("N", range(1, 10))
@pytest.mark.parametrize("K", [44, 45, 46, 47])
@pytest.mark.parametrize("dname", ["f64", "f32"])
def test_bb_parity_every_stride_residue(N, K, dname):
    """Sub-meshes of cube_mesh(2) with K = 44..47 tets (non-convex domains with extra boundary
    faces): K Np mod 4 takes every value the order allows, so each stride-residue variant of the
    fused kernel (template FSR: 4 in fp32, 2 in fp64) is compared element-wise with the oracle; the
    last TMA window runs past the end of the state arrays (sub-16-byte tail copied by hand) and
    odd K ends on a partial tile (incl. the fp64 stage's guarded HBM reads of the LSRK register)."""
    base = cube_mesh(2)
    m = from_arrays(base.vertices, base.tets[:K])
    assert m.K == K
    rng = np.random.default_rng(40 + 10 * N + K)
    kap, rho = rng.uniform(0.5, 2.0, m.K), rng.uniform(0.5, 2.0, m.K)
    dtype = DT[dname]
    sy = WaveSystem(m, BernsteinRefOps.build(N), Materials(kap, rho), dtype=dtype)
    ref = orc.OracleSystem(orc.mesh_arrays(m), orc.bernstein_tables(N), kap, rho, dtype)
    q = rng.standard_normal((4, m.K, sy.Np)).astype(dtype)
    for mode in ("optimal", "factorized"):
        assert rel_l2(sy.rhs(FieldState(q.copy(), "bernstein"), mode), ref.rhs(q.copy(), mode)) < TOL[dname], mode
    assert rel_l2(sy.volume_rhs(FieldState(q.copy(), "bernstein")), ref.volume_rhs(q.copy())) < TOL[dname]
    assert rel_l2(sy.surface_rhs(FieldState(q.copy(), "bernstein"), "optimal"),
                  ref.surface_rhs(q.copy(), "optimal")) < TOL[dname]
    dt = stable_dt(m, N, float(np.sqrt(kap / rho).max()))
    stage_vs_oracle(sy, ref, q, rng.standard_normal(q.shape).astype(dtype), dt, "optimal")
    st = lsrk4_step(sy, FieldState(q.copy(), "bernstein"), dt, "optimal")
    assert rel_l2(st.q, ref.lsrk4_step(q.copy(), dt, "optimal")) < TOL[dname]


# ------------------------------------------------------------------ config-2 size vs the oracle
@pytest.fixture(scope="module")
def c2_arrays(c2_mesh):
    return orc.mesh_arrays(c2_mesh)


_C2_MAPS = {}


@pytest.mark.parametrize("N", range(1, 10))
def test_config2_stage_vs_oracle(c2_mesh, c2_arrays, N):
    """configs[1] mesh cube_mesh(26), K = 105,456 (FSR 0): the fused stage element-wise against the
    oracle, fp64 and fp32 -- every element for N <= 3, three 1,024-element windows (start, middle,
    end: boundary and interior elements) above, where the numpy oracle of the whole mesh is slow."""
    m = c2_mesh
    K = m.K
    rows = None if N <= 3 else [(0, 1024), (K // 2, K // 2 + 1024), (K - 1024, K)]
    key = (N, rows is None)
    tabs = orc.bernstein_tables(N)
    if key not in _C2_MAPS:
        _C2_MAPS.clear()
        _C2_MAPS[key] = orc.trace_maps(c2_arrays["vertices"], c2_arrays["tets"], c2_arrays["etoe"],
                                       c2_arrays["etof"], tabs.face_pts, tabs.trace, tabs.Np, c2_arrays["h_elem"], rows)
    rng = np.random.default_rng(2600 + N)
    kap, rho = np.ones(K), np.ones(K)
    dt = stable_dt(m, N, 1.0)
    for dname in ("f64", "f32"):
        dtype = DT[dname]
        sy = WaveSystem(m, BernsteinRefOps.build(N), Materials(kap, rho), dtype=dtype)
        ref = orc.OracleSystem(c2_arrays, tabs, kap, rho, dtype, maps=_C2_MAPS[key])
        q = rng.standard_normal((4, K, sy.Np)).astype(dtype)
        res = rng.standard_normal((4, K, sy.Np)).astype(dtype)
        stage_vs_oracle(sy, ref, q, res, dt, "optimal", rows)
        del sy
