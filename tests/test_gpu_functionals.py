"""Device functionals and the finite-precision study (BASELINE configs[3]) on the GPU.

Anchors: the host float64 formulas of the reference (solver.py:282-312) for the
functionals, and reference error values / trajectories computed by the reference
itself on the CPU (tests/golden/make_sensitivity.py -> golden_sensitivity.npz).
"""

from pathlib import Path

import numpy as np
import pytest

from conftest import rel_l2
from paper_1512_06025_b200 import (BernsteinRefOps, ErrorFunctional, FieldState, Materials, NodalRefOps, WaveSystem,
                                   cube_mesh, discrete_energy, initial_state, integrate, stable_dt)

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden" / "golden_sensitivity.npz"


@pytest.fixture(scope="module")
def sens():
    if not GOLD.exists():
        pytest.skip("golden_sensitivity.npz not generated")
    return np.load(GOLD)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_device_energy_and_error_match_host(dtype):
    import torch

    m = cube_mesh(3)
    rng = np.random.default_rng(3)
    mat = Materials(rng.uniform(0.5, 2.0, m.K), rng.uniform(0.5, 2.0, m.K))
    sy = WaveSystem(m, BernsteinRefOps.build(4), mat, dtype=dtype)
    q = rng.standard_normal((4, m.K, sy.Np)).astype(dtype)
    e_host = discrete_energy(sy, FieldState(q.astype(np.float64), "bernstein"))
    e_dev = discrete_energy(sy, FieldState(torch.as_tensor(q).cuda(), "bernstein"))
    assert abs(e_dev - e_host) <= 1e-13 * abs(e_host)
    ef = ErrorFunctional(m, sy.ops_double)
    st = initial_state(m, 4, "bernstein", dtype=dtype, tau=0.3)
    h = ef(FieldState(st.q.copy(), "bernstein", 0.31))
    d = ef(FieldState(torch.as_tensor(st.q).cuda(), "bernstein", 0.31))
    assert abs(d - h) <= 1e-12 * abs(h)


def _run(n, N, dtype, tau=0.5, lift="optimal"):
    import torch

    m = cube_mesh(n)
    sy = WaveSystem(m, BernsteinRefOps.build(N), Materials.homogeneous(m.K), dtype=dtype)
    st = initial_state(m, N, "bernstein", dtype=dtype)
    dt = stable_dt(m, N, 1.0)
    nst = int(np.ceil(tau / dt))
    st = FieldState(torch.as_tensor(st.q).cuda(), "bernstein")
    st = integrate(sy, st, tau / nst, nst, lift, energy_guard=None)
    return ErrorFunctional(m, sy.ops_double)(st)


@pytest.mark.parametrize("n,N", [(2, N) for N in range(1, 10)] + [(4, N) for N in range(1, 7)])
def test_convergence_errors_match_reference(sens, n, N):
    """float64: the error after tau = 0.5 equals the reference's to roundoff; float32: same
    value where discretisation error dominates, same magnitude where roundoff does."""
    e64 = _run(n, N, np.float64)
    r64 = float(sens[f"conv_f64_n{n}_N{N}"])
    assert abs(e64 - r64) <= 1e-6 * r64 + 1e-12, (e64, r64)
    e32 = _run(n, N, np.float32)
    r32 = float(sens[f"conv_f32_n{n}_N{N}"])
    assert abs(e32 - r64) <= 1e-4 * r64 + 3e-6, (e32, r64)       # float32 floor ~1e-6
    assert 1 / 3 <= (e32 + 1e-7) / (r32 + 1e-7) <= 3, (e32, r32)


@pytest.mark.parametrize("N", range(1, 10))
def test_convergence_states_match_reference(N):
    """configs[3] at the north-star float64 tolerance: the whole state after the convergence run
    (cube_mesh(2), tau = 0.5, factorized lift -- the reference default; 5..392 steps) equals the
    reference's own final state to 1e-12 relative L2 (golden_sens_states.npz, produced by
    make_sens_states.py on the reference), and so does the error functional."""
    import torch

    g = np.load(GOLD.parent / "golden_sens_states.npz")
    m = cube_mesh(2)
    sy = WaveSystem(m, BernsteinRefOps.build(N), Materials.homogeneous(m.K))
    st = initial_state(m, N, "bernstein")
    nst = int(g[f"nst_N{N}"])
    assert nst == int(np.ceil(0.5 / stable_dt(m, N, 1.0)))
    st = integrate(sy, FieldState(torch.as_tensor(st.q).cuda(), "bernstein"), 0.5 / nst, nst, "factorized",
                   energy_guard=None)
    assert rel_l2(st.q.cpu().numpy(), g[f"q_N{N}"]) < 1e-12
    e, r = ErrorFunctional(m, sy.ops_double)(st), float(g[f"err_N{N}"])
    assert abs(e - r) <= 1e-10 * r + 1e-15, (e, r)   # the functional's own cancellation: |p_h - p| << |p|


def test_reference_divergence_reproduced(sens):
    """N = 1 at cfl = 0.5 diverges on cube_mesh(16) in the reference (error ~1.12 at tau = 0.5);
    the device path reproduces the reference's value, not a stabilised one."""
    e = _run(16, 1, np.float64)
    r = float(sens["conv_f64_n16_N1"])
    assert r > 1.0 and abs(e - r) <= 1e-9 * r, (e, r)


def test_roundoff_band_criterion_8(sens):
    """Reference acceptance criterion 8 (test_acceptance.py:222-250) on the GPU, float32 N=5,
    cube_mesh(4), tau <= 5: errors inside [5e-8, 1e-5], Bernstein <= 2x nodal, and each
    trajectory within 2x of the reference's own samples."""
    import torch

    N, n, tmax = 5, 4, 5.0
    m = cube_mesh(n)
    mat = Materials.homogeneous(m.K)
    dt = stable_dt(m, N, 1.0)
    nst = int(np.ceil(tmax / dt))
    dt = tmax / nst
    every = max(1, nst // 100)
    traj = {}
    for basis, Ops in (("bernstein", BernsteinRefOps), ("nodal", NodalRefOps)):
        sy = WaveSystem(m, Ops.build(N), mat, dtype=np.float32)
        st = initial_state(m, N, basis, dtype=np.float32)
        ef = ErrorFunctional(m, sy.ops_double)
        samples = []
        integrate(sy, FieldState(torch.as_tensor(st.q).cuda(), basis), dt, nst, "optimal",
                  callback=lambda step, s: samples.append(ef(s)) if step % every == 0 else None)
        traj[basis] = np.array(samples)
        assert traj[basis].min() > 5e-8 and traj[basis].max() < 1e-5, basis
        ref = sens[f"band_{basis}"]
        assert len(ref) == len(traj[basis])
        assert np.all(traj[basis] <= 2 * ref) and np.all(ref <= 2 * traj[basis]), basis
    assert (traj["bernstein"] / traj["nodal"]).max() <= 2.0


@pytest.mark.parametrize("basis", ["bernstein", "nodal"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_initial_state_device_matches_host(basis, dtype):
    from paper_1512_06025_b200 import initial_state_device

    m = cube_mesh(3)
    for N in (1, 4, 9):
        host = initial_state(m, N, basis, dtype=dtype, tau=0.37)
        dev = initial_state_device(m, N, basis, dtype=dtype, tau=0.37, chunk=50)   # several chunks
        got = dev.q.cpu().numpy()
        assert got.dtype == dtype and dev.time == 0.37
        tol = 1e-13 if dtype == np.float64 else 1e-6
        assert rel_l2(got, host.q) < tol, (N, rel_l2(got, host.q))
