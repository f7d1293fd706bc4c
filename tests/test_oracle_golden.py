"""Pin the CPU oracle against vectors produced by the reference itself (CPU only)."""

import numpy as np
import pytest

import bbdg_oracle as orc
from conftest import TOL, rel_l2
from paper_1512_06025_b200 import mesh as msh

MODES = ("factorized", "optimal", "dense")


def _sys(n, N, dtype, nodal=None):
    m = msh.cube_mesh(n)
    kap, rho = np.ones(m.K), np.ones(m.K)
    tables = orc.bernstein_tables(N) if nodal is None else nodal
    return orc.OracleSystem(orc.mesh_arrays(m), tables, kap, rho, dtype)


@pytest.mark.parametrize("N", range(1, 10))
@pytest.mark.parametrize("dname", ["f64", "f32"])
def test_oracle_matches_reference_bb(golden_bb, N, dname):
    g = golden_bb
    dtype = np.float64 if dname == "f64" else np.float32
    sy = _sys(int(g[f"N{N}_n"]), N, dtype)
    q = g[f"N{N}_q"].astype(dtype)
    # the oracle is a line-by-line restatement: float64 agrees to rounding noise
    tol = 1e-13 if dname == "f64" else 1e-6
    assert rel_l2(sy.volume_rhs(q), g[f"N{N}_{dname}_vol"]) < tol
    for mode in MODES:
        assert rel_l2(sy.surface_rhs(q, mode), g[f"N{N}_{dname}_surf_{mode}"]) < tol, mode
    assert rel_l2(sy.rhs(q), g[f"N{N}_{dname}_rhs"]) < tol
    qs = sy.lsrk4_step(q.copy(), float(g[f"N{N}_dt"]))
    assert rel_l2(qs, g[f"N{N}_{dname}_step"]) < tol


@pytest.mark.parametrize("N", range(1, 7))
def test_oracle_matches_reference_nodal(golden_nodal, golden_setup, N):
    s = golden_setup
    tables = orc.NodalTables(N, s[f"N{N}_nodal_Dr"], s[f"N{N}_nodal_Ds"], s[f"N{N}_nodal_Dt"],
                             s[f"N{N}_nodal_dense_L"], s[f"N{N}_nodal_trace"], s[f"N{N}_nodal_nodes"])
    sy = _sys(2, N, np.float64, nodal=tables)
    q = golden_nodal[f"N{N}_q"]
    assert rel_l2(sy.volume_rhs(q), golden_nodal[f"N{N}_vol"]) < 1e-13
    assert rel_l2(sy.rhs(q, "dense"), golden_nodal[f"N{N}_rhs"]) < 1e-13
    qs = sy.lsrk4_step(q.copy(), float(golden_nodal[f"N{N}_dt"]), "dense")
    assert rel_l2(qs, golden_nodal[f"N{N}_step"]) < 1e-13


def test_oracle_trace_maps_match_reference(golden_setup):
    s = golden_setup
    m = {k: s[f"mesh_{k}"] for k in ("vertices", "tets", "jac", "rst_dx", "normals", "jf", "etoe", "etof", "h_elem")}
    for N in range(1, 5):
        t = orc.bernstein_tables(N)
        g, b = orc.trace_maps(m["vertices"], m["tets"], m["etoe"], m["etof"], t.face_pts, t.trace, t.Np, m["h_elem"])
        assert np.array_equal(g, s[f"N{N}_gather"])
        assert np.array_equal(b, s[f"N{N}_boundary"])


def test_oracle_tables_match_reference(golden_setup):
    s = golden_setup
    for N in range(1, 10):
        t = orc.bernstein_tables(N)
        assert np.array_equal(t.L0.dense(), s[f"N{N}_L0"])
        assert np.abs(t.EL.dense() - s[f"N{N}_EL"]).max() == 0.0
        assert np.abs(t.dense_L - s[f"N{N}_dense_L"]).max() <= 1e-12 * np.abs(s[f"N{N}_dense_L"]).max()
        assert np.array_equal(np.stack(t.dcols), s[f"N{N}_dcols"])


def test_oracle_config1_ten_steps(golden_c1):
    """Config 1 (cube_mesh(6), N=3, 10 LSRK4 steps) against the reference's own run."""
    from paper_1512_06025_b200.solver import initial_state  # host-side IC (float64 nodal interpolation)

    m = msh.cube_mesh(6)
    sy = orc.OracleSystem(orc.mesh_arrays(m), orc.bernstein_tables(3), np.ones(m.K), np.ones(m.K))
    q = initial_state(m, 3, "bernstein").q
    dt = float(golden_c1["dt"])
    for _ in range(10):
        q = sy.lsrk4_step(q, dt, "factorized")
    assert rel_l2(q, golden_c1["q_final_f64_factorized"]) < 1e-13
