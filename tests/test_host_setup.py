"""Host-side setup (mesh, compact connectivity, operator tables) vs the reference (CPU)."""

import numpy as np
import pytest

from paper_1512_06025_b200 import bernstein as bb, mesh as msh, multiindex as mi, nodal as nd
from paper_1512_06025_b200.solver import Materials, stable_dt

MESH_KEYS = ("vertices", "tets", "jac", "rst_dx", "normals", "jf", "etoe", "etof", "h_elem")


def test_cube_mesh_matches_reference(golden_setup):
    m = msh.cube_mesh(2)
    for k in MESH_KEYS:
        a, b = getattr(m, k), golden_setup[f"mesh_{k}"]
        assert a.shape == b.shape, k
        if a.dtype.kind in "iu":
            assert np.array_equal(a, b), k
        else:
            assert np.abs(a - b).max() <= 1e-15 * max(1.0, np.abs(b).max()), k


@pytest.mark.parametrize("N", range(1, 5))
def test_compact_codes_reproduce_reference_gather(golden_setup, N):
    """(nbr elem, nbr face, vertex permutation) -> the reference's coordinate-matched gather, bit-exact."""
    m = msh.cube_mesh(2)
    g, b = msh.build_trace_maps(m, bb.BernsteinRefOps.build(N).trace, mi.tet_dim(N))
    assert np.array_equal(g, golden_setup[f"N{N}_gather"])
    assert np.array_equal(b, golden_setup[f"N{N}_boundary"])
    gn, _ = msh.build_trace_maps(m, nd.NodalRefOps.build(N).trace, mi.tet_dim(N))
    assert np.array_equal(gn, golden_setup[f"N{N}_nodal_gather"])


@pytest.mark.parametrize("N", [2, 4])
def test_reference_signature_build_trace_maps(golden_setup, N):
    """The reference's 4-argument form build_trace_maps(mesh, face_ref_points, face_positions, Np)
    (mesh.py:158) gives the reference gather and checks the coordinates; a Mesh built from the
    reference's nine fields (no permutation codes) derives them."""
    m = msh.cube_mesh(2)
    ops = bb.BernsteinRefOps.build(N)
    fp = np.stack([ops.face_ref_points(f) for f in range(4)])
    g, b = msh.build_trace_maps(m, fp, ops.trace, ops.Np)
    assert np.array_equal(g, golden_setup[f"N{N}_gather"]) and np.array_equal(b, golden_setup[f"N{N}_boundary"])
    bare = msh.Mesh(*[getattr(m, k) for k in MESH_KEYS])
    assert np.array_equal(bare.face_perm, m.face_perm)
    assert np.array_equal(msh.build_trace_maps(bare, fp, ops.trace, ops.Np)[0], g)
    bad = fp.copy()
    bad[0, [0, 1]] = bad[0, [1, 0]]                    # swap two face points: no longer conforming
    with pytest.raises(ValueError):
        msh.build_trace_maps(m, bad, ops.trace, ops.Np)


@pytest.mark.parametrize("N", range(1, 10))
def test_reference_operator_objects(golden_setup, N):
    """derivative_ops / build_L0 / build_lift expose the reference's sparse-row operators
    (bernstein.py:182-298) with the same dense values and row widths."""
    s = golden_setup
    ds = bb.derivative_ops(N)
    assert np.array_equal(np.stack([o.cols for o in ds.ops]), s[f"N{N}_dcols"])
    assert np.array_equal(ds.values, s[f"N{N}_dvals"])
    lf = bb.build_lift(N)
    assert np.abs(lf.L0.toarray() - s[f"N{N}_L0"]).max() < 1e-13 * np.abs(s[f"N{N}_L0"]).max()
    assert np.abs(lf.EL.toarray() - s[f"N{N}_EL"]).max() < 1e-13 * np.abs(s[f"N{N}_EL"]).max()
    assert lf.L0.row_width <= 7 and lf.EL.row_width <= mi.face_dim(N) + 3
    assert all(r.row_width <= 3 for r in lf.reductions) and len(lf.reductions) == N
    for f in (0, 3):
        Lo = bb.dense_lift_oracle(N, f)
        fact = lf.EL.toarray()[:, f * lf.Nfp:(f + 1) * lf.Nfp] @ lf.L0.toarray()
        assert np.abs(fact - Lo).max() / np.abs(Lo).max() < 1e-8


def test_face_codes_packing():
    m = msh.cube_mesh(3)
    nbr, code = m.face_codes()
    assert nbr.dtype == np.int32 and code.dtype == np.int8
    c = code.astype(np.int32) & 0xFF
    assert np.array_equal(c & 3, m.etof)
    assert np.array_equal((c >> 5) & 1, m.boundary.astype(np.int32))
    assert ((c >> 2) & 7).max() < 6
    # the cube mesh only needs 3 of the 6 orientations (survey, section 7 item 7)
    assert len(np.unique(((c >> 2) & 7)[~m.boundary])) <= 6


@pytest.mark.parametrize("N", range(1, 10))
def test_bernstein_tables_match_reference(golden_setup, N):
    s = golden_setup
    assert np.array_equal(bb.BernsteinRefOps.build(N).trace, s[f"N{N}_trace"])
    assert np.abs(bb.L0_dense(N) - s[f"N{N}_L0"]).max() < 1e-13 * np.abs(s[f"N{N}_L0"]).max()
    assert np.abs(bb.el_dense(N) - s[f"N{N}_EL"]).max() < 1e-13 * np.abs(s[f"N{N}_EL"]).max()
    assert np.array_equal(bb.dense_lift(N), s[f"N{N}_dense_L"])
    assert np.array_equal(bb.mass_matrix(N), s[f"N{N}_mass"])
    vals, cols = bb.derivative_tables(N)
    assert np.array_equal(vals, s[f"N{N}_dvals"])
    assert np.array_equal(cols, s[f"N{N}_dcols"])
    cols, vals = bb.ell_table(bb.el_dense(N))
    assert cols.shape[1] <= mi.face_dim(N) + 3          # reference bernstein.py:287-288


@pytest.mark.parametrize("N", range(1, 10))
def test_nodal_ops_match_reference(golden_setup, N):
    o = nd.NodalRefOps.build(N)
    for k in ("nodes", "Dr", "Ds", "Dt", "dense_L"):
        ref = golden_setup[f"N{N}_nodal_{k}"]
        assert np.abs(getattr(o, k) - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max()), k
    assert np.array_equal(o.trace, golden_setup[f"N{N}_nodal_trace"])


def test_closed_form_positions():
    for N in range(1, 12):
        idx = mi.simplex_indices(N, 3)
        assert np.array_equal(mi.pos3(N, idx[:, 0], idx[:, 1], idx[:, 2]), np.arange(len(idx)))
        idx2 = mi.simplex_indices(N, 2)
        assert np.array_equal(mi.pos2(N, idx2[:, 0], idx2[:, 1]), np.arange(len(idx2)))


def test_mesh_validation_and_dt():
    m = msh.cube_mesh(2)
    with pytest.raises(ValueError):
        Materials(np.array([1.0, -1.0]), np.ones(2))
    base = stable_dt(m, 2, 1.0)
    assert stable_dt(m, 4, 1.0) == pytest.approx(base / 4.0)
    assert stable_dt(msh.cube_mesh(4), 2, 1.0) == pytest.approx(base / 2.0)
    with pytest.raises(ValueError):
        stable_dt(m, 2, 1.0, cfl=0.0)
    with pytest.raises(ValueError):
        msh.cube_mesh(0)


def test_mesh_ascii_roundtrip(tmp_path):
    m = msh.cube_mesh(2)
    msh.save_mesh_ascii(tmp_path / "m.txt", m)
    m2 = msh.load_mesh_ascii(tmp_path / "m.txt")
    assert np.array_equal(m.tets, m2.tets) and np.array_equal(m.etoe, m2.etoe)
    (tmp_path / "bad.txt").write_text("8 6\n0 0 0\n")
    with pytest.raises(ValueError):
        msh.load_mesh_ascii(tmp_path / "bad.txt")


def test_large_mesh_builds_fast():
    import time
    t = time.perf_counter()
    m = msh.cube_mesh(26)                 # config C2, K = 105,456
    assert m.K == 105456
    assert time.perf_counter() - t < 20.0  # reference: ~66 s with trace maps
