"""Generate golden vectors by running the REFERENCE package itself.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Run in the build container (the reference is not present on the GPU box);
the outputs are committed as small compressed .npz fixtures:

  golden_bb.npz     Bernstein: seed-2024 random states on cube_mesh(2) (N=1..4)
                    and cube_mesh(1) (N=5..9); volume_rhs, surface_rhs x 3 lift
                    modes, rhs, one lsrk4_step -- float64 and float32
  golden_nodal.npz  nodal: rhs + one lsrk4_step on cube_mesh(2), N=1..6, and on
                    cube_mesh(1), N=7..9, float64
  golden_c1.npz     config 1: cube_mesh(6), N=3, initial_state, 10 LSRK4 steps
                    at stable_dt(m,3,1.0): final states and norms for every lift
                    mode, float64 and float32
  golden_setup.npz  mesh arrays + trace gathers (cube_mesh(2)) and the
                    reference operator tables for N=1..9
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from bbdg import mesh as msh, solver as sol  # noqa: E402  (the reference)
from bbdg.bernstein import BernsteinRefOps  # noqa: E402
from bbdg.nodal import NodalRefOps  # noqa: E402

OUT = Path(__file__).resolve().parent
MODES = ("factorized", "optimal", "dense")


def bb_cases():
    data = {}
    for N in range(1, 10):
        n = 2 if N <= 4 else 1
        m = msh.cube_mesh(n)
        mat = sol.Materials.homogeneous(m.K)
        ops = BernsteinRefOps.build(N)
        rng = np.random.default_rng(2024 + N)
        q = rng.standard_normal((4, m.K, ops.Np))
        dt = sol.stable_dt(m, N, 1.0)
        data[f"N{N}_n"] = n
        data[f"N{N}_dt"] = dt
        data[f"N{N}_q"] = q
        for dname, dtype in (("f64", np.float64), ("f32", np.float32)):
            sy = sol.WaveSystem(m, ops, mat, dtype=dtype)
            qq = q.astype(dtype)
            st = sol.FieldState(qq.copy(), "bernstein")
            data[f"N{N}_{dname}_vol"] = sy.volume_rhs(st)
            for mode in MODES:
                data[f"N{N}_{dname}_surf_{mode}"] = sy.surface_rhs(st, mode)
            data[f"N{N}_{dname}_rhs"] = sy.rhs(st)
            st2 = sol.lsrk4_step(sy, sol.FieldState(qq.copy(), "bernstein"), dt, "factorized")
            data[f"N{N}_{dname}_step"] = st2.q
    np.savez_compressed(OUT / "golden_bb.npz", **data)


def nodal_cases():
    data = {}
    for N in range(1, 10):
        m = msh.cube_mesh(2 if N <= 6 else 1)
        mat = sol.Materials.homogeneous(m.K)
        ops = NodalRefOps.build(N)
        rng = np.random.default_rng(4048 + N)
        q = rng.standard_normal((4, m.K, ops.Np))
        sy = sol.WaveSystem(m, ops, mat)
        dt = sol.stable_dt(m, N, 1.0)
        data[f"N{N}_q"] = q
        data[f"N{N}_dt"] = dt
        data[f"N{N}_vol"] = sy.volume_rhs(sol.FieldState(q.copy(), "nodal"))
        data[f"N{N}_rhs"] = sy.rhs(sol.FieldState(q.copy(), "nodal"))
        data[f"N{N}_step"] = sol.lsrk4_step(sy, sol.FieldState(q.copy(), "nodal"), dt).q
    np.savez_compressed(OUT / "golden_nodal.npz", **data)


def c1_case():
    m = msh.cube_mesh(6)
    mat = sol.Materials.homogeneous(m.K)
    N = 3
    dt = sol.stable_dt(m, N, 1.0)
    data = {"dt": dt, "K": m.K}
    for dname, dtype in (("f64", np.float64), ("f32", np.float32)):
        sy = sol.WaveSystem(m, BernsteinRefOps.build(N), mat, dtype=dtype)
        for mode in MODES:
            st = sol.initial_state(m, N, "bernstein", dtype=dtype)
            st = sol.integrate(sy, st, dt, 10, lift_mode=mode, energy_guard=None)
            data[f"q_final_{dname}_{mode}"] = st.q
            data[f"norm_{dname}_{mode}"] = float(np.linalg.norm(st.q.astype(np.float64)))
            data[f"l2err_{dname}_{mode}"] = sol.l2_error(sy, st)
    np.savez_compressed(OUT / "golden_c1.npz", **data)


def setup_case():
    from bbdg import bernstein as bb

    data = {}
    m = msh.cube_mesh(2)
    for k in ("vertices", "tets", "jac", "rst_dx", "normals", "jf", "etoe", "etof", "h_elem"):
        data[f"mesh_{k}"] = getattr(m, k)
    for N in range(1, 10):
        ops = BernsteinRefOps.build(N)
        fp = np.stack([ops.face_ref_points(f) for f in range(4)])
        g, b = msh.build_trace_maps(m, fp, ops.trace, ops.Np)
        if N <= 4:
            data[f"N{N}_gather"] = g
            data[f"N{N}_boundary"] = b
        data[f"N{N}_trace"] = ops.trace
        data[f"N{N}_L0"] = ops.lift.L0.toarray()
        data[f"N{N}_EL"] = ops.lift.EL.toarray()
        data[f"N{N}_dense_L"] = ops.dense_L
        data[f"N{N}_mass"] = ops.mass
        data[f"N{N}_dcols"] = np.stack([o.cols for o in ops.derivs.ops])
        data[f"N{N}_dvals"] = ops.derivs.values
        nops = NodalRefOps.build(N)
        for k in ("nodes", "Dr", "Ds", "Dt", "dense_L", "trace"):
            data[f"N{N}_nodal_{k}"] = getattr(nops, k)
        if N <= 4:
            fpn = np.stack([nops.face_ref_points(f) for f in range(4)])
            data[f"N{N}_nodal_gather"] = msh.build_trace_maps(m, fpn, nops.trace, nops.Np)[0]
    np.savez_compressed(OUT / "golden_setup.npz", **data)


if __name__ == "__main__":
    bb_cases()
    nodal_cases()
    c1_case()
    setup_case()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
