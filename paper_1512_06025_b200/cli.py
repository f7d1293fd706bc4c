"""Command-line driver for the drop-in solver (reference ``cli.py``: the ``solve`` and
``convergence`` subcommands).

    python -m paper_1512_06025_b200.cli solve --n 3 --mesh 4 --tmax 1.0 [--basis both] [--save-state]
    python -m paper_1512_06025_b200.cli convergence --n 1..3 --meshes 2,4,8 --tmax 0.5

Same arguments, outputs and exit codes as the reference (``cli.py:281-424``): CSV files with 17
significant digits (``solve_<basis>_N<k>.csv``: step,tau,l2_error_p,energy; ``convergence.csv``:
basis,N,meshes,errors,observed_order), the mesh summary and final-error lines on stdout, exit 0 on
success, 1 when the energy guard aborts an unstable run, 2 on a usage error.  Every time step runs
on the GPU; the state stays in HBM and the error / energy samples are evaluated there too
(bbdg_error_l2, bbdg_energy), so a run costs one 8-byte read-back per sample.  The kernels are
deterministic (owner-computes, fixed-order reductions), so reruns are byte-identical.

The operator-diagnostic subcommands of the reference (``ops``, ``check``: conditioning, extrema,
eigen identities, op counts) are out of scope and exit with code 2.
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np

_FMT = "%.17g"


def _fmt(x) -> str:
    if isinstance(x, str):
        return x
    if isinstance(x, (int, np.integer)):
        return str(int(x))
    return _FMT % float(x)


def _write_csv(path, header, rows):
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    with open(path, "w") as fh:
        fh.write(",".join(header) + "\n")
        for row in rows:
            fh.write(",".join(_fmt(x) for x in row) + "\n")


def _degrees(text: str) -> list[int]:
    if ".." in text:
        lo, hi = text.split("..")
        out = list(range(int(lo), int(hi) + 1))
    else:
        out = [int(tok) for tok in text.split(",") if tok]
    if not out:
        raise ValueError("empty degree range")
    return out


def _bases(arg: str) -> list[str]:
    return ["bernstein", "nodal"] if arg == "both" else [arg]


def _system(mesh, N, basis, nodes, dtype):
    from . import BernsteinRefOps, Materials, NodalRefOps, WaveSystem

    ops = BernsteinRefOps.build(N) if basis == "bernstein" else NodalRefOps.build(N, nodes)
    return WaveSystem(mesh, ops, Materials.homogeneous(mesh.K), dtype=dtype)


def _device_state(state):
    import torch

    from . import FieldState

    return FieldState(torch.as_tensor(state.q).cuda(), state.basis, state.time)


def cmd_solve(args) -> int:
    from . import ErrorFunctional, cube_mesh, discrete_energy, initial_state, integrate, load_mesh_ascii, save_state
    from . import stable_dt
    from .mesh import mesh_stats

    degrees = _degrees(args.n)
    if len(degrees) != 1:
        raise ValueError("solve expects exactly one degree")
    N = degrees[0]
    dtype = np.float32 if args.precision == "single" else np.float64
    os.makedirs(args.out, exist_ok=True)
    for basis in _bases(args.basis):
        m = load_mesh_ascii(args.mesh_file) if args.mesh_file else cube_mesh(args.mesh)
        system = _system(m, N, basis, args.nodes, dtype)
        print("mesh: " + " ".join(f"{k}={_fmt(v)}" for k, v in mesh_stats(m).items()))
        state = _device_state(initial_state(m, N, basis, dtype=dtype, node_kind=args.nodes))
        err = ErrorFunctional(m, system.ops_double)
        series = []
        if args.tmax <= 0.0:
            series.append((0, 0.0, err(state), discrete_energy(system, state)))
            nsteps = 0
        else:
            dt = stable_dt(m, N, float(system.mat.c.max()), args.cfl)
            nsteps = int(np.ceil(args.tmax / dt))
            dt = args.tmax / nsteps
            every = max(1, nsteps // args.samples)

            def sample(step, s):
                if step % every == 0 or step == nsteps:
                    series.append((step, s.time, err(s), discrete_energy(system, s)))

            try:
                state = integrate(system, state, dt, nsteps, lift_mode=args.lift_mode, callback=sample)
            except RuntimeError as exc:
                print(f"aborted: {exc}", file=sys.stderr)
                return 1
        path = os.path.join(args.out, f"solve_{basis}_N{N}.csv")
        _write_csv(path, ["step", "tau", "l2_error_p", "energy"], series)
        print(f"{basis}: N={N} steps={nsteps} final_error={_fmt(series[-1][2])} wrote {path}")
        if args.save_state:
            save_state(os.path.join(args.out, f"state_{basis}_N{N}.bin"), state)
    return 0


def cmd_convergence(args) -> int:
    from . import cube_mesh, initial_state, integrate, l2_error, stable_dt

    degrees = _degrees(args.n)
    meshes = [int(tok) for tok in args.meshes.split(",") if tok]
    if len(meshes) < 2:
        raise ValueError("need at least two mesh resolutions")
    os.makedirs(args.out, exist_ok=True)
    rows = []
    for basis in _bases(args.basis):
        for N in degrees:
            errs = []
            for n in meshes:
                m = cube_mesh(n)
                system = _system(m, N, basis, args.nodes, np.float64)
                state = _device_state(initial_state(m, N, basis, node_kind=args.nodes))
                nsteps = int(np.ceil(args.tmax / stable_dt(m, N, 1.0, args.cfl)))
                state = integrate(system, state, args.tmax / nsteps, nsteps, args.lift_mode)
                errs.append(l2_error(system, state))
            # observed order: slope of log(error) against log(h), h = 1/n
            order = float(np.polyfit(np.log([1.0 / n for n in meshes]), np.log(errs), 1)[0])
            rows.append((basis, N, ";".join(str(n) for n in meshes), " ".join(_fmt(e) for e in errs), order))
            print(f"{basis} N={N}: errors={errs} observed_order={order:.2f}")
    path = os.path.join(args.out, "convergence.csv")
    _write_csv(path, ["basis", "N", "meshes", "errors", "observed_order"], rows)
    print(f"wrote {path}")
    return 0


def _out_of_scope(command) -> int:
    print(f"error: '{command}' (operator diagnostics) is not part of this drop-in; use the reference "
          "package for it", file=sys.stderr)
    return 2


def _parser():
    p = argparse.ArgumentParser(prog="bbdg", description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    sub = p.add_subparsers(dest="command", required=True)

    def common(sp):
        sp.add_argument("--n", default="1..9", help="degree or range, e.g. 4 or 1..9")
        sp.add_argument("--basis", choices=["bernstein", "nodal", "both"], default="bernstein")
        sp.add_argument("--nodes", choices=["warp_blend", "equispaced"], default="warp_blend")
        sp.add_argument("--out", default="out", help="output directory")
        sp.add_argument("--seed", type=int, default=2024)
        sp.add_argument("--mesh", type=int, default=4, help="cells per axis of the cube mesh")
        sp.add_argument("--mesh-file", default=None, help="ASCII mesh file instead of --mesh")
        sp.add_argument("--cfl", type=float, default=0.5)
        sp.add_argument("--lift-mode", choices=["dense", "factorized", "optimal"], default="factorized")

    sp = sub.add_parser("solve", help="wave equation run")
    common(sp)
    sp.add_argument("--tmax", type=float, default=1.0)
    sp.add_argument("--precision", choices=["double", "single"], default="double")
    sp.add_argument("--samples", type=int, default=50, help="time-series sample count")
    sp.add_argument("--save-state", action="store_true")
    sp.set_defaults(func=cmd_solve, n="3")

    sp = sub.add_parser("convergence", help="mesh refinement sweep")
    common(sp)
    sp.add_argument("--meshes", default="2,4", help="comma-separated cells per axis")
    sp.add_argument("--tmax", type=float, default=0.5)
    sp.set_defaults(func=cmd_convergence, n="2")

    for name in ("ops", "check"):
        sub.add_parser(name, help="operator diagnostics (out of scope of this drop-in)")
    return p


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else list(argv)
    if argv and argv[0] in ("ops", "check"):
        return _out_of_scope(argv[0])
    parser = _parser()
    args = parser.parse_args(argv)
    try:
        return args.func(args)
    except (ValueError, FileNotFoundError) as exc:
        parser.exit(2, f"error: {exc}\n")


if __name__ == "__main__":
    sys.exit(main())
