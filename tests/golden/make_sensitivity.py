"""Reference error trajectories for the finite-precision study (BASELINE configs[3], C4),
produced by running the REFERENCE package itself on the CPU:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_sensitivity.py [--quick]

Run in the build container (the reference is not on the GPU box); the output
``golden_sensitivity.npz`` is committed.  Contents:

  conv_{dtype}_n{n}_N{N}   L2 pressure error at tau = 0.5 of the standing wave
                           (initial_state, stable_dt(m, N, 1.0) rounded to land on
                           tau), Bernstein basis, factorized lift, cube_mesh(n),
                           float64 and float32; n in (2, 4), N = 1..9 (n = 4 up to
                           N = 6 unless --full); plus conv_f64_n16_N1, where the
                           reference scheme itself diverges (N = 1, cfl = 0.5)
  band_{basis}             criterion 8 of the reference acceptance suite
                           (test_acceptance.py:222-250): float32, N = 5,
                           cube_mesh(4), tau <= 5, error sampled every nst // 100
                           steps, Bernstein and nodal
  band_tau                 the sample times
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from bbdg import mesh as msh, solver as sol  # noqa: E402  (the reference)
from bbdg.bernstein import BernsteinRefOps  # noqa: E402
from bbdg.nodal import NodalRefOps  # noqa: E402

OUT = Path(__file__).resolve().parent


def conv_case(n, N, dtype, tau=0.5):
    m = msh.cube_mesh(n)
    sy = sol.WaveSystem(m, BernsteinRefOps.build(N), sol.Materials.homogeneous(m.K), dtype=dtype)
    st = sol.initial_state(m, N, "bernstein", dtype=dtype)
    dt = sol.stable_dt(m, N, 1.0)
    nst = int(np.ceil(tau / dt))
    st = sol.integrate(sy, st, tau / nst, nst, energy_guard=None)
    return sol.l2_error(sy, st)


def band():
    N, n, tmax = 5, 4, 5.0
    m = msh.cube_mesh(n)
    mat = sol.Materials.homogeneous(m.K)
    dt = sol.stable_dt(m, N, 1.0)
    nst = int(np.ceil(tmax / dt))
    dt = tmax / nst
    every = max(1, nst // 100)
    out = {}
    for basis, Ops in (("bernstein", BernsteinRefOps), ("nodal", NodalRefOps)):
        sy = sol.WaveSystem(m, Ops.build(N), mat, dtype=np.float32)
        st = sol.initial_state(m, N, basis, dtype=np.float32)
        err = sol.ErrorFunctional(m, sy.ops_double)
        samples, taus = [], []

        def cb(step, s, err=err, samples=samples, taus=taus):
            if step % every == 0:
                samples.append(err(s))
                taus.append(step * dt)

        sol.integrate(sy, st, dt, nst, callback=cb)
        out[f"band_{basis}"] = np.array(samples)
        out["band_tau"] = np.array(taus)
    out["band_meta"] = np.array([N, n, tmax, nst, every], dtype=np.float64)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true", help="n = 4 for every N (slow)")
    ap.add_argument("--no-band", action="store_true")
    a = ap.parse_args()
    data = {}
    for dname, dtype in (("f64", np.float64), ("f32", np.float32)):
        for n in (2, 4):
            for N in range(1, 10):
                if n == 4 and N > 6 and not a.full:
                    continue
                t0 = time.time()
                data[f"conv_{dname}_n{n}_N{N}"] = np.array(conv_case(n, N, dtype))
                print(f"conv {dname} n={n} N={N}: {float(data[f'conv_{dname}_n{n}_N{N}']):.6e} "
                      f"({time.time() - t0:.1f} s)", flush=True)
    # the reference scheme itself diverges for N = 1 at cfl = 0.5 on cube_mesh(16) (error ~1.1):
    # pinned so the GPU reproduces it rather than 'fixing' it
    data["conv_f64_n16_N1"] = np.array(conv_case(16, 1, np.float64))
    print(f"conv f64 n=16 N=1: {float(data['conv_f64_n16_N1']):.6e}", flush=True)
    if not a.no_band:
        t0 = time.time()
        data.update(band())
        print(f"band: {time.time() - t0:.1f} s", flush=True)
    np.savez_compressed(OUT / "golden_sensitivity.npz", **data)


if __name__ == "__main__":
    main()
