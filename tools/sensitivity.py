"""Finite-precision sensitivity study on the GPU (BASELINE configs[3], paper Figs. 5-6).

    python tools/sensitivity.py [--out profiles/round1_sensitivity.json] [--tmax 25]

A. Spatial convergence: L2 pressure error of the standing wave at tau = 0.5 on
   cube_mesh(n), n in (2, 4, 8, 16), N = 1..9, float64 vs float32 (optimal lift),
   with observed orders log2(e_n / e_2n).
B. Long-time roundoff sensitivity: error trajectories to tau = tmax on
   cube_mesh(4) for N in (3, 5, 7, 9), float32 vs float64, sampled 100 times.
All states stay on the device (device error functional, no host copies of q).
The CPU reference values for the small cases are in tests/golden/golden_sensitivity.npz.
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def run(n, N, dtype, tau, samples=0):
    import torch

    from paper_1512_06025_b200 import (BernsteinRefOps, ErrorFunctional, FieldState, Materials, WaveSystem,
                                       cube_mesh, initial_state, integrate, stable_dt)

    m = cube_mesh(n)
    sy = WaveSystem(m, BernsteinRefOps.build(N), Materials.homogeneous(m.K), dtype=dtype)
    st = initial_state(m, N, "bernstein", dtype=dtype)
    dt = stable_dt(m, N, 1.0)
    nst = int(np.ceil(tau / dt))
    ef = ErrorFunctional(m, sy.ops_double)
    traj = []
    every = max(1, nst // samples) if samples else 0

    def cb(step, s):
        if every and step % every == 0:
            traj.append((step * tau / nst, ef(s)))

    st = integrate(sy, FieldState(torch.as_tensor(st.q).cuda(), "bernstein"), tau / nst, nst, "optimal",
                   callback=cb if samples else None, energy_guard=None)
    return ef(st), nst, traj


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/round1_sensitivity.json")
    ap.add_argument("--tmax", type=float, default=25.0)
    a = ap.parse_args()
    res = {"convergence": {}, "trajectories": {}}
    t0 = time.time()
    for dname, dt in (("f64", np.float64), ("f32", np.float32)):
        for N in range(1, 10):
            row = {}
            for n in (2, 4, 8, 16):
                e, nst, _ = run(n, N, dt, 0.5)
                row[n] = e
            orders = {f"{n}->{2 * n}": float(np.log2(row[n] / row[2 * n])) for n in (2, 4, 8)}
            res["convergence"][f"{dname}_N{N}"] = {"errors": {str(k): v for k, v in row.items()}, "orders": orders}
            print(f"{dname} N={N} " + " ".join(f"n={k}:{v:.3e}" for k, v in row.items()) + "  orders "
                  + " ".join(f"{v:.2f}" for v in orders.values()), flush=True)
    for N in (3, 5, 7, 9):
        for dname, dt in (("f64", np.float64), ("f32", np.float32)):
            e, nst, traj = run(4, N, dt, a.tmax, samples=100)
            res["trajectories"][f"{dname}_N{N}"] = {"steps": nst, "tau": [t for t, _ in traj],
                                                    "error": [x for _, x in traj]}
            errs = np.array([x for _, x in traj])
            print(f"traj {dname} N={N} n=4 steps={nst} err min {errs.min():.3e} max {errs.max():.3e} "
                  f"final {e:.3e}", flush=True)
    res["wall_s"] = time.time() - t0
    Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
