"""Final float64 states of the finite-precision study's convergence runs (BASELINE configs[3]),
produced by running the REFERENCE package itself on the CPU:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_sens_states.py

For cube_mesh(2), N = 1..9: the standing wave from initial_state, integrated to tau = 0.5 with
stable_dt(m, N, 1.0) rounded to land on tau (factorized lift, as make_sensitivity.conv_case),
stored as ``q_N{N}`` (4, 48, Np) with the step count ``nst_N{N}`` and the L2 error ``err_N{N}``.
The GPU test compares whole states at the north-star float64 tolerance (1e-12 relative L2)
instead of only the scalar error functional.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from bbdg import mesh as msh, solver as sol  # noqa: E402  (the reference)
from bbdg.bernstein import BernsteinRefOps  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    data = {}
    m = msh.cube_mesh(2)
    tau = 0.5
    for N in range(1, 10):
        t0 = time.time()
        sy = sol.WaveSystem(m, BernsteinRefOps.build(N), sol.Materials.homogeneous(m.K))
        st = sol.initial_state(m, N, "bernstein")
        dt = sol.stable_dt(m, N, 1.0)
        nst = int(np.ceil(tau / dt))
        st = sol.integrate(sy, st, tau / nst, nst, energy_guard=None)
        data[f"q_N{N}"] = st.q
        data[f"nst_N{N}"] = np.array(nst)
        data[f"err_N{N}"] = np.array(sol.l2_error(sy, st))
        print(f"N={N}: {nst} steps, error {float(data[f'err_N{N}']):.6e} ({time.time() - t0:.1f} s)", flush=True)
    np.savez_compressed(OUT / "golden_sens_states.npz", **data)


if __name__ == "__main__":
    main()
