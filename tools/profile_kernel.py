"""Launch one hot-path kernel a few times for ncu (no timing printed -- numbers
taken under a profiler are never bench values).

    python tools/profile_kernel.py --N 9 --dtype f32 --op stage --lift optimal [--n 26] [--reps 3]
"""

import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=9)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--op", default="stage", choices=["stage", "volume", "surface", "rhs", "update"])
    ap.add_argument("--lift", default="optimal")
    ap.add_argument("--basis", default="bernstein")
    ap.add_argument("--n", type=int, default=26)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--box", default=None, help="nx,ny,nz: a device-built BoxMesh (e.g. the bench's fill mesh)")
    ap.add_argument("--xblock", type=int, default=1, help="element order of the box (x-layers per slab)")
    a = ap.parse_args()
    import torch

    from paper_1512_06025_b200 import BernsteinRefOps, Materials, NodalRefOps, WaveSystem, cube_mesh
    from paper_1512_06025_b200.solver import RK4A, RK4B, _device_update

    ops = BernsteinRefOps.build(a.N) if a.basis == "bernstein" else NodalRefOps.build(a.N)
    dt = np.float32 if a.dtype == "f32" else np.float64
    if a.box:
        from paper_1512_06025_b200.mesh_device import BoxMesh

        m = BoxMesh(*[int(x) for x in a.box.split(",")], xblock=a.xblock)
        sy = WaveSystem(m, ops, Materials(np.float64(1.0), np.float64(1.0)), dtype=dt, legacy_records=False)
    else:
        m = cube_mesh(a.n)
        sy = WaveSystem(m, ops, Materials.homogeneous(m.K), dtype=dt)
    g = torch.Generator(device="cuda").manual_seed(1)
    q = torch.randn((4, m.K, sy.Np), dtype=sy.torch_dtype, device="cuda", generator=g)
    q2, res = torch.empty_like(q), torch.randn_like(q)
    rhs = q2   # (volume / surface / rhs write it; no fourth state buffer: the fill boxes hold three)
    for _ in range(a.reps):
        if a.op == "stage":
            sy.stage_into(q, q2, res, RK4A[1], RK4B[1], 1e-3, a.lift)
        elif a.op == "volume":
            sy.volume_into(q, rhs)
        elif a.op == "surface":
            sy.surface_into(q, rhs, a.lift)
        elif a.op == "rhs":
            sy.rhs_into(q, rhs, a.lift)
        else:
            _device_update(q2, res, q, RK4A[1], RK4B[1], 1e-3)   # as bench.py's breakdown
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
