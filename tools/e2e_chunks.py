"""Pinned-state lsrk4_step wall time vs the host pipeline's chunk count (cube_mesh(40), fp32):
python tools/e2e_chunks.py [orders] [max_chunks,...]."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1512_06025_b200 import BernsteinRefOps, FieldState, Materials, WaveSystem, cube_mesh, lsrk4_step  # noqa
from paper_1512_06025_b200 import stable_dt  # noqa: E402
from paper_1512_06025_b200.solver import host_chunk_plan  # noqa: E402

orders = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "4,8,9").split(",")]
counts = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "12,24,48,96").split(",")]
m = cube_mesh(40)
for N in orders:
    sy = WaveSystem(m, BernsteinRefOps.build(N), Materials.homogeneous(m.K), np.float32)
    dt = stable_dt(m, N, 1.0)
    pinned = torch.empty((4, m.K, sy.Np), dtype=torch.float32, pin_memory=True)
    pinned.normal_()
    row = []
    for c in counts:
        sy._chunks = host_chunk_plan(m.etoe, sy.Np, 4, max_chunks=c)
        if sy._chunks is None:
            row.append(f"{c}:-")
            continue
        st = FieldState(pinned.numpy(), "bernstein")
        lsrk4_step(sy, st, dt, "optimal")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            lsrk4_step(sy, st, dt, "optimal")
        row.append(f"{c}({len(sy._chunks[0]) - 1},r{sy._chunks[1]}):{(time.perf_counter() - t0) * 1e3 / 3:.1f}")
    print(f"N={N}", " ".join(row), flush=True)
    del sy, pinned
    torch.cuda.empty_cache()
