"""Wall-clock lsrk4_step on a host numpy state (pinned vs pageable), cube_mesh(n), fp32:
python tools/e2e_time.py [orders] [n]."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1512_06025_b200 import BernsteinRefOps, FieldState, Materials, WaveSystem, cube_mesh, lsrk4_step  # noqa
from paper_1512_06025_b200 import stable_dt  # noqa: E402

orders = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "5,9").split(",")]
m = cube_mesh(int(sys.argv[2]) if len(sys.argv) > 2 else 40)
print("cpus", os.cpu_count(), "threads", os.environ.get("BBDG_COPY_THREADS"), flush=True)
for N in orders:
    sy = WaveSystem(m, BernsteinRefOps.build(N), Materials.homogeneous(m.K), np.float32)
    dt = stable_dt(m, N, 1.0)
    pinned = torch.empty((4, m.K, sy.Np), dtype=torch.float32, pin_memory=True)
    pinned.normal_()
    page = pinned.numpy().copy()
    row = {}
    for kind, arr in (("pinned", pinned.numpy()), ("pageable", page)):
        st = FieldState(arr, "bernstein")
        lsrk4_step(sy, st, dt, "optimal")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            lsrk4_step(sy, st, dt, "optimal")
        row[kind] = (time.perf_counter() - t0) * 1e3 / 3
    gd = 5 * 4 * m.K * sy.Np / 1e9
    print(f"N={N} state {page.nbytes / 1e9:.2f} GB  pinned {row['pinned']:.1f} ms ({gd / row['pinned'] * 1e3:.1f} GDOF/s)"
          f"  pageable {row['pageable']:.1f} ms ({gd / row['pageable'] * 1e3:.1f} GDOF/s)", flush=True)
    del sy, pinned, page
    torch.cuda.empty_cache()
