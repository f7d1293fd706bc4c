"""H2D bandwidth before/after running the stage kernels, blocking vs non-blocking."""
import json, sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def bw(fn, nbytes, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes / ((time.perf_counter() - t0) / reps) / 1e9


from paper_1512_06025_b200 import BernsteinRefOps, Materials, WaveSystem, cube_mesh
from paper_1512_06025_b200.solver import stable_dt
m = cube_mesh(40)
sy = WaveSystem(m, BernsteinRefOps.build(9), Materials.homogeneous(m.K), dtype=np.float32)
host = torch.empty((4, m.K, 220), dtype=torch.float32, pin_memory=True)
host.normal_()
nb = host.numel() * 4
out = {}
q = host.cuda()
out["nonblocking_before"] = bw(lambda: q.copy_(host, non_blocking=True), nb)
out["blocking_before"] = bw(lambda: q.copy_(host), nb)
tmp, res = torch.empty_like(q), torch.empty_like(q)
dt = stable_dt(m, 9, 1.0)
for _ in range(3):
    sy.step_into(q, tmp, res, dt, "optimal")
torch.cuda.synchronize()
out["nonblocking_after_steps"] = bw(lambda: q.copy_(host, non_blocking=True), nb)
out["blocking_after_steps"] = bw(lambda: q.copy_(host), nb)
out["d2h_nonblocking_after"] = bw(lambda: host.copy_(q, non_blocking=True), nb)
q.normal_()
out["h2d_after_q_normal"] = bw(lambda: q.copy_(host, non_blocking=True), nb)
out["d2h_after_q_normal"] = bw(lambda: host.copy_(q, non_blocking=True), nb)
print(json.dumps(out))
