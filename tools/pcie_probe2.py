"""Why is H2D slower inside the e2e probe than in pcie_bw? Same copy, different process histories."""
import json, os, sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def bw(host, dev, reps=5):
    dev.copy_(host, non_blocking=True); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        dev.copy_(host, non_blocking=True)
    b.record(); torch.cuda.synchronize()
    return host.numel() * host.element_size() / (a.elapsed_time(b) / reps * 1e-3) / 1e9


out = {"affinity": len(os.sched_getaffinity(0))}
n = 338 << 20
h = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
out["fresh_untouched"] = bw(h, d)
h.normal_()
out["fresh_touched"] = bw(h, d)
from paper_1512_06025_b200 import BernsteinRefOps, Materials, WaveSystem, cube_mesh
m = cube_mesh(40)
sy = WaveSystem(m, BernsteinRefOps.build(9), Materials.homogeneous(m.K), dtype=np.float32)
out["old_buffer_after_setup"] = bw(h, d)
h2 = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
out["new_buffer_after_setup"] = bw(h2, d)
h2.normal_()
out["new_buffer_touched"] = bw(h2, d)
h3 = torch.empty((4, m.K, 220), dtype=torch.float32, pin_memory=True)
h3.normal_()
d3 = torch.empty_like(h3, device="cuda")
out["shaped_like_probe"] = bw(h3, d3)
print(json.dumps(out))
