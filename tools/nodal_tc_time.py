"""Time the fp32 tcgen05 nodal rhs ("blocked") against the node-per-thread dense kernel on
cube_mesh(26) and check the two agree: python tools/nodal_tc_time.py [orders]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_1512_06025_b200 import Materials, NodalRefOps, WaveSystem, cube_mesh

orders = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1-9").replace("-", ",").split(",")]
if len(orders) == 2 and orders[1] > orders[0] + 1:
    orders = list(range(orders[0], orders[1] + 1))
mesh = cube_mesh(26)
for N in orders:
    sn = WaveSystem(mesh, NodalRefOps.build(N), Materials.homogeneous(mesh.K), np.float32)
    q = torch.randn((4, mesh.K, sn.Np), device="cuda", dtype=torch.float32)
    a, b = torch.empty_like(q), torch.empty_like(q)
    sn.rhs_into(q, a, "dense")
    sn.rhs_into(q, b, "blocked")
    torch.cuda.synchronize()
    err = float((a - b).norm() / a.norm())
    res = {}
    for mode, out in (("dense", a), ("blocked", b)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            sn.rhs_into(q, out, mode)
        e1.record()
        torch.cuda.synchronize()
        res[mode] = e0.elapsed_time(e1) / 5
    flops = 2 * mesh.K * 4 * (3 * sn.Np ** 2 + sn.Np * 4 * sn.ops.Nfp)
    print(f"N={N} dense {res['dense']:.3f} ms blocked {res['blocked']:.3f} ms "
          f"({flops / res['blocked'] / 1e9:.1f} useful TF/s, x{res['dense'] / res['blocked']:.2f}) rel_err {err:.2e}",
          flush=True)
