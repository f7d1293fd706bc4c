import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1512_06025_b200 import *
from paper_1512_06025_b200.solver import RK4A, RK4B
for n in (8, 12, 16, 20):
    m = cube_mesh(n)
    for N in (1, 2, 3):
        sy = WaveSystem(m, BernsteinRefOps.build(N), Materials.homogeneous(m.K))
        q = torch.randn((4, m.K, sy.Np), dtype=torch.float64, device="cuda")
        a, b = torch.empty_like(q), torch.empty_like(q)
        sy.rhs_into(q, a, "optimal"); sy.rhs_into(q, b, "factorized")
        res1, res2 = torch.zeros_like(q), torch.zeros_like(q)
        o1, o2 = torch.empty_like(q), torch.empty_like(q)
        sy.stage_into(q, o1, res1, RK4A[1], RK4B[1], 1e-3, "optimal"); sy.stage_into(q, o2, res2, RK4A[1], RK4B[1], 1e-3, "factorized")
        d = (a-b).norm()/b.norm(); d2=(o1-o2).norm()/o2.norm()
        bad = ((a-b).abs().amax(dim=(0,2)) > 1e-8*b.abs().max()).nonzero().flatten()
        print(n, N, m.K, f"rhs {d:.2e} stage {d2:.2e}", "bad elems", bad[:10].tolist(), len(bad), flush=True)
