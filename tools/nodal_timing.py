"""BB fused stage / rhs vs nodal NPT (dense) vs nodal blocked (tensor-core) rhs on cube_mesh(26)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_1512_06025_b200 import BernsteinRefOps, Materials, NodalRefOps, WaveSystem, cube_mesh

    m = cube_mesh(int(sys.argv[1]) if len(sys.argv) > 1 else 26)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def t(fn, reps=5):
        fn()
        tot = 0.0
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            b.synchronize()
            tot += a.elapsed_time(b)
        return tot / reps

    for dt in (np.float32, np.float64):
        for N in range(1, 10):
            sb = WaveSystem(m, BernsteinRefOps.build(N), Materials.homogeneous(m.K), dtype=dt)
            sn = WaveSystem(m, NodalRefOps.build(N), Materials.homogeneous(m.K), dtype=dt)
            q = torch.randn((4, m.K, sb.Np), device="cuda", dtype=sb.torch_dtype)
            r = torch.empty_like(q)
            tb = t(lambda: sb.rhs_into(q, r, "optimal"))
            tn = t(lambda: sn.rhs_into(q, r, "dense"))
            tk = t(lambda: sn.rhs_into(q, r, "blocked"))
            fl = 2 * m.K * 4 * (3 * sb.Np ** 2 + sb.Np * 4 * sb.ops.Nfp)
            print(f"{np.dtype(dt).name} N={N} bb_rhs {tb:.3f} ms  nodal_npt {tn:.3f}  nodal_blocked {tk:.3f} "
                  f"({fl / tk / 1e9:.1f} TFLOP/s useful)  bb/blocked speedup {tk / tb:.2f}", flush=True)
            del sb, sn, q, r
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
