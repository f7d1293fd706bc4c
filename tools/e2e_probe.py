"""Break down the end-to-end lsrk4_step on a pinned host state (N, dtype, cube_mesh(n)):
device-only step, plain H2D + step + D2H, and the chunk-pipelined bbdg_step_host.

    python tools/e2e_probe.py --N 9 --n 40
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=9)
    ap.add_argument("--n", type=int, default=40)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--max-chunks", type=int, default=48)
    ap.add_argument("--split", default="1", help="comma list: chunk = band / split")
    a = ap.parse_args()
    import torch

    from paper_1512_06025_b200 import BernsteinRefOps, FieldState, Materials, WaveSystem, cube_mesh, lsrk4_step
    from paper_1512_06025_b200.solver import host_chunk_plan, stable_dt

    dtype = np.float32 if a.dtype == "f32" else np.float64
    m = cube_mesh(a.n)
    sy = WaveSystem(m, BernsteinRefOps.build(a.N), Materials.homogeneous(m.K), dtype=dtype)
    dt = stable_dt(m, a.N, 1.0)
    host = torch.empty((4, m.K, sy.Np), dtype=sy.torch_dtype, pin_memory=True)
    host.normal_()
    q = host.cuda()
    tmp, res = torch.empty_like(q), torch.empty_like(q)
    out = {}

    def wall(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3 / reps

    out["device_step_ms"] = wall(lambda: sy.step_into(q, tmp, res, dt, "optimal"))
    out["h2d_ms"] = wall(lambda: q.copy_(host))
    out["d2h_ms"] = wall(lambda: host.copy_(q))
    st = FieldState(host.numpy(), "bernstein")
    sy._chunks = None
    out["plain_ms"] = wall(lambda: lsrk4_step(sy, st, dt, "optimal"))
    band = int(np.abs(m.etoe - np.arange(m.K)[:, None]).max())
    for sp in map(int, a.split.split(",")):
        sy._chunks = host_chunk_plan(m.etoe, sy.Np, np.dtype(dtype).itemsize, max_chunks=a.max_chunks,
                                     chunk=None if sp == 1 else -(-band // sp))
        out[f"split{sp}"] = {"chunks": len(sy._chunks[0]) - 1, "reach": sy._chunks[1],
                             "pipelined_ms": wall(lambda: lsrk4_step(sy, st, dt, "optimal"))}
    # the enqueue cost alone (host time of the C call before the final sync)
    from paper_1512_06025_b200 import _lib
    b, r = sy._chunks
    hs, ds = sy._copy_streams
    cs = torch.cuda.current_stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.check(sy._lib.bbdg_step_host(sy._ctx, host.data_ptr(), q.data_ptr(), tmp.data_ptr(), res.data_ptr(), dt,
                                      1, b.ctypes.data, len(b) - 1, r, cs.cuda_stream, hs.cuda_stream,
                                      ds.cuda_stream))
    out["enqueue_ms"] = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    out["after_sync_ms"] = (time.perf_counter() - t0) * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
