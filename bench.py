"""Benchmark: GDOF-updates/s per RK stage of the BB-DG hot path, N = 1..9.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--dtype f32|f64] [--n 26] [--orders 1-9] [--lift optimal]

Workload (BASELINE.json configs[1]): cube_mesh(26) = 105,456 tets, Bernstein
basis, orders N = 1..9, homogeneous materials, standard-normal synthetic
state (seed 2024).  One bench "step" = one fused LSRK4 stage (volume +
surface + update, ``bbdg_lsrk_stage``) at every order of the sweep; the
headline value is the sweep's whole-job DOF throughput
sum_N 4 K Np(N) / sum_N t_stage(N).  L2 (126 MB) is flushed with a 256 MB
write before every timed launch, outside the event window.

Per-order extras: volume / surface (3 lift modes) / update kernels timed
separately, the nodal NPT comparison, and the roofline fraction of each
against MEASURED_PEAKS.json.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "GDOF-updates/sec per RK stage vs order N=1..9; per-kernel % HBM/FLOP roofline"
UNIT = "GDOF/s"


def np_of(N):
    return (N + 1) * (N + 2) * (N + 3) // 6


def nfp_of(N):
    return (N + 1) * (N + 2) // 2


def parse_orders(s):
    out = []
    for part in s.split(","):
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


# ---------------------------------------------------------------------- algorithmic byte model
def stage_bytes(N, s, K):
    """Fused stage: q_in, q_out, res r/w (16 Np) + neighbour traces (16 Nfp) + geometry (36) words
    + 20 B connectivity per element."""
    return K * ((16 * np_of(N) + 16 * nfp_of(N) + 36) * s + 20)


def volume_bytes(N, s, K):
    return K * (8 * np_of(N) + 12) * s


def surface_bytes(N, s, K):
    return K * ((8 * np_of(N) + 16 * nfp_of(N) + 36) * s + 20)


def update_bytes(N, s, K):
    return K * 20 * np_of(N) * s


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------- clocks sampler
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")
        for ln in getattr(self, "lines", []):
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------- GPU arm
def build_system(mesh, N, dtype, basis="bernstein"):
    from paper_1512_06025_b200 import BernsteinRefOps, Materials, NodalRefOps, WaveSystem

    ops = BernsteinRefOps.build(N) if basis == "bernstein" else NodalRefOps.build(N)
    return WaveSystem(mesh, ops, Materials.homogeneous(mesh.K), dtype=dtype)


def time_launches(torch, fn, flush, reps):
    """Mean device time (ms) of fn over reps launches, L2 flushed before each (outside the events)."""
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


def run_ours(args, rank, world):
    import torch

    from paper_1512_06025_b200 import cube_mesh, lsrk4_step, FieldState, stable_dt
    from paper_1512_06025_b200.solver import RK4A, RK4B

    dev = int(os.environ.get("LOCAL_RANK", rank)) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dtype = np.float32 if args.dtype == "f32" else np.float64
    s = 4 if args.dtype == "f32" else 8
    if world > 1:
        # weak scaling: a box of world x n^3 cells, one n^3-cell x-slab per rank
        from paper_1512_06025_b200.mesh import box_mesh

        mesh = box_mesh(world * args.n, args.n, args.n, lo=(-0.5 * world, -0.5, -0.5), hi=(0.5 * world, 0.5, 0.5))
    else:
        mesh = cube_mesh(args.n)
    K = mesh.K // world
    orders = parse_orders(args.orders)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    gen = torch.Generator(device="cuda").manual_seed(2024 + rank)
    systems = {}
    for N in orders:
        if world > 1:
            from paper_1512_06025_b200 import BernsteinRefOps, Materials
            from paper_1512_06025_b200.dist import DistWaveSystem

            sy = DistWaveSystem(mesh, BernsteinRefOps.build(N), Materials.homogeneous(mesh.K), dtype, rank, world,
                                align=6 * args.n * args.n)
            sy.Np, sy.torch_dtype = sy.local.Np, sy.local.torch_dtype
        else:
            sy = build_system(mesh, N, dtype)
        q = torch.randn((4, K, sy.Np), generator=gen, device="cuda", dtype=sy.torch_dtype)
        systems[N] = dict(sy=sy, q=q, q2=torch.empty_like(q), res=torch.randn_like(q), rhs=torch.empty_like(q),
                          dt=stable_dt(mesh, N, 1.0))

    def stage(N):
        d = systems[N]
        d["sy"].stage_into(d["q"], d["q2"], d["res"], RK4A[1], RK4B[1], d["dt"], args.lift)

    # warm-up
    for _ in range(args.warmup):
        for N in orders:
            stage(N)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()

    # timed region: K steps, each one fused stage at every order, L2 flushed between launches
    per_n = {N: 0.0 for N in orders}
    with Clocks(dev) as clk:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            for N in orders:
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                stage(N)
                b.record()
                b.synchronize()
                per_n[N] += a.elapsed_time(b)
        torch.cuda.synchronize()
    total_ms = sum(per_n.values())
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
        torch.distributed.barrier()
    dofs_per_step = sum(4 * K * np_of(N) for N in orders)
    value = world * dofs_per_step * args.steps / (total_ms * 1e-3) / 1e9

    peak, peak_kind = load_peaks()
    out = dict(per_order={}, value=value, ms_per_step=total_ms / args.steps, clocks=clk.summary())
    # per-order stage rooflines + kernel breakdown (outside the headline timing)
    dominant = None
    for N in orders:
        d = systems[N]
        t_stage = per_n[N] / args.steps
        bytes_ = stage_bytes(N, s, K)
        ach = bytes_ / (t_stage * 1e-3) / 1e9
        row = {"gdofs_stage": 4 * K * np_of(N) / (t_stage * 1e-3) / 1e9, "stage_ms": t_stage,
               "stage_gbs": ach, "stage_frac": ach / peak}
        if not args.quick and world == 1:
            sy, q, rhs = d["sy"], d["q"], d["rhs"]
            reps = max(3, args.steps)
            tv = time_launches(torch, lambda: sy.volume_into(q, rhs), flush, reps)
            row["volume_ms"], row["volume_frac"] = tv, volume_bytes(N, s, K) / (tv * 1e-3) / 1e9 / peak
            for mode in ("factorized", "optimal", "dense"):
                ts = time_launches(torch, lambda: sy.surface_into(q, rhs, mode), flush, reps)
                row[f"surface_{mode}_ms"] = ts
                row[f"surface_{mode}_frac"] = surface_bytes(N, s, K) / (ts * 1e-3) / 1e9 / peak
            from paper_1512_06025_b200.solver import _device_update
            tu = time_launches(torch, lambda: _device_update(d["q2"], d["res"], rhs, RK4A[1], RK4B[1], d["dt"]),
                               flush, reps)
            row["update_ms"], row["update_frac"] = tu, update_bytes(N, s, K) / (tu * 1e-3) / 1e9 / peak
            row["unfused_gdofs"] = 4 * K * np_of(N) / ((tv + row["surface_optimal_ms"] + tu) * 1e-3) / 1e9
            if N <= 9 and args.nodal:
                sn = build_system(mesh, N, dtype, "nodal")
                qn, rn = torch.randn_like(q), torch.empty_like(q)
                tn = time_launches(torch, lambda: sn.rhs_into(qn, rn, "dense"), flush, max(2, reps // 2))
                row["nodal_npt_rhs_ms"] = tn
                row["bb_over_nodal_rhs"] = tn / time_launches(torch, lambda: sy.rhs_into(q, rhs, args.lift), flush,
                                                              reps)
                del sn
        out["per_order"][str(N)] = row
        if dominant is None or per_n[N] > per_n[dominant]:
            dominant = N
    Nd = dominant
    t_d = per_n[Nd] / args.steps
    ach = stage_bytes(Nd, s, K) / (t_d * 1e-3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get(args.dtype, {}).get(str(Nd))
    out["roofline"] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                       "traffic": traffic, "kernel": f"tile_kernel<{args.dtype},N={Nd},OP_STAGE,{args.lift}>",
                       "peak_kind": peak_kind,
                       "bytes_per_launch": stage_bytes(Nd, s, K)}
    out["gpu_launches"] = args.steps * len(orders)

    # end-to-end through the public API with host (numpy) buffers
    e2e_ms, h2d, d2h = 0.0, 0, 0
    e2e_reps = 2 if args.quick else max(2, min(args.steps, 5))
    for N in (orders if world == 1 else []):
        d = systems[N]
        host = torch.empty((4, K, d["sy"].Np), dtype=d["sy"].torch_dtype, pin_memory=True)
        host.copy_(d["q"])
        hq = host.numpy()
        st = FieldState(hq, "bernstein")
        lsrk4_step(d["sy"], st, d["dt"], args.lift)  # warm
        torch.cuda.synchronize()
        for _ in range(e2e_reps):
            t0 = time.perf_counter()
            lsrk4_step(d["sy"], st, d["dt"], args.lift)
            torch.cuda.synchronize()
            e2e_ms += (time.perf_counter() - t0) * 1e3
        h2d += hq.nbytes
        d2h += hq.nbytes
    e2e_dofs = sum(5 * 4 * K * np_of(N) for N in orders) * e2e_reps
    out["e2e"] = {"value": world * e2e_dofs / (e2e_ms * 1e-3) / 1e9 if e2e_ms else None, "unit": UNIT,
                  "h2d_bytes_per_step": h2d,
                  "d2h_bytes_per_step": d2h,
                  "what": "lsrk4_step (5 fused stages) on a pinned numpy state per order: H2D + stages + D2H"}
    return out, K


# ---------------------------------------------------------------------- CPU arm (oracle port)
def cpu_sweep(orders, n, dtype, reps=1, lift="factorized", budget_s=None):
    """Time one LSRK stage (rhs + update) per order with the oracle on cube_mesh(n)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import bbdg_oracle as orc

    from paper_1512_06025_b200 import cube_mesh

    m = cube_mesh(n)
    arrays = orc.mesh_arrays(m)
    tot_t, tot_dofs = 0.0, 0
    rng = np.random.default_rng(2024)
    for N in orders:
        sy = orc.OracleSystem(arrays, orc.bernstein_tables(N), np.ones(m.K), np.ones(m.K), dtype)
        q = rng.standard_normal((4, m.K, sy.t.Np)).astype(dtype)
        res = np.zeros_like(q)
        for _ in range(reps):
            t0 = time.perf_counter()
            k = sy.rhs(q, lift)
            res *= dtype(orc.RK4A[1])
            res += dtype(1e-3) * k
            q += dtype(orc.RK4B[1]) * res
            tot_t += time.perf_counter() - t0
            tot_dofs += 4 * m.K * sy.t.Np
    return tot_dofs / tot_t / 1e9, m.K, tot_t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--n", type=int, default=26, help="cube_mesh(n): K = 6 n^3")
    ap.add_argument("--orders", default="1-9")
    ap.add_argument("--lift", default="optimal", choices=["optimal", "factorized", "dense"])
    ap.add_argument("--cpu-n", type=int, default=8, help="oracle sample mesh cube_mesh(cpu_n)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nodal", dest="nodal", action="store_false", help="skip the nodal NPT comparison")
    ap.add_argument("--quick", action="store_true", help="skip the per-kernel breakdown")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    orders = parse_orders(args.orders)
    dtype = np.float32 if args.dtype == "f32" else np.float64
    config = {"workload": f"BB-DG acoustic LSRK4 stage sweep N={args.orders}, cube_mesh({args.n}) K={6 * args.n ** 3}"
                          f"{' per GPU (box of ' + str(world) + ' slabs)' if world > 1 else ''}, "
                          f"{args.lift} lift", "K": 6 * args.n ** 3, "orders": orders, "lift": args.lift,
              "l2": "flushed (256 MB write) before every timed launch", "materials": "homogeneous",
              "parallelism": f"element slabs x{world}, NCCL face-trace halo" if world > 1 else "1 GPU"}

    if args.impl == "reference":
        if rank != 0:
            return
        ncores = os.cpu_count() or 1
        os.environ.setdefault("OMP_NUM_THREADS", str(ncores))
        vals = []
        for _ in range(args.warmup if args.warmup < 1 else 1):
            cpu_sweep(orders, max(2, args.cpu_n // 2), dtype)
        for _ in range(args.steps):
            v, Ks, _ = cpu_sweep(orders, args.cpu_n, dtype)
            vals.append(v)
        v = float(np.mean(vals))
        sample = f"one LSRK stage per order N={args.orders} on cube_mesh({args.cpu_n}) (K={Ks}), factorized lift"
        print(json.dumps({"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
                          "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                          "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (standard normal, seed 2024)",
                          "config": config,
                          "cpu_baseline": {"value": v, "unit": UNIT, "cores": ncores, "kind": "port",
                                           "sample": sample},
                          "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    import torch

    if world > 1:
        torch.distributed.init_process_group("nccl")
    out, K = run_ours(args, rank, world)
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    line = {"metric": METRIC, "value": out["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": out["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.dtype, "data": "synthetic (standard normal, seed 2024)",
            "config": config, "roofline": out["roofline"], "e2e": out["e2e"], "gpu_launches": out["gpu_launches"],
            "clocks": out["clocks"], "per_order": out["per_order"]}
    if not args.no_cpu_baseline:
        v, Ks, t = cpu_sweep(orders, args.cpu_n, dtype)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                                "sample": f"oracle port, one LSRK stage per order N={args.orders} on "
                                          f"cube_mesh({args.cpu_n}) (K={Ks}), factorized lift, {t:.1f} s"}
    print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
