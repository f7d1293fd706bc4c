"""Benchmark: GDOF-updates/s per RK stage of the BB-DG hot path, N = 1..9.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--dtype f32|f64] [--n 26] [--orders 1-9] [--lift optimal]

Workload (BASELINE.json configs[2], the kernel sweep): cube_mesh(40) =
384,000 tets per GPU, Bernstein basis, orders N = 1..9, homogeneous
materials, standard-normal synthetic state (seed 2024).  One bench "step" =
one fused LSRK4 stage (volume + surface + update, ``bbdg_lsrk_stage``) at
every order of the sweep; the headline value is the sweep's whole-job DOF
throughput sum_N 4 K Np(N) / sum_N t_stage(N).  Orders run one after another
(bounded memory); L2 (126 MB) is flushed with a 256 MB write before every
timed launch, outside the event window.

Per-order extras: volume / surface (3 lift modes) / update kernels timed
separately with their roofline fractions against MEASURED_PEAKS.json, the
end-to-end lsrk4_step on a host state, and (configs[1]) the BB vs nodal
comparison on cube_mesh(26).
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
    """Mean device time (ms) of fn over reps launches, L2 flushed before each (outside the events).
    One untimed call first: the first launch of a kernel pays CUDA's lazy module load."""
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


def run_ours(args, rank, world):
    import torch

    from paper_1512_06025_b200 import cube_mesh, lsrk4_step, FieldState, stable_dt
    from paper_1512_06025_b200.solver import RK4A, RK4B

    dev = int(os.environ.get("LOCAL_RANK", rank)) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dtype = np.float32 if args.dtype == "f32" else np.float64
    s = 4 if args.dtype == "f32" else 8
    mesh_n = {}   # per-order cube size in --fill mode

    def fill_n(N):
        """cube_mesh(n) whose q, q_out, res + geometry records use args.fill of the device memory."""
        total = torch.cuda.get_device_properties(dev).total_memory
        per_elem = 12 * np_of(N) * s + 2 * 36 * s + 20
        # capped at n = 140 (16.5 M tets): the host-side setup arrays of WaveSystem stay < ~20 GB
        return min(140, int((args.fill * total / per_elem / 6) ** (1.0 / 3.0)))

    if world > 1:
        # weak scaling: a box of world x n^3 cells, one n^3-cell x-slab per rank
        from paper_1512_06025_b200.mesh import box_mesh

        mesh = box_mesh(world * args.n, args.n, args.n, lo=(-0.5 * world, -0.5, -0.5), hi=(0.5 * world, 0.5, 0.5))
    elif args.fill > 0:
        mesh = None
    else:
        mesh = cube_mesh(args.n)
    K = mesh.K // world if mesh is not None else 0
    orders = parse_orders(args.orders)
    Ks = {}
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    peak, peak_kind = load_peaks()

    def make_system(N):
        if world > 1:
            from paper_1512_06025_b200 import BernsteinRefOps, Materials
            from paper_1512_06025_b200.dist import DistWaveSystem

            sy = DistWaveSystem(mesh, BernsteinRefOps.build(N), Materials.homogeneous(mesh.K), dtype, rank, world,
                                align=6 * args.n * args.n)
            sy.Np, sy.torch_dtype = sy.local.Np, sy.local.torch_dtype
            return sy
        return build_system(mesh, N, dtype)

    # one order at a time (bounded memory): W warm-up stages, then K timed stages, each launch
    # bracketed by CUDA events with the L2 flushed before it (outside the events)
    per_n, rows = {}, {}
    gen = torch.Generator(device="cuda").manual_seed(2024 + rank)
    with Clocks(dev) as clk:
        for N in orders:
            if args.fill > 0:
                from paper_1512_06025_b200.mesh_device import cube_mesh_device

                mesh_n[N] = fill_n(N)
                mesh = cube_mesh_device(mesh_n[N])
                torch.cuda.empty_cache()   # return the builder's scratch before the context allocates
                K = mesh.K
            Ks[N] = K
            sy = make_system(N)
            q = torch.randn((4, K, sy.Np), generator=gen, device="cuda", dtype=sy.torch_dtype)
            q2, res = torch.empty_like(q), torch.randn_like(q)
            dt = stable_dt(mesh, N, 1.0)

            def stage():
                sy.stage_into(q, q2, res, RK4A[1], RK4B[1], dt, args.lift)

            for _ in range(args.warmup):
                stage()
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            tot = 0.0
            for _ in range(args.steps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                stage()
                b.record()
                b.synchronize()
                tot += a.elapsed_time(b)
            torch.cuda.synchronize()
            per_n[N] = tot
            t_stage = tot / args.steps
            ach = stage_bytes(N, s, K) / (t_stage * 1e-3) / 1e9   # K of this order's mesh
            row = {"gdofs_stage": 4 * K * np_of(N) / (t_stage * 1e-3) / 1e9, "stage_ms": t_stage,
                   "stage_gbs": ach, "stage_frac": ach / peak}
            if not args.quick and world == 1 and args.fill <= 0:
                rhs = torch.empty_like(q)
                reps = max(3, args.steps)
                tv = time_launches(torch, lambda: sy.volume_into(q, rhs), flush, reps)
                row["volume_ms"], row["volume_frac"] = tv, volume_bytes(N, s, K) / (tv * 1e-3) / 1e9 / peak
                for mode in ("factorized", "optimal", "dense"):
                    ts = time_launches(torch, lambda: sy.surface_into(q, rhs, mode), flush, reps)
                    row[f"surface_{mode}_ms"] = ts
                    row[f"surface_{mode}_frac"] = surface_bytes(N, s, K) / (ts * 1e-3) / 1e9 / peak
                from paper_1512_06025_b200.solver import _device_update
                tu = time_launches(torch, lambda: _device_update(q2, res, rhs, RK4A[1], RK4B[1], dt), flush, reps)
                row["update_ms"], row["update_frac"] = tu, update_bytes(N, s, K) / (tu * 1e-3) / 1e9 / peak
                row["unfused_gdofs"] = 4 * K * np_of(N) / ((tv + row["surface_optimal_ms"] + tu) * 1e-3) / 1e9
                del rhs
            # end to end through the public API with a pinned host state: H2D + 5 stages + D2H
            # (N > 1: each rank's slab through DistWaveSystem.step_into, max over ranks)
            if args.fill > 0:
                rows[str(N)] = row
                row["K"] = K
                row["hbm_fraction"] = (12 * np_of(N) * s + 2 * 36 * s + 20) * K / torch.cuda.get_device_properties(
                    dev).total_memory
                del sy, q, q2, res
                mesh = None
                torch.cuda.empty_cache()
                continue
            host = torch.empty((4, K, sy.Np), dtype=sy.torch_dtype, pin_memory=True)
            host.copy_(q)
            reps = 2 if args.quick else max(2, min(args.steps, 5))
            if world == 1:
                st = FieldState(host.numpy(), "bernstein")
                lsrk4_step(sy, st, dt, args.lift)   # warm
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for _ in range(reps):
                    lsrk4_step(sy, st, dt, args.lift)
                torch.cuda.synchronize()
                e2e = (time.perf_counter() - t0) * 1e3 / reps
                del st
            else:
                qd, qt, rd = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)

                def e2e_step():
                    qd.copy_(host, non_blocking=True)
                    sy.step_into(qd, qt, rd, dt, args.lift)
                    host.copy_(qd, non_blocking=True)
                    torch.cuda.synchronize()

                e2e_step()
                torch.distributed.barrier()
                t0 = time.perf_counter()
                for _ in range(reps):
                    e2e_step()
                e2e = (time.perf_counter() - t0) * 1e3 / reps
                tt = torch.tensor([e2e], device="cuda", dtype=torch.float64)
                torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
                e2e = float(tt.item())
                del qd, qt, rd
            row["e2e_ms_step"] = e2e
            row["e2e_bytes"] = 2 * host.numel() * host.element_size()
            del host
            rows[str(N)] = row
            del sy, q, q2, res
            torch.cuda.empty_cache()
    total_ms = sum(per_n.values())
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
        torch.distributed.barrier()
    dofs_per_step = sum(4 * Ks[N] * np_of(N) for N in orders)
    value = world * dofs_per_step * args.steps / (total_ms * 1e-3) / 1e9
    out = dict(per_order=rows, value=value, ms_per_step=total_ms / args.steps, clocks=clk.summary())
    Nd = max(orders, key=lambda N: per_n[N])   # dominant kernel: the order with the largest stage time
    t_d = per_n[Nd] / args.steps
    ach = stage_bytes(Nd, s, Ks[Nd]) / (t_d * 1e-3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get(args.dtype, {}).get(f"n{args.n}", {}).get(str(Nd))
    out["roofline"] = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                       "traffic": traffic, "kernel": f"opt_kernel<{args.dtype},N={Nd},OP_STAGE> ({args.lift} lift)",
                       "peak_kind": peak_kind, "bytes_per_launch": stage_bytes(Nd, s, Ks[Nd])}
    out["gpu_launches"] = args.steps * len(orders)
    if args.fill > 0:
        out["e2e"] = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                      "what": "not measured in --fill mode (a host copy of an HBM-filling state does not fit)"}
        out["fill_meshes"] = {str(N): {"n": mesh_n[N], "K": Ks[N]} for N in orders}
        return out, Ks[orders[-1]]
    e2e_ms = sum(r["e2e_ms_step"] for r in rows.values())
    e2e_dofs = sum(5 * 4 * K * np_of(N) for N in orders)
    out["e2e"] = {"value": world * e2e_dofs / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
                  "h2d_bytes_per_step": world * sum(r["e2e_bytes"] // 2 for r in rows.values()),
                  "d2h_bytes_per_step": world * sum(r["e2e_bytes"] // 2 for r in rows.values()),
                  "what": ("lsrk4_step (5 fused stages) on a pinned numpy state per order: H2D + stages + D2H "
                           "(chunk-pipelined through bbdg_step_host for states >= 32 MB: copies overlap stages)"
                           if world == 1 else "per rank: pinned host slab H2D + DistWaveSystem.step_into (5 "
                           "exchanged stages) + D2H, max over ranks")}
    if world == 1 and args.nodal and not args.quick:
        out["comparison"] = compare_bases(args, dtype, flush)
    return out, K


def compare_bases(args, dtype, flush):
    """configs[1]: BB (fused stage / rhs) vs nodal DG rhs -- node-per-thread dense (paper NPT) and
    block-partitioned tensor-core (paper EPT) -- on cube_mesh(26), per order."""
    import torch

    from paper_1512_06025_b200 import cube_mesh
    from paper_1512_06025_b200.solver import RK4A, RK4B

    mesh = cube_mesh(26)
    out = {"mesh": f"cube_mesh(26) K={mesh.K}", "per_order": {}}
    for N in parse_orders(args.orders):
        sb, sn = build_system(mesh, N, dtype), build_system(mesh, N, dtype, "nodal")
        q = torch.randn((4, mesh.K, sb.Np), device="cuda", dtype=sb.torch_dtype)
        q2, res, rhs = torch.empty_like(q), torch.randn_like(q), torch.empty_like(q)
        reps = 3
        tb = time_launches(torch, lambda: sb.rhs_into(q, rhs, args.lift), flush, reps)
        ts = time_launches(torch, lambda: sb.stage_into(q, q2, res, RK4A[1], RK4B[1], 1e-3, args.lift), flush, reps)
        tn = time_launches(torch, lambda: sn.rhs_into(q, rhs, "dense"), flush, reps)
        tk = time_launches(torch, lambda: sn.rhs_into(q, rhs, "blocked"), flush, reps)
        flops = 2 * mesh.K * 4 * (3 * sb.Np ** 2 + sb.Np * 4 * sb.ops.Nfp)   # useful nodal GEMM flops
        out["per_order"][str(N)] = {"bb_rhs_ms": tb, "bb_stage_ms": ts, "nodal_npt_rhs_ms": tn,
                                    "nodal_blocked_rhs_ms": tk, "nodal_blocked_tflops": flops / tk / 1e9,
                                    "bb_over_nodal_npt": tn / tb, "bb_over_nodal_blocked": tk / tb}
        del sb, sn, q, q2, res, rhs
        torch.cuda.empty_cache()
    return out


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
    ap.add_argument("--n", type=int, default=40, help="cube_mesh(n): K = 6 n^3 per GPU")
    ap.add_argument("--orders", default="1-9")
    ap.add_argument("--lift", default="optimal", choices=["optimal", "factorized", "dense"])
    ap.add_argument("--cpu-n", type=int, default=16, help="oracle sample mesh cube_mesh(cpu_n)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nodal", dest="nodal", action="store_false", help="skip the nodal NPT comparison")
    ap.add_argument("--quick", action="store_true", help="skip the per-kernel breakdown")
    ap.add_argument("--fill", type=float, default=0.0,
                    help="configs[2] HBM-filling sweep: per order a cube_mesh (built on the GPU) whose q, q_out, res "
                         "use this fraction of device memory (1 GPU; no breakdown / e2e)")
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
    if args.fill > 0:
        line["config"]["workload"] = (f"BB-DG acoustic LSRK4 stage sweep N={args.orders}, HBM-filling cube meshes "
                                      f"({args.fill:.2f} of device memory for q, q_out, res), built on the GPU")
        line["config"]["K"] = {N: v["K"] for N, v in out["fill_meshes"].items()}
        line["config"]["fill"] = out["fill_meshes"]
    if "comparison" in out:
        line["comparison"] = out["comparison"]
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
