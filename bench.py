"""Benchmark: GDOF-updates/s per RK stage of the BB-DG hot path vs order N = 1..9, with the
per-kernel fraction of the HBM roofline (BASELINE.json configs[2]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--dtypes f32,f64] [--orders 1-9] [--fill 0.8] [--strong] [--quick]

Workload (configs[2]): per order N = 1..9 an HBM-filling box mesh of Kuhn tetrahedra, built on
the device (mesh_device.BoxMesh -> bbdg_ctx_set_box_mesh: no host arrays), whose state q, the
stage output and the LSRK register plus the geometry records fill `--fill` of the GPU's memory;
Bernstein basis, homogeneous materials, standard-normal synthetic state (seed 2024).  One bench
"step" = one fused LSRK stage (volume + surface + update, ``bbdg_lsrk_stage``) at every order of
the sweep, fp32 (the headline `value`) and fp64 (`per_dtype`); value = sum_N 4 K_N Np(N) /
sum_N t_stage(N).  Every launch streams >= 1.4 GB, far above the 126 MB L2, so L2 is not flushed.

Per order (1 GPU): the volume, surface and update kernels timed separately on the same mesh with
their roofline fractions (MEASURED_PEAKS.json), the end-to-end lsrk4_step on a host numpy state
(pinned and pageable) on a host-fitting cube_mesh(40), and (configs[1]) BB vs nodal DG on
cube_mesh(26).  Under torchrun (N > 1) every rank owns an x-layer slab of one box (weak scaling:
an HBM-filling slab per rank; --strong: the 1-GPU mesh split N ways) with the NCCL face-trace halo
overlapped with the interior elements; times are the max over ranks.
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
WORKLOAD = ("BB-DG acoustic wave, fused LSRK4 stage sweep N={orders} on HBM-filling Kuhn box meshes "
            "(configs[2]), {lift} lift")


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


def resident_bytes(N, s, K):
    """Device memory of one order's run: q, q_out, res + the fused geometry record + connectivity."""
    return K * ((12 * np_of(N) + 36) * s + 20)


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------- clocks sampler
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def __exit__(self, *exc):
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
        for ln in self.lines:
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
# element order of the HBM-filling boxes: slabs of 4 x-layers, (y, z, x) inside a slab, so every neighbour
# except those across a slab face lies within a few MB (L2) of its element (bbdg_ctx_set_box_mesh).
# Measured per order (fp32 stage frac, xblock 1 -> 4): N=1 0.81 -> 0.85, N=9 0.43 -> 0.46, but the
# element-per-thread kernels' trace gather at N = 2, 3 prefers the reference order (0.56 -> 0.52).
XBLOCK = None   # --xblock overrides the per-order choice


def xblock_of(N):
    return XBLOCK if XBLOCK else (1 if N in (2, 3) else 4)


def fill_box(N, s, budget_bytes, ranks=1, xblock=1):
    """A Kuhn box (nx, n, n) whose resident bytes fit budget_bytes (per rank: nx a multiple of
    `ranks` layers per rank), as cubic as possible."""
    from paper_1512_06025_b200.mesh_device import BoxMesh

    per = resident_bytes(N, s, 1)
    k_max = min(int(budget_bytes // per), (1 << 29) - 1)     # int32 face ids: 4 K < 2^31
    n = max(1, int((k_max / 6) ** (1.0 / 3.0)))
    nx = max(xblock, k_max // (6 * n * n) // xblock * xblock)
    return BoxMesh(nx * ranks, n, n, lo=(-0.5 * ranks, -0.5, -0.5), hi=(0.5 * ranks, 0.5, 0.5), xblock=xblock)


def events_time(torch, fn, reps, sync_group=None):
    """Device time (ms) of `reps` back-to-back calls of fn, bracketed by barrier + synchronize."""
    torch.cuda.synchronize()
    if sync_group:
        torch.distributed.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    if sync_group:
        torch.distributed.barrier()
    return a.elapsed_time(b)


def max_over_ranks(torch, x, world):
    if world == 1:
        return x
    t = torch.tensor([x], device="cuda", dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def run_dtype(args, dname, rank, world, dev, peak, clocks):
    import torch

    from paper_1512_06025_b200 import BernsteinRefOps, Materials, WaveSystem, stable_dt
    from paper_1512_06025_b200.dist import DistWaveSystem
    from paper_1512_06025_b200.solver import RK4A, RK4B, _device_update

    dtype = np.float32 if dname == "f32" else np.float64
    s = 4 if dname == "f32" else 8
    total_mem = torch.cuda.get_device_properties(dev).total_memory
    orders = parse_orders(args.orders)
    rows, per_n, Ks = {}, {}, {}
    gen = torch.Generator(device="cuda").manual_seed(2024 + rank)
    for N in orders:
        torch.cuda.empty_cache()
        budget = args.fill * (total_mem - torch.cuda.memory_allocated(dev))
        if world == 1:
            box = fill_box(N, s, budget, 1, xblock_of(N))
            sy = WaveSystem(box, BernsteinRefOps.build(N), Materials(np.float64(1.0), np.float64(1.0)), dtype,
                            legacy_records=False)
            K = box.K
        else:
            if args.strong:   # the 1-GPU mesh, split over the ranks (needs nx >= world layers)
                from paper_1512_06025_b200.mesh_device import BoxMesh

                one = fill_box(N, s, budget, 1, xblock_of(N))
                box = BoxMesh(max(one.nx, world * xblock_of(N)), one.ny, one.nz, xblock=xblock_of(N))
            else:             # weak: an HBM-filling slab per rank
                box = fill_box(N, s, budget, world, xblock_of(N))
            sy = DistWaveSystem(box, BernsteinRefOps.build(N), Materials(np.float64(1.0), np.float64(1.0)), dtype,
                                rank, world, legacy_records=False)
            K = sy.K
        Ks[N] = K
        q = torch.randn((4, K, np_of(N)), generator=gen, device="cuda", dtype=sy.torch_dtype)
        q2, res = torch.empty_like(q), torch.randn_like(q)
        dt = stable_dt(box, N, 1.0)

        def stage():
            sy.stage_into(q, q2, res, RK4A[1], RK4B[1], dt, args.lift)

        for _ in range(args.warmup):
            stage()
        t = events_time(torch, stage, args.steps, world > 1)
        t = max_over_ranks(torch, t, world)
        per_n[N] = t
        t_stage = t / args.steps
        ach = stage_bytes(N, s, K) / (t_stage * 1e-3) / 1e9
        row = {"K": K, "box": [box.nx, box.ny, box.nz], "xblock": box.xblock,
               "hbm_fraction": resident_bytes(N, s, K) / total_mem,
               "gdofs_stage": world * 4 * K * np_of(N) / (t_stage * 1e-3) / 1e9, "stage_ms": t_stage,
               "stage_gbs": ach, "stage_frac": ach / peak}
        if world == 1 and not args.quick:
            reps = max(3, args.steps // 2)
            sy.volume_into(q, q2)
            tv = events_time(torch, lambda: sy.volume_into(q, q2), reps) / reps
            sy.surface_into(q, q2, args.lift)
            ts = events_time(torch, lambda: sy.surface_into(q, q2, args.lift), reps) / reps
            tu = events_time(torch, lambda: _device_update(q2, res, q, RK4A[1], RK4B[1], dt), reps) / reps
            row.update(volume_ms=tv, volume_frac=volume_bytes(N, s, K) / (tv * 1e-3) / 1e9 / peak,
                       surface_ms=ts, surface_frac=surface_bytes(N, s, K) / (ts * 1e-3) / 1e9 / peak,
                       update_ms=tu, update_frac=update_bytes(N, s, K) / (tu * 1e-3) / 1e9 / peak,
                       unfused_gdofs=4 * K * np_of(N) / ((tv + ts + tu) * 1e-3) / 1e9)
        rows[str(N)] = row
        del sy, q, q2, res
    total_ms = sum(per_n.values())
    dofs = sum(4 * Ks[N] * np_of(N) for N in orders)
    value = world * dofs * args.steps / (total_ms * 1e-3) / 1e9
    Nd = max(orders, key=lambda N: per_n[N])
    t_d = per_n[Nd] / args.steps
    ach = stage_bytes(Nd, s, Ks[Nd]) / (t_d * 1e-3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        tr = json.loads(tp.read_text()).get("fill", {}).get(dname, {}).get(str(Nd))
        if tr and tr.get("K") == Ks[Nd]:
            traffic = tr["dram_bytes"]
    roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": traffic,
            "kernel": f"bbdg::opt_kernel<{'float' if s == 4 else 'double'}, {Nd}, 3 (OP_STAGE), FSR>",
            "bytes_per_launch": stage_bytes(Nd, s, Ks[Nd]),
            "bytes_model": "K ((16 Np + 16 Nfp + 36) s + 20): q in/out, res r/w, neighbour traces, geometry record, "
                           "connectivity"}
    return {"value": value, "ms_per_step": total_ms / args.steps, "per_order": rows, "roofline": roof,
            "launches": args.steps * len(orders)}


def e2e_host(args, dname):
    """lsrk4_step through the public API on a host numpy state (cube_mesh(e2e_n)): H2D + 5 stages + D2H,
    per order, for a pinned and a pageable array."""
    import torch

    from paper_1512_06025_b200 import BernsteinRefOps, FieldState, Materials, WaveSystem, cube_mesh, lsrk4_step
    from paper_1512_06025_b200 import stable_dt

    dtype = np.float32 if dname == "f32" else np.float64
    m = cube_mesh(args.e2e_n)
    out = {"mesh": f"cube_mesh({args.e2e_n}) K={m.K}", "per_order": {}}
    tot = {"pinned": 0.0, "pageable": 0.0}
    dofs, nbytes = 0, 0
    for N in parse_orders(args.orders):
        sy = WaveSystem(m, BernsteinRefOps.build(N), Materials.homogeneous(m.K), dtype)
        dt = stable_dt(m, N, 1.0)
        pinned = torch.empty((4, m.K, sy.Np), dtype=sy.torch_dtype, pin_memory=True)
        pinned.normal_()
        page = pinned.numpy().copy()
        row = {}
        for kind, arr in (("pinned", pinned.numpy()), ("pageable", page)):
            st = FieldState(arr, "bernstein")
            lsrk4_step(sy, st, dt, args.lift)   # warm
            torch.cuda.synchronize()
            reps = 3
            t0 = time.perf_counter()
            for _ in range(reps):
                lsrk4_step(sy, st, dt, args.lift)   # returns with the host array updated
            row[f"{kind}_ms_step"] = (time.perf_counter() - t0) * 1e3 / reps
            tot[kind] += row[f"{kind}_ms_step"]
        out["per_order"][str(N)] = row
        dofs += 5 * 4 * m.K * sy.Np
        nbytes += pinned.numel() * pinned.element_size()
        del sy, pinned, page
        torch.cuda.empty_cache()
    out["value"] = dofs / (tot["pinned"] * 1e-3) / 1e9
    out["pageable_value"] = dofs / (tot["pageable"] * 1e-3) / 1e9
    out["bytes_per_step"] = nbytes
    return out


def compare_bases(args, dname):
    """configs[1]: BB (fused stage / rhs, and the paper's non-optimal ELL and dense lifts) vs nodal
    DG rhs -- node-per-thread dense (paper NPT) and block-partitioned tensor-core (paper EPT) -- on
    cube_mesh(26), per order."""
    import torch

    from paper_1512_06025_b200 import BernsteinRefOps, Materials, NodalRefOps, WaveSystem, cube_mesh
    from paper_1512_06025_b200.solver import RK4A, RK4B

    dtype = np.float32 if dname == "f32" else np.float64
    mesh = cube_mesh(26)
    out = {"mesh": f"cube_mesh(26) K={mesh.K}", "per_order": {}}
    for N in parse_orders(args.orders):
        sb = WaveSystem(mesh, BernsteinRefOps.build(N), Materials.homogeneous(mesh.K), dtype)
        sn = WaveSystem(mesh, NodalRefOps.build(N), Materials.homogeneous(mesh.K), dtype)
        q = torch.randn((4, mesh.K, sb.Np), device="cuda", dtype=sb.torch_dtype)
        q2, res, rhs = torch.empty_like(q), torch.randn_like(q), torch.empty_like(q)
        reps = 3

        def tm(fn):
            fn()
            return events_time(torch, fn, reps) / reps

        tb = tm(lambda: sb.rhs_into(q, rhs, args.lift))
        ts = tm(lambda: sb.stage_into(q, q2, res, RK4A[1], RK4B[1], 1e-3, args.lift))
        te = tm(lambda: sb.surface_into(q, rhs, "ell"))
        tdn = tm(lambda: sb.surface_into(q, rhs, "dense"))
        tso = tm(lambda: sb.surface_into(q, rhs, args.lift))
        tn = tm(lambda: sn.rhs_into(q, rhs, "dense"))
        tk = tm(lambda: sn.rhs_into(q, rhs, "blocked"))
        flops = 2 * mesh.K * 4 * (3 * sb.Np ** 2 + sb.Np * 4 * sb.ops.Nfp)   # useful nodal GEMM flops
        out["per_order"][str(N)] = {"bb_rhs_ms": tb, "bb_stage_ms": ts, "bb_surface_sweeps_ms": tso,
                                    "bb_surface_ell_ms": te, "bb_surface_dense_ms": tdn,
                                    "nodal_npt_rhs_ms": tn, "nodal_blocked_rhs_ms": tk,
                                    "nodal_blocked_tflops": flops / tk / 1e9,
                                    "bb_over_nodal_npt": tn / tb, "bb_over_nodal_blocked": tk / tb}
        del sb, sn, q, q2, res, rhs
        torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------- CPU arm (the reference algorithm)
_CPU = {}


def _cpu_init():
    try:   # one BLAS thread per worker process: the workers already cover the cores
        from threadpoolctl import threadpool_limits

        _CPU["limits"] = threadpool_limits(1)
    except ImportError:
        pass


def _cpu_chunk(args):
    N, lo, hi, mode = args
    sy, q, res, dt = _CPU[N]
    sy.stage(q, res, RK4A_1, RK4B_1, dt, mode, lo, hi)   # rows of [lo, hi): q_out, res_out (not shipped back)
    return hi - lo


RK4A_1 = -567301805773.0 / 1357537059087.0
RK4B_1 = 5161836677717.0 / 13612068292357.0


def cpu_sweep(orders, n, dtype, lifts=("optimal", "factorized"), procs=None, reps=1):
    """One LSRK stage per order with the oracle port (the reference algorithm: gather + einsum
    ELL rows, solver.py:139-214) on cube_mesh(n), element ranges split over `procs` forked
    workers (one BLAS thread each).  Setup (tables, coordinate-matched trace maps) is built once,
    before the workers fork, and is not timed.  Returns [{lift: (GDOF/s, seconds)}] per rep, K, procs."""
    import multiprocessing as mp

    sys.path.insert(0, str(ROOT / "oracle"))
    import bbdg_oracle as orc

    from paper_1512_06025_b200 import cube_mesh, stable_dt

    procs = procs or os.cpu_count() or 1
    m = cube_mesh(n)
    arrays = orc.mesh_arrays(m)
    rng = np.random.default_rng(2024)
    for N in orders:
        sy = orc.OracleSystem(arrays, orc.bernstein_tables(N), np.ones(m.K), np.ones(m.K), dtype)
        _CPU[N] = (sy, rng.standard_normal((4, m.K, sy.t.Np)).astype(dtype),
                   rng.standard_normal((4, m.K, sy.t.Np)).astype(dtype), stable_dt(m, N, 1.0))
    cuts = np.linspace(0, m.K, procs + 1).astype(int)
    results = []
    with mp.get_context("fork").Pool(procs, initializer=_cpu_init) as pool:
        for _ in range(reps):
            out = {}
            for lift in lifts:
                t_tot, dofs = 0.0, 0
                for N in orders:
                    t0 = time.perf_counter()
                    pool.map(_cpu_chunk, [(N, int(a), int(b), lift) for a, b in zip(cuts[:-1], cuts[1:]) if b > a])
                    t_tot += time.perf_counter() - t0
                    dofs += 4 * m.K * np_of(N)
                out[lift] = (dofs / t_tot / 1e9, t_tot)
            results.append(out)
    for N in orders:
        _CPU.pop(N, None)
    return results, m.K, procs


def cpu_sample_text(orders, n, K, lift, t, procs):
    return (f"oracle port of the reference algorithm (numpy gather + einsum, solver.py:139-214), one LSRK stage "
            f"per order N={orders} on cube_mesh({n}) (K={K}), {lift} lift, element ranges over {procs} processes, "
            f"{t:.1f} s")


# ---------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtypes", default="f32,f64", help="first = the headline value")
    ap.add_argument("--orders", default="1-9")
    ap.add_argument("--lift", default="optimal", choices=["optimal", "factorized"])
    ap.add_argument("--fill", type=float, default=0.8, help="fraction of free device memory per order")
    ap.add_argument("--strong", action="store_true", help="N>1: split the 1-GPU mesh (default: weak scaling)")
    ap.add_argument("--quick", action="store_true", help="stage sweep only (no breakdown, e2e, comparison)")
    ap.add_argument("--e2e-n", type=int, default=40)
    ap.add_argument("--cpu-n", type=int, default=16, help="oracle sample mesh cube_mesh(cpu_n)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nodal", dest="nodal", action="store_false")
    ap.add_argument("--no-e2e", dest="e2e", action="store_false", help="skip the host-state end-to-end leg")
    ap.add_argument("--xblock", type=int, default=None, help="element order of the fill boxes (x-layers per slab)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    global XBLOCK
    if args.xblock:
        XBLOCK = args.xblock
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    dnames = args.dtypes.split(",")
    orders = parse_orders(args.orders)
    head = dnames[0]
    scaling = "strong" if (args.strong and world > 1) else "weak"
    config = {"workload": WORKLOAD.format(orders=args.orders, lift=args.lift), "orders": orders, "lift": args.lift,
              "mesh": f"per order a device-built Kuhn box filling {args.fill:.2f} of free HBM, element order in "
                      f"slabs of {XBLOCK or 4} x-layers{'' if XBLOCK else ' (N = 2, 3: the reference x-slab order)'}"
                      + (f" per rank (x-layer slabs, {scaling} scaling)" if world > 1 else ""),
              "l2": "not flushed: every launch streams >= 1.4 GB (inputs larger than the 126 MB L2)",
              "materials": "homogeneous (kappa = rho = 1)",
              "parallelism": f"{world} GPUs: element slabs, NCCL face-trace halo" if world > 1 else "1 GPU"}
    base = {"metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": head,
            "data": "synthetic (standard normal, seed 2024)", "config": config}

    if args.impl == "reference":
        if rank != 0:
            return
        dtype = np.float32 if head == "f32" else np.float64
        reps, K, procs = cpu_sweep(orders, args.cpu_n, dtype, lifts=(args.lift,), reps=args.warmup + args.steps)
        timed = [r[args.lift] for r in reps[args.warmup:]]   # the first `warmup` sweeps warm the workers
        v = float(np.mean([x[0] for x in timed]))
        res = {args.lift: (v, float(np.mean([x[1] for x in timed])))}
        sample = cpu_sample_text(args.orders, args.cpu_n, K, args.lift, res[args.lift][1], procs)
        print(json.dumps(dict(base, impl="reference", value=v, ms_per_step=None,
                              cpu_baseline={"value": v, "unit": UNIT, "cores": procs, "kind": "port",
                                            "sample": sample},
                              e2e={"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})))
        return

    import torch

    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.distributed.init_process_group("nccl")
    dev = int(os.environ.get("LOCAL_RANK", rank)) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    peak, peak_kind = load_peaks()
    per_dtype = {}
    with Clocks(dev) as clk:
        for d in dnames:
            per_dtype[d] = run_dtype(args, d, rank, world, dev, peak, clk)
    line = dict(base, value=per_dtype[head]["value"], ms_per_step=per_dtype[head]["ms_per_step"],
                roofline=dict(per_dtype[head]["roofline"], peak_kind=peak_kind),
                gpu_launches=sum(r["launches"] for r in per_dtype.values()), clocks=clk.summary(),
                per_order=per_dtype[head]["per_order"],
                per_dtype={d: {"value": r["value"], "ms_per_step": r["ms_per_step"], "roofline": r["roofline"],
                               "per_order": r["per_order"]} for d, r in per_dtype.items()})
    if world > 1:
        line["nccl"] = {"backend": "nccl", "nranks": world, "version": ".".join(map(str, torch.cuda.nccl.version()))}
    if world == 1 and not args.quick and args.e2e:
        e2e = e2e_host(args, head)
        line["e2e"] = {"value": e2e["value"], "unit": UNIT, "h2d_bytes_per_step": e2e["bytes_per_step"],
                       "d2h_bytes_per_step": e2e["bytes_per_step"], "pageable_value": e2e["pageable_value"],
                       "what": f"lsrk4_step (5 fused stages) on a host numpy state per order, {e2e['mesh']}: H2D + "
                               "stages + D2H in the timed region (pinned: chunk-pipelined bbdg_step_host; "
                               "pageable_value: an ordinary numpy array through the pinned staging rings of bbdg_step_pageable)", "per_order": e2e["per_order"]}
    else:
        line["e2e"] = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                       "what": "not measured in --quick / --no-e2e / multi-GPU mode"}
    if world == 1 and not args.quick and args.nodal:
        line["comparison"] = compare_bases(args, head)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        dtype = np.float32 if head == "f32" else np.float64
        reps, K, procs = cpu_sweep(orders, args.cpu_n, dtype, lifts=(args.lift, "factorized"), reps=2)
        res = reps[-1]
        line["cpu_baseline"] = {"value": res[args.lift][0], "unit": UNIT, "cores": procs, "kind": "port",
                                "sample": cpu_sample_text(args.orders, args.cpu_n, K, args.lift, res[args.lift][1],
                                                          procs),
                                "factorized_value": res["factorized"][0]}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
