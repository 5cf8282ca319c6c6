#!/usr/bin/env python
"""Benchmark of the DFS spectral Poisson grid solve (BASELINE.json metric:
sphere Poisson DOF/s, FP64; DOF = M*N/2 per right-hand side).

One step = one grid-level solve of one batch of synthetic input: physical
samples f -> DFS doubling -> 2D transforms -> Msin^2 -> per-mode banded solves
with the k=0 constraint -> inverse transforms -> physical u.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

N > 1: launched under torchrun, one rank per GPU; the solve is slab-
decomposed (strong scaling of one RHS) with the two transposes fused into the
stage kernels as NVLink peer stores through CUDA IPC mappings (--transport
p2p, default) or as NCCL all-to-alls (--transport nccl, the baseline); for C4
the RHS are sharded instead (weak scaling, no exchange).
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PUBLISHED_DOF_PER_S = 1e8 / 60.0  # 1e8 DOF in ~60 s, config C3


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"])
    ap.add_argument("--cpu-sample-cols", type=int, default=0)
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def count(self) -> int:
        return len(self.lines)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------- CPU reference
def cpu_reference_sample(cfg, threads: int, ncols: int):
    """The reference CPU implementation of the path on a bounded sample of the
    workload: its per-column / per-row building blocks (analyze_1d columns and
    rows, Msin^2 + band_solve per lambda mode with solve()'s thread pool,
    synthesize_1d columns and rows), timed on `ncols` columns and as many rows,
    extrapolated to the full M x N pipeline (N columns, M rows per RHS)."""
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        raise RuntimeError("oracle/_ref is not built")
    R = Reference()
    t = R.time_sample(cfg.M, cfg.N, ncols, ncols, threads)
    per_rhs = cfg.N * (t[0] + t[2] + t[3]) + cfg.M * (t[1] + t[4])
    total = per_rhs * cfg.nrhs
    dofs = cfg.dof * cfg.nrhs
    sample = (f"reference (oracle/_ref, unmodified /root/reference/proj/src + FFTW-API shim) on {ncols} of "
              f"{cfg.N} lambda columns and {ncols} of {cfg.M} theta rows of {cfg.name}, extrapolated: "
              f"theta FFT/col {t[0]*1e3:.3f} ms, lambda FFT/row {t[1]*1e3:.3f} ms, Msin2+band_solve/col "
              f"{t[2]*1e3:.3f} ms ({threads} threads), inverse theta/col {t[3]*1e3:.3f} ms, inverse lambda/row "
              f"{t[4]*1e3:.3f} ms; transforms single-threaded as shipped")
    return dofs / total, total, sample


def run_reference_arm(args, cfg, rank):
    if rank != 0:
        return
    threads = min(os.cpu_count() or 1, 16)
    ncols = args.cpu_sample_cols or max(8, min(256, int(2e6 // max(cfg.M, cfg.N))))
    for _ in range(args.warmup):
        cpu_reference_sample(cfg, threads, max(4, ncols // 4))
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        v, _, sample = cpu_reference_sample(cfg, threads, ncols)
        vals.append(v)
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": "sphere Poisson DOF/s (FP64)", "value": value, "unit": "DOF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cfg.dof * cfg.nrhs / value, "higher_is_better": True,
        "scaling": "strong" if cfg.nrhs == 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_block(cfg, args.gpus),
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    if cfg.name == "C3":
        line["vs_baseline"] = value / PUBLISHED_DOF_PER_S
    print(json.dumps(line), flush=True)


def big_inputs(cfg) -> bool:
    """f, u and the half spectrum of one step exceed the 126 MB L2 by 2x."""
    return (8 * (cfg.M // 2 + 1) * cfg.N * 2 + 16 * (cfg.M // 2 + 1) * (cfg.N // 2 + 1)) * cfg.nrhs > 256e6


def config_block(cfg, ngpus):
    par = f"slab{ngpus}" if (ngpus > 1 and cfg.nrhs == 1) else (f"rhs{ngpus}" if ngpus > 1 else "single")
    return {"workload": f"{cfg.name}: {cfg.note}", "M": cfg.M, "N": cfg.N, "nrhs": cfg.nrhs,
            "sh_degree": cfg.L, "coeff_decay": cfg.p, "dof_per_rhs": cfg.dof, "parallelism": par,
            "l2": "inputs larger than L2 (no flush)" if big_inputs(cfg) else "L2 flushed between steps (256 MB write)",
            "transport": None}


# ---------------------------------------------------------------- our arm
def main():
    args = parse()
    from paper_1510_08094_b200 import inputs
    cfg = inputs.CONFIGS[args.config]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, cfg, rank)

    import torch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    from paper_1510_08094_b200.poisson import Plan
    hbm_peak, peak_kind = measured_peaks()
    rows = cfg.M // 2 + 1
    slab = world > 1 and cfg.nrhs == 1
    nrhs_local = cfg.nrhs if world == 1 or slab else cfg.nrhs // world

    # ---- inputs (untimed): seeded SH sums synthesised on the device
    plan = Plan(cfg.M, cfg.N, nrhs_local if not slab else 1, local)
    f = torch.empty((nrhs_local, rows, cfg.N), dtype=torch.float64, device=dev)
    for r in range(nrhs_local):
        gr = (rank * nrhs_local + r) if not slab else r
        c = torch.from_numpy(inputs.sh_coeffs(args.seed + gr, cfg.L, cfg.p)).to(dev)
        plan.shgen(cfg.L, c, f[r])
    u = torch.empty_like(f)
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream(dev)
    plan.set_stream(stream.cuda_stream)

    if slab:
        from paper_1510_08094_b200.distributed import SlabSolver, slab_bounds
        solver = SlabSolver(cfg.M, cfg.N, rank, world, device=dev, transport=args.transport)
        solver._plan.set_stream(stream.cuda_stream)
        rb = solver.rb
        f_rows = f[0, rb[rank]: rb[rank + 1]].contiguous()
        u_rows = torch.empty_like(f_rows)

        def step():
            solver.solve(f_rows, u_rows)
    else:
        def step():
            plan.solve_grid(f if nrhs_local > 1 else f[0], u if nrhs_local > 1 else u[0], sync=False)

    # below 2x L2 the step's working set would stay cache-resident: write a
    # 256 MB buffer between timed steps (its time is excluded: events bracket
    # each step when flushing)
    flush = None if big_inputs(cfg) else torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=dev)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()

    # untimed steps around the timed region so that the clock sampler sees
    # the GPU under this load (same count on every rank)
    t0 = time.perf_counter()
    step()
    barrier()
    t_one = time.perf_counter() - t0
    if dist is not None:
        tt = torch.tensor([t_one], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_one = tt.item()
    n_pre = max(1, min(2000, int(math.ceil(0.4 / max(t_one, 1e-6)))))
    n_post = max(1, n_pre // 2)

    # ---- timed region (device-resident inputs)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        # keep the GPU under this load until the sampler reports (nvidia-smi
        # needs ~100 ms to start), so samples are taken under load right
        # before and (below) right after the timed steps
        for _ in range(n_pre):
            step()
        barrier()
        if flush is None:
            ev0.record(stream)
            for _ in range(args.steps):
                step()
            ev1.record(stream)
            barrier()
            ms_total = ev0.elapsed_time(ev1)
        else:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for a, b in evs:
                flush.fill_(1.0)
                a.record(stream)
                step()
                b.record(stream)
            barrier()
            ms_total = sum(a.elapsed_time(b) for a, b in evs)
        for _ in range(n_post):
            step()
        barrier()
    if dist is not None:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = t.item()
    ms_step = ms_total / args.steps
    dofs_step = cfg.dof * cfg.nrhs
    value = dofs_step / (ms_step * 1e-3)
    launches = 3 * args.steps

    # parity guard on the timed output (analytic solution), rank 0 / single GPU
    err = None
    if not slab:
        ue = torch.empty_like(f[0])
        c = torch.from_numpy(inputs.sh_coeffs(args.seed + rank * nrhs_local, cfg.L, cfg.p, solution=True)).to(dev)
        plan.shgen(cfg.L, c, ue)
        plan.solve_grid(f if nrhs_local > 1 else f[0], u if nrhs_local > 1 else u[0])
        err = ((u[0] - ue).abs().max() / ue.abs().max()).item()

    # ---- per-stage device times (roofline of the dominant kernel)
    stage = None
    if not slab:
        plan.enable_stage_timing(True)
        acc = {"lambda_fwd_ms": 0.0, "theta_ms": 0.0, "lambda_inv_ms": 0.0}
        for _ in range(args.steps):
            plan.solve_grid(f if nrhs_local > 1 else f[0], u if nrhs_local > 1 else u[0])
            st = plan.stage_times()
            for k in acc:
                acc[k] += st[k] / args.steps
        plan.enable_stage_timing(False)
        stage = acc

    # ---- end to end through the public API with host buffers
    e2e = None
    if slab:
        # rows of f in from pinned host memory, rows of u back, every step
        fh = torch.empty(f_rows.shape, dtype=torch.float64, pin_memory=True)
        uh = torch.empty(f_rows.shape, dtype=torch.float64, pin_memory=True)
        fh.copy_(f_rows.cpu())

        def step_e2e():
            f_rows.copy_(fh, non_blocking=True)
            solver.solve(f_rows, u_rows)
            uh.copy_(u_rows, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()

        for _ in range(max(1, args.warmup)):
            step_e2e()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(args.steps):
            step_e2e()
        e1.record(stream)
        barrier()
        wall = time.perf_counter() - t0
        t = torch.tensor([max(e0.elapsed_time(e1), 1e3 * wall)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = t.item() / args.steps
        nb = rows * cfg.N * 8
        e2e = {"value": dofs_step / (ms_e2e * 1e-3), "unit": "DOF/s", "h2d_bytes_per_step": nb,
               "d2h_bytes_per_step": nb, "ms_per_step": ms_e2e}
    if not slab:
        fh = torch.empty(f.shape, dtype=torch.float64, pin_memory=True)
        uh = torch.empty(f.shape, dtype=torch.float64, pin_memory=True)
        fh.copy_(f.cpu())
        fnp, unp = fh.numpy(), uh.numpy()
        args_f = fnp if nrhs_local > 1 else fnp[0]
        args_u = unp if nrhs_local > 1 else unp[0]
        # pipelined host-memory solves (SK_ASYNC): every step copies its f in
        # and its u out; consecutive steps overlap copies with compute
        for _ in range(max(1, args.warmup)):
            plan.solve_grid(args_f, args_u, sync=False)
        plan.sync()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            plan.solve_grid(args_f, args_u, sync=False)
        plan.sync()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ms_e2e = 1e3 * wall / args.steps
        nb = f.numel() * 8
        e2e = {"value": dofs_step / (ms_e2e * 1e-3), "unit": "DOF/s", "h2d_bytes_per_step": nb,
               "d2h_bytes_per_step": nb, "ms_per_step": ms_e2e}

    # ---- CPU baseline (rank 0, N = 1, bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = min(os.cpu_count() or 1, 16)
            ncols = args.cpu_sample_cols or max(8, min(256, int(2e6 // max(cfg.M, cfg.N))))
            v, _, sample = cpu_reference_sample(cfg, threads, ncols)
            cpu = {"value": v, "unit": "DOF/s", "cores": threads, "kind": "reference", "sample": sample}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "DOF/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {exc}"}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # algorithmic bytes per launch
    R, C, N = rows, cfg.N // 2 + 1, cfg.N
    nr = nrhs_local
    bytes_stage = {
        "lambda_fwd_ms": nr * (8 * R * N + 16 * R * C),
        "theta_ms": nr * (2 * 16 * R * C),
        "lambda_inv_ms": nr * (16 * R * C + 8 * R * N),
    }
    roof = None
    if stage:
        dom = max(stage, key=stage.get)
        achieved = bytes_stage[dom] / (stage[dom] * 1e-3) / 1e9
        tr = None
        prof = {}
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            with open(tp) as fh:
                prof = json.load(fh).get(cfg.name, {})
            tr = prof.get(dom.replace("_ms", ""))
        roof = {"bound": "hbm", "kernel": dom.replace("_ms", ""), "achieved": achieved, "peak": hbm_peak,
                "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": tr, "peak_kind": peak_kind,
                "stage_ms": stage, "stage_share": {k: v / sum(stage.values()) for k, v in stage.items()},
                "pipeline_bytes_per_step": sum(bytes_stage.values()),
                "pipeline_frac": sum(bytes_stage.values()) / (ms_step * 1e-3) / 1e9 / hbm_peak,
                "canonical_bytes_per_step": (64 * cfg.M * cfg.N + 16 * R * cfg.N) * cfg.nrhs,
                "canonical_frac": (64 * cfg.M * cfg.N + 16 * R * cfg.N) * cfg.nrhs / (ms_step * 1e-3) / 1e9 / (hbm_peak * world)}
        if dom == "theta_ms" and "theta_fp64_pipe" in prof:
            # the theta stage is not HBM-bound: its ncu profile (profiles/) shows
            # the FP64 pipe and shared memory near 30 % at 16 warps/SM (latency)
            roof["theta_profile"] = {"fp64_pipe_frac": prof["theta_fp64_pipe"],
                                     "warps_per_sm": prof.get("theta_warps_per_sm"),
                                     "note": "latency-bound; ncu --set full, profiles/r1_phases_and_ab.md"}
    line = {
        "metric": "sphere Poisson DOF/s (FP64)", "value": value, "unit": "DOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if slab else ("weak" if world > 1 else "strong"),
        "vs_baseline": value / PUBLISHED_DOF_PER_S if cfg.name == "C3" else None,
        "dtype": "f64", "data": "synthetic: seeded spherical-harmonic sums generated on the device",
        "config": {**config_block(cfg, world), "transport": args.transport if slab else None},
        "gpu_launches": launches, "clocks": clk.summary(),
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "parity_rel_err_vs_analytic": err,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
