#!/usr/bin/env python
"""Benchmark of the DFS spectral Poisson grid solve (BASELINE.json metric:
sphere Poisson DOF/s, FP64; DOF = M*N/2 per right-hand side).

One step = one grid-level solve of one batch of synthetic input: physical
samples f -> DFS doubling -> 2D transforms -> Msin^2 -> per-mode banded solves
with the k=0 constraint -> inverse transforms -> physical u.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

N > 1: one rank per GPU — launched by the driver under torchrun, or, when
WORLD_SIZE is unset, re-launched by this script under torch.distributed.run
with N ranks.  The solve is slab-decomposed (strong scaling of one RHS) with
the two transposes fused into the stage kernels as NVLink peer stores through
CUDA IPC mappings (--transport p2p, default) or as NCCL all-to-alls
(--transport nccl, the baseline); for C4 the RHS are sharded instead (weak
scaling, no exchange).  With fewer GPUs than ranks (a one-GPU test box),
ranks share devices round-robin: the host plumbing then runs on gloo and the
transport is p2p (same-device IPC mappings; ranks meet only at host
barriers, no kernel waits on another rank) — a functional run, not a scaling
measurement (config.shared_gpus says so).
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
BLOCKS = 16  # a reference step is 1/BLOCKS of the stock composition


def host_facts():
    """nproc and the lscpu model of the host the CPU numbers were taken on."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.lower().startswith("model name"):
                model = ln.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def reference_block(R, cfg, b, threads):
    """Block b (of BLOCKS) of the reference's own grid composition on full-size
    matrices (oracle/_ref ref_time_stock_sample): sample_dfs of M/BLOCKS rows,
    analyze_2d's column stage on N/BLOCKS consecutive lambda-mode columns and
    its row stage on the M/BLOCKS rows, Msin^2 + solve()'s column solves on
    its thread pool, sample_grid's column and row stages -- the reference's
    loops and access patterns; BLOCKS consecutive blocks cover the whole
    composition once per right-hand side.  Returns (seconds, DOF processed)."""
    nc, nr = cfg.N // BLOCKS, cfg.M // BLOCKS
    t = R.time_stock_sample(cfg.M, cfg.N, (b % BLOCKS) * nc, nc, (b % BLOCKS) * nr, nr, threads)
    return float(t[5]), cfg.dof / BLOCKS


def fft_shim_factor(cfg):
    """The FFT arithmetic of the reference build comes from the FFTW-API shim
    (oracle/skfft, FFTW3 is not installed): its time per transform at the
    config's two lengths against numpy's pocketfft on the same host."""
    import numpy as np
    from oracle.oracle import Reference
    R = Reference()
    out = {}
    for n in sorted({cfg.M, cfg.N}):
        x = np.random.default_rng(0).standard_normal(n) + 1j * np.random.default_rng(1).standard_normal(n)
        reps = max(3, int(2e6 // n))
        R.analyze_1d(x)
        t0 = time.perf_counter()
        for _ in range(reps):
            R.analyze_1d(x)
        t_shim = (time.perf_counter() - t0) / reps
        np.fft.fft(x)
        t0 = time.perf_counter()
        for _ in range(reps):
            np.fft.fft(x) * (1.0 / n)
        t_np = (time.perf_counter() - t0) / reps
        out[str(n)] = {"shim_ms": 1e3 * t_shim, "pocketfft_ms": 1e3 * t_np, "shim_over_pocketfft": t_shim / t_np}
    return out


def cpu_reference_blocks(cfg, threads: int, nblocks: int, first: int = 0):
    """Time `nblocks` consecutive stock-composition blocks of the workload;
    returns (DOF/s over them, seconds, DOF)."""
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        raise RuntimeError("oracle/_ref is not built")
    R = Reference()
    secs = dofs = 0.0
    for b in range(first, first + nblocks):
        s, d = reference_block(R, cfg, b, threads)
        secs += s
        dofs += d
    return dofs * cfg.nrhs / (secs * cfg.nrhs), secs, dofs


def solve_thread_scaling(cfg):
    """BASELINE.md CPU plan step 2: the reference's solve() (coefficient space,
    bench_poisson's timing) with min(nproc, 16) threads and with 1 thread, on
    one stock block of columns."""
    from oracle.oracle import Reference
    R = Reference()
    nc, nr = cfg.N // BLOCKS, cfg.M // BLOCKS
    res = {}
    for th in sorted({1, min(os.cpu_count() or 1, 16)}):
        R.time_stock_sample(cfg.M, cfg.N, 0, nc, 0, 2, th)
        t = R.time_stock_sample(cfg.M, cfg.N, 0, nc, 0, 2, th)
        res[f"solve_{th}thr_dof_per_s"] = (cfg.M * cfg.N / 2) / (t[2] * cfg.N)
    return res


VALIDATION = os.path.join(ROOT, "profiles", "r2_reference_validation.json")


def validation_note(cfg):
    """Block sum vs the full composition measured in one piece (profiles/)."""
    if not os.path.exists(VALIDATION):
        return None
    with open(VALIDATION) as fh:
        v = json.load(fh).get(cfg.name)
    return v


def run_reference_arm(args, cfg, rank):
    if rank != 0:
        return
    threads = min(os.cpu_count() or 1, 16)
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (the reference build) is missing"}))
        return
    need = 4 * 16 * cfg.M * cfg.N  # the stock sampler's four full-size complex matrices
    try:
        ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        ram = None
    if ram is not None and need > 0.6 * ram:
        print(json.dumps({"impl": "reference", "unavailable": f"the reference composition at {cfg.name} needs "
                          f"~{need / 1e9:.0f} GB of full-size matrices; host has {ram / 1e9:.0f} GB"}))
        return
    R = Reference()
    for w in range(args.warmup):
        reference_block(R, cfg, w, threads)
    secs = dofs = 0.0
    per = []
    t0 = time.perf_counter()
    for st in range(args.steps):
        s, d = reference_block(R, cfg, args.warmup + st, threads)
        per.append(s)
        secs += s
        dofs += d
    wall = time.perf_counter() - t0
    value = dofs / secs
    sample = (f"reference (oracle/_ref: unmodified /root/reference/proj/src + FFTW-API shim over skfft), its stock "
              f"grid composition sample_dfs -> analyze_2d -> Msin^2 -> solve ({threads} threads) -> sample_grid, "
              f"one step = 1/{BLOCKS} of it (N/{BLOCKS} consecutive lambda-mode columns and M/{BLOCKS} theta rows "
              f"through every stage, on full-size {cfg.M} x {cfg.N} matrices); {BLOCKS} steps = one whole solve; "
              "transforms single-threaded as shipped")
    cb = {"value": value, "unit": "DOF/s", "cores": threads, "kind": "reference", "sample": sample, **host_facts()}
    v = validation_note(cfg)
    if v:
        cb["validation"] = v
    line = {
        "impl": "reference", "metric": "sphere Poisson DOF/s (FP64)", "value": value, "unit": "DOF/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
        "scaling": "strong" if cfg.nrhs == 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_block(cfg, args.gpus), "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall, "step_fraction_of_solve": 1.0 / (BLOCKS * cfg.nrhs),
        "full_solve_s": BLOCKS * cfg.nrhs * secs / args.steps,
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
def relaunch(args) -> int:
    """--gpus N > 1 without a launcher: run this script under
    torch.distributed.run with N ranks on this node (127.0.0.1)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


def main():
    args = parse()
    from paper_1510_08094_b200 import inputs
    cfg = inputs.CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; reporting the {world} ranks that ran",
              file=sys.stderr)
    if args.impl == "reference":
        return run_reference_arm(args, cfg, rank)

    import torch
    ndev = torch.cuda.device_count()
    shared = world > ndev  # more ranks than GPUs: ranks share devices round-robin
    local_dev = local % ndev
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    dist = None
    red_dev = dev  # device of the small tensors the host plumbing reduces
    if world > 1:
        import torch.distributed as dist
        if shared:
            # NCCL needs one rank per device; the data path does not use the
            # collectives (p2p transport), only barriers and small reductions
            dist.init_process_group("gloo")
            red_dev = torch.device("cpu")
            if args.transport != "p2p" and rank == 0:
                print("bench.py: ranks share GPUs: --transport nccl needs one GPU per rank; using p2p",
                      file=sys.stderr)
            args.transport = "p2p"
        else:
            dist.init_process_group("nccl", device_id=dev)
            if args.transport == "p2p" and cfg.nrhs == 1:
                # the fused transposes store into the peers' buffers: every GPU
                # pair of the job must have peer access (NVLink / NVSwitch);
                # the answer is reduced so that all ranks take the same path
                ok = all(torch.cuda.can_device_access_peer(local_dev, d) for d in range(min(world, ndev)) if d != local_dev)
                t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MIN)
                if t.item() == 0:
                    if rank == 0:
                        print("bench.py: no peer access between all GPUs; using --transport nccl", file=sys.stderr)
                    args.transport = "nccl"

    from paper_1510_08094_b200.poisson import Plan
    hbm_peak, peak_kind = measured_peaks()
    rows = cfg.M // 2 + 1
    slab = world > 1 and cfg.nrhs == 1
    nrhs_local = cfg.nrhs if world == 1 or slab else cfg.nrhs // world

    # ---- inputs (untimed): seeded SH sums synthesised on the device
    stream = torch.cuda.current_stream(dev)
    if slab:
        # one plan per rank (the solver's); the full input is synthesised once
        # and only this rank's rows are kept
        from paper_1510_08094_b200.distributed import SlabSolver
        solver = SlabSolver(cfg.M, cfg.N, rank, world, device=dev, transport=args.transport)
        plan = solver._plan
        rb = solver.rb
        full = torch.empty((rows, cfg.N), dtype=torch.float64, device=dev)
        plan.shgen(cfg.L, torch.from_numpy(inputs.sh_coeffs(args.seed, cfg.L, cfg.p)).to(dev), full)
        f_rows = full[rb[rank]: rb[rank + 1]].clone()  # (a row slice is a view of full)
        plan.shgen(cfg.L, torch.from_numpy(inputs.sh_coeffs(args.seed, cfg.L, cfg.p, solution=True)).to(dev), full)
        ue_rows = full[rb[rank]: rb[rank + 1]].clone()
        del full
        u_rows = torch.empty_like(f_rows)
        f = u = None
        torch.cuda.synchronize()
        plan.set_stream(stream.cuda_stream)

        def step():
            solver.solve(f_rows, u_rows)
    else:
        plan = Plan(cfg.M, cfg.N, nrhs_local, local_dev)
        f = torch.empty((nrhs_local, rows, cfg.N), dtype=torch.float64, device=dev)
        for r in range(nrhs_local):
            c = torch.from_numpy(inputs.sh_coeffs(args.seed + rank * nrhs_local + r, cfg.L, cfg.p)).to(dev)
            plan.shgen(cfg.L, c, f[r])
        u = torch.empty_like(f)
        torch.cuda.synchronize()
        plan.set_stream(stream.cuda_stream)

        def step():
            plan.solve_grid(f if nrhs_local > 1 else f[0], u if nrhs_local > 1 else u[0], sync=False)

    # below 2x L2 the step's working set would stay cache-resident: write a
    # 256 MB buffer between timed steps (its time is excluded: events bracket
    # each step when flushing)
    flush = None if big_inputs(cfg) else torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=dev)
    if slab and dist is not None:
        dist.barrier()

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
        tt = torch.tensor([t_one], dtype=torch.float64, device=red_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_one = tt.item()
    n_pre = max(1, min(2000, int(math.ceil(0.4 / max(t_one, 1e-6)))))
    n_post = max(1, n_pre // 2)

    # ---- timed region (device-resident inputs)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_dev) as clk:
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
        t = torch.tensor([ms_total], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = t.item()
    ms_step = ms_total / args.steps
    dofs_step = cfg.dof * cfg.nrhs
    value = dofs_step / (ms_step * 1e-3)
    launches = 3 * args.steps

    # parity guard on the timed output (analytic solution); slab: every rank's
    # rows against the analytic rows, max over ranks
    err = None
    if slab:
        solver.solve(f_rows, u_rows)
        torch.cuda.synchronize()
        e = torch.tensor([((u_rows - ue_rows).abs().max() / ue_rows.abs().max()).item() if u_rows.numel() else 0.0],
                         dtype=torch.float64, device=red_dev)
        dist.all_reduce(e, op=dist.ReduceOp.MAX)
        err = e.item()
    else:
        ue = torch.empty_like(f[0])
        c = torch.from_numpy(inputs.sh_coeffs(args.seed + rank * nrhs_local, cfg.L, cfg.p, solution=True)).to(dev)
        plan.shgen(cfg.L, c, ue)
        plan.solve_grid(f if nrhs_local > 1 else f[0], u if nrhs_local > 1 else u[0])
        err = ((u[0] - ue).abs().max() / ue.abs().max()).item()

    # ---- per-stage device times (roofline of the dominant kernel); slab
    # mode: per rank, each stage including its fused peer-store transpose,
    # the max over ranks
    stage = None
    acc = {"lambda_fwd_ms": 0.0, "theta_ms": 0.0, "lambda_inv_ms": 0.0}
    sp = solver._plan if slab else plan
    sp.enable_stage_timing(True)
    for _ in range(args.steps):
        if slab:
            solver.solve(f_rows, u_rows)
        else:
            plan.solve_grid(f if nrhs_local > 1 else f[0], u if nrhs_local > 1 else u[0])
        st = sp.stage_times()
        for k in acc:
            acc[k] += st[k] / args.steps
    sp.enable_stage_timing(False)
    if dist is not None:
        t = torch.tensor([acc[k] for k in sorted(acc)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        acc = {k: v for k, v in zip(sorted(acc), t.tolist())}
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
        t = torch.tensor([max(e0.elapsed_time(e1), 1e3 * wall)], dtype=torch.float64, device=red_dev)
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
        # the interconnect's share: the same bytes in and out at once on two
        # streams, no solve (what a fully overlapped pipeline could reach)
        try:
            s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
            dsrc = torch.empty_like(f)
            torch.cuda.synchronize()
            reps = 3
            t0 = time.perf_counter()
            for _ in range(reps):
                with torch.cuda.stream(s_in):
                    f.copy_(fh, non_blocking=True)
                with torch.cuda.stream(s_out):
                    uh.copy_(dsrc, non_blocking=True)
            torch.cuda.synchronize()
            e2e["copies_only_ms"] = 1e3 * (time.perf_counter() - t0) / reps
            del dsrc
        except RuntimeError:
            pass

    # ---- CPU baseline (rank 0, N = 1, bounded sample: 2 of the 16 stock blocks)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = min(os.cpu_count() or 1, 16)
            v, secs, _ = cpu_reference_blocks(cfg, threads, 2)
            cpu = {"value": v, "unit": "DOF/s", "cores": threads, "kind": "reference",
                   "sample": (f"reference (oracle/_ref) stock grid composition, 2 of its {BLOCKS} blocks "
                              f"(N/{BLOCKS} columns + M/{BLOCKS} rows through every stage on full-size matrices, "
                              f"{secs:.1f} s of CPU work; solve() on {threads} threads, transforms single-threaded)"),
                   **host_facts(), **solve_thread_scaling(cfg), "fft_shim": fft_shim_factor(cfg)}
            vn = validation_note(cfg)
            if vn:
                cpu["validation"] = vn
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "DOF/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {exc}"}

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # algorithmic bytes per launch; slab mode: this rank's share
    R, C, N = rows, cfg.N // 2 + 1, cfg.N
    nr = nrhs_local
    if slab:
        rows_r, cols_r = solver.rows_r, solver.cols_r
        bytes_stage = {
            "lambda_fwd_ms": 8 * rows_r * N + 16 * rows_r * C,
            "theta_ms": 2 * 16 * R * cols_r,
            "lambda_inv_ms": 16 * rows_r * C + 8 * rows_r * N,
        }
    else:
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
        if os.path.exists(tp) and world == 1:
            with open(tp) as fh:
                prof = json.load(fh).get(cfg.name, {})
            tr = prof.get(dom.replace("_ms", ""))
        reduced = (16 * R * N + 64 * R * C) * cfg.nrhs  # whole job, symmetry-reduced variant
        roof = {"bound": "hbm", "kernel": dom.replace("_ms", ""), "achieved": achieved, "peak": hbm_peak,
                "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": tr, "peak_kind": peak_kind,
                "stage_ms": stage, "stage_share": {k: v / sum(stage.values()) for k, v in stage.items()},
                "pipeline_bytes_per_step": reduced,
                "pipeline_frac": reduced / (ms_step * 1e-3) / 1e9 / (hbm_peak * world),
                "canonical_bytes_per_step": (64 * cfg.M * cfg.N + 16 * R * cfg.N) * cfg.nrhs,
                "canonical_frac": (64 * cfg.M * cfg.N + 16 * R * cfg.N) * cfg.nrhs / (ms_step * 1e-3) / 1e9 / (hbm_peak * world)}
        if slab:
            # SURVEY §8d combined roofline for the declared symmetry-reduced
            # variant: t_roof(P) = B/(P BW_HBM) + 2 * 16 R C (P-1)/P^2 / BW_NVL
            # (serialised phases; max() of the two is the overlap bound), and
            # the achieved NVLink GB/s of each fused transpose (the bytes this
            # rank stores into its peers' buffers over the stage's time)
            P = world
            bw_nvl = 770.0  # GB/s per direction, measured peer copy (B200_PROFILING.md)
            nvl_bytes = 2 * 16 * R * C * (P - 1) / P ** 2
            t_h = reduced / (P * hbm_peak * 1e9)
            t_n = nvl_bytes / (bw_nvl * 1e9)
            fwd_peer = 16 * rows_r * (C - cols_r)
            ret_peer = 16 * cols_r * (R - rows_r)
            roof["slab"] = {
                "P": P, "t_roof_ms": 1e3 * (t_h + t_n), "t_roof_overlap_ms": 1e3 * max(t_h, t_n),
                "frac": 1e3 * (t_h + t_n) / ms_step, "nvlink_bytes_per_gpu": nvl_bytes,
                "nvlink_peak_gbs": bw_nvl, "nvlink_peak_kind": "measured peer copy (B200_PROFILING.md)",
                "transpose_fwd_gbs": fwd_peer / (stage["lambda_fwd_ms"] * 1e-3) / 1e9,
                "transpose_ret_gbs": ret_peer / (stage["theta_ms"] * 1e-3) / 1e9,
                "shared_gpus": shared,
            }
        if dom == "theta_ms" and "theta_fp64_pipe" in prof:
            # the theta stage is not HBM-bound: its ncu profile (profiles/) shows
            # the FP64 pipe and shared memory near 30 % at 16 warps/SM (latency)
            roof["theta_profile"] = {"fp64_pipe_frac": prof["theta_fp64_pipe"],
                                     "warps_per_sm": prof.get("theta_warps_per_sm"),
                                     "note": "latency-bound; ncu --set full, profiles/r2_theta_sym_c3.md"}
    line = {
        "metric": "sphere Poisson DOF/s (FP64)", "value": value, "unit": "DOF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if slab else ("weak" if world > 1 else "strong"),
        "vs_baseline": value / PUBLISHED_DOF_PER_S if cfg.name == "C3" else None,
        "dtype": "f64", "data": "synthetic: seeded spherical-harmonic sums generated on the device",
        "config": {**config_block(cfg, world), "transport": args.transport if slab else None,
                   "devices": min(world, ndev), "shared_gpus": shared},
        "gpu_launches": launches, "clocks": clk.summary(),
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "parity_rel_err_vs_analytic": err,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
