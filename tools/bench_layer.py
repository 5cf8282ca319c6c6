"""Throughput of the widened boundary entry points on one B200 (device-resident
inputs, CUDA events on the plan's stream, best and median of reps), against
the HBM roofline of MEASURED_PEAKS.json, with the reference's CPU time for the
same call on a smaller sample (oracle/_ref, when built) for scale.

    python tools/bench_layer.py > profiles/r1_layer_bench.jsonl

Algorithmic bytes per call:
  assemble_poisson  16 M N (F written once; the K x (M + N) factors are L2-resident)
  analyze_2d        2 passes x (16 + 16) m n  (read + transposed write)
  sample_grid       rows n_out 32 + n_out m_out (16 + 16) (two passes)
  sample_dfs        8 (m/2+1) n read + 16 m n written
"""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1510_08094_b200.poisson import Plan  # noqa: E402


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p))["hbm_gbs"] if os.path.exists(p) else 6650.0


def timed(plan, fn, reps=10, warm=3):
    st = torch.cuda.current_stream()
    plan.set_stream(st.cuda_stream)
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), statistics.median(ts)


def ref_lib():
    try:
        from oracle.oracle import Reference, reference_available
        return Reference() if reference_available() else None
    except Exception:
        return None


def cpu_time(fn, reps=2):
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def main():
    pk = peak()
    R = ref_lib()
    dev = torch.device("cuda")
    out = []
    g = torch.Generator(device="cuda").manual_seed(0)

    def crand(*shape):
        return torch.complex(torch.randn(*shape, generator=g, device=dev, dtype=torch.float64),
                             torch.randn(*shape, generator=g, device=dev, dtype=torch.float64))

    # assemble_poisson at C3 size: K terms of 2048 theta / lambda modes
    for M, N, K in [(20000, 10000, 12), (20000, 10000, 64), (4096, 2048, 12)]:
        plan = Plan(M, N)
        d, col, row = crand(K), crand(K, 2048), crand(K, 2048)
        F = torch.empty((M, N), dtype=torch.complex128, device=dev)
        best, med = timed(plan, lambda: plan.assemble(d, col, row, 0.0, F))
        by = 16.0 * M * N
        rec = {"op": "assemble_poisson", "M": M, "N": N, "K": K, "ms": best, "ms_median": med,
               "achieved_gbs": by / best / 1e6, "peak_gbs": pk, "frac": by / best / 1e6 / pk,
               "flops_per_entry": 8 * K}
        if R is not None and M * N <= 1 << 23:
            dn, cn, rn = (x.cpu().numpy() for x in (d, col, row))
            rec["cpu_reference_ms"] = 1e3 * cpu_time(lambda: R.assemble_lowrank(dn, cn, rn, 0.0, M, N))
        out.append(rec)
        plan.close()
    # analyze_2d / sample_grid on large complex grids
    xp = Plan(8, 4)
    for m, n in [(8192, 8192), (4096, 10000), (2048, 2048)]:
        grid = crand(m, n)
        X = torch.empty_like(grid)
        best, med = timed(xp, lambda: xp.analyze_2d(grid, X))
        by = 2 * 32.0 * m * n
        rec = {"op": "analyze_2d", "m": m, "n": n, "ms": best, "ms_median": med, "achieved_gbs": by / best / 1e6,
               "peak_gbs": pk, "frac": by / best / 1e6 / pk}
        if R is not None and m * n <= 1 << 22:
            gn = grid.cpu().numpy()
            rec["cpu_reference_ms"] = 1e3 * cpu_time(lambda: R.analyze_2d(gn))
        out.append(rec)
        G = torch.empty_like(grid)
        best, med = timed(xp, lambda: xp.sample_grid(X, m, n, G))
        rec = {"op": "sample_grid", "m": m, "n": n, "ms": best, "ms_median": med, "achieved_gbs": by / best / 1e6,
               "peak_gbs": pk, "frac": by / best / 1e6 / pk}
        if R is not None and m * n <= 1 << 22:
            Xn = X.cpu().numpy()
            rec["cpu_reference_ms"] = 1e3 * cpu_time(lambda: R.sample_grid(Xn, m, n))
        out.append(rec)
    # DFS doubling at C3
    m, n = 20000, 10000
    phys = torch.randn(m // 2 + 1, n, generator=g, device=dev, dtype=torch.float64)
    grid = torch.empty((m, n), dtype=torch.complex128, device=dev)
    best, med = timed(xp, lambda: xp.sample_dfs(phys, m, grid))
    by = 8.0 * (m // 2 + 1) * n + 16.0 * m * n
    out.append({"op": "sample_dfs", "m": m, "n": n, "ms": best, "ms_median": med, "achieved_gbs": by / best / 1e6,
                "peak_gbs": pk, "frac": by / best / 1e6 / pk})
    # Bluestein transforms (prime factor > 7): 602 = 2 * 7 * 43 and 4 * 1031
    for m, n in [(602, 602), (4124, 1024)]:
        grid = crand(m, n)
        X = torch.empty_like(grid)
        best, med = timed(xp, lambda: xp.analyze_2d(grid, X))
        by = 2 * 32.0 * m * n
        rec = {"op": "analyze_2d (Bluestein)", "m": m, "n": n, "ms": best, "ms_median": med,
               "achieved_gbs": by / best / 1e6, "peak_gbs": pk, "frac": by / best / 1e6 / pk}
        if R is not None and m * n <= 1 << 22:
            gn = grid.cpu().numpy()
            rec["cpu_reference_ms"] = 1e3 * cpu_time(lambda: R.analyze_2d(gn))
        out.append(rec)
    # the reference-semantics grid solve (composition of the device stages)
    for M, N in [(4096, 2048), (2048, 1024)]:
        plan = Plan(M, N)
        rows = M // 2 + 1
        from paper_1510_08094_b200 import inputs
        f = torch.empty((rows, N), dtype=torch.float64, device=dev)
        plan.shgen(64, torch.from_numpy(inputs.sh_coeffs(3, 64, 2.0)).cuda(), f)
        best, med = timed(plan, lambda: plan.solve_grid_exact(f))
        rec = {"op": "solve_grid_exact", "M": M, "N": N, "ms": best, "ms_median": med,
               "dof_per_s": M * N / 2 / (best * 1e-3)}
        out.append(rec)
        plan.close()
    # GE building blocks (lowrank.hpp:73-93) on a doubled grid resident on the device:
    # one step = pivot search (reads the upper half: 16 (m/2+1) n bytes) + cross + update
    # (reads and writes the grid: 32 m n bytes, max|.| fused); CPU reference on a smaller grid
    xp = Plan(8, 4)
    for m, n in [(4096, 4096), (2048, 2048)]:
        grid0 = crand(m, n)
        jm = (m - torch.arange(m, device=dev)) % m
        km = (torch.arange(n, device=dev) + n // 2) % n
        grid0 = 0.5 * (grid0 + grid0[jm][:, km])  # BMC-symmetric noise (full rank: every step does work)
        grid = grid0.clone()
        out_g = torch.empty_like(grid)
        p = xp.pivot_search(grid)
        bs, ms_ = timed(xp, lambda: xp.pivot_search(grid))
        bu, mu_ = timed(xp, lambda: xp.ge_step(grid, p, out_g))
        steps = 16
        t0 = time.perf_counter()
        piv, resid = xp.ge_run(grid, tau=0.0, max_steps=steps)
        torch.cuda.synchronize()
        run_ms = 1e3 * (time.perf_counter() - t0) / max(len(piv), 1)
        by = 16.0 * (m // 2 + 1) * n + 32.0 * m * n
        rec = {"op": "ge_step (pivot_search + update)", "m": m, "n": n, "search_ms": bs, "update_ms": bu,
               "run_ms_per_step": run_ms, "steps": len(piv), "achieved_gbs": by / (bs + bu) / 1e6, "peak_gbs": pk,
               "frac": by / (bs + bu) / 1e6 / pk, "update_gbs": 32.0 * m * n / bu / 1e6}
        if R is not None and m * n <= 1 << 22:
            gn = grid0.cpu().numpy()
            pr = R.pivot_search(gn)
            rec["cpu_reference_ms"] = 1e3 * (cpu_time(lambda: R.pivot_search(gn)) + cpu_time(lambda: R.ge_step(gn, pr)))
        out.append(rec)
    xp.close()
    for r in out:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
