"""K5 coeff_solve (the drop-in for spherekit::solve) on the GPU beside the
reference's own bench_poisson (poisson.cpp:188-230) on the host cores.

GPU rows: bench_poisson's workload shape (band-limited random columns, the
k = 0 mean removed, Msin^2 applied; poisson.cpp:194-216) generated on the
device with the same band and sizes, device-resident F and X, best of reps
of one sk_solve_coeffs (CUDA events on the plan stream, K5 only), plus the
e2e time with host F and X (the reference's value semantics).  The
algorithmic bytes of K5 are 32 B per entry (F in, X out); the kernel also
writes and re-reads the elimination (r, d') (80 B per entry).
Reference rows: Reference.bench_poisson at min(nproc, 16) threads and 1
thread (bench_poisson's own best-of-reps timing).

    python tools/bench_coeff.py --sizes 512,1024,2048,4096 --c3 --out profiles/r2_coeff_bench.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def device_problem(torch, M, N, seed):
    """Band-limited random F like bench_poisson (|k|, |j| <= max(2, s/8)),
    k = 0 column made mean-free, Msin^2 applied column-wise (on the device)."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    band_j, band_k = max(2, M // 8), max(2, N // 8)
    X = torch.zeros((M, N), dtype=torch.complex128, device="cuda")
    j0, j1 = M // 2 - band_j, M // 2 + band_j + 1
    k0, k1 = N // 2 - band_k, N // 2 + band_k + 1
    blk = (torch.rand((j1 - j0, k1 - k0, 2), generator=g, device="cuda", dtype=torch.float64) * 2 - 1)
    X[j0:j1, k0:k1] = torch.view_as_complex(blk.contiguous())
    X[M // 2, N // 2] = 0.0
    # Msin^2 along columns: (-1/4, 1/2, -1/4) at offsets (-2, 0, 2), 1/4 on the first and last rows
    F = 0.5 * X
    F[0] = 0.25 * X[0]
    F[-1] = 0.25 * X[-1]
    F[2:] -= 0.25 * X[:-2]
    F[:-2] -= 0.25 * X[2:]
    F[:, N // 2] = 0.0  # zero surface mean
    return F.contiguous()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="512,1024,2048,4096")
    ap.add_argument("--c3", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-ref", action="store_true")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    from paper_1510_08094_b200.poisson import Plan
    shapes = [(int(s), int(s)) for s in args.sizes.split(",") if s]
    if args.c3:
        shapes.append((20000, 10000))
    rows = []
    for M, N in shapes:
        F = device_problem(torch, M, N, 7)
        X = torch.empty_like(F)
        with Plan(M, N) as plan:
            plan.enable_stage_timing(True)
            best = float("inf")
            for _ in range(args.reps + 1):
                plan.solve_coeffs(F, X)
                best = min(best, plan.stage_times()["coeff_solve_ms"])
            Fh = F.cpu().numpy()
            Xh = np.empty_like(Fh)
            plan.solve_coeffs(Fh, Xh)
            t0 = time.perf_counter()
            for _ in range(max(1, args.reps // 2)):
                plan.solve_coeffs(Fh, Xh)
            e2e = (time.perf_counter() - t0) / max(1, args.reps // 2)
        dof = M * N / 2
        row = {"M": M, "N": N, "k5_ms": best, "k5_dof_per_s": dof / (best * 1e-3),
               "k5_algorithmic_gbs": 32 * M * N / (best * 1e-3) / 1e9,
               "k5_moved_gbs": 80 * M * N / (best * 1e-3) / 1e9, "e2e_host_ms": 1e3 * e2e,
               "e2e_dof_per_s": dof / e2e}
        print(json.dumps(row), flush=True)
        rows.append(row)
        del F, X
    ref = []
    if not args.no_ref:
        from oracle.oracle import Reference, reference_available
        if reference_available():
            R = Reference()
            sizes = [s for s, _ in shapes if s <= 4096]
            for th in sorted({min(os.cpu_count() or 1, 16), 1}):
                secs, reps = R.bench_poisson(sizes, th)
                for s, t, r in zip(sizes, secs, reps):
                    d = {"size": s, "threads": th, "seconds": t, "reps": r, "dof_per_s": s * s / 2 / t}
                    print(json.dumps(d), flush=True)
                    ref.append(d)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump({"gpu": rows, "reference_bench_poisson": ref, "nproc": os.cpu_count()}, fh, indent=1)


if __name__ == "__main__":
    main()
