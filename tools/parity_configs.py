"""Config-scale parity against the reference itself (SURVEY §8d "generate
once, hash, feed identical bytes to both paths").

For each config the bench's seeded spherical-harmonic input is generated on
the device (sk_shgen), copied to the host and hashed (SHA-256 of the float64
bytes); the SAME bytes go through

  * the reference's own grid composition (oracle/_ref: sample_dfs ->
    analyze_2d -> Msin^2 -> solve -> sample_grid; solve() on
    min(nproc, 16) threads as thread_budget caps it), and
  * the device: sk_solve_grid (real grid path, with X_half) and, where the
    transform lengths fit one CTA, sk_solve_grid_exact,

and the errors are max|x_gpu - x_ref| / max|x_ref| (test_poisson.cpp:142-149).
A white-noise (under-resolved) table at small sizes records how far the real
grid path's Hermitian output sits from Re(U_ref) — the declared semantic
difference — and that sk_solve_grid_exact closes it.

    python tools/parity_configs.py --configs C2,C4,C3 --out profiles/r2_parity_configs.json

ORACLE / TEST INFRASTRUCTURE: imports oracle/ only as the checker."""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C4,C3")
    ap.add_argument("--c4-rhs", type=int, default=4)
    ap.add_argument("--noise", default="64x48,256x128,512x256,2048x1024")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()

    import torch
    from conftest import ref_grid, zero_mean_noise
    from oracle.oracle import Oracle, Reference, phys_from_doubled
    from paper_1510_08094_b200 import inputs
    from paper_1510_08094_b200.poisson import Plan

    ref = Reference()
    orc = Oracle()
    threads = min(os.cpu_count() or 1, 16)
    rows_out = []
    for name in [c for c in args.configs.split(",") if c]:
        cfg = inputs.CONFIGS[name]
        nrhs = args.c4_rhs if name == "C4" else cfg.nrhs
        M, N, R = cfg.M, cfg.N, cfg.M // 2 + 1
        for r in range(nrhs):
            seed = 11 + r
            with Plan(M, N) as plan:
                fd = torch.empty((R, N), dtype=torch.float64, device="cuda")
                plan.shgen(cfg.L, torch.from_numpy(inputs.sh_coeffs(seed, cfg.L, cfg.p)).cuda(), fd)
                torch.cuda.synchronize()
                f = fd.cpu().numpy()
                del fd
                sha = hashlib.sha256(f.tobytes()).hexdigest()
                t0 = time.perf_counter()
                u, Xh = plan.solve_grid(f, coeffs=True)
                t_gpu = time.perf_counter() - t0
                exact = None
                if M <= 12000 and N <= 12000:
                    U_ex, X_ex = plan.solve_grid_exact(f, coeffs=True)
                    exact = (U_ex, X_ex)
            t0 = time.perf_counter()
            X_ref, U_ref = ref.grid_pipeline(f, M, threads=threads)
            t_ref = time.perf_counter() - t0
            u_ref = phys_from_doubled(U_ref, M)
            row = {
                "config": name, "rhs": r, "M": M, "N": N, "L": cfg.L, "p": cfg.p, "seed": seed,
                "f_sha256": sha, "ref_seconds": t_ref, "ref_threads": threads, "gpu_call_seconds": t_gpu,
                "u_rel_err_vs_ref": rel(u, u_ref.real),
                "ref_u_imag_rel": float(np.abs(u_ref.imag).max() / np.abs(u_ref).max()),
                "X_half_rel_err_vs_ref": rel(Xh[: N // 2], X_ref[:, N // 2:].T),
                "X_nyquist_rel_err_vs_ref": float(np.abs(Xh[N // 2] - X_ref[:, 0]).max() / np.abs(X_ref).max()),
            }
            # k = 0 column separately (unpivoted chains vs the reference's bordered elimination)
            row["X_k0_rel_err_vs_ref"] = float(np.abs(Xh[0] - X_ref[:, N // 2]).max() / np.abs(X_ref).max())
            if exact is not None:
                row["exact_U_rel_err_vs_ref"] = rel(exact[0], U_ref)
                row["exact_X_rel_err_vs_ref"] = rel(exact[1], X_ref)
            print(json.dumps(row), flush=True)
            rows_out.append(row)
            del X_ref, U_ref, u_ref
    noise = []
    for spec in [s for s in args.noise.split(",") if s]:
        m, n = (int(x) for x in spec.split("x"))
        f = zero_mean_noise(orc, m, n, 3 + m)
        X_ref, U_ref, u_herm = ref_grid(ref, f, m, threads=threads)
        with Plan(m, n) as plan:
            u = plan.solve_grid(f)
            U_ex, X_ex = plan.solve_grid_exact(f, coeffs=True)
        u_ref = phys_from_doubled(U_ref, m)
        row = {
            "white_noise": f"{m}x{n}",
            "grid_path_vs_Re_u_ref": rel(u, u_ref.real),
            "ref_own_Im_u_rel": float(np.abs(u_ref.imag).max() / np.abs(u_ref).max()),
            "grid_path_vs_hermitian_completion_of_X_ref": rel(u, u_herm),
            "exact_U_vs_U_ref": rel(U_ex, U_ref),
            "exact_X_vs_X_ref": rel(X_ex, X_ref),
        }
        print(json.dumps(row), flush=True)
        noise.append(row)
    if args.out:
        import platform
        with open(args.out, "w") as fh:
            json.dump({"configs": rows_out, "white_noise": noise, "host": platform.node(),
                       "nproc": os.cpu_count(), "gpu": torch.cuda.get_device_name(0)}, fh, indent=1)


if __name__ == "__main__":
    main()
