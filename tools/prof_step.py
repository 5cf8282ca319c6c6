"""Minimal driver for ncu captures: one config's grid solve, a few times,
device-resident inputs (no bench.py extras)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_08094_b200 import inputs  # noqa: E402
from paper_1510_08094_b200.poisson import Plan  # noqa: E402

cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rows = cfg.M // 2 + 1
with Plan(cfg.M, cfg.N, cfg.nrhs) as plan:
    f = torch.empty((cfg.nrhs, rows, cfg.N), dtype=torch.float64, device="cuda")
    for r in range(cfg.nrhs):
        plan.shgen(cfg.L, torch.from_numpy(inputs.sh_coeffs(11 + r, cfg.L, cfg.p)).cuda(), f[r])
    u = torch.empty_like(f)
    for _ in range(reps):
        plan.solve_grid(f if cfg.nrhs > 1 else f[0], u if cfg.nrhs > 1 else u[0])
    torch.cuda.synchronize()
    plan.enable_stage_timing(True)
    plan.solve_grid(f if cfg.nrhs > 1 else f[0], u if cfg.nrhs > 1 else u[0])
    print(cfg.name, plan.stage_times(), plan.info())
