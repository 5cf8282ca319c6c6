"""Stage times of the grid solve at an arbitrary size (band-limited input):
python tools/size_probe.py M N [reps].  Used to compare column lengths /
CTA residency (e.g. M = 10000 against C3's M = 20000 at equal DOF)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_08094_b200 import inputs  # noqa: E402
from paper_1510_08094_b200.poisson import Plan  # noqa: E402

M, N = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
rows = M // 2 + 1
Lsh = 64
with Plan(M, N, 1) as plan:
    f = torch.empty((rows, N), dtype=torch.float64, device="cuda")
    plan.shgen(Lsh, torch.from_numpy(inputs.sh_coeffs(11, Lsh, 2.0)).cuda(), f)
    u = torch.empty_like(f)
    for _ in range(3):
        plan.solve_grid(f, u)
    torch.cuda.synchronize()
    plan.enable_stage_timing(True)
    acc = {}
    for _ in range(reps):
        plan.solve_grid(f, u)
        for k, v in plan.stage_times().items():
            acc.setdefault(k, []).append(v)
    info = plan.info()
    print(M, N, {k: round(float(np.median(v)), 4) for k, v in acc.items()},
          {k: info[k] for k in ("theta_split", "theta_threads", "lambda_threads", "theta_smem", "lambda_smem", "chain_solver", "variants")})
