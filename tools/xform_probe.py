"""One analyze_2d + sample_grid at a given size (device-resident), for ncu captures:
python tools/xform_probe.py M N [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_08094_b200.poisson import Plan  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
with Plan(8, 8) as plan:
    g = torch.randn((m, n), dtype=torch.complex128, device="cuda")
    X = torch.empty_like(g)
    g2 = torch.empty_like(g)
    for _ in range(reps):
        plan.analyze_2d(g, X)
        plan.sample_grid(X, m, n, g2)
    torch.cuda.synchronize()
    print(m, n, float((g - g2).abs().max()))
