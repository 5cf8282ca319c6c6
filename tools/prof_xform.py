"""Minimal driver for ncu captures of the standalone transforms: analyze_2d and
sample_grid of an m x n complex grid, device tensors.  python tools/prof_xform.py [m] [n]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_08094_b200.poisson import Plan  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
g = torch.randn((m, n), dtype=torch.complex128, device="cuda")
with Plan(m, n) as plan:
    for _ in range(3):
        X = plan.analyze_2d(g)
        G = plan.sample_grid(X, m, n)
    torch.cuda.synchronize()
    print("round trip", float((G - g).abs().max() / g.abs().max()))
