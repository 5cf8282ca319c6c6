"""Robustness sweep of the grid solve across kernel-selection boundaries: rough
zero-mean data at many (M, N), compared with the reference's own composition
(oracle/_ref; TEST INFRASTRUCTURE, the checker only).  python tools/sweep_sizes.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import ref_grid, zero_mean_noise  # noqa: E402
from oracle.oracle import Oracle, Reference  # noqa: E402
from paper_1510_08094_b200.poisson import Plan  # noqa: E402

O, R = Oracle(), Reference()
sizes = [(16, 16), (24, 20), (40, 12), (100, 30), (200, 24), (256, 40), (300, 20), (600, 28), (1024, 24), (1200, 16),
         (2000, 20), (3000, 16), (4096, 16), (5000, 12), (6000, 12), (8192, 12), (9000, 8), (14000, 8), (20000, 8),
         (24, 600), (40, 1200), (32, 4096), (24, 5000), (16, 10000)]
worst = 0.0
for m, n in sizes:
    f = zero_mean_noise(O, m, n, m + 3 * n)
    with Plan(m, n) as plan:
        u = plan.solve_grid(f)
        info = plan.info()
    _, _, ur = ref_grid(R, f, m)
    e = float(np.abs(u - ur).max() / np.abs(ur).max())
    worst = max(worst, e)
    print(f"{m:6d} x {n:6d}  rel err vs reference {e:.2e}  variants {info['variants']:4d} theta thr {info['theta_threads']} "
          f"split {info['theta_split']} chain {info['chain_solver']}", flush=True)
    assert e <= 1e-10, (m, n, e)
print("worst", worst)
