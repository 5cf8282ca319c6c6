"""Phase probes of the split lambda kernels (rows of N/2 = 16384 on CTA pairs;
-DSK_PHASES build, tools/build_phases.sh).  python tools/phases_split.py [M] [N]"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1510_08094_b200 import _lib
_lib.LIB_PATH = os.environ.get("SK_PHASES_LIB", os.path.join(ROOT, "tools", "libsk_poisson_phases.so"))
import torch
from paper_1510_08094_b200 import inputs
from paper_1510_08094_b200.poisson import Plan

M = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
N = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
plan = Plan(M, N)
rows = M // 2 + 1
f = torch.empty((rows, N), dtype=torch.float64, device="cuda")
plan.shgen(20, torch.from_numpy(inputs.sh_coeffs(1, 20, 2.0)).cuda(), f)
u = torch.empty_like(f)
for _ in range(3):
    plan.solve_grid(f, u)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (4096 * 24))()
assert _lib.load().sk_debug_phases(buf) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 24).astype(np.int64)[: min(4096, 2 * rows)]
for title, cols, names in [("lambda_fwd_split", [14, 15, 16, 17, 18], ["second table", "row load + first split stage", "half FFT", "real split + stores"]),
                           ("lambda_inv_split", [19, 20, 21, 22, 23], ["second table", "mode gather + pack", "half inverse FFT", "cluster barrier + recombination + stores"])]:
    t = a[:, cols]
    d = np.diff(t, axis=1)
    tot = d.sum(axis=1).mean()
    print(f"{title}: {tot:.0f} cycles per CTA after the first table")
    for i, nm in enumerate(names):
        print(f"  {nm:42s} {d[:, i].mean():9.0f} cyc  {100 * d[:, i].mean() / tot:5.1f}%")
