"""Per-phase cycle breakdown of theta_large_kernel (debug build with
-DSK_PHASES: tools/libsk_poisson_phases.so).  Usage: python tools/phases_large.py C5"""
import os, sys, ctypes
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1510_08094_b200 import _lib
_lib.LIB_PATH = os.path.join(ROOT, "tools", "libsk_poisson_phases.so")
import torch
from paper_1510_08094_b200 import inputs
from paper_1510_08094_b200.poisson import Plan

cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
plan = Plan(cfg.M, cfg.N)
print(plan.info())
rows = cfg.M // 2 + 1
f = torch.empty((rows, cfg.N), dtype=torch.float64, device="cuda")
plan.shgen(min(cfg.L, 256), torch.from_numpy(inputs.sh_coeffs(1, min(cfg.L, 256), cfg.p)).cuda(), f)
u = torch.empty_like(f)
for _ in range(2):
    plan.solve_grid(f, u)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (4096 * 24))()
assert _lib.load().sk_debug_phases(buf) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 24).astype(np.int64)[:, :14]
names = ["chain setup", "pivot TMA issue + twiddles", "fold+decimation (global loads)", "local fft fwd",
         "cluster sync + radix-Q combine", "mean + boundary values", "pivot wait", "chain part (cluster scans)",
         "x0 / export / sync", "inverse radix-Q split", "local fft inv", "cluster sync", "recombination + stores",
         "final cluster sync"]
d = np.diff(a, axis=1)
tot = a[:, 13] - a[:, 0]
print(f"{cfg.name}: mean cycles per CTA {tot.mean():.0f}")
for i in range(13):
    print(f"  {names[i + 1]:32s} {d[:, i].mean():9.0f} cyc  {100 * d[:, i].mean() / tot.mean():5.1f}%")

# lambda split kernels (probes 14..18 forward, 19..23 inverse; the first 4096 CTAs)
b = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 24).astype(np.int64)
for nm, cols, labels in [("lambda_fwd_split", range(14, 19), ["setup + twiddles N", "twiddles h + row loads", "fft", "split + scattered stores"]),
                         ("lambda_inv_split", list(range(19, 24)), ["setup + twiddles N", "twiddles h + gathers + pack", "fft inv", "DSMEM recombine + row stores"])]:
    c = list(cols)
    dd = np.diff(b[:, c], axis=1)
    t = b[:, c[-1]] - b[:, c[0]]
    print(f"{nm}: mean cycles per CTA {t.mean():.0f} (to the last probe)")
    for i, lab in enumerate(labels):
        print(f"  {lab:32s} {dd[:, i].mean():9.0f} cyc  {100 * dd[:, i].mean() / t.mean():5.1f}%")
