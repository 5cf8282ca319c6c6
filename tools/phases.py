"""Per-phase cycle breakdown of theta_kernel (debug build with -DSK_PHASES:
tools/libsk_poisson_phases.so).  Usage: python tools/phases.py C3"""
import ctypes, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1510_08094_b200 import _lib
_lib.LIB_PATH = os.path.join(ROOT, "tools", "libsk_poisson_phases.so")
import torch
from paper_1510_08094_b200 import inputs
from paper_1510_08094_b200.poisson import Plan

cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
plan = Plan(cfg.M, cfg.N)
rows = cfg.M // 2 + 1
f = torch.empty((rows, cfg.N), dtype=torch.float64, device="cuda")
plan.shgen(cfg.L, torch.from_numpy(inputs.sh_coeffs(1, cfg.L, cfg.p)).cuda(), f)
u = torch.empty_like(f)
for _ in range(3):
    plan.solve_grid(f, u)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (4096 * 24))()
assert _lib.load().sk_debug_phases(buf) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 24).astype(np.int64)
n = min(4096, 2 * (cfg.N // 2 + 1))
a = a[:n]
names = ["bars+issue+twiddles+TMA wait", "fold", "fft fwd", "mean+inner+chain+ solve", "pivot- TMA wait",
         "chain- solve", "x0/fmax/export", "fft inv", "cluster sync+combine+stores", "final cluster sync", ""]
if plan.info()["variants"] & 64:  # theta_sym_kernel's probes
    names = ["loads (column TMA wait)", "fold + paired stage 0", "restricted fwd stages", "window wait+mean+inner",
             "both chains", "x0/fmax/export", "fft inv", "cluster sync+combine+stores", "final cluster sync", "", ""]
last = 9 if plan.info()["variants"] & 64 else 10
d = np.diff(a[:, :last + 1], axis=1)
tot = (a[:, last] - a[:, 0])
print(f"{cfg.name}: CTAs sampled {n}, mean cycles per CTA {tot.mean():.0f}")
for i in range(last):
    print(f"  {names[i]:28s} {d[:, i].mean():9.0f} cyc  {100 * d[:, i].mean() / tot.mean():5.1f}%")

sub = a[:, 12:18]
if (sub > 0).all():
    sn = ["loads+sync", "pass1 (F, fwd map)", "scan1", "pass2 (sweep, bwd map)", "scan2", "pass3 (back subst)"]
    base = a[:, 4:5] if plan.info()["variants"] & 64 else a[:, 3:4]
    dd = np.diff(np.concatenate([base, sub], axis=1), axis=1)
    for i, nm in enumerate(sn):
        print(f"    chain+ {nm:18s} {dd[:, i].mean():8.0f} cyc")

# lambda kernels (their own probe table)
lb = (ctypes.c_ulonglong * (2 * 4096 * 8))()
if hasattr(_lib.load(), "sk_debug_phases_lambda") and _lib.load().sk_debug_phases_lambda(lb) == 0:
    la = np.frombuffer(lb, dtype=np.uint64).reshape(2, 4096, 8).astype(np.int64)
    nr = min(4096, cfg.M // 2 + 1)
    for w, (title, nm) in enumerate([("lambda_fwd (row pairs)", ["barrier init + tables + row TMA wait", "forward FFT",
                                                               "real split -> natural order", "cluster barrier",
                                                               "paired stores (half remote)", "exit barrier"]),
                                     ("lambda_inv", ["tables + mode gather (TMA) wait", "C2R pack", "inverse FFT",
                                                     "row store"])]):
        t = la[w, :nr, :len(nm) + 1]
        if (t > 0).all():
            d = np.diff(t, axis=1)
            tot = d.sum(axis=1).mean()
            print(f"{title}: mean cycles per CTA {tot:.0f}")
            for i, n_ in enumerate(nm):
                print(f"  {n_:38s} {d[:, i].mean():9.0f} cyc  {100 * d[:, i].mean() / tot:5.1f}%")
