import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import ref_grid, zero_mean_noise
from oracle.oracle import Oracle, Reference
from paper_1510_08094_b200.poisson import Plan
O, R = Oracle(), Reference()
ms = [int(x) for x in sys.argv[1].split(",")]
n = 32
for m in ms:
    f = zero_mean_noise(O, m, n, m * n)
    X_ref, U_ref, u_herm = ref_grid(R, f, m)
    try:
        with Plan(m, n) as plan:
            u, Xh = plan.solve_grid(f, coeffs=True)
            info = plan.info()
    except Exception as e:
        print(m, "unsupported", str(e)[:60]); continue
    E = np.abs(Xh[: n // 2] - X_ref[:, n // 2:].T)
    sc = np.abs(X_ref).max()
    bad = np.nonzero(E.max(axis=1) > 1e-10 * sc)[0]
    print(m, "L", m // 2, "L%4", (m // 2) % 4, "variants", info["variants"], f"X err {E.max()/sc:.2e}", "bad k", bad[:6], flush=True)
