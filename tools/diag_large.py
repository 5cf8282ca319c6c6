import sys, numpy as np
sys.path.insert(0, '.')
import paper_1510_08094_b200 as pkg
from paper_1510_08094_b200 import inputs
from oracle.oracle import Oracle
o = Oracle()
for (m, n, L) in [(16384, 48, 20), (32768, 48, 20), (64, 32768, 20), (64, 16384, 20)]:
    c = inputs.sh_coeffs(m // 7 + n, L, 2.0)
    f = o.shgen(m, n, L, c)
    ue = o.shgen(m, n, L, inputs.sh_coeffs(m // 7 + n, L, 2.0, solution=True))
    _, _, u_ref, _ = o.grid_pipeline(f, m, threads=8)
    with pkg.Plan(m, n) as plan:
        info = plan.info(); u = plan.solve_grid(f)
    s = np.abs(ue).max()
    print(m, n, info.get("theta_split"), "gpu-ref %.2e gpu-exact %.2e ref-exact %.2e" % (
        np.abs(u - u_ref).max() / s, np.abs(u - ue).max() / s, np.abs(u_ref - ue).max() / s), flush=True)
    d = (u - ue)
    print("   row0", d[0, :3], "rowmid", d[m // 4, :3], "rowlast", d[-1, :3])
