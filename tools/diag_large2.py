import sys, numpy as np
sys.path.insert(0, '.')
import paper_1510_08094_b200 as pkg
from paper_1510_08094_b200 import inputs
from oracle.oracle import Oracle
o = Oracle()
m, n, L = 32768, 16, 8
c = inputs.sh_coeffs(11, L, 2.0)
f = o.shgen(m, n, L, c)
X, _, u_ref, _ = o.grid_pipeline(f, m, threads=8)
with pkg.Plan(m, n) as plan:
    u, Xh = plan.solve_grid(f, coeffs=True)
Lh = m // 2
for k in range(0, 4):
    g = Xh[k]            # index i = t + M/2
    r = X[:, k + n // 2]
    d = np.abs(g - r)
    idx = np.argsort(d)[::-1][:8]
    print("k", k, "max|X|", np.abs(r).max(), "maxerr", d.max())
    for i in idx:
        print("   t=%d gpu=%s ref=%s" % (i - Lh, g[i], r[i]))
# rough data
rng = np.random.default_rng(1)
f2 = rng.standard_normal((m // 2 + 1, n))
with pkg.Plan(m, n) as plan:
    plan.solve_grid(f2); mu = plan.last_mean()
f2 -= mu.real / (4 * np.pi)
ur = o.grid_pipeline_real(f2, m, threads=8)
with pkg.Plan(m, n) as plan:
    u2 = plan.solve_grid(f2)
d=u2-ur; print(d[0,:3], d[m//4,:3], d[-1,:3]); print("rough rel err", np.abs(u2 - ur).max() / np.abs(ur).max())
