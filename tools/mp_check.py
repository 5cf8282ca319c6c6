"""A/B of theta_sym_kernel against the pair kernel (SK_THETA_MP=0) on rough
zero-mean data, and C3 stage times (debug tool)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

if len(sys.argv) > 1 and sys.argv[1] == "child":
    from conftest import zero_mean_noise
    from oracle.oracle import Oracle
    from paper_1510_08094_b200.poisson import Plan
    O = Oracle()
    out = {}
    for spec in sys.argv[3].split(","):
        m, n = (int(x) for x in spec.split("x"))
        f = zero_mean_noise(O, m, n, m + n)
        with Plan(m, n) as plan:
            u, Xh = plan.solve_grid(f, coeffs=True)
            out[spec + "_u"] = u
            out[spec + "_X"] = Xh
            out[spec + "_v"] = np.array([plan.info()["variants"]])
    np.savez(sys.argv[2], **out)
    sys.exit(0)

specs = sys.argv[1] if len(sys.argv) > 1 else "32768x24,65536x16,32768x48"
res = {}
for name, env in [("sym", {}), ("pair", {"SK_THETA_MP": "0"})]:
    path = f"/tmp/mp_{name}.npz"
    subprocess.run([sys.executable, __file__, "child", path, specs], check=True, env=dict(os.environ, **env))
    res[name] = np.load(path)
for spec in specs.split(","):
    a, b = res["sym"], res["pair"]
    eu = np.abs(a[spec + "_u"] - b[spec + "_u"]).max() / np.abs(b[spec + "_u"]).max()
    ex = np.abs(a[spec + "_X"] - b[spec + "_X"]).max() / np.abs(b[spec + "_X"]).max()
    print(spec, "variants sym/pair", int(a[spec + "_v"][0]), int(b[spec + "_v"][0]), f"u rel {eu:.2e}  X rel {ex:.2e}")
