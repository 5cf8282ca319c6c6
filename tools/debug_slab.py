import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from oracle.oracle import Oracle
from paper_1510_08094_b200 import inputs
from paper_1510_08094_b200.poisson import Plan
from paper_1510_08094_b200.distributed import slab_bounds
O = Oracle()
m, n, L = 160, 96, 24
f = O.shgen(m, n, L, inputs.sh_coeffs(9, L, 2.0))
rows, cols = m // 2 + 1, n // 2 + 1
dev = torch.device("cuda")
with Plan(m, n) as plan:
    u1 = plan.solve_grid(f); u2 = plan.solve_grid(f)
    print("repeat bitwise:", np.array_equal(u1, u2))
    # P=1 via stages
    fd = torch.from_numpy(f).to(dev)
    spec = torch.empty(2 * rows * cols, dtype=torch.float64, device=dev)
    plan.stage_lambda_fwd(1, [0, rows], [0, cols], 0, fd, spec)
    s1 = spec.clone()
    plan.stage_theta(1, [0, rows], [0, cols], 0, spec)
    t1 = spec.clone()
    for P in (2, 4):
        rb, cb = slab_bounds(rows, P), slab_bounds(cols, P)
        # theta on column slabs using P=1-row layout pieces
        S = s1.view(torch.complex128).view(cols, rows)
        out = torch.empty_like(S)
        for d in range(P):
            nc = cb[d + 1] - cb[d]
            parts = [S[cb[d]:cb[d + 1], rb[s]:rb[s + 1]].contiguous().view(-1) for s in range(P)]
            recv = torch.cat(parts).view(torch.float64).contiguous()
            plan.stage_theta(P, rb, cb, d, recv)
            R = recv.view(torch.complex128)
            off = 0
            for s in range(P):
                rs = rb[s + 1] - rb[s]
                out[cb[d]:cb[d + 1], rb[s]:rb[s + 1]] = R[off: off + nc * rs].view(nc, rs)
                off += nc * rs
        T1 = t1.view(torch.complex128).view(cols, rows)
        diff = (out - T1).abs()
        bad = torch.nonzero(diff > 0)
        print("P", P, "theta bitwise:", bool((diff == 0).all().item()), "max diff", diff.max().item(), "bad cols", sorted(set(bad[:, 0].tolist()))[:20], "n bad", bad.shape[0])
    # detail for P=2, column 5
    P = 2
    rb, cb = slab_bounds(rows, P), slab_bounds(cols, P)
    S = s1.view(torch.complex128).view(cols, rows)
    d = 0
    nc = cb[1] - cb[0]
    parts = [S[cb[d]:cb[d + 1], rb[s]:rb[s + 1]].contiguous().view(-1) for s in range(P)]
    recv = torch.cat(parts).view(torch.float64).contiguous()
    before = recv.clone()
    plan.stage_theta(P, rb, cb, d, recv)
    R = recv.view(torch.complex128); B = before.view(torch.complex128)
    T1 = t1.view(torch.complex128).view(cols, rows)
    k = 5
    got = torch.cat([R[nc * rb[s] + k * (rb[s+1]-rb[s]): nc * rb[s] + (k+1) * (rb[s+1]-rb[s])] for s in range(P)])
    inp = torch.cat([B[nc * rb[s] + k * (rb[s+1]-rb[s]): nc * rb[s] + (k+1) * (rb[s+1]-rb[s])] for s in range(P)])
    print("input col equal to S:", bool((inp == S[k]).all().item()))
    dd = (got - T1[k]).abs()
    print("col", k, "ndiff", int((dd > 0).sum().item()), "first", torch.nonzero(dd > 0)[:10].view(-1).tolist())
    print("got[:4]", got[:4].tolist()); print("ref[:4]", T1[k][:4].tolist())
