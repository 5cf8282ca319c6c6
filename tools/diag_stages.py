"""Per-stage GPU diagnostics against dense numpy formulas (debug tool)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1510_08094_b200.poisson import Plan


def lap_dense(M):
    L = M // 2
    A = np.zeros((M, M))
    for i in range(M):
        t = i - L
        if i - 2 >= 0: A[i, i - 2] = (t - 2) * (t - 1) / 4
        if i + 2 < M: A[i, i + 2] = (t + 2) * (t + 1) / 4
        A[i, i] = -t * t / 2
        if i == 0: A[i, i] = -t * (t - 1) / 4
        if i == M - 1: A[i, i] = -t * (t + 1) / 4
    return A


def msin2_dense(M):
    S = np.zeros((M, M))
    for i in range(M):
        if i - 2 >= 0: S[i, i - 2] = -0.25
        if i + 2 < M: S[i, i + 2] = -0.25
        S[i, i] = 0.25 if i in (0, M - 1) else 0.5
    return S


def theta_ref(a, kappa, M):
    L = M // 2
    s = -1.0 if kappa % 2 else 1.0
    g = np.zeros(M, complex)
    for i in range(M):
        p = i - L
        g[i] = a[p] if p >= 0 else s * a[-p]
    t = np.arange(M) - L
    X = (1.0 / M) * ((-1.0) ** np.abs(t)) * np.fft.fft(g)[t % M]
    F = msin2_dense(M) @ X
    A = lap_dense(M) - kappa * kappa * np.eye(M)
    if kappa == 0:
        w = np.array([2.0 / (1 - tt * tt) if tt % 2 == 0 else 0.0 for tt in t])
        A[L, :] = 2 * np.pi * w
        F = F.copy(); F[L] = 0
    x = np.linalg.solve(A, F)
    p = np.arange(L + 1)
    v = np.exp(2j * np.pi * np.outer(p, t) / M) @ x
    return v, X, x


def main(M, N):
    rows, cols = M // 2 + 1, N // 2 + 1
    rng = np.random.default_rng(0)
    rb, cb = [0, rows], [0, cols]
    dev = torch.device("cuda")
    with Plan(M, N) as plan:
        print("info", plan.info())
        f = rng.standard_normal((rows, N))
        spec = torch.empty(2 * rows * cols, dtype=torch.float64, device=dev)
        plan.stage_lambda_fwd(1, rb, cb, 0, torch.from_numpy(f).to(dev), spec)
        torch.cuda.synchronize()
        S = spec.cpu().numpy().view(np.complex128).reshape(cols, rows)
        ref = (np.fft.rfft(f, axis=1) / N * ((-1.0) ** np.arange(cols))).T
        print("lambda_fwd rel err", np.abs(S - ref).max() / np.abs(ref).max())
        # theta on random column data
        a = rng.standard_normal((cols, rows)) + 1j * rng.standard_normal((cols, rows))
        buf = torch.from_numpy(a.copy().view(np.float64).reshape(-1)).to(dev)
        plan.stage_theta(1, rb, cb, 0, buf)
        torch.cuda.synchronize()
        V = buf.cpu().numpy().view(np.complex128).reshape(cols, rows)
        worst = 0
        for kappa in sorted(set([0, 1, 2, 3, cols // 2, cols - 2, cols - 1])):
            v, X, x = theta_ref(a[kappa], kappa, M)
            e = np.abs(V[kappa] - v).max() / np.abs(v).max()
            worst = max(worst, e)
            print(f"  theta kappa={kappa} rel err {e:.3e}")
        # lambda inverse
        b = rng.standard_normal((cols, rows)) + 1j * rng.standard_normal((cols, rows))
        bt = torch.from_numpy(b.copy().view(np.float64).reshape(-1)).to(dev)
        u = torch.empty((rows, N), dtype=torch.float64, device=dev)
        plan.stage_lambda_inv(1, rb, cb, 0, bt, u)
        torch.cuda.synchronize()
        Vk = (b * ((-1.0) ** np.arange(cols))[:, None]).T
        uref = np.fft.irfft(Vk, n=N, axis=1) * N
        print("lambda_inv rel err", np.abs(u.cpu().numpy() - uref).max() / np.abs(uref).max())


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        M, N = map(int, arg.split("x"))
        print("=== M x N =", M, N)
        main(M, N)
