"""CPU, gloo, world_size 2 (and 3): the slab-decomposed orchestration
(SlabSolver: row/mode slabs, all-to-all split sizes and block layouts)
produces exactly the single-process result.  The per-rank stage work is a
numpy stand-in with the same buffer layouts as the CUDA stages (the CUDA
stages themselves are checked on the GPU, tests/test_gpu_parity.py
test_slab_stages_bitwise_equal_single_gpu)."""
import os
import socket

import numpy as np
import pytest


class NumpyStages:
    """Layout-faithful stand-in: lambda_fwd = analyze_1d of each row (k >= 0),
    theta = a column-global map per lambda mode, lambda_inv = synthesis."""

    def __init__(self, M, N):
        self.M, self.N = M, N
        self.rows, self.cols = M // 2 + 1, N // 2 + 1
        self.sign = (-1.0) ** np.arange(self.cols)

    def lambda_fwd(self, P, rb, cb, rank, f_rows, send):
        import torch
        X = np.fft.rfft(f_rows.numpy(), axis=1) / self.N * self.sign  # (rows_r, cols)
        send.copy_(torch.from_numpy(np.ascontiguousarray(X.T).view(np.float64).ravel()))

    def theta_map(self, cols, kappas):
        return cols * (1.0 + kappas[:, None]) + 0.25 * np.cumsum(cols, axis=1)[:, ::-1]

    def theta(self, P, rb, cb, rank, recv):
        import torch
        c0, c1 = cb[rank], cb[rank + 1]
        nc = c1 - c0
        buf = recv.numpy().view(np.complex128)
        cols = np.zeros((nc, self.rows), complex)
        for s in range(P):
            rs = rb[s + 1] - rb[s]
            cols[:, rb[s]: rb[s + 1]] = buf[nc * rb[s]: nc * rb[s + 1]].reshape(nc, rs)
        # statistics as the CUDA theta stage reports them: the k = 0 owner the
        # surface mean (here the mean of the k = 0 column), everyone max |F|
        self._stats = (cols[0].real.mean() if c0 == 0 and nc else 0.0, 0.0, float(np.abs(cols).max()) if nc else 0.0)
        out = self.theta_map(cols, np.arange(c0, c1, dtype=float))
        for s in range(P):
            buf[nc * rb[s]: nc * rb[s + 1]] = out[:, rb[s]: rb[s + 1]].ravel()
        recv.copy_(torch.from_numpy(buf.view(np.float64)))

    def stats(self):
        return self._stats

    def lambda_inv(self, P, rb, cb, rank, back, u_rows):
        import torch
        rr = rb[rank + 1] - rb[rank]
        V = back.numpy().view(np.complex128).reshape(self.cols, rr).T * self.sign
        u_rows.copy_(torch.from_numpy(np.fft.irfft(V, n=self.N, axis=1) * self.N))

    def full(self, f):
        X = np.fft.rfft(f, axis=1) / self.N * self.sign
        V = self.theta_map(X.T.copy(), np.arange(self.cols, dtype=float)).T
        return np.fft.irfft(V * self.sign, n=self.N, axis=1) * self.N


def _worker(rank, world, port, M, N, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1510_08094_b200._lib import precondition_error
    from paper_1510_08094_b200.distributed import SlabSolver, gather_rows
    rng = np.random.default_rng(7)
    f = rng.standard_normal((M // 2 + 1, N))
    f -= f.mean()  # zero surface mean (of the stand-in's statistic)
    st = NumpyStages(M, N)
    solver = SlabSolver(M, N, rank, world, device=torch.device("cpu"), backend=st)
    rows = torch.from_numpy(f[solver.rb[rank]: solver.rb[rank + 1]].copy())
    u = solver.solve(rows)
    allu = gather_rows(u, solver.rb)
    # a nonzero-mean right-hand side raises precondition_error on EVERY rank
    raised = False
    try:
        solver.solve(rows + 1.0)
    except precondition_error:
        raised = True
    flags = [None] * world
    dist.all_gather_object(flags, raised)
    if rank == 0:
        q.put((allu.numpy(), st.full(f), flags))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,M,N", [(2, 40, 24), (3, 38, 30)])
def test_slab_orchestration_gloo(world, M, N):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, ref, raised = q.get(timeout=90)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    assert raised == [True] * world, raised


def test_slab_bounds_cover():
    from paper_1510_08094_b200.distributed import slab_bounds
    for total in (1, 7, 10001, 5001):
        for P in (1, 2, 3, 8):
            b = slab_bounds(total, P)
            assert b[0] == 0 and b[-1] == total and all(b[i] <= b[i + 1] for i in range(P))


# ------------------------------------------------------------ fused peer path
def _p2p_worker(rank, world, port, M, N, L, q):
    """One rank of the fused-transpose (CUDA IPC peer-store) slab solve.  On
    the single-GPU test box both ranks share device 0: the peer mappings are
    then same-device IPC mappings, the kernels are exactly those of a
    multi-GPU run, and the ranks only meet at host barriers between stages
    (no kernel waits on another rank)."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1510_08094_b200 import inputs
    from paper_1510_08094_b200.distributed import SlabSolver, gather_rows
    from paper_1510_08094_b200.poisson import Plan
    dev = torch.device("cuda", 0)
    rows = M // 2 + 1
    c = torch.from_numpy(inputs.sh_coeffs(11, L, 2.0)).to(dev)
    with Plan(M, N) as plan:
        f = torch.empty((rows, N), dtype=torch.float64, device=dev)
        plan.shgen(L, c, f)
        u1 = plan.solve_grid(f).cpu()
    solver = SlabSolver(M, N, rank, world, device=dev, transport="p2p")
    mine = f[solver.rb[rank]: solver.rb[rank + 1]].contiguous()
    u = solver.solve(mine)
    u = solver.solve(mine)  # second solve reuses the mapped buffers
    torch.cuda.synchronize()
    allu = gather_rows(u.cpu(), solver.rb)
    # a nonzero-mean right-hand side raises the reference's precondition_error
    # on every rank (as sk_solve_grid does on one GPU)
    from paper_1510_08094_b200._lib import precondition_error
    raised = False
    try:
        solver.solve(mine + 1.0)
    except precondition_error:
        raised = True
    flags = [None] * world
    dist.all_gather_object(flags, raised)
    solver.close()
    if rank == 0:
        q.put((allu.numpy(), u1.numpy(), flags))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,M,N,L", [(2, 512, 256, 40), (3, 240, 200, 30), (2, 64, 3000, 12),
                                           (2, 6000, 64, 20), (3, 12000, 48, 16), (2, 32768, 48, 12),
                                           (2, 48, 32768, 12), (3, 30, 32768, 10)])  # theta_sym, multi-pass theta, split lambda rows
def test_p2p_fused_transposes_bitwise(world, M, N, L):
    """The fused peer-store slab solve equals the single-GPU grid solve bit
    for bit (the theta stage is slab-invariant); 64 x 3000 runs the forward
    lambda stage on 4-CTA clusters with 64-byte peer stores, 6000 / 12000 x
    N the theta_sym kernel, 32768 x 48 the multi-pass theta stage with peer
    stores and M x 32768 the lambda rows split over CTA pairs (peer stores
    forward, the per-parity TMA gather on the rank's own rows inverse): the
    kernels of C3 and C5 on several GPUs."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, M, N, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, ref, raised = q.get(timeout=240)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(got, ref)
    assert raised == [True] * world, raised
