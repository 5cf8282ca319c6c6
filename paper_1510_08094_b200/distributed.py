"""Slab-decomposed grid solve over several GPUs (one process per GPU).

The lambda stages work on physical theta rows, the theta stage on lambda
modes; the two transposes between them are all-to-all exchanges over NCCL
(torch.distributed plumbing, NVLink/NVSwitch on a B200 box).  The reference
is single-process (its only parallelism is std::thread over lambda columns,
poisson.cpp:147-159); SURVEY §8e.

Block layout of the exchanges: rank r's send buffer after the
forward lambda stage is [k][p - row_b[r]] for all modes k, so the block for
destination d is the contiguous range k in [col_b[d], col_b[d+1]); rank d's
receive buffer is the concatenation over sources s of [k - col_b[d]][p -
row_b[s]] blocks, which the theta stage reads piecewise and overwrites in
place; the return exchange sends the same blocks back.

Two transports (``SlabSolver(transport=...)``):

* ``"p2p"`` (the product on a GPU box): the exchanges are fused into the
  stage kernels.  Every rank allocates its receive / return buffers with
  ``sk_device_alloc``, the CUDA IPC handles are exchanged once through
  torch.distributed, and each rank maps every peer's buffers.  The forward
  lambda kernel then stores mode k of its rows straight into the receive
  buffer of the rank owning k, and the theta kernel stores row p of its
  solved columns straight into the return buffer of the rank owning p (NVLink
  stores over NVSwitch); no collective moves data.  The hand-over between
  stages is stream-ordered: each rank records an interprocess CUDA event
  behind each stage, and a peer's stream waits on it before the stage that
  reads what it wrote (``PeerEvents``); the host only orders every record
  before the matching waits with a barrier that runs while the stage itself
  is still on the GPU, so no stream drains between stages and no kernel ever
  waits on another rank.
* ``"nccl"``: the two exchanges as ``all_to_all_single`` over NCCL — the
  comparison baseline.

The per-rank stage work is pluggable (``backend``) so that the host-side
orchestration can be exercised on CPU with gloo (tests/test_distributed.py);
the product backend is the CUDA library (``CudaStages``).
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np


def slab_bounds(total: int, parts: int) -> List[int]:
    """Contiguous near-equal split of range(total) into `parts` slabs."""
    return [(total * i) // parts for i in range(parts + 1)]


class CudaStages:
    """The three stage entry points of libsk_poisson.so for one rank."""

    def __init__(self, plan):
        self.plan = plan

    def lambda_fwd(self, P, rb, cb, rank, f_rows, send):
        self.plan.stage_lambda_fwd(P, rb, cb, rank, f_rows, send)

    def theta(self, P, rb, cb, rank, recv):
        self.plan.stage_theta(P, rb, cb, rank, recv)

    def lambda_inv(self, P, rb, cb, rank, back, u_rows):
        self.plan.stage_lambda_inv(P, rb, cb, rank, back, u_rows)

    def stats(self):
        """(mean re, mean im, max|F|) of this rank's last theta stage: the
        k = 0 owner contributes the surface mean 2 pi w^T f~_0, every rank the
        max |F| of its modes (poisson.cpp:101-117).  Waits for that stage only
        (sk_stage_stats), not for what is queued behind it."""
        return self.plan.stage_stats()


class PeerBuffers:
    """A device buffer per rank, shared with every other rank through CUDA
    IPC: ``ptrs[d]`` is rank d's buffer as mapped in this process."""

    def __init__(self, nbytes: int, device_index: int, group=None):
        import ctypes

        import torch.distributed as dist

        from . import _lib
        self._lib = _lib.load()
        self.device = device_index
        own = ctypes.c_void_p()
        _lib.check(self._lib.sk_device_alloc(device_index, max(int(nbytes), 16), ctypes.byref(own)))
        self.own = int(own.value)
        h = ctypes.create_string_buffer(64)
        _lib.check(self._lib.sk_ipc_handle(ctypes.c_void_p(self.own), h))
        handles = [None] * dist.get_world_size(group)
        dist.all_gather_object(handles, bytes(h.raw), group=group)
        me = dist.get_rank(group)
        self.ptrs, self._opened = [], []
        for d, hd in enumerate(handles):
            if d == me:
                self.ptrs.append(self.own)
                continue
            q = ctypes.c_void_p()
            _lib.check(self._lib.sk_ipc_open(device_index, ctypes.create_string_buffer(hd, 64), ctypes.byref(q)))
            self.ptrs.append(int(q.value))
            self._opened.append(int(q.value))

    def close(self):
        import ctypes
        for q in self._opened:
            self._lib.sk_ipc_close(ctypes.c_void_p(q))
        self._opened = []
        if self.own:
            self._lib.sk_device_free(ctypes.c_void_p(self.own))
            self.own = 0


class PeerEvents:
    """An interprocess CUDA event per rank (sk_ipc_event_create), opened by
    every other rank: ``evs[d]`` is rank d's event in this process."""

    def __init__(self, device_index: int, group=None):
        import ctypes

        import torch.distributed as dist

        from . import _lib
        self._lib = _lib.load()
        own = ctypes.c_void_p()
        h = ctypes.create_string_buffer(64)
        _lib.check(self._lib.sk_ipc_event_create(device_index, h, ctypes.byref(own)))
        self.own = int(own.value)
        handles = [None] * dist.get_world_size(group)
        dist.all_gather_object(handles, bytes(h.raw), group=group)
        me = dist.get_rank(group)
        self.evs, self._opened = [], []
        for d, hd in enumerate(handles):
            if d == me:
                self.evs.append(self.own)
                continue
            e = ctypes.c_void_p()
            _lib.check(self._lib.sk_ipc_event_open(device_index, ctypes.create_string_buffer(hd, 64), ctypes.byref(e)))
            self.evs.append(int(e.value))
            self._opened.append(int(e.value))

    def close(self):
        import ctypes
        for e in self._opened + ([self.own] if self.own else []):
            self._lib.sk_event_destroy(ctypes.c_void_p(e))
        self._opened, self.own = [], 0


class SlabSolver:
    """One rank of the P-way slab-decomposed grid solve.

    ``solve(f_rows)`` takes this rank's physical rows (row_b[r]..row_b[r+1])
    of f, shape (rows_r, N) float64, and returns the same rows of u.
    """

    def __init__(self, M: int, N: int, rank: int, world: int, device=None, backend=None, group=None,
                 transport: str = "nccl"):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.M, self.N, self.rank, self.P = M, N, rank, world
        self.rows, self.cols = M // 2 + 1, N // 2 + 1
        self.rb = slab_bounds(self.rows, world)
        self.cb = slab_bounds(self.cols, world)
        self.group = group
        # Host-side coordination (ordering event records before waits, the
        # precondition reduction of three host doubles) goes through a CPU
        # (gloo) group when the job's backend is NCCL: an NCCL barrier or
        # all-reduce is stream-ordered behind the queued stage kernels, so
        # waiting for it on the host would drain the stream between stages.
        self.host_group = group
        if dist.is_initialized() and dist.get_backend(group) == "nccl":
            ranks = dist.get_process_group_ranks(group) if group is not None else None
            self.host_group = dist.new_group(ranks=ranks, backend="gloo")
        self.device = device if device is not None else torch.device("cpu")
        if backend is None:
            from .poisson import Plan
            self._plan = Plan(M, N, 1, device.index if hasattr(device, "index") and device.index is not None else 0)
            backend = CudaStages(self._plan)
        self.backend = backend
        r = rank
        self.rows_r = self.rb[r + 1] - self.rb[r]
        self.cols_r = self.cb[r + 1] - self.cb[r]
        # exchange sizes in doubles (complex = 2 doubles)
        self.send_split = [2 * (self.cb[d + 1] - self.cb[d]) * self.rows_r for d in range(world)]
        self.recv_split = [2 * self.cols_r * (self.rb[s + 1] - self.rb[s]) for s in range(world)]
        self.transport = transport
        kw = dict(dtype=torch.float64, device=self.device)
        if transport == "p2p":
            if backend is not None and not isinstance(backend, CudaStages):
                raise ValueError("the p2p transport needs the CUDA stages")
            dev = device.index if device is not None and device.index is not None else 0
            # receive buffer: cols_r x all rows; return buffer: all modes x rows_r (complex)
            self.recv_pb = PeerBuffers(8 * sum(self.recv_split), dev, group)
            self.back_pb = PeerBuffers(8 * sum(self.send_split), dev, group)
            self.recv, self.back = self.recv_pb.own, self.back_pb.own
            # one event per stage and rank: forward lambda done (its stores into
            # the peers' receive buffers landed), theta done (return buffers),
            # inverse lambda done (this rank's return buffer free again)
            self.ev_fwd = PeerEvents(dev, group)
            self.ev_theta = PeerEvents(dev, group)
            self.ev_inv = PeerEvents(dev, group)
        elif transport == "nccl":
            self.send = torch.empty(sum(self.send_split), **kw)
            self.recv = torch.empty(sum(self.recv_split), **kw)
            self.back = torch.empty(sum(self.send_split), **kw)
        else:
            raise ValueError(f"unknown transport {transport!r}")

    def solve(self, f_rows, u_rows=None):
        torch, dist = self.torch, self.dist
        if u_rows is None:
            u_rows = torch.empty_like(f_rows)
        P, rb, cb, r = self.P, self.rb, self.cb, self.rank
        if self.transport == "p2p":
            plan = self.backend.plan
            peers = [d for d in range(P) if d != r]
            plan.stage_lambda_fwd_peer(P, rb, cb, r, f_rows, self.recv_pb.ptrs)
            plan.event_record(self.ev_fwd.own)
            self._host_barrier()  # every rank's record is queued before any wait below
            for d in peers:
                plan.stream_wait(self.ev_fwd.evs[d])  # their stores into our receive buffer
                plan.stream_wait(self.ev_inv.evs[d])  # they have read their return buffers (last solve)
            plan.stage_theta_peer(P, rb, cb, r, self.recv, self.back_pb.ptrs)
            plan.event_record(self.ev_theta.own)
            self._host_barrier()
            for d in peers:
                plan.stream_wait(self.ev_theta.evs[d])  # their stores into our return buffer
            plan.stage_lambda_inv(P, rb, cb, r, self.back, u_rows)
            plan.event_record(self.ev_inv.own)
            # the statistics of this rank's theta stage (the inverse stage is
            # already queued behind it); raised on every rank together
            self.check_precondition()
            return u_rows
        self.backend.lambda_fwd(P, rb, cb, r, f_rows, self.send)
        dist.all_to_all_single(self.recv, self.send, self.recv_split, self.send_split, group=self.group)
        self.backend.theta(P, rb, cb, r, self.recv)
        dist.all_to_all_single(self.back, self.recv, self.send_split, self.recv_split, group=self.group)
        self.backend.lambda_inv(P, rb, cb, r, self.back, u_rows)
        # the theta stage's statistics stay valid through lambda_inv; checking
        # after it keeps the exchanges queued back to back
        self.check_precondition()
        return u_rows

    def _host_barrier(self):
        """Orders every rank's event records before the peers' waits (host
        side only: the stages keep running on the GPUs meanwhile)."""
        self.dist.barrier(group=self.host_group)

    def close(self):
        if self.transport == "p2p":
            self.backend.plan.sync()
            self.dist.barrier(group=self.group)  # no peer still reads our buffers
            self.recv_pb.close()
            self.back_pb.close()
            for ev in (self.ev_fwd, self.ev_theta, self.ev_inv):
                ev.close()

    def check_precondition(self):
        """All-reduce of the mean / max|F| statistics of the last theta stage
        and the reference's nonzero-mean test (poisson.cpp:111-116): every
        rank sees the same reduced values, so every rank raises the
        reference's precondition_error together (the single-GPU sk_solve_grid
        raises it for the same input)."""
        torch, dist = self.torch, self.dist
        stats = getattr(self.backend, "stats", None)
        if stats is None:
            return
        mre, mim, fmax = stats()
        # three host doubles: reduced on the CPU group (no stream is touched)
        t = torch.tensor([mre, mim, fmax], dtype=torch.float64)
        m = t[2:].clone()
        dist.all_reduce(t, group=self.host_group)
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=self.host_group)
        mu = complex(t[0].item(), t[1].item())
        fscale = m.item()
        if fscale != 0.0 and abs(mu) > 1e-6 * 4.0 * np.pi * fscale:
            from ._lib import precondition_error
            raise precondition_error("poisson solve: right-hand side has a nonzero surface mean")


def emulate_slabs(f: np.ndarray, M: int, N: int, P: int) -> np.ndarray:
    """Run the P-rank slab path on ONE GPU, the all-to-all replaced by device
    copies between the per-rank buffers (no rank waits on another)."""
    import torch

    from .poisson import Plan
    rows, cols = M // 2 + 1, N // 2 + 1
    rb, cb = slab_bounds(rows, P), slab_bounds(cols, P)
    dev = torch.device("cuda")
    fd = torch.from_numpy(np.ascontiguousarray(f)).to(dev)
    with Plan(M, N) as plan:
        st = CudaStages(plan)
        sends = []
        for r in range(P):
            rr = rb[r + 1] - rb[r]
            s = torch.empty(2 * cols * rr, dtype=torch.float64, device=dev)
            st.lambda_fwd(P, rb, cb, r, fd[rb[r]: rb[r + 1]].contiguous(), s)
            sends.append(s)
        recvs = []
        for d in range(P):
            parts = [sends[s][2 * cb[d] * (rb[s + 1] - rb[s]): 2 * cb[d + 1] * (rb[s + 1] - rb[s])] for s in range(P)]
            recv = torch.cat(parts).contiguous()
            st.theta(P, rb, cb, d, recv)
            recvs.append(recv)
        u = torch.empty((rows, N), dtype=torch.float64, device=dev)
        for s in range(P):
            rs = rb[s + 1] - rb[s]
            parts = [recvs[d][2 * (cb[d + 1] - cb[d]) * rb[s]: 2 * (cb[d + 1] - cb[d]) * rb[s + 1]] for d in range(P)]
            back = torch.cat(parts).contiguous()
            ur = torch.empty((rs, N), dtype=torch.float64, device=dev)
            st.lambda_inv(P, rb, cb, s, back, ur)
            u[rb[s]: rb[s + 1]] = ur
        torch.cuda.synchronize()
        return u.cpu().numpy()


def gather_rows(u_rows, rows_bounds: Sequence[int], group=None):
    """Collect all ranks' row slabs on every rank (for tests / small cases);
    slabs are padded to a common height for the collective."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    hmax = max(rows_bounds[i + 1] - rows_bounds[i] for i in range(world))
    pad = torch.zeros((hmax, u_rows.shape[1]), dtype=u_rows.dtype, device=u_rows.device)
    pad[: u_rows.shape[0]] = u_rows
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([parts[i][: rows_bounds[i + 1] - rows_bounds[i]] for i in range(world)])
