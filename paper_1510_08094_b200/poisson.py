"""Host-side mirror of the reference Poisson interface (namespace spherekit).

Reference                                         here
------------------------------------------------  ------------------------------------
PoissonProblem{m, n, f}      poisson.hpp:23-26    PoissonProblem(m, n, f)
PoissonSolution{x}           poisson.hpp:28-30    PoissonSolution(x)
solve(pb)                    poisson.hpp:47       solve(pb)            -> sk_solve_coeffs
ResidualReport               poisson.hpp:49-53    ResidualReport
residual(pb, sol)            poisson.hpp:54       residual(pb, sol)    -> sk_residual
bench_poisson(sizes)         poisson.hpp:62       bench_poisson(sizes)
integration_weights(m)       poisson.hpp:21       integration_weights(m)
assemble_poisson(f, m, n,     poisson.hpp:40-41    assemble_poisson(f, m, n, report) -> sk_assemble
  AssembleReport*)
LowRankSphereFun / AssembleReport                 LowRankSphereFun / AssembleReport
analyze_2d(BMCGrid)          fourier.hpp:107      analyze_2d(grid)     -> sk_analyze_2d
sample_grid(X, m, n)         fourier.hpp:108      sample_grid(X, m, n) -> sk_sample_grid
sample_dfs(f, m, n)          sphere_domain.hpp:61 sample_dfs(phys, m)  -> sk_sample_dfs (of samples)
sample_dfs -> analyze_2d -> Msin^2 -> solve ->    solve_grid(f_phys)   -> sk_solve_grid (real, Hermitian)
  sample_grid (the grid-level composition)        solve_grid_exact(f_phys) -> sk_solve_grid_exact
                                                    (the reference's complex doubled grid, every input)

Matrices are numpy complex128 arrays in the reference layout (row i = theta
mode i - m/2, column kc = lambda mode kc - n/2).  Errors raise the
reference's exception types (size_error, precondition_error,
structure_error).  Everything computes on the GPU through libsk_poisson.so.
"""
from __future__ import annotations

import ctypes
import dataclasses
import time
from typing import Optional

import numpy as np

from . import _lib
from ._lib import DeviceError, UnsupportedError, precondition_error, size_error, structure_error

__all__ = [
    "Plan", "PoissonProblem", "PoissonSolution", "ResidualReport", "BenchRow", "solve", "residual", "solve_grid",
    "bench_poisson", "integration_weights", "size_error", "precondition_error", "structure_error", "DeviceError",
    "UnsupportedError", "LowRankSphereFun", "AssembleReport", "assemble_poisson", "analyze_2d", "sample_grid",
    "sample_dfs", "solve_grid_exact", "coefficients_from_half", "rhs_coefficients",
]


def _ptr(a) -> Optional[int]:
    """Raw address of a numpy array or a torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, int):  # raw device address (sk_device_alloc / sk_ipc_open)
        return a
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())  # torch.Tensor


def _pinned_like(a: np.ndarray) -> np.ndarray:
    """A page-locked host array shaped like `a` (torch's pinned allocator; the
    numpy view keeps the tensor alive)."""
    import torch
    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    return t.numpy()


def _is_device(a) -> bool:
    return not isinstance(a, np.ndarray) and getattr(a, "is_cuda", False)


class Plan:
    """An M x N problem (M = doubled theta count, N = lambda count) with
    ``nrhs`` right-hand sides on one CUDA device: owns device buffers, FFT
    tables and a stream (sk_plan_create)."""

    def __init__(self, M: int, N: int, nrhs: int = 1, device: int = 0):
        self.lib = _lib.load()
        self.M, self.N, self.nrhs, self.device = int(M), int(N), int(nrhs), int(device)
        h = ctypes.c_void_p()
        _lib.check(self.lib.sk_plan_create(self.M, self.N, self.nrhs, self.device, ctypes.byref(h)))
        self._h = h

    # -- lifecycle
    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self.lib.sk_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream_ptr: int) -> None:
        _lib.check(self.lib.sk_plan_set_stream(self._h, ctypes.c_void_p(stream_ptr)))
        self._stream = stream_ptr

    def _follow_torch(self, t) -> None:
        """Device tensors: run on torch's current stream of that device, so the
        library's reads/writes are ordered with the surrounding torch work."""
        if _is_device(t):
            import torch
            sp = torch.cuda.current_stream(t.device).cuda_stream
            if getattr(self, "_stream", None) != sp:
                self.set_stream(sp)

    def sync(self) -> None:
        """Wait for all queued work (including pipelined host solves, whose
        deferred precondition errors are raised here)."""
        try:
            _lib.check(self.lib.sk_sync(self._h))
        finally:
            self._inflight = []

    def info(self) -> dict:
        a = (ctypes.c_longlong * 16)()
        _lib.check(self.lib.sk_plan_info(self._h, a))
        keys = ["M", "N", "nrhs", "device", "grid_ok", "rows", "theta_split", "theta_threads", "lambda_threads",
                "last_launches", "theta_smem", "lambda_smem", "chain_solver", "variants"]
        return {k: int(a[i]) for i, k in enumerate(keys)}

    @property
    def grid_supported(self) -> bool:
        return bool(self.info()["grid_ok"])

    def enable_stage_timing(self, on: bool = True) -> None:
        _lib.check(self.lib.sk_enable_stage_timing(self._h, 1 if on else 0))

    def stage_times(self) -> dict:
        t = (ctypes.c_double * 4)()
        _lib.check(self.lib.sk_stage_times(self._h, t))
        return {"lambda_fwd_ms": t[0], "theta_ms": t[1], "lambda_inv_ms": t[2], "coeff_solve_ms": t[3]}

    def last_launches(self) -> int:
        return self.info()["last_launches"]

    # -- coefficient space (drop-in for spherekit::solve)
    def solve_coeffs(self, F, X=None, sync: bool = True):
        """F: (nrhs, M, N) or (M, N) complex128, numpy (host) or torch CUDA."""
        dev = _is_device(F)
        if X is None:
            if dev:
                import torch
                X = torch.empty_like(F)
            else:
                F = np.ascontiguousarray(F, dtype=np.complex128)
                X = np.empty_like(F)
        self._check_shape(F, (self.M, self.N))
        self._follow_torch(F)
        flags = (_lib.SK_DEVICE if dev else _lib.SK_HOST) | (0 if sync else _lib.SK_ASYNC)
        _lib.check(self.lib.sk_solve_coeffs(self._h, _ptr(F), _ptr(X), flags))
        return X

    def residual(self, F, X):
        dev = _is_device(F)
        if not dev:
            F = np.ascontiguousarray(F, dtype=np.complex128)
            X = np.ascontiguousarray(X, dtype=np.complex128)
        out = (ctypes.c_double * 3)()
        self._follow_torch(F)
        _lib.check(self.lib.sk_residual(self._h, _ptr(F), _ptr(X), out, _lib.SK_DEVICE if dev else _lib.SK_HOST))
        return ResidualReport(out[0], out[1], out[2])

    # -- grid space
    def solve_grid(self, f, u=None, coeffs: bool = False, sync: bool = True):
        """f: (nrhs, M/2+1, N) or (M/2+1, N) float64 physical samples.
        Returns u (same shape), and with ``coeffs`` also the k >= 0 solution
        coefficients X_half[k][i] = X[i][k + N/2] ((N/2+1) x M complex)."""
        dev = _is_device(f)
        rows = self.M // 2 + 1
        self._check_shape(f, (rows, self.N))
        Xh = None
        if dev:
            import torch
            if u is None:
                u = torch.empty_like(f)
            if coeffs:
                Xh = torch.empty((self.nrhs, self.N // 2 + 1, self.M), dtype=torch.complex128, device=f.device)
        else:
            f = np.ascontiguousarray(f, dtype=np.float64)
            if u is None:
                # asynchronous host solves copy into u on a side stream: a pageable
                # destination would make that copy synchronous, so allocate pinned
                u = _pinned_like(f) if not sync else np.empty_like(f)
            if coeffs:
                Xh = np.empty((self.nrhs, self.N // 2 + 1, self.M), np.complex128)
        self._follow_torch(f)
        flags = (_lib.SK_DEVICE if dev else _lib.SK_HOST) | (0 if sync else _lib.SK_ASYNC)
        if not sync and not dev:
            # pipelined host solve: every (f, u) pair must outlive its queued
            # copies, i.e. stay referenced until sync() (the C contract)
            self._inflight = getattr(self, "_inflight", []) + [(f, u)]
        _lib.check(self.lib.sk_solve_grid(self._h, _ptr(f), _ptr(u), _ptr(Xh), flags))
        if coeffs:
            if self.nrhs == 1:
                Xh = Xh[0]
            return u, Xh
        return u

    def solve_grid_exact(self, f, coeffs: bool = False):
        """The reference's own grid composition on the device (sk_solve_grid_exact):
        sample_dfs -> analyze_2d -> Msin^2 -> solve -> sample_grid with all N
        lambda modes solved.  f: (nrhs, M/2+1, N) or (M/2+1, N) float64.
        Returns the complex doubled grid U ((nrhs,) M x N, BMCGrid layout) and,
        with ``coeffs``, the full M x N solution coefficients X."""
        dev = _is_device(f)
        self._check_shape(f, (self.M // 2 + 1, self.N))
        shp = (self.nrhs, self.M, self.N) if (len(f.shape) > 2 or self.nrhs > 1) else (self.M, self.N)
        if dev:
            import torch
            U = torch.empty(shp, dtype=torch.complex128, device=f.device)
            X = torch.empty(shp, dtype=torch.complex128, device=f.device) if coeffs else None
        else:
            f = np.ascontiguousarray(f, dtype=np.float64)
            U = np.empty(shp, np.complex128)
            X = np.empty(shp, np.complex128) if coeffs else None
        self._follow_torch(f)
        _lib.check(self.lib.sk_solve_grid_exact(self._h, _ptr(f), _ptr(U), _ptr(X),
                                                _lib.SK_DEVICE if dev else _lib.SK_HOST))
        return (U, X) if coeffs else U

    def last_mean(self):
        out = (ctypes.c_double * 3)()
        _lib.check(self.lib.sk_last_mean(self._h, out))
        return complex(out[0], out[1]), out[2]

    def shgen(self, L: int, coeffs_dev, phys_dev) -> None:
        self._follow_torch(phys_dev)
        _lib.check(self.lib.sk_shgen(self._h, int(L), _ptr(coeffs_dev), _ptr(phys_dev)))

    # -- slab stages (multi-GPU)
    def _bounds(self, P, row_b, col_b):
        rb = (ctypes.c_int * (P + 1))(*row_b)
        cb = (ctypes.c_int * (P + 1))(*col_b)
        return rb, cb

    def stage_lambda_fwd(self, P, row_b, col_b, rank, f_rows, send):
        rb, cb = self._bounds(P, row_b, col_b)
        self._follow_torch(f_rows)
        _lib.check(self.lib.sk_stage_lambda_fwd(self._h, P, rb, cb, rank, _ptr(f_rows), _ptr(send)))

    def stage_theta(self, P, row_b, col_b, rank, recv):
        rb, cb = self._bounds(P, row_b, col_b)
        self._follow_torch(recv)
        _lib.check(self.lib.sk_stage_theta(self._h, P, rb, cb, rank, _ptr(recv)))

    def stage_lambda_fwd_peer(self, P, row_b, col_b, rank, f_rows, peer_recv):
        """Forward lambda stage storing straight into every rank's receive
        buffer (peer_recv[d]: rank d's buffer mapped in this process)."""
        rb, cb = self._bounds(P, row_b, col_b)
        self._follow_torch(f_rows)
        tab = (ctypes.c_void_p * P)(*[_ptr(b) for b in peer_recv])
        _lib.check(self.lib.sk_stage_lambda_fwd_peer(self._h, P, rb, cb, rank, _ptr(f_rows), tab))

    def stage_theta_peer(self, P, row_b, col_b, rank, recv, peer_back):
        """Theta stage storing the solved rows straight into every rank's
        return buffer."""
        rb, cb = self._bounds(P, row_b, col_b)
        self._follow_torch(recv)
        tab = (ctypes.c_void_p * P)(*[_ptr(b) for b in peer_back])
        _lib.check(self.lib.sk_stage_theta_peer(self._h, P, rb, cb, rank, _ptr(recv), tab))

    def event_record(self, event: int) -> None:
        """Record an (interprocess) event on the plan's stream (sk_event_record)."""
        _lib.check(self.lib.sk_event_record(self._h, ctypes.c_void_p(event)))

    def stream_wait(self, event: int) -> None:
        """Make the plan's stream wait for an event (sk_stream_wait_event)."""
        _lib.check(self.lib.sk_stream_wait_event(self._h, ctypes.c_void_p(event)))

    def stage_stats(self):
        """(mean re, mean im, max|F|) of the last theta stage entry point,
        waiting for that stage only (sk_stage_stats)."""
        out = (ctypes.c_double * 3)()
        _lib.check(self.lib.sk_stage_stats(self._h, out))
        return out[0], out[1], out[2]

    def stage_lambda_inv(self, P, row_b, col_b, rank, back, u_rows):
        rb, cb = self._bounds(P, row_b, col_b)
        self._follow_torch(back)
        _lib.check(self.lib.sk_stage_lambda_inv(self._h, P, rb, cb, rank, _ptr(back), _ptr(u_rows)))

    # -- assemble / standalone transforms
    def assemble(self, d, col, row, vscale: float = 0.0, F=None):
        """assemble_poisson on raw low-rank factors (sk_assemble): d (K,),
        col (K, mf), row (K, nf) complex -> (F (M, N) complex, report[3])."""
        dev = _is_device(d)
        if dev:
            import torch
            K, mf, nf = int(d.shape[0]), int(col.shape[-1]), int(row.shape[-1])
            if F is None:
                F = torch.empty((self.M, self.N), dtype=torch.complex128, device=d.device)
        else:
            d, col, row = (np.ascontiguousarray(x, dtype=np.complex128) for x in (d, col, row))
            K = d.shape[0]
            col = col[None] if col.ndim == 1 else col  # a single term may come as a vector
            row = row[None] if row.ndim == 1 else row
            mf, nf = col.shape[1], row.shape[1]
            if F is None:
                F = np.empty((self.M, self.N), np.complex128)
        if col.shape[0] != K or row.shape[0] != K:
            raise size_error("assemble_poisson: factor counts differ")
        rep = (ctypes.c_double * 3)()
        self._follow_torch(d)
        _lib.check(self.lib.sk_assemble(self._h, K, mf, nf, _ptr(d), _ptr(col), _ptr(row), float(vscale), _ptr(F),
                                        rep, _lib.SK_DEVICE if dev else _lib.SK_HOST))
        return F, [rep[0], rep[1], rep[2]]

    def analyze_2d(self, grid, X=None):
        """analyze_2d of an m x n complex doubled grid (sk_analyze_2d)."""
        dev = _is_device(grid)
        m, n = (int(x) for x in grid.shape[-2:])
        if dev:
            import torch
            X = torch.empty((m, n), dtype=torch.complex128, device=grid.device) if X is None else X
        else:
            grid = np.ascontiguousarray(grid, dtype=np.complex128)
            X = np.empty((m, n), np.complex128) if X is None else X
        self._follow_torch(grid)
        _lib.check(self.lib.sk_analyze_2d(self._h, m, n, _ptr(grid), _ptr(X), _lib.SK_DEVICE if dev else _lib.SK_HOST))
        return X

    def sample_grid(self, X, m_out: int, n_out: int, grid=None):
        """sample_grid of rows x cols coefficients on an m_out x n_out grid."""
        dev = _is_device(X)
        rows, cols = (int(x) for x in X.shape[-2:])
        if dev:
            import torch
            grid = torch.empty((m_out, n_out), dtype=torch.complex128, device=X.device) if grid is None else grid
        else:
            X = np.ascontiguousarray(X, dtype=np.complex128)
            grid = np.empty((m_out, n_out), np.complex128) if grid is None else grid
        self._follow_torch(X)
        _lib.check(self.lib.sk_sample_grid(self._h, rows, cols, _ptr(X), int(m_out), int(n_out), _ptr(grid),
                                           _lib.SK_DEVICE if dev else _lib.SK_HOST))
        return grid

    def sample_dfs(self, phys, m: Optional[int] = None, grid=None):
        """DFS doubling of physical samples ((m/2+1) x n real) -> m x n complex."""
        dev = _is_device(phys)
        rows, n = (int(x) for x in phys.shape[-2:])
        m = 2 * (rows - 1) if m is None else int(m)
        if rows != m // 2 + 1:
            raise size_error("sample_dfs: expected m/2 + 1 physical rows")
        if dev:
            import torch
            grid = torch.empty((m, n), dtype=torch.complex128, device=phys.device) if grid is None else grid
        else:
            phys = np.ascontiguousarray(phys, dtype=np.float64)
            grid = np.empty((m, n), np.complex128) if grid is None else grid
        self._follow_torch(phys)
        _lib.check(self.lib.sk_sample_dfs(self._h, m, n, _ptr(phys), _ptr(grid), _lib.SK_DEVICE if dev else _lib.SK_HOST))
        return grid

    # -- structure-preserving GE on a doubled grid (lowrank.hpp:73-93)
    def pivot_search(self, grid, alpha: float = 0.01, half: bool = False):
        """pivot_search (lowrank.cpp:84-112) of an m x n complex doubled grid:
        a PivotBlock, or None where the grid vanishes on the pivot set.
        half: grid is the (m/2+1) x n upper half, row i <-> theta_i = 2 pi i/m,
        as construct's phase 1 keeps it (lowrank.cpp:246-252)."""
        dev = _is_device(grid)
        m, n = (int(x) for x in grid.shape[-2:])
        m = 2 * (m - 1) if half else m
        if not dev:
            grid = np.ascontiguousarray(grid, dtype=np.complex128)
        self._follow_torch(grid)
        oi = (ctypes.c_int * 3)()
        od = (ctypes.c_double * 10)()
        _lib.check(self.lib.sk_ge_pivot_search(self._h, m, n, _ptr(grid), float(alpha), oi, od,
                                               (_lib.SK_DEVICE if dev else _lib.SK_HOST) | (_lib.SK_GE_HALF if half else 0)))
        return PivotBlock._from(oi, od) if oi[0] else None

    def ge_step(self, grid, p: "PivotBlock", out=None, half: bool = False):
        """ge_step (lowrank.cpp:127-162): grid minus the rank-<=2 update of
        pivot p, bit-identical to the reference (half: as in pivot_search;
        the phase-1 update lowrank.cpp:362-392)."""
        dev = _is_device(grid)
        rows, n = (int(x) for x in grid.shape[-2:])
        m = 2 * (rows - 1) if half else rows
        if dev:
            import torch
            out = torch.empty_like(grid) if out is None else out
        else:
            grid = np.ascontiguousarray(grid, dtype=np.complex128)
            out = np.empty((rows, n), np.complex128) if out is None else out
        self._follow_torch(grid)
        pd = (ctypes.c_double * 10)(*p._doubles())
        _lib.check(self.lib.sk_ge_step(self._h, m, n, _ptr(grid), pd, _ptr(out),
                                       (_lib.SK_DEVICE if dev else _lib.SK_HOST) | (_lib.SK_GE_HALF if half else 0)))
        return out

    def ge_run(self, grid, tau: float, alpha: float = 0.01, max_steps: int = 1024, half: bool = False):
        """The elimination loop with the grid resident on the device (in place
        for device tensors; host arrays are copied in and back): returns
        (pivots, resid) with resid[0] = max|grid| before the first step and
        resid[s + 1] after step s."""
        dev = _is_device(grid)
        m, n = (int(x) for x in grid.shape[-2:])
        m = 2 * (m - 1) if half else m
        if not dev and not (isinstance(grid, np.ndarray) and grid.dtype == np.complex128 and grid.flags.c_contiguous):
            raise size_error("ge_run: a C-contiguous complex128 array is updated in place")
        self._follow_torch(grid)
        ns = ctypes.c_int(0)
        pi = (ctypes.c_int * (2 * max_steps))()
        pd = (ctypes.c_double * (10 * max_steps))()
        rs = (ctypes.c_double * (max_steps + 1))()
        _lib.check(self.lib.sk_ge_run(self._h, m, n, _ptr(grid), float(alpha), float(tau), int(max_steps), ctypes.byref(ns),
                                      pi, pd, rs, (_lib.SK_DEVICE if dev else _lib.SK_HOST) | (_lib.SK_GE_HALF if half else 0)))
        k = ns.value
        piv = [PivotBlock._from((1, pi[2 * i], pi[2 * i + 1]), pd[10 * i: 10 * i + 10]) for i in range(k)]
        return piv, [rs[i] for i in range(k + 1)]

    def _check_shape(self, a, tail):
        shp = tuple(a.shape)
        if shp[-2:] != tuple(tail):
            raise size_error(f"expected trailing shape {tail}, got {shp}")
        lead = int(np.prod(shp[:-2])) if len(shp) > 2 else 1
        if lead != self.nrhs:
            raise size_error(f"expected {self.nrhs} right-hand side(s), got {lead}")


# ------------------------------------------------------------ reference API
@dataclasses.dataclass
class PoissonProblem:
    m: int
    n: int
    f: np.ndarray  # m x n complex128: 2D Fourier coefficients of sin(theta)^2 f~


@dataclasses.dataclass
class PoissonSolution:
    x: np.ndarray  # m x n complex128: 2D Fourier coefficients of u~


@dataclasses.dataclass
class ResidualReport:
    interior_max: float = 0.0
    replaced_row_abs: float = 0.0
    constraint_abs: float = 0.0


@dataclasses.dataclass
class BenchRow:
    size: int
    reps: int
    seconds: float


_plans: dict = {}


def _plan(m: int, n: int, nrhs: int = 1) -> Plan:
    key = (m, n, nrhs)
    p = _plans.get(key)
    if p is None:
        p = Plan(m, n, nrhs)
        _plans[key] = p
    return p


def _check_sizes(m, n):
    if m <= 0 or n <= 0 or m % 2 or n % 2:
        raise size_error("poisson solve: sizes must be positive and even")


def solve(pb: PoissonProblem) -> PoissonSolution:
    """spherekit::solve (poisson.cpp:121-161) on the GPU: bit-identical X for
    every k != 0 column; k = 0 to rounding."""
    _check_sizes(pb.m, pb.n)
    F = np.ascontiguousarray(pb.f, dtype=np.complex128)
    if F.shape != (pb.m, pb.n):
        raise size_error("poisson solve: f must be m x n")
    return PoissonSolution(_plan(pb.m, pb.n).solve_coeffs(F))


def residual(pb: PoissonProblem, sol: PoissonSolution) -> ResidualReport:
    """spherekit::residual (poisson.cpp:163-186)."""
    _check_sizes(pb.m, pb.n)
    return _plan(pb.m, pb.n).residual(pb.f, sol.x)


def solve_grid(f_phys: np.ndarray, m: Optional[int] = None, coeffs: bool = False):
    """Physical samples f ((m/2+1) x n, theta_p = 2 pi p/m, lambda_q = -pi +
    2 pi q/n) -> physical solution u of Lap u = f, integral(u) = 0."""
    rows, n = f_phys.shape[-2:]
    m = 2 * (rows - 1) if m is None else m
    _check_sizes(m, n)
    return _plan(m, n).solve_grid(f_phys, coeffs=coeffs)


def solve_grid_exact(f_phys: np.ndarray, m: Optional[int] = None, coeffs: bool = False):
    """The reference's grid composition (sample_dfs -> analyze_2d -> Msin^2 ->
    solve -> sample_grid) on the GPU: the complex m x n doubled grid u, every
    lambda mode solved, for any input (see Plan.solve_grid_exact)."""
    rows, n = f_phys.shape[-2:]
    m = 2 * (rows - 1) if m is None else m
    _check_sizes(m, n)
    return _plan(m, n).solve_grid_exact(f_phys, coeffs=coeffs)


def coefficients_from_half(X_half, m: int, n: int) -> np.ndarray:
    """The full m x n coefficient matrix of the real grid solve from its
    k >= 0 half X_half[k][i] (sk_solve_grid): the k < 0 columns are the
    Hermitian mirror X(t, -k) = conj X(-t, k) (the unpaired t = -m/2 row maps
    to itself), k = -n/2 is the Nyquist column X_half[n/2]."""
    Xh = np.asarray(X_half)
    L = m // 2
    t = np.arange(m) - L
    tt = np.where(t == -L, -L, -t) + L
    X = np.empty((m, n), np.complex128)
    X[:, n // 2:] = Xh[: n // 2].T
    X[:, 0] = Xh[n // 2]
    for kc in range(1, n // 2):
        X[:, kc] = np.conj(Xh[n // 2 - kc][tt])
    return X


def rhs_coefficients(f_phys, m: Optional[int] = None) -> np.ndarray:
    """F = Msin^2 analyze_2d(sample_dfs(f)) of physical samples: the
    PoissonProblem the grid solve answers; the transforms run on
    the device, the Msin^2 column apply in the reference's accumulation order
    (banded.cpp:8-19)."""
    rows, n = f_phys.shape[-2:]
    m = 2 * (rows - 1) if m is None else m
    A = analyze_2d(sample_dfs(np.ascontiguousarray(f_phys, np.float64), m))
    d = np.full((m, 1), 0.5)
    d[0] = d[-1] = 0.25
    F = d * A
    F[2:] = -0.25 * A[:-2] + F[2:]   # acc = (-1/4) x_{i-2}, then + diag x_i
    F[:-2] = F[:-2] + (-0.25) * A[2:]  # then + (-1/4) x_{i+2}
    return F


def integration_weights(m: int) -> np.ndarray:
    """poisson.cpp:42-50: w_k = 2/(1-k^2) for even k, 0 for odd k."""
    k = np.arange(m) - m // 2
    w = np.zeros(m, np.complex128)
    even = (k % 2) == 0
    w[even] = 2.0 / (1.0 - k[even].astype(np.float64) ** 2)
    return w


def bench_poisson(sizes, reps: Optional[int] = None):
    """poisson.cpp:188-230: best-of-reps time of one coefficient-space solve
    per size on the synthetic band-limited workload (same RNG stream)."""
    from .inputs import bench_problem
    rows = []
    for i, s in enumerate(sizes):
        if s < 16 or s % 2:
            raise size_error("bench_poisson: sizes must be even and >= 16")
        F = bench_problem(list(sizes[: i + 1]))
        plan = _plan(s, s)
        r = reps if reps is not None else max(3, int(4e7 / (float(s) * s)))
        best = float("inf")
        for _ in range(r):
            t0 = time.perf_counter()
            plan.solve_coeffs(F)
            best = min(best, time.perf_counter() - t0)
        rows.append(BenchRow(s, r, best))
    return rows


@dataclasses.dataclass
class PivotBlock:
    """One 2x2 GE pivot (lowrank.hpp:19-26): (lambda_star, theta_star) pairs
    with (lambda_star - pi, -theta_star); a, b the grid values at the pair,
    (m_even, m_odd) the spectral form of the eps-pseudoinverse of [a b; b a].
    t, k: the node indices (theta_star = 2 pi t/m, lambda_star = lambda_k)."""
    lambda_star: float
    theta_star: float
    a: complex
    b: complex
    m_even: complex
    m_odd: complex
    t: int = -1
    k: int = -1

    @classmethod
    def _from(cls, oi, od):
        c = [complex(od[2 * i], od[2 * i + 1]) for i in range(4)]
        return cls(float(od[9]), float(od[8]), c[0], c[1], c[2], c[3], int(oi[1]), int(oi[2]))

    def _doubles(self):
        v = []
        for z in (self.a, self.b, self.m_even, self.m_odd):
            v += [z.real, z.imag]
        return v + [self.theta_star, self.lambda_star]


# ------------------------------------------------- assemble / Fourier layer
@dataclasses.dataclass
class LowRankSphereFun:
    """The factors of a low-rank sphere function (lowrank.hpp:47-59):
    f~(lambda, theta) = sum_j d[j] a_j(theta) b_j(lambda), with col_coeffs[j]
    the theta coefficients of a_j (mode t at t + mf/2) and row_coeffs[j] the
    lambda coefficients of b_j.  (The constructor from an expression or a
    callable is outside this hot path; factors come from the caller.)"""
    d: np.ndarray
    col_coeffs: np.ndarray  # (K, mf) complex
    row_coeffs: np.ndarray  # (K, nf) complex
    vscale: float = 0.0

    def rank(self) -> int:
        return int(np.asarray(self.d).shape[0])


@dataclasses.dataclass
class AssembleReport:
    mean_removed: bool = False
    removed_mean: complex = 0j


def assemble_poisson(f: LowRankSphereFun, m: int, n: int, report: Optional[AssembleReport] = None) -> PoissonProblem:
    """spherekit::assemble_poisson (poisson.cpp:52-86) on the GPU: F =
    sum_j d_j (Msin^2 a_j) b_j^T with the reference's mean removal;
    bit-identical to the reference."""
    if m % 2 or n % 2 or m <= 0 or n <= 0:
        raise size_error("assemble_poisson: sizes must be positive and even")
    F, rep = _plan(m, n).assemble(f.d, f.col_coeffs, f.row_coeffs, f.vscale)
    if report is not None:
        report.mean_removed = bool(rep[0])
        report.removed_mean = complex(rep[1], rep[2])
    return PoissonProblem(m, n, F)


def _xplan() -> Plan:
    return _plan(8, 4)  # any plan: the standalone transforms take their own sizes


def analyze_2d(grid) -> np.ndarray:
    """spherekit::analyze_2d (fourier.cpp:170-188): m x n doubled sample grid
    -> m x n coefficient matrix (row i = theta mode i - m/2)."""
    return _xplan().analyze_2d(grid)


def sample_grid(X, m: int, n: int) -> np.ndarray:
    """spherekit::sample_grid (fourier.cpp:190-209): coefficients -> m x n
    grid values, zero-padding or truncating the modes."""
    return _xplan().sample_grid(X, m, n)


def pivot_search(grid, alpha: float = 0.01):
    """spherekit::pivot_search (lowrank.hpp:89)."""
    return _xplan().pivot_search(grid, alpha)


def ge_step(grid, p: PivotBlock) -> np.ndarray:
    """spherekit::ge_step (lowrank.hpp:93)."""
    return _xplan().ge_step(grid, p)


def sample_dfs(phys, m: Optional[int] = None) -> np.ndarray:
    """spherekit::sample_dfs (sphere_domain.cpp:46-52) applied to physical
    samples: the DFS-doubled m x n grid."""
    return _xplan().sample_dfs(phys, m)
