"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes front-end for
  * ``oracle/libsk_oracle.so``        — the C++ restatement of the reference hot
    path (oracle/sk_oracle.cpp), and
  * ``oracle/_ref/libspherekit_ref.so`` — the UNMODIFIED reference sources
    (/root/reference/proj/src) built by ``make -C oracle ref`` with the FFTW-API
    shim; only present where it was built (it travels to the GPU box with the
    repo snapshot but /root/reference does not).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU reference — never as part of the product path.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libsk_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspherekit_ref.so")
REF_SRC = "/root/reference/proj/src"

_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build(ref: bool = True) -> None:
    """Compile the restatement (and, when the reference tree is present, the
    reference library).  Building the checker is not using it."""
    subprocess.run(["make", "-s", "-C", HERE, "libsk_oracle.so"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


class _Lib:
    prefix = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = ctypes.CDLL(path)
        getattr(self.lib, self.prefix + "last_error").restype = ctypes.c_char_p

    def _call(self, name, *args):
        rc = getattr(self.lib, self.prefix + name)(*args)
        if rc != 0:
            raise OracleError(rc, getattr(self.lib, self.prefix + "last_error")().decode())

    # ---- coefficient space
    def solve(self, F, threads=1):
        m, n = F.shape
        F = np.ascontiguousarray(F, np.complex128)
        X = np.zeros_like(F)
        self._call("solve", _I(m), _I(n), _ptr(F), _ptr(X), _I(threads))
        return X

    def residual(self, F, X):
        m, n = F.shape
        out = np.zeros(3)
        self._call("residual", _I(m), _I(n), _ptr(np.ascontiguousarray(F, np.complex128)),
                   _ptr(np.ascontiguousarray(X, np.complex128)), _ptr(out))
        return out

    def msin2_columns(self, X):
        m, n = X.shape
        X = np.ascontiguousarray(X, np.complex128)
        F = np.zeros_like(X)
        self._call("msin2_columns", _I(m), _I(n), _ptr(X), _ptr(F))
        return F

    def band_solve(self, band, b, kl, ku):
        n = b.shape[0]
        x = np.zeros(n, np.complex128)
        self._call("band_solve", _I(n), _I(kl), _I(ku), _ptr(np.ascontiguousarray(band, np.complex128)),
                   _ptr(np.ascontiguousarray(b, np.complex128)), _ptr(x))
        return x

    def band_solve_dense_row(self, band, kl, ku, skip, w, wrhs, b):
        n = b.shape[0]
        x = np.zeros(n, np.complex128)
        self._call("band_solve_dense_row", _I(n), _I(kl), _I(ku), _ptr(np.ascontiguousarray(band, np.complex128)),
                   _I(skip), _ptr(np.ascontiguousarray(w, np.complex128)), _D(wrhs.real), _D(wrhs.imag),
                   _ptr(np.ascontiguousarray(b, np.complex128)), _ptr(x))
        return x

    def div_sin(self, c):
        c = np.ascontiguousarray(c, np.complex128)
        out = np.zeros_like(c)
        self._call("div_sin", _I(c.shape[0]), _ptr(c), _ptr(out))
        return out

    # ---- transforms
    def analyze_1d(self, s):
        s = np.ascontiguousarray(s, np.complex128)
        c = np.zeros_like(s)
        self._call("analyze_1d", _I(s.shape[0]), _ptr(s), _ptr(c))
        return c

    def synthesize_1d(self, c, n_out):
        c = np.ascontiguousarray(c, np.complex128)
        g = np.zeros(n_out, np.complex128)
        self._call("synthesize_1d", _I(c.shape[0]), _ptr(c), _I(n_out), _ptr(g))
        return g

    def analyze_2d(self, grid):
        m, n = grid.shape
        grid = np.ascontiguousarray(grid, np.complex128)
        X = np.zeros_like(grid)
        self._call("analyze_2d", _I(m), _I(n), _ptr(grid), _ptr(X))
        return X

    # ---- structure-preserving GE on a doubled grid (lowrank.hpp:73-93)
    def pivot_search(self, grid, alpha=0.01):
        """(t, k, a, b, m_even, m_odd, theta_star, lambda_star) or None."""
        m, n = grid.shape
        oi = (ctypes.c_int * 3)()
        od = np.zeros(10)
        self._call("pivot_search", _I(m), _I(n), _ptr(np.ascontiguousarray(grid, np.complex128)),
                   ctypes.c_double(alpha), oi, _ptr(od))
        if not oi[0]:
            return None
        c = od[:8].view(np.complex128)
        return (int(oi[1]), int(oi[2]), complex(c[0]), complex(c[1]), complex(c[2]), complex(c[3]), float(od[8]),
                float(od[9]))

    def ge_step(self, grid, piv):
        """piv as returned by pivot_search."""
        m, n = grid.shape
        t, k, a, b, me, mo, th, lam = piv
        pd = np.array([a.real, a.imag, b.real, b.imag, me.real, me.imag, mo.real, mo.imag, th, lam])
        out = np.zeros((m, n), np.complex128)
        self._call("ge_step", _I(m), _I(n), _ptr(np.ascontiguousarray(grid, np.complex128)), _ptr(pd), _ptr(out))
        return out

    def sample_grid(self, X, m_out, n_out):
        r, c = X.shape
        g = np.zeros((m_out, n_out), np.complex128)
        self._call("sample_grid", _I(r), _I(c), _ptr(np.ascontiguousarray(X, np.complex128)), _I(m_out), _I(n_out),
                   _ptr(g))
        return g

    # ---- generators
    def bench_problem(self, sizes):
        sizes = list(sizes)
        s = sizes[-1]
        arr = (ctypes.c_int * len(sizes))(*sizes)
        F = np.zeros((s, s), np.complex128)
        self._call("bench_problem", _I(len(sizes)), arr, _ptr(F))
        return F

    def random_mean_zero_problem(self, m, n, seed):
        F = np.zeros((m, n), np.complex128)
        self._call("random_mean_zero_problem", _I(m), _I(n), ctypes.c_uint(seed), _ptr(F))
        return F


class Oracle(_Lib):
    """The C++ restatement (always available once built)."""
    prefix = "sko_"

    def __init__(self, path=ORACLE_SO):
        super().__init__(path)

    def ge_half_step(self, e, alpha=0.01):
        """One phase-1 step (lowrank.cpp:345-392) on the (g/2+1) x g upper half
        grid: ((bi, bk, a, b, m_even, m_odd), updated e) or None."""
        h, g = e.shape
        assert h == g // 2 + 1
        oi = (ctypes.c_int * 3)()
        od = np.zeros(8)
        out = np.zeros((h, g), np.complex128)
        self._call("ge_half_step", _I(g), _ptr(np.ascontiguousarray(e, np.complex128)), ctypes.c_double(alpha), oi,
                   _ptr(od), _ptr(out))
        if not oi[0]:
            return None
        c = od.view(np.complex128)
        return (int(oi[1]), int(oi[2]), complex(c[0]), complex(c[1]), complex(c[2]), complex(c[3])), out

    def build_lap(self, m):
        lap = np.zeros((m, 5))
        self._call("build_lap", _I(m), _ptr(lap))
        return lap

    def integration_weights(self, m):
        w = np.zeros(m)
        self._call("integration_weights", _I(m), _ptr(w))
        return w

    def assemble(self, d, col, row, vscale, m, n):
        """assemble_poisson on raw low-rank factors -> (F, [removed?, mu.re, mu.im])."""
        d, col, row = (np.ascontiguousarray(x, np.complex128) for x in (d, col, row))
        K, mf, nf = d.shape[0], col.shape[1], row.shape[1]
        F = np.zeros((m, n), np.complex128)
        rep = np.zeros(3)
        self._call("assemble", _I(K), _I(mf), _I(nf), _ptr(d), _ptr(col), _ptr(row), ctypes.c_double(vscale), _I(m),
                   _I(n), _ptr(F), _ptr(rep))
        return F, rep

    def dfs_double(self, phys, m):
        n = phys.shape[1]
        g = np.zeros((m, n), np.complex128)
        self._call("dfs_double", _I(m), _I(n), _ptr(np.ascontiguousarray(phys, np.float64)), _ptr(g))
        return g

    def grid_pipeline(self, phys, m, threads=1):
        """Returns (X, u_doubled, u_phys, mean)."""
        n = phys.shape[1]
        X = np.zeros((m, n), np.complex128)
        U = np.zeros((m, n), np.complex128)
        up = np.zeros((m // 2 + 1, n))
        mean = np.zeros(2)
        self._call("grid_pipeline", _I(m), _I(n), _ptr(np.ascontiguousarray(phys, np.float64)), _ptr(X), _ptr(U),
                   _ptr(up), _I(threads), _ptr(mean))
        return X, U, up, complex(mean[0], mean[1])

    def grid_pipeline_real(self, phys, m, threads=1):
        """The composition for real data with the k < 0 half taken as the
        Hermitian mirror of k > 0 (X(t,-k) = conj X(-t,k); the unpaired
        t = -M/2 row maps to itself) before synthesis — the real-output
        variant the GPU grid path implements.  Identical to grid_pipeline for
        band-limited data; for rough data the reference's own output is
        complex (its truncated operators are not mirror-symmetric)."""
        n = phys.shape[1]
        X, _, _, _ = self.grid_pipeline(phys, m, threads)
        L = m // 2
        t = np.arange(m) - L
        tt = np.where(t == -L, -L, -t) + L
        Xm = X.copy()
        for kc in range(1, n // 2):
            k = kc - n // 2
            Xm[:, kc] = np.conj(X[tt, n // 2 - k])
        U = self.sample_grid(Xm, m, n)
        return phys_from_doubled(U, m).real

    def shgen(self, m, n, L, coeffs, threads=8):
        phys = np.zeros((m // 2 + 1, n))
        self._call("shgen", _I(m), _I(n), _I(L), _ptr(np.ascontiguousarray(coeffs, np.float64)), _ptr(phys),
                   _I(threads))
        return phys


class Reference(_Lib):
    """The reference library itself (oracle/_ref), where it was built."""
    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)

    def build_lap(self, m):
        lap = np.zeros((m, 5), np.complex128)
        self._call("build_lap", _I(m), _ptr(lap))
        return lap

    def integration_weights(self, m):
        w = np.zeros(m, np.complex128)
        self._call("integration_weights", _I(m), _ptr(w))
        return w

    def sample_dfs_phys(self, phys, m):
        n = phys.shape[1]
        g = np.zeros((m, n), np.complex128)
        self._call("sample_dfs_phys", _I(m), _I(n), _ptr(np.ascontiguousarray(phys, np.float64)), _ptr(g))
        return g

    def grid_pipeline(self, phys, m, threads=1):
        """Returns (X, u_doubled)."""
        n = phys.shape[1]
        X = np.zeros((m, n), np.complex128)
        U = np.zeros((m, n), np.complex128)
        self._call("grid_pipeline", _I(m), _I(n), _ptr(np.ascontiguousarray(phys, np.float64)), _ptr(X), _ptr(U),
                   _I(threads))
        return X, U

    def grid_pipeline_timed(self, phys, m, threads=1):
        """grid_pipeline with its phases timed: (X, U, t[sample_dfs, analyze_2d,
        Msin^2, solve, sample_grid] seconds)."""
        n = phys.shape[1]
        X = np.zeros((m, n), np.complex128)
        U = np.zeros((m, n), np.complex128)
        t = np.zeros(5)
        self._call("grid_pipeline_timed", _I(m), _I(n), _ptr(np.ascontiguousarray(phys, np.float64)), _ptr(X),
                   _ptr(U), _I(threads), _ptr(t))
        return X, U, t

    def assemble_fn(self, fn_id, params, m, n):
        par = np.ascontiguousarray(params, np.float64) if params is not None and len(params) else None
        F = np.zeros((m, n), np.complex128)
        mean = np.zeros(3)
        self._call("assemble_fn", _I(fn_id), _ptr(par), _I(0 if par is None else len(par)), _I(m), _I(n), _ptr(F),
                   _ptr(mean))
        return F, mean

    def construct_fn(self, fn_id, params):
        """construct(f) of a test function -> (d[K], col[K, mf], row[K, nf], vscale)."""
        par = np.ascontiguousarray(params, np.float64) if params is not None and len(params) else None
        npar = _I(0 if par is None else len(par))
        K, mf, nf = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        vs = ctypes.c_double()
        self._call("construct_fn", _I(fn_id), _ptr(par), npar, ctypes.byref(K), ctypes.byref(mf), ctypes.byref(nf),
                   None, None, None, ctypes.byref(vs))
        d = np.zeros(K.value, np.complex128)
        col = np.zeros((K.value, mf.value), np.complex128)
        row = np.zeros((K.value, nf.value), np.complex128)
        self._call("construct_fn", _I(fn_id), _ptr(par), npar, ctypes.byref(K), ctypes.byref(mf), ctypes.byref(nf),
                   _ptr(d), _ptr(col), _ptr(row), ctypes.byref(vs))
        return d, col, row, vs.value

    def assemble_lowrank(self, d, col, row, vscale, m, n):
        d, col, row = (np.ascontiguousarray(x, np.complex128) for x in (d, col, row))
        K, mf, nf = d.shape[0], col.shape[1], row.shape[1]
        F = np.zeros((m, n), np.complex128)
        mean = np.zeros(3)
        self._call("assemble_lowrank", _I(K), _I(mf), _I(nf), _ptr(d), _ptr(col), _ptr(row), ctypes.c_double(vscale),
                   _I(m), _I(n), _ptr(F), _ptr(mean))
        return F, mean

    def sample_dfs_fn(self, fn_id, params, m, n):
        par = np.ascontiguousarray(params, np.float64) if params is not None and len(params) else None
        g = np.zeros((m, n), np.complex128)
        self._call("sample_dfs_fn", _I(fn_id), _ptr(par), _I(0 if par is None else len(par)), _I(m), _I(n), _ptr(g))
        return g

    def bench_poisson(self, sizes, threads):
        k = len(sizes)
        s = (ctypes.c_int * k)(*sizes)
        secs = (ctypes.c_double * k)()
        reps = (ctypes.c_int * k)()
        self._call("bench_poisson", _I(k), s, _I(threads), secs, reps)
        return list(secs), list(reps)

    def time_stock_sample(self, m, n, kc0, ncols, j0, nrows, threads):
        """The reference's stock grid composition on a block of ncols columns
        and nrows rows of full-size matrices (ref_time_stock_sample): per-unit
        seconds t[0..4], the sample's wall time t[5], sample_dfs per row t[6]."""
        t = np.zeros(7)
        self._call("time_stock_sample", _I(m), _I(n), _I(kc0), _I(ncols), _I(j0), _I(nrows), _I(threads), _ptr(t))
        return t

    def time_sample(self, m, n, ncols, nrows, threads):
        t = np.zeros(5)
        self._call("time_sample", _I(m), _I(n), _I(ncols), _I(nrows), _I(threads), _ptr(t))
        return t


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def phys_from_doubled(U, m):
    """Physical rows p = 0..M/2 of a doubled grid (p = M/2 from row 0)."""
    rows = [U[m // 2 + p] if p < m // 2 else U[0] for p in range(m // 2 + 1)]
    return np.stack(rows)
