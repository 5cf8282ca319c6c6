"""Command-line front end: the reference CLI's Poisson routes on the device.

    python -m paper_1510_08094_b200 poisson  --in f.sgrid --out u.sgrid [--exact] [--coeffs x.sgrid]
    python -m paper_1510_08094_b200 solve    --in F.sgrid --out X.sgrid
    python -m paper_1510_08094_b200 residual --rhs F.sgrid --sol X.sgrid
    python -m paper_1510_08094_b200 bench    [--sizes 256,512,1024,2048] [--grid]

Mirrors `spherekit poisson` / `residual` / `bench` (tools/spherekit_main.cpp
:289-306, :338-351, :353-368): the same summary lines, the same bench table
(size, reps, sec/solve, ratio, Mdof/s) and the same exit-code contract
(2 argument errors, 3 precondition / size / structure errors, 4 I/O errors,
1 anything else; spherekit_main.cpp:375-406).  The reference reads and writes
low-rank functions as JSON `.sfun` (sfun_io.cpp:51-118), which at 1e8 DOF is
impractical (solution_to_fun writes N terms x M coefficients as text,
spherekit_main.cpp:58-81) and whose construction from an expression is
outside this hot path; here grids and coefficient matrices travel in a binary
container (`.sgrid`, below) or as `.npy`.

`.sgrid` layout (little endian): magic b"SKG1", uint32 kind, int32 M, int32 N,
int32 nrhs, then the float64 payload
  kind 0: physical samples, nrhs x (M/2+1) x N real (row p: theta = 2 pi p / M);
  kind 1: coefficients, nrhs x M x N complex (reference Matrix layout);
  kind 2: doubled grid, nrhs x M x N complex (BMCGrid layout).
"""
from __future__ import annotations

import argparse
import struct
import sys
import time

import numpy as np

MAGIC = b"SKG1"
KIND_PHYS, KIND_COEFFS, KIND_DOUBLED = 0, 1, 2


class CliError(Exception):
    """Argument error (exit code 2, the reference's parse_error)."""


class IoError(Exception):
    """File error (exit code 4, the reference's io_error)."""


def save_sgrid(path: str, a: np.ndarray, kind: int, M: int, N: int) -> None:
    a = np.ascontiguousarray(a)
    nrhs = a.shape[0] if a.ndim == 3 else 1
    dtype = np.float64 if kind == KIND_PHYS else np.complex128
    try:
        with open(path, "wb") as fh:
            fh.write(MAGIC + struct.pack("<Iiii", kind, M, N, nrhs))
            fh.write(a.astype(dtype, copy=False).tobytes())
    except OSError as exc:
        raise IoError(f"cannot write {path}: {exc}") from exc


def load_sgrid(path: str):
    """-> (array, kind, M, N); `.npy` files hold a (M/2+1) x N real grid
    (kind 0) or an M x N complex matrix (kind 1)."""
    try:
        if path.endswith(".npy"):
            a = np.load(path)
            if np.iscomplexobj(a):
                return a, KIND_COEFFS, a.shape[-2], a.shape[-1]
            return a.astype(np.float64), KIND_PHYS, 2 * (a.shape[-2] - 1), a.shape[-1]
        with open(path, "rb") as fh:
            head = fh.read(20)
            if len(head) != 20 or head[:4] != MAGIC:
                raise IoError(f"{path}: not an .sgrid file")
            kind, M, N, nrhs = struct.unpack("<Iiii", head[4:])
            data = fh.read()
    except OSError as exc:
        raise IoError(f"cannot read {path}: {exc}") from exc
    if kind == KIND_PHYS:
        shape, dtype = (nrhs, M // 2 + 1, N), np.float64
    elif kind in (KIND_COEFFS, KIND_DOUBLED):
        shape, dtype = (nrhs, M, N), np.complex128
    else:
        raise IoError(f"{path}: unknown kind {kind}")
    need = int(np.prod(shape)) * np.dtype(dtype).itemsize
    if len(data) != need:
        raise IoError(f"{path}: payload has {len(data)} bytes, expected {need}")
    a = np.frombuffer(data, dtype=dtype).reshape(shape)
    return (a[0] if nrhs == 1 else a), kind, M, N


def _parser():
    ap = argparse.ArgumentParser(prog="python -m paper_1510_08094_b200",
                                 description="DFS spectral Poisson solver on the unit sphere (B200)")
    sub = ap.add_subparsers(dest="cmd")
    p = sub.add_parser("poisson", help="grid-level solve: physical samples -> solution")
    p.add_argument("--in", dest="inp")
    p.add_argument("--expr", default=None)
    p.add_argument("--out", required=True)
    p.add_argument("--exact", action="store_true",
                   help="the reference's own composition (complex doubled grid, every lambda mode solved)")
    p.add_argument("--coeffs", default=None, help="also write the solution coefficients")
    s = sub.add_parser("solve", help="coefficient-space solve (spherekit::solve)")
    s.add_argument("--in", dest="inp", required=True)
    s.add_argument("--out", required=True)
    r = sub.add_parser("residual", help="residual report of a coefficient-space solution")
    r.add_argument("--rhs", required=True)
    r.add_argument("--sol", required=True)
    b = sub.add_parser("bench", help="bench_poisson on the device")
    b.add_argument("--sizes", default="256,512,1024,2048")
    b.add_argument("--grid", action="store_true", help="time the grid-level solve instead")
    return ap


class _ArgParser(argparse.ArgumentParser):
    def error(self, message):
        raise CliError(message)


def _parse(argv):
    ap = _parser()
    ap.__class__ = _ArgParser
    for act in ap._actions:
        if isinstance(act, argparse._SubParsersAction):
            for sp in act.choices.values():
                sp.__class__ = _ArgParser
    args = ap.parse_args(argv)
    if args.cmd is None:
        raise CliError("a subcommand is required (poisson, solve, residual, bench)")
    return args


def _sizes(text: str):
    try:
        sizes = [int(x) for x in text.split(",") if x.strip()]
    except ValueError as exc:
        raise CliError(f"bad --sizes {text!r}") from exc
    if not sizes:
        raise CliError("--sizes is empty")
    return sizes


def bench_table(rows, out=sys.stdout) -> None:
    """The reference's bench table (spherekit_main.cpp:355-366)."""
    out.write("%8s %6s %12s %8s %10s\n" % ("size", "reps", "sec/solve", "ratio", "Mdof/s"))
    prev = 0.0
    for r in rows:
        dofs = float(r.size) * r.size / 2.0
        ratio = ("%8.2f" % (r.seconds / prev)) if prev > 0 else "%8s" % "-"
        out.write("%8d %6d %12.5f %s %10.1f\n" % (r.size, r.reps, r.seconds, ratio, dofs / r.seconds / 1e6))
        prev = r.seconds


def _grid_bench(sizes):
    from . import poisson as pz
    from .inputs import sh_coeffs
    rows = []
    for s in sizes:
        if s % 2:
            raise pz.size_error("bench: sizes must be even")
        M, N = 2 * s, s
        plan = pz.Plan(M, N)
        try:
            import torch
            f = torch.empty((M // 2 + 1, N), dtype=torch.float64, device="cuda")
            L = max(1, min(N // 2 - 1, s // 4))
            plan.shgen(L, torch.from_numpy(sh_coeffs(1, L, 2.0)).cuda(), f)
            u = torch.empty_like(f)
            reps = max(3, int(4e7 / (float(s) * s)))
            best = float("inf")
            for _ in range(reps + 1):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                plan.solve_grid(f, u)
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
        finally:
            plan.close()
        rows.append(pz.BenchRow(s, reps, best))
    return rows


def run(argv) -> int:
    args = _parse(argv)
    from . import poisson as pz
    if args.cmd == "poisson":
        if args.expr is not None:
            raise CliError("poisson --expr: building a function from an expression (the reference's low-rank "
                           "constructor) is not part of this solver; pass sampled values with --in")
        if not args.inp:
            raise CliError("poisson: --in is required")
        f, kind, M, N = load_sgrid(args.inp)
        if kind != KIND_PHYS:
            raise CliError("poisson --in: expected physical samples (kind 0)")
        if args.exact:
            U, X = pz.solve_grid_exact(f, M, coeffs=True)
            save_sgrid(args.out, U, KIND_DOUBLED, M, N)
        else:
            u, Xh = pz.solve_grid(f, M, coeffs=True)
            save_sgrid(args.out, u, KIND_PHYS, M, N)
            X = pz.coefficients_from_half(Xh, M, N)
        F = pz.rhs_coefficients(f, M)
        rr = pz.residual(pz.PoissonProblem(M, N, F), pz.PoissonSolution(X))
        sys.stdout.write("poisson solve %dx%d: residual %.3g, constraint %.3g\n" % (M, N, rr.interior_max,
                                                                                  rr.constraint_abs))
        if args.coeffs:
            save_sgrid(args.coeffs, X, KIND_COEFFS, M, N)
        return 0
    if args.cmd == "solve":
        F, kind, M, N = load_sgrid(args.inp)
        if kind != KIND_COEFFS:
            raise CliError("solve --in: expected coefficients (kind 1)")
        X = pz.solve(pz.PoissonProblem(M, N, F)).x
        save_sgrid(args.out, X, KIND_COEFFS, M, N)
        return 0
    if args.cmd == "residual":
        F, k1, M, N = load_sgrid(args.rhs)
        X, k2, M2, N2 = load_sgrid(args.sol)
        if k1 != KIND_COEFFS or k2 != KIND_COEFFS or (M, N) != (M2, N2):
            raise CliError("residual: --rhs and --sol must be coefficient matrices of one size")
        rr = pz.residual(pz.PoissonProblem(M, N, F), pz.PoissonSolution(X))
        sys.stdout.write("interior residual:      %.6g\n" % rr.interior_max)
        sys.stdout.write("replaced-row residual:  %.6g\n" % rr.replaced_row_abs)
        sys.stdout.write("constraint |2pi w'X0|:  %.6g\n" % rr.constraint_abs)
        return 0
    if args.cmd == "bench":
        sizes = _sizes(args.sizes)
        rows = _grid_bench(sizes) if args.grid else pz.bench_poisson(sizes)
        bench_table(rows)
        return 0
    return 1


def main(argv=None) -> int:
    from ._lib import DeviceError, UnsupportedError, precondition_error, size_error, structure_error
    try:
        return run(sys.argv[1:] if argv is None else argv)
    except CliError as exc:
        sys.stderr.write(f"error: {exc}\n")
        return 2
    except IoError as exc:
        sys.stderr.write(f"error: {exc}\n")
        return 4
    except (precondition_error, size_error, structure_error, UnsupportedError) as exc:
        sys.stderr.write(f"error: {exc}\n")
        return 3
    except (DeviceError, Exception) as exc:  # noqa: BLE001
        sys.stderr.write(f"internal error: {exc}\n")
        return 1
