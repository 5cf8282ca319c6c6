"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference sources (/root/reference/proj/src, compiled by
``make -C oracle ref`` into oracle/_ref/libspherekit_ref.so with the FFTW-API
shim) on the known-answer cases of the reference's own tests and on seeded
workloads, and stores inputs and outputs as small .npz files.  The fixtures
are committed so the GPU box (where /root/reference does not exist) can check
against them.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, OracleError, Reference, build  # noqa: E402
from paper_1510_08094_b200.inputs import sh_coeffs  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print("wrote", path, {k: v.shape for k, v in arrays.items()})


def main(only=None):
    build(ref=True)
    R = Reference()
    O = Oracle()
    if only:
        {"lowrank": lowrank_fixtures, "transforms": transform_fixtures, "ge": ge_fixtures}[only](R)
        return

    # test_poisson.cpp:53-67 — l = 1 eigenfunction cos(theta), 64 x 64
    F, mean = R.assemble_fn(0, None, 64, 64)
    X = R.solve(F)
    save("kat_cos_theta_64", F=F, X=X, mean_report=mean, residual=R.residual(F, X))

    # test_poisson.cpp:186-206 — mean removal of 1 + cos(theta), 32 x 32, u = -cos(theta)/2
    F, mean = R.assemble_fn(1, None, 32, 32)
    X = R.solve(F)
    U = R.sample_grid(X, 32, 32)
    save("kat_mean_removal_32", F=F, X=X, mean_report=mean, U=U)

    # ... and the skewed problem that must raise precondition_error
    bad = np.zeros((16, 16), np.complex128)
    bad[8, 8] = 0.5
    bad[10, 8] = -0.25
    bad[6, 8] = -0.25
    try:
        R.solve(bad)
        raised = 0
    except OracleError as e:
        raised = e.code
    save("kat_precondition_16", F=bad, expected_code=np.array(raised))

    # test_poisson.cpp:77-103 / acceptance c07 — Y_l^m eigenfunctions (a few), 64 x 64
    for (l, m) in [(2, 1), (3, -2), (4, 0)]:
        F, _ = R.assemble_fn(2, np.array([l, m, 1.0]), 64, 64)
        X = R.solve(F)
        save(f"kat_ylm_{l}_{m}_64", F=F, X=X, lm=np.array([l, m]))

    # acceptance c10 — sin(50 xyz) at 150 x 150 (non-power-of-two, radix 3/5)
    F, _ = R.assemble_fn(3, None, 150, 150)
    X = R.solve(F)
    save("kat_sin50xyz_150", F=F, X=X, residual=R.residual(F, X))

    # bench_poisson's workload (poisson.cpp:190-216), sizes 16..256 (stream shared across sizes)
    for s in (16, 64, 256):
        chain = [x for x in (16, 64, 256) if x <= s]
        F = R.bench_problem(chain)
        save(f"bench_problem_{s}", F=F, X=R.solve(F, threads=4), sizes=np.array(chain))

    # poisson_oracle.hpp random_mean_zero_problem, seeds as in test_poisson.cpp:137-152
    for s in (16, 32):
        for rep in range(2):
            seed = 600 + 10 * s + rep
            F = R.random_mean_zero_problem(s, s, seed)
            save(f"rmz_{s}_{seed}", F=F, X=R.solve(F), seed=np.array(seed))

    # test_banded.cpp:67-87 — bordered solve of the zero-mode system, m = 32
    rng = np.random.default_rng(77)
    b = rng.uniform(-1, 1, 32) + 1j * rng.uniform(-1, 1, 32)
    lap = R.build_lap(32)
    w = R.integration_weights(32)
    x = R.band_solve_dense_row(lap, 2, 2, 16, w, 0j, b)
    save("bordered_zero_mode_32", lap=lap, w=w, b=b, x=x)

    # grid pipeline on seeded spherical-harmonic sums
    for (m, n, L, seed) in [(32, 64, 6, 11), (64, 64, 12, 12), (150, 150, 20, 13), (128, 96, 30, 14)]:
        c = sh_coeffs(seed, L, 2.0)
        phys = O.shgen(m, n, L, c)
        X, U = R.grid_pipeline(phys, m)
        cu = sh_coeffs(seed, L, 2.0, solution=True)
        u_exact = O.shgen(m, n, L, cu)
        save(f"grid_sh_{m}x{n}_L{L}", phys=phys, X=X, U=U, u_exact=u_exact, L=np.array(L), seed=np.array(seed))

    # analyze_1d / synthesize_1d conventions (test_fourier.cpp:29-63)
    xs = -np.pi + 2 * np.pi * np.arange(16) / 16
    save("fourier_pure_modes_16", const=R.analyze_1d(np.ones(16, complex)),
         e3=R.analyze_1d(np.exp(3j * xs)), cos=R.analyze_1d(np.cos(xs) + 0j))

    lowrank_fixtures(R)
    transform_fixtures(R)
    ge_fixtures(R)


def lowrank_fixtures(R):
    """assemble_poisson (poisson.cpp:52-86) on the low-rank factors that the
    reference's construct() (lowrank.cpp:608-721) produces for the test
    functions; sizes that truncate (m < theta modes) and pad."""
    cases = [("cos_theta", 0, None, [(64, 64)]),
             ("one_plus_cos", 1, None, [(32, 32), (16, 24)]),              # mean removal (test_poisson.cpp:186-206)
             ("ylm_pair", 2, np.array([3, -2, 1.0, 5, 1, 0.5]), [(64, 48)]),
             ("sin50xyz", 3, None, [(150, 150), (512, 384)]),             # K = 12, 256 modes: truncate / pad
             ("sinsin_cos2", 4, None, [(32, 64)])]                        # nonzero mean
    for name, fid, par, sizes in cases:
        d, col, row, vscale = R.construct_fn(fid, par)
        for m, n in sizes:
            F, rep = R.assemble_lowrank(d, col, row, vscale, m, n)
            save(f"assemble_{name}_{m}x{n}", d=d, col=col, row=row, vscale=np.array(vscale), F=F, rep=rep)


def transform_fixtures(R):
    """analyze_2d / sample_grid (fourier.cpp:170-209) on seeded complex grids,
    with sample_grid zero-padding and truncating, and the DFS doubling of
    physical samples (sphere_domain.cpp:19-26, :46-52)."""
    rng = np.random.default_rng(1510)
    for m, n, outs in [(16, 24, [(16, 24), (32, 40), (8, 12)]), (150, 150, [(150, 150), (96, 200)]),
                       (64, 48, [(64, 48), (70, 42)])]:
        g = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
        X = R.analyze_2d(g)
        arrs = {"grid": g, "X": X}
        for mo, no in outs:
            arrs[f"S_{mo}x{no}"] = R.sample_grid(X, mo, no)
        save(f"transforms_{m}x{n}", **arrs)
    for m, n in [(8, 6), (20, 16)]:
        phys = rng.standard_normal((m // 2 + 1, n))
        save(f"dfs_double_{m}x{n}", phys=phys, grid=R.sample_dfs_phys(phys, m))


def ge_grids():
    """Doubled BMC grids for the GE building blocks, after the reference's
    own test constructions (test_lowrank.cpp:68-190, acceptance_main.cpp:
    262-285): a rank-1 product, symmetrised trigonometric sums, cos(theta)
    (pivot ties on the pole rows), and seeded exact-rank BMC functions with
    complex coefficients."""
    def grid(m, n, fn):
        th = -np.pi + 2 * np.pi * np.arange(m) / m
        la = -np.pi + 2 * np.pi * np.arange(n) / n
        T, L = np.meshgrid(th, la, indexing="ij")
        return np.asarray(fn(T, L), dtype=np.complex128)

    def bmc(g):  # g(-theta, lambda + pi) = g(theta, lambda), written as the reference's tests do
        m, n = g.shape
        out = g.copy()
        for j in range(m):
            for k in range(n):
                out[(m - j) % m, (k + n // 2) % n] = out[j, k]
        return out

    def rand_rank(m, n, K, seed):
        r = np.random.default_rng(seed)

        def f(T, L):
            acc = 0
            for _ in range(K):
                p = int(r.integers(0, 2))
                a = int(r.integers(1, 6))
                b = 2 * int(r.integers(0, 4)) + p
                c = r.normal() + 1j * r.normal()
                acc = acc + c * (np.cos(a * T) if p == 0 else np.sin(a * T)) * np.exp(1j * b * L)
            return acc
        return bmc(grid(m, n, f))

    return {
        "rank1_32x32": grid(32, 32, lambda T, L: (np.cos(2 * T) + 2.0) * (np.sin(2 * L) + 0.4)),
        "sym_32x48": bmc(grid(32, 48, lambda T, L: np.cos(2 * T) * np.cos(2 * L) + np.sin(T) * np.sin(L)
                              + 0.3 * np.sin(2 * T) * np.sin(3 * L))),
        "sym4_32x32": bmc(grid(32, 32, lambda T, L: np.cos(2 * T) * np.cos(2 * L) + np.sin(T) * np.sin(L)
                               + 0.25 * np.sin(2 * T) * np.sin(4 * L) + 0.4)),
        "cos_theta_16x16": grid(16, 16, lambda T, L: np.cos(T) + 0 * L),
        "rand6_32x32": rand_rank(32, 32, 6, 515),
        "rand12_64x96": rand_rank(64, 96, 12, 7),
    }


def ge_fixtures(R):
    """pivot_search (lowrank.cpp:84-112) and ge_step (:127-162) of the
    reference, stepped until the residual is at rounding level (at most 10
    steps): per step the pivot (t, k, a, b, m_even, m_odd, theta*, lambda*)
    and, for the first two steps and the last, the updated grid."""
    for name, g in ge_grids().items():
        arrs = {"grid": g}
        cur, scale = g, np.abs(g).max()
        piv_i, piv_d, keep = [], [], []
        for step in range(10):
            p = R.pivot_search(cur)
            if p is None:
                break
            t, k, a, b, me, mo, th, lam = p
            piv_i.append([t, k])
            piv_d.append([a.real, a.imag, b.real, b.imag, me.real, me.imag, mo.real, mo.imag, th, lam])
            cur = R.ge_step(cur, p)
            if step < 2:
                arrs[f"after_{step}"] = cur
            if np.abs(cur).max() < 1e-13 * scale:
                break
        arrs.update(piv_i=np.array(piv_i, np.int64), piv_d=np.array(piv_d), final=cur)
        save(f"ge_{name}", **arrs)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
