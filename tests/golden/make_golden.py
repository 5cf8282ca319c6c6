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
        {"lowrank": lowrank_fixtures, "transforms": transform_fixtures}[only](R)
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


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else None)
