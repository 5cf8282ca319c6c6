"""CPU: pin the oracle (C++ restatement) against the reference's golden
vectors and, where it was built, against the reference library itself."""
import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden


def _golden_solves():
    out = []
    for f in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        d = np.load(f)
        if "F" in d and "X" in d:
            out.append(os.path.basename(f)[:-4])
    return out


@pytest.mark.parametrize("name", _golden_solves())
def test_oracle_solve_bit_identical_to_reference_golden(oracle, name):
    d = golden(name)
    X = oracle.solve(d["F"], threads=2)
    assert np.array_equal(X, d["X"])


def test_kat_cos_theta(oracle):
    # test_poisson.cpp:53-67: X = -1/4 at (i=31,33; kc=32), else 0, to 1e-13
    d = golden("kat_cos_theta_64")
    X = oracle.solve(d["F"])
    expect = np.zeros((64, 64), complex)
    expect[31, 32] = expect[33, 32] = -0.25
    assert np.abs(X - expect).max() < 1e-13
    r = oracle.residual(d["F"], X)
    assert r[0] < 1e-12 and r[2] < 1e-12


def test_precondition_error(oracle):
    from oracle.oracle import OracleError
    d = golden("kat_precondition_16")
    assert int(d["expected_code"]) == 2
    with pytest.raises(OracleError) as e:
        oracle.solve(d["F"])
    assert e.value.code == 2


def test_zero_rhs_gives_zero(oracle):
    X = oracle.solve(np.zeros((16, 16), complex))
    assert not X.any()


def test_size_errors(oracle):
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as e:
        oracle.solve(np.zeros((15, 16), complex))
    assert e.value.code == 1


def test_bordered_zero_mode(oracle):
    d = golden("bordered_zero_mode_32")
    x = oracle.band_solve_dense_row(d["lap"], 2, 2, 16, d["w"], 0j, d["b"])
    assert np.array_equal(x, d["x"])


@pytest.mark.parametrize("name", [os.path.basename(f)[:-4] for f in sorted(glob.glob(os.path.join(GOLDEN, "grid_sh_*.npz")))])
def test_oracle_grid_pipeline_matches_reference(oracle, name):
    d = golden(name)
    m = d["X"].shape[0]
    X, U, up, mean = oracle.grid_pipeline(d["phys"], m)
    assert np.array_equal(X, d["X"]) and np.array_equal(U, d["U"])
    # and the reference composition reproduces the analytic solution
    assert np.abs(up - d["u_exact"]).max() <= 1e-13 * np.abs(d["u_exact"]).max()


def test_fourier_conventions(oracle):
    d = golden("fourier_pure_modes_16")
    xs = -np.pi + 2 * np.pi * np.arange(16) / 16
    assert np.abs(oracle.analyze_1d(np.ones(16, complex)) - d["const"]).max() < 1e-15
    c = oracle.analyze_1d(np.exp(3j * xs))
    assert np.abs(c - d["e3"]).max() < 1e-15
    assert abs(c[8 + 3] - 1) < 1e-15


def test_lap_and_weights_match_reference(oracle, reference):
    for m in (8, 16, 150, 512, 4096):
        assert np.array_equal(oracle.build_lap(m), reference.build_lap(m).real)
        assert not reference.build_lap(m).imag.any()
        assert np.array_equal(oracle.integration_weights(m), reference.integration_weights(m).real)


@pytest.mark.parametrize("s", [64, 512])
def test_oracle_vs_reference_bench_problem(oracle, reference, s):
    F = reference.bench_problem([s])
    assert np.array_equal(F, oracle.bench_problem([s]))
    assert np.array_equal(oracle.solve(F, 4), reference.solve(F, 4))


def test_oracle_vs_reference_dfs_and_fft(oracle, reference):
    rng = np.random.default_rng(5)
    for m, n in [(8, 6), (150, 150), (64, 602)]:
        phys = rng.standard_normal((m // 2 + 1, n))
        assert np.array_equal(oracle.dfs_double(phys, m), reference.sample_dfs_phys(phys, m))
        g = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
        assert np.array_equal(oracle.analyze_2d(g), reference.analyze_2d(g))
        X = reference.analyze_2d(g)
        assert np.array_equal(oracle.sample_grid(X, m, n), reference.sample_grid(X, m, n))


def _names(prefix):
    return [os.path.basename(f)[:-4] for f in sorted(glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))]


@pytest.mark.parametrize("name", _names("assemble_"))
def test_oracle_assemble_bit_identical_to_reference_golden(oracle, name):
    # assemble_poisson (poisson.cpp:52-86) on the reference's own construct() factors
    d = golden(name)
    m, n = d["F"].shape
    F, rep = oracle.assemble(d["d"], d["col"], d["row"], float(d["vscale"]), m, n)
    assert np.array_equal(F, d["F"]) and np.array_equal(rep, d["rep"])


def test_oracle_assemble_vs_reference_random_factors(oracle, reference):
    rng = np.random.default_rng(77)
    for K, mf, nf, m, n in [(3, 10, 8, 16, 12), (5, 40, 30, 24, 64), (1, 2, 2, 8, 8)]:
        c = lambda *s: rng.standard_normal(s) + 1j * rng.standard_normal(s)  # noqa: E731
        d, col, row = c(K), c(K, mf), c(K, nf)
        for vs in (0.0, 1e30):  # mean removed / kept
            F1, r1 = oracle.assemble(d, col, row, vs, m, n)
            F2, r2 = reference.assemble_lowrank(d, col, row, vs, m, n)
            assert np.array_equal(F1, F2) and np.array_equal(r1, r2)


@pytest.mark.parametrize("name", _names("transforms_"))
def test_oracle_transforms_match_reference_golden(oracle, name):
    # analyze_2d / sample_grid with zero-pad / truncation (fourier.cpp:55-66, :170-209)
    d = golden(name)
    X = oracle.analyze_2d(d["grid"])
    assert np.abs(X - d["X"]).max() <= 1e-15 * np.abs(d["X"]).max()
    for k in d.files:
        if k.startswith("S_"):
            mo, no = map(int, k[2:].split("x"))
            S = oracle.sample_grid(d["X"], mo, no)
            assert np.abs(S - d[k]).max() <= 1e-13 * np.abs(d[k]).max()


@pytest.mark.parametrize("name", _names("dfs_double_"))
def test_oracle_dfs_double_golden(oracle, name):
    d = golden(name)
    assert np.array_equal(oracle.dfs_double(d["phys"], d["grid"].shape[0]), d["grid"])


@pytest.mark.parametrize("m,n", [(60, 8), (30, 6), (22, 10), (64, 8), (150, 12), (44, 4)])
def test_dfs_doubling_pole_row_matches_reference(oracle, reference, m, n):
    """The reference's sample_dfs evaluates theta_j = -pi + 2 pi j/m in floating
    point (sphere_domain.hpp:54) and glides every theta < 0
    (sphere_domain.cpp:19-26): for m = 22, 30, 44, 60, ... theta_{m/2} rounds
    below zero, so the pole row p = 0 is read at longitude lambda -+ pi.  The
    restatement's index map reproduces the reference bit for bit."""
    rng = np.random.default_rng(m * n)
    phys = rng.standard_normal((m // 2 + 1, n))
    np.testing.assert_array_equal(oracle.dfs_double(phys, m), reference.sample_dfs_phys(phys, m))


# ---------------------------------------------- GE building blocks (lowrank.hpp:73-93)
def _ge_names():
    return [os.path.basename(f)[:-4] for f in sorted(glob.glob(os.path.join(GOLDEN, "ge_*.npz")))]


def _bits_equal(a, b):
    a, b = np.ascontiguousarray(a, np.complex128), np.ascontiguousarray(b, np.complex128)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("name", _ge_names())
def test_oracle_ge_bit_identical_to_reference_golden(oracle, name):
    """pivot_search (lowrank.cpp:84-112) and ge_step (:127-162) of the
    restatement against the reference's own output, step by step: the same
    pivots (node, values, pseudoinverse weights) and the same bits (zero
    signs included) in every updated grid."""
    g = golden(name)
    cur = g["grid"]
    for s, (pi, pd) in enumerate(zip(g["piv_i"], g["piv_d"])):
        p = oracle.pivot_search(cur)
        assert p is not None and (p[0], p[1]) == (int(pi[0]), int(pi[1]))
        mine = np.array([p[2].real, p[2].imag, p[3].real, p[3].imag, p[4].real, p[4].imag, p[5].real, p[5].imag,
                         p[6], p[7]])
        assert np.array_equal(mine, pd), (name, s)
        cur = oracle.ge_step(cur, p)
        if f"after_{s}" in g.files:
            assert _bits_equal(cur, g[f"after_{s}"]), (name, s)
    assert _bits_equal(cur, g["final"])


def test_oracle_ge_vs_reference_random(oracle, reference):
    rng = np.random.default_rng(84)
    for m, n in [(16, 20), (24, 16), (40, 64)]:
        cur = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))  # (no BMC symmetry needed)
        for _ in range(4):
            po, pr = oracle.pivot_search(cur, 0.05), reference.pivot_search(cur, 0.05)
            assert po == pr
            nxt = oracle.ge_step(cur, po)
            assert _bits_equal(nxt, reference.ge_step(cur, pr))
            cur = nxt
    assert oracle.pivot_search(np.zeros((16, 16), complex)) is None


@pytest.mark.parametrize("name", ["ge_rand6_32x32", "ge_sym4_32x32"])  # exactly BMC-symmetric fixtures
def test_oracle_phase1_half_step_equals_reference_full_step(oracle, name):
    """construct's phase-1 loop body on the upper half grid (lowrank.cpp:
    345-392; internal to the reference) restated: on BMC-symmetric data it
    picks the pivots of the reference's public pivot_search and leaves, on
    the stored rows, exactly the bits of the reference's ge_step on the
    doubled grid (the golden fixtures hold both)."""
    g = golden(name)
    grid = g["grid"]
    m = grid.shape[0]
    half = np.concatenate([grid[m // 2:], grid[:1]])  # theta_i = 2 pi i/m, i = 0..m/2 (theta = pi is doubled row 0)
    for s, (pi, pd) in enumerate(zip(g["piv_i"], g["piv_d"])):
        (bi, bk, a, b, me, mo), half = oracle.ge_half_step(half)
        assert (bi, bk) == (int(pi[0]), int(pi[1]))
        assert np.array_equal(np.array([a.real, a.imag, b.real, b.imag, me.real, me.imag, mo.real, mo.imag]), pd[:8])
        if f"after_{s}" in g.files:
            full = g[f"after_{s}"]
            assert _bits_equal(half, np.concatenate([full[m // 2:], full[:1]]))
    full = g["final"]
    assert _bits_equal(half, np.concatenate([full[m // 2:], full[:1]]))
