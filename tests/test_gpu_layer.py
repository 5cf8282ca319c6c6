"""GPU parity of the widened boundary: assemble_poisson,
analyze_2d, sample_grid (zero-pad / truncate) and DFS doubling, through the C
ABI, against the reference's golden vectors and the oracle."""
import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: GPU tests need a B200 (there is no CPU fallback)")
    import paper_1510_08094_b200 as p
    return p


def _names(prefix):
    return [os.path.basename(f)[:-4] for f in sorted(glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))]


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def _c(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


# ------------------------------------------------------------ assemble_poisson
@pytest.mark.parametrize("name", _names("assemble_"))
def test_assemble_bit_identical_to_reference_golden(pkg, name):
    # poisson.cpp:52-86 on the reference's own construct() factors
    d = golden(name)
    m, n = d["F"].shape
    f = pkg.LowRankSphereFun(d["d"], d["col"], d["row"], float(d["vscale"]))
    rep = pkg.AssembleReport()
    pb = pkg.assemble_poisson(f, m, n, rep)
    np.testing.assert_array_equal(pb.f, d["F"])
    assert rep.mean_removed == bool(d["rep"][0])
    assert rep.removed_mean == complex(d["rep"][1], d["rep"][2])


@pytest.mark.parametrize("K,mf,nf,m,n,vs", [(3, 10, 8, 16, 12, 0.0), (5, 40, 30, 24, 64, 1e30), (1, 2, 2, 8, 8, 0.0),
                                           (7, 300, 200, 128, 96, 0.0), (40, 64, 64, 256, 512, 0.0),
                                           (0, 4, 4, 8, 8, 0.0), (2, 0, 6, 10, 6, 0.0)])
def test_assemble_random_factors_vs_oracle(pkg, oracle, K, mf, nf, m, n, vs):
    rng = np.random.default_rng(K * 1000 + mf)
    d, col, row = _c(rng, K), _c(rng, K, mf), _c(rng, K, nf)
    d[:K // 3] = 0  # exact-zero terms are skipped by the reference (poisson.cpp:66)
    F0, r0 = oracle.assemble(d, col, row, vs, m, n)
    with pkg.Plan(m, n) as plan:
        F, r = plan.assemble(d, col, row, vs)
    np.testing.assert_array_equal(F, F0)
    np.testing.assert_array_equal(np.array(r), r0)


def test_assemble_device_tensors(pkg, oracle):
    import torch
    rng = np.random.default_rng(11)
    d, col, row = _c(rng, 4), _c(rng, 4, 20), _c(rng, 4, 18)
    F0, r0 = oracle.assemble(d, col, row, 1.0, 32, 24)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    with pkg.Plan(32, 24) as plan:
        F, r = plan.assemble(t(d), t(col), t(row), 1.0)
        torch.cuda.synchronize()
    np.testing.assert_array_equal(F.cpu().numpy(), F0)
    np.testing.assert_array_equal(np.array(r), r0)


def test_assemble_then_solve_is_the_reference_composition(pkg):
    # assemble -> solve: the reference CLI's `poisson` route (spherekit_main.cpp:292-299)
    d = golden("assemble_sin50xyz_150x150")
    f = pkg.LowRankSphereFun(d["d"], d["col"], d["row"], float(d["vscale"]))
    pb = pkg.assemble_poisson(f, 150, 150)
    kat = golden("kat_sin50xyz_150")
    np.testing.assert_array_equal(pb.f, kat["F"])
    X = pkg.solve(pb).x
    r = pkg.residual(pb, pkg.PoissonSolution(X))
    assert r.interior_max <= 1e-10 * np.abs(pb.f).max() and r.constraint_abs <= 1e-12


def test_assemble_size_errors(pkg):
    with pkg.Plan(8, 8) as plan:
        with pytest.raises(pkg.size_error):
            plan.assemble(np.ones(1, complex), np.ones((1, 3), complex), np.ones((1, 2), complex))
    with pytest.raises(pkg.size_error):
        pkg.assemble_poisson(pkg.LowRankSphereFun(np.ones(1), np.ones((1, 2)), np.ones((1, 2))), 7, 8)


# -------------------------------------------------- analyze_2d / sample_grid
@pytest.mark.parametrize("name", _names("transforms_"))
def test_transforms_match_reference_golden(pkg, name):
    d = golden(name)
    X = pkg.analyze_2d(d["grid"])
    assert _rel(X, d["X"]) <= 1e-14
    for k in d.files:
        if k.startswith("S_"):
            mo, no = map(int, k[2:].split("x"))
            assert _rel(pkg.sample_grid(d["X"], mo, no), d[k]) <= 1e-13, k


@pytest.mark.parametrize("m,n", [(4, 2), (6, 10), (128, 96), (1000, 700), (2048, 4096)])
def test_transforms_vs_oracle_and_round_trip(pkg, oracle, m, n):
    rng = np.random.default_rng(m + n)
    g = _c(rng, m, n)
    X = pkg.analyze_2d(g)
    if m * n <= 1 << 20:
        assert _rel(X, oracle.analyze_2d(g)) <= 1e-14
        outs = [(2 * m, 2 * n)] + ([(m // 2, n // 2)] if m % 4 == 0 and n % 4 == 0 else [])
        for mo, no in outs:  # zero-pad and truncate
            assert _rel(pkg.sample_grid(X, mo, no), oracle.sample_grid(X, mo, no)) <= 1e-13
    # round trip (test_fourier.cpp:198-211): sample_grid(analyze_2d(g)) = g
    assert _rel(pkg.sample_grid(X, m, n), g) <= 1e-13


@pytest.mark.parametrize("m,n,gather", [(64, 10000, "1"), (10000, 48, "1"), (96, 8192, "1"), (8192, 64, "1"),
                                        (48, 9000, "1"), (1000, 700, "0"), (96, 8192, "0"), (6, 10, "0")])
def test_transforms_gather_and_transposed_passes(pkg, oracle, m, n, gather, monkeypatch):
    """The two pass structures of the 2-D transforms: columns gathered by the
    copy engine with contiguous stores (default when both lengths are plain
    smooth transforms whose columns fit the register staging: 20 elements per
    thread, unswizzled analysis unstaged) and row loads with transposed stores
    (SK_XFORM_GATHER=0, Bluestein lengths); against the
    oracle, zero-padded / truncated synthesis and the round trip."""
    import subprocess, sys, json, os, textwrap
    # the switch is read once per process: run the case in a child
    code = textwrap.dedent(f"""
        import sys, json
        import numpy as np
        sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
        import paper_1510_08094_b200 as pkg
        from oracle.oracle import Oracle
        o = Oracle()
        m, n = {m}, {n}
        rng = np.random.default_rng(m + n)
        g = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
        rel = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())
        X = pkg.analyze_2d(g)
        out = dict(analyze=rel(X, o.analyze_2d(g)), round_trip=rel(pkg.sample_grid(X, m, n), g))
        mo = 2 * m if m <= 4000 else m // 2
        no = n // 2 if n % 4 == 0 else n
        out["resample"] = rel(pkg.sample_grid(X, mo, no), o.sample_grid(X, mo, no))
        print(json.dumps(out))
    """)
    env = dict(os.environ, SK_XFORM_GATHER=gather)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["analyze"] <= 1e-14, out
    assert out["round_trip"] <= 1e-13 and out["resample"] <= 1e-13, out


def test_transforms_device_tensors(pkg):
    import torch
    rng = np.random.default_rng(3)
    g = _c(rng, 60, 84)
    X0 = pkg.analyze_2d(g)
    with pkg.Plan(8, 4) as plan:
        gt = torch.from_numpy(g).cuda()
        X = plan.analyze_2d(gt)
        G = plan.sample_grid(X, 60, 84)
        torch.cuda.synchronize()
    np.testing.assert_array_equal(X.cpu().numpy(), X0)
    assert _rel(G.cpu().numpy(), g) <= 1e-13


def test_transform_errors(pkg):
    with pytest.raises(pkg.size_error):
        pkg.analyze_2d(np.zeros((6, 5), complex))
    with pytest.raises(pkg.size_error):
        pkg.sample_grid(np.zeros((6, 4), complex), 5, 4)



@pytest.mark.parametrize("m,n", [(8, 602), (602, 16), (22, 34), (150, 602)])
def test_transforms_bluestein_vs_reference(pkg, reference, m, n):
    """Transform lengths with a prime factor > 7 (602 = 2 * 7 * 43, 22, 34) run
    Bluestein convolutions on the device: analyze_2d and sample_grid (equal,
    padded and truncated sizes) against the reference itself, and the round
    trip of acceptance c11 (acceptance_main.cpp:242-257) to 1e-13."""
    rng = np.random.default_rng(m * n)
    g = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    X = pkg.analyze_2d(g)
    Xr = reference.analyze_2d(g)
    assert _rel(X, Xr) <= 1e-13
    for mo, no in [(m, n), (m + 4, n + 2), (max(2, m - 4), max(2, n - 2))]:
        assert _rel(pkg.sample_grid(Xr, mo, no), reference.sample_grid(Xr, mo, no)) <= 1e-13
    assert _rel(pkg.sample_grid(X, m, n), g) <= 1e-13


# ------------------------------------------------------------- DFS doubling
@pytest.mark.parametrize("name", _names("dfs_double_"))
def test_sample_dfs_golden(pkg, name):
    d = golden(name)
    np.testing.assert_array_equal(pkg.sample_dfs(d["phys"], d["grid"].shape[0]), d["grid"])


def test_sample_dfs_then_analyze_matches_grid_pipeline(pkg):
    # the grid-level composition's first two steps against the reference's
    d = golden("grid_sh_64x64_L12")
    g = pkg.sample_dfs(d["phys"], 64)
    X = pkg.analyze_2d(g)
    from oracle.oracle import Oracle
    Xo = Oracle().analyze_2d(Oracle().dfs_double(d["phys"], 64))
    assert _rel(X, Xo) <= 1e-14


# ------------------------------------------------- cluster exit barriers
_EXIT_SCRIPT = r'''
import os, sys, numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, os.path.join(sys.argv[1], "tests"))
from conftest import zero_mean_noise
from oracle.oracle import Oracle
from paper_1510_08094_b200.poisson import Plan
orc = Oracle()
out = {}
# lambda_fwd CTA pairs + theta pair kernel (64 x 3000), theta cluster kernel
# (32768 x 24), lambda split kernels (64 x 32768), and a full-occupancy grid
for m, n in [(64, 3000), (32768, 24), (64, 32768), (4000, 3000)]:
    f = zero_mean_noise(orc, m, n, m + n)
    with Plan(m, n) as plan:
        for rep in range(4):
            out[f"{m}x{n}_{rep}"] = plan.solve_grid(f)
np.savez(sys.argv[2], **out)
'''


def test_exit_barrier_variants_bitwise(tmp_path):
    """Every cluster kernel ending in cluster_exit_barrier (theta pair,
    theta cluster, lambda_fwd pairs, lambda_inv split) gives bit-identical
    results with the relaxed arrive (default) and with the release-ordered
    cluster.sync() (SK_PAIR_SYNC_EXIT=1), repeatedly and under full
    occupancy (theta_common.cuh contract)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "exit.py"
    script.write_text(_EXIT_SCRIPT)
    res = {}
    for name, extra in [("relaxed", {}), ("sync", {"SK_PAIR_SYNC_EXIT": "1"})]:
        env = dict(os.environ, **extra)
        subprocess.run([sys.executable, str(script), root, str(tmp_path / f"{name}.npz")], check=True, env=env,
                       timeout=600)
        res[name] = np.load(tmp_path / f"{name}.npz")
    keys = sorted(res["relaxed"].files)
    assert keys and keys == sorted(res["sync"].files)
    for k in keys:
        assert np.array_equal(res["relaxed"][k], res["sync"][k]), k
        base = k.rsplit("_", 1)[0] + "_0"
        assert np.array_equal(res["relaxed"][k], res["relaxed"][base]), k


@pytest.mark.parametrize("m,n", [(60, 8), (30, 6), (22, 10), (64, 8)])
def test_sample_dfs_pole_row_quirk(pkg, oracle, m, n):
    """sk_sample_dfs replicates the reference's floating-point pole row (for
    m = 22, 30, 60 theta_{m/2} < 0 in the reference: the row p = 0 glides),
    bit for bit against the reference-pinned restatement."""
    rng = np.random.default_rng(m + n)
    phys = rng.standard_normal((m // 2 + 1, n))
    np.testing.assert_array_equal(pkg.sample_dfs(phys, m), oracle.dfs_double(phys, m))


# ---------------------------------------------- GE building blocks (lowrank.hpp:73-93)
def _bits_equal(a, b):
    a, b = np.ascontiguousarray(a, np.complex128), np.ascontiguousarray(b, np.complex128)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def _piv_doubles(p):
    return np.array([p.a.real, p.a.imag, p.b.real, p.b.imag, p.m_even.real, p.m_even.imag, p.m_odd.real, p.m_odd.imag,
                     p.theta_star, p.lambda_star])


@pytest.mark.parametrize("name", _names("ge_"))
def test_ge_steps_bit_identical_to_reference_golden(pkg, name):
    """sk_ge_pivot_search / sk_ge_step against the reference's own output
    (tests/golden/ge_*: test_lowrank.cpp:68-190's constructions): the same
    pivots and the same bits in every updated grid, step by step; then the
    device-resident loop sk_ge_run reproduces the whole run."""
    g = golden(name)
    cur = g["grid"]
    with pkg.Plan(8, 8) as plan:
        for s, (pi, pd) in enumerate(zip(g["piv_i"], g["piv_d"])):
            p = plan.pivot_search(cur)
            assert p is not None and (p.t, p.k) == (int(pi[0]), int(pi[1])), (name, s)
            assert np.array_equal(_piv_doubles(p), pd), (name, s)
            cur = plan.ge_step(cur, p)
            if f"after_{s}" in g.files:
                assert _bits_equal(cur, g[f"after_{s}"]), (name, s)
        assert _bits_equal(cur, g["final"])
        run = np.array(g["grid"], dtype=np.complex128, order="C")
        piv, resid = plan.ge_run(run, tau=1e-13 * np.abs(g["grid"]).max(), max_steps=10)
        assert len(piv) == len(g["piv_i"]) and [(p.t, p.k) for p in piv] == [tuple(int(v) for v in r) for r in g["piv_i"]]
        assert _bits_equal(run, g["final"])
        assert resid[0] == np.abs(g["grid"]).max() or abs(resid[0] / np.abs(g["grid"]).max() - 1) < 1e-15
        assert abs(resid[-1] - np.abs(g["final"]).max()) <= 1e-15 * resid[0]


def test_ge_run_device_resident_large(pkg, oracle):
    """A 512 x 768 exact-rank BMC grid on the device: the elimination ends at
    rounding level within rank/1 steps, preserves the BMC symmetry EXACTLY
    (test_lowrank.cpp:98-128's property, every step being symmetric), and its
    first steps agree bit for bit with the oracle's."""
    import torch
    m, n, K = 512, 768, 16
    rng = np.random.default_rng(3)
    th = -np.pi + 2 * np.pi * np.arange(m) / m
    la = -np.pi + 2 * np.pi * np.arange(n) / n
    g = np.zeros((m, n), np.complex128)
    for _ in range(K):
        par = int(rng.integers(0, 2))
        a, b = int(rng.integers(1, 40)), 2 * int(rng.integers(0, 30)) + par
        col = np.cos(a * th) if par == 0 else np.sin(a * th)
        g += (rng.normal() + 1j * rng.normal()) * np.outer(col, np.exp(1j * b * la))
    jm, km = (m - np.arange(m)) % m, (np.arange(n) + n // 2) % n
    g = 0.5 * (g + g[jm][:, km])  # exact BMC symmetry: g(-theta, lambda + pi) = g(theta, lambda)
    assert np.array_equal(g, g[jm][:, km])
    with pkg.Plan(8, 8) as plan:
        cur = g.copy()
        for _ in range(2):
            p, po = plan.pivot_search(cur), oracle.pivot_search(cur)
            assert (p.t, p.k) == (po[0], po[1]) and p.m_even == po[4] and p.m_odd == po[5]
            cur = plan.ge_step(cur, p)
            assert _bits_equal(cur, oracle.ge_step(g if _ == 0 else prev, po))
            prev = cur
        gd = torch.from_numpy(g.copy()).cuda()
        piv, resid = plan.ge_run(gd, tau=1e-12 * np.abs(g).max(), max_steps=64)
        r = gd.cpu().numpy()
    assert len(piv) <= K and resid[-1] <= 1e-12 * resid[0]
    assert np.array_equal(r, r[jm][:, km])


def test_ge_errors(pkg):
    with pkg.Plan(8, 8) as plan:
        with pytest.raises(pkg.size_error):
            plan.pivot_search(np.zeros((15, 16), complex))
        assert plan.pivot_search(np.zeros((16, 16), complex)) is None  # lowrank.cpp:103
        g = np.ones((16, 16), complex)
        p = plan.pivot_search(g)
        bad = pkg.PivotBlock(0.456, 0.123, p.a, p.b, p.m_even, p.m_odd)  # not a grid node (test_lowrank.cpp:127)
        with pytest.raises(ValueError):
            plan.ge_step(g, bad)


@pytest.mark.parametrize("name", ["ge_rand6_32x32", "ge_sym4_32x32", "ge_sym_32x48", "ge_rand12_64x96"])
def test_ge_half_grid_mode(pkg, oracle, name):
    """SK_GE_HALF: the elimination on the (m/2+1) x n upper half grid, as
    construct's phase 1 keeps it (lowrank.cpp:246-252, :345-392): the same
    pivots as on the doubled grid and, on the stored rows, the same bits as
    the reference's ge_step (golden) and as the oracle's phase-1 step."""
    g = golden(name)
    grid = g["grid"]
    m, n = grid.shape
    up = lambda a: np.ascontiguousarray(np.concatenate([a[m // 2:], a[:1]]))  # noqa: E731
    half = up(grid)
    with pkg.Plan(8, 8) as plan:
        cur = half
        for s, (pi, pd) in enumerate(zip(g["piv_i"], g["piv_d"])):
            p = plan.pivot_search(cur, half=True)
            assert (p.t, p.k) == (int(pi[0]), int(pi[1])) and np.array_equal(_piv_doubles(p), pd)
            nxt = plan.ge_step(cur, p, half=True)
            if m == n:
                _, oh = oracle.ge_half_step(cur)
                assert _bits_equal(nxt, oh)
            if f"after_{s}" in g.files:
                assert _bits_equal(nxt, up(g[f"after_{s}"]))
            cur = nxt
        assert _bits_equal(cur, up(g["final"]))
        run = half.copy()
        piv, resid = plan.ge_run(run, tau=1e-13 * np.abs(grid).max(), max_steps=10, half=True)
        assert [(p.t, p.k) for p in piv] == [tuple(int(v) for v in r) for r in g["piv_i"]]
        assert _bits_equal(run, up(g["final"]))
