"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the oracle, plus size-independent properties at full size."""
import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, ref_grid, zero_mean_noise

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: GPU tests need a B200 (there is no CPU fallback)")
    import paper_1510_08094_b200 as p
    return p


def _coeff_cases():
    out = []
    for f in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        d = np.load(f)
        if "F" in d and "X" in d:
            out.append(os.path.basename(f)[:-4])
    return out


def _assert_reference_bits(X, Xref, n):
    """Bit-identical for every k != 0 column; k = 0 to rounding."""
    cols = np.arange(n) != n // 2
    np.testing.assert_array_equal(X[:, cols], Xref[:, cols])
    scale = max(np.abs(Xref).max(), 1e-300)
    assert np.abs(X[:, n // 2] - Xref[:, n // 2]).max() <= 1e-15 * scale + 1e-300


@pytest.mark.parametrize("name", _coeff_cases())
def test_coeff_solve_matches_reference_golden(pkg, name):
    d = golden(name)
    F = d["F"]
    m, n = F.shape
    sol = pkg.solve(pkg.PoissonProblem(m, n, F))
    _assert_reference_bits(sol.x, d["X"], n)


@pytest.mark.parametrize("s", [512, 1024, 2048])
def test_coeff_solve_bench_workload_vs_oracle(pkg, oracle, s):
    F = oracle.bench_problem([s])
    with pkg.Plan(s, s) as plan:
        X = plan.solve_coeffs(F)
    _assert_reference_bits(X, oracle.solve(F, threads=8), s)


def test_bench_poisson_mirror(pkg, oracle):
    """bench_poisson (poisson.cpp:188-230) on the device: the reference's
    sizes -> (size, reps, seconds) rows, the same RNG stream across sizes
    (the generator is not reseeded between sizes), its size check, and the
    problem it times solved bit-identically to the reference's solve."""
    import paper_1510_08094_b200 as sk
    rows = sk.bench_poisson([64, 128], reps=2)
    assert [r.size for r in rows] == [64, 128] and all(r.reps == 2 and r.seconds > 0 for r in rows)
    with pytest.raises(sk.size_error):
        sk.bench_poisson([15])
    from paper_1510_08094_b200.inputs import bench_problem
    F = bench_problem([64, 128])  # the second problem of the stream
    assert np.array_equal(F, oracle.bench_problem([64, 128]))
    with pkg.Plan(128, 128) as plan:
        X = plan.solve_coeffs(F)
    _assert_reference_bits(X, oracle.solve(F, threads=4), 128)


@pytest.mark.parametrize("m,n,seed", [(64, 32, 1), (32, 64, 2), (150, 40, 3), (18, 22, 4)])
def test_coeff_solve_rectangular_vs_oracle(pkg, oracle, m, n, seed):
    F = oracle.random_mean_zero_problem(m, n, seed)
    X = pkg.solve(pkg.PoissonProblem(m, n, F)).x
    _assert_reference_bits(X, oracle.solve(F), n)


def test_coeff_solve_errors(pkg):
    d = golden("kat_precondition_16")
    with pytest.raises(pkg.precondition_error):
        pkg.solve(pkg.PoissonProblem(16, 16, d["F"]))
    with pytest.raises(pkg.size_error):
        pkg.solve(pkg.PoissonProblem(15, 16, np.zeros((15, 16), complex)))
    X = pkg.solve(pkg.PoissonProblem(16, 16, np.zeros((16, 16), complex))).x
    assert not X.any()


def test_kat_cos_theta_and_residual(pkg):
    d = golden("kat_cos_theta_64")
    pb = pkg.PoissonProblem(64, 64, d["F"])
    sol = pkg.solve(pb)
    expect = np.zeros((64, 64), complex)
    expect[31, 32] = expect[33, 32] = -0.25
    assert np.abs(sol.x - expect).max() < 1e-13
    r = pkg.residual(pb, sol)
    assert r.interior_max < 1e-12 and r.constraint_abs < 1e-12
    ref = d["residual"]
    assert abs(r.interior_max - ref[0]) <= 1e-15 and abs(r.constraint_abs - ref[2]) <= 1e-15


def test_residual_vs_oracle(pkg, oracle):
    F = oracle.random_mean_zero_problem(32, 32, 5)
    X = oracle.solve(F)
    with pkg.Plan(32, 32) as plan:
        r = plan.residual(F, X)
        ro = oracle.residual(F, X)
        assert abs(r.interior_max - ro[0]) <= 1e-15 and abs(r.replaced_row_abs - ro[1]) <= 1e-15
        assert abs(r.constraint_abs - ro[2]) <= 1e-15
        X2 = X.copy()
        X2[7, 9] += 1e-3  # test_poisson.cpp:176-184
        assert plan.residual(F, X2).interior_max > 1e-5


def test_coeff_solve_batched_rhs(pkg, oracle):
    Fs = np.stack([oracle.random_mean_zero_problem(64, 64, 100 + r) for r in range(5)])
    with pkg.Plan(64, 64, nrhs=5) as plan:
        X = plan.solve_coeffs(Fs)
    for r in range(5):
        _assert_reference_bits(X[r], oracle.solve(Fs[r]), 64)


# ------------------------------------------------------------- grid path
def _grid_cases():
    return [os.path.basename(f)[:-4] for f in sorted(glob.glob(os.path.join(GOLDEN, "grid_sh_*.npz")))]


@pytest.mark.parametrize("name", _grid_cases())
def test_grid_solve_matches_reference_golden(pkg, name):
    from oracle.oracle import phys_from_doubled
    d = golden(name)
    m, n = d["X"].shape
    with pkg.Plan(m, n) as plan:
        u, Xh = plan.solve_grid(d["phys"], coeffs=True)
    uref = phys_from_doubled(d["U"], m).real
    assert np.abs(u - uref).max() <= 1e-10 * np.abs(uref).max()
    Xref = d["X"][:, n // 2:].T  # k = 0..N/2-1 columns
    assert np.abs(Xh[: n // 2] - Xref).max() <= 1e-10 * np.abs(d["X"]).max()
    # the analytic solution
    assert np.abs(u - d["u_exact"]).max() <= 1e-12 * np.abs(d["u_exact"]).max()


@pytest.mark.parametrize("m,n,L", [(512, 256, 32), (112, 98, 20), (160, 90, 30), (40, 12, 4), (8, 4, 1)])
def test_grid_solve_vs_reference(pkg, oracle, reference, m, n, L):
    """Band-limited input through the grid path against the reference's own
    composition (oracle/_ref): its complex u (real part; the imaginary part is
    rounding for band-limited data) and its coefficients X."""
    from oracle.oracle import phys_from_doubled
    from paper_1510_08094_b200 import inputs
    c = inputs.sh_coeffs(m + n, L, 2.0)
    f = oracle.shgen(m, n, L, c)
    X_ref, U_ref, _ = ref_grid(reference, f, m)
    u_ref = phys_from_doubled(U_ref, m)
    assert np.abs(u_ref.imag).max() <= 1e-12 * np.abs(u_ref).max()
    with pkg.Plan(m, n) as plan:
        u, Xh = plan.solve_grid(f, coeffs=True)
    assert np.abs(u - u_ref.real).max() <= 1e-10 * np.abs(u_ref).max()
    assert np.abs(Xh[: n // 2] - X_ref[:, n // 2:].T).max() <= 1e-10 * np.abs(X_ref).max()


@pytest.mark.parametrize("m,n", [(64, 48), (256, 128), (150, 150), (60, 32), (120, 40), (30, 64)])
def test_grid_solve_rough_data_vs_reference(pkg, oracle, reference, m, n):
    """Non-band-limited (white-noise) data with zero mean, against the
    reference's own composition (oracle/_ref).  The reference solves every
    lambda mode k >= 0 exactly as the grid path does: the solution
    coefficients X_half must match its X to 1e-10.  Its k < 0 columns differ
    from the Hermitian mirror of k > 0 when the data reach the truncation rows
    (its theta operators are not mirror-symmetric at j = -M/2), so its u is
    complex there; the real grid path synthesises the Hermitian completion of
    the reference's own X, which the reference's sample_grid computes here
    (ref_grid: u_herm).  The reference's complex u itself is matched by
    sk_solve_grid_exact (tests/test_gpu_exact.py)."""
    f = zero_mean_noise(oracle, m, n, 3 + m)
    X_ref, _, u_herm = ref_grid(reference, f, m)
    with pkg.Plan(m, n) as plan:
        u, Xh = plan.solve_grid(f, coeffs=True)
    assert np.abs(Xh[: n // 2] - X_ref[:, n // 2:].T).max() <= 1e-10 * np.abs(X_ref).max()
    assert np.abs(Xh[n // 2] - X_ref[:, 0]).max() <= 1e-10 * np.abs(X_ref).max()  # Nyquist k = -N/2
    assert np.abs(u - u_herm).max() <= 1e-10 * np.abs(u_herm).max()


_SWEEP = [(16, 16), (24, 20), (100, 30), (200, 24), (300, 20), (600, 28), (1024, 24), (1200, 16), (2000, 20),
          (3000, 16), (4096, 16), (5000, 12), (8192, 12), (9000, 8), (14000, 8), (20000, 8), (24, 600), (40, 1200),
          (32, 4096), (24, 5000), (16, 10000), (36, 18), (84, 42), (500, 250), (1470, 14), (14, 1470)]


@pytest.mark.parametrize("m,n", _SWEEP)
def test_grid_size_sweep_vs_reference(pkg, oracle, reference, m, n):
    """Rough zero-mean data across the plan's kernel-selection boundaries
    (segment / register / shared-memory chain solvers, high-occupancy and
    swizzled variants, theta_sym, row-pair lambda kernels, radices 3 / 5 / 7)
    against the reference's own composition (oracle/_ref), the comparands of
    test_grid_solve_rough_data_vs_reference.  Half lengths with a prime factor
    > 7 belong to sk_solve_grid_exact (tests/test_gpu_exact.py)."""
    f = zero_mean_noise(oracle, m, n, m + 3 * n)
    X_ref, _, u_herm = ref_grid(reference, f, m)
    with pkg.Plan(m, n) as plan:
        u, Xh = plan.solve_grid(f, coeffs=True)
    assert np.abs(Xh[: n // 2] - X_ref[:, n // 2:].T).max() <= 1e-10 * np.abs(X_ref).max()
    assert np.abs(u - u_herm).max() <= 1e-10 * np.abs(u_herm).max()


@pytest.mark.parametrize("m,n", [(44, 26), (1204, 22), (26, 1204)])
def test_grid_unsupported_lengths_fail_loudly(pkg, oracle, m, n):
    """Half lengths with a prime factor > 7 are outside the real grid path
    (DESIGN section 7): it reports SK_ERR_UNSUPPORTED instead of computing
    anything, and the same data go through sk_solve_grid_exact."""
    from paper_1510_08094_b200._lib import UnsupportedError
    f = zero_mean_noise(oracle, m, n, 5)
    with pytest.raises(UnsupportedError):
        with pkg.Plan(m, n) as plan:
            plan.solve_grid(f)
    with pkg.Plan(m, n) as plan:
        U = plan.solve_grid_exact(f)
    assert np.isfinite(U).all()


def test_grid_precondition_error(pkg):
    m, n = 32, 16
    f = np.ones((m // 2 + 1, n))
    with pkg.Plan(m, n) as plan:
        with pytest.raises(pkg.precondition_error):
            plan.solve_grid(f)


def test_shgen_vs_oracle(pkg, oracle):
    import torch
    from paper_1510_08094_b200 import inputs
    m, n, L = 96, 80, 30
    c = inputs.sh_coeffs(5, L, 2.0)
    ref = oracle.shgen(m, n, L, c)
    with pkg.Plan(m, n) as plan:
        cd = torch.from_numpy(c).cuda()
        out = torch.empty((m // 2 + 1, n), dtype=torch.float64, device="cuda")
        plan.shgen(L, cd, out)
        torch.cuda.synchronize()
    assert np.abs(out.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max()


def test_grid_batched_rhs_bitwise(pkg, oracle):
    from paper_1510_08094_b200 import inputs
    m, n, L = 128, 64, 20
    fs = np.stack([oracle.shgen(m, n, L, inputs.sh_coeffs(40 + r, L, 1.5)) for r in range(3)])
    with pkg.Plan(m, n, nrhs=3) as plan:
        ub = plan.solve_grid(fs)
    with pkg.Plan(m, n) as plan:
        for r in range(3):
            assert np.array_equal(plan.solve_grid(fs[r]), ub[r])


@pytest.mark.parametrize("P", [2, 3, 4])
def test_slab_stages_bitwise_equal_single_gpu(pkg, oracle, P):
    """The multi-rank slab path (stage entry points + the all-to-all block
    layout) emulated on one GPU with device copies: bit-identical to the
    single-GPU solve."""
    import torch
    from paper_1510_08094_b200 import distributed as dist_mod, inputs
    m, n, L = 160, 96, 24
    f = oracle.shgen(m, n, L, inputs.sh_coeffs(9, L, 2.0))
    with pkg.Plan(m, n) as plan:
        u1 = plan.solve_grid(f)
    u = dist_mod.emulate_slabs(f, m, n, P)
    assert np.array_equal(u, u1)


def test_grid_full_size_analytic_C2(pkg):
    """Size-independent property at config C2 (4096 x 2048, L = 512): the
    grid solve reproduces the analytic solution -sum c_lm Y/(l(l+1))."""
    import torch
    from paper_1510_08094_b200 import inputs
    cfg = inputs.CONFIGS["C2"]
    with pkg.Plan(cfg.M, cfg.N) as plan:
        rows = cfg.M // 2 + 1
        f = torch.empty((rows, cfg.N), dtype=torch.float64, device="cuda")
        ue = torch.empty_like(f)
        plan.shgen(cfg.L, torch.from_numpy(inputs.sh_coeffs(2, cfg.L, cfg.p)).cuda(), f)
        plan.shgen(cfg.L, torch.from_numpy(inputs.sh_coeffs(2, cfg.L, cfg.p, solution=True)).cuda(), ue)
        u = plan.solve_grid(f)
        torch.cuda.synchronize()
        err = (u - ue).abs().max().item() / ue.abs().max().item()
    assert err <= 1e-10, err


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_grid_full_size_analytic(pkg, name):
    """The same property at the bench workloads: C3 (20000 x 10000, L = 2000,
    the paper-scale single RHS) and C4 (64 RHS of 2048 x 1024, L = 256, one
    batched plan): every right-hand side against its analytic solution."""
    import torch
    from paper_1510_08094_b200 import inputs
    cfg = inputs.CONFIGS[name]
    rows = cfg.M // 2 + 1
    with pkg.Plan(cfg.M, cfg.N, cfg.nrhs) as plan:
        f = torch.empty((cfg.nrhs, rows, cfg.N), dtype=torch.float64, device="cuda")
        for r in range(cfg.nrhs):
            plan.shgen(cfg.L, torch.from_numpy(inputs.sh_coeffs(11 + r, cfg.L, cfg.p)).cuda(), f[r])
        u = plan.solve_grid(f if cfg.nrhs > 1 else f[0])
        if cfg.nrhs == 1:
            u = u.unsqueeze(0)
        del f
        ue = torch.empty((rows, cfg.N), dtype=torch.float64, device="cuda")
        worst = 0.0
        for r in range(cfg.nrhs):
            plan.shgen(cfg.L, torch.from_numpy(inputs.sh_coeffs(11 + r, cfg.L, cfg.p, solution=True)).cuda(), ue)
            worst = max(worst, ((u[r] - ue).abs().max() / ue.abs().max()).item())
    assert worst <= 1e-10, worst


# ------------------------------------------------- cluster-split kernels
@pytest.mark.parametrize("m,n,L", [(32768, 48, 20), (64, 32768, 20), (32768, 32768 // 64, 24)])
def test_grid_split_kernels_vs_reference(pkg, oracle, reference, m, n, L):
    """theta length M/2 = 16384 runs the 8-CTA cluster kernel, lambda length
    N/2 = 16384 the CTA-pair kernels; both against the reference's own
    composition (oracle/_ref)."""
    from oracle.oracle import phys_from_doubled
    from paper_1510_08094_b200 import inputs
    c = inputs.sh_coeffs(m // 7 + n, L, 2.0)
    f = oracle.shgen(m, n, L, c)
    _, U_ref, _ = ref_grid(reference, f, m)
    u_ref = phys_from_doubled(U_ref, m).real
    with pkg.Plan(m, n) as plan:
        info = plan.info()
        u = plan.solve_grid(f)
    assert info["theta_split"] in (2, 8)
    assert np.abs(u - u_ref).max() <= 1e-10 * np.abs(u_ref).max()


@pytest.mark.parametrize("m,n", [(32768, 24), (64, 32768)])
def test_grid_split_kernels_rough_data(pkg, oracle, reference, m, n):
    """Random (non-band-limited) zero-mean data through the cluster kernels:
    every spectral entry is O(1), so a wrong pivot, twiddle or cross-CTA
    carry shows up at full size."""
    f = zero_mean_noise(oracle, m, n, m + n)
    X_ref, _, u_ref = ref_grid(reference, f, m)
    with pkg.Plan(m, n) as plan:
        u, Xh = plan.solve_grid(f, coeffs=True)
    assert np.abs(Xh[: n // 2] - X_ref[:, n // 2:].T).max() <= 1e-10 * np.abs(X_ref).max()
    assert np.abs(u - u_ref).max() <= 1e-10 * np.abs(u_ref).max()


@pytest.mark.parametrize("m,n,tma", [(64, 32768, "1"), (64, 32768, "0"), (30, 32768, "1"), (18, 36864, "1"),
                                     (18, 36864, "0"), (16, 20480, "1")])
def test_lambda_split_gather_paths(pkg, oracle, reference, m, n, tma, monkeypatch):
    """Rows split over a CTA pair (N/2 beyond one CTA's shared memory): the
    inverse gathers each CTA's modes (k = c mod 2) through per-parity tensor
    maps (default when a thread's mode pairs fit its registers), or with
    per-thread loads (SK_SPLIT_TMA=0, and lengths beyond that limit); rough
    data against the reference's composition, odd row counts included."""
    monkeypatch.setenv("SK_SPLIT_TMA", tma)
    f = zero_mean_noise(oracle, m, n, m + n)
    X_ref, _, u_ref = ref_grid(reference, f, m)
    with pkg.Plan(m, n) as plan:
        u, Xh = plan.solve_grid(f, coeffs=True)
    assert np.abs(Xh[: n // 2] - X_ref[:, n // 2:].T).max() <= 1e-10 * np.abs(X_ref).max()
    assert np.abs(u - u_ref).max() <= 1e-10 * np.abs(u_ref).max()


@pytest.mark.parametrize("m,n,theta_hi,lambda_hi", [(2048, 1024, True, True), (4096, 2048, True, True),
                                                     (20000, 10000, False, False), (512, 256, True, True)])
def test_plan_kernel_variants(pkg, m, n, theta_hi, lambda_hi):
    """Short columns / rows select the high-occupancy kernel variants (C4,
    C2, C1); the paper-scale plan keeps the 128-register kernels."""
    with pkg.Plan(m, n) as plan:
        v = plan.info()["variants"]
    assert bool(v & 1) == theta_hi and bool(v & 2) == lambda_hi, v


@pytest.mark.parametrize("m,n,nrhs", [(512, 256, 1), (2048, 1024, 3), (60, 32, 2), (1000, 360, 1), (4096, 64, 2),
                                        (500, 48, 1), (20, 24, 1), (1536, 40, 1)])
def test_fwd_rows_gather_bitwise(pkg, oracle, reference, m, n, nrhs, monkeypatch):
    """The row-major forward spectrum (lambda_fwd writes each row's modes
    contiguously, theta_kernel gathers its raw column through two tensor maps:
    boxes of 256 rows and the tail box; default for large batches of short
    columns, C4) against the mode-major stores: the same values take another
    route, so the solves agree bit for bit (several RHS, row counts with every
    tail-box size, swizzled and unswizzled plans), and against the reference."""
    f = np.stack([zero_mean_noise(oracle, m, n, 3 * m + n + r) for r in range(nrhs)])
    fin = f if nrhs > 1 else f[0]
    monkeypatch.setenv("SK_FWD_ROWS", "1")
    with pkg.Plan(m, n, nrhs) as plan:
        assert plan.info()["variants"] & 1024, plan.info()
        u1 = plan.solve_grid(fin)
    monkeypatch.setenv("SK_FWD_ROWS", "0")
    with pkg.Plan(m, n, nrhs) as plan:
        assert not plan.info()["variants"] & 1024
        u0 = plan.solve_grid(fin)
    assert np.array_equal(u0, u1)
    _, _, u_ref = ref_grid(reference, f[0], m)
    assert np.abs((u1[0] if nrhs > 1 else u1) - u_ref).max() <= 1e-10 * np.abs(u_ref).max()


def test_fwd_rows_default_policy(pkg):
    """On for theta_kernel solves of at least 2^23 spectral entries (C4: 64
    RHS of 2048 x 1024), off for a single small grid and for C3's theta_sym
    columns."""
    with pkg.Plan(2048, 1024, 64) as plan:
        assert plan.info()["variants"] & 1024
    with pkg.Plan(2048, 1024) as plan:
        assert not plan.info()["variants"] & 1024
    with pkg.Plan(20000, 10000) as plan:
        assert not plan.info()["variants"] & 1024


@pytest.mark.parametrize("m,n", [(256, 1024), (128, 2048), (96, 512), (64, 4096)])
def test_grid_pow2_rows_rough_data(pkg, oracle, reference, m, n):
    """Power-of-two lambda rows (N/2 = 256 .. 2048) run the lambda kernels on
    XOR-swizzled slots (per-thread row loads, swizzled pack and store); rough
    zero-mean data makes every slot of the permutation matter."""
    f = zero_mean_noise(oracle, m, n, 7 * m + n)
    X_ref, _, u_ref = ref_grid(reference, f, m)
    with pkg.Plan(m, n) as plan:
        u, Xh = plan.solve_grid(f, coeffs=True)
    assert np.abs(Xh[: n // 2] - X_ref[:, n // 2:].T).max() <= 1e-10 * np.abs(X_ref).max()
    assert np.abs(u - u_ref).max() <= 1e-10 * np.abs(u_ref).max()


def test_slab_stages_cluster_kernels_bitwise(pkg, oracle):
    from paper_1510_08094_b200 import distributed as dist_mod, inputs
    m, n, L = 32768, 40, 12
    f = oracle.shgen(m, n, L, inputs.sh_coeffs(3, L, 2.0))
    with pkg.Plan(m, n) as plan:
        u1 = plan.solve_grid(f)
    assert np.array_equal(dist_mod.emulate_slabs(f, m, n, 3), u1)


def test_grid_full_size_analytic_C5(pkg):
    """Config C5 (65536 x 32768, 1.07e9 DOF, L = 8192) against the analytic
    solution: the size-independent check at the largest configuration."""
    import torch
    from paper_1510_08094_b200 import inputs
    cfg = inputs.CONFIGS["C5"]
    rows = cfg.M // 2 + 1
    with pkg.Plan(cfg.M, cfg.N) as plan:
        f = torch.empty((rows, cfg.N), dtype=torch.float64, device="cuda")
        plan.shgen(cfg.L, torch.from_numpy(inputs.sh_coeffs(5, cfg.L, cfg.p)).cuda(), f)
        u = plan.solve_grid(f)
        del f
        ue = torch.empty_like(u)
        plan.shgen(cfg.L, torch.from_numpy(inputs.sh_coeffs(5, cfg.L, cfg.p, solution=True)).cuda(), ue)
        torch.cuda.synchronize()
        err = ((u - ue).abs().max() / ue.abs().max()).item()
    assert err <= 1e-10, err


def test_pipelined_host_solves(pkg, oracle):
    """SK_HOST | SK_ASYNC: consecutive host-memory solves overlap through two
    device slots; each result equals the synchronous solve bit for bit, and a
    nonzero-mean input is reported by a later call or by sync()."""
    from paper_1510_08094_b200 import inputs
    m, n, L = 256, 128, 20
    fs = [oracle.shgen(m, n, L, inputs.sh_coeffs(40 + i, L, 2.0)) for i in range(5)]
    with pkg.Plan(m, n) as plan:
        ref = [plan.solve_grid(f) for f in fs]
        outs = [np.empty_like(f) for f in fs]
        for f, u in zip(fs, outs):
            plan.solve_grid(f, u, sync=False)
        plan.sync()
        for a, b in zip(outs, ref):
            assert np.array_equal(a, b)
        bad = fs[0] + 1.0
        ub = np.empty_like(bad)
        with pytest.raises(pkg.precondition_error):
            plan.solve_grid(bad, ub, sync=False)
            plan.solve_grid(fs[1], np.empty_like(bad), sync=False)
            plan.solve_grid(fs[2], np.empty_like(bad), sync=False)
            plan.sync()


@pytest.mark.parametrize("m,n", [(64, 3000), (128, 3000), (40, 2400), (54, 3000), (50, 3000), (60, 3000)])
def test_lambda_row_groups_bitwise(pkg, oracle, reference, m, n, monkeypatch):
    """Long non-power-of-two lambda rows run the forward lambda transform on
    CTA pairs (row pairs, 32-byte stores; default), on 4-CTA clusters
    (SK_LAMBDA_QUAD=1: row quads, 64-byte stores; the default for peer
    stores) or one row per CTA (SK_LAMBDA_QUAD=0 SK_LAMBDA_PAIR=0); row counts
    M/2+1 = 33, 65, 21, 28, 26, 31 cover every padding case.  All three are
    bit-identical, and against the reference on rough zero-mean data."""
    f = zero_mean_noise(oracle, m, n, m * n)
    monkeypatch.setenv("SK_LAMBDA_QUAD", "1")
    with pkg.Plan(m, n) as plan:
        assert plan.info()["variants"] & 128, plan.info()
        u = plan.solve_grid(f)
    monkeypatch.setenv("SK_LAMBDA_QUAD", "0")
    with pkg.Plan(m, n) as plan:
        assert not plan.info()["variants"] & 128 and plan.info()["variants"] & 16
        u2 = plan.solve_grid(f)
    monkeypatch.setenv("SK_LAMBDA_PAIR", "0")
    with pkg.Plan(m, n) as plan:
        assert not plan.info()["variants"] & 16
        u1 = plan.solve_grid(f)
    assert np.array_equal(u, u1) and np.array_equal(u2, u1)
    _, _, u_ref = ref_grid(reference, f, m)
    assert np.abs(u - u_ref).max() <= 1e-10 * np.abs(u_ref).max()


@pytest.mark.parametrize("m,n,paired", [(64, 3000, True), (54, 3000, True), (40, 2400, False)])
def test_lambda_inv_row_pairs_bitwise(pkg, oracle, reference, m, n, paired, monkeypatch):
    """The opt-in inverse lambda transform on CTA pairs (SK_LAMBDA_PAIR_INV=1:
    2-row TMA boxes, the peer's modes through DSMEM; used when the row's box
    count is even: L = 1500 -> 6 boxes, L = 1200 -> 5 boxes falls back):
    bit-identical to the one-row-per-CTA kernel for odd (33) and even (28)
    row counts, and against the oracle."""
    f = zero_mean_noise(oracle, m, n, m * n + 1)
    with pkg.Plan(m, n) as plan:
        assert not plan.info()["variants"] & 32
        u1 = plan.solve_grid(f)
    monkeypatch.setenv("SK_LAMBDA_PAIR_INV", "1")
    with pkg.Plan(m, n) as plan:
        assert bool(plan.info()["variants"] & 32) == paired, plan.info()
        u = plan.solve_grid(f)
    assert np.array_equal(u, u1)
    _, _, u_ref = ref_grid(reference, f, m)
    assert np.abs(u - u_ref).max() <= 1e-10 * np.abs(u_ref).max()


@pytest.mark.parametrize("m,n", [(64, 3000), (54, 3000), (40, 2400), (50, 3000), (128, 10000)])
def test_lambda_duo_bitwise(pkg, oracle, reference, m, n, monkeypatch):
    """The opt-in lambda stages on row pairs inside one CTA (SK_LAMBDA_DUO=1,
    lambda_duo.cu: local 32-byte (p, p+1) stores, 2-row TMA boxes in the
    inverse; measured slower at C3 than two independent CTAs per SM, so not
    the default): bit-identical to the one-row-per-CTA kernels for odd (33,
    21) and even (28, 26) row counts and at C3's row length, and against the
    reference on rough zero-mean data."""
    f = zero_mean_noise(oracle, m, n, m * n + 2)
    monkeypatch.setenv("SK_LAMBDA_DUO", "1")
    with pkg.Plan(m, n) as plan:
        assert plan.info()["variants"] & 512, plan.info()
        u = plan.solve_grid(f)
    monkeypatch.setenv("SK_LAMBDA_DUO", "0")
    monkeypatch.setenv("SK_LAMBDA_PAIR", "0")
    with pkg.Plan(m, n) as plan:
        assert not plan.info()["variants"] & (512 | 16)
        u1 = plan.solve_grid(f)
    assert np.array_equal(u, u1)
    _, _, u_ref = ref_grid(reference, f, m)
    assert np.abs(u - u_ref).max() <= 1e-10 * np.abs(u_ref).max()


@pytest.mark.parametrize("m,n", [(2048, 64), (4096, 24), (512, 48), (256, 40), (64, 32), (32, 16)])
def test_pair_chains_matches_two_solves(pkg, oracle, reference, m, n, monkeypatch):
    """Short even columns (C1, C2, C4: theta_kernel's segment solver) take both
    chains of a parity from ONE solve (solve_chains_pair_fast: x- = s x+ +
    Phi Delta, the pairing of theta_sym.cu on the unpruned transform).  On
    rough zero-mean data (every lambda mode excited, the truncation rows
    included) it agrees with the two separate solves (SK_PAIR_CHAINS=0) to
    rounding and with the reference to 1e-10."""
    f = zero_mean_noise(oracle, m, n, 3 * m + n)
    with pkg.Plan(m, n) as plan:
        u = plan.solve_grid(f)
    monkeypatch.setenv("SK_PAIR_CHAINS", "0")
    with pkg.Plan(m, n) as plan:
        u2 = plan.solve_grid(f)
    assert np.abs(u - u2).max() <= 1e-12 * np.abs(u2).max()
    _, _, u_ref = ref_grid(reference, f, m)
    assert np.abs(u - u_ref).max() <= 1e-10 * np.abs(u_ref).max()


@pytest.mark.parametrize("m,n", [(512, 256), (2048, 64), (6000, 64), (12000, 48), (64, 3000), (65536, 24), (256, 32768)])
def test_repeated_solves_bitwise(pkg, oracle, m, n):
    """Every kernel family of the grid path — the paired segment solver on short
    columns, theta_sym, the multi-pass theta stage (M/2 = 32768), lambda row
    pairs and the split lambda rows — gives the same bits on every one of 12
    consecutive solves of rough data (a shared-memory or DSMEM race, or a
    barrier released too early, shows up as run-to-run differences; this pool
    has no compute-sanitizer)."""
    f = zero_mean_noise(oracle, m, n, 7 * m + n)
    with pkg.Plan(m, n) as plan:
        u0 = plan.solve_grid(f).copy()
        for _ in range(11):
            assert np.array_equal(plan.solve_grid(f), u0)


def test_bench_multi_rank_launcher():
    """bench.py --gpus 2 without a launcher re-runs itself under
    torch.distributed.run with 2 ranks (on a one-GPU box both share GPU 0:
    gloo plumbing, p2p transport): n_gpus = 2, a slab roofline, parity."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--config", "C1", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "slab2"
    assert line["roofline"] is not None and line["roofline"]["slab"]["P"] == 2
    assert line["parity_rel_err_vs_analytic"] <= 1e-10


# --------------------------------------------- theta_sym_kernel (C3 path)
@pytest.mark.parametrize("m,n", [(6000, 64), (12000, 48), (4200, 40), (20000, 24)])
def test_theta_sym_rough_data_vs_reference(pkg, oracle, reference, m, n):
    """Long even theta columns whose plan starts with a power-of-two radix
    over an odd span run theta_sym_kernel (pruned forward transform through
    the column's mirror symmetry, both chains of a parity from one solve plus
    the boundary correction).  White-noise zero-mean data against the
    reference's own composition: X to 1e-10, u to 1e-10 of the Hermitian
    completion of the reference's X."""
    f = zero_mean_noise(oracle, m, n, 5 * m + n)
    X_ref, _, u_ref = ref_grid(reference, f, m)
    with pkg.Plan(m, n) as plan:
        assert plan.info()["variants"] & 64, plan.info()
        u, Xh = plan.solve_grid(f, coeffs=True)
    assert np.abs(Xh[: n // 2] - X_ref[:, n // 2:].T).max() <= 1e-10 * np.abs(X_ref).max()
    assert np.abs(Xh[n // 2] - X_ref[:, 0]).max() <= 1e-10 * np.abs(X_ref).max()
    assert np.abs(u - u_ref).max() <= 1e-10 * np.abs(u_ref).max()


@pytest.mark.parametrize("m,n", [(12000, 48), (6000, 64)])
def test_theta_sym_matches_pair_kernel(pkg, oracle, m, n, monkeypatch):
    """theta_sym_kernel against the pair kernel it replaces (SK_THETA_SYM=0)
    on the same rough data: equal to rounding (different but exact
    arithmetic), and the pair kernel's fast chain solver stays inside its
    digit-reversal window past the chain ends (M = 12000)."""
    f = zero_mean_noise(oracle, m, n, m - n)
    with pkg.Plan(m, n) as plan:
        u = plan.solve_grid(f)
    monkeypatch.setenv("SK_THETA_SYM", "0")
    with pkg.Plan(m, n) as plan:
        assert not plan.info()["variants"] & 64
        u0 = plan.solve_grid(f)
    assert np.abs(u - u0).max() <= 1e-12 * np.abs(u0).max()
