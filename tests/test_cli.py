"""CLI front end (paper_1510_08094_b200/cli.py, the reference's `spherekit
poisson / residual / bench` routes, tools/spherekit_main.cpp:289-368): the
binary container, the exit-code contract and the bench table on CPU; the
device routes end to end on the GPU."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, "-m", "paper_1510_08094_b200", *args], capture_output=True, text=True,
                       cwd=ROOT, timeout=300)
    return r.returncode, r.stdout, r.stderr


def test_sgrid_round_trip(tmp_path):
    from paper_1510_08094_b200.cli import KIND_COEFFS, KIND_PHYS, load_sgrid, save_sgrid
    rng = np.random.default_rng(0)
    f = rng.standard_normal((9, 12))
    save_sgrid(str(tmp_path / "f.sgrid"), f, KIND_PHYS, 16, 12)
    g, kind, M, N = load_sgrid(str(tmp_path / "f.sgrid"))
    assert (kind, M, N) == (KIND_PHYS, 16, 12) and np.array_equal(g, f)
    X = rng.standard_normal((2, 16, 12)) + 1j * rng.standard_normal((2, 16, 12))
    save_sgrid(str(tmp_path / "x.sgrid"), X, KIND_COEFFS, 16, 12)
    Y, kind, M, N = load_sgrid(str(tmp_path / "x.sgrid"))
    assert kind == KIND_COEFFS and np.array_equal(Y, X)


def test_exit_codes(tmp_path):
    # argument errors -> 2 (parse_error), I/O errors -> 4 (io_error), as spherekit_main.cpp:375-406
    assert _run()[0] == 2
    assert _run("poisson", "--out", str(tmp_path / "u.sgrid"), "--expr", "x*y")[0] == 2
    assert _run("bench", "--sizes", "a,b")[0] == 2
    assert _run("solve", "--in", str(tmp_path / "missing.sgrid"), "--out", str(tmp_path / "x.sgrid"))[0] == 4
    (tmp_path / "junk.sgrid").write_bytes(b"not a grid")
    assert _run("residual", "--rhs", str(tmp_path / "junk.sgrid"), "--sol", str(tmp_path / "junk.sgrid"))[0] == 4


def test_bench_table_format():
    import io
    from paper_1510_08094_b200.cli import bench_table
    from paper_1510_08094_b200.poisson import BenchRow
    out = io.StringIO()
    bench_table([BenchRow(256, 610, 0.001), BenchRow(512, 152, 0.004)], out)
    lines = out.getvalue().splitlines()
    assert lines[0].split() == ["size", "reps", "sec/solve", "ratio", "Mdof/s"]
    assert lines[1].split()[3] == "-" and float(lines[2].split()[3]) == pytest.approx(4.0)


@pytest.mark.gpu
def test_cli_poisson_and_residual_on_device(tmp_path, oracle, reference):
    """poisson --in samples: the grid solve (and --exact, the reference's
    composition) against the reference; solve + residual in coefficient space
    print the reference's report lines."""
    from conftest import ref_grid, zero_mean_noise
    from paper_1510_08094_b200.cli import KIND_COEFFS, KIND_PHYS, load_sgrid, save_sgrid
    from paper_1510_08094_b200 import inputs
    m, n = 64, 48
    # band-limited samples: the real grid path solves the reference's problem (residual ~ rounding)
    fb = oracle.shgen(m, n, 12, inputs.sh_coeffs(3, 12, 2.0))
    save_sgrid(str(tmp_path / "fb.sgrid"), fb, KIND_PHYS, m, n)
    rc, out, err = _run("poisson", "--in", str(tmp_path / "fb.sgrid"), "--out", str(tmp_path / "ub.sgrid"),
                        "--coeffs", str(tmp_path / "x.sgrid"))
    assert rc == 0, err
    assert out.startswith("poisson solve 64x48: residual")
    assert float(out.split("residual")[1].split(",")[0]) < 1e-12
    # white noise: the real grid path is the Hermitian completion of the reference's X ...
    f = zero_mean_noise(oracle, m, n, 4)
    save_sgrid(str(tmp_path / "f.sgrid"), f, KIND_PHYS, m, n)
    rc, out, err = _run("poisson", "--in", str(tmp_path / "f.sgrid"), "--out", str(tmp_path / "u.sgrid"))
    assert rc == 0, err
    u, kind, M, N = load_sgrid(str(tmp_path / "u.sgrid"))
    X_ref, U_ref, u_herm = ref_grid(reference, f, m)
    assert kind == KIND_PHYS and np.abs(u - u_herm).max() <= 1e-10 * np.abs(u_herm).max()
    # ... and --exact is the reference's own composition (every lambda mode solved)
    rc, out, err = _run("poisson", "--in", str(tmp_path / "f.sgrid"), "--out", str(tmp_path / "U.sgrid"), "--exact")
    assert rc == 0, err
    assert float(out.split("residual")[1].split(",")[0]) < 1e-12
    U, kind, _, _ = load_sgrid(str(tmp_path / "U.sgrid"))
    assert np.abs(U - U_ref).max() <= 1e-10 * np.abs(U_ref).max()
    F = oracle.random_mean_zero_problem(32, 32, 9)
    save_sgrid(str(tmp_path / "F.sgrid"), F, KIND_COEFFS, 32, 32)
    assert _run("solve", "--in", str(tmp_path / "F.sgrid"), "--out", str(tmp_path / "X.sgrid"))[0] == 0
    X, _, _, _ = load_sgrid(str(tmp_path / "X.sgrid"))
    cols = np.arange(32) != 16
    np.testing.assert_array_equal(X[:, cols], reference.solve(F)[:, cols])
    rc, out, _ = _run("residual", "--rhs", str(tmp_path / "F.sgrid"), "--sol", str(tmp_path / "X.sgrid"))
    assert rc == 0 and "interior residual:" in out and "constraint |2pi w'X0|:" in out
    # nonzero mean -> precondition_error -> exit code 3
    save_sgrid(str(tmp_path / "bad.sgrid"), np.ones((m // 2 + 1, n)), KIND_PHYS, m, n)
    assert _run("poisson", "--in", str(tmp_path / "bad.sgrid"), "--out", str(tmp_path / "b.sgrid"))[0] == 3


@pytest.mark.gpu
def test_cli_bench_table_on_device():
    rc, out, err = _run("bench", "--sizes", "64,128")
    assert rc == 0, err
    lines = out.splitlines()
    assert lines[0].split()[0] == "size" and len(lines) == 3
    rc, out, err = _run("bench", "--sizes", "64,128", "--grid")
    assert rc == 0, err and len(out.splitlines()) == 3
