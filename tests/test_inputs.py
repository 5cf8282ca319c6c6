"""CPU: the package's input generators reproduce the reference's RNG streams."""
import numpy as np
import pytest

from paper_1510_08094_b200 import inputs


@pytest.mark.parametrize("sizes", [[16], [16, 64], [16, 64, 256]])
def test_bench_problem_bitwise(oracle, sizes):
    assert np.array_equal(inputs.bench_problem(sizes), oracle.bench_problem(sizes))


@pytest.mark.parametrize("m,n,seed", [(16, 16, 760), (32, 32, 921), (64, 32, 3)])
def test_random_mean_zero_bitwise(oracle, m, n, seed):
    assert np.array_equal(inputs.random_mean_zero_problem(m, n, seed), oracle.random_mean_zero_problem(m, n, seed))


def test_sh_coeffs_properties():
    c = inputs.sh_coeffs(7, 40, 2.0)
    assert c.shape == (41 * 41,) and c[0] == 0.0
    assert np.array_equal(c, inputs.sh_coeffs(7, 40, 2.0))
    # counter-based: a prefix is independent of L
    assert np.array_equal(inputs.sh_coeffs(7, 10, 2.0), c[: 11 * 11] * 1.0)
    z = inputs.normals(1, np.arange(200000))
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01
    u = inputs.sh_coeffs(7, 40, 2.0, solution=True)
    l = np.floor(np.sqrt(np.arange(41 * 41)))
    assert np.allclose(u[1:], -c[1:] / (l[1:] * (l[1:] + 1)))


def test_configs_match_baseline():
    import json, os
    base = json.load(open(os.path.join(os.path.dirname(os.path.dirname(__file__)), "BASELINE.json")))
    assert len(base["configs"]) == 5
    assert inputs.CONFIGS["C3"].dof == 100_000_000
    assert inputs.CONFIGS["C5"].dof == 65536 * 32768 // 2
