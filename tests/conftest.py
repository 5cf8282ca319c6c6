import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100) device; run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import ORACLE_SO, Oracle, build
    if not os.path.exists(ORACLE_SO):
        build(ref=False)
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference, reference_available
    if not reference_available():
        pytest.skip("oracle/_ref (the reference compiled from /root/reference) is not built here")
    return Reference()


def ref_grid(reference, f, m, threads=8):
    """The reference's own grid composition (oracle/_ref: sample_dfs ->
    analyze_2d -> Msin^2 -> solve -> sample_grid) on physical samples f.
    Returns (X_ref, U_ref, u_herm): the reference's M x N coefficients and
    complex doubled grid, and the real physical-row grid synthesised by the
    reference's sample_grid from X_ref with its k < 0 half replaced by the
    Hermitian mirror of k > 0 (X(t,-k) = conj X(-t,k); the unpaired t = -M/2
    row maps to itself) -- the semantics of the real grid path sk_solve_grid."""
    import numpy as np
    from oracle.oracle import phys_from_doubled
    n = f.shape[-1]
    X, U = reference.grid_pipeline(f, m, threads=threads)
    L = m // 2
    t = np.arange(m) - L
    tt = np.where(t == -L, -L, -t) + L
    Xm = X.copy()
    for kc in range(1, n // 2):
        k = kc - n // 2
        Xm[:, kc] = np.conj(X[tt, n // 2 - k])
    u_herm = phys_from_doubled(reference.sample_grid(Xm, m, n), m).real
    return X, U, u_herm


def zero_mean_noise(oracle, m, n, seed):
    """White-noise physical samples with the surface mean removed (the
    constant 1 has 2 pi w^T e_0 = 4 pi): the rough-data workload."""
    import numpy as np
    rng = np.random.default_rng(seed)
    f = rng.standard_normal((m // 2 + 1, n))
    A = oracle.analyze_2d(oracle.dfs_double(f, m))
    mu = (oracle.integration_weights(m) * A[:, n // 2]).sum() / 2.0
    return f - mu.real


def golden(name):
    import numpy as np
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def pytest_collection_modifyitems(config, items):
    """Without an explicit -m, GPU tests are skipped where no device exists."""
    if config.getoption("-m"):
        return
    try:
        import torch
        have = torch.cuda.is_available()
    except Exception:
        have = False
    if have:
        return
    skip = pytest.mark.skip(reason="no CUDA device (run with -m gpu on a B200)")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
