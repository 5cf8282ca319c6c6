"""CPU: the C-ABI library loads and exports every symbol include/sk_poisson.h
declares; host-side argument checks and the error contract (no compute)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "sk_poisson.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sk_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1510_08094_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_1510_08094_b200 import build
        build.build()
    return _lib.load()


def test_header_declares_expected_api():
    from paper_1510_08094_b200 import _lib
    assert _header_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    from paper_1510_08094_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (sk_[a-z_0-9]+)", out))
    for sym in _header_symbols():
        assert sym in exported, sym
        assert getattr(lib, sym) is not None


def test_library_is_sm100a_only(lib):
    from paper_1510_08094_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(8\d|90)\b", out)


def test_version_and_error_strings(lib):
    assert b"sm_100a" in lib.sk_version()
    assert lib.sk_last_error() is not None


def test_size_error_before_device_probe():
    import paper_1510_08094_b200 as p
    with pytest.raises(p.size_error):
        p.Plan(15, 16)
    with pytest.raises(p.size_error):
        p.Plan(16, 0)


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    import paper_1510_08094_b200 as p
    with pytest.raises(p.DeviceError):
        p.Plan(16, 16)


def test_null_arguments_rejected(lib):
    import ctypes
    from paper_1510_08094_b200 import _lib
    assert lib.sk_plan_create(16, 16, 1, 0, None) == _lib.SK_ERR_ARGUMENT
    assert lib.sk_solve_coeffs(None, None, None, 0) == _lib.SK_ERR_ARGUMENT
    assert lib.sk_plan_destroy(None) == _lib.SK_OK
    info = (ctypes.c_longlong * 16)()
    assert lib.sk_plan_info(None, info) == _lib.SK_ERR_ARGUMENT
