"""ctypes binding of the C ABI in ``include/sk_poisson.h``.

The product path is the in-tree ``libsk_poisson.so`` (sm_100a).  There is no
CPU fallback: if the library is missing or no device is present every compute
call raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SK_LIB_PATH") or os.path.join(HERE, "libsk_poisson.so")  # override: A/B builds

SK_OK = 0
SK_ERR_SIZE = 1
SK_ERR_PRECONDITION = 2
SK_ERR_SINGULAR = 3
SK_ERR_CUDA = 4
SK_ERR_UNSUPPORTED = 5
SK_ERR_ARGUMENT = 6
SK_ERR_NCCL = 7

SK_HOST = 0
SK_DEVICE = 1
SK_ASYNC = 2
SK_GE_HALF = 8

# Every symbol declared in include/sk_poisson.h (checked by tests/test_abi.py).
EXPORTS = [
    "sk_plan_create", "sk_plan_destroy", "sk_plan_set_stream", "sk_sync", "sk_solve_coeffs", "sk_residual",
    "sk_solve_grid", "sk_last_mean", "sk_shgen", "sk_stage_lambda_fwd", "sk_stage_theta", "sk_stage_lambda_inv",
    "sk_plan_info", "sk_stage_times", "sk_enable_stage_timing", "sk_last_error", "sk_version",
    "sk_stage_lambda_fwd_peer", "sk_stage_theta_peer", "sk_device_alloc", "sk_device_free", "sk_ipc_handle",
    "sk_ipc_open", "sk_ipc_close", "sk_assemble", "sk_analyze_2d", "sk_sample_grid", "sk_sample_dfs",
    "sk_solve_grid_exact", "sk_ipc_event_create", "sk_ipc_event_open", "sk_event_destroy", "sk_event_record",
    "sk_stream_wait_event", "sk_stage_stats", "sk_ge_pivot_search", "sk_ge_step", "sk_ge_run",
]


# Exception types named after the reference's (types.hpp:43-65).
class size_error(ValueError):
    """Reference spherekit::size_error (std::invalid_argument)."""


class precondition_error(RuntimeError):
    """Reference spherekit::precondition_error."""


class structure_error(RuntimeError):
    """Reference spherekit::structure_error."""


class DeviceError(RuntimeError):
    """CUDA failure, or no usable sm_100 device (there is no CPU fallback)."""


class UnsupportedError(ValueError):
    """Size outside the FFT factorisation / on-chip limits of this build."""


_ERRORS = {
    SK_ERR_SIZE: size_error,
    SK_ERR_PRECONDITION: precondition_error,
    SK_ERR_SINGULAR: structure_error,
    SK_ERR_CUDA: DeviceError,
    SK_ERR_UNSUPPORTED: UnsupportedError,
    SK_ERR_ARGUMENT: ValueError,
    SK_ERR_NCCL: RuntimeError,
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libsk_poisson.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1510_08094_b200.build` "
            "(the solver has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    I = ctypes.c_int
    U = ctypes.c_uint
    D = ctypes.POINTER(ctypes.c_double)
    IP = ctypes.POINTER(ctypes.c_int)
    sig = {
        "sk_plan_create": (I, [I, I, I, I, ctypes.POINTER(P)]),
        "sk_plan_destroy": (I, [P]),
        "sk_plan_set_stream": (I, [P, P]),
        "sk_sync": (I, [P]),
        "sk_solve_coeffs": (I, [P, P, P, U]),
        "sk_residual": (I, [P, P, P, D, U]),
        "sk_solve_grid": (I, [P, P, P, P, U]),
        "sk_last_mean": (I, [P, D]),
        "sk_shgen": (I, [P, I, P, P]),
        "sk_stage_lambda_fwd": (I, [P, I, IP, IP, I, P, P]),
        "sk_stage_theta": (I, [P, I, IP, IP, I, P]),
        "sk_stage_lambda_inv": (I, [P, I, IP, IP, I, P, P]),
        "sk_plan_info": (I, [P, ctypes.POINTER(ctypes.c_longlong)]),
        "sk_stage_times": (I, [P, D]),
        "sk_enable_stage_timing": (I, [P, I]),
        "sk_stage_lambda_fwd_peer": (I, [P, I, IP, IP, I, P, ctypes.POINTER(P)]),
        "sk_stage_theta_peer": (I, [P, I, IP, IP, I, P, ctypes.POINTER(P)]),
        "sk_device_alloc": (I, [I, ctypes.c_size_t, ctypes.POINTER(P)]),
        "sk_device_free": (I, [P]),
        "sk_ipc_handle": (I, [P, ctypes.c_char_p]),
        "sk_ipc_open": (I, [I, ctypes.c_char_p, ctypes.POINTER(P)]),
        "sk_ipc_close": (I, [P]),
        "sk_assemble": (I, [P, I, I, I, P, P, P, ctypes.c_double, P, D, U]),
        "sk_analyze_2d": (I, [P, I, I, P, P, U]),
        "sk_sample_grid": (I, [P, I, I, P, I, I, P, U]),
        "sk_sample_dfs": (I, [P, I, I, P, P, U]),
        "sk_solve_grid_exact": (I, [P, P, P, P, U]),
        "sk_ipc_event_create": (I, [I, ctypes.c_char_p, ctypes.POINTER(P)]),
        "sk_ipc_event_open": (I, [I, ctypes.c_char_p, ctypes.POINTER(P)]),
        "sk_event_destroy": (I, [P]),
        "sk_event_record": (I, [P, P]),
        "sk_stream_wait_event": (I, [P, P]),
        "sk_stage_stats": (I, [P, D]),
        "sk_ge_pivot_search": (I, [P, I, I, P, ctypes.c_double, IP, D, U]),
        "sk_ge_step": (I, [P, I, I, P, D, P, U]),
        "sk_ge_run": (I, [P, I, I, P, ctypes.c_double, ctypes.c_double, I, IP, IP, D, D, U]),
        "sk_last_error": (ctypes.c_char_p, []),
        "sk_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != SK_OK:
        msg = load().sk_last_error().decode()
        raise _ERRORS.get(rc, RuntimeError)(msg)
