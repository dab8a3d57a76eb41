"""ctypes binding of the native C-ABI library (include/pf_b200.h).

There is no fallback: if ``_build/libpf_b200.so`` is missing and cannot be
built, or no CUDA device is present when a device entry point is called, the
call raises.  The product path never runs a CPU restatement of the kernels.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import build as _build

_lock = threading.Lock()
_lib = None


class NativeError(RuntimeError):
    """A pf_* entry point returned an error status."""


def lib():
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                # PF_B200_LIB selects a tuning variant built with build.py --variant
                path = os.environ.get("PF_B200_LIB") or _build.LIB
                if not os.path.exists(path):
                    try:
                        _build.build()
                    except Exception as exc:  # noqa: BLE001
                        raise NativeError(
                            f"native library {path} is missing and could not be built: {exc}") from exc
                _lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
                _declare(_lib)
    return _lib


_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)


_gen = None


def gen_lib():
    """libpf_gen.so (include/pf_gen.h): host-only input generation."""
    global _gen
    if _gen is None:
        with _lock:
            if _gen is None:
                if not os.path.exists(_build.GEN_LIB):
                    try:
                        _build.build_gen()
                    except Exception as exc:  # noqa: BLE001
                        raise NativeError(f"{_build.GEN_LIB} is missing and could not be built: {exc}") from exc
                L = C.CDLL(_build.GEN_LIB)
                _declare_gen(L)
                _gen = L
    return _gen


def _declare_gen(L):
    L.pf_ksp_run.restype = C.c_void_p
    L.pf_ksp_run.argtypes = [C.c_int32, C.c_int64, _i64p, _i64p, _f64p, _f64p, C.c_int64, _i64p, _i64p,
                             C.c_int32, C.c_int32]
    L.pf_ksp_sizes.argtypes = [C.c_void_p, _i64p, _i64p]
    L.pf_ksp_export.argtypes = [C.c_void_p, _i64p, _i64p, _i64p]
    L.pf_ksp_free.argtypes = [C.c_void_p]
    L.pf_validate_paths.restype = C.c_int64
    L.pf_validate_paths.argtypes = [C.c_int64, _i64p, _i64p, _i64p, C.c_int64, _i64p, _i64p, _i64p, _i64p]


def _declare(L):
    from . import _abi
    _abi.declare(L)


def last_error() -> str:
    buf = C.create_string_buffer(4096)
    lib().pf_last_error(buf, C.c_size_t(len(buf)))
    return buf.value.decode(errors="replace")


_INPUT_ERROR = None


def _input_error_type():
    """PF_ERR_INPUT is the reference's InputError (model.py:20); the type is
    also a NativeError so callers catching either keep working."""
    global _INPUT_ERROR
    if _INPUT_ERROR is None:
        from .topology import InputError

        class NativeInputError(InputError, NativeError):
            pass
        _INPUT_ERROR = NativeInputError
    return _INPUT_ERROR


def check(status: int) -> None:
    if status != 0:
        msg = f"pf status {status}: {last_error()}"
        if status == 1:  # PF_ERR_INPUT
            raise _input_error_type()(msg)
        raise NativeError(msg)
