"""ctypes binding of the C ABI (include/moa_b200.h) — the backend plug point.

This plays the role of the reference's backend selection (_backend.py:5-12):
the compiled library is loaded once at import.  There is no fallback: when
``libmoa_b200.so`` is absent or a call fails, the product raises BackendError.
ctypes releases the GIL around foreign calls, so concurrent Python threads can
launch concurrently, as the reference's nogil loop allows (_ckernel.pyx:81).
"""

from __future__ import annotations

import ctypes
import threading

from .build import LIB_PATH
from .errors import BackendError

DTYPE_F64 = 0
DTYPE_F32 = 1
DTYPE_I32 = 2
DTYPE_I64 = 3
FLAG_ACCUMULATE = 1
FLAG_EXACT = 2

# every symbol include/moa_b200.h declares
EXPORTS = ("moa_product_rows", "moa_product_rows_host", "moa_last_error", "moa_abi_version",
           "moa_device_count", "moa_launch_count", "moa_plan_kernel", "moa_host_alloc",
           "moa_host_free")

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None
_load_error: str | None = None

_i64 = ctypes.c_int64


def _bind(lib: ctypes.CDLL) -> None:
    lib.moa_product_rows.restype = ctypes.c_int
    lib.moa_product_rows.argtypes = [
        ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
        _i64, _i64, _i64, _i64, _i64, _i64,
        ctypes.c_int, ctypes.c_int, _i64, _i64, ctypes.c_uint32, ctypes.c_void_p]
    lib.moa_product_rows_host.restype = ctypes.c_int
    lib.moa_product_rows_host.argtypes = [
        ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
        _i64, _i64, _i64, _i64, _i64, _i64,
        ctypes.c_int, ctypes.c_int, _i64, _i64, ctypes.c_uint32, ctypes.c_int]
    lib.moa_last_error.restype = ctypes.c_char_p
    lib.moa_last_error.argtypes = []
    lib.moa_abi_version.restype = ctypes.c_int
    lib.moa_abi_version.argtypes = []
    lib.moa_device_count.restype = ctypes.c_int
    lib.moa_device_count.argtypes = []
    lib.moa_launch_count.restype = ctypes.c_uint64
    lib.moa_launch_count.argtypes = []
    lib.moa_host_alloc.restype = ctypes.c_void_p
    lib.moa_host_alloc.argtypes = [ctypes.c_size_t]
    lib.moa_host_free.restype = None
    lib.moa_host_free.argtypes = [ctypes.c_void_p]
    lib.moa_plan_kernel.restype = ctypes.c_char_p
    lib.moa_plan_kernel.argtypes = [ctypes.c_int, _i64, _i64, _i64, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_uint32]


def load() -> ctypes.CDLL:
    """The loaded library; raises BackendError (loudly) if it is not built."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                _load_error = (f"CUDA backend {LIB_PATH} is not built; run "
                               f"`python -m paper_0907_0792_b200.build`")
                raise BackendError(_load_error)
            try:
                lib = ctypes.CDLL(str(LIB_PATH))
            except OSError as exc:  # pragma: no cover - depends on the host
                _load_error = f"cannot load {LIB_PATH}: {exc}"
                raise BackendError(_load_error) from exc
            try:
                _bind(lib)
            except AttributeError as exc:  # a stale build missing a newer entry point
                _load_error = f"{LIB_PATH} is out of date ({exc}); rebuild it"
                raise BackendError(_load_error) from exc
            _lib = lib
    return _lib


def available() -> bool:
    try:
        load()
        return True
    except BackendError:
        return False


def product_rows(dtype: int, res_ptr: int, a_ptr: int, b_ptr: int,
                 noproc: int, rowsinred: int, elsinop: int,
                 lstride: int, rstride: int, restride: int,
                 combine_code: int, reduce_code: int, start: int, step: int,
                 flags: int, stream: int) -> None:
    """moa_product_rows on raw device pointers; raises BackendError on failure."""
    lib = load()
    rc = lib.moa_product_rows(dtype, res_ptr, a_ptr, b_ptr, noproc, rowsinred, elsinop,
                              lstride, rstride, restride, combine_code, reduce_code,
                              start, step, flags, stream)
    if rc != 0:
        msg = lib.moa_last_error().decode(errors="replace")
        raise BackendError(f"moa_product_rows failed ({rc}): {msg}")


def product_rows_host(dtype: int, res_ptr: int, a_ptr: int, b_ptr: int,
                      noproc: int, rowsinred: int, elsinop: int,
                      lstride: int, rstride: int, restride: int,
                      combine_code: int, reduce_code: int, start: int, step: int,
                      flags: int, device: int) -> None:
    """moa_product_rows_host on raw HOST pointers (blocks until res is written);
    raises BackendError on failure."""
    lib = load()
    rc = lib.moa_product_rows_host(dtype, res_ptr, a_ptr, b_ptr, noproc, rowsinred, elsinop,
                                   lstride, rstride, restride, combine_code, reduce_code,
                                   start, step, flags, device)
    if rc != 0:
        msg = lib.moa_last_error().decode(errors="replace")
        raise BackendError(f"moa_product_rows_host failed ({rc}): {msg}")


def plan_kernel(dtype: int, noproc: int, rowsinred: int, elsinop: int,
                combine_code: int, reduce_code: int, flags: int = 0) -> str:
    return load().moa_plan_kernel(dtype, noproc, rowsinred, elsinop, combine_code,
                                  reduce_code, flags).decode()


def host_alloc(nbytes: int) -> int:
    """moa_host_alloc: page-locked, huge-page-backed host memory (0 on failure)."""
    return int(load().moa_host_alloc(nbytes) or 0)


def host_free(ptr: int) -> None:
    if _lib is not None:
        _lib.moa_host_free(ptr)


def launch_count() -> int:
    return int(load().moa_launch_count())


def abi_version() -> int:
    return int(load().moa_abi_version())
