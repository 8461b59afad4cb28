"""B200 backend module for the reference package (drop in as moaprod/_b200kernel.py).

``product_rows`` has the signature and the contract of the reference's
compiled loop ``_ckernel.product_rows`` (_ckernel.pyx:75-88): numpy float64
buffers, rows ``start, start+step, ...`` folded INTO ``res`` (which the
reference's ``_Runner`` prefilled with the reduce identity, kernel.py:149),
callable concurrently from ``execute_parallel``'s threads on disjoint row
sets of one ``res`` (parallel.py:26-43).  It is one call of the library's
host-buffer entry point ``moa_product_rows_host`` (include/moa_b200.h) with
MOA_FLAG_ACCUMULATE: the library moves the caller's rows of A and res and
all of B to the GPU, runs the fold there, and writes back exactly the
caller's rows of res, so concurrent callers never overwrite each other's
rows.  Nothing but ctypes and numpy is imported; no torch in the reference's
process.

Rounding.  By default every call carries MOA_FLAG_EXACT too, so (multiply,
add) folds with the reference's separate multiply and add in l order and the
module is bit-identical to the compiled loop and the pure-Python backend for
every op pair (the reference's tests/test_kernel.py::test_bitwise_equal_backends
holds with it registered).  $MOA_B200_TENSOR_CORES=1 drops the flag: (multiply,
add) with rowsinred >= 8 then runs on the FP64 tensor cores (DMMA, fused
multiply-adds), accurate to K*2^-52*max|A|*max|B| instead of bit-identical.

``product_rows_overwrite`` is the same call for a runner that does NOT prefill
res with the identity (kernel.py:149): each row of the set is written from the
identity in registers (bit-identical to prefill + accumulate), so res only
travels device -> host and the 8-byte-per-element prefill pass disappears.
INTEGRATION.md shows the two-line _Runner branch that uses it.

The reference's execute_parallel calls this from W threads, worker k with
rows k, k+W, ... (parallel.py:37-43); worker k runs on GPU DEVICES[k mod
len(DEVICES)], so the reference's own fork-join spreads its row sets over the
GPUs of the box.  The library is found through $MOA_B200_LIB (default: the
in-tree build), the GPUs through $MOA_B200_DEVICES (comma-separated indices;
default: every visible device).  Registration in the reference's _backend.py
(:5-14) is two lines; see INTEGRATION.md.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

_DEFAULT = Path(__file__).resolve().parents[1] / "paper_0907_0792_b200" / "libmoa_b200.so"
_lib = ctypes.CDLL(os.environ.get("MOA_B200_LIB", str(_DEFAULT)))
_i64 = ctypes.c_int64
_ARGS = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         _i64, _i64, _i64, _i64, _i64, _i64, ctypes.c_int, ctypes.c_int, _i64, _i64,
         ctypes.c_uint32]
_lib.moa_product_rows_host.restype = ctypes.c_int
_lib.moa_product_rows_host.argtypes = _ARGS + [ctypes.c_int]        # ... flags, device
_lib.moa_product_rows.restype = ctypes.c_int
_lib.moa_product_rows.argtypes = _ARGS + [ctypes.c_void_p]          # ... flags, stream
_lib.moa_last_error.restype = ctypes.c_char_p
_lib.moa_device_count.restype = ctypes.c_int
MOA_DTYPE_F64 = 0
MOA_FLAG_ACCUMULATE = 1
MOA_FLAG_EXACT = 2
# reference rounding unless the caller opts into the tensor-core route
ROUND_FLAGS = 0 if os.environ.get("MOA_B200_TENSOR_CORES") == "1" else MOA_FLAG_EXACT
DEVICES = ([int(d) for d in os.environ["MOA_B200_DEVICES"].split(",") if d.strip()]
           if os.environ.get("MOA_B200_DEVICES") else
           list(range(max(1, _lib.moa_device_count()))))


def _call(flags, res, a, b, noproc, rowsinred, elsinop, lstride, rstride, restride,
          combine_code, reduce_code, start, step):
    res = np.asarray(res)
    if res.dtype != np.float64 or not res.flags.c_contiguous or not res.flags.writeable:
        raise TypeError("res must be a writeable contiguous float64 buffer")
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    rc = _lib.moa_product_rows_host(MOA_DTYPE_F64, res.ctypes.data, a.ctypes.data, b.ctypes.data,
                                    noproc, rowsinred, elsinop, lstride, rstride, restride,
                                    combine_code, reduce_code, start, step,
                                    flags | ROUND_FLAGS, DEVICES[start % len(DEVICES)])
    if rc != 0:
        raise RuntimeError(_lib.moa_last_error().decode())


def product_rows(res, a, b, noproc, rowsinred, elsinop, lstride, rstride, restride,
                 combine_code, reduce_code, start, step):
    """Drop-in for _ckernel.product_rows (same arguments, float64 buffers):
    folds rows start::step INTO res."""
    _call(MOA_FLAG_ACCUMULATE, res, a, b, noproc, rowsinred, elsinop, lstride, rstride,
          restride, combine_code, reduce_code, start, step)


def product_rows_overwrite(res, a, b, noproc, rowsinred, elsinop, lstride, rstride, restride,
                           combine_code, reduce_code, start, step):
    """product_rows for an un-prefilled res: rows start::step are WRITTEN with
    the fold from the reduce identity (what prefill + product_rows gives)."""
    _call(0, res, a, b, noproc, rowsinred, elsinop, lstride, rstride, restride,
          combine_code, reduce_code, start, step)
