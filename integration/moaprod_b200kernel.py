"""B200 backend module for the reference package (drop in as moaprod/_b200kernel.py).

``product_rows`` has the signature and the contract of the reference's
compiled loop ``_ckernel.product_rows`` (_ckernel.pyx:75-88): numpy float64
buffers, rows ``start, start+step, ...`` folded INTO ``res`` (which the
reference's ``_Runner`` prefilled with the reduce identity, kernel.py:149),
callable concurrently from ``execute_parallel``'s threads on disjoint row
sets of one ``res`` (parallel.py:26-43).  The fold runs on the GPU through
``moa_product_rows`` (include/moa_b200.h) with MOA_FLAG_ACCUMULATE; only the
caller's rows are written back, so concurrent callers never overwrite each
other's rows.

The library is found through $MOA_B200_LIB (default: the in-tree build).
Registration in the reference's _backend.py (:5-14) is two lines; see
INTEGRATION.md.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np
import torch

_DEFAULT = Path(__file__).resolve().parents[1] / "paper_0907_0792_b200" / "libmoa_b200.so"
_lib = ctypes.CDLL(os.environ.get("MOA_B200_LIB", str(_DEFAULT)))
_i64 = ctypes.c_int64
_lib.moa_product_rows.restype = ctypes.c_int
_lib.moa_product_rows.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  _i64, _i64, _i64, _i64, _i64, _i64,
                                  ctypes.c_int, ctypes.c_int, _i64, _i64,
                                  ctypes.c_uint32, ctypes.c_void_p]
_lib.moa_last_error.restype = ctypes.c_char_p
MOA_DTYPE_F64 = 0
MOA_FLAG_ACCUMULATE = 1


def product_rows(res, a, b, noproc, rowsinred, elsinop, lstride, rstride, restride,
                 combine_code, reduce_code, start, step):
    """Drop-in for _ckernel.product_rows (same arguments, float64 buffers)."""
    if start >= noproc or elsinop == 0:
        return
    dev = torch.device("cuda", torch.cuda.current_device())
    ta = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)
    tb = torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64)).to(dev)
    rows = np.arange(start, noproc, step, dtype=np.int64)
    idx = (rows[:, None] * restride + np.arange(elsinop, dtype=np.int64)).ravel()
    tr = torch.from_numpy(np.asarray(res)).to(dev)  # res holds the running fold
    stream = torch.cuda.current_stream(dev)
    rc = _lib.moa_product_rows(MOA_DTYPE_F64, tr.data_ptr(), ta.data_ptr(), tb.data_ptr(),
                               noproc, rowsinred, elsinop, lstride, rstride, restride,
                               combine_code, reduce_code, start, step,
                               MOA_FLAG_ACCUMULATE, stream.cuda_stream)
    if rc != 0:
        raise RuntimeError(_lib.moa_last_error().decode())
    host = tr.cpu().numpy()  # synchronises the stream
    res[idx] = host[idx]     # only this caller's rows
