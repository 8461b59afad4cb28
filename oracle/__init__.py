"""TEST INFRASTRUCTURE — the CPU checkers for the MoA generalized product.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and the
``--impl reference`` arm) may import this package; the product path never does
(tests/test_boundary.py enforces it).  Three checkers, each pinned to the
reference:

* ``port``: moa_oracle.c, a plain-C restatement of _ckernel.product_rows
  (_ckernel.pyx:37-88) and of parallel.execute_parallel (parallel.py:26-43),
  built by Makefile into _build/.  Bit-identical to the reference; pinned by
  tests/test_oracle_pins.py against tests/golden/ (vectors the reference
  itself produced, tests/golden/make_golden.py).
* ``ref``: the reference's own compiled hot loop, _ref/_ckernel*.so, built by
  Makefile from /root/reference/pkg/src/moaprod/_ckernel.pyx with the
  reference's flags.  Used as the CPU baseline when present.
* ``odometer_inner`` / ``odometer_outer``: pure-Python restatements of the
  reference's naive oracle (oracle.py:17-72) for tiny cases.
"""

from __future__ import annotations

import ctypes
import os
import shutil
import subprocess
import sys
import threading
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ORACLE_DIR = Path(__file__).resolve().parent
PORT_LIB = ORACLE_DIR / "_build" / "libmoa_oracle.so"
REF_DIR = ORACLE_DIR / "_ref"
REFERENCE_PYX = Path("/root/reference/pkg/src/moaprod/_ckernel.pyx")

_lock = threading.Lock()
_port = None
_ref = None


def build(ref: bool | None = None) -> None:
    """make the C port (and the reference kernel when its source is present)."""
    targets = ["oracle"]
    if ref is None:
        ref = REFERENCE_PYX.exists() and shutil.which("cython") is not None
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), f"PYTHON={sys.executable}", *targets],
                   check=True)


def port() -> ctypes.CDLL:
    global _port
    with _lock:
        if _port is None:
            if not PORT_LIB.exists():
                build(ref=False)
            lib = ctypes.CDLL(str(PORT_LIB))
            i64, vp = ctypes.c_int64, ctypes.c_void_p
            lib.oracle_product_rows.argtypes = [vp, vp, vp] + [i64] * 6 + [ctypes.c_int] * 2 + [i64] * 2
            lib.oracle_product_rows.restype = None
            lib.oracle_product_rows_f32in.argtypes = lib.oracle_product_rows.argtypes
            lib.oracle_product_rows_f32in.restype = None
            lib.oracle_product_parallel.argtypes = [vp, vp, vp, ctypes.c_int] + [i64] * 6 + \
                [ctypes.c_int] * 3
            lib.oracle_product_parallel.restype = ctypes.c_int
            _port = lib
    return _port


def ref_kernel():
    """The reference's compiled product_rows module, or None if not built here."""
    global _ref
    with _lock:
        if _ref is None:
            if not any(REF_DIR.glob("_ckernel*.so")):
                return None
            sys.path.insert(0, str(REF_DIR))
            try:
                import _ckernel  # noqa: PLC0415
            finally:
                sys.path.remove(str(REF_DIR))
            _ref = _ckernel
    return _ref


def _ptr(x: np.ndarray) -> int:
    return x.ctypes.data


def identity(reduce_code: int) -> float:
    return (0.0, 1.0, float("inf"), float("-inf"))[reduce_code]


def product(a: np.ndarray, b: np.ndarray, M: int, K: int, N: int, comb: int, red: int, *,
            lda: int | None = None, ldb: int | None = None, workers: int = 1,
            res: np.ndarray | None = None) -> np.ndarray:
    """C[M x N] (float64) of the unified loop, via the C port.

    a, b: flat float64 or float32 arrays (float32 is upcast like the reference);
    ``res`` (float64, length M*N) is accumulated into if given, else a fresh
    identity-filled buffer is used (kernel.py:149).
    """
    lda = K if lda is None else lda
    ldb = N if ldb is None else ldb
    # integer operands are upcast like the reference does (arrays.py:77-78)
    if a.dtype.kind in "iu":
        a = a.astype(np.float64)
    if b.dtype.kind in "iu":
        b = b.astype(np.float64)
    f32 = a.dtype == np.float32
    if (b.dtype == np.float32) != f32:
        a, b = a.astype(np.float64), b.astype(np.float64)
        f32 = False
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if res is None:
        res = np.full(M * N, identity(red), dtype=np.float64)
    lib = port()
    if workers == 1:
        fn = lib.oracle_product_rows_f32in if f32 else lib.oracle_product_rows
        fn(_ptr(res), _ptr(a), _ptr(b), M, K, N, lda, ldb, N, comb, red, 0, 1)
    else:
        rc = lib.oracle_product_parallel(_ptr(res), _ptr(a), _ptr(b), int(f32), M, K, N, lda,
                                         ldb, N, comb, red, workers)
        if rc != 0:
            raise RuntimeError(f"oracle_product_parallel failed: {rc}")
    return res


def reference_product(a: np.ndarray, b: np.ndarray, M: int, K: int, N: int, comb: int,
                      red: int, *, workers: int = 1) -> np.ndarray:
    """The same product through the reference's own compiled loop (oracle/_ref).

    Driven the way the reference's execute_parallel drives it
    (parallel.py:37-43): one identity-filled buffer, ``workers`` threads, worker
    k calling product_rows(..., start=k, step=workers).
    """
    ck = ref_kernel()
    if ck is None:
        raise RuntimeError("reference kernel not built (oracle/_ref); run `make -C oracle ref`")
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    res = np.full(M * N, identity(red), dtype=np.float64)
    args = (res, a, b, M, K, N, K, N, N, comb, red)
    if workers == 1:
        ck.product_rows(*args, 0, 1)
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            for f in [pool.submit(ck.product_rows, *args, k, workers) for k in range(workers)]:
                f.result()
    return res


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


# ---- naive odometer oracle (oracle.py:17-72), tiny cases only -----------------

def _odometer(shape):
    if any(e == 0 for e in shape):
        return
    idx = [0] * len(shape)
    while True:
        yield tuple(idx)
        for axis in range(len(shape) - 1, -1, -1):
            idx[axis] += 1
            if idx[axis] < shape[axis]:
                break
            idx[axis] = 0
        else:
            return


def _offset(idx, shape):
    off = 0
    for i, e in zip(idx, shape):
        off = off * e + i
    return off


_COMB = [lambda x, y: x + y, lambda x, y: x - y, lambda x, y: x * y, None,
         lambda x, y: x if x < y else y, lambda x, y: x if x > y else y]
_RED = [lambda x, y: x + y, lambda x, y: x * y, lambda x, y: x if x < y else y,
        lambda x, y: x if x > y else y]


def _div(x, y):
    with np.errstate(all="ignore"):
        return float(np.float64(x) / np.float64(y))


_COMB[3] = _div


def odometer_inner(a, shape_a, b, shape_b, comb: int, red: int) -> np.ndarray:
    """result[u, v] = fold_p reduce(identity, combine(a[u, p], b[p, v])), p ascending."""
    u_shape, v_shape, p_ext = tuple(shape_a[:-1]), tuple(shape_b[1:]), shape_a[-1]
    out = []
    for u in _odometer(u_shape):
        for v in _odometer(v_shape):
            acc = identity(red)
            for p in range(p_ext):
                x = float(a[_offset(u + (p,), shape_a)])
                y = float(b[_offset((p,) + v, shape_b)])
                acc = _RED[red](acc, _COMB[comb](x, y))
            out.append(acc)
    return np.array(out, dtype=np.float64)


def odometer_outer(a, shape_a, b, shape_b, comb: int) -> np.ndarray:
    """result[u ++ v] = combine(a[u], b[v]) (the reference oracle applies no reduce)."""
    out = [_COMB[comb](float(a[_offset(u, shape_a)]), float(b[_offset(v, shape_b)]))
           for u in _odometer(tuple(shape_a)) for v in _odometer(tuple(shape_b))]
    return np.array(out, dtype=np.float64)
