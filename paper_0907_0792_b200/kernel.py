"""Plans (the 2-D collapse of rho A and rho B) and the device runner.

Both products are the reference's single loop nest (kernel.py:3-11):

    res[i*restride + j] = reduce(res[i*restride + j],
                                 combine(a[l + i*lstride], b[l*rstride + j]))

A KernelPlan is exactly the reference's (kernel.py:36-52) and *is* the 2-D
view the GPU works on: C[noproc x elsinop] from A[noproc x rowsinred]
(row stride lstride) and B[rowsinred x elsinop] (row stride rstride).  The
outer product is the rowsinred = 1 case (kernel.py:95-108).

``_Runner`` replaces the reference's runner (kernel.py:138-170): it stages the
operands on the GPU, allocates the result WITHOUT an identity prefill (the
kernels start every fold from the identity in registers, which gives the same
bits), and ``run_rows(start, step)`` calls the C ABI for the rows
start, start+step, ... on the current CUDA stream.
"""

from __future__ import annotations

import ctypes
import enum
import warnings
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native
from .arrays import MoaArray, Shape, as_shape, element_count
from .errors import PlanError, RankError, ShapeError
from .ops import MUL_ADD, OpPair

MAX_INDEX = 2**63 - 1

# The CUDA library is this build's compiled backend, so it answers to the
# reference's name (_backend.py:12, BACKENDS ``("compiled", "python")``);
# "cuda" is accepted as an alias.  The reference's "python" backend is the
# pure-Python loop (_purekernel.py); this build has no CPU path, so asking for
# it raises ValueError, as the reference does for an unavailable backend
# (_backend.py:23-24).
BACKENDS = ("compiled",)
DEFAULT_BACKEND = "compiled"
_BACKEND_ALIASES = {None: "compiled", "auto": "compiled", "compiled": "compiled",
                    "cuda": "compiled"}


class ProductMode(enum.Enum):
    INNER = "inner"
    OUTER = "outer"


@dataclass(frozen=True)
class KernelPlan:
    """Loop bounds and flat strides of one product (same fields as the reference).

    noproc: result rows (M); rowsinred: contraction length (K); elsinop: result
    row length (N); lstride / rstride / restride: flat row strides of A, B, C.
    """

    mode: ProductMode
    noproc: int
    rowsinred: int
    elsinop: int
    lstride: int
    rstride: int
    restride: int
    result_shape: Shape


def _checked(plan: KernelPlan) -> KernelPlan:
    """Reject plans whose index products leave the 63-bit range (kernel.py:55-65)."""
    m, k, n = plan.noproc, plan.rowsinred, plan.elsinop
    if max(m * n, m * k, k * n, m, k, n) > MAX_INDEX:
        raise ShapeError(f"product of shapes {plan.result_shape} needs indices beyond "
                         f"the 63-bit range")
    return plan


def plan_inner(shape_a, shape_b) -> KernelPlan:
    """Contract the last axis of A with the first of B: result drop-last(A) ++ drop-first(B)."""
    sa, sb = as_shape(shape_a), as_shape(shape_b)
    if not sa or not sb:
        raise RankError("inner product needs operands of rank >= 1")
    if sa[-1] != sb[0]:
        raise ShapeError(f"contraction extents differ: last axis of A is {sa[-1]}, "
                         f"first axis of B is {sb[0]}")
    k = sa[-1]
    n = element_count(sb[1:])
    return _checked(KernelPlan(ProductMode.INNER, element_count(sa[:-1]), k, n,
                               k, n, n, sa[:-1] + sb[1:]))


def plan_outer(shape_a, shape_b) -> KernelPlan:
    """Pair every element of A with every element of B: result shape A ++ B."""
    sa, sb = as_shape(shape_a), as_shape(shape_b)
    n = element_count(sb)
    return _checked(KernelPlan(ProductMode.OUTER, element_count(sa), 1, n, 1, n, n, sa + sb))


def _check_plan(plan: KernelPlan, a: MoaArray, b: MoaArray) -> None:
    """Re-derive the plan from the operands; any difference is a PlanError."""
    planner = plan_inner if plan.mode is ProductMode.INNER else plan_outer
    try:
        expected = planner(a.shape, b.shape)
    except (ShapeError, RankError) as exc:
        raise PlanError(f"plan does not fit the operands: {exc}") from exc
    if expected != plan:
        raise PlanError(f"plan {plan} is inconsistent with operand shapes "
                        f"{a.shape} and {b.shape}")


def resolve_backend(backend: str | None, ops: OpPair) -> str:
    """Map a backend name to the native backend; custom callables are refused.

    The reference falls back to pure Python for OpPairs of arbitrary callables
    (kernel.py:126-135).  This build has no CPU path, so such pairs raise
    ValueError — the same error the reference gives when the compiled backend
    is requested explicitly.
    """
    if backend == "python":
        raise ValueError("python backend requested but this build has no CPU path "
                         "(the products run on the CUDA backend only)")
    if backend not in _BACKEND_ALIASES:
        raise ValueError(f"unknown backend {backend!r}; choose from {BACKENDS}")
    if ops.codes() is None:
        raise ValueError("the CUDA backend supports built-in op pairs only; "
                         "this OpPair carries custom callables")
    return _BACKEND_ALIASES[backend]


def _torch():
    import torch
    return torch


_F32, _F64 = np.dtype(np.float32), np.dtype(np.float64)
_I32, _I64 = np.dtype(np.int32), np.dtype(np.int64)


def result_dtype(a: MoaArray, b: MoaArray) -> np.dtype:
    """Element type of a product.

    float64 unless both operands are float32 (-> float32) or both are integers
    (-> int64 if either is int64, else int32).  Mixing floats and integers
    computes in float64, as the reference does for everything."""
    da, db = a.dtype, b.dtype
    if da == db:
        return da
    ints = (_I32, _I64)
    if da in ints and db in ints:
        return _I64
    return _F64


_NP_CODES = {_F64: _native.DTYPE_F64, _F32: _native.DTYPE_F32, _I32: _native.DTYPE_I32,
             _I64: _native.DTYPE_I64}


def native_dtype(dt) -> int:
    """ABI dtype code for a numpy or torch dtype."""
    code = _NP_CODES.get(dt) if isinstance(dt, np.dtype) else None
    if code is not None:
        return code
    name = str(dt).replace("torch.", "")
    return {"float64": _native.DTYPE_F64, "float32": _native.DTYPE_F32,
            "int32": _native.DTYPE_I32, "int64": _native.DTYPE_I64}[name]


def torch_dtype(dt: np.dtype):
    torch = _torch()
    return {_F64: torch.float64, _F32: torch.float32, _I32: torch.int32,
            _I64: torch.int64}[np.dtype(dt)]


def stage(x: MoaArray, device, dtype: np.dtype):
    """x's elements as a flat CUDA tensor of ``dtype`` on ``device`` (no copy if already so)."""
    tdt = torch_dtype(dtype)
    if x.is_device:
        t = x.data
        if t.device != device or t.dtype != tdt:
            t = t.to(device=device, dtype=tdt, non_blocking=True)
        return t
    return stage_host(x.data, device, dtype)


def stage_host(host: np.ndarray, device, dtype: np.dtype):
    """Copy a flat host vector to ``device`` as ``dtype`` (async if it is pinned)."""
    torch = _torch()
    if host.dtype != dtype:
        host = host.astype(dtype)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)  # frozen arrays are read only
        t = torch.from_numpy(host)
    return t.to(device=device, non_blocking=True)


def launch(plan: KernelPlan, res, a_dev, b_dev, ops: OpPair, *, start: int = 0,
           step: int = 1, exact: bool = False, accumulate: bool = False, stream=None) -> None:
    """One moa_product_rows call on device tensors (no validation beyond dtypes).

    res, a_dev, b_dev: flat CUDA tensors of one dtype on one device.  The call
    is asynchronous on ``stream`` (default: the current stream of res's device).
    """
    torch = _torch()
    if not (res.dtype == a_dev.dtype == b_dev.dtype):
        raise TypeError("operands and result must share one dtype")
    codes = ops.codes()
    if codes is None:
        raise ValueError("custom OpPair callables have no device implementation")
    _check_extents(plan, res, a_dev, b_dev, start, step)
    if stream is None:
        stream = torch.cuda.current_stream(res.device)
    flags = (_native.FLAG_EXACT if exact else 0) | (_native.FLAG_ACCUMULATE if accumulate else 0)
    _native.product_rows(native_dtype(res.dtype), res.data_ptr(), a_dev.data_ptr(), b_dev.data_ptr(),
                         plan.noproc, plan.rowsinred, plan.elsinop,
                         plan.lstride, plan.rstride, plan.restride,
                         codes[0], codes[1], start, step, flags, stream.cuda_stream)


def _check_extents(plan: KernelPlan, res, a_dev, b_dev, start: int, step: int) -> None:
    """The kernels index raw pointers: refuse tensors that are not flat,
    contiguous, on one CUDA device, and long enough for the rows addressed."""
    for name, t in (("res", res), ("a", a_dev), ("b", b_dev)):
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous CUDA tensor")
    if not (res.device == a_dev.device == b_dev.device):
        raise ValueError("res, a and b must be on one device")
    if step < 1 or start < 0 or start >= plan.noproc or plan.elsinop == 0:
        return  # nothing is touched (the C ABI rejects step < 1 / start < 0)
    last = start + (plan.noproc - 1 - start) // step * step
    need = {"res": last * plan.restride + plan.elsinop}
    if plan.rowsinred:
        need["a"] = last * plan.lstride + plan.rowsinred
        need["b"] = (plan.rowsinred - 1) * plan.rstride + plan.elsinop
    have = {"res": res.numel(), "a": a_dev.numel(), "b": b_dev.numel()}
    for name, n in need.items():
        if have[name] < n:
            raise ValueError(f"{name} holds {have[name]} elements; the plan addresses {n}")


def launch_host(plan: KernelPlan, res: np.ndarray, a: np.ndarray, b: np.ndarray, ops: OpPair,
                *, start: int = 0, step: int = 1, exact: bool = False,
                accumulate: bool = False, device: int | None = None) -> None:
    """One moa_product_rows_host call on flat HOST numpy buffers — the
    reference's ``product_rows(res, a, b, ...)`` contract (_ckernel.pyx:75-88)
    with the product on ``device``.  Writes rows start::step of ``res`` (folds
    into them with ``accumulate``) and returns when they hold the result."""
    if not (res.dtype == a.dtype == b.dtype):
        raise TypeError("operands and result must share one dtype")
    for name, x in (("res", res), ("a", a), ("b", b)):
        if x.ndim != 1 or not x.flags.c_contiguous:
            raise ValueError(f"{name} must be a flat contiguous array")
    if not res.flags.writeable:
        raise ValueError("res must be writeable")
    codes = ops.codes()
    if codes is None:
        raise ValueError("custom OpPair callables have no device implementation")
    if step >= 1 and 0 <= start < plan.noproc and plan.elsinop:
        last = start + (plan.noproc - 1 - start) // step * step
        need = {"res": last * plan.restride + plan.elsinop}
        if plan.rowsinred:
            need["a"] = last * plan.lstride + plan.rowsinred
            need["b"] = (plan.rowsinred - 1) * plan.rstride + plan.elsinop
        for name, n in need.items():
            have = {"res": res, "a": a, "b": b}[name].size
            if have < n:
                raise ValueError(f"{name} holds {have} elements; the plan addresses {n}")
    if device is None:
        device = _torch().cuda.current_device()
    flags = (_native.FLAG_EXACT if exact else 0) | (_native.FLAG_ACCUMULATE if accumulate else 0)
    _native.product_rows_host(native_dtype(res.dtype), res.ctypes.data, a.ctypes.data,
                              b.ctypes.data, plan.noproc, plan.rowsinred, plan.elsinop,
                              plan.lstride, plan.rstride, plan.restride, codes[0], codes[1],
                              start, step, flags, int(device))


class _Runner:
    """One planned product on one GPU, ready to run row sets into one result."""

    def __init__(self, plan: KernelPlan, a: MoaArray, b: MoaArray, ops: OpPair,
                 backend: str | None = None, *, exact: bool = False, device=None):
        _check_plan(plan, a, b)
        self.backend = resolve_backend(backend, ops)
        _native.load()  # fail loudly before touching CUDA
        torch = _torch()
        self.plan, self.ops, self.exact = plan, ops, exact
        self.dtype = result_dtype(a, b)
        self.host_result = not (a.is_device or b.is_device)
        if device is None:
            device = (a.data.device if a.is_device else b.data.device if b.is_device
                      else torch.device("cuda", torch.cuda.current_device()))
        self.device = torch.device(device)
        self._a = stage(a, self.device, self.dtype)
        self._b = stage(b, self.device, self.dtype)
        tdt = torch_dtype(self.dtype)
        self._res = torch.empty(plan.noproc * plan.elsinop, dtype=tdt, device=self.device)

    def run_rows(self, start: int, step: int) -> None:
        launch(self.plan, self._res, self._a, self._b, self.ops, start=start, step=step,
               exact=self.exact)

    def finish(self) -> MoaArray:
        torch = _torch()
        if not self.host_result:
            return MoaArray._wrap(self.plan.result_shape, self._res)
        out = torch.empty(self._res.numel(), dtype=self._res.dtype, pin_memory=True)
        d2h_split(out, self._res, torch.cuda.current_stream(self.device))
        return MoaArray._wrap(self.plan.result_shape, out.numpy())


_D2H_SPLIT_BYTES = 64 << 20


def d2h_split(dst, src, stream, parts: int = 4) -> None:
    """Copy device ``src`` into pinned ``dst`` and wait for it.

    Large results are split over ``parts`` streams: several copy-engine queues
    draw a little more of the host link than one (tools/e2e_probe.py:
    54.8 -> 56.9 GB/s on B200)."""
    torch = _torch()
    nbytes = src.numel() * src.element_size()
    if nbytes < _D2H_SPLIT_BYTES:
        with torch.cuda.stream(stream):
            dst.copy_(src, non_blocking=True)
        stream.synchronize()
        return
    n = src.numel()
    step = -(-n // parts)
    streams = [torch.cuda.Stream(src.device) for _ in range(parts)]
    for i, s in enumerate(streams):
        s.wait_stream(stream)
        with torch.cuda.stream(s):
            dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)
    for s in streams:
        s.synchronize()


def execute_sequential(plan: KernelPlan, a: MoaArray, b: MoaArray, ops: OpPair = MUL_ADD,
                       *, backend: str | None = None, exact: bool = False) -> MoaArray:
    """Run the planned product over all result rows.

    Device operands: one launch.  Host operands: the native executor
    (``execute_host``), which streams large products in row blocks so the
    copies overlap the kernels; the bits are those of one launch because rows
    are independent.
    """
    if not (a.is_device or b.is_device):
        _check_plan(plan, a, b)
        resolve_backend(backend, ops)
        return execute_host(plan, a, b, ops, exact=exact)
    runner = _Runner(plan, a, b, ops, backend, exact=exact)
    runner.run_rows(0, 1)
    return runner.finish()


_HUGE_PAGE = 2 << 20
_PINNED_RESULT_BYTES = 256 << 10  # host_runtime.cu kDirectBytes
_TRACE = bool(__import__("os").environ.get("MOA_HOST_TRACE"))


def host_empty(n: int, dtype) -> np.ndarray:
    """Uninitialised host memory for a result of ``n`` elements.

    Large results come from the library's host block cache
    (``moa_host_alloc``): huge-page-backed, first-touched by its copy threads
    and page-locked with cudaHostRegister (~40 ms per GiB the first time,
    against 0.39 s per GiB for cudaHostAlloc on a B200 host,
    profiles/r02_host_probe.json), so the result's copy-back runs at link
    speed; when the array is garbage-collected the block returns to the cache
    and the next result of a similar size reuses it.  Results from 256 KiB up
    take such a block too (one 2 MiB page at least): below that the executor
    copies pageable memory directly, above it a pageable result would be
    staged through its copy threads, while a page-locked one of <= 1 MiB is
    written by the kernel itself (csrc/host_exec.cu direct_out_bytes).
    Smaller results are plain numpy memory."""
    dt = np.dtype(dtype)
    nbytes = n * dt.itemsize
    if nbytes < _PINNED_RESULT_BYTES:
        return np.empty(n, dt)
    ptr = _native.host_alloc(nbytes)
    if not ptr:  # pragma: no cover - host out of memory
        return np.empty(n, dt)
    buf = (ctypes.c_char * nbytes).from_address(ptr)
    weakref.finalize(buf, _native.host_free, ptr)
    return np.frombuffer(buf, dtype=dt, count=n)


def execute_host(plan: KernelPlan, a: MoaArray, b: MoaArray, ops: OpPair = MUL_ADD, *,
                 exact: bool = False, device=None) -> MoaArray:
    """Host operands -> host result through the native executor
    (moa_product_rows_host, csrc/host_exec.cu): A, B and the result move with
    2-D copies — page-locked buffers directly, pageable ones (plain numpy)
    staged through page-locked slots by the executor's copy threads — and
    large products stream in row blocks with the copies overlapping the
    kernels (B in k-chunks behind the first block).  The result is ordinary
    pageable memory (``host_empty``)."""
    import time as _time
    t0 = _time.perf_counter()
    torch = _torch()
    _native.load()
    dtype = result_dtype(a, b)
    host_a = np.ascontiguousarray(a.data if a.data.dtype == dtype else a.data.astype(dtype)).ravel()
    host_b = np.ascontiguousarray(b.data if b.data.dtype == dtype else b.data.astype(dtype)).ravel()
    t1 = _time.perf_counter()
    out = host_empty(plan.noproc * plan.elsinop, dtype)
    t2 = _time.perf_counter()
    dev = torch.cuda.current_device() if device is None else torch.device(device).index
    launch_host(plan, out, host_a, host_b, ops, exact=exact, device=dev)
    t3 = _time.perf_counter()
    res = MoaArray._wrap(plan.result_shape, out)
    if _TRACE:
        import sys as _sys
        print(f"[execute_host] operands={1e3 * (t1 - t0):.3f} alloc={1e3 * (t2 - t1):.3f} "
              f"call={1e3 * (t3 - t2):.3f} wrap={1e3 * (_time.perf_counter() - t3):.3f} ms",
              file=_sys.stderr)
    return res
