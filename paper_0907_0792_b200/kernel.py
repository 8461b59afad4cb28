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

import enum
import warnings
from dataclasses import dataclass

import numpy as np

from . import _native
from .arrays import MoaArray, Shape, as_shape, element_count
from .errors import PlanError, RankError, ShapeError
from .ops import MUL_ADD, OpPair

MAX_INDEX = 2**63 - 1

BACKENDS = ("cuda",)
DEFAULT_BACKEND = "cuda"
# names accepted for the native backend; "compiled" keeps reference call sites working
_BACKEND_ALIASES = {None: "cuda", "auto": "cuda", "cuda": "cuda", "compiled": "cuda"}


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
    if backend not in _BACKEND_ALIASES:
        raise ValueError(f"unknown backend {backend!r}; choose from {BACKENDS}")
    if ops.codes() is None:
        raise ValueError("the CUDA backend supports built-in op pairs only; "
                         "this OpPair carries custom callables")
    return _BACKEND_ALIASES[backend]


def _torch():
    import torch
    return torch


def result_dtype(a: MoaArray, b: MoaArray) -> np.dtype:
    """float32 only when both operands are float32 (the reference is float64)."""
    f32 = np.dtype(np.float32)
    return f32 if (a.dtype == f32 and b.dtype == f32) else np.dtype(np.float64)


def _native_dtype(dt: np.dtype) -> int:
    return _native.DTYPE_F32 if dt == np.dtype(np.float32) else _native.DTYPE_F64


def stage(x: MoaArray, device, dtype: np.dtype):
    """x's elements as a flat CUDA tensor of ``dtype`` on ``device`` (no copy if already so)."""
    torch = _torch()
    tdt = torch.float32 if dtype == np.dtype(np.float32) else torch.float64
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
    if stream is None:
        stream = torch.cuda.current_stream(res.device)
    flags = (_native.FLAG_EXACT if exact else 0) | (_native.FLAG_ACCUMULATE if accumulate else 0)
    dt = _native.DTYPE_F32 if res.dtype == torch.float32 else _native.DTYPE_F64
    _native.product_rows(dt, res.data_ptr(), a_dev.data_ptr(), b_dev.data_ptr(),
                         plan.noproc, plan.rowsinred, plan.elsinop,
                         plan.lstride, plan.rstride, plan.restride,
                         codes[0], codes[1], start, step, flags, stream.cuda_stream)


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
        tdt = torch.float32 if self.dtype == np.dtype(np.float32) else torch.float64
        self._res = torch.empty(plan.noproc * plan.elsinop, dtype=tdt, device=self.device)

    def run_rows(self, start: int, step: int) -> None:
        launch(self.plan, self._res, self._a, self._b, self.ops, start=start, step=step,
               exact=self.exact)

    def finish(self) -> MoaArray:
        torch = _torch()
        if not self.host_result:
            return MoaArray._wrap(self.plan.result_shape, self._res)
        out = torch.empty(self._res.numel(), dtype=self._res.dtype, pin_memory=True)
        out.copy_(self._res, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return MoaArray._wrap(self.plan.result_shape, out.numpy())


def execute_sequential(plan: KernelPlan, a: MoaArray, b: MoaArray, ops: OpPair = MUL_ADD,
                       *, backend: str | None = None, exact: bool = False) -> MoaArray:
    """Run the planned product over all result rows in one launch."""
    runner = _Runner(plan, a, b, ops, backend, exact=exact)
    runner.run_rows(0, 1)
    return runner.finish()
