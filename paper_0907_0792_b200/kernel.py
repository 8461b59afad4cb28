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


def native_dtype(dt) -> int:
    """ABI dtype code for a numpy or torch dtype."""
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

    Device operands: one launch.  Host operands of a large product: the rows
    are streamed in blocks (``_stream_chunks``) so the copy of A's next block
    and of C's previous block overlap the kernel; the bits are those of one
    launch because rows are independent.
    """
    if not (a.is_device or b.is_device):
        blocks = _stream_blocks(plan, result_dtype(a, b), ops)
        if len(blocks) > 1:
            _check_plan(plan, a, b)
            resolve_backend(backend, ops)
            return _execute_streamed(plan, a, b, ops, blocks, exact=exact)
    runner = _Runner(plan, a, b, ops, backend, exact=exact)
    runner.run_rows(0, 1)
    return runner.finish()


_STREAM_MIN_OUT_BYTES = 128 << 20
_WAVES_PER_CHUNK = 24  # >= 24 waves of CTAs per block keeps the tail wave small


_EDGE_MIN_WAVES = 6    # ... and >= 6 waves in each half-size end block


def edge_blocks(noproc: int, middle: int = 3, align: int = 128) -> list[range]:
    """Row blocks for streaming: a 3/16 first block, ``middle`` equal blocks,
    a 1/16 last block (sizes rounded to ``align`` rows).  The first block is
    computed k-chunk by k-chunk while B lands, so it must be long enough to
    cover B's transfer and the next block's A rows (B is 16% of c4's compute
    time at the measured host link); the last block's C rows are the copy no
    compute can hide, so it is small.  Middle blocks stay long enough that
    their partial last wave of CTAs costs little.  (A copy/compute timeline
    model over the BASELINE configs picked these fractions: c4 273 -> 260 ms
    against half-size end blocks.)"""
    from .parallel import row_blocks  # local: parallel imports this module
    first = noproc * 3 // 16
    first -= first % align
    last = noproc // 16
    last -= last % align
    if first <= 0 or last <= 0:
        return row_blocks(noproc, middle + 2)
    mid = noproc - first - last
    size = -(-mid // middle)
    size += -size % align
    bounds = [0] + [min(first + i * size, noproc - last) for i in range(middle)] + \
        [noproc - last, noproc]
    return [range(bounds[i], bounds[i + 1]) for i in range(len(bounds) - 1)
            if bounds[i + 1] > bounds[i]]


def _stream_blocks(plan: KernelPlan, dtype: np.dtype, ops: OpPair = MUL_ADD) -> list[range]:
    """Row blocks for the streamed host path (one block = do not stream)."""
    from .parallel import row_blocks  # local: parallel imports this module
    m = plan.noproc
    if plan.rowsinred < 2:  # outer products are pure D2H; blocks cannot hide it
        return [range(0, m)]
    out_bytes = m * plan.elsinop * np.dtype(dtype).itemsize
    if ops.codes() == (2, 0) and np.dtype(dtype) == np.dtype(np.float64):
        tiles, per_wave = -(-m // 64) * -(-plan.elsinop // 128), 296  # dmma.cu
    else:
        tiles, per_wave = -(-m // 128) * -(-plan.elsinop // 128), 296  # semiring.cu
    if out_bytes >= 8 * _STREAM_MIN_OUT_BYTES and tiles >= 8 * _EDGE_MIN_WAVES * per_wave:
        return edge_blocks(m)
    by_waves = tiles // (per_wave * _WAVES_PER_CHUNK)
    return row_blocks(m, int(max(1, min(8, out_bytes // _STREAM_MIN_OUT_BYTES, by_waves))))


def _execute_streamed(plan: KernelPlan, a: MoaArray, b: MoaArray, ops: OpPair, chunks,
                      *, exact: bool = False, device=None) -> MoaArray:
    """Host operands -> host result with copies overlapped with compute.

    For each row block: H2D of its A rows on a copy stream, the kernel on the
    compute stream, D2H of its C rows on a second copy stream, with two-deep
    device buffers.  Every row needs all of B, so a host B is copied in
    slab-aligned k-chunks behind the first block's A rows, and the first
    block is computed chunk by chunk as they land (later chunks accumulate,
    MOA_FLAG_ACCUMULATE; the same k order, so the same bits, whenever the fold
    is stored in its own type) — B's transfer then hides behind compute
    instead of preceding it.
    """
    from .distributed import k_chunks  # local: distributed imports this module
    from .parallel import row_blocks  # local: parallel imports this module
    torch = _torch()
    _native.load()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else \
        torch.device(device)
    dtype = result_dtype(a, b)
    tdt = torch_dtype(dtype)
    m, n, lda = plan.noproc, plan.elsinop, plan.lstride
    comp = torch.cuda.current_stream(dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    out = torch.empty(m * n, dtype=tdt, pin_memory=True)
    # chunks: a number of equal row blocks, or the blocks themselves
    blocks = [r for r in (row_blocks(m, chunks) if isinstance(chunks, int) else chunks) if len(r)]
    k = plan.rowsinred
    # k-chunks accumulate through the result buffer, so the fold must not be
    # carried in a wider type than it is stored in (float32 data folded in
    # float64: sums, products, and multiply/divide with min/max)
    wide = np.dtype(dtype) == np.float32 and (ops.reduce_name in ("add", "multiply") or
                                              ops.combine_name in ("multiply", "divide"))
    chunked = not b.is_device and not wide
    # the first block takes B in k-chunks as they land; with half-size end
    # blocks, eight chunks keep that block's per-chunk compute above the
    # per-chunk transfer while the first chunk (the exposed part) stays small
    b_chunks = k_chunks(k, 8 if len(blocks) >= 5 else len(blocks)) if chunked else [(0, k)]
    if not chunked:
        b_dev = stage(b, dev, dtype)
        b_ready = [None]
    else:
        b_dev = torch.empty(k * n, dtype=tdt, device=dev)
        host_b = b.data if b.data.dtype == dtype else b.data.astype(dtype)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)
            host_b_t = torch.from_numpy(host_b)
        b_ready = []
    rows_max = max(len(r) for r in blocks)
    a_buf = [torch.empty(rows_max * lda, dtype=tdt, device=dev) for _ in range(2)]
    c_buf = [torch.empty(rows_max * n, dtype=tdt, device=dev) for _ in range(2)]
    a_free = [None, None]
    c_free = [None, None]
    host_a = a.data if a.data.dtype == dtype else a.data.astype(dtype)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)
        host_a_t = torch.from_numpy(host_a)
    for idx, rows in enumerate(blocks):
        slot, r0, r1 = idx % 2, rows.start, rows.stop
        na, nc = (r1 - r0) * lda, (r1 - r0) * n
        with torch.cuda.stream(s_in):
            if a_free[slot] is not None:
                s_in.wait_event(a_free[slot])
            a_buf[slot][:na].copy_(host_a_t[r0 * lda:r1 * lda], non_blocking=True)
            a_ready = torch.cuda.Event()
            a_ready.record(s_in)
            if idx == 0 and chunked:  # B's k-chunks queue behind block 0's rows
                for k0, k1 in b_chunks:
                    b_dev[k0 * n:k1 * n].copy_(host_b_t[k0 * n:k1 * n], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(s_in)
                    b_ready.append(ev)
        comp.wait_event(a_ready)
        if c_free[slot] is not None:
            comp.wait_event(c_free[slot])
        if idx == 0:
            for j, (k0, k1) in enumerate(b_chunks):
                if b_ready[j] is not None:
                    comp.wait_event(b_ready[j])
                part = KernelPlan(plan.mode, r1 - r0, k1 - k0, n, lda, plan.rstride, plan.restride,
                                  plan.result_shape)
                launch(part, c_buf[slot][:nc], a_buf[slot][k0:na], b_dev[k0 * n:], ops,
                       exact=exact, accumulate=j > 0, stream=comp)
        else:
            sub = KernelPlan(plan.mode, r1 - r0, k, n, lda, plan.rstride, plan.restride,
                             plan.result_shape)
            launch(sub, c_buf[slot][:nc], a_buf[slot][:na], b_dev, ops, exact=exact, stream=comp)
        done = torch.cuda.Event()
        done.record(comp)
        a_free[slot] = done
        with torch.cuda.stream(s_out):
            s_out.wait_event(done)
            out[r0 * n:r1 * n].copy_(c_buf[slot][:nc], non_blocking=True)
            copied = torch.cuda.Event()
            copied.record(s_out)
            c_free[slot] = copied
    s_out.synchronize()
    comp.synchronize()
    return MoaArray._wrap(plan.result_shape, out.numpy())
