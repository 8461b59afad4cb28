"""The paper's BLAS comparator, as the vendor FP64 GEMM.

Same interface as the reference's ``moaprod.gemm`` (gemm.py:23-98):
``GemmParams`` (alpha, beta, m, n, k with the same validation),
``gemm_baseline(params, a, b, c)`` = alpha*A*B + beta*C on row-major arrays
(C is left unchanged), and the column-major helpers.  The reference ports the
paper's dgemm.f column loop; on B200 the comparator that
matters is cuBLAS DGEMM, so the product runs as ``torch.addmm`` on float64 CUDA
tensors (beta = 0 ignores C, as dgemm does).  ``workers`` is accepted for
signature parity; the result does not depend on it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .arrays import MoaArray
from .errors import ShapeError


@dataclass(frozen=True)
class GemmParams:
    """Scaling factors and dimensions: C is m x n, A is m x k, B is k x n."""

    alpha: float
    beta: float
    m: int
    n: int
    k: int

    def __post_init__(self):
        for name in ("m", "n", "k"):
            v = getattr(self, name)
            if v < 1:
                raise ShapeError(f"dimension {name} must be >= 1, got {v}")


def to_colmajor(a: MoaArray, rows: int, cols: int) -> np.ndarray:
    """Flat column-major copy of a rows x cols row-major array."""
    if a.shape != (rows, cols):
        raise ShapeError(f"expected shape ({rows}, {cols}), got {a.shape}")
    return np.ascontiguousarray(a.host_data().reshape(rows, cols).T).ravel().copy()


def from_colmajor(flat: np.ndarray, rows: int, cols: int) -> MoaArray:
    """Row-major array from a flat column-major buffer."""
    return MoaArray._wrap((rows, cols), np.ascontiguousarray(flat.reshape(cols, rows).T).ravel())


def _device_gemm(params: GemmParams, a_rm, b_rm, c_rm):
    """alpha * A @ B + beta * C on the current CUDA device (row-major 2-D tensors)."""
    import torch
    if params.beta == 0.0:
        out = torch.mm(a_rm, b_rm)
        return out if params.alpha == 1.0 else out.mul_(params.alpha)
    return torch.addmm(c_rm, a_rm, b_rm, beta=params.beta, alpha=params.alpha)


def run_colmajor(params: GemmParams, a_cm: np.ndarray, b_cm: np.ndarray, c_cm: np.ndarray,
                 workers: int = 1, *, backend: str | None = None) -> None:
    """C = alpha*A*B + beta*C in place on flat column-major float64 buffers."""
    import torch
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    m, n, k = params.m, params.n, params.k
    dev = torch.device("cuda")
    a = torch.from_numpy(np.asarray(a_cm, dtype=np.float64)).to(dev).view(k, m).t()
    b = torch.from_numpy(np.asarray(b_cm, dtype=np.float64)).to(dev).view(n, k).t()
    c = torch.from_numpy(np.asarray(c_cm, dtype=np.float64)).to(dev).view(n, m).t()
    out = _device_gemm(params, a, b, c)
    c_cm[:] = out.t().contiguous().view(-1).cpu().numpy()


def gemm_baseline(params: GemmParams, a: MoaArray, b: MoaArray, c: MoaArray, *,
                  workers: int = 1, backend: str | None = None) -> MoaArray:
    """alpha*A*B + beta*C on row-major arrays; returns a new array (c unchanged).

    Host operands take the same path as the MoA products (kernel.stage_host
    in, pinned result out through kernel.d2h_split), and C is not read when
    beta == 0 (as dgemm), so the harness compares like with like."""
    import torch

    from .kernel import d2h_split, stage_host
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    m, n, k = params.m, params.n, params.k
    for arr, shape, name in ((a, (m, k), "A"), (b, (k, n), "B"), (c, (m, n), "C")):
        if arr.shape != shape:
            raise ShapeError(f"{name}: expected shape {shape}, got {arr.shape}")
    dev = torch.device("cuda", torch.cuda.current_device())
    f64 = np.dtype(np.float64)

    def dev2d(x: MoaArray, r: int, cc: int):
        t = x.data.to(device=dev, dtype=torch.float64) if x.is_device else stage_host(x.data, dev, f64)
        return t.view(r, cc)

    c_dev = dev2d(c, m, n) if params.beta != 0.0 else None
    out = _device_gemm(params, dev2d(a, m, k), dev2d(b, k, n), c_dev)
    flat = out.contiguous().view(-1)
    if a.is_device or b.is_device or c.is_device:
        return MoaArray._wrap((m, n), flat)
    host = torch.empty(flat.numel(), dtype=torch.float64, pin_memory=True)
    d2h_split(host, flat, torch.cuda.current_stream(dev))
    return MoaArray._wrap((m, n), host.numpy())
