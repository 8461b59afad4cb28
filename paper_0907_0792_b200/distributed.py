"""One process per GPU: row-sharded products with one broadcast of B.

This is the multi-GPU form of the reference's fork-join over result rows
(parallel.py:19-43): rank r of a ``torch.distributed`` group owns the
contiguous block of result rows ``row_block(noproc, world, r)`` and the
matching rows of A.  The only exchange the path has is B, which every row
needs: rank 0 holds it and one ``broadcast`` (NCCL over NVLink/NVSwitch on
B200, gloo on CPU) gives every rank a copy.  No reduction follows, because
rows are independent; result blocks stay on their GPU unless ``gather_rows``
is asked for them.

The per-rank compute is ``row_kernel(plan_block, c_block, a_block, b, ops)``,
by default the CUDA backend (``kernel.launch``).  The injection point exists
so the host logic (partitioning, broadcast, gather) can be tested with gloo on
CPU; it is not a fallback — the default has no CPU path.
"""

from __future__ import annotations

from typing import Callable

import numpy as np

from .kernel import KernelPlan, d2h_split, launch
from .ops import MUL_ADD, OpPair


def _torch():
    import torch
    return torch


def _dist():
    import torch.distributed as dist
    return dist


def row_block(noproc: int, world: int, rank: int) -> tuple[int, int]:
    """[r0, r1) rows owned by ``rank``: ceil-sized contiguous blocks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    size = -(-noproc // world) if noproc else 0
    return min(rank * size, noproc), min((rank + 1) * size, noproc)


def block_plan(plan: KernelPlan, r0: int, r1: int) -> KernelPlan:
    """The plan of rows [r0, r1) of ``plan`` as a stand-alone product."""
    return KernelPlan(plan.mode, r1 - r0, plan.rowsinred, plan.elsinop, plan.lstride,
                      plan.rstride, plan.restride, plan.result_shape)


def broadcast_operand(b, plan: KernelPlan, *, src: int = 0, group=None, device=None,
                      dtype=None):
    """B (rowsinred x elsinop, flat) on every rank; ``b`` is only read on ``src``.

    Every rank must post the same byte count, so ``src`` sends B in ``dtype``
    (the dtype the other ranks allocate), casting if ``b`` differs, and checks
    B's length against the plan before the collective."""
    torch, dist = _torch(), _dist()
    n = plan.rowsinred * plan.elsinop
    if dist.get_rank(group) == src:
        buf = b.reshape(-1)
        if buf.numel() != n:
            raise ValueError(f"B holds {buf.numel()} elements; the plan needs {n}")
        buf = buf.to(device=device if device is not None else buf.device,
                     dtype=dtype if dtype is not None else buf.dtype)
        buf = buf.contiguous()
    else:
        buf = torch.empty(n, dtype=dtype if dtype is not None else b.dtype,
                          device=device if device is not None else "cpu")
    dist.broadcast(buf, src=src, group=group)
    return buf


def _cuda_rows(plan: KernelPlan, c, a, b, ops: OpPair, exact: bool = False) -> None:
    launch(plan, c, a, b, ops, exact=exact)


def k_chunks(K: int, chunks: int, align: int = 16) -> list[tuple[int, int]]:
    """Split [0, K) into up to ``chunks`` ranges whose inner boundaries are
    multiples of ``align`` (the DMMA kernel's k-slab), so accumulating the
    chunks replays exactly the DMMA sequence of one pass."""
    if chunks <= 1 or K <= align:
        return [(0, K)]
    step = -(-K // chunks)
    step = -(-step // align) * align
    out = [(k0, min(K, k0 + step)) for k0 in range(0, K, step)]
    if len(out) > 1 and out[-1][1] - out[-1][0] < align:
        # a short tail joins the previous chunk: every chunk keeps >= align
        # k-steps, so its kernel route is the whole product's (capi.cu route())
        out[-2:] = [(out[-2][0], K)]
    return out


# (combine, reduce) codes whose fold replays exactly when split into k-chunks
# accumulated into C: min/max of sums or differences — the fold is one
# compare-select chain either way, C holds the running value exactly (no
# float32 rounding can move it: a nonzero sum of two floats never rounds to
# zero, and rounding is monotone), and the fast tropical loops seed from C
_CHUNKABLE_FOLDS = {(0, 2), (0, 3), (1, 2), (1, 3)}


def bcast_chunk_align(ops: OpPair, dtype) -> int | None:
    """k alignment of the chunks for a pipelined broadcast of B, or None when
    chunked accumulation would not reproduce one pass bit for bit."""
    torch = _torch()
    codes = ops.codes()
    if codes == (2, 0):
        return 16 if dtype == torch.float64 else None  # the DMMA k-slab (f64 DMMA route only)
    if codes in _CHUNKABLE_FOLDS and dtype in (torch.float32, torch.float64, torch.int32,
                                               torch.int64):
        return 32  # the tropical / semiring k-slab
    return None


def sharded_product(plan: KernelPlan, a_block, b, ops: OpPair = MUL_ADD, *, group=None,
                    src: int = 0, exact: bool = False, out=None,
                    row_kernel: Callable | None = None, bcast_chunks: int = 1):
    """This rank's result block of ``plan``.

    a_block: this rank's rows of A (flat, rows row_block(...)), on this rank's
    device; b: the full B on rank ``src`` (ignored elsewhere).  Returns the flat
    result block (rows r0..r1 of C) on the same device as a_block.

    ``bcast_chunks > 1`` pipelines the broadcast of B with the compute for
    (multiply, add) on float64 and for (add|subtract, min|max): B is broadcast
    in k-chunks (asynchronously, in order) and the kernel for chunk i runs as
    soon as chunk i has arrived, accumulating into C (MOA_FLAG_ACCUMULATE)
    while later chunks are still on the wire.  Chunk boundaries are multiples
    of the kernels' k-slab, and those folds replay exactly under chunked
    accumulation (``bcast_chunk_align``), so the result is bitwise identical
    to one pass; other pairs broadcast B whole.
    """
    torch, dist = _torch(), _dist()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    r0, r1 = row_block(plan.noproc, world, rank)
    sub = block_plan(plan, r0, r1)
    if a_block.numel() != (r1 - r0) * plan.lstride:
        raise ValueError(f"rank {rank} owns rows [{r0}, {r1}) = {(r1 - r0) * plan.lstride} "
                         f"A elements, got {a_block.numel()}")
    c = out if out is not None else torch.empty(sub.noproc * sub.elsinop,
                                                dtype=a_block.dtype, device=a_block.device)
    align = bcast_chunk_align(ops, a_block.dtype)
    pipelined = (bcast_chunks > 1 and row_kernel is None and align is not None
                 and not (exact and ops.codes() == (2, 0)))
    if not pipelined:
        b_all = broadcast_operand(b, plan, src=src, group=group, device=a_block.device,
                                  dtype=a_block.dtype)
        if sub.noproc:
            (row_kernel or (lambda p, c_, a_, b_, o: _cuda_rows(p, c_, a_, b_, o, exact)))(
                sub, c, a_block, b_all, ops)
        return c
    # pipelined: async, in-order broadcasts of B's k-chunks; compute chases them
    n, k = plan.elsinop, plan.rowsinred
    b_all = torch.empty(k * n, dtype=a_block.dtype, device=a_block.device)
    b_src = None
    if rank == src:
        b_src = b.reshape(-1)
        if b_src.numel() != k * n:
            raise ValueError(f"B holds {b_src.numel()} elements; the plan needs {k * n}")
    chunks = k_chunks(k, bcast_chunks, align)
    works = []
    for k0, k1 in chunks:
        if b_src is not None:
            # src stages chunk by chunk (from host memory too), in A's dtype so
            # every rank's broadcast of the chunk posts equal byte counts
            b_all[k0 * n:k1 * n].copy_(b_src[k0 * n:k1 * n], non_blocking=True)
        works.append(dist.broadcast(b_all[k0 * n:k1 * n], src=src, group=group, async_op=True))
    for i, ((k0, k1), work) in enumerate(zip(chunks, works)):
        work.wait()  # the current stream waits for this chunk only
        if sub.noproc:
            part = KernelPlan(plan.mode, sub.noproc, k1 - k0, n, plan.lstride, plan.rstride,
                              plan.restride, plan.result_shape)
            launch(part, c, a_block[k0:], b_all[k0 * n:], ops, exact=exact, accumulate=i > 0)
    return c


def gather_rows(c_block, plan: KernelPlan, *, dst: int = 0, group=None):
    """Concatenate every rank's result block on ``dst`` (None elsewhere)."""
    torch, dist = _torch(), _dist()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    size = -(-plan.noproc // world) if plan.noproc else 0
    n = plan.elsinop
    padded = torch.zeros(size * n, dtype=c_block.dtype, device=c_block.device)
    padded[:c_block.numel()] = c_block
    if dist.get_backend(group) == "nccl":
        full = torch.empty(world * size * n, dtype=c_block.dtype, device=c_block.device)
        dist.all_gather_into_tensor(full, padded, group=group)
        return full[:plan.noproc * n] if rank == dst else None
    parts = [torch.empty_like(padded) for _ in range(world)] if rank == dst else None
    dist.gather(padded, parts, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat(parts)[:plan.noproc * n]


def sharded_product_host(plan: KernelPlan, a_block_host, b_host, ops: OpPair = MUL_ADD, *,
                         device, group=None, src: int = 0, exact: bool = False,
                         bcast_chunks: int = 8):
    """Host-buffer form of ``sharded_product``: this rank's A rows go to
    ``device``; on ``src`` B goes up in k-chunks, each broadcast as soon as it
    is on the device and folded by every rank while later chunks are still in
    flight (where the fold replays exactly, ``bcast_chunk_align``; else B goes
    whole); the result block comes back into page-locked host memory
    (``kernel.host_empty``), returned as a numpy vector."""
    torch = _torch()
    from .kernel import host_empty
    a_dev = _to_device(a_block_host, device)
    b_arg = None
    if b_host is not None:
        b_arg = b_host if isinstance(b_host, torch.Tensor) else torch.from_numpy(b_host)
        if not b_arg.is_cuda and bcast_chunk_align(ops, a_dev.dtype) is None:
            b_arg = _to_device(b_arg, device)
    c = sharded_product(plan, a_dev, b_arg, ops, group=group, src=src, exact=exact,
                        bcast_chunks=bcast_chunks)
    out = host_empty(c.numel(), np.dtype(str(c.dtype).replace("torch.", "")))
    d2h_split(torch.from_numpy(out), c, torch.cuda.current_stream(c.device))
    return out


def _to_device(x, device):
    torch = _torch()
    if not isinstance(x, torch.Tensor):
        x = torch.from_numpy(x)
    return x.to(device, non_blocking=True)
