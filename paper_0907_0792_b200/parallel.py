"""Row-partitioned execution over the GPUs of one process.

The reference's only parallel strategy is fork-join over result rows: worker
k owns rows k, k+W, ... and runs the sequential loop on them (parallel.py:19-43,
PAPER.md:505-507).  Rows are independent and every kernel folds each element
in the same order whatever rows it is given, so any partition gives the same
bits (tests/test_acceptance.py:84-103 analogue).

On B200 the fork-join unit is a GPU: ``execute_parallel(..., workers=W)``
splits the rows into ``min(W, len(devices))`` contiguous blocks, one per GPU
(contiguous blocks keep A and C rows dense for the tile loaders), sends B to
every GPU with one NCCL broadcast from the home GPU (pipelined in k-chunks with
the blocks' kernels where the fold allows) and launches the blocks
concurrently, one stream per block.
With a single GPU the whole product is one launch.  Workers beyond the device
count, like surplus reference workers, do nothing.  For one process per GPU
(torchrun) see ``distributed.py``.
"""

from __future__ import annotations


from . import _native
from .arrays import MoaArray
from .kernel import (KernelPlan, _Runner, _check_plan, execute_host, host_empty, launch,
                     resolve_backend, result_dtype, stage, stage_host, torch_dtype)
from .ops import MUL_ADD, OpPair


def partition_rows(noproc: int, workers: int) -> list[range]:
    """The reference's round-robin ownership: worker k gets rows k, k+workers, ..."""
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    return [range(k, noproc, workers) for k in range(workers)]


def row_blocks(noproc: int, parts: int) -> list[range]:
    """Contiguous, nearly equal row blocks (ceil-sized; trailing blocks may be empty)."""
    if parts < 1:
        raise ValueError(f"parts must be >= 1, got {parts}")
    size = -(-noproc // parts) if noproc else 0
    return [range(min(p * size, noproc), min((p + 1) * size, noproc)) for p in range(parts)]


def _torch():
    import torch
    return torch


def execute_parallel(plan: KernelPlan, a: MoaArray, b: MoaArray, ops: OpPair = MUL_ADD,
                     workers: int = 1, *, backend: str | None = None, devices=None,
                     exact: bool = False, bcast_chunks: int | None = None) -> MoaArray:
    """Run the planned product with ``workers`` row partitions over the GPUs.

    ``devices``: CUDA device indices to use (default: every visible GPU); the
    same index may repeat, which runs several blocks on one GPU.  The result is
    bitwise identical for every ``workers``/``devices`` choice.

    B, which every block needs, reaches the GPUs as ONE NCCL broadcast from the
    home GPU (``torch.cuda.comm.broadcast``: a single-process communicator over
    NVLink/NVSwitch) instead of a copy per GPU.  Where chunked accumulation
    replays one pass bit for bit (``distributed.bcast_chunk_align``) the
    broadcast goes out in ``bcast_chunks`` k-chunks on a communication stream
    per GPU and each GPU's kernel for chunk i starts as soon as chunk i has
    landed, accumulating, while later chunks are on the wire (default: 4
    chunks when more than one distinct GPU takes part, else 1).
    """
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    torch = _torch()
    if devices is None:
        devices = list(range(torch.cuda.device_count())) or [0]
    devices = list(devices)[:workers]
    if len(devices) <= 1:
        if not (a.is_device or b.is_device):  # host operands: the native executor
            _check_plan(plan, a, b)
            resolve_backend(backend, ops)
            return execute_host(plan, a, b, ops, exact=exact,
                                device=devices[0] if devices else None)
        runner = _Runner(plan, a, b, ops, backend, exact=exact,
                         device=None if not devices else _device_for(a, b, devices[0]))
        runner.run_rows(0, 1)
        return runner.finish()

    from contextlib import ExitStack

    from .distributed import bcast_chunk_align, k_chunks
    _check_plan(plan, a, b)
    resolve_backend(backend, ops)
    _native.load()
    dtype = result_dtype(a, b)
    tdt = torch_dtype(dtype)
    host_result = not (a.is_device or b.is_device)
    home = a.data.device if a.is_device else b.data.device if b.is_device else \
        torch.device("cuda", devices[0])
    blocks = [(torch.device("cuda", d), rows)
              for d, rows in zip(devices, row_blocks(plan.noproc, len(devices))) if len(rows)]
    m, k, n = plan.noproc, plan.rowsinred, plan.elsinop
    distinct = []
    for dev, _ in blocks:
        if dev not in distinct:
            distinct.append(dev)
    a_home = stage(a, home, dtype) if a.is_device else None
    b_home = stage(b, home, dtype)
    # B on every GPU: the home copy, and one receive buffer per other GPU
    b_on = {dev: (b_home if dev == home else torch.empty(k * n, dtype=tdt, device=dev))
            for dev in distinct}
    others = [dev for dev in distinct if dev != home]
    align = bcast_chunk_align(ops, tdt)
    chunkable = align is not None and not (exact and ops.codes() == (2, 0))
    if bcast_chunks is None:
        bcast_chunks = 4 if others else 1
    chunks = k_chunks(k, bcast_chunks, align) if chunkable and k else [(0, k)]
    comm = {dev: torch.cuda.Stream(dev) for dev in distinct}
    b_ready = torch.cuda.Event()
    b_ready.record(torch.cuda.current_stream(home))
    comm[home].wait_event(b_ready)

    pieces = []
    for dev, rows in blocks:
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(home))
        with torch.cuda.device(dev), torch.cuda.stream(s):
            r0, r1 = rows.start, rows.stop
            if a_home is not None:
                a_blk = a_home[r0 * plan.lstride:r1 * plan.lstride].to(dev, non_blocking=True)
            else:
                a_blk = stage_host(a.data[r0 * plan.lstride:r1 * plan.lstride], dev, dtype)
            c_blk = torch.empty((r1 - r0) * n, dtype=tdt, device=dev)
        pieces.append((dev, s, r0, r1, c_blk, a_blk))

    for i, (k0, k1) in enumerate(chunks):
        if others and k1 > k0:
            # one NCCL broadcast of B's rows [k0, k1) from home, on the
            # communication streams (current for the call on every GPU)
            with ExitStack() as stack:
                for dev in distinct:
                    stack.enter_context(torch.cuda.stream(comm[dev]))
                torch.cuda.comm.broadcast(b_home[k0 * n:k1 * n],
                                          out=[b_on[dev][k0 * n:k1 * n] for dev in others])
        landed = {}
        for dev in distinct:
            landed[dev] = torch.cuda.Event()
            landed[dev].record(comm[dev])
        for dev, s, r0, r1, c_blk, a_blk in pieces:
            s.wait_event(landed[dev])
            part = KernelPlan(plan.mode, r1 - r0, k1 - k0, n, plan.lstride, plan.rstride,
                              plan.restride, plan.result_shape)
            launch(part, c_blk, a_blk[k0:], b_on[dev][k0 * n:], ops, exact=exact,
                   accumulate=i > 0, stream=s)

    if host_result:
        out = host_empty(m * n, dtype)
        out_t = torch.from_numpy(out)
        for dev, s, r0, r1, c_blk, _ in pieces:
            with torch.cuda.device(dev), torch.cuda.stream(s):
                out_t[r0 * n:r1 * n].copy_(c_blk, non_blocking=True)
        for _, s, *_ in pieces:
            s.synchronize()
        for st in comm.values():
            st.synchronize()
        return MoaArray._wrap(plan.result_shape, out)
    res = torch.empty(m * n, dtype=tdt, device=home)
    cur = torch.cuda.current_stream(home)
    for dev, s, r0, r1, c_blk, _ in pieces:
        cur.wait_stream(s)
        c_blk.record_stream(cur)
        res[r0 * n:r1 * n].copy_(c_blk, non_blocking=True)
    for _, s, *_ in pieces:
        s.synchronize()
    for st in comm.values():
        st.synchronize()
    return MoaArray._wrap(plan.result_shape, res)


def _device_for(a: MoaArray, b: MoaArray, index: int):
    if a.is_device:
        return a.data.device
    if b.is_device:
        return b.data.device
    return _torch().device("cuda", index)
