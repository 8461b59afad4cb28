"""Row-partitioned execution over the GPUs of one process.

The reference's only parallel strategy is fork-join over result rows: worker
k owns rows k, k+W, ... and runs the sequential loop on them (parallel.py:19-43,
PAPER.md:505-507).  Rows are independent and every kernel folds each element
in the same order whatever rows it is given, so any partition gives the same
bits (tests/test_acceptance.py:84-103 analogue).

On B200 the fork-join unit is a GPU: ``execute_parallel(..., workers=W)``
splits the rows into ``min(W, len(devices))`` contiguous blocks, one per GPU
(contiguous blocks keep A and C rows dense for the tile loaders), copies B to
every GPU once (a device-to-device copy over NVLink when B is already
device-resident) and launches the blocks concurrently, one stream per GPU.
With a single GPU the whole product is one launch.  Workers beyond the device
count, like surplus reference workers, do nothing.  For one process per GPU
(torchrun) see ``distributed.py``.
"""

from __future__ import annotations


from . import _native
from .arrays import MoaArray
from .kernel import (KernelPlan, _Runner, _check_plan, execute_host, launch, resolve_backend,
                     result_dtype, stage, stage_host, torch_dtype)
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
                     exact: bool = False) -> MoaArray:
    """Run the planned product with ``workers`` row partitions over the GPUs.

    ``devices``: CUDA device indices to use (default: every visible GPU); the
    same index may repeat, which runs several blocks on one GPU.  The result is
    bitwise identical for every ``workers``/``devices`` choice.
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

    _check_plan(plan, a, b)
    resolve_backend(backend, ops)
    _native.load()
    dtype = result_dtype(a, b)
    tdt = torch_dtype(dtype)
    host_result = not (a.is_device or b.is_device)
    home = a.data.device if a.is_device else b.data.device if b.is_device else \
        torch.device("cuda", devices[0])
    blocks = row_blocks(plan.noproc, len(devices))
    m, k, n = plan.noproc, plan.rowsinred, plan.elsinop
    a_home = stage(a, home, dtype) if a.is_device else None
    b_home = stage(b, home, dtype)
    pieces = []
    for dev_idx, rows in zip(devices, blocks):
        dev = torch.device("cuda", dev_idx)
        if len(rows) == 0:
            continue
        with torch.cuda.device(dev):
            s = torch.cuda.Stream(dev)
            s.wait_stream(torch.cuda.current_stream(home))
            with torch.cuda.stream(s):
                r0, r1 = rows.start, rows.stop
                if a_home is not None:
                    a_blk = a_home[r0 * plan.lstride:r1 * plan.lstride].to(dev, non_blocking=True)
                else:
                    a_blk = stage_host(a.data[r0 * plan.lstride:r1 * plan.lstride], dev, dtype)
                b_blk = b_home.to(dev, non_blocking=True)
                c_blk = torch.empty((r1 - r0) * n, dtype=tdt, device=dev)
                sub = KernelPlan(plan.mode, r1 - r0, k, n, plan.lstride, plan.rstride,
                                 plan.restride, plan.result_shape)
                launch(sub, c_blk, a_blk, b_blk, ops, exact=exact, stream=s)
                pieces.append((dev, s, r0, r1, c_blk, a_blk, b_blk))
    if host_result:
        out = torch.empty(m * n, dtype=tdt, pin_memory=True)
        for dev, s, r0, r1, c_blk, *_ in pieces:
            with torch.cuda.stream(s):
                out[r0 * n:r1 * n].copy_(c_blk, non_blocking=True)
        for _, s, *_ in pieces:
            s.synchronize()
        return MoaArray._wrap(plan.result_shape, out.numpy())
    res = torch.empty(m * n, dtype=tdt, device=home)
    cur = torch.cuda.current_stream(home)
    for dev, s, r0, r1, c_blk, *_ in pieces:
        cur.wait_stream(s)
        c_blk.record_stream(cur)
        res[r0 * n:r1 * n].copy_(c_blk, non_blocking=True)
    for _, s, *_ in pieces:
        s.synchronize()
    return MoaArray._wrap(plan.result_shape, res)


def _device_for(a: MoaArray, b: MoaArray, index: int):
    if a.is_device:
        return a.data.device
    if b.is_device:
        return b.data.device
    return _torch().device("cuda", index)
