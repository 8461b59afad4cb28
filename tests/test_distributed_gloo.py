"""The N>1 host path (row blocks, the broadcast of B, gathering the result) on
CPU with the gloo backend, world size 2 and 3.  The per-rank compute is the
C oracle injected through ``row_kernel`` — the device kernel is covered by the
GPU tests; this checks the sharding logic around it."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_rows(plan, c, a, b, ops):
    import oracle
    comb, red = ops.codes()
    got = oracle.product(a.numpy(), b.numpy(), plan.noproc, plan.rowsinred, plan.elsinop,
                         comb, red, lda=plan.lstride, ldb=plan.rstride)
    c.copy_(torch.from_numpy(got))


def _worker(rank, world, port, mode, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import paper_0907_0792_b200 as moa
        from paper_0907_0792_b200.distributed import gather_rows, row_block, sharded_product

        rng = np.random.default_rng(5)
        if mode in ("inner", "inner_b_f32"):
            m, k, n = 37, 11, 9
            plan = moa.plan_inner((m, k), (k, n))
            ops = moa.op_pair("add", "min")
        else:
            m, k, n = 23, 1, 17
            plan = moa.plan_outer((m,), (n,))
            ops = moa.op_pair("subtract", "max")
        a = rng.uniform(-1, 1, m * k)
        b = rng.uniform(-1, 1, k * n)
        if mode == "inner_b_f32":
            # B handed to rank 0 in another dtype than A: rank 0 must still
            # post A's dtype to the broadcast (equal byte counts on every rank)
            b = b.astype(np.float32).astype(np.float64)
        r0, r1 = row_block(m, world, rank)
        a_blk = torch.from_numpy(a[r0 * plan.lstride:r1 * plan.lstride].copy())
        # only rank 0 holds B; the others must receive it through the broadcast
        b_arg = (torch.from_numpy(b.astype(np.float32)) if mode == "inner_b_f32"
                 else torch.from_numpy(b)) if rank == 0 else None
        blk = sharded_product(plan, a_blk, b_arg, ops, row_kernel=_oracle_rows)
        assert blk.numel() == (r1 - r0) * n
        full = gather_rows(blk, plan)
        if rank == 0:
            comb, red = ops.codes()
            want = oracle.product(a, b, m, k, n, comb, red)
            q.put(("ok", np.array_equal(full.numpy(), want)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:  # surface worker failures in the parent
        q.put(("error", repr(exc)))
        raise


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("mode", ["inner", "outer", "inner_b_f32"])
def test_sharded_product_gloo(world, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = []
    while not q.empty():
        results.append(q.get())
    assert all(p.exitcode == 0 for p in procs), results
    assert ("ok", True) in results, results


def test_bcast_chunk_alignment_only_for_replayable_folds():
    """Pipelined broadcasts of B are offered only where chunked accumulation
    replays one pass bit for bit: (x,+) on float64 (DMMA k-slab 16) and
    (add|subtract, min|max) on every dtype (k-slab 32)."""
    import torch

    import paper_0907_0792_b200 as moa
    from paper_0907_0792_b200.distributed import bcast_chunk_align, k_chunks
    assert bcast_chunk_align(moa.MUL_ADD, torch.float64) == 16
    assert bcast_chunk_align(moa.MUL_ADD, torch.float32) is None
    for comb in ("add", "subtract"):
        for red in ("min", "max"):
            for dt in (torch.float32, torch.float64, torch.int32, torch.int64):
                assert bcast_chunk_align(moa.op_pair(comb, red), dt) == 32
    for comb, red in (("add", "add"), ("multiply", "min"), ("divide", "max"), ("min", "min")):
        assert bcast_chunk_align(moa.op_pair(comb, red), torch.float32) is None
    chunks = k_chunks(16384, 8, 32)
    assert chunks[0] == (0, 2048) and chunks[-1] == (14336, 16384)
    assert all(k0 % 32 == 0 for k0, _ in chunks)
