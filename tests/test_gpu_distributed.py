"""The one-process-per-GPU path with the real CUDA kernels: two ranks on the
single GPU of the test box, gloo for the (host-mediated) broadcast and gather.
The ranks' kernels never wait on each other, so sharing one GPU is safe; NCCL
itself needs one GPU per rank and is exercised by the driver's scaling run.
Checks that row-sharded results equal one launch bit for bit."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_0907_0792_b200 as moa
        from paper_0907_0792_b200.distributed import gather_rows, row_block, sharded_product
        rng = np.random.default_rng(11)
        ok = True
        for ops, dt, (m, k, n) in ((moa.op_pair("multiply", "add"), torch.float64, (777, 300, 513)),
                                   (moa.op_pair("add", "min"), torch.float32, (640, 257, 384)),
                                   (moa.op_pair("divide", "max"), torch.float64, (33, 5, 70))):
            a = torch.from_numpy(rng.random(m * k)).to(dt).cuda()
            b = torch.from_numpy(rng.random(k * n)).to(dt).cuda()
            plan = moa.plan_inner((m, k), (k, n))
            r0, r1 = row_block(m, world, rank)
            blk = sharded_product(plan, a[r0 * k:r1 * k], b if rank == 0 else None, ops)
            full = gather_rows(blk, plan)
            if rank == 0:
                ref = moa.inner(moa.MoaArray((m, k), a), moa.MoaArray((k, n), b), ops).data
                ok &= bool(torch.equal(full.view(-1), ref.view(-1)))
        # pipelined broadcast of B in k-chunks (float64 (x,+)): same bits
        m, k, n = 500, 300, 384
        a = torch.from_numpy(rng.random(m * k)).cuda()
        b = torch.from_numpy(rng.random(k * n)).cuda()
        plan = moa.plan_inner((m, k), (k, n))
        r0, r1 = row_block(m, world, rank)
        blk = sharded_product(plan, a[r0 * k:r1 * k], b if rank == 0 else None, moa.MUL_ADD,
                              bcast_chunks=4)
        full = gather_rows(blk, plan)
        if rank == 0:
            ref = moa.inner(moa.MoaArray((m, k), a), moa.MoaArray((k, n), b)).data
            ok &= bool(torch.equal(full.view(-1), ref.view(-1)))
        # ... and for (add|subtract, min|max), fast folds and the exact loop
        # (NaN / -0 / negative data), float32 and int32: same bits
        m, k, n = 300, 203, 388
        for ops, dt, poison in ((moa.op_pair("add", "min"), torch.float32, None),
                                (moa.op_pair("subtract", "max"), torch.float32, "negative"),
                                (moa.op_pair("add", "max"), torch.float32, "nan"),
                                (moa.op_pair("add", "min"), torch.float64, "negzero"),
                                (moa.op_pair("subtract", "min"), torch.int32, None)):
            av = rng.random(m * k) * 100
            bv = rng.random(k * n) * 100
            av[rng.random(m * k) < 0.05] = np.inf if dt.is_floating_point else 7
            if poison == "negative":
                av -= 50
            elif poison == "nan":
                av[rng.random(m * k) < 0.01] = np.nan
            elif poison == "negzero":
                av[rng.random(m * k) < 0.05] = -0.0
                bv[rng.random(k * n) < 0.05] = -0.0
            a = torch.from_numpy(av).to(dt).cuda()
            b = torch.from_numpy(bv).to(dt).cuda()
            plan = moa.plan_inner((m, k), (k, n))
            r0, r1 = row_block(m, world, rank)
            blk = sharded_product(plan, a[r0 * k:r1 * k], b if rank == 0 else None, ops,
                                  bcast_chunks=3)
            full = gather_rows(blk, plan)
            if rank == 0:
                ref = moa.inner(moa.MoaArray((m, k), a), moa.MoaArray((k, n), b), ops).data
                same = torch.equal(full.view(-1).view(torch.uint8), ref.view(-1).view(torch.uint8))
                ok &= bool(same)
        # the host-buffer form used by bench.py's e2e leg
        from paper_0907_0792_b200.distributed import sharded_product_host
        m, k, n = 100, 64, 96
        a = rng.random(m * k)
        b = rng.random(k * n)
        plan = moa.plan_inner((m, k), (k, n))
        r0, r1 = row_block(m, world, rank)
        blk = sharded_product_host(plan, a[r0 * k:r1 * k].copy(), b if rank == 0 else None,
                                   moa.MUL_ADD, device=torch.device("cuda", 0))
        want = moa.inner(moa.MoaArray((m, k), a), moa.MoaArray((k, n), b)).data[r0 * n:r1 * n]
        ok &= bool(np.array_equal(blk, want))
        q.put((rank, ok))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as exc:
        q.put((rank, repr(exc)))
        raise


def test_row_sharded_product_two_ranks_one_gpu():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = dict(q.get() for _ in range(q.qsize()))
    assert all(p.exitcode == 0 for p in procs), results
    assert results == {0: True, 1: True}, results
