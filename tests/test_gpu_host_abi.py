"""moa_product_rows_host — the host-buffer form of the boundary (the exact
drop-in for _ckernel.product_rows, _ckernel.pyx:75-88): against the
device-pointer entry point on the same data (bitwise) and the CPU oracle,
for every dtype, row sets start::step, accumulate mode, padded and
overlapping strides, pageable and page-locked buffers, the streamed (row
block) schedule, and its argument errors."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_0907_0792_b200 as moa
from paper_0907_0792_b200 import op_pair
from paper_0907_0792_b200.errors import BackendError
from paper_0907_0792_b200.kernel import KernelPlan, launch, launch_host, plan_inner, plan_outer
from parity import assert_bits_equal, assert_within, sum_tolerance

pytestmark = pytest.mark.gpu

DTYPES = (np.float64, np.float32, np.int32, np.int64)


def _torch():
    import torch
    return torch


def _operands(rng, n, dt):
    if np.dtype(dt).kind == "i":
        return rng.integers(-50, 50, n).astype(dt)
    return (rng.random(n) * 4 - 1).astype(dt)


def _device_result(plan, res0, a, b, ops, **kw):
    torch = _torch()
    res = torch.from_numpy(res0.copy()).cuda()
    launch(plan, res, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), ops, **kw)
    return res.cpu().numpy()


@pytest.mark.parametrize("dt", DTYPES)
def test_host_entry_equals_device_entry(dt, rng):
    """Same bits as moa_product_rows on device copies of the same buffers, for
    row sets start::step, write-only and accumulate, across op pairs."""
    m, k, n = 77, 45, 66
    a, b = _operands(rng, m * k, dt), _operands(rng, k * n, dt)
    plan = plan_inner((m, k), (k, n))
    pairs = [op_pair("multiply", "add"), op_pair("add", "min"), op_pair("subtract", "max"),
             op_pair("max", "multiply"), op_pair("divide", "min")]
    for ops in pairs:
        for start, step in ((0, 1), (1, 3), (5, 2), (76, 4)):
            for acc in (False, True):
                res0 = _operands(rng, m * n, dt)
                want = _device_result(plan, res0, a, b, ops, start=start, step=step, accumulate=acc)
                got = res0.copy()
                launch_host(plan, got, a, b, ops, start=start, step=step, accumulate=acc)
                assert_bits_equal(got, want, f"{dt.__name__} {ops} {start}::{step} acc={acc}")


def test_host_entry_matches_oracle_and_touches_only_its_rows(rng):
    m, k, n = 60, 33, 47
    a, b = rng.random(m * k) * 2 - 1, rng.random(k * n) * 2 - 1
    plan = plan_inner((m, k), (k, n))
    sentinel = -7.25
    res = np.full(m * n, sentinel)
    launch_host(plan, res, a, b, op_pair("add", "max"), start=2, step=5)
    want = oracle.product(a, b, m, k, n, 0, 3).reshape(m, n)
    got = res.reshape(m, n)
    rows = np.arange(2, m, 5)
    assert_bits_equal(got[rows].ravel(), want[rows].ravel())
    others = np.setdiff1d(np.arange(m), rows)
    assert np.all(got[others] == sentinel)
    # (multiply, add) on the tensor cores: within the north-star tolerance
    res = np.empty(m * n)
    launch_host(plan, res, a, b, moa.MUL_ADD)
    assert_within(res, oracle.product(a, b, m, k, n, 2, 0), sum_tolerance(k, a, b))


def test_host_entry_padded_and_overlapping_strides(rng):
    """lstride > K (padded A rows), rstride > N (padded B rows) and a row set
    whose A rows overlap (lstride*step < K: the span path)."""
    m, k, n = 40, 24, 30
    ops = op_pair("add", "min")
    # padded A rows (lstride = 31) and B rows (rstride = 37); C rows restride 35
    lstride, rstride, restride = 31, 37, 35
    a = rng.random(m * lstride)
    b = rng.random(k * rstride)
    plan = KernelPlan("inner", m, k, n, lstride, rstride, restride, (m, n))
    res0 = np.full(m * restride, 3.5)
    want = _device_result(plan, res0, a, b, ops, start=1, step=2)
    got = res0.copy()
    launch_host(plan, got, a, b, ops, start=1, step=2)
    assert_bits_equal(got, want, "padded")
    # overlapping A rows: lstride 10 < K = 24 (rows share elements)
    plan = KernelPlan("inner", m, k, n, 10, n, n, (m, n))
    a = rng.random((m - 1) * 10 + k)
    b = rng.random(k * n)
    res0 = np.zeros(m * n)
    want = _device_result(plan, res0, a, b, ops)
    got = res0.copy()
    launch_host(plan, got, a, b, ops)
    assert_bits_equal(got, want, "overlapping A rows")


def test_host_entry_outer_fill_and_page_locked_buffers(rng):
    torch = _torch()
    x, y = rng.random(300) * 2 - 1, rng.random(513) * 2 - 1
    res = np.empty(300 * 513)
    launch_host(plan_outer((300,), (513,)), res, x, y, moa.MUL_ADD)
    assert_bits_equal(res, (np.multiply.outer(x, y) + 0.0).ravel())
    # K = 0: the identity everywhere (write-only), nothing under accumulate
    res = np.full(6, 9.0)
    launch_host(plan_inner((2, 0), (0, 3)), res, np.empty(0), np.empty(0), op_pair("add", "min"))
    assert np.all(res == np.inf)
    res = np.full(6, 9.0)
    launch_host(plan_inner((2, 0), (0, 3)), res, np.empty(0), np.empty(0), op_pair("add", "min"),
                accumulate=True)
    assert np.all(res == 9.0)
    # page-locked host buffers (the overlapped path) give the same bits
    m, k, n = 90, 64, 128
    a, b = rng.random(m * k), rng.random(k * n)
    pa = torch.empty(m * k, dtype=torch.float64, pin_memory=True).numpy()
    pb = torch.empty(k * n, dtype=torch.float64, pin_memory=True).numpy()
    pr = torch.empty(m * n, dtype=torch.float64, pin_memory=True).numpy()
    pa[:], pb[:] = a, b
    plan = plan_inner((m, k), (k, n))
    launch_host(plan, pr, pa, pb, op_pair("multiply", "max"))
    assert_bits_equal(pr, oracle.product(a, b, m, k, n, 2, 3))


@pytest.mark.parametrize("dt,ops", [(np.float64, moa.MUL_ADD),
                                    (np.float32, op_pair("add", "min")),
                                    (np.float32, op_pair("multiply", "add"))])
def test_host_entry_streamed_blocks_equal_one_launch(dt, ops, rng):
    """Results of >= 1 GiB run the streamed schedule (4/16 first block computed
    per k-chunk of B, middle blocks, 1/16 last block; float32 sums take B
    whole): bitwise equal to one device launch."""
    torch = _torch()
    esz = np.dtype(dt).itemsize
    m, k, n = (8192, 96, 16384) if esz == 8 else (16384, 96, 16384)
    a = (rng.random(m * k) * 100).astype(dt)
    b = (rng.random(k * n) * 100).astype(dt)
    plan = plan_inner((m, k), (k, n))
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    want = torch.empty(m * n, dtype=ad.dtype, device="cuda")
    launch(plan, want, ad, bd, ops)
    want = want.cpu().numpy()
    del ad, bd
    res = torch.empty(m * n, dtype=torch.from_numpy(a[:1]).dtype, pin_memory=True).numpy()
    launch_host(plan, res, a, b, ops)
    assert_bits_equal(res, want, f"{dt.__name__} {ops}")
    # and with accumulate (res prefilled with the identity, as the reference does)
    res[:] = ops.reduce_identity
    launch_host(plan, res, a, b, ops, accumulate=True)
    assert_bits_equal(res, want, f"{dt.__name__} {ops} accumulate")


def test_host_entry_argument_errors(rng):
    from paper_0907_0792_b200 import _native
    a, b, res = np.zeros(12), np.zeros(12), np.zeros(9)
    with pytest.raises(BackendError, match="step"):
        _native.product_rows_host(0, res.ctypes.data, a.ctypes.data, b.ctypes.data,
                                  3, 4, 3, 4, 3, 3, 2, 0, 0, 0, 0, 0)
    with pytest.raises(BackendError, match="dtype"):
        _native.product_rows_host(9, res.ctypes.data, a.ctypes.data, b.ctypes.data,
                                  3, 4, 3, 4, 3, 3, 2, 0, 0, 1, 0, 0)
    with pytest.raises(BackendError, match="overlap"):
        _native.product_rows_host(0, res.ctypes.data, a.ctypes.data, b.ctypes.data,
                                  3, 4, 3, 4, 3, 1, 2, 0, 0, 1, 0, 0)
    with pytest.raises(BackendError, match="cudaSetDevice"):
        _native.product_rows_host(0, res.ctypes.data, a.ctypes.data, b.ctypes.data,
                                  3, 4, 3, 4, 3, 3, 2, 0, 0, 1, 0, 99)
    # surplus worker / empty rows: no work, no error
    _native.product_rows_host(0, res.ctypes.data, a.ctypes.data, b.ctypes.data,
                              3, 4, 3, 4, 3, 3, 2, 0, 5, 1, 0, 0)


@pytest.mark.parametrize("dt,ops", [(np.float64, moa.MUL_ADD), (np.float32, op_pair("add", "min")),
                                    (np.float64, op_pair("subtract", "max"))])
def test_host_entry_ramped_k_chunks(dt, ops, monkeypatch, rng):
    """Long contractions (K >= 1024) split the first block's k-range as a ramp
    (~K/32 first, each next 1.25x, 16-aligned): many uneven accumulating
    chunks, still the bits of one device launch — write-only, accumulate from
    the identity, and a strided row set."""
    torch = _torch()
    monkeypatch.setenv("MOA_HOST_BLOCK_BYTES", str(2 << 20))  # forces the streamed schedule
    m, k, n = 2100, 1100, 128   # 128-row blocks; K = 1100: a ramp of 10 chunks
    a = (rng.random(m * k) * 100).astype(dt)
    b = (rng.random(k * n) * 100).astype(dt)
    plan = plan_inner((m, k), (k, n))
    want = _device_result(plan, np.zeros(m * n, dtype=dt), a, b, ops)
    for acc, pin in ((False, True), (True, True), (False, False)):
        res0 = np.full(m * n, ops.reduce_identity if acc else 0, dtype=dt)
        res = _pinned_like(res0) if pin else res0.copy()
        launch_host(plan, res, a, b, ops, accumulate=acc)
        assert_bits_equal(res, want, f"{dt.__name__} {ops} acc={acc} pinned={pin}")
    res = np.full(m * n, 7, dtype=dt)
    launch_host(plan, res, a, b, ops, start=1, step=2)
    got, ref = res.reshape(m, n), want.reshape(m, n)
    assert_bits_equal(got[1::2].ravel(), ref[1::2].ravel(), f"{dt.__name__} {ops} rows 1::2")
    assert np.all(got[0::2] == 7)


def test_host_entry_bounded_blocks(monkeypatch, rng):
    """Every block's A and C rows stay within $MOA_HOST_BLOCK_BYTES (4 GiB by
    default): a small cap forces many blocks for an outer product (equal
    blocks) and for a sub-GiB inner product (4/16 first block per k-chunk,
    extra middle blocks); results bitwise equal one device launch."""
    torch = _torch()
    monkeypatch.setenv("MOA_HOST_BLOCK_BYTES", str(3 << 20))  # 3 MiB
    x, y = rng.random(2000) * 2 - 1, rng.random(700) * 2 - 1
    res = np.empty(2000 * 700)
    launch_host(plan_outer((2000,), (700,)), res, x, y, op_pair("subtract", "max"))
    assert_bits_equal(res, np.subtract.outer(x, y).ravel())
    for ops, dt in ((moa.MUL_ADD, np.float64), (op_pair("add", "min"), np.float32),
                    (op_pair("divide", "max"), np.float64)):
        m, k, n = 2100, 96, 640  # 6.9 MiB of A+C rows: 512-row first block, 128-row last
        a = (rng.random(m * k) * 100 + 1).astype(dt)
        b = (rng.random(k * n) * 100 + 1).astype(dt)
        plan = plan_inner((m, k), (k, n))
        want = _device_result(plan, np.zeros(m * n, dtype=dt), a, b, ops)
        for acc in (False, True):
            res = np.full(m * n, ops.reduce_identity if acc else 0, dtype=dt)
            pinned = torch.empty(m * n, dtype=torch.from_numpy(res[:1]).dtype,
                                 pin_memory=True).numpy()
            pinned[:] = res
            launch_host(plan, pinned, a, b, ops, accumulate=acc)
            assert_bits_equal(pinned, want, f"{ops} {dt.__name__} acc={acc}")
        # a strided row set (rows 1, 3, 5, ...) through the same multi-block
        # schedule: A rows and result rows move by 2-D copies
        res = np.full(m * n, 5, dtype=dt)
        launch_host(plan, res, a, b, ops, start=1, step=2)
        got, ref = res.reshape(m, n), want.reshape(m, n)
        assert_bits_equal(got[1::2].ravel(), ref[1::2].ravel(), f"{ops} {dt.__name__} rows 1::2")
        assert np.all(got[0::2] == 5)


def _pinned_like(x):
    torch = _torch()
    t = torch.empty(x.size, dtype=torch.from_numpy(x[:1]).dtype, pin_memory=True).numpy()
    t[:] = x
    return t


@pytest.mark.parametrize("dt", DTYPES)
def test_direct_out_into_page_locked_res(dt, rng):
    """Write-only single-block products with a page-locked res (pinned, and
    registered moa_host_alloc memory) of <= 1 MiB store their rows straight
    into res through its device mapping: the bits of the device entry point,
    only the row set's rows written, for inner (every kernel family) and
    outer products."""
    from paper_0907_0792_b200 import _native
    m, k, n = 300, 132, 260   # f64 result 609 KiB   # 16-byte rows: TMA kernels; odd K below: cp.async ones
    for kk in (k, 67):
        a, b = _operands(rng, m * kk, dt), _operands(rng, kk * n, dt)
        plan = plan_inner((m, kk), (kk, n))
        pa, pb = _pinned_like(a), _pinned_like(b)
        for ops in (moa.MUL_ADD, op_pair("add", "min"), op_pair("subtract", "max"),
                    op_pair("divide", "add"), op_pair("max", "multiply")):
            for start, step in ((0, 1), (3, 4)):
                res0 = np.full(m * n, 5, dtype=dt)
                want = _device_result(plan, res0, a, b, ops, start=start, step=step)
                got = _pinned_like(res0)
                launch_host(plan, got, pa, pb, ops, start=start, step=step)
                assert_bits_equal(got, want, f"{dt.__name__} {ops} K={kk} {start}::{step}")
    # registered (huge-page) host block as res
    esz = np.dtype(dt).itemsize
    ptr = _native.host_alloc(m * n * esz)
    try:
        import ctypes
        buf = (ctypes.c_char * (m * n * esz)).from_address(ptr)
        got = np.frombuffer(buf, dtype=dt)
        got[:] = 0
        a, b = _operands(rng, m * k, dt), _operands(rng, k * n, dt)
        plan = plan_inner((m, k), (k, n))
        want = _device_result(plan, np.zeros(m * n, dtype=dt), a, b, op_pair("add", "max"))
        launch_host(plan, got, _pinned_like(a), _pinned_like(b), op_pair("add", "max"))
        assert_bits_equal(got, want, f"{dt.__name__} registered res")
        del got, buf
    finally:
        _native.host_free(ptr)
    # outer product straight into pinned res
    x, y = _operands(rng, 300, dt), _operands(rng, 400, dt)
    plan = plan_outer((300,), (400,))
    want = _device_result(plan, np.zeros(300 * 400, dtype=dt), x, y, op_pair("multiply", "add"))
    got = _pinned_like(np.zeros(300 * 400, dtype=dt))
    launch_host(plan, got, _pinned_like(x), _pinned_like(y), op_pair("multiply", "add"))
    assert_bits_equal(got, want, f"{dt.__name__} outer")


@pytest.mark.parametrize("acc", [False, True])
def test_row_parts_into_page_locked_res(acc, rng):
    """Results of >= 64 MiB into page-locked res run as four row parts whose
    copy-out overlaps the next part's kernel: the bits of the device entry
    point for the DMMA, tropical and outer routes, a strided row set (only its
    rows written) and overlapping A rows (the whole span of A goes first)."""
    m, k, n = 16384, 33, 1024
    cases = [(np.float64, moa.MUL_ADD, 1, k), (np.float64, moa.MUL_ADD, 2, k),
             (np.float32, op_pair("add", "min"), 1, k), (np.float64, op_pair("max", "add"), 1, 20)]
    for dt, ops, step, lstride in cases:   # every row set >= 64 MiB of result
        a = _operands(rng, (m - 1) * lstride + k, dt)
        b = _operands(rng, k * n, dt)
        plan = KernelPlan("inner", m, k, n, lstride, n, n, (m, n))
        res0 = _operands(rng, m * n, dt)
        kw = dict(step=step, accumulate=acc)
        want = _device_result(plan, res0, a, b, ops, **kw)
        got = _pinned_like(res0)
        launch_host(plan, got, _pinned_like(a), _pinned_like(b), ops, **kw)
        assert_bits_equal(got, want, f"{dt.__name__} {ops} step={step} lstride={lstride} acc={acc}")
    # outer product (K = 1): 8192 x 2048 f64 = 128 MiB
    x, y = _operands(rng, 8192, np.float64), _operands(rng, 2048, np.float64)
    plan = plan_outer((8192,), (2048,))
    res0 = _operands(rng, 8192 * 2048, np.float64)
    want = _device_result(plan, res0, x, y, moa.MUL_ADD, accumulate=acc)
    got = _pinned_like(res0)
    launch_host(plan, got, _pinned_like(x), _pinned_like(y), moa.MUL_ADD, accumulate=acc)
    assert_bits_equal(got, want, f"outer acc={acc}")


@pytest.mark.parametrize("dt,ops", [(np.float64, moa.MUL_ADD), (np.float64, op_pair("add", "min")),
                                    (np.float32, op_pair("multiply", "max")),
                                    (np.int32, op_pair("add", "min"))])
def test_accumulate_into_identity_result_skips_its_upload(dt, ops, rng):
    """MOA_FLAG_ACCUMULATE into a result of >= 32 MiB that holds only the
    reduce identity (the reference's prefill) runs write-only — the same bits
    by construction — and one other value anywhere in the row set keeps the
    fold from res: both equal the device entry's accumulate, pageable and
    page-locked, whole set and a strided row set."""
    m, k, n = 9000, 20, 1000
    a, b = _operands(rng, m * k, dt), _operands(rng, k * n, dt)
    plan = plan_inner((m, k), (k, n))
    ident = ops.reduce_identity if np.dtype(dt).kind == "f" else \
        {"add": 0, "multiply": 1, "min": np.iinfo(dt).max, "max": np.iinfo(dt).min}[ops.reduce_name]
    for start, step in ((0, 1), (2, 2)):
        for poke in (None, (m // 2) * n + 7):
            res0 = np.full(m * n, ident, dtype=dt)
            if poke is not None:
                res0[poke] = dt(3) if np.dtype(dt).kind == "i" else dt(-3.5)
                res0[poke + 2 * n] = res0[poke]   # the row set 2::2 sees it too
            want = _device_result(plan, res0, a, b, ops, start=start, step=step, accumulate=True)
            for pin in (False, True):
                got = _pinned_like(res0) if pin else res0.copy()
                launch_host(plan, got, a, b, ops, start=start, step=step, accumulate=True)
                assert_bits_equal(got, want, f"{np.dtype(dt).name} {ops} {start}::{step} "
                                             f"poke={poke} pinned={pin}")


def test_large_pageable_result_prefaulted_in_place(rng):
    """A pageable result of >= 32 MiB is prefaulted before the copy-back
    (huge-page advice + MADV_POPULATE_WRITE over its span): fresh np.empty
    memory and a strided row set whose other rows hold data — those rows keep
    their contents, the set's rows get the device entry's bits."""
    m, k, n = 13200, 24, 1000   # 106 MB of float64 result; rows 1::3 alone 35 MB
    a, b = rng.random(m * k) * 2 - 1, rng.random(k * n) * 2 - 1
    plan = plan_inner((m, k), (k, n))
    for ops in (moa.MUL_ADD, op_pair("add", "min")):
        want = _device_result(plan, np.zeros(m * n), a, b, ops)
        fresh = np.empty(m * n)
        launch_host(plan, fresh, a, b, ops)
        assert_bits_equal(fresh, want, f"{ops} fresh")
        res0 = rng.random(m * n)
        res = res0.copy()
        launch_host(plan, res, a, b, ops, start=1, step=3)
        got, ref = res.reshape(m, n), want.reshape(m, n)
        assert_bits_equal(got[1::3].ravel(), ref[1::3].ravel(), f"{ops} rows 1::3")
        keep = np.setdiff1d(np.arange(m), np.arange(1, m, 3))
        assert_bits_equal(got[keep].ravel(), res0.reshape(m, n)[keep].ravel(), f"{ops} other rows")


@pytest.mark.parametrize("acc", [False, True])
def test_pageable_staging_equals_page_locked(acc, rng):
    """Pageable host buffers above the direct-copy size are staged through
    page-locked slots by the executor's copy threads (host_runtime.cu): many
    8 MiB chunks, strided row sets gathered and scattered by the threads,
    accumulate mode reading res through the slots — the same bits as the
    page-locked path."""
    m, k, n = 1500, 700, 2300   # A 8 MiB, B 12.3 MiB, C 26 MiB: several chunks each
    a, b = rng.random(m * k) * 2 - 1, rng.random(k * n) * 2 - 1
    plan = plan_inner((m, k), (k, n))
    for ops in (moa.MUL_ADD, op_pair("add", "min")):
        for start, step in ((0, 1), (3, 5)):
            res0 = rng.random(m * n) if acc else np.full(m * n, -1.5)
            pinned = _pinned_like(res0)
            launch_host(plan, pinned, _pinned_like(a), _pinned_like(b), ops, start=start,
                        step=step, accumulate=acc)
            pageable = res0.copy()
            launch_host(plan, pageable, a, b, ops, start=start, step=step, accumulate=acc)
            assert_bits_equal(pageable, pinned, f"{ops} {start}::{step} acc={acc}")
            if step > 1:  # rows outside the set untouched
                keep = np.setdiff1d(np.arange(m), np.arange(start, m, step))
                assert_bits_equal(pageable.reshape(m, n)[keep].ravel(),
                                  res0.reshape(m, n)[keep].ravel())


def test_pageable_rows_wider_than_a_staging_slot(rng):
    """Result rows longer than one 8 MiB staging slot move in row segments."""
    m, n = 3, 1_300_000          # 10.4 MB per float64 row
    x, y = rng.random(m) * 2 - 1, rng.random(n) * 2 - 1
    res = np.empty(m * n)
    launch_host(plan_outer((m,), (n,)), res, x, y, moa.MUL_ADD)
    assert_bits_equal(res, (np.multiply.outer(x, y) + 0.0).ravel())
    # and a K > 1 product whose B rows exceed a slot (pageable B, A, res)
    k = 4
    a, b = rng.random(m * k), rng.random(k * n)
    res = np.empty(m * n)
    launch_host(plan_inner((m, k), (k, n)), res, a, b, op_pair("add", "max"))
    assert_bits_equal(res, oracle.product(a, b, m, k, n, 0, 3))


def test_concurrent_pageable_callers_share_the_slots(rng):
    """16 threads at once on pageable buffers (more slot demand than the
    per-GPU slot budget): every caller still gets its exact result."""
    from concurrent.futures import ThreadPoolExecutor
    m, k, n = 600, 64, 1800
    a, b = rng.random(m * k), rng.random(k * n)
    plan = plan_inner((m, k), (k, n))
    want = oracle.product(a, b, m, k, n, 0, 2)

    def one(i):
        res = np.full(m * n, np.nan)
        launch_host(plan, res, a, b, op_pair("add", "min"))
        return res
    with ThreadPoolExecutor(16) as pool:
        for got in pool.map(one, range(48)):
            assert_bits_equal(got, want)


def test_short_lived_threads_reuse_pooled_queues(rng):
    """The reference's execute_parallel makes a new thread pool per call
    (parallel.py:37-41); queue sets are pooled per device, not per thread, so
    hundreds of short-lived calling threads neither leak streams nor fail."""
    from concurrent.futures import ThreadPoolExecutor
    m, k, n = 40, 16, 24
    a, b = rng.random(m * k), rng.random(k * n)
    plan = plan_inner((m, k), (k, n))
    want = oracle.product(a, b, m, k, n, 2, 3)
    for _ in range(60):
        res = np.empty(m * n)
        with ThreadPoolExecutor(4) as pool:
            list(pool.map(lambda w: launch_host(plan, res, a, b, op_pair("multiply", "max"),
                                                start=w, step=4), range(4)))
        assert_bits_equal(res, want)


def test_host_result_blocks_are_page_locked_and_reused(rng):
    """Public-API results from 256 KiB up live in moa_host_alloc blocks: huge-page
    backed and page-locked (the copy-back needs no staging), returned to the
    cache when the array dies and reused by the next result of that size."""
    import gc
    torch = _torch()
    from paper_0907_0792_b200 import MoaArray, _native
    x, y = rng.random(1000) * 2 - 1, rng.random(3000) * 2 - 1
    out = moa.outer(MoaArray((1000,), x), MoaArray((3000,), y))
    assert_bits_equal(out.data, (np.multiply.outer(x, y) + 0.0).ravel())
    ptr = out.data.ctypes.data
    assert ptr % (2 << 20) == 0
    t = torch.from_numpy(out.data)
    assert t.is_pinned()  # registered with CUDA
    del out, t
    gc.collect()
    out2 = moa.outer(MoaArray((1000,), y[:1000]), MoaArray((3000,), y))
    assert out2.data.ctypes.data == ptr  # the idle block was reused
    assert_bits_equal(out2.data, (np.multiply.outer(y[:1000], y) + 0.0).ravel())
    # a 320 KiB result is page-locked too (kernel stores straight into it)
    small = moa.outer(MoaArray((200,), x[:200]), MoaArray((200,), y[:200]))
    assert torch.from_numpy(small.data).is_pinned()
    assert_bits_equal(small.data, (np.multiply.outer(x[:200], y[:200]) + 0.0).ravel())
    # the raw allocator: distinct live blocks, reuse after free
    p1, p2 = _native.host_alloc(5 << 20), _native.host_alloc(5 << 20)
    assert p1 and p2 and p1 != p2
    _native.host_free(p1)
    assert _native.host_alloc(5 << 20) == p1
