"""Parity at BASELINE.json's full sizes (all five configs), on the GPU.

* exact-mode and bit-exact routes are compared with the sha256 of the
  reference's own output rows (tests/golden/configs.json) — bit parity at full
  K and N;
* the FP64 tensor-core route is compared with the C port (itself pinned to
  the reference, tests/test_oracle_pins.py) on the same rows within
  K*2^-52*max|A|*max|B|;
* size-independent properties cover the whole output: the outer product
  equals numpy's exact elementwise product everywhere, exact and DMMA routes
  agree within tolerance everywhere.
"""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

import oracle
import paper_0907_0792_b200 as moa
from conftest import GOLDEN
from paper_0907_0792_b200 import MoaArray
from paper_0907_0792_b200.workloads import WORKLOADS
from parity import assert_bits_equal, assert_within, sum_tolerance

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

PINS = json.loads((GOLDEN / "configs.json").read_text())


def _arrays(key, device=True):
    w = WORKLOADS[key]
    a, b = w.generate()
    A = MoaArray(w.shape_a, a, dtype=w.dtype)
    B = MoaArray(w.shape_b, b, dtype=w.dtype)
    if device:
        A, B = A.to_device(), B.to_device()
    return w, a, b, A, B


def _rows(out_dev, rows, n):
    import torch
    idx = torch.tensor(rows, device=out_dev.device)
    return out_dev.view(-1, n).index_select(0, idx).cpu().numpy()


def _product(w, A, B, **kw):
    fn = moa.inner if w.mode == "inner" else moa.outer
    return fn(A, B, w.ops, **kw)


@pytest.mark.parametrize("key", ["c1", "c3", "c4"])
def test_mul_add_configs(key):
    w, a, b, A, B = _arrays(key)
    m, k, n = w.mkn
    pins = PINS[key]
    rows = pins["rows"]
    fast = _product(w, A, B)
    exact = _product(w, A, B, exact=True)
    got_exact = _rows(exact.data, rows, n)
    assert hashlib.sha256(got_exact.tobytes()).hexdigest() == pins["sha256_f64"]
    tol = sum_tolerance(k, a, b)
    got_fast = _rows(fast.data, rows, n)
    a_rows = np.concatenate([a[i * k:(i + 1) * k] for i in rows])
    want = oracle.product(a_rows, b, len(rows), k, n, 2, 0, workers=oracle.host_cores())
    assert_within(got_fast, want.reshape(len(rows), n), tol, key)
    # whole output: tensor-core route within tolerance of the reference-exact route
    import torch
    err = torch.max(torch.abs(fast.data - exact.data)).item()
    assert err <= tol, f"{key}: max |dmma - exact| {err:.3e} > {tol:.3e}"


def test_outer_config_c2_every_element():
    w, a, b, A, B = _arrays("c2")
    out = _product(w, A, B)
    assert out.shape == (32, 16, 16, 8, 16, 16, 8)
    m, _, n = w.mkn
    rows = PINS["c2"]["rows"]
    got_rows = _rows(out.data, rows, n)
    assert hashlib.sha256(got_rows.tobytes()).hexdigest() == PINS["c2"]["sha256_f64"]
    want = (np.multiply.outer(a, b) + 0.0).ravel()  # reduce(0.0, a*b): exact in numpy too
    assert_bits_equal(out.data.cpu().numpy(), want, "c2")


def test_tropical_config_c5_bit_exact():
    w, a, b, A, B = _arrays("c5")
    out = _product(w, A, B)
    assert out.dtype == np.float32
    m, k, n = w.mkn
    rows = PINS["c5"]["rows"]
    got = _rows(out.data, rows, n)
    assert hashlib.sha256(got.tobytes()).hexdigest() == PINS["c5"]["sha256_f32"]
    # size-independent checks over the whole output: an element is +inf iff
    # every pair in its fold has an inf operand, and no NaN appears
    import torch
    assert not torch.isnan(out.data).any().item()
    fin_a = torch.from_numpy(np.isfinite(a).reshape(m, k).astype(np.float32)).cuda()
    fin_b = torch.from_numpy(np.isfinite(b).reshape(k, n).astype(np.float32)).cuda()
    finite_pairs = fin_a @ fin_b  # count of finite pairs per element (exact in f32 < 2^24)
    assert torch.equal(torch.isinf(out.data.view(m, n)), finite_pairs == 0)


def _bits_equal_dev(got, want, msg):
    """Bitwise equality of two CUDA float32 tensors, NaN payloads aside."""
    import torch
    gn, wn = torch.isnan(got), torch.isnan(want)
    assert torch.equal(gn, wn), f"{msg}: NaN positions differ"
    g = got.masked_fill(gn, 0).view(torch.int32)
    w = want.masked_fill(wn, 0).view(torch.int32)
    diff = int((g != w).sum().item())
    assert diff == 0, f"{msg}: {diff} of {g.numel()} elements differ"


@pytest.mark.parametrize("poison", ["none", "negatives", "nan_negzero"])
def test_c5_whole_output_bitwise_against_exact_fold(poison):
    """All 268M elements of the c5 product on the fast route, bit for bit
    against the exact fold: the same inputs upcast to float64 through the
    exact K2 route (bit-pinned to the reference's goldens and to the
    reference's own c5 rows) and rounded once to float32 on the device — the
    reference's result (arrays.py:77-78 upcasts, then float32 is the one
    rounding).  ``none`` is BASELINE c5 (unsigned-order VIMNMX3 fold);
    ``negatives`` forces the FMNMX3 fold (signed operands, no NaN or -0
    result possible); ``nan_negzero`` forces the exact loop (a NaN and -0.0
    in A) — every one of the device-chosen folds checked at full size."""
    import torch
    w, a, b, _, _ = _arrays("c5", device=False)
    m, k, n = w.mkn
    a = a.copy()
    if poison == "negatives":
        rng = np.random.default_rng(44)
        idx = rng.choice(a.size, 1 << 16, replace=False)
        a[idx] = -a[idx]
        a[idx[:7]] = -np.inf
    elif poison == "nan_negzero":
        a[12345] = np.nan
        a[(m - 1) * k + 17] = np.nan
        a[777] = -0.0
    A = MoaArray(w.shape_a, a, dtype=np.float32).to_device()
    B = MoaArray(w.shape_b, b, dtype=np.float32).to_device()
    fast = moa.inner(A, B, w.ops).data
    A64 = MoaArray._wrap(w.shape_a, A.data.to(torch.float64))
    B64 = MoaArray._wrap(w.shape_b, B.data.to(torch.float64))
    assert moa.kernel._native.plan_kernel(0, m, k, n, 0, 2) == "semiring_exact"
    ref = moa.inner(A64, B64, w.ops).data.to(torch.float32)
    del A64, B64
    _bits_equal_dev(fast, ref, f"c5 {poison}")
    if poison == "none":  # and the reference's own rows, hashed
        got = _rows(fast, PINS["c5"]["rows"], n)
        assert hashlib.sha256(got.tobytes()).hexdigest() == PINS["c5"]["sha256_f32"]


def test_c5_rows_sharded_any_gpu_count_bitwise():
    """Row blocks for 2/4/8 shards reproduce the one-shot result bit for bit."""
    import torch
    w, a, b, A, B = _arrays("c5")
    m, k, n = w.mkn
    full = _product(w, A, B).data
    for parts in (2, 8):
        for rows in moa.row_blocks(m, parts)[:2]:
            r0, r1 = rows.start, rows.stop
            sub = moa.inner(MoaArray((r1 - r0, k), A.data[r0 * k:r1 * k]), B, w.ops)
            assert torch.equal(sub.data, full[r0 * n:r1 * n])


def test_index_math_beyond_2_31_elements():
    """Results with more than 2^31 elements (64-bit offsets in every kernel):
    the last rows, where 32-bit offsets would wrap, match the oracle."""
    import torch
    from paper_0907_0792_b200.kernel import launch, plan_inner, plan_outer
    rng = np.random.default_rng(5)
    # outer product, float32: 70000 x 32768 = 2.29e9 elements
    m, n = 70000, 32768
    a = rng.random(m, dtype=np.float32)
    b = rng.random(n, dtype=np.float32)
    c = torch.empty(m * n, dtype=torch.float32, device="cuda")
    launch(plan_outer((m,), (n,)), c, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(),
           moa.op_pair("add", "max"))
    tail = c[(m - 3) * n:].cpu().numpy().reshape(3, n)
    assert_bits_equal(tail, (a[-3:, None] + b[None, :]).astype(np.float32))
    del c
    # inner products with M*N > 2^31: DMMA (f64) and tropical (f32)
    for ops, dt, (m, k, n) in ((moa.MUL_ADD, np.float64, (50000, 8, 45000)),
                               (moa.op_pair("add", "min"), np.float32, (50000, 6, 45000))):
        a = rng.random(m * k).astype(dt)
        b = rng.random(k * n).astype(dt)
        tdt = torch.float64 if dt == np.float64 else torch.float32
        c = torch.empty(m * n, dtype=tdt, device="cuda")
        launch(plan_inner((m, k), (k, n)), c, torch.from_numpy(a).cuda(),
               torch.from_numpy(b).cuda(), ops)
        got = c[(m - 2) * n:].cpu().numpy()
        comb, red = ops.codes()
        want = oracle.product(a[(m - 2) * k:], b, 2, k, n, comb, red)
        if dt == np.float64:
            assert_within(got, want, sum_tolerance(k, a, b))
        else:
            assert_bits_equal(got, want.astype(np.float32))
        del c
        torch.cuda.empty_cache()
