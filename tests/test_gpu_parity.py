"""GPU parity: every golden case the reference produced, through the public API
(which calls the C ABI), plus the properties the reference's tests assert
(unification, determinism across workers, psi-row law) and the edge cases of
the device kernels (ragged tiles, unaligned rows, row subsets, accumulate).

Bar: bit-exact (NaN payload aside) for every pair except (multiply, add) on
float64 without ``exact``, which runs on the FP64 tensor cores and must be
within K*2^-52*max|A|*max|B| (BASELINE.json north_star)."""

from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
import paper_0907_0792_b200 as moa
from paper_0907_0792_b200 import MoaArray, op_pair
from paper_0907_0792_b200.kernel import KernelPlan, launch, plan_inner, plan_outer
from parity import assert_bits_equal, assert_within, sum_tolerance

pytestmark = [pytest.mark.gpu, pytest.mark.filterwarnings("ignore::RuntimeWarning")]

MUL, ADD = 2, 0


def _torch():
    import torch
    return torch


def _run(case, exact=False, device=False, workers=1):
    dt = case.a.dtype
    a = MoaArray(case.shape_a, case.a, dtype=dt)
    b = MoaArray(case.shape_b, case.b, dtype=dt)
    if device:
        a, b = a.to_device(), b.to_device()
    ops = op_pair(list(moa.COMBINE_OPS)[case.comb], list(moa.REDUCE_OPS)[case.red])
    fn = moa.inner if case.mode == "inner" else moa.outer
    out = fn(a, b, ops, workers=workers, exact=exact)
    want_shape = (case.shape_a[:-1] + case.shape_b[1:]) if case.mode == "inner" \
        else case.shape_a + case.shape_b
    assert out.shape == want_shape
    return out.host_data()


DMMA_MIN_K = 8  # capi.cu kDmmaMinK: below it (multiply, add) takes the exact fold


def _is_dmma(case) -> bool:
    return case.comb == MUL and case.red == ADD and case.a.dtype == np.float64 and \
        case.mode == "inner" and case.shape_a[-1] >= DMMA_MIN_K


def _check(case, got, exact=False):
    want = case.out
    if got.dtype.kind == "i":  # integer-valued reference result, exact
        assert got.dtype == case.a.dtype, repr(case)
        np.testing.assert_array_equal(got, want.astype(got.dtype), err_msg=repr(case))
    elif got.dtype == np.float32:
        assert_bits_equal(got, want.astype(np.float32), repr(case))
    elif _is_dmma(case) and not exact:
        k = case.shape_a[-1]
        assert_within(got, want, sum_tolerance(k, case.a, case.b), repr(case))
    else:
        assert_bits_equal(got, want, repr(case))


def test_golden_cases_bitwise(golden_small):
    """Every golden case on the default route, specials included: bit-exact,
    except (multiply, add) float64 with K >= 8 (DMMA), within the sum bound."""
    for case in golden_small:
        _check(case, _run(case))


def test_default_route_is_the_reference_below_one_dmma_k_group(golden_small):
    """Every (multiply, add) float64 golden case with K < 8 — the reference's
    special-value cases (NaN, +-inf, +-0, subnormals, +-1e308) among them —
    is bit-exact on the default route, not just within tolerance."""
    seen = 0
    for case in golden_small:
        if case.comb == MUL and case.red == ADD and case.a.dtype == np.float64 and \
                case.mode == "inner" and 0 < case.shape_a[-1] < DMMA_MIN_K:
            assert_bits_equal(_run(case), case.out, repr(case))
            seen += 1
    assert seen >= 15


def _random_array(rng, rank, max_extent=5):
    shape = tuple(int(e) for e in rng.integers(1, max_extent + 1, size=rank))
    return MoaArray(shape, rng.random(math.prod(shape)) * 3.0 - 1.0)


def test_criterion_1_oracle_equivalence_default_route():
    """reference tests/test_acceptance.py:34-53 on the default (fast) routes:
    1000 random cases over every built-in pair, half inner products of ranks
    1..4 with extents 1..5, half outer products, values in [-1, 2); each
    element within rtol 1e-12 (atol 0) of the oracle, min/max folds exact."""
    rng = np.random.default_rng(1001)
    pairs = list(moa.builtin_pairs())
    for case in range(1000):
        ops = pairs[case % len(pairs)]
        comb, red = ops.codes()
        if rng.random() < 0.5:
            ra, rb = int(rng.integers(1, 5)), int(rng.integers(1, 5))
            shared = int(rng.integers(1, 6))
            sa = tuple(int(e) for e in rng.integers(1, 6, size=ra - 1)) + (shared,)
            sb = (shared,) + tuple(int(e) for e in rng.integers(1, 6, size=rb - 1))
            a = MoaArray(sa, rng.random(math.prod(sa)) * 3.0 - 1.0)
            b = MoaArray(sb, rng.random(math.prod(sb)) * 3.0 - 1.0)
            got = moa.inner(a, b, ops)
            m, k = math.prod(sa[:-1]), shared
            n = math.prod(sb[1:])
        else:
            a = _random_array(rng, int(rng.integers(1, 5)))
            b = _random_array(rng, int(rng.integers(1, 5)))
            got = moa.outer(a, b, ops)
            m, k, n = a.count, 1, b.count
        want = oracle.product(a.data, b.data, m, k, n, comb, red)
        if ops.reduce_name in ("min", "max"):
            np.testing.assert_array_equal(got.data, want, err_msg=f"case {case} {ops}")
        else:
            np.testing.assert_allclose(got.data, want, rtol=1e-12, atol=0.0, equal_nan=True,
                                       err_msg=f"case {case} {ops}")


def _special_operand(rng, size, span):
    """Uniform [-1, 1) with NaN, +-inf, +-0 and subnormals, each at rate 1/span."""
    x = rng.uniform(-1.0, 1.0, size)
    kinds = rng.integers(0, span, size)
    x[kinds == 0] = np.nan
    x[kinds == 1] = np.inf
    x[kinds == 2] = -np.inf
    x[kinds == 3] = 0.0
    x[kinds == 4] = -0.0
    sub = kinds == 5
    x[sub] = rng.uniform(-1, 1, int(sub.sum())) * 2.0**-1060  # subnormal
    return x


@pytest.mark.parametrize("mkn", [(96, 8, 40),       # smallest DMMA K
                                 (200, 64, 136),    # 16x32 TMA tiles
                                 (2048, 48, 512),   # 64x64 TMA tiles
                                 (301, 37, 203)])   # unaligned: cp.async kernel
def test_dmma_route_ieee_specials(mkn, rng):
    """The FP64 tensor-core route on NaN, +-inf, +-0 and subnormal operands:
    the same NaN positions and the same infinities (signs included) as the
    reference's loop, finite elements within K*2^-52*max|A|*max|B| over the
    finite operands.  The one exception is overflow near DBL_MAX (the fused
    DMMA step does not overflow where the reference's separate product does),
    so values near 1e308 stay out of this set; include/moa_b200.h says so."""
    m, k, n = mkn
    for span in (600, 40):  # sparse specials (mostly finite results), dense
        a = _special_operand(rng, m * k, span)
        b = _special_operand(rng, k * n, span)
        assert moa.kernel._native.plan_kernel(0, m, k, n, MUL, ADD) == "dmma"
        got = moa.inner(MoaArray((m, k), a), MoaArray((k, n), b)).data
        want = oracle.product(a, b, m, k, n, MUL, ADD)
        fa, fb = a[np.isfinite(a)], b[np.isfinite(b)]
        assert_within(got, want, sum_tolerance(k, fa, fb), f"{mkn} span {span}")
        assert np.isnan(want).any()
        if span == 600:
            assert np.isfinite(want).mean() > 0.3


def test_golden_cases_exact_mode_bitwise_everywhere(golden_small):
    """exact=True reproduces the reference's (multiply, add) rounding too."""
    for case in golden_small:
        got = _run(case, exact=True)
        if got.dtype.kind == "i":
            np.testing.assert_array_equal(got, case.out.astype(got.dtype), err_msg=repr(case))
        elif got.dtype == np.float32:
            assert_bits_equal(got, case.out.astype(np.float32), repr(case))
        else:
            assert_bits_equal(got, case.out, repr(case))


def test_golden_cases_device_resident(golden_small):
    for case in golden_small[::5]:
        _check(case, _run(case, device=True))


def test_golden_cases_parallel_workers(golden_small):
    for case in golden_small[::11]:
        for w in (2, 3, 8):
            _check(case, _run(case, workers=w))


def test_hand_answers():
    a = MoaArray((2, 3), [1, 2, 3, 4, 5, 6])
    b = MoaArray((3, 4), range(12))
    c = moa.inner(a, b)
    assert moa.psi_select((0,), c).data.tolist() == [32.0, 38.0, 44.0, 50.0]
    assert c.data.tolist() == [32, 38, 44, 50, 68, 83, 98, 113]
    assert moa.inner(MoaArray((3,), [1, 2, 3]), MoaArray((3,), [4, 5, 6])).item() == 32.0
    assert moa.outer(MoaArray((2,), [1, 2]), MoaArray((2,), [10, 20])).data.tolist() == \
        [10, 20, 20, 40]
    trop = moa.inner(MoaArray((2,), [1, 2]), MoaArray((2,), [10, 20]), op_pair("add", "min"))
    assert trop.item() == 11.0
    e = moa.inner(MoaArray((2, 0), []), MoaArray((0, 3), []), op_pair("multiply", "min"))
    assert e.data.tolist() == [math.inf] * 6
    z = moa.inner(MoaArray((0, 3), []), MoaArray((3, 4), range(12)))
    assert z.shape == (0, 4) and z.count == 0
    assert moa.execute_parallel(moa.plan_inner((2, 3), (3, 4)), a, b, workers=3).data.tolist() == \
        [32, 38, 44, 50, 68, 83, 98, 113]


def test_outer_signed_zero_semantics():
    a, b = MoaArray((), [-1.0]), MoaArray((), [0.0])
    assert not np.signbit(moa.outer(a, b).item())                           # (x,+): +0.0
    assert np.signbit(moa.outer(a, b, op_pair("multiply", "min")).item())   # (x,min): -0.0
    assert np.signbit(moa.outer(a, b, op_pair("multiply", "multiply")).item())


def test_min_fold_nan_not_sticky_and_zero_tie():
    # fold over [5, NaN, 7] gives 7; a min(-0, +0) tie gives the later +0
    a = MoaArray((1, 3), [5.0, math.nan, 7.0])
    b = MoaArray((3, 1), [0.0, 0.0, 0.0])
    for dt in (np.float64, np.float32):
        got = moa.inner(MoaArray(a.shape, a.data, dtype=dt), MoaArray(b.shape, b.data, dtype=dt),
                        op_pair("add", "min")).item()
        assert got == 7.0
    z = moa.inner(MoaArray((1, 2), [-0.0, 0.0]), MoaArray((2, 1), [0.0, 0.0]),
                  op_pair("add", "min")).item()
    assert z == 0.0 and not np.signbit(z)


def test_outer_unifies_with_rowsinred_one_inner(rng):
    """reference tests/test_acceptance.py:56-68: outer == K=1 inner, bitwise."""
    for _ in range(60):
        sa = tuple(int(e) for e in rng.integers(1, 5, size=int(rng.integers(0, 4))))
        sb = tuple(int(e) for e in rng.integers(1, 5, size=int(rng.integers(0, 4))))
        a = MoaArray(sa, rng.random(math.prod(sa)) * 3 - 1)
        b = MoaArray(sb, rng.random(math.prod(sb)) * 3 - 1)
        for ops in (op_pair("multiply", "add"), op_pair("divide", "max")):
            via_outer = moa.outer(a, b, ops)
            via_inner = moa.inner(moa.reshape(a, (a.count, 1)), moa.reshape(b, (1, b.count)), ops)
            assert_bits_equal(via_outer.data, via_inner.data)


def test_psi_row_law(rng):
    for ops in (op_pair("multiply", "add"), op_pair("add", "min")):
        a = MoaArray((4, 3), rng.random(12))
        b = MoaArray((3, 5), rng.random(15))
        c = moa.inner(a, b, ops, exact=True)
        for i in range(4):
            acc = [ops.reduce_identity] * 5
            for l in range(3):
                ail = moa.psi_select((i, l), a).item()
                row = moa.psi_select((l,), b).data
                acc = [ops.reduce(acc[j], ops.combine(ail, float(row[j]))) for j in range(5)]
            assert_bits_equal(moa.psi_select((i,), c).data, np.array(acc))


# ---- kernel-level edge cases through the C ABI --------------------------------

def _dev(x, dtype=None):
    torch = _torch()
    t = torch.from_numpy(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def _pairs_sample():
    return [op_pair(c, r) for c in moa.COMBINE_OPS for r in moa.REDUCE_OPS]


@pytest.mark.parametrize("mkn", [(1, 1, 1), (5, 17, 3), (129, 33, 130), (64, 16, 64),
                                 (300, 41, 257), (7, 1, 300), (1000, 3, 9)])
def test_ragged_shapes_all_pairs_vs_port(mkn, rng):
    m, k, n = mkn
    a = rng.random(m * k) * 3 - 1
    b = rng.random(k * n) * 3 - 1
    for ops in _pairs_sample():
        c, r = ops.codes()
        want = oracle.product(a, b, m, k, n, c, r)
        got = moa.inner(MoaArray((m, k), a), MoaArray((k, n), b), ops).data
        if (c, r) == (MUL, ADD) and k > 1:
            assert_within(got, want, sum_tolerance(k, a, b), f"{mkn} {ops}")
        else:
            assert_bits_equal(got, want, f"{mkn} {ops}")


@pytest.mark.parametrize("mkn", [(129, 33, 130), (300, 41, 257)])
def test_float32_all_pairs_with_specials_vs_port(mkn, rng):
    """float32 storage, every pair, data with zeros, infinities, NaN and
    subnormals: the reference's float64 result rounded once, bit for bit
    (including (multiply, add), which runs as DFMA on exact float products)."""
    m, k, n = mkn
    a = ((rng.random(m * k) * 3 - 1) * 10.0 ** rng.integers(-3, 4, m * k)).astype(np.float32)
    b = ((rng.random(k * n) * 3 - 1) * 10.0 ** rng.integers(-3, 4, k * n)).astype(np.float32)
    for x in (a, b):
        idx = rng.choice(x.size, size=x.size // 20, replace=False)
        x[idx] = rng.choice(np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -3e-39],
                                     dtype=np.float32), size=idx.size)
    for ops in _pairs_sample():
        c, r = ops.codes()
        want = oracle.product(a, b, m, k, n, c, r).astype(np.float32)
        got = moa.inner(MoaArray((m, k), a, dtype=np.float32), MoaArray((k, n), b, dtype=np.float32),
                        ops).data
        assert_bits_equal(got, want, f"{mkn} {ops}")


def test_round_robin_row_sets_fill_the_same_result(rng):
    """Worker k of W launching rows k::W into one buffer == one full launch
    (parallel.py:38-42 on the device), for every kernel route."""
    torch = _torch()
    m, k, n = 333, 45, 270
    a = rng.random(m * k) * 3 - 1
    b = rng.random(k * n) * 3 - 1
    plan = plan_inner((m, k), (k, n))
    for ops in (op_pair("multiply", "add"), op_pair("add", "min"), op_pair("divide", "max")):
        for dt in (torch.float64, torch.float32):
            ad, bd = _dev(a, dt), _dev(b, dt)
            full = torch.empty(m * n, dtype=dt, device="cuda")
            launch(plan, full, ad, bd, ops)
            for w in (2, 3, 8):
                part = torch.full((m * n,), float("nan"), dtype=dt, device="cuda")
                for kk in range(w):
                    launch(plan, part, ad, bd, ops, start=kk, step=w)
                assert_bits_equal(part.cpu().numpy(), full.cpu().numpy(), f"{ops} {dt} W={w}")


def test_outer_row_sets(rng):
    torch = _torch()
    m, n = 1000, 4096
    a, b = rng.random(m) * 3 - 1, rng.random(n) * 3 - 1
    plan = plan_outer((m,), (n,))
    ad, bd = _dev(a), _dev(b)
    full = torch.empty(m * n, dtype=torch.float64, device="cuda")
    launch(plan, full, ad, bd, moa.MUL_ADD)
    part = torch.full((m * n,), float("nan"), dtype=torch.float64, device="cuda")
    for kk in range(5):
        launch(plan, part, ad, bd, moa.MUL_ADD, start=kk, step=5)
    assert_bits_equal(part.cpu().numpy(), full.cpu().numpy())
    assert_bits_equal(full.cpu().numpy(), (np.multiply.outer(a, b) + 0.0).ravel())


@pytest.mark.parametrize("dt", [np.float64, np.float32, np.int32, np.int64])
@pytest.mark.parametrize("mn", [(300, 512), (301, 70), (64, 9)])  # vec / scalar / flat kernels
def test_outer_kernels_every_dtype_and_accumulate(dt, mn, rng):
    """The three outer-product kernels for every element type, write-only and
    accumulating, all 24 pairs: the reference's fold of one term into res."""
    torch = _torch()
    m, n = mn
    if np.dtype(dt).kind == "i":
        a = rng.integers(-50, 50, m).astype(dt)
        b = rng.integers(-50, 50, n).astype(dt)
        init = rng.integers(-50, 50, m * n).astype(dt)
    else:
        a = ((rng.random(m) * 3 - 1) * 10.0 ** rng.integers(-2, 3, m)).astype(dt)
        b = ((rng.random(n) * 3 - 1) * 10.0 ** rng.integers(-2, 3, n)).astype(dt)
        b[::17] = 0.0
        init = (rng.random(m * n) * 3 - 1).astype(dt)
    plan = plan_outer((m,), (n,))
    for ops in _pairs_sample():
        c, r = ops.codes()
        for acc in (False, True):
            res = _dev(init.copy()) if acc else torch.empty(m * n, dtype=_dev(a).dtype, device="cuda")
            launch(plan, res, _dev(a), _dev(b), ops, accumulate=acc)
            got = res.cpu().numpy()
            if np.dtype(dt).kind == "i":
                wi = oracle.product(a.astype(np.float64), b.astype(np.float64), m, 1, n, c, r,
                                    res=init.astype(np.float64) if acc else None)
                if c == 3:  # integer division truncates (x/0 = 0); compare on the exact cases
                    continue
                np.testing.assert_array_equal(got, wi.astype(dt), err_msg=f"{ops} acc={acc}")
            else:
                want = oracle.product(a, b, m, 1, n, c, r,
                                      res=init.astype(np.float64) if acc else None)
                assert_bits_equal(got, want.astype(dt), f"{np.dtype(dt).name} {ops} acc={acc}")


def test_accumulate_mode_matches_reference_semantics(rng):
    """MOA_FLAG_ACCUMULATE folds into res's contents, like _ckernel.product_rows."""
    torch = _torch()
    m, k, n = 70, 37, 90
    a = rng.random(m * k) * 3 - 1
    b = rng.random(k * n) * 3 - 1
    init = rng.random(m * n) * 3 - 1
    plan = plan_inner((m, k), (k, n))
    for ops in _pairs_sample():
        c, r = ops.codes()
        want = oracle.product(a, b, m, k, n, c, r, res=init.copy())
        res = _dev(init.copy())
        launch(plan, res, _dev(a), _dev(b), ops, accumulate=True, exact=True)
        assert_bits_equal(res.cpu().numpy(), want, f"{ops}")
        if (c, r) == (MUL, ADD):
            res = _dev(init.copy())
            launch(plan, res, _dev(a), _dev(b), ops, accumulate=True)
            tol = sum_tolerance(k, a, b) + (k + 1) * 2.0**-52 * float(np.max(np.abs(init)))
            assert_within(res.cpu().numpy(), want, tol, f"{ops}")


def test_unaligned_operands_and_odd_strides(rng):
    """Element offsets that break 16/32-byte alignment take the narrow-copy
    paths; results must not change."""
    torch = _torch()
    m, k, n = 150, 35, 133
    a = rng.random(m * k + 1) * 3 - 1
    b = rng.random(k * n + 1) * 3 - 1
    plan = plan_inner((m, k), (k, n))
    for ops in (op_pair("multiply", "add"), op_pair("add", "min"), op_pair("multiply", "max")):
        c, r = ops.codes()
        want = oracle.product(a[1:], b[1:], m, k, n, c, r)
        ad, bd = _dev(a), _dev(b)
        res = torch.empty(m * n + 1, dtype=torch.float64, device="cuda")
        launch(plan, res[1:], ad[1:], bd[1:], ops)
        got = res[1:].cpu().numpy()
        if (c, r) == (MUL, ADD):
            assert_within(got, want, sum_tolerance(k, a, b))
        else:
            assert_bits_equal(got, want)
    # outer with odd N and misaligned result: scalar path
    m, n = 333, 1001
    x, y = rng.random(m + 1), rng.random(n)
    res = torch.empty(m * n + 1, dtype=torch.float64, device="cuda")
    launch(plan_outer((m,), (n,)), res[1:], _dev(x)[1:], _dev(y), op_pair("subtract", "max"))
    assert_bits_equal(res[1:].cpu().numpy(), np.subtract.outer(x[1:], y).ravel())


def test_dmma_tile_configs_bitwise_identical(rng):
    """Every (multiply, add) kernel configuration — TMA 64x64 (aligned, many
    rows), cp.async 64x128 / 64x64 (rows misaligned for TMA), cp.async 32x32
    (few rows) — accumulates in the same k order, so shared rows are bitwise
    equal (the GPU-count determinism argument)."""
    torch = _torch()
    m, k, n = 4096, 300, 2048
    a = rng.random(m * k + 1) * 2 - 1
    b = rng.random(k * n) * 2 - 1
    bd = _dev(b)
    outs = []
    for shift in (0, 1):  # shift 1: 8-byte aligned A rows, TMA ineligible
        ad = _dev(a)[shift:shift + m * k]
        full = torch.empty(m * n, dtype=torch.float64, device="cuda")
        launch(plan_inner((m, k), (k, n)), full, ad, bd, moa.MUL_ADD)
        full = full.cpu().numpy()
        # rows: 64 (small), 130 (small), 400 (TMA / cp.async medium), 96 (small)
        for r0, r1 in ((0, 64), (1000, 1130), (1000, 1400), (4000, 4096)):
            sub = torch.empty((r1 - r0) * n, dtype=torch.float64, device="cuda")
            launch(plan_inner((r1 - r0, k), (k, n)), sub, ad[r0 * k:r1 * k], bd, moa.MUL_ADD)
            assert_bits_equal(sub.cpu().numpy(), full[r0 * n:r1 * n], f"shift={shift} {r0}:{r1}")
        want = oracle.product(a[shift:shift + 64 * k], b, 64, k, n, MUL, ADD)
        assert_within(full[:64 * n], want, sum_tolerance(k, a, b))
        outs.append(full)
    # same A values at both alignments except the one-element shift: compare
    # the aligned run on a[1:] through a copy instead
    ad = _dev(np.ascontiguousarray(a[1:1 + m * k]))
    again = torch.empty(m * n, dtype=torch.float64, device="cuda")
    launch(plan_inner((m, k), (k, n)), again, ad, bd, moa.MUL_ADD)
    assert_bits_equal(again.cpu().numpy(), outs[1], "TMA vs cp.async large tiles")


def test_dmma_tma_edges_bitwise_equal_cp_async_path(rng):
    """The TMA-staged kernel (dmma_tma.cu, taken when >= 148 64x64 tiles and
    even row strides) against the cp.async kernels on row subsets: ragged M and
    N, K not a multiple of the 16-deep slab (TMA zero fill), round-robin rows
    (lda = K*step), and accumulate mode — all bitwise equal, and within the
    north_star tolerance of the reference."""
    torch = _torch()
    m, k, n = 1000, 38, 2102
    a = rng.random(m * k) * 2 - 1
    b = rng.random(k * n) * 2 - 1
    init = rng.random(m * n) * 2 - 1
    ad, bd = _dev(a), _dev(b)
    plan = plan_inner((m, k), (k, n))
    for acc in (False, True):
        full = _dev(init.copy())
        launch(plan, full, ad, bd, moa.MUL_ADD, accumulate=acc)
        full = full.cpu().numpy()
        for r0, r1 in ((0, 64), (936, 1000), (400, 650)):
            sub = _dev(init[r0 * n:r1 * n].copy())
            launch(plan_inner((r1 - r0, k), (k, n)), sub, ad[r0 * k:r1 * k], bd, moa.MUL_ADD,
                   accumulate=acc)
            assert_bits_equal(sub.cpu().numpy(), full[r0 * n:r1 * n], f"acc={acc} rows {r0}:{r1}")
        want = oracle.product(a, b, m, k, n, MUL, ADD, res=init.copy() if acc else None)
        tol = sum_tolerance(k, a, b) + (k + 1) * 2.0**-52 * float(np.max(np.abs(init)))
        assert_within(full, want, tol, f"acc={acc}")
    # every other row (lda = 2K, ldc = 2N), as execute_parallel's round-robin
    # row sets give
    big = rng.random(2 * m * k) * 2 - 1
    res = torch.zeros(2 * m * n, dtype=torch.float64, device="cuda")
    launch(plan_inner((2 * m, k), (k, n)), res, _dev(big), bd, moa.MUL_ADD, start=1, step=2)
    got = res.cpu().numpy().reshape(2 * m, n)
    assert not got[0::2].any()
    rows = np.ascontiguousarray(big.reshape(2 * m, k)[1::2]).ravel()
    ref = torch.empty(64 * n, dtype=torch.float64, device="cuda")
    launch(plan_inner((64, k), (k, n)), ref, _dev(rows[:64 * k]), bd, moa.MUL_ADD)
    assert_bits_equal(got[1::2][:64].ravel(), ref.cpu().numpy())
    assert_within(got[1::2].ravel(), oracle.product(rows, b, m, k, n, MUL, ADD),
                  sum_tolerance(k, rows, b))


@pytest.mark.parametrize("mkn", [(70, 610, 258),    # <= 148 16x32 tiles: 8-stage ring, refills
                                 (600, 610, 300),   # > 148 tiles: 4-stage ring
                                 (256, 256, 256)])  # BASELINE c1: whole K in flight
def test_dmma_tiny_tma_bitwise_equal_cp_async_path(mkn, rng):
    """Problems below one wave of 64x64 tiles take the 16x32-tile TMA kernel
    when rows are 16-byte aligned and the cp.async tiles otherwise: same k
    order, so bitwise equal, in write-only and accumulate mode, with ragged M/N
    and K past the pipeline depth (ring refills)."""
    torch = _torch()
    m, k, n = mkn
    a = rng.random(m * k + 1) * 2 - 1
    b = rng.random(k * n) * 2 - 1
    init = rng.random(m * n) * 2 - 1
    bd = _dev(b)
    aligned = _dev(np.ascontiguousarray(a[1:]))
    shifted = _dev(a)[1:]  # 8-byte aligned A rows: TMA ineligible
    plan = plan_inner((m, k), (k, n))
    for acc in (False, True):
        outs = []
        for ad in (aligned, shifted):
            c = _dev(init.copy())
            launch(plan, c, ad, bd, moa.MUL_ADD, accumulate=acc)
            outs.append(c.cpu().numpy())
        assert_bits_equal(outs[0], outs[1], f"acc={acc}")
        want = oracle.product(a[1:], b, m, k, n, MUL, ADD, res=init.copy() if acc else None)
        tol = sum_tolerance(k, a, b) + (k + 1) * 2.0**-52 * float(np.max(np.abs(init)))
        assert_within(outs[0], want, tol, f"acc={acc}")
    torch.cuda.synchronize()


def test_dmma_accumulate_launches_repeat_bitwise(rng):
    """Accumulate-mode TMA DMMA launches over a zero-filled C, repeated: every
    one equals the write-only launch bit for bit (an mbarrier-init / TMA-issue
    ordering race once broke a few warps' results intermittently, only in
    this mode); the float32 tropical TMA kernel likewise."""
    torch = _torch()
    m, k, n = 4096, 256, 4096  # ~1 launch in 20 went wrong here before the fix
    a, b = _dev(rng.random(m * k) * 100), _dev(rng.random(k * n) * 100)
    plan = plan_inner((m, k), (k, n))
    want = torch.empty(m * n, dtype=torch.float64, device="cuda")
    launch(plan, want, a, b, moa.MUL_ADD)
    c = torch.empty_like(want)
    for trial in range(80):
        c.zero_()
        launch(plan, c, a, b, moa.MUL_ADD, accumulate=True)
        assert torch.equal(c, want), f"accumulate launch {trial}"
    # the 16x32-tile TMA kernel with its ring refilling (K = 1024 > 8 stages x 32)
    mt, kt_, nt = 256, 1024, 256
    at, bt = _dev(rng.random(mt * kt_) * 100), _dev(rng.random(kt_ * nt) * 100)
    plan_t = plan_inner((mt, kt_), (kt_, nt))
    want_t = torch.empty(mt * nt, dtype=torch.float64, device="cuda")
    launch(plan_t, want_t, at, bt, moa.MUL_ADD)
    ct = torch.empty_like(want_t)
    for trial in range(80):
        ct.zero_()
        launch(plan_t, ct, at, bt, moa.MUL_ADD, accumulate=True)
        assert torch.equal(ct, want_t), f"16x32-tile accumulate launch {trial}"
    ops = op_pair("add", "min")
    a32, b32 = a.float(), b.float()
    want32 = torch.empty(m * n, dtype=torch.float32, device="cuda")
    launch(plan, want32, a32, b32, ops)
    c32 = torch.empty_like(want32)
    for trial in range(30):
        c32.fill_(float("inf"))
        launch(plan, c32, a32, b32, ops, accumulate=True)
        assert torch.equal(c32, want32), f"tropical accumulate launch {trial}"


@pytest.mark.parametrize("dt,mkn", [(np.float32, (257, 131, 300)),   # odd K, unaligned: cp.async
                                    (np.float32, (1000, 132, 1004)),  # 16-byte rows: TMA kernel
                                    (np.float64, (257, 131, 300))])   # exact fold, specials
def test_tropical_fast_and_exact_loops_agree(dt, mkn, rng):
    """(add|subtract, min|max): the float32 fast folds (clean data) and the
    compare-select loop (float64, and data with NaN/-0) all equal the
    reference.  (A float64 fmin/fmax fold was tried: sm_100a has no DMNMX, it
    lowers to DSETP + selects and ran 24% slower than compare-select.)"""
    m, k, n = mkn  # odd K: the last k of the last tile takes the scalar tail
    for comb in ("add", "subtract"):
        for red in ("min", "max"):
            ops = op_pair(comb, red)
            c, r = ops.codes()
            a = (rng.random(m * k) * 100).astype(dt)
            b = (rng.random(k * n) * 100).astype(dt)
            a[rng.random(m * k) < 0.05] = np.inf
            b[rng.random(k * n) < 0.05] = np.inf if comb == "add" else -np.inf
            for poison in (None, "nan", "negzero", "negative"):
                aa, bb = a.copy(), b.copy()
                if poison == "negative":  # sign bits set: FMNMX3 loop instead of VIMNMX3
                    aa = aa - dt(50)
                elif poison == "nan":
                    aa[rng.random(m * k) < 0.01] = np.nan
                elif poison == "negzero":
                    aa[rng.random(m * k) < 0.05] = -0.0
                    bb[rng.random(k * n) < 0.05] = -0.0 if comb == "add" else 0.0
                want = oracle.product(aa, bb, m, k, n, c, r).astype(dt)
                got = moa.inner(MoaArray((m, k), aa, dtype=dt),
                                MoaArray((k, n), bb, dtype=dt), ops).data
                assert got.dtype == dt
                assert_bits_equal(got, want, f"{ops} poison={poison}")


def _identity(ops, dt):
    if np.dtype(dt).kind == "f":
        return ops.reduce_identity
    info = np.iinfo(dt)
    return {"add": 0, "multiply": 1, "min": info.max, "max": info.min}[ops.reduce_name]


@pytest.mark.parametrize("mkn", [(200, 132, 260), (130, 67, 97)])  # aligned / unaligned
def test_accumulate_from_identity_equals_write_only_every_route(mkn, rng):
    """The reference's contract for its loop (kernel.py:149 + _ckernel.pyx:51,70):
    folding into a result prefilled with the reduce identity gives the same
    bits as the write-only launch — for all 24 (combine, reduce) pairs on
    every dtype, through every kernel route (TMA and cp.async tiles, fast and
    exact folds, DPX, division)."""
    torch = _torch()
    m, k, n = mkn
    plan = plan_inner((m, k), (k, n))
    for dt in (np.float64, np.float32, np.int32, np.int64):
        if np.dtype(dt).kind == "f":
            a, b = (rng.random(m * k) * 9 + 0.5).astype(dt), (rng.random(k * n) * 9 + 0.5).astype(dt)
        else:
            a, b = rng.integers(1, 9, m * k).astype(dt), rng.integers(1, 9, k * n).astype(dt)
        ad, bd = _dev(a), _dev(b)
        for ops in moa.builtin_pairs():
            w = torch.empty(m * n, dtype=ad.dtype, device="cuda")
            launch(plan, w, ad, bd, ops)
            acc = torch.full((m * n,), _identity(ops, dt), dtype=ad.dtype, device="cuda")
            launch(plan, acc, ad, bd, ops, accumulate=True)
            assert_bits_equal(acc.cpu().numpy(), w.cpu().numpy(),
                              f"{np.dtype(dt).name} {ops} {mkn}")


@pytest.mark.parametrize("mkn", [(200, 132, 260), (130, 67, 97)])
def test_row_sets_equal_full_launch_every_route(mkn, rng):
    """execute_parallel's determinism (tests/test_acceptance.py:84-103 of the
    reference): the rows 0::2 and 1::2 launched separately, and a contiguous
    row block launched as its own product, give the bits of one full launch —
    for all 24 pairs on every dtype (so sharding rows over workers or GPUs
    never changes a result)."""
    torch = _torch()
    m, k, n = mkn
    plan = plan_inner((m, k), (k, n))
    r0, r1 = m // 3, m // 3 + 64
    for dt in (np.float64, np.float32, np.int32, np.int64):
        if np.dtype(dt).kind == "f":
            a, b = (rng.random(m * k) * 9 + 0.5).astype(dt), (rng.random(k * n) * 9 + 0.5).astype(dt)
        else:
            a, b = rng.integers(1, 9, m * k).astype(dt), rng.integers(1, 9, k * n).astype(dt)
        ad, bd = _dev(a), _dev(b)
        for ops in moa.builtin_pairs():
            full = torch.empty(m * n, dtype=ad.dtype, device="cuda")
            launch(plan, full, ad, bd, ops)
            parts = torch.empty_like(full)
            launch(plan, parts, ad, bd, ops, start=0, step=2)
            launch(plan, parts, ad, bd, ops, start=1, step=2)
            assert_bits_equal(parts.cpu().numpy(), full.cpu().numpy(),
                              f"{np.dtype(dt).name} {ops} rows k::2")
            blk = torch.empty((r1 - r0) * n, dtype=ad.dtype, device="cuda")
            launch(plan_inner((r1 - r0, k), (k, n)), blk, ad[r0 * k:r1 * k], bd, ops)
            assert_bits_equal(blk.cpu().numpy(), full[r0 * n:r1 * n].cpu().numpy(),
                              f"{np.dtype(dt).name} {ops} rows {r0}:{r1}")


@pytest.mark.parametrize("mkn", [(300, 132, 260),    # TMA kernel, 64x128 tiles
                                 (257, 131, 300),    # cp.async kernel
                                 (2049, 37, 2052)])  # TMA kernel, >= 256 128x128 tiles, ragged
def test_tropical_accumulate_seeds(mkn, rng):
    """float32 (add|subtract|multiply, min|max) under MOA_FLAG_ACCUMULATE with
    the reference's identity prefill (+-inf), with negative and with mixed
    seeds: the unsigned-order max fold replaces negative seeds by +0 (they can
    never win against results >= +0), a min fold with negative seeds leaves
    the fast loop (multiply has no FMNMX3 kernel: it once ran nothing and left
    the -inf prefill in place).  Bitwise vs the reference's fold from res."""
    torch = _torch()
    m, k, n = mkn
    a = (rng.random(m * k) * 100).astype(np.float32)
    b = (rng.random(k * n) * 100).astype(np.float32)
    ad, bd = _dev(a), _dev(b)
    plan = plan_inner((m, k), (k, n))
    for comb in ("add", "subtract", "multiply"):
        for red in ("min", "max"):
            ops = op_pair(comb, red)
            c, r = ops.codes()
            seeds = {"identity": np.full(m * n, ops.reduce_identity, dtype=np.float32),
                     "negative": -(rng.random(m * n) * 50).astype(np.float32) - 1,
                     "mixed": ((rng.random(m * n) - 0.5) * 20000).astype(np.float32)}
            for name, seed in seeds.items():
                res = _dev(seed.copy())
                launch(plan, res, ad, bd, ops, accumulate=True)
                want = oracle.product(a, b, m, k, n, c, r,
                                      res=seed.astype(np.float64)).astype(np.float32)
                assert_bits_equal(res.cpu().numpy(), want, f"{ops} seed={name}")


@pytest.mark.parametrize("mkn", [(300, 132, 260), (257, 131, 300)])  # TMA / cp.async kernels
def test_max_times_fast_fold(mkn, rng):
    """float32 (multiply, min|max): non-negative data runs the FMUL2 +
    unsigned-order fold; zeros with infinities (0 x inf = NaN), negative
    values, -0 and NaN fall back to the exact loop.  Bitwise vs the reference."""
    m, k, n = mkn
    base_a = rng.random(m * k).astype(np.float32) * np.float32(3)
    base_b = rng.random(k * n).astype(np.float32) * np.float32(3)
    base_a[rng.random(m * k) < 0.03] = 0.0
    base_b[rng.random(k * n) < 0.03] = 1e-30  # products that underflow to +0
    for red in ("max", "min"):
        ops = op_pair("multiply", red)
        c, r = ops.codes()
        for poison in (None, "inf_and_zero", "negative", "negzero", "nan", "inf_only"):
            a, b = base_a.copy(), base_b.copy()
            if poison == "inf_and_zero":
                b[::53] = np.inf
            elif poison == "negative":
                a[::7] *= -1
            elif poison == "negzero":
                a[::41] = -0.0
            elif poison == "nan":
                b[::61] = np.nan
            elif poison == "inf_only":
                a[a == 0] = 0.5
                b[::53] = np.inf
            want = oracle.product(a, b, m, k, n, c, r).astype(np.float32)
            got = moa.inner(MoaArray((m, k), a, dtype=np.float32), MoaArray((k, n), b, dtype=np.float32),
                            ops).data
            assert_bits_equal(got, want, f"{ops} poison={poison}")


@pytest.mark.parametrize("mkn", [(20000, 48, 8), (12000, 4, 4), (9600, 132, 16), (12000, 2, 2)])
def test_tma_kernels_on_skinny_shapes(mkn, rng):
    """Boxes wider than the matrix (N below the 16/128-column TMA box, K below
    the 16/32-deep slab): the out-of-bounds fill must not leak into results.
    (x,+) float64 against the cp.async kernel on a row subset (bitwise) and the
    reference (tolerance); (add,min) float32 bitwise against the reference."""
    torch = _torch()
    m, k, n = mkn
    a = rng.random(m * k) * 2 - 1
    b = rng.random(k * n) * 2 - 1
    ad, bd = _dev(a), _dev(b)
    full = torch.empty(m * n, dtype=torch.float64, device="cuda")
    launch(plan_inner((m, k), (k, n)), full, ad, bd, moa.MUL_ADD)
    sub = torch.empty(64 * n, dtype=torch.float64, device="cuda")
    launch(plan_inner((64, k), (k, n)), sub, ad[:64 * k], bd, moa.MUL_ADD)
    full = full.cpu().numpy()
    assert_bits_equal(sub.cpu().numpy(), full[:64 * n])
    assert_within(full, oracle.product(a, b, m, k, n, MUL, ADD), sum_tolerance(k, a, b))
    if k % 4 == 0 and n % 4 == 0:  # 16-byte rows: the TMA tropical kernel
        a32 = (rng.random(m * k) * 100).astype(np.float32)
        b32 = (rng.random(k * n) * 100).astype(np.float32)
        ops = op_pair("add", "min")
        got = moa.inner(MoaArray((m, k), a32, dtype=np.float32), MoaArray((k, n), b32, dtype=np.float32),
                        ops).data
        assert_bits_equal(got, oracle.product(a32, b32, m, k, n, 0, 2).astype(np.float32))


@pytest.mark.parametrize("mkn", [(300, 132, 260), (257, 131, 300)])  # TMA / cp.async kernels
def test_tropical_accumulate_folds_previous_contents(mkn, rng):
    """MOA_FLAG_ACCUMULATE on float32 tropical pairs (what the reference-side
    binding sends, with res prefilled by the identity): the fast folds start
    from C's contents when the pre-scan of C allows, else the exact loop runs;
    every case equals the reference's fold into res."""
    torch = _torch()
    m, k, n = mkn
    a = (rng.random(m * k) * 100).astype(np.float32)
    b = (rng.random(k * n) * 100).astype(np.float32)
    plan = plan_inner((m, k), (k, n))
    for comb, red in (("add", "min"), ("add", "max"), ("subtract", "min"), ("subtract", "max")):
        ops = op_pair(comb, red)
        c, r = ops.codes()
        ident = np.float32(ops.reduce_identity)
        inits = {"identity": np.full(m * n, ident, dtype=np.float32),
                 "positive": (rng.random(m * n) * 150).astype(np.float32),
                 "signed": ((rng.random(m * n) - 0.5) * 300).astype(np.float32)}
        nan = inits["positive"].copy()
        nan[::97] = np.nan
        negz = inits["positive"].copy()
        negz[::89] = -0.0
        inits.update(nan=nan, negzero=negz)
        for name, init in inits.items():
            res = _dev(init.copy())
            launch(plan, res, _dev(a), _dev(b), ops, accumulate=True)
            want = oracle.product(a, b, m, k, n, c, r, res=init.astype(np.float64)).astype(np.float32)
            assert_bits_equal(res.cpu().numpy(), want, f"{ops} init={name}")


def test_tropical_tma_strided_rows_odd_k(rng):
    """Round-robin row sets (lda = K*step) keep the TMA-staged tropical kernel
    eligible with an odd K, so its lone-k tail runs; bitwise vs the reference."""
    torch = _torch()
    m, k, n, step = 400, 131, 260, 4
    for comb, red in (("add", "min"), ("subtract", "max")):
        ops = op_pair(comb, red)
        c, r = ops.codes()
        a = rng.random(step * m * k, dtype=np.float32) * np.float32(100)
        b = rng.random(k * n, dtype=np.float32) * np.float32(100)
        for shift in (0.0, 50.0):  # non-negative sums (VIMNMX3) and signed (FMNMX3)
            aa = a - np.float32(shift)
            res = torch.zeros(step * m * n, dtype=torch.float32, device="cuda")
            # start 0: the first row stays 16-byte aligned (TMA base requirement)
            launch(plan_inner((step * m, k), (k, n)), res, _dev(aa), _dev(b), ops, start=0,
                   step=step)
            got = res.cpu().numpy().reshape(step * m, n)
            rows = np.ascontiguousarray(aa.reshape(step * m, k)[0::step]).ravel()
            want = oracle.product(rows, b, m, k, n, c, r).astype(np.float32)
            assert_bits_equal(got[0::step].ravel(), want, f"{ops} shift={shift}")
            assert not np.delete(got, np.s_[0::step], axis=0).any()


@pytest.mark.parametrize("k,m,n", [(70, 2048, 2432), (67, 2048, 2432), (67, 2049, 2436)])
def test_tropical_quad_step_on_full_grids(k, m, n, rng):
    """Grids of >= 256 128x128 tiles run the TMA tropical kernel's 128x128
    tiles (256 threads, four-k step; tail: one k-pair and/or a lone k; ragged
    last row and column tiles); every fast fold mode — unsigned order
    (VIMNMX3), signed (FMNMX3), max-times (FMUL2) — bitwise vs the reference
    and vs the exact loop."""
    cases = (("add", "min", 0.0), ("subtract", "max", 50.0), ("multiply", "max", 0.0))
    for comb, red, shift in cases:
        ops = op_pair(comb, red)
        c, r = ops.codes()
        a = rng.random(m * k, dtype=np.float32) * np.float32(100) - np.float32(shift)
        b = rng.random(k * n, dtype=np.float32) * np.float32(100)
        if comb == "add":
            a[rng.random(m * k) < 0.05] = np.inf
        A = MoaArray((m, k), a, dtype=np.float32)
        B = MoaArray((k, n), b, dtype=np.float32)
        got = moa.inner(A, B, ops).data
        want = oracle.product(a, b, m, k, n, c, r, workers=8).astype(np.float32)
        assert_bits_equal(got, want, f"{ops} k={k}")
        assert_bits_equal(moa.inner(A, B, ops, exact=True).data, want, f"{ops} k={k} exact")


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
def test_prescan_sees_every_element(offset, rng):
    """The float32 pre-scan decides which fold is exact, so it must see every
    element: one negative value (breaks the unsigned-order fold) or one NaN in
    the last k (the reference's fold ends on it) placed first, last, or inside
    a 16-byte vector of an operand that starts `offset` floats past an aligned
    address — contiguous (one segment) and round-robin rows (strided scan)."""
    torch = _torch()
    m, k, n = 37, 67, 41
    ops = op_pair("add", "min")
    base_a = (rng.random(m * k + 8) * 100).astype(np.float32)
    base_b = (rng.random(k * n + 8) * 100).astype(np.float32)
    for where in ("a_first", "a_last", "a_mid", "b_first", "b_last", "nan_last_k"):
        aa, bb = base_a.copy(), base_b.copy()
        av, bv = aa[offset:offset + m * k], bb[offset:offset + k * n]
        if where == "a_first":
            av[0] = -1.5
        elif where == "a_last":
            av[-1] = -1.5
        elif where == "a_mid":
            av[m * k // 2 + 1] = -0.25
        elif where == "b_first":
            bv[0] = -3.0
        elif where == "b_last":
            bv[-1] = -3.0
        else:
            av[5 * k + k - 1] = np.nan
        want = oracle.product(av, bv, m, k, n, 0, 2).astype(np.float32)
        res = torch.empty(m * n, dtype=torch.float32, device="cuda")
        ad, bd = _dev(aa)[offset:offset + m * k], _dev(bb)[offset:offset + k * n]
        launch(plan_inner((m, k), (k, n)), res, ad, bd, ops)
        assert_bits_equal(res.cpu().numpy(), want, f"{where} offset={offset}")
        # rows 1, 3, 5, ... : the A scan walks strided rows
        rows = np.ascontiguousarray(av.reshape(m, k)[1::2]).ravel()
        res2 = torch.zeros(m * n, dtype=torch.float32, device="cuda")
        launch(plan_inner((m, k), (k, n)), res2, ad, bd, ops, start=1, step=2)
        got = res2.cpu().numpy().reshape(m, n)[1::2].ravel()
        want2 = oracle.product(rows, bv, rows.size // k, k, n, 0, 2).astype(np.float32)
        assert_bits_equal(got, want2, f"{where} offset={offset} strided")


def _division_operands(rng, n, dt):
    """n dividends and n divisors spanning every exponent, mantissas of all
    ones, powers of two, the reciprocal path's range edges, zeros,
    subnormals, infinities and NaN (div_by_rcp in moa_common.cuh)."""
    if dt == np.float64:
        bits = rng.integers(0, 2**63, size=n, dtype=np.uint64) | \
            (rng.integers(0, 2, size=n, dtype=np.uint64) << np.uint64(63))
        x = bits.view(np.float64).copy()
        edges = [2.0**400, 2.0**-400, np.nextafter(2.0**400, 0), np.nextafter(2.0**-400, 0),
                 2.0 - 2.0**-52, 1.0 - 2.0**-53, 1.5, 3.0, 2.0**-1074, 2.0**-1022, 1.7976931348623157e308]
    else:
        bits = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
        x = bits.view(np.float32).copy()
        edges = [2.0**40, 2.0**-40, float(np.nextafter(np.float32(2.0**40), np.float32(0))),
                 float(np.nextafter(np.float32(2.0**-40), np.float32(0))), 2.0 - 2.0**-23,
                 1.0 - 2.0**-24, 1.5, 3.0, 2.0**-149, 2.0**-126, 3.4028234663852886e38]
    k = n // 4
    x[:k] = (rng.random(k) * 2 - 1) * 10.0 ** rng.integers(-5, 6, size=k)  # everyday values
    e = np.array(edges + [-v for v in edges] + [0.0, -0.0, np.inf, -np.inf, np.nan], dtype=dt)
    x[k:k + e.size] = e
    x[k + e.size:k + e.size + 64] = 2.0 ** rng.integers(-60, 60, size=64)  # powers of two
    return rng.permutation(x)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_division_by_reciprocal_is_correctly_rounded(dt, rng):
    """Every quotient the exact loop forms with div_by_rcp equals RN(a/b): K=2
    folds whose second term cannot change the first (a zero added, an
    infinity that loses the min/max), so each result element is one quotient."""
    n = 1024
    a_col, b_row = _division_operands(rng, n, dt), _division_operands(rng, n, dt)
    for red, filler in (("add", 0.0), ("min", np.inf), ("max", -np.inf)):
        ops = op_pair("divide", red)
        c, r = ops.codes()
        a = np.empty((n, 2), dtype=dt)
        a[:, 0], a[:, 1] = a_col, filler
        b = np.empty((2, n), dtype=dt)
        b[0], b[1] = b_row, 1.0
        want = oracle.product(a.ravel(), b.ravel(), n, 2, n, c, r)
        got = moa.inner(MoaArray((n, 2), a.ravel(), dtype=dt), MoaArray((2, n), b.ravel(), dtype=dt),
                        ops).data
        assert_bits_equal(got, want.astype(dt), f"{np.dtype(dt).name} divide/{red}")
        if red == "add":  # the quotients themselves, against numpy's IEEE division
            with np.errstate(all="ignore"):
                q = (a_col[:, None].astype(np.float64) / b_row[None, :].astype(np.float64))
            ref = ((0.0 + q) + 0.0).astype(dt).ravel()
            assert_bits_equal(got, ref, f"{np.dtype(dt).name} quotients")
            # the outer product's streaming kernel (one reciprocal per column)
            out = moa.outer(MoaArray((n,), a_col, dtype=dt), MoaArray((n,), b_row, dtype=dt),
                            ops).data
            assert_bits_equal(out, (0.0 + q).astype(dt).ravel(), f"{np.dtype(dt).name} outer")


@pytest.mark.parametrize("dt", [np.int32, np.int64])
def test_integer_division_by_reciprocal_exact(dt, rng):
    """Integer quotients through the float64 reciprocal (idiv_by_rcp) equal
    truncating division for full-range operands and the edges: 0, +-1, MIN,
    MAX, powers of two, exact multiples (where the estimate falls one short)."""
    info = np.iinfo(dt)
    n = 1024

    def operands():
        x = rng.integers(info.min, info.max, size=n, endpoint=True, dtype=np.int64).astype(dt)
        k = n // 4
        x[:k] = rng.integers(-1000, 1000, size=k)
        edges = [0, 1, -1, 2, -2, 3, info.min, info.max, info.min + 1, info.max - 1,
                 info.max // 2, info.min // 2, 7, -7, 1 << 20, -(1 << 20)]
        x[k:k + len(edges)] = edges
        p2 = rng.integers(0, info.bits - 1, size=64)
        x[k + len(edges):k + len(edges) + 64] = [(1 << int(e)) * (1 if i % 2 else -1)
                                                 for i, e in enumerate(p2)]
        return rng.permutation(x)

    xs, ys = operands(), operands()
    # exact multiples: dividends q*y for random (q, y) pairs
    ys[:128] = rng.integers(-50000, 50000, size=128)
    xs[:128] = ys[:128].astype(object) * rng.integers(-40000, 40000, size=128)
    a = np.empty((n, 2), dtype=dt)
    a[:, 0], a[:, 1] = xs, 0
    b = np.empty((2, n), dtype=dt)
    b[0], b[1] = ys, 1
    got = moa.inner(MoaArray((n, 2), a.ravel(), dtype=dt), MoaArray((2, n), b.ravel(), dtype=dt),
                    op_pair("divide", "add")).data.reshape(n, n)
    xo, yo = xs.astype(object)[:, None], ys.astype(object)[None, :]
    mag = np.vectorize(lambda x, y: 0 if y == 0 else (abs(x) // abs(y)) * (1 if (x < 0) == (y < 0) else -1),
                       otypes=[object])(xo, yo)
    span = 1 << info.bits
    want = ((mag - info.min) % span + info.min).astype(dt)  # MIN / -1 wraps to MIN
    np.testing.assert_array_equal(got, want)
    out = moa.outer(MoaArray((n,), xs, dtype=dt), MoaArray((n,), ys, dtype=dt),
                    op_pair("divide", "add")).data.reshape(n, n)
    np.testing.assert_array_equal(out, want)


def test_launch_counter_advances():
    from paper_0907_0792_b200 import _native
    before = _native.launch_count()
    moa.inner(MoaArray((3, 3), range(9)), MoaArray((3, 3), range(9)))
    assert _native.launch_count() > before


def test_host_operands_through_native_executor_equal_device_launch(rng):
    """Host operands go through the native executor (moa_product_rows_host):
    the public API's result equals one device launch bit for bit, for float64
    and float32 pairs (fast folds, float64-folded float32, exact division),
    mixed-dtype operands, and through execute_parallel on one GPU.  (The
    streamed row-block schedule is covered at >= 1 GiB in
    tests/test_gpu_host_abi.py.)"""
    m, k, n = 1000, 300, 777
    a = rng.random(m * k) * 2 - 1
    b = rng.random(k * n) * 2 - 1
    for ops, dt in ((op_pair("multiply", "add"), np.float64), (op_pair("add", "min"), np.float32),
                    (op_pair("max", "multiply"), np.float64), (op_pair("divide", "max"), np.float64),
                    (op_pair("multiply", "add"), np.float32), (op_pair("subtract", "max"), np.float32)):
        A, B = MoaArray((m, k), a, dtype=dt), MoaArray((k, n), b, dtype=dt)
        want = moa.inner(A.to_device(), B.to_device(), ops).host_data()
        got = moa.inner(A, B, ops)
        assert got.shape == (m, n) and got.data.dtype == np.dtype(dt)
        assert_bits_equal(got.data, want, f"{ops} {dt.__name__}")
        assert_bits_equal(moa.execute_parallel(moa.plan_inner(A.shape, B.shape), A, B, ops,
                                               workers=1).data, want, f"{ops} parallel")
    # mixed float32 x float64 operands compute in float64
    A32 = MoaArray((m, k), a, dtype=np.float32)
    B64 = MoaArray((k, n), b)
    want = moa.inner(A32.to_device(), B64.to_device(), op_pair("add", "min")).host_data()
    assert_bits_equal(moa.inner(A32, B64, op_pair("add", "min")).data, want, "mixed dtypes")


def test_kernels_never_write_outside_their_rows(rng):
    """Canary check (compute-sanitizer is closed on this pool): every route
    writes exactly the result elements of its rows — sentinels before, after
    and between the owned rows stay untouched."""
    torch = _torch()
    sentinel = -12345.678
    # (start, step) 1, 3: odd row strides (cp.async routes); 0, 2 with even K:
    # 16-byte aligned rows, so the TMA kernels (16x32 / 64x64 DMMA, tropical) run
    cases = [((70, 33, 45), op_pair("multiply", "add"), 1, 3),
             ((70, 33, 45), op_pair("add", "min"), 1, 3),
             ((70, 1, 257), op_pair("multiply", "add"), 1, 3),
             ((70, 0, 45), op_pair("add", "max"), 1, 3),
             ((129, 20, 131), op_pair("divide", "multiply"), 1, 3),
             ((5, 40, 2048), op_pair("min", "max"), 1, 3),
             ((70, 34, 46), op_pair("multiply", "add"), 0, 2),
             ((4000, 36, 2370), op_pair("multiply", "add"), 0, 2),
             ((300, 40, 260), op_pair("add", "min"), 0, 2)]
    for (m, k, n), ops, start, step in cases:
        for dt in (torch.float64, torch.float32):
            a = _dev(rng.random(m * k) * 2 - 1, dt)
            b = _dev(rng.random(k * n) * 2 - 1, dt)
            plan = plan_inner((m, k), (k, n))
            pad = 37
            buf = torch.full((m * n + 2 * pad,), sentinel, dtype=dt, device="cuda")
            launch(plan, buf[pad:pad + m * n], a, b, ops, start=start, step=step)
            host = buf.cpu().numpy()
            want_sent = np.ones(m * n + 2 * pad, dtype=bool)
            for i in range(start, m, step):
                want_sent[pad + i * n:pad + (i + 1) * n] = False
            got_sent = host == np.array(sentinel, dtype=host.dtype)
            assert np.array_equal(got_sent[want_sent], np.ones(want_sent.sum(), bool)), \
                f"write outside owned rows {(m, k, n)} {ops} {dt}"
            owned = host[~want_sent]
            assert not np.any(owned == np.array(sentinel, dtype=host.dtype)), \
                f"owned element left unwritten {(m, k, n)} {ops} {dt}"


def test_integer_semantics_beyond_the_reference():
    """Integer-only behaviour (no float64 reference): wraparound, truncating
    division with x/0 = 0, and the type's max/min as the min/max identities."""
    i32 = np.int32
    big = MoaArray((1, 2), [2**31 - 1, 5], dtype=i32)
    one = MoaArray((2, 1), [1, 1], dtype=i32)
    assert moa.inner(big, one).data.tolist() == [np.int32(2**31 - 1 + 5 - 2**32)]
    num = MoaArray((4,), [7, -7, 5, -2**31], dtype=i32)
    den = MoaArray((4,), [2, 2, 0, -1], dtype=i32)
    q = moa.outer(num, den, op_pair("divide", "max")).data.reshape(4, 4)
    assert q[0].tolist() == [3, 3, 0, -7] and q[1].tolist() == [-3, -3, 0, 7]
    assert q[3].tolist()[3] == -2**31  # MIN / -1 wraps
    for dt, info in ((np.int32, np.iinfo(np.int32)), (np.int64, np.iinfo(np.int64))):
        e = moa.inner(MoaArray((2, 0), [], dtype=dt), MoaArray((0, 3), [], dtype=dt),
                      op_pair("add", "min"))
        assert e.data.dtype == dt and e.data.tolist() == [info.max] * 6
        e = moa.inner(MoaArray((2, 0), [], dtype=dt), MoaArray((0, 3), [], dtype=dt),
                      op_pair("add", "max"))
        assert e.data.tolist() == [info.min] * 6


def test_integer_large_random_matches_int_reference(rng):
    """Tile-crossing integer products against numpy's exact int64 matmul."""
    for dt in (np.int32, np.int64):
        m, k, n = 300, 129, 257
        a = rng.integers(-1000, 1000, size=(m, k)).astype(dt)
        b = rng.integers(-1000, 1000, size=(k, n)).astype(dt)
        got = moa.inner(MoaArray((m, k), a.ravel(), dtype=dt), MoaArray((k, n), b.ravel(), dtype=dt))
        assert got.data.dtype == dt
        np.testing.assert_array_equal(got.data.reshape(m, n), (a.astype(np.int64) @ b).astype(dt))
        mn = moa.inner(MoaArray((m, k), a.ravel(), dtype=dt), MoaArray((k, n), b.ravel(), dtype=dt),
                       op_pair("add", "min"))
        want = (a[:, :, None].astype(np.int64) + b[None, :, :]).min(axis=1).astype(dt)
        np.testing.assert_array_equal(mn.data.reshape(m, n), want)


def test_integer_tropical_wraps(rng):
    """int32/int64 (add|subtract, min|max) over full-range values: the sums
    wrap (two's complement) before the fold, as in the exact loop's wrap_add;
    int32 runs on the DPX add-then-min/max instruction (VIADDMNMX)."""
    for dt in (np.int32, np.int64):
        info = np.iinfo(dt)
        m, k, n = 70, 45, 130
        a = rng.integers(info.min, info.max, size=(m, k), endpoint=True, dtype=np.int64).astype(dt)
        b = rng.integers(info.min, info.max, size=(k, n), endpoint=True, dtype=np.int64).astype(dt)
        a[0, :4] = [info.max, info.min, 0, -1]
        b[:4, 0] = [info.max, info.min, 1, info.min]
        for comb, red in (("add", "min"), ("add", "max"), ("subtract", "min"), ("subtract", "max")):
            with np.errstate(over="ignore"):
                s3 = (a[:, :, None] + b[None, :, :]) if comb == "add" else (a[:, :, None] - b[None, :, :])
            want = s3.min(axis=1) if red == "min" else s3.max(axis=1)
            got = moa.inner(MoaArray((m, k), a.ravel(), dtype=dt), MoaArray((k, n), b.ravel(), dtype=dt),
                            op_pair(comb, red)).data.reshape(m, n)
            np.testing.assert_array_equal(got, want, err_msg=f"{np.dtype(dt).name} {comb}/{red}")


@pytest.mark.parametrize("k,lstride,m,n", [(68, 68, 300, 260), (67, 68, 300, 260),
                                           (130, 132, 300, 260), (13, 16, 2049, 2052)])
def test_int32_tropical_tma_route_wraps(k, lstride, m, n, rng):
    """int32 (add|subtract, min|max) with 16-byte aligned rows runs the TMA
    tropical kernel (one VIADDMNMX per pair, four-k step, pair and lone-k
    tails when K is odd; 64x128 tiles, and 128x128 ones from 256 of them):
    full-range values, two's-complement wrap before the fold, write-only and
    accumulate, bitwise vs numpy."""
    torch = _torch()
    info = np.iinfo(np.int32)
    a = rng.integers(info.min, info.max, size=(m, lstride), endpoint=True, dtype=np.int64).astype(np.int32)
    b = rng.integers(info.min, info.max, size=(k, n), endpoint=True, dtype=np.int64).astype(np.int32)
    a[0, :4] = [info.max, info.min, 0, -1]
    b[:4, 0] = [info.max, info.min, 1, info.min]
    plan = KernelPlan("inner", m, k, n, lstride, n, n, (m, n))
    ad, bd = _dev(a.ravel()), _dev(b.ravel())
    for comb, red in (("add", "min"), ("add", "max"), ("subtract", "min"), ("subtract", "max")):
        with np.errstate(over="ignore"):
            s3 = (a[:, :k, None] + b[None, :, :]) if comb == "add" else (a[:, :k, None] - b[None, :, :])
        want = s3.min(axis=1) if red == "min" else s3.max(axis=1)
        res = torch.empty(m * n, dtype=torch.int32, device="cuda")
        launch(plan, res, ad, bd, op_pair(comb, red))
        np.testing.assert_array_equal(res.cpu().numpy().reshape(m, n), want,
                                      err_msg=f"{comb}/{red} k={k}")
        # accumulate: fold into previous contents (the exact loop's semantics)
        init = rng.integers(info.min, info.max, size=(m, n), endpoint=True,
                            dtype=np.int64).astype(np.int32)
        res = _dev(init.ravel().copy())
        launch(plan, res, ad, bd, op_pair(comb, red), accumulate=True)
        want_acc = np.minimum(init, want) if red == "min" else np.maximum(init, want)
        np.testing.assert_array_equal(res.cpu().numpy().reshape(m, n), want_acc,
                                      err_msg=f"{comb}/{red} k={k} accumulate")


@pytest.mark.parametrize("mkn", [(700, 1000, 520),    # cp.async kernels
                                 (2000, 1000, 520),   # TMA kernel (>= 148 64x64 tiles)
                                 (2000, 33, 520)])    # chunks 16+17: a 1-wide tail joins
                                                      # its neighbour (else it would take
                                                      # the outer route's rounding)
def test_k_chunked_accumulation_replays_one_pass(mkn, rng):
    """Accumulating k-chunks (slab-aligned) with MOA_FLAG_ACCUMULATE gives the
    bits of one DMMA pass — what the pipelined broadcast of B relies on."""
    torch = _torch()
    from paper_0907_0792_b200.distributed import k_chunks
    m, k, n = mkn
    a, b = _dev(rng.random(m * k) * 2 - 1), _dev(rng.random(k * n) * 2 - 1)
    one = torch.empty(m * n, dtype=torch.float64, device="cuda")
    launch(plan_inner((m, k), (k, n)), one, a, b, moa.MUL_ADD)
    for chunks in (2, 3, 8):
        c = torch.empty(m * n, dtype=torch.float64, device="cuda")
        for i, (k0, k1) in enumerate(k_chunks(k, chunks)):
            part = moa.KernelPlan(moa.ProductMode.INNER, m, k1 - k0, n, k, n, n, (m, n))
            launch(part, c, a[k0:], b[k0 * n:], moa.MUL_ADD, accumulate=i > 0)
        assert torch.equal(c, one), chunks


def test_concurrent_invocations_are_reentrant(rng):
    """reference tests/test_parallel.py:86-96: the executor is reentrant
    across host threads sharing operands (ctypes releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    m, k, n = 300, 200, 260
    a = MoaArray((m, k), rng.random(m * k))
    b = MoaArray((k, n), rng.random(k * n))
    plan = moa.plan_inner(a.shape, b.shape)
    for ops in (moa.MUL_ADD, op_pair("add", "min")):
        want = moa.execute_sequential(plan, a, b, ops).data
        with ThreadPoolExecutor(max_workers=6) as pool:
            futs = [pool.submit(moa.execute_parallel, plan, a, b, ops, 1 + i % 4)
                    for i in range(12)]
            for f in futs:
                assert_bits_equal(f.result().data, want)


def test_workers_over_repeated_devices_bitwise(rng):
    """execute_parallel's multi-block path (several blocks on the one GPU)
    reproduces the single launch bit for bit, host and device operands."""
    m, k, n = 517, 130, 333
    a = MoaArray((m, k), rng.random(m * k))
    b = MoaArray((k, n), rng.random(k * n))
    plan = moa.plan_inner(a.shape, b.shape)
    for ops in (moa.MUL_ADD, op_pair("subtract", "max")):
        want = moa.execute_sequential(plan, a, b, ops).data
        for devs in ([0, 0], [0, 0, 0, 0, 0]):
            got = moa.execute_parallel(plan, a, b, ops, workers=len(devs), devices=devs)
            assert_bits_equal(got.data, want)
            got = moa.execute_parallel(plan, a.to_device(), b.to_device(), ops,
                                       workers=len(devs), devices=devs)
            assert got.is_device
            assert_bits_equal(got.host_data(), want)


@pytest.mark.parametrize("chunks", [2, 3, 5])
def test_execute_parallel_chunked_broadcast_schedule_bitwise(chunks, rng):
    """The k-chunked schedule execute_parallel uses with several GPUs (B's
    broadcast in k-chunks, each block's kernel accumulating chunk by chunk on
    its own stream, chunk i waiting on chunk i's arrival event) reproduces one
    launch bit for bit; on a one-GPU box the blocks share GPU 0 and the
    broadcast itself is skipped, the chunk pipeline is not."""
    m, k, n = 611, 260, 333
    for ops, dt in ((moa.MUL_ADD, np.float64), (op_pair("add", "min"), np.float32),
                    (op_pair("subtract", "max"), np.float64), (op_pair("divide", "max"), np.float64)):
        a = MoaArray((m, k), rng.random(m * k) * 10 + 1, dtype=dt)
        b = MoaArray((k, n), rng.random(k * n) * 10 + 1, dtype=dt)
        plan = moa.plan_inner(a.shape, b.shape)
        want = moa.execute_sequential(plan, a, b, ops).data
        for devs in ([0, 0], [0, 0, 0]):
            got = moa.execute_parallel(plan, a, b, ops, workers=len(devs), devices=devs,
                                       bcast_chunks=chunks)
            assert_bits_equal(got.data, want, f"{ops} {dt.__name__} {devs} chunks={chunks}")
            got = moa.execute_parallel(plan, a.to_device(), b.to_device(), ops, workers=len(devs),
                                       devices=devs, bcast_chunks=chunks)
            assert_bits_equal(got.host_data(), want, f"{ops} {dt.__name__} device")


def test_oracle_api_mirrors_reference_definitions(golden_small):
    """oracle_inner / oracle_outer (reference oracle.py:33-72) exported for API
    parity: inner = the exact fold, outer = combine with no reduce."""
    for case in golden_small[::9]:
        if case.a.dtype != np.float64:
            continue
        ops = op_pair(list(moa.COMBINE_OPS)[case.comb], list(moa.REDUCE_OPS)[case.red])
        a, b = MoaArray(case.shape_a, case.a), MoaArray(case.shape_b, case.b)
        if case.mode == "inner":
            assert_bits_equal(moa.oracle_inner(a, b, ops).data, case.out, repr(case))
        else:
            want = oracle.odometer_outer(case.a, case.shape_a, case.b, case.shape_b, case.comb)
            assert_bits_equal(moa.oracle_outer(a, b, ops).data, want, repr(case))
    neg = moa.oracle_outer(MoaArray((), [-1.0]), MoaArray((), [0.0]))
    assert np.signbit(neg.item())  # combine only: (-1)*0 = -0.0, no "+ 0.0"


def test_launch_refuses_short_or_foreign_buffers():
    torch = _torch()
    plan = plan_inner((10, 4), (4, 6))
    a = torch.zeros(40, dtype=torch.float64, device="cuda")
    b = torch.zeros(24, dtype=torch.float64, device="cuda")
    c = torch.zeros(60, dtype=torch.float64, device="cuda")
    launch(plan, c, a, b, moa.MUL_ADD)
    with pytest.raises(ValueError, match="res holds"):
        launch(plan, c[:59], a, b, moa.MUL_ADD)
    with pytest.raises(ValueError, match="a holds"):
        launch(plan, c, a[:39], b, moa.MUL_ADD)
    with pytest.raises(ValueError, match="b holds"):
        launch(plan, c, a, b[:23], moa.MUL_ADD)
    with pytest.raises(ValueError, match="contiguous CUDA"):
        launch(plan, c, a.cpu(), b, moa.MUL_ADD)
    with pytest.raises(ValueError, match="contiguous CUDA"):
        launch(plan, c.view(6, 10).t(), a, b, moa.MUL_ADD)
    launch(plan, c[:54], a, b, moa.MUL_ADD, start=0, step=4)  # rows 0, 4, 8 -> needs 8*6+6 = 54
