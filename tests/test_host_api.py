"""Host layer: shapes, psi, plans, op pairs, partitions — the reference's own
unit tests (tests/test_arrays.py, test_ops.py, test_kernel.py plan parts,
test_parallel.py partition parts) restated against this package.  CPU only."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_0907_0792_b200 as moa
from paper_0907_0792_b200 import (BoundsError, MoaArray, PlanError, RankError, ShapeError,
                                  builtin_pairs, op_pair, plan_inner, plan_outer, psi_select,
                                  reshape)
from paper_0907_0792_b200.kernel import (MAX_INDEX, ProductMode, _check_plan, resolve_backend)
from paper_0907_0792_b200.ops import COMBINE_OPS, REDUCE_OPS, OpPair


# ---- arrays (reference tests/test_arrays.py) ---------------------------------

def test_element_count():
    assert moa.element_count((2, 3)) == 6
    assert moa.element_count(()) == 1
    assert moa.element_count((4, 0, 7)) == 0


def test_row_major_offset_and_strides():
    assert moa.row_major_offset((1, 2), (2, 3)) == 5
    assert moa.row_major_offset((1, 0, 2), (2, 3, 4)) == 14
    assert moa.row_major_strides((2, 3, 4)) == (12, 4, 1)
    with pytest.raises(BoundsError):
        moa.row_major_offset((2, 0), (2, 3))
    with pytest.raises(BoundsError):
        moa.row_major_offset((0,), (2, 3))


def test_offset_is_bijection():
    shape = (2, 3, 4)
    offs = sorted(moa.row_major_offset((i, j, k), shape)
                  for i in range(2) for j in range(3) for k in range(4))
    assert offs == list(range(24))


def test_negative_extent_rejected():
    with pytest.raises(ShapeError):
        moa.as_shape((2, -1))


def test_moaarray_copy_freeze_and_count_check():
    src = np.arange(6.0)
    a = MoaArray((2, 3), src)
    src[0] = 99.0
    assert a.data[0] == 0.0
    assert a.data.dtype == np.float64
    with pytest.raises(ValueError):
        a.data[0] = 1.0
    with pytest.raises(AttributeError):
        a.shape = (3, 2)
    with pytest.raises(ShapeError):
        MoaArray((2, 2), [1.0, 2.0, 3.0])


def test_moaarray_float32_storage_only_on_request():
    x = np.arange(4, dtype=np.float32)
    assert MoaArray((4,), x).dtype == np.float64  # the reference upcasts
    assert MoaArray((4,), x, dtype=np.float32).dtype == np.float32
    assert MoaArray((4,), x, dtype=np.int32).dtype == np.int32
    with pytest.raises(TypeError):
        MoaArray((4,), x, dtype=np.int8)


def test_result_dtype_promotion():
    from paper_0907_0792_b200.kernel import result_dtype
    def arr(dt):
        return MoaArray((1,), [1], dtype=dt)
    cases = {(np.float32, np.float32): np.float32, (np.float32, np.float64): np.float64,
             (np.int32, np.int32): np.int32, (np.int32, np.int64): np.int64,
             (np.int32, np.float32): np.float64, (np.int64, np.float64): np.float64}
    for (x, y), want in cases.items():
        assert result_dtype(arr(x), arr(y)) == np.dtype(want)
        assert result_dtype(arr(y), arr(x)) == np.dtype(want)


def test_psi_select():
    c = MoaArray((2, 4), range(8))
    assert psi_select((0,), c).data.tolist() == [0, 1, 2, 3]
    assert psi_select((), c) is c
    a = MoaArray((2, 3), range(6))
    s = psi_select((1, 2), a)
    assert s.shape == () and s.item() == 5.0
    with pytest.raises(RankError):
        psi_select((0, 0, 0), a)
    with pytest.raises(BoundsError):
        psi_select((2,), a)


def test_psi_rows_rebuild_array(rng):
    a = MoaArray((3, 2, 4), rng.random(24))
    rebuilt = np.concatenate([psi_select((i,), a).data for i in range(3)])
    np.testing.assert_array_equal(rebuilt, a.data)


def test_reshape():
    a = MoaArray((6,), range(6))
    b = reshape(a, (2, 3))
    assert b.shape == (2, 3) and b.data.tolist() == a.data.tolist()
    assert reshape(b, (6,)) == a
    with pytest.raises(ShapeError):
        reshape(MoaArray((4,), range(4)), (5,))


def test_literal_roundtrip_bit_exact(tmp_path, rng):
    a = MoaArray((2, 3), np.concatenate([rng.random(4), [math.inf, -0.0]]))
    b = moa.loads(moa.dumps(a))
    assert b.shape == a.shape
    assert b.data.tobytes() == a.data.tobytes()
    p = tmp_path / "a.txt"
    moa.dump(a, p)
    assert moa.load(p) == a
    with pytest.raises(ShapeError):
        moa.loads("2 2\n1 2 3\n")


def test_equality_treats_nan_as_equal():
    assert MoaArray((2,), [math.nan, 1.0]) == MoaArray((2,), [math.nan, 1.0])


# ---- op pairs (reference tests/test_ops.py) -----------------------------------

def test_identities_and_codes():
    assert op_pair("multiply", "add").reduce_identity == 0.0
    assert op_pair("multiply", "multiply").reduce_identity == 1.0
    assert op_pair("add", "min").reduce_identity == math.inf
    assert op_pair("add", "max").reduce_identity == -math.inf
    pairs = list(builtin_pairs())
    assert len(pairs) == 24
    for p in pairs:
        assert p.codes() == (COMBINE_OPS[p.combine_name][0], REDUCE_OPS[p.reduce_name][0])
    # codes are the C ABI (include/moa_b200.h)
    assert {k: v[0] for k, v in COMBINE_OPS.items()} == {
        "add": 0, "subtract": 1, "multiply": 2, "divide": 3, "min": 4, "max": 5}
    assert {k: v[0] for k, v in REDUCE_OPS.items()} == {
        "add": 0, "multiply": 1, "min": 2, "max": 3}


def test_identity_law(rng):
    samples = list(rng.random(50) * 2e3 - 1e3) + [0.0, 1e-300, math.inf, -math.inf, math.nan]
    for p in builtin_pairs():
        for x in samples:
            got = p.reduce(p.reduce_identity, x)
            assert got == x or (math.isnan(got) and math.isnan(x))


def test_ieee_divide_and_min_max_semantics():
    div = op_pair("divide", "add").combine
    assert div(1.0, 0.0) == math.inf and div(-1.0, 0.0) == -math.inf
    assert div(1.0, -0.0) == -math.inf and math.isnan(div(0.0, 0.0))
    assert math.isnan(div(math.nan, 0.0)) and div(math.inf, 0.0) == math.inf
    mn, mx = op_pair("add", "min").reduce, op_pair("add", "max").reduce
    assert math.isnan(mn(math.inf, math.nan)) and math.isnan(mx(-math.inf, math.nan))
    # NaN is not sticky in a fold; a +-0 tie keeps the later operand
    acc = math.inf
    for v in (5.0, math.nan, 7.0):
        acc = mn(acc, v)
    assert acc == 7.0
    assert math.copysign(1.0, mn(-0.0, 0.0)) == 1.0


def test_unknown_op_names():
    with pytest.raises(ValueError):
        op_pair("pow", "add")
    with pytest.raises(ValueError):
        op_pair("add", "subtract")
    assert OpPair(lambda x, y: x, lambda x, y: y, 0.0).codes() is None


# ---- plans (reference tests/test_kernel.py:32-86) -----------------------------

def test_plan_inner_values():
    p = plan_inner((2, 3), (3, 4))
    assert p.result_shape == (2, 4)
    assert (p.noproc, p.rowsinred, p.elsinop) == (2, 3, 4)
    assert (p.lstride, p.rstride, p.restride) == (3, 4, 4)
    p = plan_inner((5,), (5,))
    assert p.result_shape == () and (p.noproc, p.rowsinred, p.elsinop) == (1, 5, 1)
    p = plan_inner((2, 3, 4), (4, 5))
    assert p.result_shape == (2, 3, 5) and (p.noproc, p.rowsinred, p.elsinop) == (6, 4, 5)
    assert p.mode is ProductMode.INNER


def test_plan_inner_errors():
    with pytest.raises(ShapeError, match=r"3.*4|4.*3"):
        plan_inner((2, 3), (4, 5))
    with pytest.raises(RankError):
        plan_inner((), (3,))
    with pytest.raises(RankError):
        plan_inner((3,), ())
    big = 2**32
    with pytest.raises(ShapeError):
        plan_inner((big, big, 2), (2, big))
    with pytest.raises(ShapeError):
        plan_inner((big, big, 0), (0, big, big))
    assert MAX_INDEX == 2**63 - 1


def test_plan_outer_values():
    assert plan_outer((2, 3), (3, 4)).result_shape == (2, 3, 3, 4)
    p = plan_outer((), (3,))
    assert p.result_shape == (3,) and (p.noproc, p.rowsinred, p.elsinop) == (1, 1, 3)
    p = plan_outer((2,), (2,))
    assert (p.noproc, p.rowsinred, p.elsinop, p.lstride) == (2, 1, 2, 1)
    assert p.mode is ProductMode.OUTER
    with pytest.raises(ShapeError):
        plan_outer((2**40,), (2**40,))


def test_baseline_config_plans():
    """The 2-D collapse of every BASELINE config."""
    from paper_0907_0792_b200.workloads import WORKLOADS
    p = plan_outer(WORKLOADS["c2"].shape_a, WORKLOADS["c2"].shape_b)
    assert (p.noproc, p.rowsinred, p.elsinop) == (65536, 1, 2048)
    assert p.result_shape == (32, 16, 16, 8, 16, 16, 8)
    p = plan_inner(WORKLOADS["c3"].shape_a, WORKLOADS["c3"].shape_b)
    assert (p.noproc, p.rowsinred, p.elsinop) == (32768, 256, 4096)
    assert p.result_shape == (32, 32, 32, 64, 64)
    for key in ("c1", "c4", "c5"):
        w = WORKLOADS[key]
        p = plan_inner(w.shape_a, w.shape_b)
        assert (p.noproc, p.rowsinred, p.elsinop) == w.mkn


def test_check_plan_detects_mismatch():
    import dataclasses
    a = MoaArray((2, 3), range(6))
    b = MoaArray((3, 4), range(12))
    _check_plan(plan_inner(a.shape, b.shape), a, b)
    with pytest.raises(PlanError):
        _check_plan(plan_inner((2, 3), (3, 4)), MoaArray((3, 3), range(9)), b)
    with pytest.raises(PlanError):
        _check_plan(dataclasses.replace(plan_inner(a.shape, b.shape), lstride=1), a, b)
    with pytest.raises(PlanError):
        _check_plan(plan_inner((2, 3), (3, 4)), MoaArray((2, 2), range(4)), b)


def test_backend_names_and_custom_callables():
    assert resolve_backend(None, moa.MUL_ADD) == "compiled"
    assert resolve_backend("auto", moa.MUL_ADD) == "compiled"
    assert resolve_backend("compiled", moa.MUL_ADD) == "compiled"
    assert resolve_backend("cuda", moa.MUL_ADD) == "compiled"
    with pytest.raises(ValueError):
        resolve_backend("rust", moa.MUL_ADD)
    with pytest.raises(ValueError):
        resolve_backend("python", moa.MUL_ADD)  # no CPU path in this build
    with pytest.raises(ValueError):
        resolve_backend(None, OpPair(lambda x, y: x * y, lambda x, y: x + y, 0.0))
    assert moa.active_backend() == "compiled"  # the reference's name (_backend.py:12)


# ---- partitions (reference tests/test_parallel.py:18-33) ----------------------

def test_partition_rows_round_robin():
    for noproc in (0, 1, 2, 7, 16):
        for workers in range(1, 9):
            owned = moa.partition_rows(noproc, workers)
            assert len(owned) == workers
            assert sorted(i for r in owned for i in r) == list(range(noproc))
    assert [list(r) for r in moa.partition_rows(7, 3)] == [[0, 3, 6], [1, 4], [2, 5]]
    with pytest.raises(ValueError):
        moa.partition_rows(4, 0)


def test_row_blocks_contiguous_cover():
    for noproc in (0, 1, 5, 16, 16384, 65537):
        for parts in range(1, 9):
            blocks = moa.row_blocks(noproc, parts)
            assert len(blocks) == parts
            flat = [i for r in blocks for i in r]
            assert flat == list(range(noproc))
    with pytest.raises(ValueError):
        moa.row_blocks(4, 0)


def test_distributed_row_block_matches_row_blocks():
    from paper_0907_0792_b200.distributed import row_block
    for noproc in (0, 3, 16384):
        for world in (1, 2, 4, 8):
            got = [range(*row_block(noproc, world, r)) for r in range(world)]
            assert got == moa.row_blocks(noproc, world)


def test_bench_job_plans_match_rank_blocks():
    """bench.py's multi-rank plans: weak scaling gives every rank exactly one
    unit of rows, strong scaling splits one unit (checked without a GPU)."""
    import bench
    from paper_0907_0792_b200.distributed import row_block
    from paper_0907_0792_b200.workloads import WORKLOADS
    for key in ("c2", "c4"):
        w = WORKLOADS[key]
        m = w.mkn[0]
        for world in (1, 2, 4, 8):
            plan = bench.job_plan(w, world)
            blocks = [row_block(plan.noproc, world, r) for r in range(world)]
            if bench.SCALING[key] == "weak":
                assert plan.noproc == m * world
                assert all(r1 - r0 == m for r0, r1 in blocks)
            else:
                assert plan.noproc == m
                assert sum(r1 - r0 for r0, r1 in blocks) == m


def test_k_chunks_align_to_the_dmma_slab():
    from paper_0907_0792_b200.distributed import k_chunks
    for K in (1, 15, 16, 17, 33, 256, 16384, 1000, 1025):
        for n in (1, 2, 3, 8):
            ch = k_chunks(K, n)
            assert ch[0][0] == 0 and ch[-1][1] == K
            assert all(a[1] == b[0] for a, b in zip(ch, ch[1:]))
            assert all(k0 % 16 == 0 for k0, _ in ch)
            assert len(ch) <= max(1, n)
            # no short tail: every chunk keeps the whole product's route
            assert len(ch) == 1 or all(k1 - k0 >= 16 for k0, k1 in ch)


def test_launch_host_validates_before_the_abi():
    """kernel.launch_host (the host-buffer C ABI from Python) refuses what the
    raw pointers cannot express — mixed dtypes, non-flat or non-contiguous
    buffers, a read-only result, buffers shorter than the rows addressed,
    custom callables — before any native call (so this runs without a GPU)."""
    import numpy as np
    import pytest

    from paper_0907_0792_b200 import OpPair, op_pair
    from paper_0907_0792_b200.kernel import launch_host, plan_inner
    plan = plan_inner((4, 3), (3, 5))
    a, b, res = np.zeros(12), np.zeros(15), np.zeros(20)
    ops = op_pair("add", "min")
    with pytest.raises(TypeError):
        launch_host(plan, res, a.astype(np.float32), b, ops)
    with pytest.raises(ValueError, match="flat"):
        launch_host(plan, res.reshape(4, 5), a, b, ops)
    with pytest.raises(ValueError, match="flat"):
        launch_host(plan, res, np.zeros(24)[::2], b, ops)
    ro = np.zeros(20)
    ro.flags.writeable = False
    with pytest.raises(ValueError, match="writeable"):
        launch_host(plan, ro, a, b, ops)
    with pytest.raises(ValueError, match="holds"):
        launch_host(plan, np.zeros(19), a, b, ops)
    with pytest.raises(ValueError, match="holds"):
        launch_host(plan, res, np.zeros(11), b, ops)
    custom = OpPair(lambda x, y: x, lambda x, y: y, 0.0)
    with pytest.raises(ValueError, match="custom"):
        launch_host(plan, res, a, b, custom)
