"""The cuBLAS GEMM comparator (reference tests/test_gemm.py restated)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_0907_0792_b200 as moa
from paper_0907_0792_b200 import GemmParams, MoaArray, ShapeError, gemm_baseline
from paper_0907_0792_b200.gemm import from_colmajor, run_colmajor, to_colmajor


def _mats(rng, m, n, k):
    return (MoaArray((m, k), rng.random(m * k)), MoaArray((k, n), rng.random(k * n)),
            MoaArray((m, n), rng.random(m * n)))


def test_colmajor_round_trip_and_shape_check(rng):
    a = MoaArray((3, 5), rng.random(15))
    flat = to_colmajor(a, 3, 5)
    assert flat[1] == a.data[5]
    assert from_colmajor(flat, 3, 5) == a
    with pytest.raises(ShapeError):
        to_colmajor(a, 5, 3)


def test_params_validation():
    with pytest.raises(ShapeError):
        GemmParams(1.0, 0.0, 0, 3, 4)
    GemmParams(1.0, 0.0, 1, 1, 1)


@pytest.mark.gpu
def test_gemm_baseline_semantics(rng):
    a, b, c = _mats(rng, 3, 4, 2)
    zeros = MoaArray((3, 4), [0.0] * 12)
    got = gemm_baseline(GemmParams(1.0, 0.0, 3, 4, 2), a, b, zeros)
    want = oracle.product(a.data, b.data, 3, 2, 4, 2, 0)
    np.testing.assert_allclose(got.data, want, rtol=1e-12)
    a, b, c = _mats(rng, 4, 3, 5)
    np.testing.assert_array_equal(gemm_baseline(GemmParams(0.0, 1.0, 4, 3, 5), a, b, c).data, c.data)
    got = gemm_baseline(GemmParams(0.0, 2.0, 1, 1, 1), MoaArray((1, 1), [9.0]),
                        MoaArray((1, 1), [0.0]), MoaArray((1, 1), [1.0]))
    assert got.data.tolist() == [2.0]
    a, b, c = _mats(rng, 2, 2, 2)
    before = c.data.copy()
    gemm_baseline(GemmParams(1.0, 0.5, 2, 2, 2), a, b, c)
    np.testing.assert_array_equal(c.data, before)
    with pytest.raises(ShapeError):
        gemm_baseline(GemmParams(1.0, 0.0, 2, 3, 5), *_mats(rng, 2, 3, 4))


@pytest.mark.gpu
def test_gemm_matches_inner_and_colmajor_path(rng):
    for _ in range(5):
        m, n, k = (int(v) for v in rng.integers(1, 65, size=3))
        a, b, c = _mats(rng, m, n, k)
        params = GemmParams(1.5, 0.25, m, n, k)
        got = gemm_baseline(params, a, b, c)
        want = 1.5 * moa.inner(a, b, exact=True).data + 0.25 * c.data
        np.testing.assert_allclose(got.data, want, rtol=1e-12)
        c_cm = to_colmajor(c, m, n)
        run_colmajor(params, to_colmajor(a, m, k), to_colmajor(b, k, n), c_cm)
        np.testing.assert_array_equal(from_colmajor(c_cm, m, n).data, got.data)
        for w in (2, 5):
            np.testing.assert_array_equal(gemm_baseline(params, a, b, c, workers=w).data, got.data)
