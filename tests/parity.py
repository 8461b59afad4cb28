"""Comparison helpers for the parity tests."""

from __future__ import annotations

import numpy as np


def assert_bits_equal(got: np.ndarray, want: np.ndarray, msg: str = "") -> None:
    """Bit-exact equality, NaN payloads excepted (NVIDIA GPUs return the
    canonical NaN; x86 propagates the operand's payload).  Unlike
    numpy.testing.assert_array_equal this distinguishes -0.0 from +0.0."""
    got = np.asarray(got)
    want = np.asarray(want).astype(got.dtype, copy=False)
    assert got.shape == want.shape, f"{msg}: shape {got.shape} != {want.shape}"
    gn, wn = np.isnan(got), np.isnan(want)
    if not np.array_equal(gn, wn):
        i = int(np.flatnonzero(gn != wn)[0])
        raise AssertionError(f"{msg}: NaN mismatch at {i}: got {got[i]!r} want {want[i]!r}")
    ut = np.uint64 if got.dtype == np.float64 else np.uint32
    g, w = got[~gn].view(ut), want[~wn].view(ut)
    if not np.array_equal(g, w):
        bad = np.flatnonzero(g != w)
        i = int(bad[0])
        raise AssertionError(f"{msg}: {bad.size} elements differ; first: got "
                             f"{got[~gn][i]!r} want {want[~wn][i]!r}")


def sum_tolerance(K: int, a: np.ndarray, b: np.ndarray, eps: float = 2.0**-52) -> float:
    """BASELINE's bound for floating-point sums: K * 2^-52 * max|A| * max|B|."""
    ma = float(np.max(np.abs(a))) if a.size else 0.0
    mb = float(np.max(np.abs(b))) if b.size else 0.0
    return max(K, 1) * eps * ma * mb


def assert_within(got: np.ndarray, want: np.ndarray, tol: float, msg: str = "") -> None:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, msg
    fin = np.isfinite(want)
    assert np.array_equal(np.isfinite(got), fin), f"{msg}: finiteness differs"
    nonfin = ~fin
    assert_bits_equal(got[nonfin], want[nonfin], msg + " (non-finite)")
    if fin.any():
        err = float(np.max(np.abs(got[fin] - want[fin])))
        assert err <= tol, f"{msg}: max |err| {err:.3e} > tolerance {tol:.3e}"
