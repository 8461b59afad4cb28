"""Seeded random sweep of the device entry point (moa_product_rows, the drop-in
for _ckernel.product_rows, _ckernel.pyx:75-88) against the C oracle
(oracle/moa_oracle.c, pinned to the reference's goldens): random extents
(including K = 0 and 1; one case in ten large enough for the
large-grid kernels), all 24 (combine, reduce) pairs, four dtypes,
write-only and accumulate (the reference's fold from res, _ckernel.pyx:51,70),
exact and default routes, round-robin row sets start::step
(parallel.py:37-43), padded row strides and misaligned base pointers (TMA-
ineligible), float data with and without IEEE specials.  Bit-exact everywhere
except the float64 (multiply, add) DMMA route (K >= 8, not exact), which is
held to BASELINE's K * 2^-52 * max|A| * max|B| with identical non-finite
positions.  Integer cases keep values small and reduce with add/min/max (no
divide combine), where the reference's float64 arithmetic is exact."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_0907_0792_b200 as moa
from paper_0907_0792_b200 import op_pair
from paper_0907_0792_b200.kernel import KernelPlan, launch
from parity import assert_bits_equal, assert_within, sum_tolerance

pytestmark = pytest.mark.gpu

MUL_ADD = (2, 0)
_SPECIALS = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -2.5e-310])


def _float_operand(rng, n, dt, specials):
    x = (rng.random(n) * 8 - 3) * 2.0 ** rng.integers(-4, 5, n)
    if specials and n:
        idx = rng.random(n) < 0.06
        sp = _SPECIALS if dt == np.float64 else np.array([0.0, -0.0, np.inf, -np.inf, np.nan,
                                                          1e-45, -3e-39])
        x[idx] = rng.choice(sp, size=int(idx.sum()))
    return x.astype(dt)


def _case(rng):
    dt = rng.choice([np.float64, np.float32, np.int32, np.int64], p=[0.4, 0.3, 0.15, 0.15])
    is_int = np.dtype(dt).kind == "i"
    combs = [c for c in moa.COMBINE_OPS if not (is_int and c == "divide")]
    reds = [r for r in moa.REDUCE_OPS if not (is_int and r == "multiply")]
    ops = op_pair(str(rng.choice(combs)), str(rng.choice(reds)))
    big = rng.random() < 0.1  # >= one wave of 64x64 / 128x128 tiles: the large-grid kernels
    m = int(rng.integers(600, 1300) if big else rng.integers(1, 200))
    k = int(rng.choice([0, 1, 2, 3, 7, 8, 9, 16, 17, 31, 33, 64, 67]))
    if is_int and k == 0:
        k = 1
    n = int(rng.integers(600, 1300) if big else rng.integers(1, 200))
    step = int(rng.choice([1, 1, 2, 3, 4]))
    start = int(rng.integers(0, step + 1))
    pad = lambda: int(rng.choice([0, 0, 1, 4, 7]))  # noqa: E731
    return dt, ops, m, k, n, step, start, k + pad(), n + pad(), n + pad(), \
        bool(rng.random() < 0.5), bool(rng.random() < 0.3), int(rng.choice([0, 0, 1])), \
        bool(rng.random() < 0.3)


@pytest.mark.parametrize("seed", range(12))
def test_random_sweep_against_oracle(seed):
    import torch
    rng = np.random.default_rng(1000 + seed)
    for trial in range(50):
        (dt, ops, m, k, n, step, start, lstride, rstride, restride, acc, exact, shift,
         specials) = _case(rng)
        is_int = np.dtype(dt).kind == "i"
        c, r = ops.codes()
        if is_int:
            a = rng.integers(-9, 10, max((m - 1) * lstride + k, 0)).astype(dt)
            b = rng.integers(-9, 10, max((k - 1) * rstride + n, 0)).astype(dt)
            seed_c = rng.integers(-50, 50, m * restride).astype(dt)
        else:
            a = _float_operand(rng, max((m - 1) * lstride + k, 0), dt, specials)
            b = _float_operand(rng, max((k - 1) * rstride + n, 0), dt, specials)
            seed_c = _float_operand(rng, m * restride, dt, False)
        plan = KernelPlan("inner", m, k, n, lstride, rstride, restride, (m, n))
        # device buffers, optionally shifted by one element (TMA-ineligible bases)
        tdt = torch.from_numpy(np.zeros(1, dtype=dt)).dtype

        def dev(x):
            t = torch.zeros(x.size + shift + 1, dtype=tdt, device="cuda")
            t[shift:shift + x.size] = torch.from_numpy(x).cuda()
            return t[shift:shift + max(x.size, 1)]

        ad, bd, cd = dev(a), dev(b), dev(seed_c)
        launch(plan, cd, ad, bd, ops, start=start, step=step, exact=exact, accumulate=acc)
        got = cd[:m * restride].cpu().numpy().reshape(m, restride)
        # oracle: every row of the (padded) A through the C port, res = the seed
        # rows (accumulate) or the identity
        seed_rows = seed_c.reshape(m, restride)[:, :n]
        res0 = (np.ascontiguousarray(seed_rows).astype(np.float64).ravel() if acc else None)
        want_all = oracle.product(a.astype(np.float64) if is_int else a,
                                  b.astype(np.float64) if is_int else b, m, k, n, c, r,
                                  lda=lstride, ldb=rstride, res=res0).reshape(m, n)
        rows = np.arange(start, m, step)
        others = np.setdiff1d(np.arange(m), rows)
        msg = (f"seed {seed} trial {trial}: {np.dtype(dt).name} {ops} m={m} k={k} n={n} "
               f"{start}::{step} strides={lstride},{rstride},{restride} acc={acc} "
               f"exact={exact} shift={shift} specials={specials}")
        # rows outside the set and the row padding are untouched
        assert_bits_equal(got[others].ravel(), seed_c.reshape(m, restride)[others].ravel(),
                          msg + " (rows outside the set)")
        assert_bits_equal(got[:, n:].ravel(), seed_c.reshape(m, restride)[:, n:].ravel(),
                          msg + " (row padding)")
        g = got[rows, :n].ravel()
        w = want_all[rows].ravel()
        if is_int:
            np.testing.assert_array_equal(g, w.astype(dt), err_msg=msg)
        elif (c, r) == MUL_ADD and dt == np.float64 and k >= 8 and not exact:
            av = a.reshape(-1)
            bv = b.reshape(-1)
            tol = sum_tolerance(k, av[np.isfinite(av)], bv[np.isfinite(bv)])
            if acc:
                tol += 2.0 ** -52 * float(np.max(np.abs(seed_rows[np.isfinite(seed_rows)]),
                                                 initial=0.0)) * 2
            assert_within(g, w, tol, msg)
        else:
            with np.errstate(over="ignore"):  # float32 results beyond range round to inf
                w = w.astype(dt)
            assert_bits_equal(g, w, msg)


@pytest.mark.parametrize("seed", range(6))
def test_random_host_entry_equals_device_entry(seed, monkeypatch):
    """moa_product_rows_host (csrc/host_exec.cu) on random cases: page-locked
    or pageable A, B and res in any mix, row sets, padded strides, accumulate,
    and a block cap ($MOA_HOST_BLOCK_BYTES) that is sometimes small enough to
    force the streamed multi-block schedule (k-chunked first block) — always
    the bits of the device entry point on the same data."""
    import torch
    from paper_0907_0792_b200.kernel import launch_host
    rng = np.random.default_rng(2000 + seed)
    for trial in range(25):
        (dt, ops, m, k, n, step, start, lstride, rstride, restride, acc, exact, _shift,
         specials) = _case(rng)
        cap = int(rng.choice([0, 0, 64 << 10, 256 << 10, 1 << 20]))
        if cap:
            monkeypatch.setenv("MOA_HOST_BLOCK_BYTES", str(cap))
        else:
            monkeypatch.delenv("MOA_HOST_BLOCK_BYTES", raising=False)
        is_int = np.dtype(dt).kind == "i"
        if is_int:
            a = rng.integers(-9, 10, max((m - 1) * lstride + k, 1)).astype(dt)
            b = rng.integers(-9, 10, max((k - 1) * rstride + n, 1)).astype(dt)
            seed_c = rng.integers(-50, 50, m * restride).astype(dt)
        else:
            a = _float_operand(rng, max((m - 1) * lstride + k, 1), dt, specials)
            b = _float_operand(rng, max((k - 1) * rstride + n, 1), dt, specials)
            seed_c = _float_operand(rng, m * restride, dt, False)
        plan = KernelPlan("inner", m, k, n, lstride, rstride, restride, (m, n))
        tdt = torch.from_numpy(np.zeros(1, dtype=dt)).dtype
        cd = torch.from_numpy(seed_c.copy()).cuda()
        launch(plan, cd, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), ops,
               start=start, step=step, exact=exact, accumulate=acc)
        want = cd.cpu().numpy()

        def host(x, pin):
            if not pin:
                return x.copy()
            t = torch.empty(x.size, dtype=tdt, pin_memory=True).numpy()
            t[:] = x
            return t

        pins = rng.random(3) < 0.5
        got = host(seed_c, pins[2])
        launch_host(plan, got, host(a, pins[0]), host(b, pins[1]), ops, start=start, step=step,
                    exact=exact, accumulate=acc)
        assert_bits_equal(got, want,
                          f"seed {seed} trial {trial}: {np.dtype(dt).name} {ops} m={m} k={k} "
                          f"n={n} {start}::{step} strides={lstride},{rstride},{restride} "
                          f"acc={acc} exact={exact} pinned={list(pins)} cap={cap}")
