"""The reference-side backend module (integration/moaprod_b200kernel.py) driven
the way the reference drives its compiled loop: ``_Runner`` prefills res with
the reduce identity (kernel.py:149) and ``execute_parallel`` calls
``product_rows(res, a, b, ..., start=w, step=W)`` from W threads at once on
one shared res (parallel.py:26-43).  Results must equal the reference's loop
(oracle C port) bit for bit — (multiply, add) included, since the module
sends MOA_FLAG_EXACT by default; with $MOA_B200_TENSOR_CORES=1 (multiply, add)
runs on the FP64 tensor cores and is checked against K*2^-52*max|A|*max|B|."""

from __future__ import annotations

import importlib.util
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_0907_0792_b200 as moa
from parity import assert_bits_equal, assert_within, sum_tolerance

ROOT = Path(__file__).resolve().parents[1]


def _module():
    spec = importlib.util.spec_from_file_location("moaprod_b200kernel",
                                                  ROOT / "integration" / "moaprod_b200kernel.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_backend_module_binds_the_abi():
    """CPU-side: the module loads the library (no torch) and binds the
    host-buffer entry point with the reference's 13 arguments plus dtype,
    flags and device (and the device-pointer one with a stream)."""
    mod = _module()
    assert len(mod._lib.moa_product_rows_host.argtypes) == 16
    assert len(mod._lib.moa_product_rows.argtypes) == 16
    assert mod.MOA_FLAG_ACCUMULATE == 1
    assert callable(mod.product_rows)
    src = (ROOT / "integration" / "moaprod_b200kernel.py").read_text()
    assert "import torch" not in src


@pytest.mark.gpu
@pytest.mark.parametrize("workers", [1, 3, 8])
@pytest.mark.parametrize("tensor_cores", [False, True])
def test_reference_style_runner_with_concurrent_threads(workers, tensor_cores, rng,
                                                         monkeypatch):
    if tensor_cores:
        monkeypatch.setenv("MOA_B200_TENSOR_CORES", "1")
    mod = _module()
    m, k, n = 150, 37, 90
    a = rng.random(m * k) * 3 - 1
    b = rng.random(k * n) * 3 - 1
    for ops in (moa.op_pair("multiply", "add"), moa.op_pair("add", "min"),
                moa.op_pair("divide", "max"), moa.op_pair("max", "multiply")):
        c, r = ops.codes()
        res = np.full(m * n, ops.reduce_identity)  # _Runner's identity prefill
        with ThreadPoolExecutor(workers) as pool:
            futs = [pool.submit(mod.product_rows, res, a, b, m, k, n, k, n, n, c, r, w, workers)
                    for w in range(workers)]
            for f in futs:
                f.result()
        want = oracle.product(a, b, m, k, n, c, r)
        if (c, r) == (2, 0) and tensor_cores:
            assert_within(res, want, sum_tolerance(k, a, b), f"{ops} W={workers}")
        else:
            assert_bits_equal(res, want, f"{ops} W={workers}")


@pytest.mark.gpu
@pytest.mark.parametrize("workers", [1, 4])
def test_overwrite_variant_needs_no_prefill(workers, rng):
    """product_rows_overwrite on an UNinitialised res (a _Runner branch that
    skips the identity prefill) gives the bits of prefill + product_rows."""
    mod = _module()
    m, k, n = 130, 29, 77
    a = rng.random(m * k) * 3 - 1
    b = rng.random(k * n) * 3 - 1
    for ops in (moa.MUL_ADD, moa.op_pair("add", "max"), moa.op_pair("multiply", "multiply")):
        c, r = ops.codes()
        res = np.empty(m * n)
        res.fill(np.nan)  # garbage the overwrite must not read
        with ThreadPoolExecutor(workers) as pool:
            for f in [pool.submit(mod.product_rows_overwrite, res, a, b, m, k, n, k, n, n, c, r,
                                  w, workers) for w in range(workers)]:
                f.result()
        assert_bits_equal(res, oracle.product(a, b, m, k, n, c, r), f"{ops} W={workers}")


@pytest.mark.gpu
def test_reference_style_outer_and_empty_rows(rng):
    mod = _module()
    x, y = rng.random(40) * 2 - 1, rng.random(70) * 2 - 1
    res = np.full(40 * 70, 0.0)
    for w in range(3):
        mod.product_rows(res, x, y, 40, 1, 70, 1, 70, 70, 2, 0, w, 3)
    assert_bits_equal(res, (np.multiply.outer(x, y) + 0.0).ravel())
    before = res.copy()
    mod.product_rows(res, x, y, 40, 1, 70, 1, 70, 70, 2, 0, 45, 3)  # surplus worker: no rows
    assert_bits_equal(res, before)


@pytest.mark.gpu
def test_workers_spread_over_listed_devices(monkeypatch, rng):
    """$MOA_B200_DEVICES lists the GPUs; worker k of the reference's
    execute_parallel (rows k::W) runs on DEVICES[k mod len].  On a one-GPU box
    the list repeats device 0, which exercises the mapping."""
    monkeypatch.setenv("MOA_B200_DEVICES", "0,0,0")
    mod = _module()
    assert mod.DEVICES == [0, 0, 0]
    m, k, n = 97, 40, 61
    a, b = rng.random(m * k), rng.random(k * n)
    ops = moa.op_pair("subtract", "min")
    c, r = ops.codes()
    res = np.full(m * n, ops.reduce_identity)
    workers = 5
    with ThreadPoolExecutor(workers) as pool:
        for f in [pool.submit(mod.product_rows, res, a, b, m, k, n, k, n, n, c, r, w, workers)
                  for w in range(workers)]:
            f.result()
    assert_bits_equal(res, oracle.product(a, b, m, k, n, c, r))
