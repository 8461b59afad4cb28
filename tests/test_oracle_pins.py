"""Pin the oracle before trusting it: the C port (oracle/moa_oracle.c) and the
reference's own compiled loop (oracle/_ref) must reproduce the reference's
golden outputs bit for bit (tests/golden/, written by the reference itself via
tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

import oracle
from conftest import GOLDEN

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def _mkn(case):
    if case.mode == "outer":
        return int(np.prod(case.shape_a, dtype=np.int64)), 1, int(np.prod(case.shape_b, dtype=np.int64))
    return (int(np.prod(case.shape_a[:-1], dtype=np.int64)), case.shape_a[-1],
            int(np.prod(case.shape_b[1:], dtype=np.int64)))


def test_golden_has_every_pair(golden_small):
    seen = {(c.comb, c.red) for c in golden_small}
    assert seen == {(c, r) for c in range(6) for r in range(4)}
    tags = {c.tag for c in golden_small}
    for t in ("fig1", "dot", "tropical_dot", "empty_min", "zero_rows", "special_inner",
              "f32_tropical_specials", "negzero_add"):
        assert t in tags


def test_port_bitwise_equals_reference_goldens(golden_small):
    for case in golden_small:
        m, k, n = _mkn(case)
        got = oracle.product(case.a, case.b, m, k, n, case.comb, case.red)
        np.testing.assert_array_equal(got, case.out, err_msg=repr(case))
        assert got.tobytes() == case.out.tobytes() or np.isnan(case.out).any(), repr(case)


def test_port_parallel_bitwise_any_worker_count(golden_small):
    for case in golden_small[::7]:
        m, k, n = _mkn(case)
        for w in (2, 3, 8):
            got = oracle.product(case.a, case.b, m, k, n, case.comb, case.red, workers=w)
            np.testing.assert_array_equal(got, case.out, err_msg=repr(case))


def test_reference_kernel_build_matches_goldens(golden_small):
    if oracle.ref_kernel() is None:
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    for case in golden_small[::3]:
        m, k, n = _mkn(case)
        got = oracle.reference_product(case.a, case.b, m, k, n, case.comb, case.red, workers=2)
        np.testing.assert_array_equal(got, case.out, err_msg=repr(case))


def test_odometer_oracle_matches_goldens(golden_small):
    """The naive odometer restatement (oracle.py:33-72) agrees with the kernel's
    outputs: bitwise for inner products (same fold order), and for outer
    products up to the reduce against the identity the kernel applies."""
    for case in golden_small:
        if max(_mkn(case)) > 64:
            continue
        if case.mode == "inner":
            got = oracle.odometer_inner(case.a, case.shape_a, case.b, case.shape_b,
                                        case.comb, case.red)
            np.testing.assert_array_equal(got, case.out, err_msg=repr(case))
        else:
            got = oracle.odometer_outer(case.a, case.shape_a, case.b, case.shape_b, case.comb)
            np.testing.assert_array_equal(got, case.out, err_msg=repr(case))


def test_hand_values_in_goldens(golden_small):
    by_tag = {c.tag: c for c in golden_small}
    assert by_tag["fig1"].out.tolist() == [32, 38, 44, 50, 68, 83, 98, 113]
    assert by_tag["dot"].out.tolist() == [32.0]
    assert by_tag["tropical_dot"].out.tolist() == [11.0]
    assert by_tag["outer_hand"].out.tolist() == [10, 20, 20, 40]
    assert by_tag["singleton"].out.tolist() == [15.0]
    assert by_tag["scalar_scalar"].out.tolist() == [12.0]
    assert by_tag["empty_min"].out.tolist() == [np.inf] * 6
    assert by_tag["empty_max"].out.tolist() == [-np.inf] * 6
    # outer(-1, 0): (x, +) gives +0.0, (x, min) keeps -0.0
    assert np.signbit(by_tag["negzero_add"].out[0]) == False  # noqa: E712
    assert np.signbit(by_tag["negzero_min"].out[0]) == True  # noqa: E712
    assert by_tag["zero_rows"].out.size == 0


@pytest.mark.parametrize("key", ["c1", "c2", "c3", "c4", "c5"])
def test_port_matches_reference_at_full_size(key):
    """Row subsets of every BASELINE config at full K and N: the C port's bytes
    hash to the reference's (configs.json)."""
    from paper_0907_0792_b200.workloads import WORKLOADS
    pins = json.loads((GOLDEN / "configs.json").read_text())[key]
    w = WORKLOADS[key]
    a, b = w.generate()
    m, k, n = w.mkn
    rows = pins["rows"]
    a_rows = np.concatenate([a[i * k:(i + 1) * k] for i in rows])
    comb, red = w.ops.codes()
    got = oracle.product(a_rows, b, len(rows), k, n, comb, red, workers=oracle.host_cores())
    assert hashlib.sha256(got.tobytes()).hexdigest() == pins["sha256_f64"]
    if "sha256_f32" in pins:
        assert hashlib.sha256(got.astype(np.float32).tobytes()).hexdigest() == pins["sha256_f32"]
