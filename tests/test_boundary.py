"""The C-ABI boundary and the no-fallback rules.  CPU only (no kernel launches:
every call here returns before touching a device)."""

from __future__ import annotations

import ast
import ctypes
import re
from pathlib import Path

import pytest

import paper_0907_0792_b200 as moa
from paper_0907_0792_b200 import _native
from paper_0907_0792_b200.errors import BackendError

REPO = Path(__file__).resolve().parents[1]
HEADER = REPO / "include" / "moa_b200.h"
PKG = REPO / "paper_0907_0792_b200"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return re.findall(r"\b(moa_[a-z_]+)\s*\(", text)


def test_library_loads_and_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    decl = declared_functions()
    assert set(decl) == set(_native.EXPORTS)
    for name in decl:
        assert hasattr(lib, name), name
    assert _native.abi_version() == 101  # 1.01: moa_product_rows_host, moa_device_count


def test_header_constants_match_python_codes():
    text = HEADER.read_text()
    consts = dict(re.findall(r"#define (MOA_[A-Z0-9_]+) \(?(-?\d+)u?\)?", text))
    for name, (code, _) in moa.COMBINE_OPS.items():
        assert int(consts[f"MOA_COMBINE_{name.upper()}"]) == code
    for name, (code, _, _) in moa.REDUCE_OPS.items():
        assert int(consts[f"MOA_REDUCE_{name.upper()}"]) == code
    assert int(consts["MOA_DTYPE_F64"]) == _native.DTYPE_F64
    assert int(consts["MOA_DTYPE_F32"]) == _native.DTYPE_F32
    assert int(consts["MOA_DTYPE_I32"]) == _native.DTYPE_I32
    assert int(consts["MOA_DTYPE_I64"]) == _native.DTYPE_I64
    assert int(consts["MOA_FLAG_ACCUMULATE"]) == _native.FLAG_ACCUMULATE
    assert int(consts["MOA_FLAG_EXACT"]) == _native.FLAG_EXACT


def test_kernel_routing():
    pk = _native.plan_kernel
    assert pk(0, 16384, 16384, 16384, 2, 0) == "dmma"
    assert pk(0, 16384, 8, 16384, 2, 0) == "dmma"
    assert pk(0, 16384, 7, 16384, 2, 0) == "semiring_exact"  # write-bound: exact fold
    assert pk(0, 4, 2, 4, 2, 0) == "semiring_exact"
    assert pk(0, 16384, 16384, 16384, 2, 0, _native.FLAG_EXACT) == "semiring_exact"
    assert pk(1, 16384, 16384, 16384, 0, 2) == "semiring_fast"
    # accumulate folds C's contents too (pre-scanned with A and B)
    assert pk(1, 16384, 16384, 16384, 0, 2, _native.FLAG_ACCUMULATE) == "semiring_fast"
    assert pk(0, 16384, 16384, 16384, 0, 2) == "semiring_exact"  # no f64 fast loop
    assert pk(1, 16384, 16384, 16384, 2, 0) == "semiring_exact"  # f32 sums run in f64
    assert pk(1, 16384, 16384, 16384, 2, 3) == "semiring_fast"  # max-times (scanned)
    assert pk(2, 16384, 16384, 16384, 2, 0) == "semiring_exact"  # int32: exact integer fold
    assert pk(2, 16384, 16384, 16384, 1, 3) == "semiring_dpx"  # int32 tropical: DPX on TMA tiles
    assert pk(3, 16384, 16384, 16384, 0, 2) == "semiring_exact"  # int64 tropical
    assert pk(2, 65536, 1, 2048, 2, 0) == "outer"
    assert pk(0, 65536, 1, 2048, 2, 0) == "outer"
    assert pk(0, 2, 0, 3, 2, 2) == "fill"
    assert pk(0, 2, 0, 3, 2, 2, _native.FLAG_ACCUMULATE) == "none"
    assert pk(0, 0, 5, 3, 2, 0) == "none"
    assert pk(0, 5, 5, 0, 2, 0) == "none"


def _call(**kw):
    args = dict(dtype=0, res_ptr=0, a_ptr=0, b_ptr=0, noproc=4, rowsinred=3, elsinop=5,
                lstride=3, rstride=5, restride=5, combine_code=2, reduce_code=0, start=0,
                step=1, flags=0, stream=0)
    args.update(kw)
    _native.product_rows(**args)


@pytest.mark.parametrize("kw, msg", [
    (dict(dtype=7), "dtype"),
    (dict(dtype=-1), "dtype"),
    (dict(combine_code=6), "combine"),
    (dict(reduce_code=-1), "reduce"),
    (dict(step=0), "step"),
    (dict(start=-1), "start"),
    (dict(noproc=-2), "negative"),
    (dict(lstride=-1), "negative"),
    (dict(), "null"),
])
def test_argument_errors_raise(kw, msg):
    with pytest.raises(BackendError, match=msg):
        _call(**kw)


def test_empty_work_is_a_noop():
    _call(noproc=0)
    _call(elsinop=0)
    _call(start=4)  # surplus worker owns no rows (parallel.py:31-33)
    _call(rowsinred=0, flags=_native.FLAG_ACCUMULATE)  # empty fold into existing res


def test_product_package_never_imports_the_oracle():
    for path in PKG.rglob("*.py"):
        tree = ast.parse(path.read_text())
        for node in ast.walk(tree):
            names = []
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            assert not any(n.split(".")[0] == "oracle" for n in names), path
        assert "/root/reference" not in path.read_text(), path


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", tmp_path / "missing.so")
    with pytest.raises(BackendError, match="not built"):
        _native.load()
    a = moa.MoaArray((2,), [1.0, 2.0])
    with pytest.raises(BackendError):
        moa.inner(a, a)


def test_custom_callables_rejected_before_any_device_work():
    ops = moa.OpPair(lambda x, y: x * y + 1.0, lambda x, y: x + y, 0.0)
    a = moa.MoaArray((2,), [1.0, 2.0])
    with pytest.raises(ValueError, match="custom"):
        moa.inner(a, a, ops)


def test_plan_errors_raised_before_backend():
    a = moa.MoaArray((2, 3), range(6))
    with pytest.raises(moa.ShapeError):
        moa.inner(a, moa.MoaArray((4, 2), range(8)))
    with pytest.raises(moa.PlanError):
        moa.execute_sequential(moa.plan_inner((2, 3), (3, 4)), a, moa.MoaArray((3, 5), range(15)))
    with pytest.raises(ValueError):
        moa.execute_parallel(moa.plan_inner((2, 3), (3, 2)), a, moa.MoaArray((3, 2), range(6)),
                             workers=0)
