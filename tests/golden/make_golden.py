"""Generate the golden fixtures from the REFERENCE itself (run in the build container).

    python tests/golden/make_golden.py

Builds the reference package from /root/reference/pkg in a scratch copy under
/tmp (its own setup.py, compiled backend, flags -O3 -ffp-contract=off), imports
it as ``moaprod`` and records its outputs:

* small.npz  — ~700 small cases over all 24 (combine, reduce) pairs: random
  inner/outer products (rank <= 4, extents <= 5, values U[-1,2) like the
  reference's conftest.py:7-27), special-value cases (NaN, +-inf, +-0), medium
  products with ragged tile edges, float32 inputs (the reference upcasts,
  arrays.py:77-78), integer-valued int32/int64 inputs, the reference tests'
  hand-checked answers, and empty / zero-extent cases.  Every output comes from moaprod.inner / moaprod.outer.
* configs.json — for each BASELINE config, the reference output on a row
  subset at FULL size (full K and N), as sha256 of the float64 bytes (and of
  the float32 rounding for the float32 config) plus a few sample values.

The reference cannot travel to the GPU box; these files do.
"""

from __future__ import annotations

import hashlib
import json
import math
import shutil
import subprocess
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
SCRATCH = Path("/tmp/moaprod_ref_golden")


def load_reference():
    if not (SCRATCH / "src" / "moaprod").exists():
        shutil.rmtree(SCRATCH, ignore_errors=True)
        shutil.copytree("/root/reference/pkg", SCRATCH)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                       check=True, capture_output=True)
    sys.path.insert(0, str(SCRATCH / "src"))
    import moaprod  # noqa: PLC0415
    assert moaprod.active_backend() == "compiled", "reference compiled backend not built"
    return moaprod


def rand_shape(rng, rank, lo=1, hi=5):
    return tuple(int(e) for e in rng.integers(lo, hi + 1, size=rank))


SPECIALS = np.array([np.nan, np.inf, -np.inf, 0.0, -0.0, 1.0, -1.0, 2.5, -3.0, 1e-310,
                     1e308, -1e308, 0.5], dtype=np.float64)


def main() -> None:
    mp = load_reference()
    sys.path.insert(0, str(REPO))
    from paper_0907_0792_b200.workloads import WORKLOADS  # noqa: PLC0415

    pairs = list(mp.builtin_pairs())
    cases = []  # (mode, comb, red, shape_a, a, shape_b, b, out, tag)

    def add(mode, ops, sa, a, sb, b, tag, dtype=np.float64):
        A = mp.MoaArray(sa, np.asarray(a, dtype=np.float64))
        B = mp.MoaArray(sb, np.asarray(b, dtype=np.float64))
        fn = mp.inner if mode == "inner" else mp.outer
        out = fn(A, B, ops)
        c, r = ops.codes()
        cases.append((mode, c, r, sa, np.asarray(a, dtype=dtype), sb,
                      np.asarray(b, dtype=dtype), out.data.copy(), out.shape, tag))

    rng = np.random.default_rng(20240811)
    # random small inner/outer over every pair (conftest.py:7-27 distributions)
    for rep in range(10):
        for ops in pairs:
            ra, rb = int(rng.integers(1, 5)), int(rng.integers(1, 5))
            k = int(rng.integers(1, 6))
            sa = rand_shape(rng, ra - 1) + (k,)
            sb = (k,) + rand_shape(rng, rb - 1)
            a = rng.random(math.prod(sa)) * 3.0 - 1.0
            b = rng.random(math.prod(sb)) * 3.0 - 1.0
            add("inner", ops, sa, a, sb, b, "random_inner")
        for ops in pairs if rep < 5 else []:
            sa = rand_shape(rng, int(rng.integers(0, 5)))
            sb = rand_shape(rng, int(rng.integers(0, 5)))
            add("outer", ops, sa, rng.random(math.prod(sa)) * 3.0 - 1.0, sb,
                rng.random(math.prod(sb)) * 3.0 - 1.0, "random_outer")
    # special values: NaN, +-inf, +-0, subnormal, huge
    for rep in range(4):
        for ops in pairs:
            m, k, n = (int(v) for v in rng.integers(1, 8, size=3))
            a = rng.choice(SPECIALS, size=m * k)
            b = rng.choice(SPECIALS, size=k * n)
            add("inner", ops, (m, k), a, (k, n), b, "special_inner")
            if rep < 2:
                add("outer", ops, (m,), rng.choice(SPECIALS, size=m), (n,),
                    rng.choice(SPECIALS, size=n), "special_outer")
    # medium products with ragged tile edges (GPU tiles are 64/128 wide, BK=16)
    for ops in pairs:
        m, k, n = 37, 67, 45
        add("inner", ops, (m, k), rng.random(m * k) * 3.0 - 1.0, (k, n),
            rng.random(k * n) * 3.0 - 1.0, "medium_inner")
    for ops in (mp.op_pair("multiply", "add"), mp.op_pair("add", "min")):
        m, k, n = 131, 300, 257
        add("inner", ops, (m, k), rng.random(m * k) * 3.0 - 1.0, (k, n),
            rng.random(k * n) * 3.0 - 1.0, "large_inner")
    # float32 inputs (the reference upcasts; GPU output = float32(reference))
    for ops in pairs:
        m, k, n = 19, 41, 23
        a = (rng.random(m * k, dtype=np.float32) * np.float32(100))
        b = (rng.random(k * n, dtype=np.float32) * np.float32(100))
        a[rng.random(m * k) < 0.05] = np.inf
        b[rng.random(k * n) < 0.05] = np.inf
        add("inner", ops, (m, k), a, (k, n), b, "f32_inner", dtype=np.float32)
    for ops in (mp.op_pair("add", "min"), mp.op_pair("add", "max"),
                mp.op_pair("subtract", "min"), mp.op_pair("subtract", "max")):
        m, k, n = 130, 77, 140
        a = rng.random(m * k, dtype=np.float32) * np.float32(100)
        b = rng.random(k * n, dtype=np.float32) * np.float32(100)
        a[rng.random(m * k) < 0.05] = np.inf
        b[rng.random(k * n) < 0.05] = np.inf
        add("inner", ops, (m, k), a, (k, n), b, "f32_tropical", dtype=np.float32)
        # with specials that defeat the fast loop (NaN, -inf, -0)
        a2 = a.copy()
        a2[rng.random(m * k) < 0.02] = np.nan
        a2[rng.random(m * k) < 0.02] = -np.inf
        b2 = b.copy()
        b2[rng.random(k * n) < 0.02] = -0.0
        a2[rng.random(m * k) < 0.02] = -0.0
        add("inner", ops, (m, k), a2, (k, n), b2, "f32_tropical_specials", dtype=np.float32)
    # hand-checked answers of the reference tests
    mul_add = mp.op_pair("multiply", "add")
    add("inner", mul_add, (2, 3), [1, 2, 3, 4, 5, 6], (3, 4), list(range(12)), "fig1")
    add("inner", mul_add, (3,), [1, 2, 3], (3,), [4, 5, 6], "dot")
    add("outer", mul_add, (2,), [1, 2], (2,), [10, 20], "outer_hand")
    add("inner", mp.op_pair("add", "min"), (2,), [1, 2], (2,), [10, 20], "tropical_dot")
    add("inner", mul_add, (1, 1), [3.0], (1, 1), [5.0], "singleton")
    add("outer", mul_add, (), [3.0], (), [4.0], "scalar_scalar")
    for name in ("add", "multiply", "min", "max"):
        add("inner", mp.op_pair("multiply", name), (2, 0), [], (0, 3), [], f"empty_{name}")
        add("outer", mp.op_pair("multiply", name), (), [-1.0], (), [0.0], f"negzero_{name}")
    add("inner", mul_add, (0, 3), [], (3, 4), list(range(12)), "zero_rows")
    add("inner", mul_add, (3, 4), list(range(12)), (4, 0), [], "zero_cols")
    a = rng.random(6)
    add("outer", mp.op_pair("subtract", "add"), (3, 2), a, (3, 2), a, "sub_self")

    # integer inputs (the reference upcasts to float64; with small integer
    # values every partial result is exact, so the reference's float64 result
    # IS the integer result).  divide is excluded: integer division truncates.
    for dt in (np.int32, np.int64):
        for ops in pairs:
            if ops.combine_name == "divide":
                continue
            m, k, n = (int(v) for v in rng.integers(1, 9, size=3))
            lim = 4 if ops.reduce_name == "multiply" else 100
            a = rng.integers(-lim, lim + 1, size=m * k).astype(dt)
            b = rng.integers(-lim, lim + 1, size=k * n).astype(dt)
            add("inner", ops, (m, k), a, (k, n), b, "int_inner", dtype=dt)
            add("outer", ops, (m,), a[:m], (n,), b[:n], "int_outer", dtype=dt)
        for ops in (mp.op_pair("multiply", "add"), mp.op_pair("add", "min"),
                    mp.op_pair("subtract", "max")):
            m, k, n = 37, 67, 45
            a = rng.integers(-1000, 1001, size=m * k).astype(dt)
            b = rng.integers(-1000, 1001, size=k * n).astype(dt)
            add("inner", ops, (m, k), a, (k, n), b, "int_medium", dtype=dt)

    # float32 inputs whose products/quotients under- or overflow float32 (but
    # not float64), with both signs, zeros and subnormals: the float32 result
    # must still be the reference's float64 fold rounded once (signed-zero ties
    # from float32 underflow must not leak in).  Appended last so the earlier
    # cases keep their indices.
    for ops in pairs:
        m, k, n = 17, 29, 19
        a = ((rng.random(m * k) * 2 - 1) * 10.0 ** rng.integers(-30, 31, m * k)).astype(np.float32)
        b = ((rng.random(k * n) * 2 - 1) * 10.0 ** rng.integers(-30, 31, k * n)).astype(np.float32)
        a[rng.random(m * k) < 0.05] = 0.0
        b[rng.random(k * n) < 0.05] = -0.0
        a[rng.random(m * k) < 0.03] = 1e-45
        b[rng.random(k * n) < 0.03] = -3e-39
        add("inner", ops, (m, k), a, (k, n), b, "f32_underflow", dtype=np.float32)
    for red in ("max", "min"):  # max-times on non-negative data with tiny values
        ops = mp.op_pair("multiply", red)
        m, k, n = 40, 33, 36
        a = (rng.random(m * k) * 10.0 ** rng.integers(-25, 5, m * k)).astype(np.float32)
        b = (rng.random(k * n) * 10.0 ** rng.integers(-25, 5, k * n)).astype(np.float32)
        a[rng.random(m * k) < 0.05] = 0.0
        add("inner", ops, (m, k), a, (k, n), b, "f32_maxtimes", dtype=np.float32)

    arrays = {}
    for i, (mode, c, r, sa, a, sb, b, out, oshape, tag) in enumerate(cases):
        meta = [0 if mode == "inner" else 1, c, r, len(sa), *sa, len(sb), *sb]
        arrays[f"c{i}_meta"] = np.array(meta, dtype=np.int64)
        arrays[f"c{i}_a"] = a
        arrays[f"c{i}_b"] = b
        arrays[f"c{i}_out"] = out
        arrays[f"c{i}_tag"] = np.array(tag)
    arrays["count"] = np.array(len(cases))
    np.savez_compressed(HERE / "small.npz", **arrays)
    print(f"small.npz: {len(cases)} cases")

    # ---- full-size config pins on row subsets -------------------------------
    rows_for = {"c1": list(range(0, 256, 17)) + [255], "c2": [0, 1, 2, 777, 32768, 65535],
                "c3": [0, 1, 4095, 4096, 20000, 32767],
                "c4": [0, 1, 127, 128, 8191, 8192, 12345, 16383],
                "c5": [0, 1, 127, 128, 8191, 8192, 12345, 16383]}
    configs = {}
    for key, w in WORKLOADS.items():
        a, b = w.generate()
        m, k, n = w.mkn
        rows = rows_for[key]
        a_rows = np.concatenate([a[i * k:(i + 1) * k] for i in rows])
        A = mp.MoaArray((len(rows), k) if w.mode == "inner" else (len(rows),), a_rows)
        if w.mode == "inner":
            B = mp.MoaArray((k, n), b)
            out = mp.execute_parallel(mp.plan_inner(A.shape, B.shape), A, B,
                                      mp.op_pair(w.ops.combine_name, w.ops.reduce_name), 8)
        else:
            B = mp.MoaArray((n,), b)
            out = mp.execute_parallel(mp.plan_outer(A.shape, B.shape), A, B,
                                      mp.op_pair(w.ops.combine_name, w.ops.reduce_name), 8)
        data = out.data.reshape(len(rows), n)
        entry = {"rows": rows, "sha256_f64": hashlib.sha256(data.tobytes()).hexdigest(),
                 "samples": {str(r): [float(x) for x in data[i, :4]] for i, r in enumerate(rows)},
                 "row_absmax": [float(np.max(np.abs(data[i]))) for i in range(len(rows))]}
        if w.dtype == np.float32:
            entry["sha256_f32"] = hashlib.sha256(data.astype(np.float32).tobytes()).hexdigest()
        configs[key] = entry
        print(key, entry["sha256_f64"][:16])
    (HERE / "configs.json").write_text(json.dumps(configs, indent=1) + "\n")


if __name__ == "__main__":
    main()
