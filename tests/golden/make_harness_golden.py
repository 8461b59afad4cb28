"""Golden records of the REFERENCE's experiment harness (run in the build container).

    python tests/golden/make_harness_golden.py

Imports the reference package (built in /tmp by make_golden.load_reference)
and runs its own ``moaprod.bench.run_experiment`` (bench.py:154-177) for the
fixed experiments in ``EXPERIMENTS`` below, then its ``derive_metrics``
(bench.py:180-209) and ``emit_csv`` (bench.py:222-247).  Writes
``harness_ref.json``: for each experiment the reference's raw CSV text and,
per (mode, threads), the metric CSV text derived against the single-worker
records.  tests/test_harness.py checks this repo's harness against it: the
same CSV schema and row keys, checksums bitwise for the exact folds and within
the K*2^-52 sum bound for (multiply, add) on the tensor cores, and metric
arithmetic identical when fed the reference's own timings.
"""

from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

# (name, ExperimentConfig keyword arguments) — small sweeps the GPU test reruns
EXPERIMENTS = [
    ("inner_w1", dict(mode="moa-inner", workers=1, ell=128, n_list=(2, 4, 8, 16, 32, 64),
                      repeats=2, seed=11)),
    ("inner_w2", dict(mode="moa-inner", workers=2, ell=128, n_list=(2, 4, 8, 16, 32, 64),
                      repeats=2, seed=11)),
    ("inner_rows", dict(mode="moa-inner", workers=1, ell=37, n_list=(3, 17, 250), repeats=1,
                        seed=5, rows=70)),
    ("inner_tropical", dict(mode="moa-inner", workers=3, ell=64, n_list=(8, 100), repeats=1,
                            seed=2, rows=50, combine="add", reduce="min")),
    ("inner_short_k", dict(mode="moa-inner", workers=1, ell=5, n_list=(4, 64), repeats=1,
                           seed=3, rows=40)),
    ("outer_w1", dict(mode="moa-outer", workers=1, ell=1, n_list=(2, 4, 8, 16), repeats=1,
                      seed=4, combine="add", reduce="min")),
    ("outer_mul", dict(mode="moa-outer", workers=2, ell=1, n_list=(64, 512), repeats=1,
                       seed=6, rows=33)),
    ("gemm_w1", dict(mode="gemm-baseline", workers=1, ell=128, n_list=(2, 8, 32), repeats=2,
                     seed=11)),
]


def _csv(bench, rows, kind):
    with tempfile.NamedTemporaryFile("r", suffix=".csv") as fh:
        bench.emit_csv(fh.name, rows, kind=kind)
        return Path(fh.name).read_text()


def main() -> None:
    from make_golden import load_reference
    mp = load_reference()
    from moaprod import bench  # noqa: PLC0415
    out = {}
    for name, kw in EXPERIMENTS:
        cfg = bench.ExperimentConfig(**kw)
        res = bench.run_experiment(cfg)
        assert not res.failures, res.failures
        base = [r for r in res.records if r.threads == 1]
        metrics = bench.derive_metrics(res.records, base) if base else []
        out[name] = {"config": {k: (list(v) if isinstance(v, tuple) else v) for k, v in kw.items()},
                     "raw_csv": _csv(bench, res.records, "raw"),
                     "metrics_csv": _csv(bench, metrics, "metrics") if base else None}
    # derive_metrics across experiments: inner_w2 against inner_w1's single-worker
    # runs, read back through the reference's read_records_csv (it takes a path)
    with tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False) as f1, \
            tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False) as f2:
        f1.write(out["inner_w1"]["raw_csv"])
        f2.write(out["inner_w2"]["raw_csv"])
    w1 = bench.read_records_csv(f1.name)
    w2 = bench.read_records_csv(f2.name)
    out["metrics_w2_vs_w1"] = _csv(bench, bench.derive_metrics(w2, w1), "metrics")
    out["_generator"] = ("tests/golden/make_harness_golden.py: reference moaprod.bench "
                         f"(numpy {__import__('numpy').__version__})")
    (HERE / "harness_ref.json").write_text(json.dumps(out, indent=1))
    print(f"wrote {HERE / 'harness_ref.json'} ({len(EXPERIMENTS)} experiments)")
    del mp


if __name__ == "__main__":
    main()
