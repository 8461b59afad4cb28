"""The experiment harness and CLI (reference tests/test_bench.py, test_cli.py
restated).  CPU tests exercise config validation, metrics, CSV formats and
exit codes; GPU tests run real sweeps and one-off products."""

from __future__ import annotations

import math

import numpy as np
import pytest

from paper_0907_0792_b200 import MoaArray, dump, harness, loads
from paper_0907_0792_b200.cli import main
from paper_0907_0792_b200.harness import (ExperimentConfig, ExperimentResult, MetricRow,
                                          SizeFailure, TimingRecord, derive_metrics, emit_csv,
                                          operand_pair, read_records_csv)


def _rec(mode="moa-inner", threads=1, n=2, rep=0, secs=1.0, cs=3.5):
    return TimingRecord(mode, threads, 8, n, rep, secs, cs)


def test_config_validation():
    with pytest.raises(ValueError):
        ExperimentConfig(mode="nope")
    with pytest.raises(ValueError):
        ExperimentConfig(mode="moa-inner", workers=0)
    with pytest.raises(ValueError):
        ExperimentConfig(mode="moa-inner", ell=0)
    with pytest.raises(ValueError):
        ExperimentConfig(mode="moa-inner", repeats=0)
    with pytest.raises(ValueError):
        ExperimentConfig(mode="gemm-baseline", combine="add", reduce="min")
    ExperimentConfig(mode="moa-outer", combine="add", reduce="min")


def test_operand_pair_deterministic_and_shaped():
    a1, b1 = operand_pair(3, 2, 8, 16)
    a2, b2 = operand_pair(3, 2, 8, 16)
    assert a1.shape == (2, 8) and b1.shape == (8, 16)
    assert a1 == a2 and b1 == b2
    assert np.all((a1.data >= 0) & (a1.data < 1))
    # same generator as the reference's bench.operand_pair (bench.py:101-111)
    gen = np.random.default_rng([3, 2, 8, 16])
    np.testing.assert_array_equal(a1.data, gen.random((2, 8)).ravel())


def test_derive_metrics_ratio_and_flag():
    base = [_rec(threads=1, n=2, secs=1.0), _rec(threads=1, n=2, rep=1, secs=3.0)]
    recs = [_rec(threads=2, n=2, secs=5.0), _rec(threads=2, n=2, rep=1, secs=5.0)]
    rows = derive_metrics(recs, base)
    assert rows == [MetricRow("moa-inner", 2, 2, 5.0, 4, 2.5, True)]
    assert derive_metrics(base, base)[0].ratio == 1.0
    with pytest.warns(UserWarning):
        rows = derive_metrics([_rec(n=4)], [])
    assert rows[0].ratio is None and rows[0].no_net_benefit is None


def test_csv_round_trip_and_headers(tmp_path):
    recs = [_rec(n=4, rep=1, secs=0.1, cs=1 / 3), _rec(n=2, secs=2e-5, cs=math.pi)]
    p = tmp_path / "raw.csv"
    emit_csv(p, recs)
    lines = p.read_text().splitlines()
    assert lines[0] == "mode,threads,ell,n,repeat,seconds,checksum"
    back = read_records_csv(p)
    assert back == sorted(recs, key=lambda r: (r.mode, r.threads, r.n, r.repeat))
    m = tmp_path / "m.csv"
    emit_csv(m, derive_metrics(recs, recs))
    assert m.read_text().splitlines()[0] == \
        "mode,threads,n,mean_seconds,total_x,ratio,no_net_benefit"
    emit_csv(tmp_path / "empty.csv", [], kind="metrics")
    assert (tmp_path / "empty.csv").read_text().startswith("mode,threads,n,mean_seconds")
    with pytest.raises(ValueError):
        emit_csv(tmp_path / "x.csv", recs, kind="bogus")


def test_cli_bad_bounds_and_failure_exit_codes(tmp_path, monkeypatch, capsys):
    out = tmp_path / "raw.csv"
    assert main(["bench", "--mode", "moa-inner", "--n-min", "5", "--n-max", "2",
                 "--out", str(out)]) == 2
    assert "bad sweep bounds" in capsys.readouterr().err
    result = ExperimentResult(records=[], failures=[SizeFailure("moa-inner", 1, 8, 4, "OOM")])
    monkeypatch.setattr(harness, "run_experiment", lambda cfg: result)
    args = ["bench", "--mode", "moa-inner", "--out", str(out)]
    assert main(args) == 1
    assert main(args + ["--keep-going"]) == 0


def test_cli_metrics_command(tmp_path):
    raw1, raw2, out = tmp_path / "r1.csv", tmp_path / "r2.csv", tmp_path / "m.csv"
    emit_csv(raw1, [_rec(threads=1, n=n, secs=1.0) for n in (2, 4)])
    emit_csv(raw2, [_rec(threads=2, n=n, secs=1.5) for n in (2, 4)])
    assert main(["metrics", "--raw", str(raw2), "--baseline-raw", str(raw1),
                 "--out", str(out)]) == 0
    cells = [ln.split(",") for ln in out.read_text().splitlines()[1:]]
    assert [c[5] for c in cells] == ["1.5", "1.5"]
    assert [c[6] for c in cells] == ["false", "false"]


# ---- on the GPU ----------------------------------------------------------------

@pytest.mark.gpu
def test_sweep_modes_and_checksums(tmp_path):
    raws = {}
    for mode in ("moa-inner", "gemm-baseline"):
        out = tmp_path / f"{mode}.csv"
        assert main(["bench", "--mode", mode, "--threads", "2", "--ell", "128", "--n-min", "1",
                     "--n-max", "8", "--repeats", "2", "--seed", "9", "--out", str(out)]) == 0
        raws[mode] = read_records_csv(out)
        assert [r.n for r in raws[mode]] == [2**p for p in range(1, 9) for _ in range(2)]
        assert all(r.seconds > 0 and r.threads == 2 for r in raws[mode])
    for x, y in zip(raws["moa-inner"], raws["gemm-baseline"]):
        assert x.n == y.n and x.checksum == pytest.approx(y.checksum, rel=1e-12)
    outer = tmp_path / "outer.csv"
    assert main(["bench", "--mode", "moa-outer", "--ell", "1", "--n-max", "4",
                 "--combine", "add", "--reduce", "min", "--repeats", "1",
                 "--out", str(outer)]) == 0
    assert len(read_records_csv(outer)) == 4


@pytest.mark.gpu
def test_product_command_matches_api(tmp_path, capsys):
    import paper_0907_0792_b200 as moa
    left, right = tmp_path / "a.txt", tmp_path / "b.txt"
    dump(MoaArray((2, 3), [1, 2, 3, 4, 5, 6]), left)
    dump(MoaArray((3, 4), range(12)), right)
    assert main(["product", "--mode", "inner", "--left", str(left), "--right", str(right)]) == 0
    got = loads(capsys.readouterr().out)
    assert got.shape == (2, 4) and got.data.tolist() == [32, 38, 44, 50, 68, 83, 98, 113]
    dump(MoaArray((2,), [1, 2]), left)
    dump(MoaArray((2,), [10, 20]), right)
    out = tmp_path / "c.txt"
    assert main(["product", "--mode", "inner", "--left", str(left), "--right", str(right),
                 "--combine", "add", "--reduce", "min", "--threads", "3", "--out", str(out)]) == 0
    assert moa.load(out).item() == 11.0


def test_memory_failure_recorded_and_sweep_continues(monkeypatch):
    """reference tests/test_bench.py: a size that runs out of memory becomes a
    SizeFailure and the sweep goes on (the product itself stubbed: CPU test)."""
    real = harness.operand_pair

    def flaky(seed, rows, ell, n):
        if n == 8:
            raise MemoryError("simulated allocation failure")
        return real(seed, rows, ell, n)

    def fake_timer(config, a, b, n, out):
        out.records.append(TimingRecord(config.mode, config.workers, config.ell, n, 0, 1e-3, 0.0))

    monkeypatch.setattr(harness, "operand_pair", flaky)
    monkeypatch.setattr(harness, "_time_product", fake_timer)
    cfg = ExperimentConfig(mode="moa-inner", workers=1, ell=8, n_list=[4, 8, 16], repeats=1)
    result = harness.run_experiment(cfg)
    assert [r.n for r in result.records] == [4, 16]
    assert len(result.failures) == 1 and result.failures[0].n == 8
    assert "MemoryError" in result.failures[0].error
    with pytest.raises(ValueError):
        harness.run_experiment(ExperimentConfig(mode="moa-inner", rows=0))


@pytest.mark.gpu
def test_experiment_checksums_independent_of_workers_and_reproducible():
    sums = {}
    for workers in (1, 2, 4):
        cfg = ExperimentConfig(mode="moa-inner", workers=workers, ell=16, n_list=[8], repeats=1,
                               seed=3, rows=2)
        sums[workers] = harness.run_experiment(cfg).records[0].checksum
    assert sums[1] == sums[2] == sums[4]
    cfg = ExperimentConfig(mode="moa-inner", workers=2, ell=8, n_list=[4], repeats=2, seed=5, rows=3)
    r1, r2 = harness.run_experiment(cfg), harness.run_experiment(cfg)
    assert [r.checksum for r in r1.records] == [r.checksum for r in r2.records]
    assert all(r.threads == 2 and r.seconds > 0 for r in r1.records)


# ---- against the reference harness's own records (tests/golden/harness_ref.json,
# made by tests/golden/make_harness_golden.py from the imported reference) -------

def _ref_harness():
    import json
    from conftest import GOLDEN
    return json.loads((GOLDEN / "harness_ref.json").read_text())


def _records_from_text(tmp_path, name, text):
    p = tmp_path / f"{name}.csv"
    p.write_text(text)
    return read_records_csv(p)


def test_reference_records_round_trip_and_metrics_identical(tmp_path):
    """The reference's raw CSV parses with this harness and re-emits to the same
    text; derive_metrics + emit_csv on the reference's own timings give the
    reference's metric CSV text exactly (bench.py:180-247)."""
    ref = _ref_harness()
    for name, exp in ref.items():
        if not isinstance(exp, dict):
            continue
        recs = _records_from_text(tmp_path, name, exp["raw_csv"])
        again = tmp_path / f"{name}_again.csv"
        emit_csv(again, recs)
        assert again.read_text() == exp["raw_csv"], name
        if exp["metrics_csv"] is not None:
            m = tmp_path / f"{name}_m.csv"
            emit_csv(m, derive_metrics(recs, [r for r in recs if r.threads == 1]), kind="metrics")
            assert m.read_text() == exp["metrics_csv"], name
    w1 = _records_from_text(tmp_path, "w1", ref["inner_w1"]["raw_csv"])
    w2 = _records_from_text(tmp_path, "w2", ref["inner_w2"]["raw_csv"])
    m = tmp_path / "w2w1.csv"
    emit_csv(m, derive_metrics(w2, w1), kind="metrics")
    assert m.read_text() == ref["metrics_w2_vs_w1"]


@pytest.mark.gpu
def test_harness_records_match_the_reference_harness(tmp_path):
    """This harness run on the GPU with the reference's experiment configs:
    identical CSV schema and row keys (mode, threads, ell, n, repeat);
    checksums bit-identical for the exact folds (tropical, outer products,
    (multiply, add) below K = 8) and within the north-star sum bound
    K*2^-52*max|A|*max|B| per element for (multiply, add) on the tensor cores
    and the cuBLAS comparator."""
    ref = _ref_harness()
    for name, exp in ref.items():
        if not isinstance(exp, dict):
            continue
        cfg = ExperimentConfig(**exp["config"])
        res = harness.run_experiment(cfg)
        assert not res.failures
        ours = tmp_path / f"{name}.csv"
        emit_csv(ours, res.records)
        assert ours.read_text().splitlines()[0] == exp["raw_csv"].splitlines()[0]
        theirs = _records_from_text(tmp_path, f"{name}_ref", exp["raw_csv"])
        mine = read_records_csv(ours)
        assert [(r.mode, r.threads, r.ell, r.n, r.repeat) for r in mine] == \
            [(r.mode, r.threads, r.ell, r.n, r.repeat) for r in theirs], name
        rows = cfg.rows if cfg.rows is not None else cfg.workers
        exact = (cfg.mode == "moa-outer" or (cfg.combine, cfg.reduce) != ("multiply", "add")
                 or (cfg.mode == "moa-inner" and cfg.ell < 8))
        for x, y in zip(mine, theirs):
            if exact:
                assert x.checksum == y.checksum, (name, x, y)
            else:  # values in [0, 1): max|A| = max|B| <= 1
                count = rows * x.n
                tol = count * cfg.ell * 2.0**-52 + 4 * 2.0**-52 * abs(y.checksum) * \
                    max(1.0, math.log2(count))
                assert abs(x.checksum - y.checksum) <= tol, (name, x, y, tol)
