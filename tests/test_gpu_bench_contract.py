"""bench.py keeps the driver's JSON contract (one line, required keys, sane
values) — run as the driver runs it, in a subprocess on the GPU."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
            "gpu_launches", "roofline", "clocks"}


def _run(*args) -> dict:
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=REPO, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_default_line_contract():
    d = _run("--steps", "3", "--warmup", "3", "--no-inner")
    assert REQUIRED <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3
    assert d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] >= 3
    assert "workload" in d["config"]
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["e2e_pageable"]["value"] > 0 and d["e2e_pageable"]["first_call_ms"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert "theoretical" in r
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] > 0
    assert d["clocks"]["sm_mhz"] is not None


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["cores"] >= 1
    ours = _run("--steps", "3", "--warmup", "3", "--no-inner", "--no-cpu")
    assert d["config"] == ours["config"]   # the driver's same_config check
    for key in ("metric", "unit", "higher_is_better", "scaling", "dtype"):
        assert d[key] == ours[key]


def test_multi_rank_line_over_gloo():
    """The N>1 code path the driver's scaling run takes (torchrun, one JSON
    line from rank 0, max over ranks), exercised with two ranks sharing the
    test box's GPU over gloo (timings meaningless there; NCCL needs one GPU
    per rank): weak c2 with B broadcast once, strong c4/c5 legs with the
    k-chunked broadcast inside every step."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", str(port), "bench.py", "--gpus", "2", "--steps", "2",
                          "--warmup", "3", "--dist-backend", "gloo", "--no-cpu"],
                         cwd=REPO, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert REQUIRED <= d.keys() and d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert "once, before the timed region" in d["config"]["parallelism"]
    assert set(d["inner"]) == {"c4", "c5"}
    for leg in d["inner"].values():
        assert leg["scaling"] == "strong" and leg["rows_per_rank"] == 8192 and leg["value"] > 0
        assert leg["e2e"]["value"] > 0 and leg["e2e"]["d2h_bytes_per_step"] > 0
