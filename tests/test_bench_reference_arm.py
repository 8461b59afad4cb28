"""The reference arm of bench.py (``--impl reference``) runs the reference's own
CPU loop and nothing of this repo's CUDA path, on the same workload
description as the repo's arm (CPU test: the arm needs no GPU)."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]

_PROBE = r"""
import json, runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--config", "{cfg}", "--steps", "1",
            "--warmup", "0"]
runpy.run_path("bench.py", run_name="__main__")
maps = open("/proc/self/maps").read()
print("MAPS " + json.dumps(sorted({{ln.split()[-1] for ln in maps.splitlines()
                                   if ln.split()[-1].endswith(".so") or ".so." in ln}})))
"""


def _run(cfg: str):
    out = subprocess.run([sys.executable, "-c", _PROBE.format(cfg=cfg)], cwd=REPO,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    line = json.loads(next(ln for ln in lines if ln.startswith("{")))
    maps = json.loads(next(ln for ln in lines if ln.startswith("MAPS "))[5:])
    return line, maps


def test_reference_arm_never_loads_the_cuda_library():
    line, maps = _run("c1")
    assert not any("libmoa_b200" in p for p in maps), maps
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port")


def test_reference_arm_config_matches_the_repo_arm():
    sys.path.insert(0, str(REPO))
    import bench
    from paper_0907_0792_b200.workloads import WORKLOADS
    line, _ = _run("c1")
    assert line["config"] == json.loads(json.dumps(bench.job_config(WORKLOADS["c1"], 1)))
    for key in ("metric", "unit", "higher_is_better", "scaling", "dtype"):
        assert key in line
    assert line["metric"] == bench.METRIC["c1"][0]


def test_package_import_does_not_dlopen():
    probe = ("import paper_0907_0792_b200, paper_0907_0792_b200.workloads;"
             "print('libmoa_b200' in open('/proc/self/maps').read())")
    out = subprocess.run([sys.executable, "-c", probe], cwd=REPO, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip() == "False"


def test_cpu_sample_rows_follow_the_survey_protocol():
    sys.path.insert(0, str(REPO))
    import bench
    from paper_0907_0792_b200.workloads import WORKLOADS
    for key in ("c1", "c2", "c3"):
        assert bench.cpu_rows_for(WORKLOADS[key], 16) == WORKLOADS[key].mkn[0]
    for key in ("c4", "c5"):
        assert bench.cpu_rows_for(WORKLOADS[key], 16) == 512   # R = 32 * W
