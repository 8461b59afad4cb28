"""Shared fixtures.  Tests marked ``gpu`` need a B200 and the built library;
everything else runs on CPU (the driver runs ``-m "not gpu"`` in the build
container and ``-m gpu`` on a GPU box)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

GOLDEN = REPO / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and libmoa_b200.so")
    config.addinivalue_line("markers", "slow: full-size BASELINE workloads")


@pytest.fixture
def rng():
    return np.random.default_rng(20240811)


class GoldenCase:
    __slots__ = ("idx", "mode", "comb", "red", "shape_a", "a", "shape_b", "b", "out", "tag")

    def __repr__(self):
        return (f"GoldenCase#{self.idx}({self.tag}, {self.mode}, comb={self.comb}, "
                f"red={self.red}, {self.shape_a}x{self.shape_b})")


def load_golden_small() -> list[GoldenCase]:
    z = np.load(GOLDEN / "small.npz")
    cases = []
    for i in range(int(z["count"])):
        meta = [int(v) for v in z[f"c{i}_meta"]]
        c = GoldenCase()
        c.idx = i
        c.mode = "inner" if meta[0] == 0 else "outer"
        c.comb, c.red = meta[1], meta[2]
        ra = meta[3]
        c.shape_a = tuple(meta[4:4 + ra])
        rb = meta[4 + ra]
        c.shape_b = tuple(meta[5 + ra:5 + ra + rb])
        c.a, c.b, c.out = z[f"c{i}_a"], z[f"c{i}_b"], z[f"c{i}_out"]
        c.tag = str(z[f"c{i}_tag"])
        cases.append(c)
    return cases


@pytest.fixture(scope="session")
def golden_small():
    return load_golden_small()


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA GPU in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
