"""The five BASELINE.json workloads as seeded host generators.

There is no public dataset for this path; BASELINE.json's synthetic configs
are the workload, instantiated exactly as SURVEY.md §8(d) specifies
(``numpy.random.default_rng(seed)``, A drawn before B).  The same arrays feed
the reference oracle and the GPU build, so the parity checks and the CPU
baseline see identical inputs.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .arrays import element_count
from .ops import MUL_ADD, OpPair, op_pair


@dataclass(frozen=True)
class Workload:
    key: str
    mode: str            # "inner" | "outer"
    shape_a: tuple
    shape_b: tuple
    ops: OpPair
    dtype: np.dtype
    seed: int
    description: str

    @property
    def mkn(self) -> tuple[int, int, int]:
        if self.mode == "outer":
            return element_count(self.shape_a), 1, element_count(self.shape_b)
        return (element_count(self.shape_a[:-1]), self.shape_a[-1],
                element_count(self.shape_b[1:]))

    @property
    def flops(self) -> int:
        """Algorithmic work: 2*M*K*N (one combine + one reduce per pair)."""
        m, k, n = self.mkn
        return 2 * m * k * n

    @property
    def pairs(self) -> int:
        m, k, n = self.mkn
        return m * k * n

    @property
    def bytes(self) -> int:
        """Compulsory HBM bytes: read A and B once, write C once."""
        m, k, n = self.mkn
        isz = np.dtype(self.dtype).itemsize
        return isz * (m * k + k * n + m * n)

    def generate(self) -> tuple[np.ndarray, np.ndarray]:
        return _GENERATORS[self.key](self)


def _uniform_pair(w: Workload):
    rng = np.random.default_rng(w.seed)
    a = rng.uniform(-1.0, 1.0, element_count(w.shape_a))
    b = rng.uniform(-1.0, 1.0, element_count(w.shape_b))
    return a, b


def _tropical_pair(w: Workload):
    # draw order: A values, A mask, B values, B mask
    rng = np.random.default_rng(w.seed)
    out = []
    for shape in (w.shape_a, w.shape_b):
        n = element_count(shape)
        x = rng.random(n, dtype=np.float32) * np.float32(100)
        x[rng.random(n) < 0.05] = np.inf
        out.append(x)
    return out[0], out[1]


_N = 16384
WORKLOADS: dict[str, Workload] = {
    "c1": Workload("c1", "inner", (256, 256), (256, 256), MUL_ADD, np.dtype(np.float64), 0,
                   "matrix multiply as MoA inner product, (+,x), 256^2 . 256^2 f64"),
    "c2": Workload("c2", "outer", (32, 16, 16, 8), (16, 16, 8), MUL_ADD, np.dtype(np.float64), 1,
                   "generalized outer product, op x, rho<32 16 16 8> (x) rho<16 16 8> f64"),
    "c3": Workload("c3", "inner", (32, 32, 32, 256), (256, 64, 64), MUL_ADD,
                   np.dtype(np.float64), 2,
                   "tensor contraction rho<32 32 32 256> . rho<256 64 64> f64, K=256"),
    "c4": Workload("c4", "inner", (_N, _N), (_N, _N), MUL_ADD, np.dtype(np.float64), 3,
                   "large square (+,x) inner product 16384^2 . 16384^2 f64"),
    "c5": Workload("c5", "inner", (_N, _N), (_N, _N), op_pair("add", "min"),
                   np.dtype(np.float32), 4,
                   "tropical (min,+) inner product 16384^2 . 16384^2 f32, 5% +inf"),
}

_GENERATORS = {"c1": _uniform_pair, "c2": _uniform_pair, "c3": _uniform_pair,
               "c4": _uniform_pair, "c5": _tropical_pair}
