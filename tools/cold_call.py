"""Cold and warm end-to-end calls of the public API on plain (pageable) numpy
inputs, in a fresh process: the cost a user sees on the first c2-sized outer
product (after one tiny call has created the CUDA context and loaded the
library), then steady state.  Prints one JSON line."""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

import paper_0907_0792_b200 as moa  # noqa: E402
from paper_0907_0792_b200 import MoaArray  # noqa: E402
from paper_0907_0792_b200.workloads import WORKLOADS  # noqa: E402


def timed(fn):
    t0 = time.perf_counter()
    out = fn()
    return out, time.perf_counter() - t0


def main():
    out = {}
    _, out["tiny_first_call_s"] = timed(lambda: moa.outer(MoaArray((2,), [1.0, 2.0]),
                                                          MoaArray((2,), [3.0, 4.0])))
    for key in ("c2", "c1") + tuple(sys.argv[1:]):
        w = WORKLOADS[key]
        a, b = w.generate()
        A, B = MoaArray(w.shape_a, a, dtype=w.dtype), MoaArray(w.shape_b, b, dtype=w.dtype)
        fn = moa.outer if w.mode == "outer" else moa.inner
        res, first = timed(lambda: fn(A, B, w.ops))
        del res
        warm = []
        for _ in range(5):
            res, t = timed(lambda: fn(A, B, w.ops))
            warm.append(t)
            del res
        out[key] = {"first_call_ms": round(first * 1e3, 2),
                    "warm_ms": [round(t * 1e3, 2) for t in warm],
                    "result_bytes": w.mkn[0] * w.mkn[2] * np.dtype(w.dtype).itemsize}
        out[key]["warm_GBps_result"] = round(out[key]["result_bytes"] / min(warm) / 1e9, 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
