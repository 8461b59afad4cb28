"""Per-call timings of moa_product_rows_host (the C ABI on host buffers) for
result/input memory kinds: page-locked (torch), pageable prefaulted (np.full),
pageable fresh (kernel.host_empty).  Prints JSON lines."""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_0907_0792_b200.kernel import host_empty, launch_host, plan_inner, plan_outer  # noqa: E402
from paper_0907_0792_b200.workloads import WORKLOADS  # noqa: E402


def pinned(x):
    t = torch.empty(x.size, dtype=torch.from_numpy(x[:1]).dtype, pin_memory=True).numpy()
    t[:] = x
    return t


def run(key, kinds, reps=4):
    w = WORKLOADS[key]
    a, b = w.generate()
    m, k, n = w.mkn
    plan = (plan_inner if w.mode == "inner" else plan_outer)(w.shape_a, w.shape_b)
    pa, pb = pinned(a), pinned(b)
    for kind in kinds:
        ins, res_kind = kind.split("/")
        A, B = (pa, pb) if ins == "pin" else (a, b)
        times = []
        keep = None
        for r in range(reps):
            if res_kind == "pin":
                res = keep if keep is not None else torch.empty(m * n, dtype=torch.from_numpy(a[:1]).dtype, pin_memory=True).numpy()
                keep = res
            elif res_kind == "faulted":
                res = keep if keep is not None else np.full(m * n, 0, dtype=a.dtype)
                keep = res
            else:
                res = host_empty(m * n, a.dtype)
            t0 = time.perf_counter()
            launch_host(plan, res, A, B, w.ops)
            times.append(time.perf_counter() - t0)
            del res
        print(json.dumps({"cfg": key, "inputs": ins, "res": res_kind,
                          "ms": [round(t * 1e3, 2) for t in times]}), flush=True)


if __name__ == "__main__":
    run("c1", ["pin/pin", "page/faulted"], reps=20)
    run("c2", ["pin/pin", "pin/faulted", "pin/fresh", "page/faulted"])
    for key in sys.argv[1:]:
        run(key, ["pin/pin", "page/faulted", "page/pin"], reps=3)
