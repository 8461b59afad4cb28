"""Throughput of every (dtype, combine, reduce) route at one inner-product size.

Runs on a GPU box (tools; not part of the library):

    python tools/route_sweep.py [--n 4096] [--out gpurun_out/route_sweep.jsonl]

For each of the 4 dtypes x 24 op pairs: seeded operands of n x n (values that
keep every route on its common path: positive for the tropical fast loops,
small integers so integer products stay meaningful), one warm-up launch, then
the best of 3 CUDA-event-timed launches through ``kernel.launch`` (the C ABI).
Prints one JSON line per route with the kernel ``moa_plan_kernel`` reports and
G pairs/s (M*K*N / time).
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0907_0792_b200 as moa  # noqa: E402
from paper_0907_0792_b200 import _native  # noqa: E402
from paper_0907_0792_b200.kernel import launch, native_dtype, plan_inner  # noqa: E402


def operands(dt, n, gen):
    if np.dtype(dt).kind == "i":
        a = gen.integers(-1000, 1000, size=n * n).astype(dt)
        b = gen.integers(-1000, 1000, size=n * n).astype(dt)
    else:
        a = (gen.random(n * n) * 100).astype(dt)
        b = (gen.random(n * n) * 100).astype(dt)
    return torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--out", default="gpurun_out/route_sweep.jsonl")
    ap.add_argument("--only", default=None, help="dtype:combine:reduce, e.g. float64:add:min")
    ap.add_argument("--outer", action="store_true",
                    help="outer products (K = 1) of 65536 x 2048 instead (GB/s of result written)")
    args = ap.parse_args()
    n = args.n
    gen = np.random.default_rng(0)
    if args.outer:
        from paper_0907_0792_b200.kernel import plan_outer
        plan = plan_outer((65536,), (2048,))
    else:
        plan = plan_inner((n, n), (n, n))
    lines = []
    only = args.only.split(":") if args.only else None
    for dt in (np.float64, np.float32, np.int32, np.int64):
        if only and np.dtype(dt).name != only[0]:
            continue
        if args.outer:
            a, b = operands(dt, 256, gen)
            a, b = a[:plan.noproc], b[:plan.elsinop]
        else:
            a, b = operands(dt, n, gen)
        res = torch.empty(plan.noproc * plan.elsinop, dtype=a.dtype, device="cuda")
        for comb in moa.COMBINE_OPS:
            for red in moa.REDUCE_OPS:
                if only and (comb, red) != (only[1], only[2]):
                    continue
                ops = moa.op_pair(comb, red)
                c, r = ops.codes()
                kern = _native.plan_kernel(native_dtype(np.dtype(dt)), plan.noproc, plan.rowsinred,
                                           plan.elsinop, c, r, 0)
                launch(plan, res, a, b, ops)
                torch.cuda.synchronize()
                best = float("inf")
                for _ in range(3):
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    launch(plan, res, a, b, ops)
                    e.record()
                    e.synchronize()
                    best = min(best, s.elapsed_time(e))
                rec = {"dtype": np.dtype(dt).name, "combine": comb, "reduce": red, "kernel": kern,
                       "n": n, "ms": round(best, 4),
                       "Gpairs_s": round(n ** 3 / (best * 1e-3) / 1e9, 1)}
                if args.outer:
                    nbytes = plan.noproc * plan.elsinop * np.dtype(dt).itemsize
                    rec = {"dtype": np.dtype(dt).name, "combine": comb, "reduce": red,
                           "kernel": "outer", "M": plan.noproc, "N": plan.elsinop,
                           "ms": round(best, 4), "GB_s": round(nbytes / (best * 1e-3) / 1e9, 1)}
                lines.append(rec)
                print(json.dumps(rec), flush=True)
        del a, b, res
        torch.cuda.empty_cache()
        time.sleep(3)  # let clocks/power settle between dtype groups
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text("".join(json.dumps(x) + "\n" for x in lines))


if __name__ == "__main__":
    main()
