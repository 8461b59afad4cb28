"""Accumulate-mode throughput vs the write-only launch at 4096^3 (tools; run on
a GPU box): float32 tropical pairs should both run the fast fold, and the other
routes should lose little to the accumulate variant."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0907_0792_b200 as moa  # noqa: E402
from paper_0907_0792_b200.kernel import launch, plan_inner  # noqa: E402

n = 4096
g = np.random.default_rng(0)
plan = plan_inner((n, n), (n, n))
cases = [(np.float32, "add", "min"), (np.float32, "add", "max"), (np.float64, "add", "min"),
         (np.float64, "multiply", "add"), (np.float64, "multiply", "max"), (np.float64, "divide", "add"),
         (np.float64, "max", "max"), (np.float64, "min", "min"), (np.float64, "divide", "max"),
         (np.float64, "max", "add"), (np.float64, "multiply", "multiply")]
if len(sys.argv) > 1:  # only float64 routes
    cases = [c for c in cases if c[0] == np.float64]
for dt, comb, red in cases:
    a = torch.from_numpy((g.random(n * n) * 100).astype(dt)).cuda()
    b = torch.from_numpy((g.random(n * n) * 100 + 1).astype(dt)).cuda()
    ops = moa.op_pair(comb, red)
    for acc in (False, True):
        res = torch.full((n * n,), float(ops.reduce_identity), dtype=a.dtype, device="cuda")
        launch(plan, res, a, b, ops, accumulate=acc)
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            launch(plan, res, a, b, ops, accumulate=acc)
            e.record()
            e.synchronize()
            best = min(best, s.elapsed_time(e))
        print(f"{np.dtype(dt).name} {comb}/{red} accumulate={acc}: "
              f"{n ** 3 / (best * 1e-3) / 1e9:.1f} G pairs/s")
