"""Accumulate-mode throughput of the float32 tropical route vs the write-only
route at 4096^3 (tools; run on a GPU box): both should run the fast fold."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0907_0792_b200 as moa  # noqa: E402
from paper_0907_0792_b200.kernel import launch, plan_inner  # noqa: E402

n = 4096
g = np.random.default_rng(0)
a = torch.from_numpy((g.random(n * n) * 100).astype(np.float32)).cuda()
b = torch.from_numpy((g.random(n * n) * 100).astype(np.float32)).cuda()
plan = plan_inner((n, n), (n, n))
for red in ("min", "max"):
    ops = moa.op_pair("add", red)
    for acc in (False, True):
        res = torch.full((n * n,), float(ops.reduce_identity), dtype=torch.float32, device="cuda")
        launch(plan, res, a, b, ops, accumulate=acc)
        torch.cuda.synchronize()
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            launch(plan, res, a, b, ops, accumulate=acc)
            e.record()
            e.synchronize()
            print(f"add/{red} accumulate={acc}: {n ** 3 / (s.elapsed_time(e) * 1e-3) / 1e9:.1f} G pairs/s")
