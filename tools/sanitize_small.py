"""Small products through every kernel route, for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python tools/sanitize_small.py
(ragged edges, unaligned operands, every op pair and dtype, row subsets,
accumulate, fill and outer routes)."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0907_0792_b200 as moa  # noqa: E402
from paper_0907_0792_b200.kernel import launch, plan_inner, plan_outer  # noqa: E402

rng = np.random.default_rng(3)
n_calls = 0
for dt in (torch.float64, torch.float32):
    for ops in moa.builtin_pairs():
        for (m, k, n) in ((1, 1, 1), (37, 19, 45), (130, 33, 129), (3, 0, 5), (65, 1, 67)):
            a = torch.from_numpy(rng.random(m * k + 1) * 3 - 1).to(dt).cuda()
            b = torch.from_numpy(rng.random(k * n + 1) * 3 - 1).to(dt).cuda()
            c = torch.zeros(m * n + 1, dtype=dt, device="cuda")
            plan = plan_inner((m, k), (k, n))
            launch(plan, c[:m * n], a[:m * k], b[:k * n], ops)            # aligned
            launch(plan, c[1:], a[1:], b[1:], ops)                         # misaligned
            launch(plan, c[:m * n], a[:m * k], b[:k * n], ops, start=1, step=3)
            launch(plan, c[:m * n], a[:m * k], b[:k * n], ops, accumulate=True)
            launch(plan, c[:m * n], a[:m * k], b[:k * n], ops, exact=True)
            n_calls += 5
    x = torch.from_numpy(rng.random(300)).to(dt).cuda()
    y = torch.from_numpy(rng.random(2048)).to(dt).cuda()
    o = torch.empty(300 * 2048, dtype=dt, device="cuda")
    launch(plan_outer((300,), (2048,)), o, x, y, moa.MUL_ADD)
    n_calls += 1
torch.cuda.synchronize()
print(f"sanitize_small: {n_calls} launches ok")
