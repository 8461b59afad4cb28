"""Stress accumulate-mode launches: N repeated (x,+) float64 launches into a
zero-filled C, each compared bitwise with the write-only launch (tools)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_0907_0792_b200 as moa
from paper_0907_0792_b200.kernel import launch, plan_inner
trials = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(5)
for (m, k, n), shift in (((2048, 96, 16384), 0), ((2048, 96, 16384), 1), ((4096, 256, 4096), 0)):
    a = torch.from_numpy(rng.random(m * k + 1) * 100).cuda()[shift:shift + m * k]
    b = torch.from_numpy(rng.random(k * n) * 100).cuda()
    plan = plan_inner((m, k), (k, n))
    want = torch.empty(m * n, dtype=torch.float64, device="cuda")
    launch(plan, want, a, b, moa.MUL_ADD)
    c = torch.empty_like(want)
    fails = []
    for t in range(trials):
        c.zero_()
        launch(plan, c, a, b, moa.MUL_ADD, accumulate=True)
        bad = (c != want).nonzero().flatten()
        if bad.numel():
            r = (bad // n).cpu().numpy(); cc = (bad % n).cpu().numpy()
            fails.append((t, bad.numel(), int(r.min()), int(r.max()), int(cc.min()), int(cc.max())))
    wo = 0
    for t in range(trials // 2):
        launch(plan, c, a, b, moa.MUL_ADD)
        wo += int((c != want).sum())
    print(f"{m}x{k}x{n} shift={shift} route={moa._native.plan_kernel(0, m, k, n, 2, 0)}: "
          f"{len(fails)}/{trials} accumulate launches wrong {fails[:4]}; write-only wrong elements {wo}",
          flush=True)
