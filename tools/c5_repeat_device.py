"""Repeated device-resident c5 launches (write-only, and k-chunked with
accumulate like the host executor's first block), event-timed per launch:
does the tropical route's time vary from launch to launch?  (tools probe)"""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_0907_0792_b200 as moa
from paper_0907_0792_b200.kernel import KernelPlan, launch, plan_inner
from paper_0907_0792_b200.workloads import WORKLOADS
w = WORKLOADS["c5"]; a, b = w.generate(); m, k, n = w.mkn
ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
c = torch.empty(m * n, dtype=torch.float32, device="cuda")
plan = plan_inner((m, k), (k, n))
def timed(fn):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); fn(); e.record(); e.synchronize(); return round(s.elapsed_time(e), 1)
out = {"write_only": [timed(lambda: launch(plan, c, ad, bd, w.ops)) for _ in range(10)]}
rows = 3072
sub = KernelPlan(plan.mode, rows, k, n, k, n, n, plan.result_shape)
def chunked():
    step = 2048
    for i, k0 in enumerate(range(0, k, step)):
        part = KernelPlan(plan.mode, rows, step, n, k, n, n, plan.result_shape)
        launch(part, c, ad[k0:], bd[k0 * n:], w.ops, accumulate=i > 0)
out["block0_chunked_acc"] = [timed(chunked) for _ in range(10)]
out["block0_one_pass"] = [timed(lambda: launch(sub, c, ad, bd, w.ops)) for _ in range(5)]
print(json.dumps(out))
