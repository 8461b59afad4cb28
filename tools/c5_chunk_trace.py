"""CUPTI trace of the k-chunked accumulate schedule of c5's first block,
repeated: which kernels run, and how long, in fast and slow repetitions."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_0907_0792_b200.kernel import KernelPlan, launch, plan_inner
from paper_0907_0792_b200.workloads import WORKLOADS
w = WORKLOADS["c5"]; a, b = w.generate(); m, k, n = w.mkn
ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
c = torch.empty(m * n, dtype=torch.float32, device="cuda")
plan = plan_inner((m, k), (k, n))
rows, step = 3072, 2048
def chunked():
    for i, k0 in enumerate(range(0, k, step)):
        part = KernelPlan(plan.mode, rows, step, n, k, n, n, plan.result_shape)
        launch(part, c, ad[k0:], bd[k0 * n:], w.ops, accumulate=i > 0)
chunked(); torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(12):
        chunked()
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA],
             key=lambda e: e.time_range.start)
rows_out = [(e.name[:70], round((e.time_range.end - e.time_range.start) / 1e3, 3)) for e in evs]
from collections import defaultdict
agg = defaultdict(list)
for nm, d in rows_out:
    agg[nm].append(d)
for nm, ds in agg.items():
    print(f"{len(ds):4d}  min {min(ds):8.3f}  max {max(ds):8.3f}  sum {sum(ds):9.2f}  {nm}")
slow = [(i, nm, d) for i, (nm, d) in enumerate(rows_out) if d > 8]
print(slow[:40])
