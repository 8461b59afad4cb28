"""Repeated C-ABI calls of one config on page-locked buffers: per-call wall
times (spotting outliers), for the executor's memory-pool settings."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_0907_0792_b200.kernel import launch_host, plan_inner, plan_outer
from paper_0907_0792_b200.workloads import WORKLOADS
key = sys.argv[1]; reps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
w = WORKLOADS[key]; a, b = w.generate(); m, k, n = w.mkn
plan = (plan_inner if w.mode == "inner" else plan_outer)(w.shape_a, w.shape_b)
def pinned(x):
    t = torch.empty(x.size, dtype=torch.from_numpy(x[:1]).dtype, pin_memory=True).numpy(); t[:] = x; return t
pa, pb = pinned(a), pinned(b)
res = torch.empty(m * n, dtype=torch.from_numpy(a[:1]).dtype, pin_memory=True).numpy()
ts = []
for _ in range(reps):
    t0 = time.perf_counter(); launch_host(plan, res, pa, pb, w.ops); ts.append(time.perf_counter() - t0)
print(json.dumps({"cfg": key, "ms": [round(t * 1e3, 1) for t in ts]}))
