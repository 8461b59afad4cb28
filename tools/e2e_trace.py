"""Timeline of one end-to-end (host buffers in, host result out) product of a
BASELINE config through the public API, from a torch.profiler (CUPTI) trace:
per-stream busy time of H2D copies, kernels and D2H copies, and the span
(tools probe; not a test).  Usage: python tools/e2e_trace.py c5 [out.json] [pageable]
("pageable": plain numpy inputs and a prefaulted numpy result through the C
ABI, i.e. the staged path)"""

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_0907_0792_b200 as moa  # noqa: E402
from paper_0907_0792_b200 import MoaArray  # noqa: E402
from paper_0907_0792_b200.workloads import WORKLOADS  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "c5"
w = WORKLOADS[key]
a, b = w.generate()


def pinned(x):
    t = torch.empty(x.size, dtype=torch.from_numpy(x[:1]).dtype, pin_memory=True)
    t.numpy()[:] = x
    return t


pageable = len(sys.argv) > 3 and sys.argv[3] == "pageable"
if pageable:
    from paper_0907_0792_b200.kernel import launch_host, plan_inner, plan_outer
    plan = (plan_inner if w.mode == "inner" else plan_outer)(w.shape_a, w.shape_b)
    res = np.zeros(w.mkn[0] * w.mkn[2], dtype=a.dtype)

    def fn(_a, _b, ops):
        launch_host(plan, res, a, b, ops)
        return res
    A = B = None
else:
    ap, bp = pinned(a), pinned(b)
    A = MoaArray._wrap(w.shape_a, ap.numpy())
    B = MoaArray._wrap(w.shape_b, bp.numpy())
    fn = moa.inner if w.mode == "inner" else moa.outer
out = None
for _ in range(2):
    out = None
    out = fn(A, B, w.ops)
torch.cuda.synchronize()
out = None
t0 = time.perf_counter()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                        torch.profiler.ProfilerActivity.CPU]) as prof:
    out = fn(A, B, w.ops)
    torch.cuda.synchronize()
wall = time.perf_counter() - t0
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
rows = []
for e in evs:
    rows.append({"name": e.name[:80], "start_us": e.time_range.start, "end_us": e.time_range.end})
rows.sort(key=lambda r: r["start_us"])
t_first = rows[0]["start_us"] if rows else 0
summary = {"workload": key, "wall_ms_under_profiler": round(wall * 1e3, 2), "events": []}
for r in rows:
    summary["events"].append({"name": r["name"], "start_ms": round((r["start_us"] - t_first) / 1e3, 3),
                              "dur_ms": round((r["end_us"] - r["start_us"]) / 1e3, 3)})
span = (max(r["end_us"] for r in rows) - t_first) / 1e3 if rows else 0
summary["device_span_ms"] = round(span, 2)
txt = json.dumps(summary, indent=1)
if len(sys.argv) > 2:
    Path(sys.argv[2]).write_text(txt)
for ev in summary["events"]:
    print(f'{ev["start_ms"]:10.3f} {ev["dur_ms"]:9.3f}  {ev["name"]}')
print("span ms", summary["device_span_ms"], "wall ms", summary["wall_ms_under_profiler"])
