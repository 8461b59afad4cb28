"""Where does the end-to-end time go?  Host<->device copy rates on this box and
the phases of one public-API outer product (tools probe; not a test)."""

import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

res = {}
n = 1 << 27  # 1 GiB of float64
dev = torch.device("cuda")
d = torch.empty(n, dtype=torch.float64, device=dev)
d.fill_(1.0)


def t_events(fn, reps=3):
    best = 1e30
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


t0 = time.perf_counter()
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
res["pin_alloc_1GiB_s"] = time.perf_counter() - t0
res["d2h_pinned_GBs"] = n * 8 / t_events(lambda: h.copy_(d, non_blocking=True)) / 1e6
res["h2d_pinned_GBs"] = n * 8 / t_events(lambda: d.copy_(h, non_blocking=True)) / 1e6
pg = torch.empty(n, dtype=torch.float64)  # pageable
pg.fill_(0.0)
res["d2h_pageable_GBs"] = n * 8 / t_events(lambda: pg.copy_(d)) / 1e6

for ns in (2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = n // ns

    def multi():
        cur = torch.cuda.current_stream()
        for i, s in enumerate(streams):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                h[i * chunk:(i + 1) * chunk].copy_(d[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
    res[f"d2h_pinned_{ns}streams_GBs"] = n * 8 / t_events(multi) / 1e6

# bidirectional
s2 = torch.cuda.Stream()
h2 = torch.empty(n // 2, dtype=torch.float64, pin_memory=True)


def bidir():
    cur = torch.cuda.current_stream()
    s2.wait_stream(cur)
    with torch.cuda.stream(s2):
        d[: n // 2].copy_(h2, non_blocking=True)
    h[n // 2:].copy_(d[n // 2:], non_blocking=True)
    cur.wait_stream(s2)


res["bidir_half_each_GBs_total"] = n * 8 / t_events(bidir) / 1e6

# the public API, phase by phase
import paper_0907_0792_b200 as moa  # noqa: E402
from paper_0907_0792_b200.workloads import WORKLOADS  # noqa: E402

w = WORKLOADS["c2"]
a, b = w.generate()
ap = torch.empty(a.size, dtype=torch.float64, pin_memory=True)
ap.numpy()[:] = a
bp = torch.empty(b.size, dtype=torch.float64, pin_memory=True)
bp.numpy()[:] = b
A = moa.MoaArray._wrap(w.shape_a, ap.numpy())
B = moa.MoaArray._wrap(w.shape_b, bp.numpy())
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = moa.outer(A, B)
    res[f"api_outer_s_{i}"] = time.perf_counter() - t0
    del out
print(json.dumps({k: round(v, 4) for k, v in res.items()}))
