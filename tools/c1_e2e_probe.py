"""c1 end to end through the C ABI (moa_product_rows_host) on page-locked
buffers: wall time per call (median / best of many), the host-side phase
trace of a few calls ($MOA_HOST_TRACE), and a CUPTI timeline (torch.profiler)
of the copies and kernel of one call (tools probe; not a test).
Usage: python tools/c1_e2e_probe.py [calls=400] [m k n (default 256 256 256)] [notrace]"""

import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_0907_0792_b200 import _native  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 400
m, k, n = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (256, 256, 256)
rng = np.random.default_rng(0)


def pinned(nel):
    t = torch.empty(nel, dtype=torch.float64, pin_memory=True)
    return t, t.numpy()


ta, a = pinned(m * k)
tb, b = pinned(k * n)
tc, c = pinned(m * n)
a[:] = rng.uniform(-1, 1, m * k)
b[:] = rng.uniform(-1, 1, k * n)


def call():
    _native.product_rows_host(_native.DTYPE_F64, c.ctypes.data, a.ctypes.data, b.ctypes.data,
                              m, k, n, k, n, n, 2, 0, 0, 1, 0, 0)


for _ in range(20):
    call()
ts = []
for _ in range(calls):
    t0 = time.perf_counter()
    call()
    ts.append((time.perf_counter() - t0) * 1e6)
ts.sort()
print(f"{m}x{k}x{n} e2e C ABI (direct-out limit {os.environ.get('MOA_HOST_DIRECT_OUT_BYTES', 'default')}): median {ts[len(ts) // 2]:.1f} us, best {ts[0]:.1f} us, p90 {ts[int(len(ts) * 0.9)]:.1f} us")

import paper_0907_0792_b200 as moa  # noqa: E402
from paper_0907_0792_b200 import MoaArray  # noqa: E402

for label, A, B in (("pinned MoaArrays", MoaArray._wrap((m, k), a), MoaArray._wrap((k, n), b)),
                    ("numpy MoaArrays", MoaArray((m, k), a.copy()), MoaArray((k, n), b.copy()))):
    for _ in range(20):
        moa.inner(A, B)
    ts = []
    for _ in range(calls):
        t0 = time.perf_counter()
        moa.inner(A, B)
        ts.append((time.perf_counter() - t0) * 1e6)
    ts.sort()
    print(f"{m}x{k}x{n} e2e moa.inner on {label}: median {ts[len(ts) // 2]:.1f} us, best {ts[0]:.1f} us")

if "notrace" in sys.argv:
    sys.exit(0)
os.environ["MOA_HOST_TRACE"] = "1"
for _ in range(3):
    call()
del os.environ["MOA_HOST_TRACE"]

from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        call()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[-1].time_range.start
# the last call's device activity
last = [e for e in evs if e.time_range.start >= evs[-4].time_range.start - 1]
for e in evs[-8:]:
    print(f"  {e.name[:60]:60s} start {e.time_range.start - evs[-8].time_range.start:8.1f} us "
          f"dur {e.time_range.end - e.time_range.start:7.1f} us")
