"""c4-/c5-sized end-to-end calls through the C ABI on page-locked buffers
(float64 (x,+) 16384^3 and float32 (add, min) 16384^3 with c5's data), wall
time per call, under whatever $MOA_HOST_MID_BLOCKS the process got (tools
probe; not a test).  Usage: python tools/e2e_blocks_probe.py [calls=3] [c4|c5]"""

import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_0907_0792_b200 import _native  # noqa: E402
from paper_0907_0792_b200.workloads import WORKLOADS  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 3
which = sys.argv[2:] or ["c4", "c5"]
for key in which:
    w = WORKLOADS[key]
    a, b = w.generate()
    m, k, n = w.mkn
    dt = torch.from_numpy(a[:1]).dtype
    ta = torch.empty(a.size, dtype=dt, pin_memory=True)
    tb = torch.empty(b.size, dtype=dt, pin_memory=True)
    tc = torch.empty(m * n, dtype=dt, pin_memory=True)
    ta.numpy()[:] = a.ravel()
    tb.numpy()[:] = b.ravel()
    code = _native.DTYPE_F64 if dt == torch.float64 else _native.DTYPE_F32
    c, r = w.ops.codes()

    def call():
        _native.product_rows_host(code, tc.data_ptr(), ta.data_ptr(), tb.data_ptr(), m, k, n, k,
                                  n, n, c, r, 0, 1, 0, 0)

    call()
    ts = []
    for _ in range(calls):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    print(f"{key} C ABI mid_blocks={os.environ.get('MOA_HOST_MID_BLOCKS', 'default')}: "
          f"best {min(ts) * 1e3:.1f} ms, all {[round(t * 1e3, 1) for t in ts]}", flush=True)
    del ta, tb, tc
