"""One c4 drop-in call (product_rows_overwrite into np.empty) with
$MOA_HOST_TRACE on: the executor's host-side phases and each staged
transfer's pack/wait/prefault times (tools probe; not a test)."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from integration import moaprod_b200kernel as kb  # noqa: E402
from paper_0907_0792_b200.workloads import WORKLOADS  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "c4"
w = WORKLOADS[key]
a, b = (np.ascontiguousarray(x, dtype=np.float64).ravel() for x in w.generate())
m, k, n = w.mkn
c, r = w.ops.codes()
res = np.empty(m * n)
kb.product_rows_overwrite(res, a, b, m, k, n, k, n, n, c, r, 0, 1)
del res
os.environ["MOA_HOST_TRACE"] = "1"
for fresh in (True, False):
    res = np.empty(m * n)
    if not fresh:
        res[:] = 0.0
    t0 = time.perf_counter()
    kb.product_rows_overwrite(res, a, b, m, k, n, k, n, n, c, r, 0, 1)
    print(f"{key} overwrite, {'fresh' if fresh else 'pre-touched'} res: {(time.perf_counter() - t0) * 1e3:.1f} ms",
          file=sys.stderr, flush=True)
