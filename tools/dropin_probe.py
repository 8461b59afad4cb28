"""The reference's own call pattern through the drop-in module
(integration/moaprod_b200kernel.py): what a moaprod user gets with the B200
backend registered.  Per call, as the reference's _Runner does
(kernel.py:138-170): res = np.full(M*N, identity) (pageable), then one
product_rows(res, a, b, ...) over all rows (execute_sequential) with pageable
numpy A and B.  Also the runner branch INTEGRATION.md proposes
(product_rows_overwrite into np.empty, no prefill), and the reference's own
compiled loop (oracle/_ref) on the same buffers for comparison (16 threads,
rows k::W, as execute_parallel does).  Tools probe; not a test.
Usage: python tools/dropin_probe.py [c2 c4 ...]"""

import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from integration import moaprod_b200kernel as kb  # noqa: E402
from paper_0907_0792_b200.workloads import WORKLOADS  # noqa: E402

keys = sys.argv[1:] or ["c2", "c4"]
out = {}
for key in keys:
    w = WORKLOADS[key]
    a, b = w.generate()
    a = np.ascontiguousarray(a, dtype=np.float64).ravel()
    b = np.ascontiguousarray(b, dtype=np.float64).ravel()
    m, k, n = w.mkn
    c, r = w.ops.codes()
    ident = w.ops.reduce_identity
    args = (a, b, m, k, n, k, n, n, c, r, 0, 1)
    reps = 3 if key in ("c4", "c5") else 5

    def prefill_accumulate():
        res = np.full(m * n, ident)
        kb.product_rows(res, *args)
        return res

    def overwrite():
        res = np.empty(m * n)
        kb.product_rows_overwrite(res, *args)
        return res

    rec = {}
    for name, fn in (("prefill_accumulate", prefill_accumulate), ("overwrite", overwrite)):
        fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            res = fn()
            ts.append(time.perf_counter() - t0)
            del res
        rec[name + "_ms"] = round(min(ts) * 1e3, 1)
    if key in ("c1", "c2", "c3"):
        try:
            import oracle
            ck = oracle.ref_kernel()
            W = oracle.host_cores()

            def ref():
                res = np.full(m * n, ident)
                with ThreadPoolExecutor(max_workers=W) as pool:
                    for f in [pool.submit(ck.product_rows, res, a, b, m, k, n, k, n, n, c, r, j, W)
                              for j in range(W)]:
                        f.result()
                return res
            ts = []
            for _ in range(3):
                t0 = time.perf_counter()
                ref()
                ts.append(time.perf_counter() - t0)
            rec["reference_compiled_loop_ms"] = round(min(ts) * 1e3, 1)
            rec["reference_threads"] = W
        except Exception as exc:  # oracle/_ref not built on this box
            rec["reference_compiled_loop_ms"] = f"unavailable: {exc}"
    out[key] = rec
    print(key, rec, flush=True)
print(json.dumps(out))
