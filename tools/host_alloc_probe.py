"""Timing of the host result-block cache (kernel.host_empty -> moa_host_alloc)
under the allocation pattern of repeated products (tools probe)."""
import gc, json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_0907_0792_b200.kernel import host_empty

out = {}
for label, nbytes in (("1GiB", 1 << 30), ("2GiB", 2 << 30)):
    ts = []
    x = None
    for _ in range(6):
        x = None
        t0 = time.perf_counter()
        x = host_empty(nbytes // 8, np.float64)
        ts.append(round((time.perf_counter() - t0) * 1e3, 2))
    out[label + "_alloc_ms"] = ts
    x = None
    gc.collect()
print(json.dumps(out))
