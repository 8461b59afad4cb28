"""c2 (outer product, 1 GiB f64 result) through the C ABI on page-locked
buffers: per-call wall time, with whatever $MOA_HOST_DIRECT_OUT_BYTES the
process got (0: kernel into device memory + D2H copy; >= 1 GiB: the outer
kernel stores straight into the page-locked result over PCIe).  Also the
same kernel timed alone into host memory vs device memory with CUDA events
(tools probe; not a test).  Usage: python tools/c2_direct_probe.py [calls=10] [trace]"""

import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_0907_0792_b200 import _native  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 10
M, N = 65536, 2048
rng = np.random.default_rng(1)
ta = torch.empty(M, dtype=torch.float64, pin_memory=True)
tb = torch.empty(N, dtype=torch.float64, pin_memory=True)
tc = torch.empty(M * N, dtype=torch.float64, pin_memory=True)
ta.numpy()[:] = rng.uniform(-1, 1, M)
tb.numpy()[:] = rng.uniform(-1, 1, N)


def call():
    _native.product_rows_host(_native.DTYPE_F64, tc.data_ptr(), ta.data_ptr(), tb.data_ptr(),
                              M, 1, N, 1, N, N, 2, 0, 0, 1, 0, 0)


for _ in range(3):
    call()
ts = []
for _ in range(calls):
    t0 = time.perf_counter()
    call()
    ts.append(time.perf_counter() - t0)
ts.sort()
lim = os.environ.get("MOA_HOST_DIRECT_OUT_BYTES", "default")
print(f"c2 C ABI (direct-out limit {lim}): median {ts[len(ts) // 2] * 1e3:.2f} ms "
      f"({M * N * 8 / ts[len(ts) // 2] / 1e9:.2f} GB/s), best {ts[0] * 1e3:.2f} ms")
if "trace" in sys.argv:
    os.environ["MOA_HOST_TRACE"] = "1"
    for _ in range(3):
        t0 = time.perf_counter()
        call()
        print(f"  call {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr)
    del os.environ["MOA_HOST_TRACE"]
want = np.multiply.outer(ta.numpy(), tb.numpy()).ravel()
assert np.array_equal(tc.numpy(), want + 0.0), "c2 result differs"

# the kernel alone: into device memory vs into the page-locked result
a_d, b_d = ta.cuda(), tb.cuda()
c_d = torch.empty(M * N, dtype=torch.float64, device="cuda")
for name, dst in (("device", c_d.data_ptr()), ("host-mapped", tc.data_ptr())):
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _native.product_rows(_native.DTYPE_F64, dst, a_d.data_ptr(), b_d.data_ptr(), M, 1, N, 1,
                             N, N, 2, 0, 0, 1, 0, torch.cuda.current_stream().cuda_stream)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    print(f"outer kernel into {name} memory: {best:.3f} ms ({M * N * 8 / best / 1e6:.1f} GB/s)")
