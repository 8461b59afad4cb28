"""Device -> page-locked host copy rate of a 1 GiB result (the c2 end-to-end
bound): torch pinned (cudaHostAlloc) vs moa_host_alloc (registered huge
pages) destinations, split over 1..8 copy queues, as 1..64 row chunks
issued round-robin; plus the c2 C-ABI call itself under a CUPTI timeline
(tools probe; not a test).  Usage: python tools/d2h_probe.py"""

import ctypes
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_0907_0792_b200 import _native  # noqa: E402

NB = 1 << 30
dev = torch.empty(NB // 8, dtype=torch.float64, device="cuda")
dev.uniform_()
pinned = torch.empty(NB // 8, dtype=torch.float64, pin_memory=True)
ptr = _native.host_alloc(NB)
reg = torch.from_numpy(np.frombuffer((ctypes.c_char * NB).from_address(ptr), dtype=np.float64))
streams = [torch.cuda.Stream() for _ in range(8)]


def copy(dst, queues, chunks):
    n = dst.numel()
    per = -(-n // chunks)
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    for i in range(chunks):
        s = streams[i % queues]
        s.wait_event(ev)
        with torch.cuda.stream(s):
            dst[i * per:(i + 1) * per].copy_(dev[i * per:(i + 1) * per], non_blocking=True)
    for s in streams[:queues]:
        s.synchronize()


res = {}
for name, dst in (("cudaHostAlloc", pinned), ("registered_hugepages", reg)):
    for queues, chunks in ((1, 1), (2, 2), (4, 4), (8, 8), (4, 16), (4, 64), (2, 16), (1, 16)):
        copy(dst, queues, chunks)
        best = 1e9
        for _ in range(5):
            t0 = time.perf_counter()
            copy(dst, queues, chunks)
            best = min(best, time.perf_counter() - t0)
        res[f"{name}_q{queues}_c{chunks}_GBs"] = round(NB / best / 1e9, 2)
        print(name, queues, chunks, res[f"{name}_q{queues}_c{chunks}_GBs"], flush=True)
print(res)
