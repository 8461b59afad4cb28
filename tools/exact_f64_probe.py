"""The exact (separate multiply and add, k ascending) float64 (x,+) route —
the drop-in module's default — at 4096^3 and c4's 16384^3: CUDA-event time
and TFLOP/s against the FP64 pipe bound for two FP64 instructions per pair
(148 SMs x 64 lanes x 1.965 GHz / 2 = 9.3 T pairs/s = 18.6 TFLOP/s)
(tools probe; not a test).  Usage: python tools/exact_f64_probe.py [n ...]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0907_0792_b200 as moa  # noqa: E402
from paper_0907_0792_b200.kernel import launch, plan_inner  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or [4096, 16384]:
    a = torch.rand(n * n, dtype=torch.float64, device="cuda") * 2 - 1
    b = torch.rand(n * n, dtype=torch.float64, device="cuda") * 2 - 1
    c = torch.empty(n * n, dtype=torch.float64, device="cuda")
    plan = plan_inner((n, n), (n, n))
    launch(plan, c, a, b, moa.MUL_ADD, exact=True)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3 if n <= 8192 else 1):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        launch(plan, c, a, b, moa.MUL_ADD, exact=True)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    tf = 2.0 * n ** 3 / best / 1e9
    print(f"exact f64 (x,+) {n}^3: {best:.2f} ms, {tf:.2f} TFLOP/s, {tf / 18.6:.2f} of the "
          f"two-FP64-instruction bound", flush=True)
    del a, b, c
