"""float32 pairs folded in float64 through the production route at 4096^3 —
(x,+), (+,+), (x,min), (min,+), (x,x) — CUDA-event time per launch (tools
probe; not a test).  Round 2 used it with $MOA_F32W to compare a
register-staged float64-tile kernel that was then dropped
(profiles/r02_tune_semiring_kunroll.jsonl); the variable no longer selects
anything.  Usage: python tools/f32w_probe.py [n]"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_0907_0792_b200 as moa  # noqa: E402
from paper_0907_0792_b200.kernel import launch, plan_inner  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
a = torch.rand(n * n, device="cuda") * 4 - 1
b = torch.rand(n * n, device="cuda") * 4 - 1
c = torch.empty(n * n, device="cuda")
plan = plan_inner((n, n), (n, n))
for comb, red in (("multiply", "add"), ("add", "add"), ("multiply", "min"), ("min", "add"),
                  ("multiply", "multiply")):
    ops = moa.op_pair(comb, red)
    launch(plan, c, a, b, ops)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        launch(plan, c, a, b, ops)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    h = hash(c.cpu().numpy().tobytes())
    print(f"MOA_F32W={os.environ.get('MOA_F32W', '1')} f32 ({comb},{red}) {n}^3: {best:.3f} ms "
          f"{n ** 3 / best / 1e9:.0f} G pairs/s bits {h & 0xffffffff:08x}", flush=True)
