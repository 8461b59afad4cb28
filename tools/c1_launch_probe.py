"""c1 step timing: CUDA-graph replay vs a direct launch, events on the launching
stream, L2 flushed before each step (tools)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_0907_0792_b200 as moa
from paper_0907_0792_b200.kernel import launch, plan_inner
m = k = n = 256
rng = np.random.default_rng(0)
a = torch.from_numpy(rng.uniform(-1, 1, m * k)).cuda(); b = torch.from_numpy(rng.uniform(-1, 1, k * n)).cuda()
c = torch.empty(m * n, dtype=torch.float64, device="cuda")
plan = plan_inner((m, k), (k, n))
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
step = lambda: launch(plan, c, a, b, moa.MUL_ADD)
for _ in range(5): step()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
stream = torch.cuda.current_stream()
for name, fn in (("graph", g.replay), ("direct", step), ("graph", g.replay), ("direct", step)):
    ts = []
    for _ in range(50):
        flush.fill_(1.0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream); fn(); e.record(stream)
        e.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    ts.sort()
    print(f"{name}: median {ts[len(ts)//2]:.2f} us, best {ts[0]:.2f} us")
