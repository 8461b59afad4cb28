"""Stress the native host executor's streamed schedule: repeated
moa_product_rows_host calls on >= 1 GiB results (pinned and pageable, write-only
and accumulate, (x,+) f64 and (add,min) f32, equal and ramped k-chunks) and on a
128 MiB single-block result (row parts), each compared bitwise with one device
launch (tools)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_0907_0792_b200 as moa
from paper_0907_0792_b200 import op_pair
from paper_0907_0792_b200.kernel import launch, launch_host, plan_inner
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
rng = np.random.default_rng(9)
for dt, ops, (m, k, n) in ((np.float64, moa.MUL_ADD, (8192, 200, 16384)),
                          (np.float32, op_pair("add", "min"), (16384, 200, 16384)),
                          (np.float64, moa.MUL_ADD, (8192, 1100, 16384)),      # ramped k-chunks
                          (np.float32, op_pair("add", "min"), (16384, 1100, 16384)),
                          (np.float64, op_pair("subtract", "max"), (4096, 512, 4096))):  # row parts
    a = (rng.random(m * k) * 100).astype(dt); b = (rng.random(k * n) * 100).astype(dt)
    plan = plan_inner((m, k), (k, n))
    want = torch.empty(m * n, dtype=torch.from_numpy(a[:1]).dtype, device="cuda")
    launch(plan, want, torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), ops)
    want = want.cpu().numpy()
    pinned = torch.empty(m * n, dtype=torch.from_numpy(a[:1]).dtype, pin_memory=True).numpy()
    pageable = np.empty(m * n, dtype=dt)
    bad = []
    for r in range(reps):
        for name, res in (("pinned", pinned), ("pageable", pageable)):
            for acc in (False, True):
                res[:] = ops.reduce_identity if acc else 7
                launch_host(plan, res, a, b, ops, accumulate=acc)
                nb = int(np.count_nonzero(res.view(np.uint8) != want.view(np.uint8)))
                if nb:
                    bad.append((r, name, acc, nb))
    print(np.dtype(dt).name, ops, f"{reps * 4} calls, wrong: {bad}", flush=True)
