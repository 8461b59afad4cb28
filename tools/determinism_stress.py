"""Repeat every kernel route many times on the same data, write-only and
accumulate, and count launches whose bits differ from the first (tools; the
accumulate-mode stage race of round 1 showed up only this way)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_0907_0792_b200 as moa
from paper_0907_0792_b200 import op_pair
from paper_0907_0792_b200.kernel import launch, plan_inner, plan_outer
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(17)
cases = [  # (label, dtype, ops, (m, k, n), shift: 1 = misaligned A -> cp.async kernels)
    ("dmma TMA 64x64", np.float64, moa.MUL_ADD, (4096, 256, 4096), 0),
    ("dmma TMA 16x32", np.float64, moa.MUL_ADD, (256, 1024, 256), 0),
    ("dmma cp.async", np.float64, moa.MUL_ADD, (2048, 255, 2048), 1),
    ("tropical f32 TMA 128x128", np.float32, op_pair("add", "min"), (2048, 512, 4096), 0),
    ("tropical f32 TMA 64x128", np.float32, op_pair("add", "min"), (1000, 512, 1024), 0),
    ("tropical f32 FMNMX3 128x128", np.float32, op_pair("subtract", "max"), (2048, 512, 4096), 0),
    ("tropical f32 cp.async", np.float32, op_pair("subtract", "max"), (1024, 511, 1024), 1),
    ("int32 DPX TMA 128x128", np.int32, op_pair("add", "min"), (2048, 512, 4096), 0),
    ("int32 DPX TMA 64x128", np.int32, op_pair("add", "max"), (1000, 512, 1024), 0),
    ("f64 exact (add,min)", np.float64, op_pair("add", "min"), (1024, 256, 1024), 0),
    ("f32 max-times", np.float32, op_pair("multiply", "max"), (2048, 256, 2048), 0),
    ("f32 (divide,max) exact", np.float32, op_pair("divide", "max"), (1024, 256, 1024), 0),
    ("f64 (max,multiply)", np.float64, op_pair("max", "multiply"), (1024, 256, 1024), 0),
    ("f32 (min,min) exact", np.float32, op_pair("min", "min"), (1024, 256, 1024), 0),
    ("int32 (multiply,add)", np.int32, op_pair("multiply", "add"), (1024, 256, 1024), 0),
    ("int32 DPX cp.async", np.int32, op_pair("subtract", "max"), (1024, 255, 1024), 1),
    ("int64 (add,min)", np.int64, op_pair("add", "min"), (1024, 256, 1024), 0),
    ("f64 (divide,add)", np.float64, op_pair("divide", "add"), (1024, 256, 1024), 0),
]
torch_dt = {np.float64: torch.float64, np.float32: torch.float32, np.int32: torch.int32,
            np.int64: torch.int64}
for label, dt, ops, (m, k, n), shift in cases:
    if np.dtype(dt).kind == "i":
        a = rng.integers(-1000, 1000, m * k + 1).astype(dt); b = rng.integers(-1000, 1000, k * n).astype(dt)
    else:
        a = (rng.random(m * k + 1) * 100).astype(dt); b = (rng.random(k * n) * 100).astype(dt)
    ad = torch.from_numpy(a).cuda()[shift:shift + m * k]; bd = torch.from_numpy(b).cuda()
    plan = plan_inner((m, k), (k, n))
    first = torch.empty(m * n, dtype=torch_dt[dt], device="cuda")
    launch(plan, first, ad, bd, ops)
    bad_w = bad_a = 0
    c = torch.empty_like(first)
    for r in range(reps):
        launch(plan, c, ad, bd, ops)
        isint = np.dtype(dt).kind == "i"
        bad_w += int(not torch.equal(c if isint else c.view(torch.uint8),
                                     first if isint else first.view(torch.uint8)))
        if isint:
            info = np.iinfo(dt)
            c.fill_({"add": 0, "multiply": 1, "min": int(info.max), "max": int(info.min)}[ops.reduce_name])
        else:
            c.fill_(ops.reduce_identity)
        launch(plan, c, ad, bd, ops, accumulate=True)
        bad_a += int(not torch.equal(c if isint else c.view(torch.uint8),
                                     first if isint else first.view(torch.uint8)))
    print(f"{label:24s} {m}x{k}x{n}: {reps} write-only launches differing {bad_w}, "
          f"{reps} accumulate launches differing {bad_a}", flush=True)
x = torch.from_numpy(rng.random(65536)).cuda(); y = torch.from_numpy(rng.random(2048)).cuda()
o1 = torch.empty(65536 * 2048, dtype=torch.float64, device="cuda")
launch(plan_outer((65536,), (2048,)), o1, x, y, moa.MUL_ADD)
o2 = torch.empty_like(o1); bad = 0
for r in range(reps):
    launch(plan_outer((65536,), (2048,)), o2, x, y, moa.MUL_ADD); bad += int(not torch.equal(o1, o2))
print(f"{'outer':24s} 65536x2048: {reps} launches differing {bad}")
