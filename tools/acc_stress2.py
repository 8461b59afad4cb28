"""Characterise accumulate-mode corruption: for a failing launch, relate each
wrong element's error to per-slab partial sums (tools)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_0907_0792_b200 as moa
from paper_0907_0792_b200.kernel import launch, plan_inner
rng = np.random.default_rng(5)
m, k, n = 4096, 256, 4096
ah = rng.random(m * k) * 100; bh = rng.random(k * n) * 100
a = torch.from_numpy(ah).cuda(); b = torch.from_numpy(bh).cuda()
A = ah.reshape(m, k); B = bh.reshape(k, n)
plan = plan_inner((m, k), (k, n))
want = torch.empty(m * n, dtype=torch.float64, device="cuda")
launch(plan, want, a, b, moa.MUL_ADD)
wantn = want.cpu().numpy().reshape(m, n)
c = torch.empty_like(want)
found = 0
for t in range(int(sys.argv[1]) if len(sys.argv) > 1 else 400):
    c.zero_()
    launch(plan, c, a, b, moa.MUL_ADD, accumulate=True)
    bad = (c != want).nonzero().flatten()
    if not bad.numel():
        continue
    found += 1
    got = c.cpu().numpy().reshape(m, n)
    idx = bad.cpu().numpy()
    rows, cols = idx // n, idx % n
    print(f"trial {t}: {idx.size} wrong, rows {rows.min()}-{rows.max()} cols {cols.min()}-{cols.max()}")
    for (r, cc) in list(zip(rows, cols))[:6]:
        d = got[r, cc] - wantn[r, cc]
        S = np.array([A[r, j*16:(j+1)*16] @ B[j*16:(j+1)*16, cc] for j in range(16)])
        Sk = np.array([A[r, j] * B[j, cc] for j in range(k)])
        print(f"  ({r},{cc}) diff {d:.4f}; closest -slab {np.argmin(np.abs(d + S))} ({(d + S)[np.argmin(np.abs(d + S))]:.3g}); "
              f"closest +slab {np.argmin(np.abs(d - S))} ({(d - S)[np.argmin(np.abs(d - S))]:.3g}); "
              f"closest -kterm {np.argmin(np.abs(d + Sk))} ({(d + Sk)[np.argmin(np.abs(d + Sk))]:.3g}); "
              f"got/want {got[r, cc] / wantn[r, cc]:.6f}")
    # fraction of the warp tile and the pattern of wrong (row, col) inside it
    r0 = rows.min() // 32 * 32; c0 = cols.min() // 32 * 32
    mask = np.zeros((32, 32), int)
    for r, cc in zip(rows, cols):
        if r0 <= r < r0 + 32 and c0 <= cc < c0 + 32:
            mask[r - r0, cc - c0] = 1
    print("  rows with errors:", np.nonzero(mask.any(1))[0].tolist())
    print("  cols with errors:", np.nonzero(mask.any(0))[0].tolist())
    if found >= 3:
        break
print("trials run", t + 1, "failing", found)
