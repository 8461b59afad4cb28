"""Benchmark: BASELINE.json's metric on B200 (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Workload (``config.workload``): BASELINE.json configs[1] by default — the
generalized outer product rho<32 16 16 8> (x) rho<16 16 8> in float64, 1.07 GB of
result, metric "outer-product GB/s" (algorithmic bytes 8*(M*N + M + N) per unit).
``--config c1|c3|c4`` measure the (+,x) inner products in GFLOP/s, ``c5`` the
tropical product in G pairs/s.  At N=1 the default run also measures c1, c3, c4
and c5 device-resident (key "inner"), so one line carries both halves of the
metric ("inner-product GFLOP/s & outer-product GB/s ... % of roofline"); at
N>1 "inner" holds c4 and c5 with their result rows sharded over the ranks
(BASELINE configs 4-5: B broadcast inside every step, strong scaling).

A step is one pass of the product over one unit of synthetic input:
* ``value``: inputs resident in HBM; per step, rank 0's B is broadcast (NCCL,
  N>1 only) and the kernel writes the rank's result block.  L2 is flushed
  between timed steps (a 256 MiB write, outside the events); each step is
  bracketed by CUDA events on the launching stream; sum over steps, max over
  ranks.
* ``e2e``: the reference-facing C ABI with HOST buffers — one
  ``moa_product_rows_host`` call per step on page-locked A, B and result (H2D
  of A and B, the product, D2H of the whole result, all inside the clock) at
  N=1; ``distributed.sharded_product_host`` at N>1.  ``e2e_api`` is the same
  through the public Python API (``moa.outer``/``moa.inner`` on pinned host
  MoaArrays).
Multi-GPU (torchrun): the outer product scales weakly (each rank owns one
unit of 65,536 result rows; B broadcast from rank 0), the large inner products
strongly (result rows of one 16384^3 product split across ranks).

``--impl reference`` times the reference's own compiled hot loop
(oracle/_ref, built from /root/reference by oracle/Makefile; the C port of it
if absent) on the host cores, driven like its execute_parallel.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

from paper_0907_0792_b200.workloads import WORKLOADS  # noqa: E402

METRIC = {"c2": ("outer-product GB/s", "GB/s"),
          "c1": ("inner-product GFLOP/s", "GFLOP/s"),
          "c3": ("inner-product GFLOP/s", "GFLOP/s"),
          "c4": ("inner-product GFLOP/s", "GFLOP/s"),
          "c5": ("tropical inner-product G pairs/s", "Gpairs/s")}
SCALING = {"c2": "weak", "c1": "weak", "c3": "weak", "c4": "strong", "c5": "strong"}
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback (used only if MEASURED_PEAKS.json is absent)


# ---------------------------------------------------------------------------- peaks
def hbm_peak() -> tuple[float, str]:
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    return FALLBACK_HBM_GBS, "B200_PROFILING.md fallback"


def microbench_peaks() -> dict:
    p = REPO / "profiles" / "r01_peaks_microbench.json"
    return json.loads(p.read_text()) if p.exists() else {}


def fp64_peak() -> tuple[float, str]:
    mb = microbench_peaks()
    vals = [v for k, v in mb.items() if k.startswith("dmma_")]
    if vals:
        return max(vals), "measured DMMA mma.sync f64 microbenchmark (profiles/r01_peaks_microbench.json)"
    return 36.96, "measured DMMA microbenchmark (r01)"


def minplus_peak() -> tuple[float, str]:
    """Best measured (add, min) pair rate on the ALU/FMA pipes, G pairs/s.

    profiles/r01_minplus_mix2.json holds warp-instructions per clock per SM for
    FADD2 + FMNMX3 and FADD2 + VIMNMX3 units (64 pairs each) at 1965 MHz."""
    p = REPO / "profiles" / "r01_minplus_mix2.json"
    if p.exists():
        mix = json.loads(p.read_text())
        units = max(mix.get("fadd2_fmnmx3_pairs_winstr_per_clk_sm", 0.0),
                    mix.get("fadd2_vimnmx3_units_winstr_per_clk_sm", 0.0))
        return (units * 64 * 148 * 1.965e9 / 1e9,
                "measured FADD2+VIMNMX3 / FADD2+FMNMX3 instruction-mix microbenchmark "
                "(profiles/r01_minplus_mix2.json), best mix, 1965 MHz")
    return 24470.0, "measured FADD2+VIMNMX3 microbenchmark (r01)"


def ncu_traffic(workload: str):
    p = REPO / "profiles" / "ncu_traffic.json"
    if p.exists():
        return json.loads(p.read_text()).get(workload)
    return None


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) == 7:
                try:
                    rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:]))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        loaded = [r for r in rows if r[2] > 300.0] or rows
        reasons = sorted({names[i] for r in loaded for i, v in enumerate(r[3]) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in loaded),
                "sm_max_mhz": max(r[1] for r in rows), "reasons": reasons,
                "samples": len(loaded), "power_w_max": max(r[2] for r in rows)}


# ---------------------------------------------------------------------------- helpers
def dist_env() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def pinned_copy(x: np.ndarray):
    import torch
    t = torch.empty(x.size, dtype=torch.from_numpy(x[:1]).dtype, pin_memory=True)
    t.numpy()[:] = x
    return t


class L2Flusher:
    def __init__(self, device):
        import torch
        self.buf = torch.empty(256 * 2**20 // 4, dtype=torch.float32, device=device)

    def __call__(self):
        self.buf.fill_(1.0)


def plan_for(w):
    from paper_0907_0792_b200 import plan_inner, plan_outer
    return (plan_inner if w.mode == "inner" else plan_outer)(w.shape_a, w.shape_b)


def job_plan(w, world: int):
    """The whole job's plan: strong scaling splits one unit's rows over the
    ranks; weak scaling stacks one unit per rank (world * M result rows, each
    rank's block being exactly one unit, distributed.row_block)."""
    from paper_0907_0792_b200.distributed import block_plan
    plan = plan_for(w)
    if SCALING[w.key] == "strong" or world == 1:
        return plan
    return block_plan(plan, 0, plan.noproc * world)


def unit_amount(w, rows: int) -> float:
    """Algorithmic work of ``rows`` result rows in the metric's unit numerator."""
    m, k, n = w.mkn
    isz = np.dtype(w.dtype).itemsize
    if w.key == "c2":
        return isz * (rows * n + rows * k + (k * n))   # bytes: C rows + A rows + B
    if w.key == "c5":
        return rows * k * n                              # (add,min) pairs
    return 2.0 * rows * k * n                            # flops


def to_unit(w, amount: float, seconds: float) -> float:
    return amount / seconds / 1e9  # GB/s, GFLOP/s or G pairs/s


# ---------------------------------------------------------------------------- device leg
def measure_device(w, rows_range, a_host, b_host, steps, warmup, device, world, rank, group=None):
    """value leg + kernel-only timing for one workload (inputs resident in HBM)."""
    import torch
    import torch.distributed as dist

    from paper_0907_0792_b200 import _native
    from paper_0907_0792_b200.distributed import block_plan
    from paper_0907_0792_b200.kernel import launch

    plan = plan_for(w)
    r0, r1 = rows_range
    m, k, n = w.mkn
    tdt = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
           np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64}[np.dtype(w.dtype)]
    lda = plan.lstride
    a_dev = torch.from_numpy(np.ascontiguousarray(a_host[r0 * lda:r1 * lda])).to(device)
    b_dev = torch.from_numpy(b_host).to(device) if rank == 0 else \
        torch.empty(b_host.size, dtype=tdt, device=device)
    c_dev = torch.empty((r1 - r0) * n, dtype=tdt, device=device)
    sub = block_plan(plan, r0, r1)
    flush = L2Flusher(device)
    stream = torch.cuda.current_stream(device)

    # Strong-scaled jobs (c4/c5) broadcast B inside every step.  A weak-scaled
    # job (c2) has B resident on every rank when the clock starts (broadcast
    # once, below), so its step is the rank's own product with no collective.
    bcast_in_step = world > 1 and SCALING[w.key] == "strong"
    if bcast_in_step:
        from paper_0907_0792_b200.distributed import sharded_product
        gplan = job_plan(w, world)
        # strong-scaled jobs pipeline B's broadcast in k-chunks where the fold
        # replays exactly under chunked accumulation ((x,+) f64, (add, min))
        from paper_0907_0792_b200.distributed import bcast_chunk_align
        chunks = 8 if bcast_chunk_align(w.ops, tdt) is not None else 1

        def step():
            sharded_product(gplan, a_dev, b_dev if rank == 0 else None, w.ops, group=group,
                            out=c_dev, bcast_chunks=chunks)
    else:
        def step():
            launch(sub, c_dev, a_dev, b_dev, w.ops)

    if world > 1:
        # B on every rank (the kernel-only leg below and weak-scaled steps read b_dev)
        dist.broadcast(b_dev, src=0, group=group)
        dist.barrier()
    for _ in range(warmup):
        step()
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(device)
    # Steps without a collective are captured once into a CUDA graph, so each
    # timed step is one graph launch and the events bracket device work only
    # (no host-side launch gaps).  Steps with the broadcast inside stay eager
    # (it may run over gloo, which cannot be captured).
    # Under torchrun the NCCL watchdog thread keeps querying events, so the
    # capture is thread-local there; should it still fail, the steps stay eager.
    graph, per_step_launches = None, None
    if not bcast_in_step:
        l0 = _native.launch_count()
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, capture_error_mode="thread_local" if world > 1
                                  else "global"):
                step()
            per_step_launches = _native.launch_count() - l0
            graph.replay()
            torch.cuda.synchronize(device)
        except RuntimeError as exc:  # pragma: no cover - depends on the driver/NCCL
            print(f"[bench] rank {rank}: CUDA graph capture failed ({exc}); eager steps",
                  file=sys.stderr)
            graph, per_step_launches = None, None
            torch.cuda.synchronize(device)
    run_step = graph.replay if graph is not None else step
    launches0 = _native.launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    with ClockSampler(device.index) as clocks:
        for s, e in evs:
            flush()
            s.record(stream)
            run_step()
            e.record(stream)
        torch.cuda.synchronize(device)
        launches = (per_step_launches * steps if graph is not None
                    else _native.launch_count() - launches0)
        step_ms = sum(s.elapsed_time(e) for s, e in evs)
        # Short timed regions end before nvidia-smi samples them: keep the same
        # load running (untimed, same count on every rank) until the sampler
        # has seen ~0.4 s of it.
        per = step_ms / steps
        if world > 1:
            t = torch.tensor([per], dtype=torch.float64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            per = t.item()
        extra = max(0, int(400.0 / max(per, 1e-3)) - steps)
        for i in range(extra):
            if i % 8 == 0:
                flush()
            run_step()
        torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(device)

    # kernel-only: the dominant kernel's launch duration on its own stream
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for s, e in kev:
        flush()
        s.record(stream)
        if graph is not None:
            graph.replay()  # a graph-captured step is exactly the product launch
        else:
            launch(sub, c_dev, a_dev, b_dev, w.ops)
        e.record(stream)
    torch.cuda.synchronize(device)
    kern_ms = [s.elapsed_time(e) for s, e in kev]
    del a_dev, b_dev, c_dev, flush
    return {"step_ms_total": step_ms, "kernel_ms_mean": sum(kern_ms) / len(kern_ms),
            "kernel_ms_min": min(kern_ms), "launches": launches, "clocks": clocks.summary(),
            "graph": graph is not None}


def roofline(w, rows: int, kernel_ms: float) -> dict:
    m, k, n = w.mkn
    if w.key == "c2":
        algo = unit_amount(w, rows)
        peak, src = hbm_peak()
        achieved = algo / (kernel_ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": ncu_traffic(w.key),
                "algorithmic_bytes_per_launch": int(algo), "peak_source": src}
    if w.key == "c5":
        pairs = rows * k * n
        peak, src = minplus_peak()
        achieved = pairs / (kernel_ms * 1e-3) / 1e9
        return {"bound": "alu", "achieved": round(achieved, 1), "peak": round(peak, 1),
                "unit": "Gpairs/s", "frac": round(achieved / peak, 4),
                "traffic": ncu_traffic(w.key), "algorithmic_pairs_per_launch": pairs,
                "peak_source": src}
    flops = 2.0 * rows * k * n
    peak, src = fp64_peak()
    achieved = flops / (kernel_ms * 1e-3) / 1e12
    return {"bound": "tensor", "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4), "traffic": ncu_traffic(w.key),
            "algorithmic_flops_per_launch": int(flops), "peak_source": src}


# ---------------------------------------------------------------------------- e2e leg
def measure_e2e(w, rows_range, a_pin, b_pin, steps, warmup, device, world, rank, group=None):
    """Public API with pinned host buffers; H2D + kernel + D2H inside the timer."""
    import torch
    import torch.distributed as dist

    import paper_0907_0792_b200 as moa
    from paper_0907_0792_b200 import MoaArray
    from paper_0907_0792_b200.distributed import sharded_product_host

    r0, r1 = rows_range
    plan = plan_for(w)
    if world == 1:
        A = MoaArray._wrap(w.shape_a, a_pin.numpy())
        B = MoaArray._wrap(w.shape_b, b_pin.numpy())
        fn = moa.inner if w.mode == "inner" else moa.outer

        def step():
            return fn(A, B, w.ops)
    else:
        gplan = job_plan(w, world)
        a_blk = a_pin[r0 * plan.lstride:r1 * plan.lstride] if SCALING[w.key] == "strong" \
            else a_pin  # weak scaling: this rank's unit is its whole A

        def step():
            return sharded_product_host(gplan, a_blk, b_pin if rank == 0 else None, w.ops,
                                        device=device, group=group)
    # results are returned in pinned host memory from torch's caching host
    # allocator; drop each step's result before the next so the cache reuses it
    out = None
    for _ in range(warmup):
        out = None
        out = step()
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    marks = []
    for _ in range(steps):
        out = None
        out = step()
        marks.append(time.perf_counter())
    torch.cuda.synchronize(device)
    elapsed = time.perf_counter() - t0
    if os.environ.get("MOA_BENCH_VERBOSE"):
        per = [round((b_ - a_) * 1e3, 2) for a_, b_ in zip([t0] + marks[:-1], marks)]
        print(f"[bench] {w.key} e2e per-step ms: {per}", file=sys.stderr)
    if world > 1:
        t = torch.tensor([elapsed], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = t.item()
    del out
    return elapsed


def measure_e2e_cabi(w, a_pin, b_pin, steps, warmup, device):
    """The reference-facing boundary with host buffers: one
    moa_product_rows_host call (include/moa_b200.h) per step on page-locked A,
    B and result; returns seconds for ``steps`` calls."""
    import torch

    from paper_0907_0792_b200.kernel import launch_host
    plan = plan_for(w)
    m, k, n = w.mkn
    res = torch.empty(m * n, dtype=a_pin.dtype, pin_memory=True).numpy()
    a, b = a_pin.numpy(), b_pin.numpy()
    for _ in range(warmup):
        launch_host(plan, res, a, b, w.ops, device=device.index)
    t0 = time.perf_counter()
    for _ in range(steps):
        launch_host(plan, res, a, b, w.ops, device=device.index)
    elapsed = time.perf_counter() - t0
    del res
    return elapsed


# ---------------------------------------------------------------------------- CPU legs
def cpu_reference_time(w, a, b, budget_s: float = 10.0, max_reps: int = 500, rows: int | None = None,
                       min_reps: int = 3):
    """Reference hot loop (oracle/_ref, else the C port) on all host cores.

    Returns (seconds per unit of ``rows`` rows, kind, cores, sample description)."""
    import oracle
    m, k, n = w.mkn
    cores = oracle.host_cores()
    rows = m if rows is None else rows
    a_s = a[:rows * (k if w.mode == "inner" else 1)]
    comb, red = w.ops.codes()
    kind = "reference" if oracle.ref_kernel() is not None else "port"
    run = (lambda: oracle.reference_product(a_s, b, rows, k, n, comb, red, workers=cores)) \
        if kind == "reference" else \
        (lambda: oracle.product(a_s, b, rows, k, n, comb, red, workers=cores))
    times = []
    t_end = time.perf_counter() + budget_s
    while len(times) < max_reps and (len(times) < min_reps or time.perf_counter() < t_end):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    sample = (f"{rows} of {m} result rows (full K={k}, N={n}), {len(times)} reps, median; "
              f"identity prefill + product_rows over {cores} threads, round-robin rows "
              f"(reference parallel.py:37-43); inputs {'float32 upcast to float64' if w.dtype == np.float32 else 'float64'}")
    return statistics.median(times), kind, cores, sample, rows


def cpu_rows_for(w) -> int:
    m, k, n = w.mkn
    return {"c1": m, "c2": m, "c3": m, "c4": 256, "c5": 256}[w.key]


def run_reference(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = WORKLOADS[args.config]
    a, b = w.generate()
    rows = cpu_rows_for(w)
    m, k, n = w.mkn
    import oracle
    kind = "reference" if oracle.ref_kernel() is not None else "port"
    cores = oracle.host_cores()
    comb, red = w.ops.codes()
    a_s = a[:rows * (k if w.mode == "inner" else 1)]

    def one():
        if kind == "reference":
            oracle.reference_product(a_s, b, rows, k, n, comb, red, workers=cores)
        else:
            oracle.product(a_s, b, rows, k, n, comb, red, workers=cores)
    for _ in range(args.warmup):
        one()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    el = time.perf_counter() - t0
    amount = unit_amount(w, rows)
    value = to_unit(w, amount * args.steps, el)
    metric, unit = METRIC[w.key]
    line = {"impl": "reference", "metric": metric, "value": round(value, 4), "unit": unit,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": SCALING[w.key], "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators of SURVEY.md §8d)",
            "config": {"workload": f"{w.key}: {w.description}", "sample_rows": rows},
            "cpu_baseline": {"value": round(value, 4), "unit": unit, "cores": cores, "kind": kind,
                             "sample": f"{rows} of {m} result rows per step (full K, N)"},
            "e2e": {"value": round(value, 4), "unit": unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- main
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-inner", action="store_true", help="skip the extra inner-product legs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--legs", nargs="*", default=None,
                    help="inner-product legs to run beside c2 (default: all of c1 c3 c4 c5)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend for N>1 (gloo only to exercise the "
                         "multi-rank code path on fewer GPUs than ranks; timings meaningless)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(local)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    w = WORKLOADS[args.config]
    m, k, n = w.mkn
    scaling = SCALING[w.key]
    a, b = w.generate()
    if scaling == "weak":
        rows_range = (0, m)   # every rank owns one full unit (weak scaling)
        job_rows = m * world
    else:
        from paper_0907_0792_b200.distributed import row_block
        rows_range = row_block(m, world, rank)
        job_rows = m

    dev = measure_device(w, rows_range, a, b, args.steps, max(args.warmup, 3), device, world, rank)
    step_ms = dev["step_ms_total"]
    kern_ms = dev["kernel_ms_mean"]
    if world > 1:
        t = torch.tensor([step_ms, kern_ms, float(dev["launches"])], dtype=torch.float64,
                         device=device)
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        step_ms, kern_ms, launches = mx[0].item(), mx[1].item(), int(sm[2].item())
    else:
        launches = dev["launches"]
    ms_per_step = step_ms / args.steps
    job_amount = unit_amount(w, job_rows) if scaling == "weak" else unit_amount(w, m)
    if scaling == "weak":
        job_amount = unit_amount(w, m) * world
    value = to_unit(w, job_amount, ms_per_step * 1e-3)

    # e2e through the public API, pinned host buffers
    a_pin, b_pin = pinned_copy(a), pinned_copy(b)
    e2e_steps = max(2, min(args.steps, 5))
    el = measure_e2e(w, rows_range, a_pin, b_pin, e2e_steps, 2, device, world, rank)
    isz = np.dtype(w.dtype).itemsize
    if scaling == "weak":
        h2d = world * (m * k + k * n) * isz if w.mode == "inner" else world * (m + n) * isz
        d2h = world * m * n * isz
    else:
        h2d = (m * k + k * n) * isz
        d2h = m * n * isz
    e2e_value = to_unit(w, job_amount * e2e_steps, el)
    e2e_api = None
    if world == 1:  # headline e2e through the C ABI; the public API beside it
        e2e_api = {"value": round(e2e_value, 3), "unit": METRIC[w.key][1],
                   "path": "moa.outer/inner on pinned host MoaArrays"}
        el = measure_e2e_cabi(w, a_pin, b_pin, e2e_steps, 2, device)
        e2e_value = to_unit(w, job_amount * e2e_steps, el)
    del a_pin, b_pin

    metric, unit = METRIC[w.key]
    line = {"metric": metric, "value": round(value, 3), "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32" if w.dtype == np.float32 else "f64",
            "data": "synthetic (seeded generators of SURVEY.md §8d; no public dataset)",
            "config": {"workload": f"{w.key}: {w.description}", "M": m, "K": k, "N": n,
                       "rows_per_rank": rows_range[1] - rows_range[0],
                       "parallelism": ("single GPU" if world == 1 else
                                       f"row-sharded x{world}, B broadcast "
                                       f"({dist.get_backend().upper()}) "
                                       + ("inside every step" if scaling == "strong" else
                                          "once, before the timed region")),
                       "l2": "flushed between timed steps (256 MiB write, outside the events)",
                       "cuda_graph": bool(dev.get("graph"))},
            "e2e": {"value": round(e2e_value, 3), "unit": unit, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": "moa_product_rows_host (C ABI) on page-locked host buffers"
                    if world == 1 else "distributed.sharded_product_host"},
            "gpu_launches": launches,
            **({"e2e_api": e2e_api} if e2e_api else {}),
            "roofline": roofline(w, rows_range[1] - rows_range[0], kern_ms),
            "kernel_ms": round(kern_ms, 4),
            "clocks": dev["clocks"]}

    if world == 1 and not args.no_inner and w.key == "c2":
        inner = {}
        for key in [k for k in ("c1", "c3", "c4", "c5") if args.legs is None or k in args.legs]:
            wi = WORKLOADS[key]
            ai, bi = wi.generate()
            mi = wi.mkn[0]
            st = 20 if key in ("c1", "c3") else 3
            d = measure_device(wi, (0, mi), ai, bi, st, 3, device, 1, 0)
            amt = unit_amount(wi, mi)
            inner[key] = {"metric": METRIC[key][0], "unit": METRIC[key][1],
                          "value": round(to_unit(wi, amt, d["step_ms_total"] / st * 1e-3), 2),
                          "kernel_ms": round(d["kernel_ms_mean"], 4),
                          "roofline": roofline(wi, mi, d["kernel_ms_mean"]),
                          "clocks": d["clocks"]}
            # the same product end to end through moa.inner on pinned host
            # arrays (H2D of A and B, the product, D2H of C inside the clock)
            ap, bp = pinned_copy(ai), pinned_copy(bi)
            e2e_st = 20 if key == "c1" else 3
            el_i = measure_e2e(wi, (0, mi), ap, bp, e2e_st, 3, device, 1, 0)
            isz_i = np.dtype(wi.dtype).itemsize
            ki, ni = wi.mkn[1], wi.mkn[2]
            el_c = measure_e2e_cabi(wi, ap, bp, e2e_st, 3, device)
            inner[key]["e2e"] = {"value": round(to_unit(wi, amt * e2e_st, el_c), 2),
                                 "unit": METRIC[key][1], "ms_per_step": round(el_c / e2e_st * 1e3, 3),
                                 "h2d_bytes_per_step": (mi * ki + ki * ni) * isz_i,
                                 "d2h_bytes_per_step": mi * ni * isz_i,
                                 "path": "moa_product_rows_host (C ABI) on page-locked host "
                                         "buffers (streamed row blocks)"}
            inner[key]["e2e_api"] = {"value": round(to_unit(wi, amt * e2e_st, el_i), 2),
                                     "unit": METRIC[key][1],
                                     "ms_per_step": round(el_i / e2e_st * 1e3, 3),
                                     "path": "moa.inner on pinned host MoaArrays (streamed row blocks)"}
            del ap, bp
            if rank == 0 and not args.no_cpu:
                # the reference's own loop on a small row sample (~1-3 s of CPU)
                rows_i = {"c1": mi, "c3": 1024, "c4": 32, "c5": 32}[key]
                t_i, kind_i, cores_i, sample_i, rows_i = cpu_reference_time(
                    wi, ai, bi, budget_s=1.5, rows=rows_i, min_reps=1)
                inner[key]["cpu_baseline"] = {
                    "value": round(to_unit(wi, unit_amount(wi, rows_i), t_i), 4),
                    "unit": METRIC[key][1], "cores": cores_i, "kind": kind_i, "sample": sample_i}
            del ai, bi
        line["inner"] = inner

    if world > 1 and not args.no_inner and w.key == "c2":
        # BASELINE configs 4-5 at N GPUs: result rows sharded over the ranks, B
        # broadcast from rank 0 inside every step (strong scaling, max over ranks)
        from paper_0907_0792_b200.distributed import row_block
        inner = {}
        for key in ("c4", "c5"):
            wi = WORKLOADS[key]
            ai, bi = wi.generate()
            mi = wi.mkn[0]
            rr = row_block(mi, world, rank)
            st = 3
            d = measure_device(wi, rr, ai, bi, st, 3, device, world, rank)
            t = torch.tensor([d["step_ms_total"], d["kernel_ms_mean"]], dtype=torch.float64,
                             device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            amt = unit_amount(wi, mi)
            inner[key] = {"metric": METRIC[key][0], "unit": METRIC[key][1], "scaling": "strong",
                          "value": round(to_unit(wi, amt, t[0].item() / st * 1e-3), 2),
                          "rows_per_rank": rr[1] - rr[0],
                          "kernel_ms": round(t[1].item(), 4),
                          "roofline": roofline(wi, rr[1] - rr[0], t[1].item()),
                          "clocks": d["clocks"]}
            del ai, bi
        line["inner"] = inner

    if world == 1 and rank == 0 and not args.no_cpu:
        t_unit, kind, cores, sample, rows = cpu_reference_time(w, a, b, rows=cpu_rows_for(w))
        line["cpu_baseline"] = {"value": round(to_unit(w, unit_amount(w, rows), t_unit), 4),
                                "unit": unit, "cores": cores, "kind": kind, "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
