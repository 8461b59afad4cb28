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
SM_COUNT = 148


# ---------------------------------------------------------------------------- peaks
# Every roofline denominator is a MEASURED figure read from a committed file;
# a missing file leaves the figure unmeasured (peak/frac null) instead of
# falling back to a hard-coded number.  The theoretical ceiling of the same
# pipe at the run's SM clock is printed beside each one.
def hbm_peak() -> tuple[float | None, str]:
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    return None, "unmeasured: MEASURED_PEAKS.json absent"


def microbench_peaks() -> dict:
    p = REPO / "profiles" / "r01_peaks_microbench.json"
    return json.loads(p.read_text()) if p.exists() else {}


def fp64_peak() -> tuple[float | None, str]:
    vals = [v for k, v in microbench_peaks().items() if k.startswith("dmma_")]
    if vals:
        return max(vals), "measured DMMA mma.sync f64 microbenchmark (profiles/r01_peaks_microbench.json)"
    return None, "unmeasured: profiles/r01_peaks_microbench.json absent"


def minplus_peak() -> tuple[float | None, str]:
    """Best measured (add, min) pair rate on the ALU/FMA pipes, G pairs/s.

    profiles/r01_minplus_mix2.json holds warp-instructions per clock per SM for
    FADD2 + FMNMX3 and FADD2 + VIMNMX3 units (64 pairs each) at 1965 MHz."""
    p = REPO / "profiles" / "r01_minplus_mix2.json"
    if p.exists():
        mix = json.loads(p.read_text())
        units = max(mix.get("fadd2_fmnmx3_pairs_winstr_per_clk_sm", 0.0),
                    mix.get("fadd2_vimnmx3_units_winstr_per_clk_sm", 0.0))
        return (units * 64 * SM_COUNT * 1.965e9 / 1e9,
                "measured FADD2+VIMNMX3 / FADD2+FMNMX3 instruction-mix microbenchmark "
                "(profiles/r01_minplus_mix2.json), best mix, 1965 MHz")
    return None, "unmeasured: profiles/r01_minplus_mix2.json absent"


def theoretical(key: str, sm_mhz: float | None) -> dict:
    """The pipe's nominal ceiling at the run's SM clock (max clock if unsampled)."""
    mhz = sm_mhz or 1965.0
    if key == "c5":
        # 64 pairs per warp need 64 adds and 32 three-input folds: 2 FADD +
        # 1 VIMNMX3 = 3 issue clocks (FADD2 would halve the adds' issue slots
        # but stalls dispatch next to ALU-pipe instructions: ncu on
        # tools/mb_dualissue.cu, profiles/r02_mb_dualissue_ncu.json), on each
        # of 4 schedulers (profiles/r02_c5_ceiling.md)
        return {"value": round(SM_COUNT * 4 * 64 / 3 * mhz * 1e6 / 1e9, 1), "unit": "Gpairs/s",
                "what": "issue limit: 2 FADD + 1 VIMNMX3 (3 issue clocks) per 64 pairs per warp, "
                        "4 schedulers x 148 SMs; FADD2 next to the fold stalls dispatch, so no "
                        "form beats it (measured)",
                "sm_mhz": mhz}
    if key == "c2":
        return {"value": None, "unit": "GB/s", "what": "write-only ceiling measured: cudaMemset "
                f"{microbench_peaks().get('memset_GBs')} GB/s (profiles/r01_peaks_microbench.json)"}
    return {"value": round(SM_COUNT * 64 * 2 * mhz * 1e6 / 1e12, 2), "unit": "TFLOP/s",
            "what": "148 SMs x 64 FP64 FMA/clk (DMMA) x 2 flop", "sm_mhz": mhz}


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


def roofline(w, rows: int, kernel_ms: float, sm_mhz: float | None = None) -> dict:
    m, k, n = w.mkn
    if w.key == "c2":
        algo = unit_amount(w, rows)
        peak, src = hbm_peak()
        achieved = algo / (kernel_ms * 1e-3) / 1e9
        out = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
               "algorithmic_bytes_per_launch": int(algo)}
    elif w.key == "c5":
        algo = rows * k * n
        peak, src = minplus_peak()
        achieved = algo / (kernel_ms * 1e-3) / 1e9
        out = {"bound": "alu", "achieved": round(achieved, 1),
               "peak": None if peak is None else round(peak, 1), "unit": "Gpairs/s",
               "algorithmic_pairs_per_launch": algo}
    else:
        algo = 2.0 * rows * k * n
        peak, src = fp64_peak()
        achieved = algo / (kernel_ms * 1e-3) / 1e12
        out = {"bound": "tensor", "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
               "algorithmic_flops_per_launch": int(algo)}
    out["frac"] = None if peak is None else round(achieved / peak, 4)
    out["traffic"] = ncu_traffic(w.key)
    out["peak_source"] = src
    out["theoretical"] = theoretical(w.key, sm_mhz)
    th = out["theoretical"]["value"]
    if th:
        out["frac_of_theoretical"] = round(achieved / th, 4)
    return out


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
        # strong scaling: this rank's rows of A (a_pin may already be just the
        # block); weak scaling: this rank's unit is its whole A
        nblk = (r1 - r0) * plan.lstride
        a_blk = a_pin[r0 * plan.lstride:r1 * plan.lstride] \
            if SCALING[w.key] == "strong" and a_pin.numel() != nblk else a_pin

        def step():
            return sharded_product_host(gplan, a_blk, b_pin if rank == 0 else None, w.ops,
                                        device=device, group=group)
    # results come back in the library's page-locked host blocks; drop each
    # step's result before the next so its block is reused
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


def measure_e2e_pageable(w, a, b, steps, warmup):
    """The public API exactly as a reference user calls it: ``MoaArray`` built
    from ordinary (pageable) numpy arrays, ``moa.outer``/``moa.inner``, the
    result handed back in host memory; returns seconds for ``steps`` calls."""
    import paper_0907_0792_b200 as moa
    from paper_0907_0792_b200 import MoaArray
    A = MoaArray(w.shape_a, a, dtype=w.dtype)
    B = MoaArray(w.shape_b, b, dtype=w.dtype)
    fn = moa.inner if w.mode == "inner" else moa.outer
    t_first = time.perf_counter()
    out = fn(A, B, w.ops)
    t_first = time.perf_counter() - t_first
    for _ in range(max(0, warmup - 1)):
        out = None
        out = fn(A, B, w.ops)
    t0 = time.perf_counter()
    for _ in range(steps):
        out = None
        out = fn(A, B, w.ops)
    elapsed = time.perf_counter() - t0
    del out
    return elapsed, t_first


# ---------------------------------------------------------------------------- CPU legs
def cpu_rows_for(w, cores: int) -> int:
    """configs 1-3 in full; configs 4-5 on R = 32*W contiguous
    rows (W = the host's cores), extrapolated x M/R (the per-row cost is constant)."""
    m = w.mkn[0]
    return m if w.key in ("c1", "c2", "c3") else min(m, 32 * cores)


def _cpu_runner(w, a, b, rows):
    """One call of the reference's execute_parallel on the first ``rows`` rows:
    an identity-filled result (kernel.py:149) and W threads, worker k running
    product_rows(..., start=k, step=W) (parallel.py:37-43), through the
    reference's own compiled loop (oracle/_ref) or, if absent, the C port.
    Inputs are float64 before the clock starts, as the reference's bench
    builds its MoaArrays outside the timer (bench.py:110-111)."""
    import oracle
    m, k, n = w.mkn
    cores = oracle.host_cores()
    a_s = np.ascontiguousarray(a[:rows * (k if w.mode == "inner" else 1)], dtype=np.float64)
    b64 = np.ascontiguousarray(b, dtype=np.float64)
    comb, red = w.ops.codes()
    kind = "reference" if oracle.ref_kernel() is not None else "port"
    fn = oracle.reference_product if kind == "reference" else oracle.product

    def run():
        fn(a_s, b64, rows, k, n, comb, red, workers=cores)
    return run, kind, cores


def cpu_reference_time(w, a, b, rows: int, reps: int = 3) -> dict:
    """Best of ``reps`` timed calls (bench.py:118-133 protocol, best instead of
    mean as SURVEY.md §8(d) asks); returns the cpu_baseline object."""
    m = w.mkn[0]
    run, kind, cores = _cpu_runner(w, a, b, rows)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        run()
        times.append(time.perf_counter() - t0)
    best = min(times)
    sample = (f"W={cores} threads, R={rows} of M={m} contiguous result rows (full K, N)"
              + ("" if rows == m else f", extrapolated x M/R = x{m / rows:g}")
              + f"; best of {reps} ({', '.join(f'{t:.3f}' for t in times)} s); identity "
              f"prefill + product_rows(start=k, step=W) per thread (reference "
              f"parallel.py:37-43); inputs "
              + ("float32 upcast to float64 before the clock" if w.dtype == np.float32
                 else "float64"))
    metric, unit = METRIC[w.key]
    return {"value": round(to_unit(w, unit_amount(w, rows), best), 4), "unit": unit,
            "cores": cores, "kind": kind, "sample": sample, "seconds_per_sample": best}


def job_config(w, world: int) -> dict:
    """The workload's description, identical on both arms (``--impl ours`` and
    ``--impl reference``), so the driver compares like with like."""
    from paper_0907_0792_b200.distributed import row_block
    m, k, n = w.mkn
    scaling = SCALING[w.key]
    rows = m if scaling == "weak" else row_block(m, world, 0)[1]
    return {"workload": f"{w.key}: {w.description}", "M": m, "K": k, "N": n,
            "ranks": world, "rows_per_rank": rows,
            "parallelism": ("single GPU" if world == 1 else
                            f"row-sharded x{world}, B broadcast from rank 0 "
                            + ("inside every step" if scaling == "strong" else
                               "once, before the timed region")),
            "l2": "flushed between timed steps (256 MiB write, outside the events)"}


def run_reference(args) -> None:
    """The reference arm: the reference's own CPU implementation of the path
    on this box's host cores, on the same workload as ``--impl ours``.  Never
    loads this repo's CUDA library (tests/test_bench_reference_arm.py)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = WORKLOADS[args.config]
    a, b = w.generate()
    import oracle
    rows = cpu_rows_for(w, oracle.host_cores())
    m = w.mkn[0]
    run, kind, cores = _cpu_runner(w, a, b, rows)
    for _ in range(args.warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()
    el = time.perf_counter() - t0
    value = to_unit(w, unit_amount(w, rows) * args.steps, el)
    metric, unit = METRIC[w.key]
    sample = (f"W={cores} threads, R={rows} of M={m} contiguous result rows per step "
              "(full K, N)" + ("" if rows == m else f", extrapolated x M/R = x{m / rows:g}"))
    line = {"impl": "reference", "metric": metric, "value": round(value, 4), "unit": unit,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": SCALING[w.key], "vs_baseline": None,
            "dtype": "f32" if w.dtype == np.float32 else "f64",
            "data": "synthetic (seeded generators of SURVEY.md §8d; no public dataset)",
            "config": job_config(w, args.gpus),
            "execution": f"reference compiled loop ({kind}, oracle/_ref) on {cores} host "
                         "threads, rank 0 only; no GPU",
            "cpu_baseline": {"value": round(value, 4), "unit": unit, "cores": cores, "kind": kind,
                             "sample": sample},
            "e2e": {"value": round(value, 4), "unit": unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def inner_leg(key, device, world, rank, group=None) -> dict:
    """One BASELINE inner config: device-resident value and roofline, and the
    same product end to end from host buffers (C ABI at N=1; the sharded
    host path at N>1)."""
    import torch
    import torch.distributed as dist

    from paper_0907_0792_b200.distributed import row_block
    wi = WORKLOADS[key]
    ai, bi = wi.generate()
    mi, ki, ni = wi.mkn
    rr = (0, mi) if world == 1 else row_block(mi, world, rank)
    st = 20 if key in ("c1", "c3") else 3
    d = measure_device(wi, rr, ai, bi, st, 3, device, world, rank, group)
    step_ms, kern_ms = d["step_ms_total"], d["kernel_ms_mean"]
    if world > 1:
        t = torch.tensor([step_ms, kern_ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        step_ms, kern_ms = t[0].item(), t[1].item()
    amt = unit_amount(wi, mi)
    isz = np.dtype(wi.dtype).itemsize
    leg = {"metric": METRIC[key][0], "unit": METRIC[key][1], "scaling": SCALING[key],
           "value": round(to_unit(wi, amt, step_ms / st * 1e-3), 2),
           "rows_per_rank": rr[1] - rr[0], "kernel_ms": round(kern_ms, 4),
           "roofline": roofline(wi, rr[1] - rr[0], kern_ms, d["clocks"].get("sm_mhz")),
           "clocks": d["clocks"], "gpu_launches": d["launches"]}
    if world == 1:
        ap, bp = pinned_copy(ai), pinned_copy(bi)
    else:  # each rank pins only what it sends: its A rows, and B on rank 0
        ap = pinned_copy(ai[rr[0] * ki:rr[1] * ki])
        bp = pinned_copy(bi) if rank == 0 else None
    e2e_st = 20 if key == "c1" else 5
    el_i = measure_e2e(wi, rr, ap, bp, e2e_st, 3, device, world, rank, group)
    if world == 1:
        with ClockSampler(device.index) as e2e_clocks:
            el_c = measure_e2e_cabi(wi, ap, bp, e2e_st, 3, device)
        leg["e2e"] = {"value": round(to_unit(wi, amt * e2e_st, el_c), 2), "unit": METRIC[key][1],
                      "ms_per_step": round(el_c / e2e_st * 1e3, 3),
                      "h2d_bytes_per_step": (mi * ki + ki * ni) * isz,
                      "d2h_bytes_per_step": mi * ni * isz,
                      "path": "moa_product_rows_host (C ABI) on page-locked host buffers "
                              "(streamed row blocks)", "clocks": e2e_clocks.summary()}
        leg["e2e_api"] = {"value": round(to_unit(wi, amt * e2e_st, el_i), 2),
                          "unit": METRIC[key][1], "ms_per_step": round(el_i / e2e_st * 1e3, 3),
                          "path": "moa.inner on pinned host MoaArrays (streamed row blocks)"}
        if key == "c4":
            el_p, first = measure_e2e_pageable(wi, ai, bi, 2, 1)
            leg["e2e_pageable"] = {"value": round(to_unit(wi, amt * 2, el_p), 2),
                                   "unit": METRIC[key][1], "ms_per_step": round(el_p / 2 * 1e3, 3),
                                   "first_call_ms": round(first * 1e3, 1),
                                   "path": "moa.inner on MoaArray(numpy) (pageable) inputs"}
    else:
        leg["e2e"] = {"value": round(to_unit(wi, amt * e2e_st, el_i), 2), "unit": METRIC[key][1],
                      "ms_per_step": round(el_i / e2e_st * 1e3, 3),
                      "h2d_bytes_per_step": (mi * ki + ki * ni) * isz,
                      "d2h_bytes_per_step": mi * ni * isz,
                      "path": "distributed.sharded_product_host: A rows per rank + B on rank 0 "
                              "from page-locked host buffers, broadcast, product, result block "
                              "back to host; max over ranks"}
    del ap, bp
    return leg, (ai, bi)


# ---------------------------------------------------------------------------- main
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-inner", action="store_true", help="skip the extra inner-product legs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline legs")
    ap.add_argument("--legs", nargs="*", default=None,
                    help="inner-product legs to run beside c2 (default: c1 c3 c4 c5 at N=1, "
                         "c4 c5 at N>1)")
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
    else:
        from paper_0907_0792_b200.distributed import row_block
        rows_range = row_block(m, world, rank)

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
    job_amount = unit_amount(w, m) * (world if scaling == "weak" else 1)
    value = to_unit(w, job_amount, ms_per_step * 1e-3)

    # e2e: host buffers, copies inside the clock
    a_pin, b_pin = pinned_copy(a), pinned_copy(b)
    e2e_steps = max(2, min(args.steps, 5))
    el = measure_e2e(w, rows_range, a_pin, b_pin, e2e_steps, 2, device, world, rank)
    isz = np.dtype(w.dtype).itemsize
    units = world if scaling == "weak" else 1
    h2d = units * ((m * k + k * n) if w.mode == "inner" else (m + n)) * isz
    d2h = units * m * n * isz
    e2e_value = to_unit(w, job_amount * e2e_steps, el)
    e2e_api = e2e_pageable = None
    if world == 1:  # headline e2e through the C ABI; the public API beside it
        e2e_api = {"value": round(e2e_value, 3), "unit": METRIC[w.key][1],
                   "path": "moa.outer/inner on pinned host MoaArrays"}
        el = measure_e2e_cabi(w, a_pin, b_pin, e2e_steps, 2, device)
        e2e_value = to_unit(w, job_amount * e2e_steps, el)
        el_p, first = measure_e2e_pageable(w, a, b, e2e_steps, 2)
        e2e_pageable = {"value": round(to_unit(w, job_amount * e2e_steps, el_p), 3),
                        "unit": METRIC[w.key][1], "first_call_ms": round(first * 1e3, 1),
                        "path": "moa.outer/inner on MoaArray(numpy) (pageable) inputs, "
                                "result returned as a host MoaArray"}
    del a_pin, b_pin

    metric, unit = METRIC[w.key]
    line = {"metric": metric, "value": round(value, 3), "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32" if w.dtype == np.float32 else "f64",
            "data": "synthetic (seeded generators of SURVEY.md §8d; no public dataset)",
            "config": job_config(w, world),
            "execution": {"dist_backend": dist.get_backend().upper() if world > 1 else None,
                          "cuda_graph": bool(dev.get("graph"))},
            "e2e": {"value": round(e2e_value, 3), "unit": unit, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "path": "moa_product_rows_host (C ABI) on page-locked host buffers"
                    if world == 1 else "distributed.sharded_product_host, max over ranks"},
            "gpu_launches": launches,
            **({"e2e_api": e2e_api} if e2e_api else {}),
            **({"e2e_pageable": e2e_pageable} if e2e_pageable else {}),
            "roofline": roofline(w, rows_range[1] - rows_range[0], kern_ms,
                                 dev["clocks"].get("sm_mhz")),
            "kernel_ms": round(kern_ms, 4),
            "clocks": dev["clocks"]}

    inputs = {}
    if not args.no_inner and w.key == "c2":
        default_legs = ("c1", "c3", "c4", "c5") if world == 1 else ("c4", "c5")
        inner = {}
        for key in [x for x in default_legs if args.legs is None or x in args.legs]:
            inner[key], inputs[key] = inner_leg(key, device, world, rank)
            if rank != 0 or args.no_cpu:
                inputs.pop(key)
        line["inner"] = inner

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    # CPU legs last, on rank 0 alone, once every other rank has exited, so no
    # GPU work or waiting rank competes for the host cores
    if not args.no_cpu:
        import oracle
        cores = oracle.host_cores()
        line["cpu_baseline"] = cpu_reference_time(w, a, b, cpu_rows_for(w, cores))
        for key, (ai, bi) in inputs.items():
            wi = WORKLOADS[key]
            line["inner"][key]["cpu_baseline"] = cpu_reference_time(wi, ai, bi,
                                                                    cpu_rows_for(wi, cores))
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
