#!/usr/bin/env python
"""Benchmark: fp64 SpTRSV on B200 — µs/solve and GFLOP/s (2·nnz/t), % of the HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config lap2d-4096]
                    [--precision fast|exact] [--executor auto|rows|chains|stencil|push]
    python bench.py --impl reference ...      # the reference's CPU path (oracle port)
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N   # column-block over N GPUs

One JSON line on stdout (rank 0). A "step" is one solve of L x = b for the
configured matrix with b = ones (the reference CLI default, cli.py:139-140).

* ``value``: GFLOP/s = 2·nnz / t, t = device time per solve over K
  back-to-back solves with b and x resident in HBM (CUDA events on the solve
  stream, barrier + synchronize on both sides, max over ranks).
* ``e2e``: the same metric through the C-ABI host-buffer call
  (``sptrsv_solve``: pinned b -> device, solve, device -> pinned x), wall clock.
* ``roofline``: the solve kernel's algorithmic bytes (SURVEY.md §8d:
  12·nnz + 4·(n+1) + 16·n) over its CUDA-event duration, against the measured
  HBM copy bandwidth in MEASURED_PEAKS.json (N > 1: the slowest rank's kernel
  against N HBMs).
* ``timing``: >= 100 repeats with mean / min / max per solve,
  kernel-only times, setup and the combined setup + solve figure
  (cli.py:199-202). Inputs under 5x the L2 size are timed with a 256 MB
  scratch write between solves (the L2-cold figure; ``l2_warm_ms`` beside it).
* ``cpu_baseline``: the C port of the reference ``solve_serial`` (oracle/) on
  one host core, full matrix (rank 0, N = 1 only).

N > 1 (torchrun, one process per GPU): block_partition(n, N) (``--partition
nnz``, the default for rmat: slabs of equal nnz, nnz_block_partition) — every GPU owns a
contiguous slab of rows (for lap2d-4096: whole 64-grid-row bands of the
stencil executor) and its x; the peer state (stencil mailboxes, or component
segments) is opened over CUDA IPC and read with one-sided loads inside the
solve (no collective in the solve); an NCCL all-reduce of one word orders
consecutive solves. Total work is fixed, so ``scaling`` is "strong".
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

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SpTRSV µs/solve and GFLOP/s (2·nnz/t) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "GFLOP/s"


def _method(config: str, precision: str, executor: str) -> str:
    """How the executor solved this config, for the bench line."""
    ex = executor.split(" ")[0]
    fast = precision == "fast"
    if ex == "stencil" and config.startswith("lap2d"):
        return ("2D wavefront, bands entered through halo bands when the plan-time error contraction allows "
                "(lap2d: <= 3e-31 |x|; SPTRSV_ST_GROUP=0: one chain)") if fast else "2D wavefront, one band chain (bitwise)"
    if ex == "stencil":
        return ("3D wavefront, z-groups entered through halo z-tiles (<= 2^-64 |x|; SPTRSV_S3_ZGROUP=0: one chain)"
                if fast else "3D wavefront, one chain (bitwise)")
    if ex == "band":
        return ("row blocks: TMA-streamed sweeps, tail chain by superblocks, coupling reach (terms <= 2^-64 dropped)"
                if fast else "band window kernel (bitwise)")
    if ex == "rows":
        return "component pool (level-ordered tickets, value-is-flag polling)"
    return ex

def algorithmic_bytes(n: int, nnz: int) -> int:
    """int32 indices/pointers, f64 values, b and x."""
    return 12 * nnz + 4 * (n + 1) + 8 * n + 8 * n


def measured_peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5,
                ).stdout.strip()
                if out:
                    self.rows.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 3 + k and r[3 + k] == "Active"})
        return {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(mx) if mx else None,
            "reasons": reasons,
            "samples": len(self.rows),
        }


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def cpu_solve(l, b, reps: int, budget_s: float) -> dict:
    """The reference's CPU solve (C port of solve_serial, reference.py:20-35), 1 core."""
    import oracle

    times, x = [], None
    t_end = time.perf_counter() + budget_s
    while len(times) < reps or (not times):
        t0 = time.perf_counter()
        x = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() > t_end:
            break
    return {"seconds": statistics.mean(times), "reps": len(times), "x": x}


def reference_arm(args, l, b, n, nnz):
    for _ in range(args.warmup):
        cpu_solve(l, b, 1, 0)
    r = cpu_solve(l, b, args.steps, 120.0)
    gflops = 2.0 * nnz / r["seconds"] / 1e9
    return {
        "metric": METRIC, "value": gflops, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": r["reps"], "warmup": args.warmup, "ms_per_step": r["seconds"] * 1e3,
        "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "n": n, "nnz": nnz, "rhs": "ones", "precision": "exact (serial)",
                   "executor": "solve_serial (C port of reference.py:20-35)", "parallelism": "1 CPU core"},
        "cpu_baseline": {"value": gflops, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"full {args.config} solve_serial (C port of reference.py:20-35, "
                                   f"-ffp-contract=off), {r['reps']} reps"},
        "e2e": {"value": gflops, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="lap2d-4096")
    ap.add_argument("--precision", choices=["fast", "exact"], default="fast")
    ap.add_argument("--executor", choices=["auto", "rows", "chains", "stencil", "push", "band"], default="auto")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--partition", choices=["auto", "block", "nnz"], default="auto",
                    help="N > 1 owner map: block_partition (reference), or contiguous slabs of equal nnz "
                         "(64-row aligned); auto: nnz for configs without grid structure (rmat), else block")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--l2", choices=["auto", "flush", "warm"], default="auto",
                    help="auto: flush a 256 MB scratch buffer between timed solves when the solve's inputs are "
                         "< 5x the L2 size, else back-to-back solves")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    ws, rank, local = dist_env()
    from paper_2012_06959_b200 import synth

    t0 = time.perf_counter()
    l = synth.config_matrix(args.config)
    gen_s = time.perf_counter() - t0
    n, nnz = l.n, l.nnz
    flops = 2.0 * nnz
    b = np.ones(n)

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(reference_arm(args, l, b, n, nnz)), flush=True)
        return

    import torch

    from paper_2012_06959_b200 import _native

    # SPTRSV_BENCH_SAME_DEVICE=1 + SPTRSV_BENCH_BACKEND=gloo: every rank on
    # cuda:0 (exercises the N > 1 path on a one-GPU box; NCCL refuses that)
    dev = 0 if os.environ.get("SPTRSV_BENCH_SAME_DEVICE") == "1" else local
    torch.cuda.set_device(dev)
    if ws > 1:
        import torch.distributed as dist

        backend = os.environ.get("SPTRSV_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{dev}"))
        else:
            dist.init_process_group(backend)
    stream = torch.cuda.Stream(dev)  # solves, events and the inter-solve all-reduce share it
    sh = stream.cuda_stream

    ts = time.perf_counter()
    if ws > 1:
        from paper_2012_06959_b200 import multi

        kind = args.partition
        if kind == "auto":
            kind = "block" if args.config.startswith(("lap2d", "lap3d", "banded")) else "nnz"
        # rows' entry counts (CSC column counts of the transpose = row counts)
        row_w = np.bincount(np.asarray(l.row_idx), minlength=n).astype(np.float64) if kind == "nnz" else None
        partition = multi.rank_partition(n, ws, kind, row_weight=row_w, align=64)
        solver = multi.DistributedSolver(l, partition, rank, device=dev, precision=args.precision)
        plan = solver.native
        owned = torch.from_numpy((partition.owner_arr == rank).astype(np.float64)).to(f"cuda:{dev}")
    else:
        solver = None
        plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, n, precision=args.precision,
                                  executor=args.executor, device=dev)
    setup_s = time.perf_counter() - ts
    info = plan.info()
    if ws > 1:
        if solver.replicated:  # no per-PE mode for this executor: every rank solves the whole system
            info["executor"] = f"{info['executor']} (replicated per rank: no per-PE mode)"
        else:
            via = {"stencil": ("local halo bands" if args.precision == "fast" else "peer mailboxes"),
                   "band": "superblock chain through peer slots"}.get(info["executor"], "peer segments")
            info["executor"] = f"{info['executor']} (PE partition, {via})"

    db = torch.from_numpy(b).to(f"cuda:{dev}")
    dx = torch.zeros_like(db)
    order_word = torch.zeros(1, device=f"cuda:{dev}")

    def one_solve():
        if ws > 1:
            # every rank finished the previous solve before any segment is reset
            torch.distributed.all_reduce(order_word)
        plan.solve_device_async(db.data_ptr(), dx.data_ptr(), sh)

    alg = algorithmic_bytes(n, nnz)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = args.l2 == "flush" or (args.l2 == "auto" and alg < 5 * l2_bytes)
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}") if flush else None

    def timed_loop(k: int, do_flush: bool) -> tuple[list[float], list[float]]:
        """k solves; per-solve device times (events on the solve stream) and kernel times."""
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * k)]
        kms = []
        for i in range(k):
            if do_flush:
                scratch.fill_(i & 0xFF)  # 256 MB > 126 MB L2, outside the timed events
            ev[2 * i].record(stream)
            one_solve()
            ev[2 * i + 1].record(stream)
            if do_flush or i >= k - 10:
                kms.append(plan.synchronize()["kernel_ms"])
        torch.cuda.synchronize(dev)
        return [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(k)], kms

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            one_solve()
        plan.synchronize()
        torch.cuda.synchronize(dev)
        if ws > 1:
            torch.distributed.barrier()
        with ClockSampler(dev) as clocks:
            torch.cuda.synchronize(dev)
            if flush:
                per_solve, kernel_ms = timed_loop(args.steps, True)
                total_ms = sum(per_solve)
            else:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(args.steps):
                    one_solve()
                e1.record(stream)
                torch.cuda.synchronize(dev)
                total_ms = e0.elapsed_time(e1)
                # per-solve spread and per-launch kernel durations (same stream)
                per_solve, kernel_ms = timed_loop(min(args.steps, 30), False)
        warm = None
        if flush:  # the back-to-back (L2-warm) figure beside the flushed one
            w0 = torch.cuda.Event(enable_timing=True)
            w1 = torch.cuda.Event(enable_timing=True)
            w0.record(stream)
            for _ in range(args.steps):
                one_solve()
            w1.record(stream)
            torch.cuda.synchronize(dev)
            warm = w0.elapsed_time(w1) / args.steps
        if ws > 1:
            torch.distributed.barrier()
        ms = total_ms / args.steps
        kern = statistics.mean(kernel_ms) if kernel_ms else ms
        if ws > 1:
            t = torch.tensor([ms, kern], device=f"cuda:{dev}")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms, kern = float(t[0].item()), float(t[1].item())
            # x: each rank holds its owned rows; the sum over ranks assembles it
            xfull = dx * owned
            torch.distributed.all_reduce(xfull)
            x_dev = xfull.cpu().numpy()
        else:
            x_dev = dx.cpu().numpy()

    # ---- end-to-end through the C ABI host-buffer call (pinned b / x) -----
    hb = torch.from_numpy(b).pin_memory()
    hx = torch.empty(n, dtype=torch.float64).pin_memory()
    hb_np, hx_np = hb.numpy(), hx.numpy()
    t_e2e = []
    e2e_streamed = 0
    if ws == 1:
        e2e_streamed = int(plan.solve(hb_np, out=hx_np)[1].get("streamed_io", 0))
        for _ in range(args.e2e_steps):
            t1 = time.perf_counter()
            plan.solve(hb_np, out=hx_np)
            t_e2e.append(time.perf_counter() - t1)
        # same solution through both paths (bitwise when the executor is
        # deterministic; fast-mode split rows add partial sums atomically)
        diff = np.abs(hx_np - x_dev) / np.maximum(np.abs(x_dev), 1.0)
        assert (not diff.size) or float(np.nanmax(diff)) <= 1e-12, float(np.nanmax(diff))
        d2h = 8 * n
    else:
        rows = solver.rows
        # a rank reads b and writes x of its own rows only: with a contiguous
        # (block) slab each GPU moves 1/N of b and x over its own PCIe link
        if rows.size and rows[-1] - rows[0] + 1 == rows.size:
            sl = slice(int(rows[0]), int(rows[-1]) + 1)
        else:
            sl = slice(0, n)
        with torch.cuda.stream(stream):  # copy -> all-reduce -> solve -> copy, ordered on one stream
            for _ in range(args.e2e_steps + 1):
                torch.distributed.barrier()
                t1 = time.perf_counter()
                db[sl].copy_(hb[sl], non_blocking=True)
                one_solve()
                plan.synchronize()
                hx[sl].copy_(dx[sl], non_blocking=False)
                t_e2e.append(time.perf_counter() - t1)
        t_e2e = t_e2e[1:]
        h2d_rank = 8 * (sl.stop - sl.start)
        d2h = 8 * (sl.stop - sl.start)
    e2e_s = statistics.mean(t_e2e)
    if ws > 1:
        t = torch.tensor([e2e_s], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return

    # ---- correctness against the C oracle -----------------------------------
    import oracle
    from paper_2012_06959_b200 import compare_solutions, residual_norm, residual_norm_2

    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_solve(l, b, 1, 0)
        x_ref = cpu["x"]
    else:
        x_ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    cmp = compare_solutions(x_dev, x_ref, 1e-12)
    res_inf = residual_norm(l, x_dev, b)[1]
    res_2 = residual_norm_2(l, x_dev, b)

    peak, peak_kind = measured_peaks()
    # N > 1: the whole job's bytes over the slowest rank's kernel, against N HBMs
    peak = peak * ws
    achieved = alg / (kern * 1e-3) / 1e9
    traffic = None
    tr = ROOT / "profiles" / "traffic.json"
    if tr.exists():
        try:
            traffic = json.loads(tr.read_text()).get(f"{args.config}/{args.precision}/{info['executor']}")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC,
        "value": flops / (ms * 1e-3) / 1e9,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "us_per_solve": ms * 1e3,
        "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {
            "workload": args.config,
            "n": n,
            "nnz": nnz,
            "n_levels": info["n_levels"],
            "rhs": "ones",
            "precision": args.precision,
            "executor": info["executor"],
            "method": _method(args.config, args.precision, info["executor"]),
            "parallelism": (f"column-block x{ws} ({partition.kind} partition), IPC peer segments" if ws > 1
                            else "single GPU"),
            "l2": (f"flushed: 256 MB scratch write between timed solves (solve inputs {alg / 1e6:.0f} MB vs "
                   f"{l2_bytes / 1e6:.0f} MB L2)") if flush else
                  f"back-to-back: solve inputs {alg / 1e6:.0f} MB vs {l2_bytes / 1e6:.0f} MB L2",
        },
        "timing": {
            "repeats": args.steps,
            "mean_ms": ms,
            "min_ms": min(per_solve),
            "max_ms": max(per_solve),
            "per_solve_sample": len(per_solve),
            "kernel_mean_ms": kern,
            "kernel_min_ms": min(kernel_ms) if kernel_ms else None,
            "l2_warm_ms": warm,
            "setup_ms": setup_s * 1e3,
            # the paper's protocol sums analysis and solve (
            # the reference's mean_combined_time, cli.py:199-202)
            "combined_ms": setup_s * 1e3 + ms,
        },
        "roofline": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": traffic,
            "peak_kind": peak_kind,
            "algorithmic_bytes": alg,
            "kernel_ms": kern,
        },
        "e2e": {
            "value": flops / e2e_s / 1e9,
            "unit": UNIT,
            "h2d_bytes_per_step": 8 * n if ws == 1 else h2d_rank * ws,
            "d2h_bytes_per_step": d2h if ws == 1 else d2h * ws,
            "ms_per_step": e2e_s * 1e3,
            "path": ("sptrsv_solve (C ABI, pinned host b/x" +
                     {1: ", band-granular H2D/D2H overlapping the kernel)",
                      2: ", zero-copy: the kernel reads b and writes x over PCIe in 128-byte lines)"}.get(
                         e2e_streamed, ")"))
            if ws == 1 else "per rank: H2D of its rows of b, solve, D2H of its rows of x (pinned)",
        },
        "cpu_baseline": None if cpu is None else {
            "value": flops / cpu["seconds"] / 1e9,
            "unit": UNIT,
            "cores": 1,
            "kind": "port",
            "sample": f"full {args.config} solve_serial (C port of reference.py:20-35), 1 rep",
            "seconds": cpu["seconds"],
        },
        "gpu_launches": args.steps * int(plan.synchronize().get("launches", 1)),
        "clocks": clocks.summary(),
        "correctness": {
            "max_rel_err_vs_oracle": cmp.max_rel_error,
            "bitwise_equal_oracle": bool(x_dev.tobytes() == x_ref.tobytes()),
            "residual_inf_rel": res_inf,
            "residual_2_rel": res_2,
        },
        "setup_ms": setup_s * 1e3,
        "generate_s": gen_s,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
