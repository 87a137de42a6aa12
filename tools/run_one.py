"""Run one executor on one matrix a few times (for ncu captures on the GPU box).

    python tools/run_one.py --config lap2d-4096 --executor stencil --precision fast --reps 2
    python tools/run_one.py --lap2d 4096 1024 --executor stencil
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2012_06959_b200 import _native, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default=None)
    ap.add_argument("--lap2d", type=int, nargs=2, default=None)
    ap.add_argument("--executor", default="auto")
    ap.add_argument("--precision", default="fast")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--spin-initial", type=int, default=1024)
    ap.add_argument("--spin-max-ns", type=int, default=64)
    args = ap.parse_args()
    if args.lap2d:
        l = synth.lap2d(*args.lap2d)
    else:
        l = synth.config_matrix(args.config or "lap2d-4096")
    t0 = time.perf_counter()
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=args.precision, executor=args.executor,
                              spin_initial=args.spin_initial, spin_max_ns=args.spin_max_ns)
    print("setup_s", round(time.perf_counter() - t0, 2), plan.info(), flush=True)
    b = np.ones(l.n)
    for _ in range(args.reps):
        _, st = plan.solve(b)
        print("kernel_ms", round(st["kernel_ms"], 4), "spins", st["spins"], flush=True)


if __name__ == "__main__":
    main()
