"""Probe the executors on shapes that isolate one cost at a time (GPU).

    python tools/chains_probe.py [--quick]

Prints one JSON line per case: kernel ms, per-step ns, device spins.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2012_06959_b200 import _native, synth  # noqa: E402


def run(name, l, executor, precision, reps=5, **kw):
    t0 = time.perf_counter()
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor=executor, **kw)
    setup = time.perf_counter() - t0
    info = plan.info()
    b = np.ones(l.n)
    plan.solve(b)
    ks, sp = [], []
    for _ in range(reps):
        _, st = plan.solve(b)
        ks.append(st["kernel_ms"])
        sp.append(st["spins"])
    k = min(ks)
    steps = info["chain_max_task_steps"] or info["n_levels"]
    print(json.dumps({
        "case": name, "executor": info["executor"], "precision": precision, "n": l.n, "nnz": l.nnz,
        "kernel_ms": round(k, 4), "ns_per_step": round(k * 1e6 / max(steps, 1), 1), "steps": steps,
        "tasks": info["chain_tasks"], "spins": int(np.median(sp)), "setup_s": round(setup, 2),
        "deps": {x: info[x] for x in ("deps_register", "deps_ring", "deps_mailbox")},
    }), flush=True)
    plan.close()


def main():
    quick = "--quick" in sys.argv
    cases = [
        ("lap2d 32x65536 (1 task, no mailboxes)", synth.lap2d(65536, 32)),
        ("lap2d 64x65536 (2 tasks)", synth.lap2d(65536, 64)),
        ("lap2d 1024x4096 (32 tasks)", synth.lap2d(4096, 1024)),
        ("lap2d 4096x4096", synth.lap2d(4096)),
    ]
    if quick:
        cases = cases[:2]
    for name, l in cases:
        for prec in ("fast", "exact"):
            run(name, l, "chains", prec)
        run(name, l, "rows", "fast", reps=2)
        run(name + " rows spin-only", l, "rows", "fast", reps=2, spin_initial=1 << 30)


if __name__ == "__main__":
    main()
