"""Probe the executors on shapes that isolate one cost at a time (GPU).

    python tools/chains_probe.py [--variants] [--cases ...]

Prints one JSON line per case: kernel ms, per-step ns, device spins; with
--variants also the chains kernel with parts of the step switched off
(probe_flags) and per-phase clock64 stamps of one warp.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2012_06959_b200 import _native, synth  # noqa: E402

NO_B, NO_STORE_X, NO_WAIT, CLOCK = 1, 2, 4, 16


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
    rec = {
        "case": name, "executor": info["executor"], "precision": precision, "flags": kw.get("probe_flags", 0),
        "n": l.n, "nnz": l.nnz, "kernel_ms": round(k, 4), "ns_per_step": round(k * 1e6 / max(steps, 1), 1),
        "steps": steps, "tasks": info["chain_tasks"], "spins": int(np.median(sp)), "setup_s": round(setup, 2),
    }
    if kw.get("probe_flags", 0) & CLOCK:
        st = plan.probe_stamps()
        d = np.diff(st, axis=1)
        step = np.diff(st[:, 0])
        rec["cycles"] = {
            "wait": float(np.median(d[:, 0])), "compute": float(np.median(d[:, 1])),
            "stores+prefetch": float(np.median(d[:, 2])), "syncwarp": float(np.median(d[:, 3])),
            "step": float(np.median(step)),
        }
    print(json.dumps(rec), flush=True)
    plan.close()


def main():
    variants = "--variants" in sys.argv
    cases = {
        "1task": ("lap2d 65536x32 (1 task, no mailboxes)", lambda: synth.lap2d(65536, 32)),
        "32task": ("lap2d 4096x1024 (32 tasks)", lambda: synth.lap2d(4096, 1024)),
        "full": ("lap2d 4096x4096", lambda: synth.lap2d(4096)),
    }
    pick = [a for a in sys.argv[1:] if a in cases] or list(cases)
    for key in pick:
        name, make = cases[key]
        l = make()
        if variants:
            for flags in (CLOCK, 0):
                run(name, l, "chains", "fast", probe_flags=flags)
        else:
            for prec in ("fast", "exact"):
                run(name, l, "stencil", prec)
                run(name, l, "chains", prec)
            run(name, l, "rows", "fast", reps=2)


if __name__ == "__main__":
    main()
