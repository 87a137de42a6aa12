"""Batched right-hand sides (f4): kernel time of k stacked solves against one
solve, lap2d-4096 (or argv[1] = config), both precisions.

    python tools/solve_many_bench.py [config] [k ...]
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2012_06959_b200 import _native, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "lap2d-4096"
ks = [int(v) for v in sys.argv[2:]] or [2, 4, 8, 16]
l = synth.config_matrix(cfg)
for prec in ("fast", "exact"):
    p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=prec, timeout=60.0)
    b = np.ones(l.n)
    p.solve(b)
    one = min(p.solve(b)[1]["kernel_ms"] for _ in range(5))
    row = {"config": cfg, "precision": prec, "executor": p.info()["executor"], "one_ms": round(one, 4)}
    for k in ks:
        bs = np.random.default_rng(k).uniform(-1, 1, (k, l.n))
        p.solve_many(bs)
        t = min(p.solve_many(bs)[1]["kernel_ms"] for _ in range(3))
        row[f"k{k}_ms"] = round(t, 4)
        row[f"k{k}_vs_one"] = round(t / one, 2)
    p.close()
    print(json.dumps(row), flush=True)
