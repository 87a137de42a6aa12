"""f1 measurement: the paper's push engine
(Alg. 2: warp per column, fp64 atomics on shared left sums and in-degree
counters) on device memory and on unified memory with system-scope atomics
(the paper's Unified-Memory design), against this repo's pull executors, per
BASELINE config, fast mode, on one B200. Reports kernel ms (min of reps),
analysis (plan build) ms and analysis + solve, the paper's protocol
("we sum up the execution time of the analysis phase and the
solver phase").

    python tools/push_vs_pull.py [config ...]   (default: all four)
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2012_06959_b200 import _native, synth  # noqa: E402

configs = sys.argv[1:] or ["lap2d-4096", "lap3d-128", "rmat-4M", "banded-8M"]
for cfg in configs:
    l = synth.config_matrix(cfg)
    b = np.ones(l.n)
    row = {"config": cfg, "n": l.n, "nnz": l.nnz}
    for name, kw in (("pull", {"executor": "auto"}), ("push", {"executor": "push"}),
                     ("push_managed", {"executor": "push", "push_managed": True})):
        t0 = time.perf_counter()
        p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="fast", timeout=120.0, **kw)
        setup_ms = (time.perf_counter() - t0) * 1e3
        ks = []
        reps = 2 if cfg == "banded-8M" and name != "pull" else 5
        for _ in range(reps):
            _, st = p.solve(b)
            ks.append(st["kernel_ms"])
        row[name] = {"executor": st["executor"], "kernel_ms": round(min(ks), 4), "setup_ms": round(setup_ms, 1),
                     "analysis_plus_solve_ms": round(setup_ms + min(ks), 1)}
        p.close()
    row["pull_speedup_vs_push"] = round(row["push"]["kernel_ms"] / row["pull"]["kernel_ms"], 1)
    row["pull_speedup_vs_push_managed"] = round(row["push_managed"]["kernel_ms"] / row["pull"]["kernel_ms"], 1)
    print(json.dumps(row), flush=True)
