"""Per-band timeline of the 2D stencil executor on lap2d-4096 (probe bit 16):
band start, first chunk ready and end (us from the earliest start), plus the
medians of the consecutive differences, for the library in SPTRSV_LIB.

    python tools/stencil_timeline.py [fast|exact] [ny]
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2012_06959_b200 import _native, synth  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fast"
ny = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
l = synth.lap2d(4096, ny)
p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=prec, executor="stencil", probe_flags=16)
b = np.ones(l.n)
p.solve(b)
ks = []
for _ in range(3):
    _, st = p.solve(b)
    ks.append(st["kernel_ms"])
nt = (ny + 63) // 64
ts = p.probe_tasks(nt).astype(np.float64)
rel = (ts - ts[:, 0].min()) / 1e3
p.close()
print(json.dumps({
    "lib": os.environ.get("SPTRSV_LIB", "default"), "precision": prec, "ny": ny, "kernel_ms": round(min(ks), 4),
    "ready_us": [round(v, 1) for v in rel[:, 1]],
    "end_us": [round(v, 1) for v in rel[:, 2]],
    "run_us": [round(v, 1) for v in rel[:, 2] - rel[:, 1]],
    "ready_gap_median": round(float(np.median(np.diff(rel[:, 1]))), 2) if nt > 1 else None,
    "run_median": round(float(np.median(rel[:, 2] - rel[:, 1])), 1),
}), flush=True)
