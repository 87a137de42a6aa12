"""Per-tile timeline of the 3D stencil executor on lap3d-128 (probe bit 16):
tile start, first chunk ready and end (us from the earliest start) in (Z, Y)
order, plus the z-hop lag (ready/end of tile (Y, Z) minus tile (Y, Z-1)) and
the tile run time, for the library in SPTRSV_LIB.

    python tools/stencil3d_timeline.py [fast|exact] [n]
"""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2012_06959_b200 import _native, synth  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "fast"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
l = synth.lap3d(n)
p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=prec, executor="stencil", probe_flags=16)
b = np.ones(l.n)
p.solve(b)
ks = []
for _ in range(3):
    _, st = p.solve(b)
    ks.append(st["kernel_ms"])
nyt, nzt = (n + 31) // 32, (n + 3) // 4
nt = nyt * nzt
ts = p.probe_tasks(nt).astype(np.float64)
rel = (ts - ts[:, 0].min()) / 1e3
p.close()
ready = rel[:, 1].reshape(nzt, nyt)
end = rel[:, 2].reshape(nzt, nyt)
print(json.dumps({
    "lib": os.environ.get("SPTRSV_LIB", "default"), "precision": prec, "n": n, "kernel_ms": round(min(ks), 4),
    "start_max_us": round(float(rel[:, 0].max()), 1),
    "ready_Y0_us": [round(v, 1) for v in ready[:, 0]],
    "end_Y0_us": [round(v, 1) for v in end[:, 0]],
    "ready_Z0_us": [round(v, 1) for v in ready[0]],
    "end_Z0_us": [round(v, 1) for v in end[0]],
    "zhop_ready_median": round(float(np.median(np.diff(ready[:, 0]))), 2),
    "zhop_end_median": round(float(np.median(np.diff(end[:, 0]))), 2),
    "yhop_end_median": round(float(np.median(np.diff(end, axis=1))), 2),
    "run_median": round(float(np.median(end - ready)), 1),
}), flush=True)
