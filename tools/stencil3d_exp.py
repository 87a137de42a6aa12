"""3D stencil executor timeline on lap3d-128: per-tile start / first-chunk-ready / end (us)."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2012_06959_b200 import _native, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
l = synth.lap3d(n)
for prec in ("fast", "exact"):
    p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=prec, executor="stencil", probe_flags=16)
    b = np.ones(l.n)
    p.solve(b)
    _, st = p.solve(b)
    nyt, nzt = (n + 31) // 32, (n + 3) // 4
    ts = p.probe_tasks(nyt * nzt).astype(np.float64)
    t0 = ts[:, 0].min()
    rel = (ts - t0) / 1e3
    grid = rel.reshape(nzt, nyt, 3)
    raw = p._probe_raw()
    pc = (raw[0:2 * nyt * nzt].reshape(-1, 2).astype(np.float64) - t0) / 1e3  # poller c0 done, compute c0 end
    pcg = pc.reshape(nzt, nyt, 2)
    print(json.dumps({"Y0_Z0..7": [[round(grid[z, 0, 1], 1), round(pcg[z, 0, 1], 1), round(pcg[z, 0, 0], 1)]
                                   for z in range(8)]}))
    print(json.dumps({"precision": prec, "kernel_ms": round(st["kernel_ms"], 4), "spins": st["spins"],
                      "ready_Y_at_Z0": [round(v, 1) for v in grid[0, :, 1]],
                      "ready_Z_at_Y0": [round(v, 1) for v in grid[::4, 0, 1]],
                      "end_Z_at_Y3": [round(v, 1) for v in grid[::4, -1, 2]],
                      "tile_duration_median": round(float(np.median(rel[:, 2] - rel[:, 1])), 1)}), flush=True)
    p.close()
