"""Band hand-over timeline of the 2D stencil executor (probe bit 256, globaltimer ns).

Band 2's chunk c needs band 1's chunk c + 4 (lane 31's blocks of steps
8(c+4) .. 8(c+4)+7 are columns 8c + 1 .. 8c + 8 of the row below). Prints the
medians over chunks 64..123 of: band 1's publish -> band 2's poller release,
poller release -> band 2's compute done waiting, and how long band 2's
compute actually waited.

    python tools/stencil_lag.py [ny] [fast|exact]
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2012_06959_b200 import _native, synth  # noqa: E402

ny = int(sys.argv[1]) if len(sys.argv) > 1 else 256
prec = sys.argv[2] if len(sys.argv) > 2 else "fast"
l = synth.lap2d(4096, ny)
p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=prec, executor="stencil", probe_flags=16 | 256)
b = np.ones(l.n)
p.solve(b)
_, st = p.solve(b)
s = p.probe_stamps(6).astype(np.float64)  # [64 chunks][6 slots]
pub, rel, wb, wa = s[:, 0], s[:, 1], s[:, 2], s[:, 3]
c = np.arange(60)
out = {
    "ny": ny, "precision": prec, "kernel_ms": round(st["kernel_ms"], 4),
    "producer_chunk_ns": float(np.median(np.diff(pub))),
    "consumer_chunk_ns": float(np.median(np.diff(wa))),
    "publish_to_poller_ns": float(np.median(rel[c] - pub[c + 4])),
    "poller_to_compute_ns": float(np.median(wa[c] - rel[c])),
    "compute_wait_ns": float(np.median(wa - wb)),
    "consumer_lag_ns": float(np.median(wa[c] - pub[c + 4])),
    "publish_of_needed_minus_wait_start_ns": float(np.median(pub[c + 4] - wb[c])),
}
print(json.dumps(out), flush=True)
