"""Count exact-mode IEEE-division fallbacks of the stencil kernel (probe bit 128)."""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2012_06959_b200 import _native, synth  # noqa: E402

for ny in (64, 4096):
    l = synth.lap2d(4096, ny)
    p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="exact", executor="stencil",
                           probe_flags=128)
    _, st = p.solve(np.ones(l.n))
    _, st = p.solve(np.ones(l.n))
    print(json.dumps({"ny": ny, "fallback_blocks": st["remote_reads"], "kernel_ms": st["kernel_ms"]}), flush=True)
    p.close()
