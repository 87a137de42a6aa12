"""Per-band timeline of a streamed host-buffer solve (lap2d-4096, pinned b/x):
kernel-relative start / first-chunk-ready / end per band, to see whether the
bands wait on the b copies or on each other."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2012_06959_b200 import _native, synth  # noqa: E402

l = synth.lap2d(4096, 4096)
hb = torch.ones(l.n, dtype=torch.float64).pin_memory().numpy()
hx = torch.empty(l.n, dtype=torch.float64).pin_memory().numpy()
import os
p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="fast", executor="stencil", probe_flags=16,
                       timeout=float(os.environ.get("TL_TIMEOUT", 60)))
for _ in range(3):
    _, st = p.solve(hb, out=hx)
ts = p.probe_tasks(64).astype(np.float64)
t0 = ts[:, 0].min()
rel = (ts - t0) / 1e3
print(json.dumps({"e2e_ms": st.get("e2e_ms"), "kernel_ms": st["kernel_ms"], "streamed": st.get("streamed_io"),
                  "ready_us": [round(v, 1) for v in rel[::4, 1]], "end_us": [round(v, 1) for v in rel[::4, 2]],
                  "ready_last": round(rel[-1, 1], 1), "end_last": round(rel[-1, 2], 1)}))
p.close()
