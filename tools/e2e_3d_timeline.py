"""Per-tile timeline of a streamed host-buffer lap3d-128 solve: when each
z-slab's first tile became ready (its b arrived) and when the slab's last tile
ended, relative to the kernel start."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2012_06959_b200 import _native, synth  # noqa: E402

l = synth.lap3d(128)
hb = torch.ones(l.n, dtype=torch.float64).pin_memory().numpy()
hx = torch.empty(l.n, dtype=torch.float64).pin_memory().numpy()
p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="fast", executor="stencil", probe_flags=16,
                       timeout=10.0)
for _ in range(3):
    _, st = p.solve(hb, out=hx)
nt = 128
ts = p.probe_tasks(nt).astype(np.float64)
rel = (ts - ts[:, 0].min()) / 1e3
print(json.dumps({"e2e_ms": st["e2e_ms"], "kernel_ms": st["kernel_ms"],
                  "slab_ready_us": [round(v, 1) for v in rel[::4, 1][::4]],
                  "slab_end_us": [round(v, 1) for v in rel[3::4, 2][::4]],
                  "start_us": [round(v, 1) for v in rel[::16, 0]]}))
p.close()
