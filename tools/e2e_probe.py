"""e2e of the host-buffer solve on lap2d-4096 (pinned b/x): overlapped band copies
(streamed_io=True) vs copy-in / solve / copy-out."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2012_06959_b200 import _native, synth  # noqa: E402

l = synth.config_matrix("lap2d-4096")
out = []
hb = torch.ones(l.n, dtype=torch.float64).pin_memory().numpy()
hx = torch.empty(l.n, dtype=torch.float64).pin_memory().numpy()
for streamed in (True, False):
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="fast", executor="stencil",
                              streamed_io=streamed)
    plan.solve(hb, out=hx)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        _, st = plan.solve(hb, out=hx)
        ts.append(time.perf_counter() - t0)
    out.append({"streamed": streamed, "e2e_ms": round(min(ts) * 1e3, 3), "kernel_ms": round(st["kernel_ms"], 3),
                "mode": st["streamed_io"]})
    plan.close()
print(json.dumps(out), flush=True)
