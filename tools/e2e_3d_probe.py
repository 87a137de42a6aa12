import sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2012_06959_b200 import _native, synth
l = synth.lap3d(128)
hb = torch.ones(l.n, dtype=torch.float64).pin_memory().numpy()
hx = torch.empty(l.n, dtype=torch.float64).pin_memory().numpy()
for streamed in ((True,) if len(sys.argv) > 1 else (True, False)):
    p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="fast", executor="stencil", streamed_io=streamed)
    res = []
    for _ in range(8):
        t = time.perf_counter(); _, st = p.solve(hb, out=hx); res.append(((time.perf_counter() - t) * 1e3, st["e2e_ms"], st["kernel_ms"], st["streamed_io"]))
    print(streamed, [tuple(round(v, 3) for v in r) for r in res[-3:]])
    p.close()
