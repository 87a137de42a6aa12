import sys, json, numpy as np
sys.path.insert(0, '.')
from paper_2012_06959_b200 import _native, synth
for ny in (64, 128, 256, 1024, 4096):
    l = synth.lap2d(4096, ny)
    for prec in ("fast",):
        p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=prec, executor="stencil")
        b = np.ones(l.n); p.solve(b)
        ks=[]; sp=[]
        for _ in range(3):
            _, st = p.solve(b); ks.append(st["kernel_ms"]); sp.append(st["spins"])
        bands = (ny + 63)//64
        steps = 1024 + 31
        print(json.dumps({"ny": ny, "bands": bands, "kernel_ms": min(ks), "spins": sp, "ns_per_band_step": min(ks)*1e6/(steps + (bands-1)*32)}), flush=True)
        p.close()
