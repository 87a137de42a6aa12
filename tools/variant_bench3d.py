"""Stencil3d kernel time on lap3d-128 (fast + exact) for the library in SPTRSV_LIB (or the default)."""
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2012_06959_b200 import _native, synth  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 128
l = synth.lap3d(nx)
b = np.ones(l.n)
res = {"lib": os.environ.get("SPTRSV_LIB", "default")}
for prec in ("fast", "exact"):
    p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=prec, executor="stencil", timeout=30.0)
    p.solve(b)
    ks = [p.solve(b)[1]["kernel_ms"] for _ in range(10)]
    res[prec] = round(min(ks), 4)
    res[prec + "_median"] = round(float(np.median(ks)), 4)
    p.close()
print(json.dumps(res), flush=True)
