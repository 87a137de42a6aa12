"""One small solve per executor, checked against the C oracle, for
compute-sanitizer runs (tools/sanitize.sh):

    compute-sanitizer --tool racecheck python tools/sanitize_case.py stencil fast
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import oracle  # noqa: E402  (the checker)
import paper_2012_06959_b200 as sp  # noqa: E402
from paper_2012_06959_b200 import _native, synth  # noqa: E402

executor, precision = sys.argv[1], sys.argv[2]
mats = {
    "stencil": lambda: synth.lap2d(128, 192),       # 3 bands, 2D wavefront
    "stencil3d": lambda: synth.lap3d(32, 64, 8),    # 3D tiles
    "band": lambda: synth.banded(3000, 64, 0.5, 1),
    "rows": lambda: synth.rmat(11, 8, 0),
    "chains": lambda: synth.lap2d(40, 40),
    "push": lambda: synth.rmat(10, 8, 0),
}
l = mats[executor]()
ex = "stencil" if executor == "stencil3d" else executor
b = np.random.default_rng(0).uniform(-1, 1, l.n)
ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor=ex, timeout=600.0)
for _ in range(2):
    x, st = plan.solve(b)
ok = x.tobytes() == ref.tobytes() if precision == "exact" and ex != "push" else sp.compare_solutions(x, ref, 1e-12).within_tol
print(f"{executor} {precision}: n={l.n} executor={st['executor']} ok={ok}", flush=True)
plan.close()
sys.exit(0 if ok else 1)
