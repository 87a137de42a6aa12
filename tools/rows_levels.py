"""Where the component pool's time goes, per level (probe bit 512: one
globaltimer stamp per row at its publish). For rmat-4M (or --config):
per-level completion time, the slowest levels, and for each level's last row
its dependency count and the delay between its newest dependency's publish
and its own ("row latency").

    python tools/rows_levels.py [--config rmat-4M] [--precision fast]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2012_06959_b200 import _native, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="rmat-4M")
ap.add_argument("--precision", default="fast")
args = ap.parse_args()
l = synth.config_matrix(args.config)
p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=args.precision, executor="rows",
                       probe_flags=512)
b = np.ones(l.n)
p.solve(b)
_, st = p.solve(b)
raw = np.empty(max(l.n, 6 * 64 + 3 * 1024), dtype=np.int64)
rc = p._lib.sptrsv_plan_probe_read(p._h, _native._ptr(raw, _native.C.c_int64), raw.size)
stamp = raw[: l.n].astype(np.float64)
level, _, _, nl = p.levels()
assert rc == 0
p.close()
t0 = stamp.min()
stamp = (stamp - t0) / 1e3  # us
# CSR of dependencies (row i depends on columns j < i)
cols = np.repeat(np.arange(l.n), np.diff(l.col_ptr))
rows = np.asarray(l.row_idx)
off = rows != cols
dep_row, dep_col = rows[off], cols[off]
deg = np.bincount(dep_row, minlength=l.n)
# newest dependency publish time per row
newest = np.full(l.n, -1.0)
np.maximum.at(newest, dep_row, stamp[dep_col])
lat = np.where(deg > 0, stamp - newest, np.nan)
done = np.full(nl, -np.inf)
np.maximum.at(done, level, stamp)
last_row = np.zeros(nl, dtype=np.int64)
order = np.lexsort((stamp, level))
lv_sorted = level[order]
ends = np.searchsorted(lv_sorted, np.arange(nl), side="right") - 1
last_row = order[ends]
dt = np.diff(np.concatenate([[0.0], done]))
worst = np.argsort(-dt)[:15]
print(json.dumps({
    "config": args.config, "kernel_ms": round(st["kernel_ms"], 4), "n_levels": int(nl),
    "level0_done_us": round(float(done[0]), 1), "last_done_us": round(float(done[-1]), 1),
    "dt_us_quantiles": [round(float(v), 2) for v in np.percentile(dt[1:], [10, 50, 90, 99])],
    "row_latency_us_quantiles_last_rows": [round(float(v), 2) for v in np.nanpercentile(lat[last_row[1:]], [10, 50, 90])],
    "last_row_deg_quantiles": [int(v) for v in np.percentile(deg[last_row[1:]], [10, 50, 90, 99])],
    "worst_levels": [{"L": int(L), "dt": round(float(dt[L]), 2), "rows": int((level == L).sum()),
                      "last_deg": int(deg[last_row[L]]), "last_lat": round(float(lat[last_row[L]]), 2)}
                     for L in worst],
    "sum_dt_by_last_deg": {k: round(float(dt[1:][m].sum()), 1) for k, m in {
        "<=32": deg[last_row[1:]] <= 32, "33-256": (deg[last_row[1:]] > 32) & (deg[last_row[1:]] <= 256),
        ">256": deg[last_row[1:]] > 256}.items()},
}), flush=True)
