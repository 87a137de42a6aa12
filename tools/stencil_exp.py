"""Stencil executor experiments (GPU): per-band step time vs band count, and
per-chunk clock stamps of the compute and loader warps (--clock).

    python tools/stencil_exp.py [--clock]
"""

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2012_06959_b200 import _native, synth  # noqa: E402


def run(ny, precision="fast", nx=4096):
    l = synth.lap2d(nx, ny)
    p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor="stencil", timeout=20.0)
    b = np.ones(l.n)
    try:
        p.solve(b)
        ks, sp = [], []
        for _ in range(3):
            _, st = p.solve(b)
            ks.append(st["kernel_ms"])
            sp.append(st["spins"])
    finally:
        p.close()
    bands = (ny + 63) // 64
    steps = nx // 4 + 31
    print(json.dumps({"ny": ny, "bands": bands, "precision": precision, "kernel_ms": round(min(ks), 4),
                      "spins": sp[-1], "ns_per_band_step": round(min(ks) * 1e6 / (steps + (bands - 1) * 32), 1)}),
          flush=True)


def clock(ny=64, precision="fast", extra=0):
    l = synth.lap2d(4096, ny)
    p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor="stencil",
                           probe_flags=16 | extra)
    b = np.ones(l.n)
    p.solve(b)
    p.solve(b)
    st = p.probe_stamps(6).astype(np.float64)
    # compute: [0] before waiting for the chunk, [1] after; loader: [2] loop top, [3] before settle,
    # [4] after settle, [5] after hand-over
    rec = {
        "compute_chunk_period": float(np.median(np.diff(st[:, 1]))),
        "compute_wait": float(np.median(st[:, 1] - st[:, 0])),
        "loader_chunk_period": float(np.median(np.diff(st[:, 2]))),
        "loader_issue": float(np.median(st[:, 3] - st[:, 2])),
        "loader_settle": float(np.median(st[:, 4] - st[:, 3])),
        "loader_handover": float(np.median(st[:, 5] - st[:, 4])),
        "loader_ahead_of_compute": float(np.median(st[:, 1] - st[:, 5])),
    }
    _, stt = p.solve(b)
    print(json.dumps({"ny": ny, "precision": precision, "probe": extra, "kernel_ms": round(stt["kernel_ms"], 4),
                      "cycles": rec}), flush=True)
    p.close()


def tasks(ny=4096, precision="fast"):
    """Per-band timeline: start, first chunk ready, end (us from kernel start)."""
    l = synth.lap2d(4096, ny)
    p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor="stencil",
                           probe_flags=16)
    b = np.ones(l.n)
    p.solve(b)
    _, st = p.solve(b)
    nt = (ny + 63) // 64
    ts = p.probe_tasks(nt).astype(np.float64)
    t0 = ts[:, 0].min()
    rel = (ts - t0) / 1e3
    gaps = np.diff(rel[:, 2])
    print(json.dumps({"ny": ny, "precision": precision, "kernel_ms": round(st["kernel_ms"], 4),
                      "first_ready_us": [round(v, 1) for v in rel[:8, 1]],
                      "end_us": [round(v, 1) for v in rel[::max(1, nt // 16), 2]],
                      "band0_us": round(rel[0, 2] - rel[0, 1], 1),
                      "end_gap_us_median": round(float(np.median(gaps)), 2) if gaps.size else None,
                      "ready_gap_us_median": round(float(np.median(np.diff(rel[:, 1]))), 2) if nt > 1 else None}),
          flush=True)
    p.close()


def main():
    if "--tasks" in sys.argv:
        for ny in (64, 256, 4096):
            tasks(ny)
        tasks(4096, "exact")
        return
    if "--clock" in sys.argv:
        # probe bit 4: helper nap = bits 8.. (ns); bit 32: compute warp alone;
        # bits 12..15: compute ablation (1 no staging, 2 no loads, 4 no shfl, 8 no publish branch)
        clock(64)
        clock(256)
        clock(256, extra=64)  # band 1
        clock(4096, extra=64)
        return
    for ny in (64, 128, 256, 1024, 4096):
        run(ny)
    run(4096, precision="exact")


if __name__ == "__main__":
    main()
