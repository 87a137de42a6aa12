"""Stencil executor experiments (GPU): per-band step time vs band count, and
probe variants that switch parts of the step off (timings only; results wrong).

    python tools/stencil_exp.py [--variants]
"""

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2012_06959_b200 import _native, synth  # noqa: E402

NO_AWAIT, NO_FENCE, NO_WAITB, NO_PREFETCH, NO_STORE = 1, 2, 4, 8, 32


def run(ny, probe=0, precision="fast"):
    l = synth.lap2d(4096, ny)
    p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor="stencil",
                           probe_flags=probe, timeout=5.0)
    b = np.ones(l.n)
    try:
        p.solve(b)
        ks, sp = [], []
        for _ in range(3):
            _, st = p.solve(b)
            ks.append(st["kernel_ms"])
            sp.append(st["spins"])
    except Exception as e:  # a probe variant may trip the watchdog
        print(json.dumps({"ny": ny, "probe": probe, "error": str(e)[:80]}), flush=True)
        return
    finally:
        p.close()
    bands = (ny + 63) // 64
    steps = 1024 + 31
    rec = {"ny": ny, "bands": bands, "probe": probe, "precision": precision, "kernel_ms": round(min(ks), 4),
           "spins": sp[-1], "ns_per_band_step": round(min(ks) * 1e6 / (steps + (bands - 1) * 32), 1)}
    print(json.dumps(rec), flush=True)


def clock_profile(ny=64, precision="fast"):
    l = synth.lap2d(4096, ny)
    p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor="stencil",
                           probe_flags=16)
    b = np.ones(l.n)
    p.solve(b)
    p.solve(b)
    st = p.probe_stamps(6)
    d = np.diff(st, axis=1)
    names = ["shfl+inbox", "compute", "stores", "prefetch+issue", "stage(next)"]
    out = {nm: float(np.median(d[:, k])) for k, nm in enumerate(names)}
    out["step"] = float(np.median(np.diff(st[:, 0])))
    print(json.dumps({"clock_cycles": out, "precision": precision}), flush=True)
    p.close()


def main():
    if "--clock" in sys.argv:
        clock_profile(64, "fast")
        clock_profile(64, "exact")
        return
    if "--variants" in sys.argv:
        for probe in (0, NO_FENCE, NO_AWAIT, NO_WAITB, NO_PREFETCH | NO_WAITB, NO_STORE,
                      NO_AWAIT | NO_FENCE | NO_WAITB | NO_PREFETCH | NO_STORE):
            run(64, probe)
        return
    for ny in (64, 128, 256, 1024, 4096):
        run(ny)
    run(4096, precision="exact")


if __name__ == "__main__":
    main()
