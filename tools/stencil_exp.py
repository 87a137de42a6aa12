"""Stencil executor experiments (GPU): per-band step time vs band count.

    python tools/stencil_exp.py
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


def main():
    for ny in (64, 128, 256, 1024, 4096):
        run(ny)
    run(4096, precision="exact")


if __name__ == "__main__":
    main()
