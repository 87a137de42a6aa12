"""Warp-stall samples of a warp-specialised kernel split by warp role.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_roles.py src.csv paper_2012_06959_b200/csrc/stencil.cu

Per CUDA source line ncu reports the warp-stall sampling counts of the SASS
it compiled to; lines of the kernel file are attributed to the device
function (role) that contains them (by definition line in the given source
file, which must be the one the profiled library was built from) and inlined
helpers from other files are reported per file. Prints
samples and the top stall reasons per role (the north star's "stall
breakdown on flag polling").
"""

from __future__ import annotations

import csv
import re
import sys
from collections import defaultdict


def roles_of(src_path: str) -> list[tuple[int, str]]:
    """(definition line, name) of every __device__/__global__ function of the file."""
    pat = re.compile(r"^(?:template <[^>]*>\s*)?__(?:device|global)__[^(]*?\b(\w+)\s*\(")
    return sorted((no, m.group(1)) for no, line in enumerate(open(src_path), start=1) if (m := pat.match(line)))


def main():
    # the source file must be the one the profiled library was built from
    csv_path, src_path = sys.argv[1], sys.argv[2]
    src_name = src_path.split("/")[-1]
    starts = roles_of(src_path)

    def role_at(line: int) -> str:
        name = "file scope"
        for no, fn in starts:
            if no <= line:
                name = fn
        return name

    samples = defaultdict(int)
    reasons = defaultdict(lambda: defaultdict(int))
    cur_file, header = None, None
    for row in csv.reader(open(csv_path)):
        if not row:
            continue
        if row[0] == "File Path":
            cur_file = row[1].split("/")[-1]
            header = None
            continue
        if row[0] == "Line No":
            header = {h: i for i, h in enumerate(row) if h not in header_seen(row, i)}
            continue
        if header is None or not row[0].isdigit():
            continue
        col = header.get("Warp Stall Sampling (All Samples)")
        if col is None or col >= len(row) or not row[col].replace(".", "").isdigit():
            continue
        s = int(float(row[col]))
        if not s:
            continue
        key = role_at(int(row[0])) if cur_file == src_name else f"{cur_file} (inlined helpers)"
        samples[key] += s
        for h, i in header.items():
            if h.startswith("stall_") and "Not Issued" not in h and i < len(row):
                try:
                    reasons[key][h[6:]] += int(float(row[i] or 0))
                except ValueError:
                    pass
    total = sum(samples.values()) or 1
    for key, s in sorted(samples.items(), key=lambda kv: -kv[1]):
        top = sorted(reasons[key].items(), key=lambda kv: -kv[1])[:5]
        print(f"{key:38s} {s:7d} samples {100.0 * s / total:5.1f}%  " + ", ".join(f"{k} {v}" for k, v in top))


def header_seen(row, i):
    """Duplicate column names (the cuda,sass view repeats "Source"): keep the first."""
    return set(row[:i])


if __name__ == "__main__":
    main()
