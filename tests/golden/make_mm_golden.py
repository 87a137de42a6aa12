"""Matrix Market golden fixtures from the REFERENCE reader (this container only).

    python tests/golden/make_mm_golden.py

Each case is a Matrix Market text and the reference's parse_matrix_market
CSC arrays (and its read of the lower triangle where that is valid). The
.npz is committed; tests never read /root/reference.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from sptrsv import mmio as ref_mmio  # noqa: E402
from sptrsv.matrix import DiagonalPolicy, extract_lower_triangular  # noqa: E402

HERE = Path(__file__).resolve().parent


def cases() -> dict[str, str]:
    rng = np.random.default_rng(5)
    out = {
        "general_dups": "%%MatrixMarket matrix coordinate real general\n% c\n3 3 6\n1 1 2.0\n2 1 0.1\n2 1 0.2\n"
                        "2 1 0.3000000000000001\n3 3 1e-300\n2 2 -0.0\n",
        "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n4 4 5\n1 1 4\n2 1 -1\n2 2 4\n3 2 -1\n4 4 2.5\n",
        "pattern": "%%MatrixMarket matrix coordinate pattern general\n3 3 4\n1 1\n2 2\n3 3\n3 1\n",
        "integer": "%%MatrixMarket matrix coordinate integer general\n2 2 3\n1 1 7\n2 1 -3\n2 2 5\n",
        "empty": "%%MatrixMarket matrix coordinate real general\n5 5 0\n",
    }
    # a larger random lower-heavy file with duplicates, shuffled entries, blank/comment lines
    n, m = 400, 4000
    r = rng.integers(0, n, m)
    c = rng.integers(0, n, m)
    r, c = np.maximum(r, c), np.minimum(r, c)
    r = np.concatenate([r, np.arange(n), r[:300]])
    c = np.concatenate([c, np.arange(n), c[:300]])
    v = np.concatenate([rng.uniform(-1, 1, m), 5.0 + rng.random(n), rng.uniform(-1, 1, 300)])
    perm = rng.permutation(r.size)
    lines = [f"{int(r[k]) + 1} {int(c[k]) + 1} {float(v[k])!r}" for k in perm]
    lines.insert(100, "")
    lines.insert(200, "% a comment in the body")
    out["random_dups"] = "%%MatrixMarket matrix coordinate real general\n" + f"{n} {n} {r.size}\n" + \
        "\n".join(lines) + "\n"
    return out


def main():
    data = {}
    for name, text in cases().items():
        a = ref_mmio.parse_matrix_market(text.encode())
        data[f"{name}/text"] = np.frombuffer(text.encode(), dtype=np.uint8)
        data[f"{name}/col_ptr"] = a.col_ptr
        data[f"{name}/row_idx"] = a.row_idx
        data[f"{name}/values"] = a.values
        try:
            low = extract_lower_triangular(a, DiagonalPolicy.INSERT_UNIT)
            data[f"{name}/lower_col_ptr"] = low.col_ptr
            data[f"{name}/lower_row_idx"] = low.row_idx
            data[f"{name}/lower_values"] = low.values
        except Exception as exc:  # recorded for the test
            data[f"{name}/lower_error"] = np.frombuffer(type(exc).__name__.encode(), dtype=np.uint8)
    np.savez_compressed(HERE / "mm_cases.npz", **data)
    print("wrote", HERE / "mm_cases.npz", len(data))


if __name__ == "__main__":
    main()
