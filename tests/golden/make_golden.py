"""Generate golden fixtures by running the REFERENCE package (this container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports the reference read-only from /root/reference/pkg/src and records, per
case: the CSC arrays, a right-hand side, the reference's ``solve_serial`` x,
``compute_in_degrees`` and ``compute_level_schedule`` output. The .npz files are
committed; nothing at test time reads /root/reference (it does not exist on
the GPU box).

Cases mirror the reference's own fixtures and tests:
* worked_3x3 / identity4 / bidiagonal / fan-out / stored-zero / shared-parent
  (conftest.py:7-34, test_analysis.py:38-82, test_reference.py:14-35)
* random_instance(seed) with random_rhs(n, seed) (conftest.py:25-34)
* the criterion-1 grid instances k = 0..23 (test_acceptance.py:59-96)
* BLOCK_DIAGONAL 4096/32 seed 2 (test_engine.py:121-132)
* lap2d-256: BASELINE configs[0], solved by the reference CPU path.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import sptrsv as ref  # noqa: E402

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))


def random_instance(seed, n_lo=16, n_hi=512, d_lo=0.001, d_hi=0.3):
    rng = np.random.default_rng(seed)
    n = int(np.exp(rng.uniform(np.log(n_lo), np.log(n_hi))))
    density = float(np.exp(rng.uniform(np.log(d_lo), np.log(d_hi))))
    return ref.random_lower(n, density, seed)


def random_rhs(n, seed):
    return np.random.default_rng((seed, 77)).uniform(-2.0, 2.0, size=n)


def record(name, l, b, out):
    x = ref.solve_serial(l, b) if b is not None else None
    sched = ref.compute_level_schedule(l)
    case = {
        "n": np.array(l.n),
        "col_ptr": l.col_ptr,
        "row_idx": l.row_idx,
        "values": l.values,
        "in_degree": ref.compute_in_degrees(l),
        "level_of": sched.level_of,
        "n_levels": np.array(sched.n_levels),
    }
    if b is not None:
        case["b"] = b
        case["x"] = x
    out[name] = case


def main():
    cases: dict[str, dict] = {}
    l3 = ref.CscMatrix.from_entries(3, {(0, 0): 2.0, (1, 0): 1.0, (1, 1): 1.0, (2, 1): 3.0, (2, 2): 4.0})
    record("worked_3x3", l3, np.array([2.0, 2.0, 7.0]), cases)
    eye = ref.generate_synthetic(ref.SyntheticSpec(ref.SyntheticKind.DIAGONAL, 4))
    record("identity4", eye, np.array([3.0, -1.0, 0.5, 8.0]), cases)
    bi = ref.generate_synthetic(ref.SyntheticSpec(ref.SyntheticKind.BIDIAGONAL, 4))
    record("bidiagonal4", bi, np.array([1.0, 0.0, 0.0, 0.0]), cases)
    bi1000 = ref.generate_synthetic(ref.SyntheticSpec(ref.SyntheticKind.BIDIAGONAL, 1000))
    record("bidiagonal1000", bi1000, random_rhs(1000, 3), cases)
    fan = {(j, j): 1.0 for j in range(8)}
    fan.update({(1, 0): 0.5, (3, 0): 0.5, (5, 0): 0.5, (7, 0): 0.5})
    record("fanout8", ref.CscMatrix.from_entries(8, fan), np.arange(8.0) - 3.0, cases)
    zero = ref.CscMatrix.from_entries(2, {(0, 0): 1.0, (1, 0): 0.0, (1, 1): 1.0})
    record("stored_zero", zero, np.array([1.0, 2.0]), cases)
    par = {(j, j): 1.0 for j in range(6)}
    par.update({(1, 0): 1.0, (3, 0): 1.0, (5, 0): 1.0})
    record("shared_parent", ref.CscMatrix.from_entries(6, par), np.ones(6), cases)
    rng = np.random.default_rng(11)
    vals = rng.uniform(1.0, 3.0, size=20) * rng.choice([-1.0, 1.0], size=20)
    diag = ref.CscMatrix(n=20, col_ptr=np.arange(21), row_idx=np.arange(20), values=vals)
    record("diagonal20", diag, rng.uniform(-5.0, 5.0, size=20), cases)
    for seed in range(12):
        l = random_instance(seed)
        record(f"random_{seed}", l, random_rhs(l.n, seed), cases)
    for k in range(24):  # criterion-1 instance generator (test_acceptance.py:66-75)
        g = [(p, t, w) for p in (1, 2, 4, 8) for t in (1, 4, 8) for w in (1, 4)][k]
        r = np.random.default_rng((2024, k))
        n_lo = max(16, g[0] * g[1])
        n = int(float(np.exp(r.uniform(np.log(n_lo), np.log(2000)))))
        density = float(np.exp(r.uniform(np.log(0.001), np.log(0.3))))
        l = ref.random_lower(n, density, seed=90_000 + k)
        if l.nnz <= 40_000:  # keep the fixture file small
            record(f"criterion1_{k}", l, random_rhs(n, seed=k), cases)
    bd = ref.generate_synthetic(ref.SyntheticSpec(ref.SyntheticKind.BLOCK_DIAGONAL, 4096, seed=2, block=32))
    record("blockdiag4096", bd, random_rhs(4096, 5), cases)

    small = {k: v for k, v in cases.items()}
    np.savez_compressed(HERE / "reference_cases.npz", **{f"{k}/{f}": v for k, c in small.items() for f, v in c.items()})

    # lap2d-256 (BASELINE configs[0]) built by our generator, solved by the reference
    from paper_2012_06959_b200 import synth

    mine = synth.lap2d(256)
    l = ref.CscMatrix(n=mine.n, col_ptr=mine.col_ptr, row_idx=mine.row_idx, values=mine.values)
    digest = hashlib.sha256(mine.col_ptr.tobytes() + mine.row_idx.tobytes() + mine.values.tobytes()).hexdigest()
    b_ones = np.ones(l.n)
    b_rand = np.random.default_rng((0, 1)).uniform(-1.0, 1.0, size=l.n)  # cli.py:141-142, seed 0
    sched = ref.compute_level_schedule(l)
    np.savez_compressed(
        HERE / "lap2d_256.npz",
        sha256=np.array(digest),
        x_ones=ref.solve_serial(l, b_ones),
        b_rand=b_rand,
        x_rand=ref.solve_serial(l, b_rand),
        in_degree=ref.compute_in_degrees(l).astype(np.int8),
        level_of=sched.level_of.astype(np.int16),
        n_levels=np.array(sched.n_levels),
    )
    print(f"{len(cases)} reference cases + lap2d_256 (n_levels={sched.n_levels}, sha256={digest[:16]}...)")


if __name__ == "__main__":
    main()
