"""Multi-process host logic of the inter-GPU layer on CPU (gloo, world_size 2).

The device side (peer loads over NVLink) cannot run here; what is checked is
everything around it: both ranks agree on the partition, segment handles are
all-gathered in rank order, each rank's owned rows are disjoint and complete,
and x assembles from the per-rank pieces. The per-PE segments themselves are
exercised on one GPU with virtual PEs (tests/test_gpu_partitioned.py).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2012_06959_b200 import multi, synth


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, kind, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        l = synth.lap2d(16, 12)
        w = np.diff(np.asarray(l.col_ptr))  # entries per column: a skewed weight
        plan = multi.rank_partition(l.n, world, kind, tasks_per_pe=3, row_weight=w)
        # a fake 64-byte "IPC handle" per rank
        handle = bytes([rank]) * 64
        handles = multi.exchange_handles(handle)
        rows = multi.owned_rows(plan.owner_arr, rank)
        # each rank "solves" its rows: value = row index * 2 (stand-in for x)
        vals = rows.astype(np.float64) * 2.0
        gathered: list = [None] * world
        dist.all_gather_object(gathered, (rows, vals))
        x = multi.assemble_x(gathered, l.n)
        out_q.put((rank, [h[0] for h in handles], int(rows.size), bool(np.array_equal(x, np.arange(l.n) * 2.0))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["block", "round-robin", "nnz"])
def test_two_ranks_exchange_handles_and_assemble_x(kind):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    results.sort()
    for rank, handle_ids, n_rows, ok in results:
        assert handle_ids == [0, 1]  # rank order
        assert ok
    assert sum(r[2] for r in results) == 16 * 12


def test_assemble_rejects_overlap():
    with pytest.raises(ValueError):
        multi.assemble_x([(np.array([0, 1]), np.zeros(2)), (np.array([1]), np.zeros(1))], 2)


def test_rank_partition_is_deterministic():
    a = multi.rank_partition(1000, 8)
    b = multi.rank_partition(1000, 8)
    np.testing.assert_array_equal(a.owner_arr, b.owner_arr)
    assert np.bincount(a.owner_arr).tolist() == [125] * 8


def test_nnz_block_partition_balances_work():
    """Contiguous slabs of equal total weight (block_partition
    leaves rmat's power-law rows 8.4x imbalanced over 8 PEs)."""
    import paper_2012_06959_b200 as sp
    rng = np.random.default_rng(0)
    w = np.floor(rng.pareto(1.2, 200_000) + 1)  # power-law row weights
    w[:5000] *= 50  # a heavy head, like low-numbered rmat rows
    for pes in (2, 4, 8):
        blk = sp.block_partition(w.size, pes)
        nnz = sp.nnz_block_partition(w, pes)
        load_blk = np.bincount(blk.owner_arr, weights=w)
        load_nnz = np.bincount(nnz.owner_arr, weights=w)
        # within one row's weight of the mean (contiguous slabs cannot do better)
        assert load_nnz.max() <= load_nnz.mean() + w.max()
        assert load_nnz.max() / load_nnz.mean() < load_blk.max() / load_blk.mean()
        # contiguous, ascending, every row owned once
        assert np.all(np.diff(nnz.owner_arr) >= 0) and nnz.owner_arr.size == w.size
        assert [t.owner_pe for t in nnz.tasks] == list(range(pes))
    # band alignment: every boundary on a multiple of 64 rows
    al = sp.nnz_block_partition(w[:64 * 1000], 8, align=64)
    assert all(t.first % 64 == 0 for t in al.tasks)
    from paper_2012_06959_b200.errors import InvalidPeCount
    with pytest.raises(InvalidPeCount):
        sp.nnz_block_partition(np.ones(3), 4)
