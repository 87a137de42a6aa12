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
        plan = multi.rank_partition(l.n, world, kind, tasks_per_pe=3)
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


@pytest.mark.parametrize("kind", ["block", "round-robin"])
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
