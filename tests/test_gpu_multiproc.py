"""GPU: one process per PE over real CUDA IPC (the deployment bench.py uses
under torchrun), here with both processes on cuda:0 and gloo for the handle
exchange and the barriers between solves (NCCL refuses two ranks per device).

Each rank builds a DistributedSolver (auto executor): for a 2D five-point L
with a band-aligned owner map that is the stencil executor partitioned, the
mailbox arrays exchanged as IPC handles; with an unaligned map the test asks
for the component pool with per-PE segments (auto would keep the stencil,
replicated per rank). Every rank solves only its own rows;
x assembled over the ranks must equal the serial oracle bit for bit (exact),
for several right-hand sides (the parity double buffers).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, nx, ny, aligned, out_q):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2012_06959_b200 import multi, synth
    from paper_2012_06959_b200.partition import PartitionPlan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        l = synth.lap2d(nx, ny)
        if aligned:  # whole 64-grid-row bands per rank
            part = multi.rank_partition(l.n, world, "block")
        else:
            part = multi.rank_partition(l.n, world, "round-robin", tasks_per_pe=5)
        assert isinstance(part, PartitionPlan)
        # (unaligned: the component pool with per-PE segments is asked for; left
        # to auto, a band-splitting map keeps the stencil replicated per rank)
        solver = multi.DistributedSolver(l, part, rank, device=0, precision="exact", timeout=30.0,
                                         executor="auto" if aligned else "rows")
        executor = solver.native.info()["executor"]
        ok = []
        rng = np.random.default_rng(7)
        for rep in range(3):
            b = rng.uniform(-1.0, 1.0, l.n)
            db = torch.from_numpy(b).cuda()
            dx = torch.full_like(db, float("nan"))
            solver.barrier()
            solver.solve_device_async(db.data_ptr(), dx.data_ptr(), 0)
            st = solver.synchronize()
            torch.cuda.synchronize()
            rows = solver.rows
            pieces: list = [None] * world
            dist.all_gather_object(pieces, (rows, dx.cpu().numpy()[rows]))
            x = multi.assemble_x(pieces, l.n)
            ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
            ok.append(x.tobytes() == ref.tobytes())
        out_q.put((rank, executor, ok, int(st["remote_reads"])))
        solver.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("aligned", [True, False])
def test_two_processes_one_device_ipc(aligned):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    world = 2
    nx, ny = (256, 256) if aligned else (64, 40)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nx, ny, aligned, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, executor, ok, remote in res:
        assert executor == ("stencil" if aligned else "rows")
        assert all(ok), (rank, ok)
    assert sum(r[3] for r in res) > 0


def _worker_band(rank, world, port, out_q, n):
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2012_06959_b200 import multi, synth
    import paper_2012_06959_b200 as sp

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        l = synth.banded(n, 64, 0.5, 3)
        part = multi.rank_partition(l.n, world, "block")
        solver = multi.DistributedSolver(l, part, rank, device=0, precision="fast", timeout=30.0)
        executor = solver.native.info()["executor"]
        oks = []
        for seed in range(3):  # repeated solves: the chain slot alternates halves by parity
            b = np.random.default_rng(seed).uniform(-1.0, 1.0, l.n)
            db = torch.from_numpy(b).cuda()
            dx = torch.full_like(db, float("nan"))
            solver.barrier()
            solver.solve_device_async(db.data_ptr(), dx.data_ptr(), 0)
            solver.synchronize()
            torch.cuda.synchronize()
            pieces: list = [None] * world
            dist.all_gather_object(pieces, (solver.rows, dx.cpu().numpy()[solver.rows]))
            x = multi.assemble_x(pieces, l.n)
            ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
            oks.append(bool(sp.compare_solutions(x, ref, 1e-12).within_tol))
        out_q.put((rank, executor, bool(solver.replicated), all(oks)))
        solver.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [6400, 6000, 25600])
def test_two_processes_band_executor(n):
    """Band blocks over two processes. n = 6400: 3200-row slabs on the 64-row
    block grid, so each rank sweeps its blocks and rank 1's stretch of the
    tail chain starts from rank 0's last tail (read from rank 0's IPC-mapped
    slot). n = 6000: slabs off the grid, so the DistributedSolver keeps the
    band executor replicated (every rank solves the whole system and keeps
    its rows) instead of degrading to the component pool. n = 25600: 200
    blocks per rank, so rank 1's superblock chain polls rank 0's slot."""
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp

    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_band, args=(r, world, port, q, n)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, executor, replicated, ok in res:
        assert executor == "band" and replicated == (n % (64 * world) != 0) and ok
