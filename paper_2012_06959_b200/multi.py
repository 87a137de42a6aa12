"""One process per GPU: the read-only inter-GPU layer over CUDA IPC + torch.distributed.

Each rank is one PE of a ``PartitionPlan`` (column-block ``block_partition`` by
default, as in BASELINE.json's multi-GPU config; ``task_round_robin_partition``
works too). A rank builds the device plan of the whole matrix, keeps only its
own components' x in its segment, exports the segment as a CUDA IPC handle and
opens every peer's segment; inside the solve its kernel reads peers' x with
one-sided loads over NVLink/NVSwitch. For a 2D five-point L whose owner map
is band-aligned (block_partition of a 4096-square grid over 1/2/4/8 PEs) the
shared state is the stencil executor's mailbox array instead: a PE solves its
own 64-grid-row bands and polls only the bottom row of the band above a PE
boundary from its owner. ``torch.distributed`` carries only the
64-byte handles at setup and a barrier between solves (a solve resets the
segments, so no rank may start solve k+1 while a peer still reads solve k);
scatter of b / gather of x, when a caller wants x on one rank, is NCCL.

The orchestration (handle exchange, ownership, x assembly) is plain Python so
the multi-process logic is testable on CPU with the gloo backend
(tests/test_multi_gloo.py).
"""

from __future__ import annotations

import numpy as np

from .partition import PartitionPlan, block_partition, nnz_block_partition, task_round_robin_partition


def rank_partition(n: int, world: int, kind: str = "block", tasks_per_pe: int = 1, row_weight=None,
                   align: int = 1) -> PartitionPlan:
    """The partition every rank must agree on (deterministic in its arguments).

    ``kind="nnz"``: contiguous slabs of equal total ``row_weight`` (entries per
    row), boundaries on multiples of ``align`` rows."""
    if kind == "block":
        return block_partition(n, world)
    if kind == "nnz":
        return nnz_block_partition(np.ones(n) if row_weight is None else row_weight, world, align)
    return task_round_robin_partition(n, world, tasks_per_pe)


def exchange_handles(local: bytes, group=None) -> list[bytes]:
    """All-gather each rank's segment handle (CPU objects over the default group)."""
    import torch.distributed as dist

    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, local, group=group)
    return [bytes(h) for h in out]


def owned_rows(owner: np.ndarray, rank: int) -> np.ndarray:
    return np.flatnonzero(np.asarray(owner) == rank)


def assemble_x(parts: list[tuple[np.ndarray, np.ndarray]], n: int) -> np.ndarray:
    """Full x from (rows, values) pieces of every rank; every row exactly once."""
    x = np.full(n, np.nan)
    seen = np.zeros(n, dtype=np.int64)
    for rows, vals in parts:
        x[rows] = vals
        seen[rows] += 1
    if not np.all(seen == 1):
        raise ValueError("pieces do not cover every component exactly once")
    return x


class DistributedSolver:
    """This rank's PE of a partitioned solve (needs a GPU and an initialised process group)."""

    def __init__(self, l, plan: PartitionPlan, rank: int, *, device: int, precision: str = "fast",
                 timeout: float = 60.0, group=None, executor: str = "auto"):
        from . import _native

        if plan.n != l.n:
            raise ValueError("partition does not match the matrix")
        self.rank = rank
        self.world = plan.n_pes
        self.group = group
        # auto: a 2D five-point L with a band-aligned owner map runs the stencil
        # executor partitioned (exact: peer mailboxes; fast on a diagonally
        # dominant L: each rank enters its bands through local halo bands and
        # reads nothing remote); a banded L in fast mode with
        # slabs on row-block boundaries the band-block executor partitioned
        # (each rank sweeps its blocks, the tail chain passes rank to rank
        # through one 64-value slot); an unstructured L the component pool with
        # per-PE segments. The structured executors without a per-PE mode (3D
        # wavefront, lane chains, the exact band window, or owner maps that
        # split bands / row blocks) would degrade to the pool (banded-8M:
        # 3.6 ms -> 13 s), so there every rank solves the whole system on its
        # own GPU and keeps its rows ("replicated": correct, no speed-up, no
        # regression).
        build = lambda: _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision,  # noqa: E731
                                           executor=executor, device=device, timeout=timeout)
        self.native = build()
        ex0 = self.native.info()["executor"]
        self.native.set_partition(plan.owner_arr, plan.n_pes, rank)
        ex1 = self.native.info()["executor"]
        # (every rank decides alike: same matrix, same partition law)
        self.replicated = ex0 != "rows" and ex0 != ex1
        if self.replicated:
            self.native.close()
            self.native = build()
        else:
            handles = exchange_handles(self.native.export_segment(), group)
            for pe, h in enumerate(handles):
                if pe != rank:
                    self.native.import_segment(pe, h)
        self.rows = owned_rows(plan.owner_arr, rank)

    def barrier(self) -> None:
        import torch.distributed as dist

        dist.barrier(group=self.group)

    def solve_device_async(self, d_b: int, d_x: int, stream: int) -> None:
        """Solve this rank's components; x of the owned rows lands in d_x (others untouched)."""
        self.native.solve_device_async(d_b, d_x, stream)

    def synchronize(self) -> dict:
        return self.native.synchronize()
