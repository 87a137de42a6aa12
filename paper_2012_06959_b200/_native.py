"""ctypes binding of the C ABI in ``include/sptrsv_b200.h``.

This is the only module that talks to the CUDA library. There is no CPU
fallback anywhere in the package: if ``libsptrsv_b200.so`` is missing or no
CUDA device is visible, every compute entry point raises
:class:`~paper_2012_06959_b200.errors.NativeUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref
from pathlib import Path

import numpy as np

from .errors import NativeUnavailable, raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "libsptrsv_b200.so"

PRECISION = {"exact": 0, "fast": 1}
EXECUTOR = {"auto": 0, "rows": 1, "chains": 2, "stencil": 3, "push": 4, "band": 5}
EXECUTOR_NAME = {v: k for k, v in EXECUTOR.items()}
PLAN_STRUCTURE_ONLY = 1
PLAN_NO_STREAMED_IO = 4
PLAN_PUSH_MANAGED = 8  # executor='push': shared state in unified memory, system-scope atomics
PLAN_DEBUG = 16  # device checks: owner-only, write-once publication (SolverConfig.debug)


class Options(C.Structure):
    _fields_ = [
        ("precision", C.c_int32),
        ("executor", C.c_int32),
        ("device", C.c_int32),
        ("flags", C.c_int32),
        ("timeout_s", C.c_double),
        ("spin_initial", C.c_int32),
        ("spin_max_ns", C.c_int32),
        ("chain_lanes", C.c_int32),
        ("probe_flags", C.c_int32),
        ("reserved", C.c_int32 * 6),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("setup_ms", C.c_double),
        ("solve_ms", C.c_double),
        ("h2d_ms", C.c_double),
        ("d2h_ms", C.c_double),
        ("kernel_ms", C.c_double),
        ("spins", C.c_int64),
        ("remote_reads", C.c_int64),
        ("launches", C.c_int64),
        ("executor", C.c_int32),
        ("n_levels", C.c_int32),
        ("e2e_ms", C.c_double),
        ("streamed_io", C.c_int32),
        ("reserved_", C.c_int32),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class PlanInfo(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("nnz", C.c_int64),
        ("n_offdiag", C.c_int64),
        ("n_levels", C.c_int32),
        ("executor", C.c_int32),
        ("setup_ms", C.c_double),
        ("chains_ready", C.c_int32),
        ("chain_tasks", C.c_int32),
        ("chain_slices", C.c_int64),
        ("chain_stream_bytes", C.c_int64),
        ("chain_mailboxes", C.c_int64),
        ("chain_max_width", C.c_int32),
        ("chain_lanes", C.c_int32),
        ("deps_total", C.c_int64),
        ("deps_in_task", C.c_int64),
        ("deps_register", C.c_int64),
        ("deps_ring", C.c_int64),
        ("deps_mailbox", C.c_int64),
        ("chain_max_task_steps", C.c_int64),
        ("schedule_ms", C.c_double),
    ]

    def as_dict(self) -> dict:
        d = {name: getattr(self, name) for name, _ in self._fields_}
        d["executor"] = EXECUTOR_NAME.get(d["executor"], "?")
        return d


_P64 = C.POINTER(C.c_int64)
_PD = C.POINTER(C.c_double)

_lib = None
_lib_lock = threading.Lock()


def library_path() -> Path:
    return LIB_PATH


def _bind(lib: C.CDLL) -> None:
    lib.sptrsv_default_options.argtypes = [C.POINTER(Options)]
    lib.sptrsv_default_options.restype = None
    lib.sptrsv_plan_create.argtypes = [_P64, _P64, _PD, C.c_int64, C.POINTER(Options), C.POINTER(C.c_void_p), _P64]
    lib.sptrsv_plan_create.restype = C.c_int
    lib.sptrsv_plan_in_degrees.argtypes = [C.c_void_p, _P64]
    lib.sptrsv_plan_in_degrees.restype = C.c_int
    lib.sptrsv_plan_levels.argtypes = [C.c_void_p, _P64, _P64, _P64, _P64]
    lib.sptrsv_plan_levels.restype = C.c_int
    lib.sptrsv_in_degrees.argtypes = [_P64, _P64, C.c_int64, C.c_int32, _P64]
    lib.sptrsv_in_degrees.restype = C.c_int
    lib.sptrsv_coo_to_csc.argtypes = [C.c_int64, _P64, _P64, _PD, C.c_int64, C.c_int32, _P64, _P64, _PD,
                                      C.POINTER(C.c_int64)]
    lib.sptrsv_coo_to_csc.restype = C.c_int
    lib.sptrsv_solve.argtypes = [C.c_void_p, _PD, _PD, C.POINTER(Stats)]
    lib.sptrsv_solve.restype = C.c_int
    lib.sptrsv_solve_device_async.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.sptrsv_solve_device_async.restype = C.c_int
    lib.sptrsv_plan_last_counters.argtypes = [C.c_void_p, _P64, _P64]
    lib.sptrsv_plan_last_counters.restype = C.c_int
    lib.sptrsv_solve_device_many_async.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]
    lib.sptrsv_solve_device_many_async.restype = C.c_int
    lib.sptrsv_solve_many.argtypes = [C.c_void_p, _PD, _PD, C.c_int32, C.POINTER(Stats)]
    lib.sptrsv_solve_many.restype = C.c_int
    lib.sptrsv_synchronize.argtypes = [C.c_void_p, C.POINTER(Stats)]
    lib.sptrsv_synchronize.restype = C.c_int
    lib.sptrsv_plan_destroy.argtypes = [C.c_void_p]
    lib.sptrsv_plan_destroy.restype = C.c_int
    lib.sptrsv_last_error.argtypes = []
    lib.sptrsv_last_error.restype = C.c_char_p
    lib.sptrsv_device_count.argtypes = []
    lib.sptrsv_device_count.restype = C.c_int
    lib.sptrsv_abi_version.argtypes = []
    lib.sptrsv_abi_version.restype = C.c_int
    lib.sptrsv_plan_get_info.argtypes = [C.c_void_p, C.POINTER(PlanInfo)]
    lib.sptrsv_plan_get_info.restype = C.c_int
    lib.sptrsv_plan_probe_read.argtypes = [C.c_void_p, _P64, C.c_int32]
    lib.sptrsv_plan_probe_read.restype = C.c_int
    lib.sptrsv_plan_set_partition.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_int32]
    lib.sptrsv_plan_set_partition.restype = C.c_int
    lib.sptrsv_plan_export_segment.argtypes = [C.c_void_p, C.c_void_p]
    lib.sptrsv_plan_export_segment.restype = C.c_int
    lib.sptrsv_plan_import_segment.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
    lib.sptrsv_plan_import_segment.restype = C.c_int
    lib.sptrsv_plan_set_peer_segment.argtypes = [C.c_void_p, C.c_int32, C.c_void_p]
    lib.sptrsv_plan_set_peer_segment.restype = C.c_int
    lib.sptrsv_plan_segment.argtypes = [C.c_void_p]
    lib.sptrsv_plan_segment.restype = C.c_void_p
    lib.sptrsv_ipc_handle_size.argtypes = []
    lib.sptrsv_ipc_handle_size.restype = C.c_int
    lib.sptrsv_solve_group.argtypes = [C.POINTER(C.c_void_p), C.c_int32, _PD, _PD, C.POINTER(Stats)]
    lib.sptrsv_solve_group.restype = C.c_int


def load_library() -> C.CDLL:
    """Load (once) the in-tree CUDA library; raises if it is absent."""
    global _lib
    with _lib_lock:
        if _lib is None:
            # SPTRSV_LIB: an alternative in-tree build (tools/variants.sh), diagnostics only
            path = Path(os.environ["SPTRSV_LIB"]) if os.environ.get("SPTRSV_LIB") else LIB_PATH
            if not path.exists():
                raise NativeUnavailable(
                    f"{LIB_PATH} is missing: run `python -m paper_2012_06959_b200.build` (there is no CPU fallback)"
                )
            lib = C.CDLL(str(path))
            _bind(lib)
            _lib = lib
        return _lib


def require_gpu() -> C.CDLL:
    lib = load_library()
    if lib.sptrsv_device_count() < 1:
        raise NativeUnavailable("no CUDA device visible: this solver runs on the GPU only")
    return lib


def _err(lib) -> str:
    msg = lib.sptrsv_last_error()
    return msg.decode() if msg else ""


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def default_options() -> Options:
    opt = Options()
    load_library().sptrsv_default_options(C.byref(opt))
    return opt


class NativePlan:
    """A device-resident plan for one matrix (C handle ``sptrsv_plan*``)."""

    def __init__(self, col_ptr, row_idx, values, n: int, *, precision="exact", executor="auto", device=0,
                 timeout=60.0, spin_initial=1024, spin_max_ns=64, structure_only=False, chain_lanes=32,
                 probe_flags=0, streamed_io=True, push_managed=False, debug=False):
        lib = require_gpu()
        self._lib = lib
        self.n = int(n)
        cp = np.ascontiguousarray(col_ptr, dtype=np.int64)
        ri = np.ascontiguousarray(row_idx, dtype=np.int64)
        va = None if values is None else np.ascontiguousarray(values, dtype=np.float64)
        opt = default_options()
        opt.precision = PRECISION[precision]
        opt.executor = EXECUTOR[executor]
        opt.device = int(device)
        opt.flags = ((PLAN_STRUCTURE_ONLY if structure_only else 0) | (0 if streamed_io else PLAN_NO_STREAMED_IO)
                     | (PLAN_PUSH_MANAGED if push_managed else 0) | (PLAN_DEBUG if debug else 0))
        opt.timeout_s = float(timeout)
        opt.spin_initial = int(spin_initial)
        opt.spin_max_ns = int(spin_max_ns)
        opt.chain_lanes = int(chain_lanes)
        opt.probe_flags = int(probe_flags)
        handle = C.c_void_p()
        bad = C.c_int64(-1)
        rc = lib.sptrsv_plan_create(_ptr(cp, C.c_int64), _ptr(ri, C.c_int64),
                                    None if va is None else _ptr(va, C.c_double), self.n, C.byref(opt),
                                    C.byref(handle), C.byref(bad))
        raise_for_status(rc, _err(lib), bad.value)
        self._h = handle
        self.precision = precision
        self.device = int(device)
        self._finalizer = weakref.finalize(self, lib.sptrsv_plan_destroy, handle)

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def close(self) -> None:
        self._finalizer()

    def info(self) -> dict:
        inf = PlanInfo()
        rc = self._lib.sptrsv_plan_get_info(self._h, C.byref(inf))
        raise_for_status(rc, _err(self._lib))
        return inf.as_dict()

    # --- PE partitions (read-only inter-PE layer) -------------------------
    def set_partition(self, owner, n_pes: int, my_pe: int = -1) -> None:
        """Own components per ``owner`` (PartitionPlan.owner_arr); my_pe < 0: all PEs on this device."""
        own = np.ascontiguousarray(owner, dtype=np.int32)
        if own.shape != (self.n,):
            raise ValueError(f"owner has shape {own.shape}, need ({self.n},)")
        rc = self._lib.sptrsv_plan_set_partition(self._h, own.ctypes.data_as(C.POINTER(C.c_int32)), int(n_pes),
                                                 int(my_pe))
        raise_for_status(rc, _err(self._lib))

    def export_segment(self) -> bytes:
        buf = C.create_string_buffer(self._lib.sptrsv_ipc_handle_size())
        rc = self._lib.sptrsv_plan_export_segment(self._h, buf)
        raise_for_status(rc, _err(self._lib))
        return buf.raw

    def import_segment(self, pe: int, handle: bytes) -> None:
        buf = C.create_string_buffer(bytes(handle), len(handle))
        rc = self._lib.sptrsv_plan_import_segment(self._h, int(pe), buf)
        raise_for_status(rc, _err(self._lib))

    def set_peer_segment(self, pe: int, device_ptr: int) -> None:
        """Wire PE ``pe``'s shared state (segment / stencil mailboxes) by device pointer (same process)."""
        rc = self._lib.sptrsv_plan_set_peer_segment(self._h, int(pe), C.c_void_p(device_ptr))
        raise_for_status(rc, _err(self._lib))

    def segment_ptr(self) -> int:
        return int(self._lib.sptrsv_plan_segment(self._h) or 0)

    _PROBE_WORDS = 6 * 64 + 3 * 1024  # DevicePlan::kProbeWords

    def _probe_raw(self) -> np.ndarray:
        out = np.zeros(self._PROBE_WORDS, dtype=np.int64)
        rc = self._lib.sptrsv_plan_probe_read(self._h, _ptr(out, C.c_int64), out.size)
        raise_for_status(rc, _err(self._lib))
        return out

    def probe_stamps(self, per_step: int = 5) -> np.ndarray:
        """Per-step (chains) or per-chunk (stencil) clock stamps, [64, per_step]."""
        return self._probe_raw()[: per_step * 64].reshape(64, per_step)

    def probe_tasks(self, n_tasks: int) -> np.ndarray:
        """Stencil per-task globaltimer stamps [n_tasks, 3]: start, first chunk ready, end (ns)."""
        return self._probe_raw()[6 * 64: 6 * 64 + 3 * min(n_tasks, 1024)].reshape(-1, 3)

    def in_degrees(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.int64)
        rc = self._lib.sptrsv_plan_in_degrees(self._h, _ptr(out, C.c_int64))
        raise_for_status(rc, _err(self._lib))
        return out

    def levels(self) -> tuple[np.ndarray, np.ndarray, np.ndarray, int]:
        n_levels = C.c_int64(0)
        rc = self._lib.sptrsv_plan_levels(self._h, None, None, None, C.byref(n_levels))
        raise_for_status(rc, _err(self._lib))
        level_of = np.empty(self.n, dtype=np.int64)
        order = np.empty(self.n, dtype=np.int64)
        level_ptr = np.empty(n_levels.value + 1, dtype=np.int64)
        rc = self._lib.sptrsv_plan_levels(self._h, _ptr(level_of, C.c_int64), _ptr(order, C.c_int64),
                                          _ptr(level_ptr, C.c_int64), C.byref(n_levels))
        raise_for_status(rc, _err(self._lib))
        return level_of, order, level_ptr, int(n_levels.value)

    def solve(self, b: np.ndarray, out: np.ndarray | None = None) -> tuple[np.ndarray, dict]:
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = out if out is not None else np.empty(self.n, dtype=np.float64)
        st = Stats()
        rc = self._lib.sptrsv_solve(self._h, _ptr(b, C.c_double), _ptr(x, C.c_double), C.byref(st))
        raise_for_status(rc, _err(self._lib))
        d = st.as_dict()
        d["executor"] = EXECUTOR_NAME.get(d["executor"], "?")
        return x, d

    def solve_many(self, bs: np.ndarray, out: np.ndarray | None = None) -> tuple[np.ndarray, dict]:
        """k right-hand sides, ``bs`` shaped (k, n) (one per row): one stacked
        launch on the 2D stencil executor, else k solves on the device."""
        bs = np.ascontiguousarray(bs, dtype=np.float64)
        if bs.ndim != 2 or bs.shape[1] != self.n:
            raise ValueError(f"right-hand sides must be shaped (k, {self.n}), got {bs.shape}")
        x = out if out is not None else np.empty_like(bs)
        st = Stats()
        rc = self._lib.sptrsv_solve_many(self._h, _ptr(bs, C.c_double), _ptr(x, C.c_double), bs.shape[0],
                                         C.byref(st))
        raise_for_status(rc, _err(self._lib))
        d = st.as_dict()
        d["executor"] = EXECUTOR_NAME.get(d["executor"], "?")
        return x, d

    def solve_device_many_async(self, d_b: int, d_x: int, k: int, stream: int = 0) -> None:
        rc = self._lib.sptrsv_solve_device_many_async(self._h, C.c_void_p(d_b), C.c_void_p(d_x), int(k),
                                                      C.c_void_p(stream))
        raise_for_status(rc, _err(self._lib))

    def last_counters(self) -> dict:
        """Device counters of this plan's last finished solve."""
        sp_, rr = np.zeros(1, dtype=np.int64), np.zeros(1, dtype=np.int64)
        rc = self._lib.sptrsv_plan_last_counters(self._h, _ptr(sp_, C.c_int64), _ptr(rr, C.c_int64))
        raise_for_status(rc, _err(self._lib))
        return {"spins": int(sp_[0]), "remote_reads": int(rr[0])}

    def solve_device_async(self, d_b: int, d_x: int, stream: int = 0) -> None:
        rc = self._lib.sptrsv_solve_device_async(self._h, C.c_void_p(d_b), C.c_void_p(d_x), C.c_void_p(stream))
        raise_for_status(rc, _err(self._lib))

    def synchronize(self) -> dict:
        st = Stats()
        rc = self._lib.sptrsv_synchronize(self._h, C.byref(st))
        raise_for_status(rc, _err(self._lib))
        d = st.as_dict()
        d["executor"] = EXECUTOR_NAME.get(d["executor"], "?")
        return d


def in_degrees_raw(col_ptr, row_idx, n: int, device: int = 0) -> np.ndarray:
    lib = require_gpu()
    cp = np.ascontiguousarray(col_ptr, dtype=np.int64)
    ri = np.ascontiguousarray(row_idx, dtype=np.int64)
    out = np.empty(n, dtype=np.int64)
    rc = lib.sptrsv_in_degrees(_ptr(cp, C.c_int64), _ptr(ri, C.c_int64), n, device, _ptr(out, C.c_int64))
    raise_for_status(rc, _err(lib))
    return out


# --- plan cache -------------------------------------------------------------
# CscMatrix is immutable (frozen arrays), so a device plan stays valid for the
# matrix object's lifetime; repeated solve() calls with the same L reuse it.
_cache: dict[int, dict] = {}
_cache_lock = threading.Lock()


def _evict(ident: int) -> None:
    with _cache_lock:
        _cache.pop(ident, None)


def plan_for(l, **kw) -> NativePlan:
    """Device plan of matrix ``l`` (identity-keyed; dropped with the matrix)."""
    key = tuple(sorted(kw.items()))
    ident = id(l)
    with _cache_lock:
        per = _cache.get(ident)
        if per is None:
            per = {}
            _cache[ident] = per
            weakref.finalize(l, _evict, ident)
        plan = per.get(key)
    if plan is None:
        plan = NativePlan(l.col_ptr, l.row_idx, None if kw.get("structure_only") else l.values, l.n, **kw)
        with _cache_lock:
            per[key] = plan
    return plan


def partitioned_plan_for(l, partition, **kw) -> NativePlan:
    """Device plan of ``l`` split into the PEs of ``partition`` (all PEs on this device).

    Cached per (matrix, partition object); the partition is kept alive with the
    entry so its identity stays a valid key.
    """
    key = ("pe", id(partition)) + tuple(sorted(kw.items()))
    ident = id(l)
    with _cache_lock:
        per = _cache.get(ident)
        if per is None:
            per = {}
            _cache[ident] = per
            weakref.finalize(l, _evict, ident)
        hit = per.get(key)
    if hit is not None and hit[0] is partition:
        return hit[1]
    kw = dict(kw)
    kw["executor"] = "rows"
    plan = NativePlan(l.col_ptr, l.row_idx, l.values, l.n, **kw)
    plan.set_partition(partition.owner_arr, partition.n_pes, -1)
    with _cache_lock:
        per[key] = (partition, plan)
    return plan


class PeGroup:
    """All PEs of a partition in this process: one plan per PE (``plans[p]`` is PE p).

    The PEs' plans sit on one device or one per GPU (P2P peer pointers); one
    ``sptrsv_solve_group`` call launches every PE's kernel concurrently and
    assembles x from each PE's own rows.
    """

    def __init__(self, plans: list[NativePlan], devices: list[int], mode: str):
        self.plans = plans
        self.devices = devices
        self.mode = mode
        self.n = plans[0].n
        self._lib = plans[0]._lib

    def info(self) -> dict:
        d = self.plans[0].info()
        d["pe_mode"] = self.mode
        return d

    def solve(self, b: np.ndarray, out: np.ndarray | None = None) -> tuple[np.ndarray, dict]:
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = out if out is not None else np.empty(self.n, dtype=np.float64)
        handles = (C.c_void_p * len(self.plans))(*[p.handle.value for p in self.plans])
        st = Stats()
        rc = self._lib.sptrsv_solve_group(handles, len(self.plans), _ptr(b, C.c_double), _ptr(x, C.c_double),
                                          C.byref(st))
        raise_for_status(rc, _err(self._lib))
        d = st.as_dict()
        d["executor"] = EXECUTOR_NAME.get(d["executor"], "?")
        d["pe_mode"] = self.mode
        d["devices"] = list(self.devices)
        d["per_pe"] = [p.last_counters() for p in self.plans]  # measured, one plan per PE
        return x, d

    def close(self) -> None:
        for p in self.plans:
            p.close()


class SharedSegment:
    """Virtual PEs sharing one published segment: the structured executors
    (band window, 3D wavefront, lane chains, or a 2D wavefront whose owner map
    splits bands) have no per-PE mode, so on one device the whole matrix runs
    on the single fast plan; the PE split only shapes the report."""

    def __init__(self, plan: NativePlan):
        self.plan = plan

    def info(self) -> dict:
        d = self.plan.info()
        d["pe_mode"] = "shared-segment"
        return d

    def solve(self, b, out=None):
        x, d = self.plan.solve(b, out=out)
        d["pe_mode"] = "shared-segment"
        d["devices"] = [self.plan.device]
        return x, d


def pe_devices(n_pes: int, base: int = 0) -> list[int]:
    """Device of each PE: ``SPTRSV_PE_DEVICES`` (comma list, dealt round-robin),
    else one PE per visible GPU round-robin from ``base`` (SURVEY.md §8a N2:
    n_pes = number of GPUs), else every PE on ``base``."""
    env = os.environ.get("SPTRSV_PE_DEVICES")
    if env:
        devs = [int(v) for v in env.split(",") if v.strip()]
    else:
        count = require_gpu().sptrsv_device_count()
        devs = [(base + k) % count for k in range(count)] if count > 1 else [base]
    return [devs[p % len(devs)] for p in range(n_pes)]


def _wire(plans: list[NativePlan]) -> None:
    for p, pl in enumerate(plans):
        for q, peer in enumerate(plans):
            if q != p:
                pl.set_peer_segment(q, peer.segment_ptr())


def pe_solver_for(l, partition, executor: str = "auto", **kw):
    """The solver behind ``solve_partitioned`` with ``n_pes > 1`` (engine.py:438-582).

    * several GPUs: one plan per PE on its own device (``pe_devices``), each
      publishing its rows into its own HBM, peers read over NVLink (P2P);
    * one GPU, 2D five-point L with whole 64-row bands per PE: one stencil
      plan per PE, peers' mailboxes in the same HBM (``mode="stencil-pes"``);
    * one GPU, banded L in fast mode with slabs on row-block boundaries: one
      band-block plan per PE, the tail chain handed from PE to PE
      (``mode="band-pes"``);
    * one GPU, unstructured L: the component pool with one segment per PE
      (``mode="pool-segments"``);
    * one GPU, any other structured L: the single fast plan
      (``SharedSegment``).
    Cached per (matrix, partition object, knobs) like ``partitioned_plan_for``.
    """
    key = ("pes", id(partition), executor) + tuple(sorted(kw.items()))
    ident = id(l)
    with _cache_lock:
        per = _cache.get(ident)
        if per is None:
            per = {}
            _cache[ident] = per
            weakref.finalize(l, _evict, ident)
        hit = per.get(key)
    if hit is not None and hit[0] is partition:
        return hit[1]
    P = partition.n_pes
    device = kw.pop("device", 0)
    devs = pe_devices(P, device)
    owner = partition.owner_arr

    def build(dev: int, ex: str = executor) -> NativePlan:
        return NativePlan(l.col_ptr, l.row_idx, l.values, l.n, executor=ex, device=dev, **kw)

    if len(set(devs)) > 1:
        plans = []
        for p in range(P):
            pl = build(devs[p])
            ex0 = pl.info()["executor"]
            pl.set_partition(owner, P, p)
            if ex0 != "rows" and pl.info()["executor"] != ex0:
                # a structured executor without a per-PE mode (3D wavefront,
                # lane chains, band window (exact), a band-splitting 2D owner
                # map, band slabs off the row-block boundaries) would
                # degrade to the component pool: one GPU runs the fast plan
                for q in plans + [pl]:
                    q.close()
                plans = None
                break
            plans.append(pl)
        if plans is not None:
            _wire(plans)
            solver = PeGroup(plans, devs, "pe-per-gpu")
        else:
            solver = SharedSegment(plan_for(l, executor=executor, device=device, **kw))
    else:
        single = plan_for(l, executor=executor, device=device, **kw)
        ex = single.info()["executor"]
        solver = None
        if ex in ("stencil", "band"):
            # 2D: whole 64-row bands per PE (partitioned wavefront); band
            # blocks (fast mode): slabs on row-block boundaries (each PE its
            # blocks' sweeps and its stretch of the tail chain)
            first = build(device, ex)
            first.set_partition(owner, P, 0)
            if first.info()["executor"] == ex:
                plans = [first]
                for p in range(1, P):
                    pl = build(device, ex)
                    pl.set_partition(owner, P, p)
                    plans.append(pl)
                _wire(plans)
                solver = PeGroup(plans, devs, ex + "-pes")
            else:
                first.close()
        if solver is None and ex in ("rows", "push"):
            pool = build(device, "rows")
            pool.set_partition(owner, P, -1)
            solver = pool
        if solver is None:
            solver = SharedSegment(single)
    with _cache_lock:
        per[key] = (partition, solver)
    return solver


def env_device() -> int:
    return int(os.environ.get("SPTRSV_DEVICE", "0"))


def coo_to_csc(n: int, rows, cols, vals, device: int | None = None):
    """COO -> (col_ptr, row_idx, values) on the GPU: column-major, duplicates summed (mmio.py:132-144)."""
    lib = require_gpu()
    r = np.ascontiguousarray(rows, dtype=np.int64)
    c = np.ascontiguousarray(cols, dtype=np.int64)
    v = np.ascontiguousarray(vals, dtype=np.float64)
    nnz = int(r.size)
    col_ptr = np.empty(n + 1, dtype=np.int64)
    row_idx = np.empty(max(nnz, 1), dtype=np.int64)
    values = np.empty(max(nnz, 1), dtype=np.float64)
    out_nnz = C.c_int64(0)
    rc = lib.sptrsv_coo_to_csc(int(n), _ptr(r, C.c_int64), _ptr(c, C.c_int64), _ptr(v, C.c_double), nnz,
                               env_device() if device is None else int(device), _ptr(col_ptr, C.c_int64),
                               _ptr(row_idx, C.c_int64), _ptr(values, C.c_double), C.byref(out_nnz))
    raise_for_status(rc, _err(lib))
    k = int(out_nnz.value)
    return col_ptr, row_idx[:k].copy(), values[:k].copy()

