/*
 * sptrsv_b200 — C ABI of the B200-native synchronization-free sparse lower
 * triangular solver (fp64, L x = b). Plain pointers and sizes only: no torch,
 * no C++ types, no exceptions cross this boundary.
 *
 * The reference package has no FFI; its operator API is the Python function
 * set re-exported from /root/reference/pkg/src/sptrsv/__init__.py:10-48. Each
 * entry point below names the reference function whose contract it serves, so
 * a binding (ctypes here) can sit exactly where the
 * reference's Python engine sits today (cli.py:149-150 `_run_engine`).
 *
 * Threading: a plan is not re-entrant; distinct plans may be used concurrently
 * (SPEC.md:451). Every call is synchronous unless its name ends in _async.
 */
#ifndef SPTRSV_B200_H
#define SPTRSV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the Python shim maps them 1:1 onto the reference exception
 * classes of errors.py (ZeroDiagonal, MissingDiagonal, MatrixStructureError,
 * DimensionMismatch, SolveTimeout, InvalidPeCount). */
enum {
  SPTRSV_OK = 0,
  SPTRSV_E_DIMENSION = 1,        /* DimensionMismatch        errors.py:62   */
  SPTRSV_E_ZERO_DIAGONAL = 2,    /* ZeroDiagonal(col)        errors.py:52   */
  SPTRSV_E_MISSING_DIAGONAL = 3, /* MissingDiagonal(col)     errors.py:46   */
  SPTRSV_E_STRUCTURE = 4,        /* MatrixStructureError     errors.py:42   */
  SPTRSV_E_TIMEOUT = 5,          /* SolveTimeout             errors.py:82   */
  SPTRSV_E_INVALID_PE = 6,       /* InvalidPeCount           errors.py:68   */
  SPTRSV_E_CUDA = 7,             /* CUDA runtime failure (no reference class) */
  SPTRSV_E_ARGUMENT = 8,         /* ValueError                               */
  SPTRSV_E_UNSUPPORTED = 9,
  SPTRSV_E_DEBUG_CHECK = 10     /* AssertionError: a SPTRSV_PLAN_DEBUG device check failed (engine.py:154-169) */
};

/* Arithmetic of the solve. EXACT reproduces solve_serial (reference.py:20-35)
 * bit for bit; FAST pre-scales rows by 1/l_ii and uses FMA (max relative
 * error vs the oracle ~1e-15, contract 1e-12). */
enum { SPTRSV_PRECISION_EXACT = 0, SPTRSV_PRECISION_FAST = 1 };

/* Which device executor runs the solve. ROWS: sync-free component pool over
 * a level-ordered ticket queue (paper Alg. 3). CHAINS: lane-chain lockstep
 * warps over contiguous row tasks. STENCIL: register-blocked wavefront for L
 * with 2D five-point lower structure (detected; any coefficients). AUTO:
 * STENCIL when the structure is detected, else CHAINS when most dependencies
 * stay inside a warp task, else ROWS. */
enum {
  SPTRSV_EXECUTOR_AUTO = 0,
  SPTRSV_EXECUTOR_ROWS = 1,
  SPTRSV_EXECUTOR_CHAINS = 2,
  SPTRSV_EXECUTOR_STENCIL = 3,
  SPTRSV_EXECUTOR_PUSH = 4, /* paper Alg. 2 / solve_shared_atomics (engine.py:324-431): warp per column, fp64
                               atomics on shared left sums + in-degree counters; rounding-level nondeterministic */
  SPTRSV_EXECUTOR_BAND = 5  /* one warp, sliding 64-row window of accumulators, column (push) order: for narrow
                               bands with little parallelism (banded-8M); exact mode bit-identical */
};

/* plan flags */
enum {
  SPTRSV_PLAN_STRUCTURE_ONLY = 1, /* analysis only: diagonal may be missing/zero, values may be NULL */
  SPTRSV_PLAN_NO_STREAMED_IO = 4, /* sptrsv_solve: copy all of b in, solve, copy all of x out (no overlap) */
  SPTRSV_PLAN_PUSH_MANAGED = 8,   /* executor "push": left sums and in-degree counters in cudaMallocManaged
                                     (unified) memory, updated with system-scope atomics -- the paper's
                                     Unified-Memory baseline, for the push/pull comparison */
  SPTRSV_PLAN_DEBUG = 16          /* device checks of the publication protocol (SolverConfig.debug,
                                     engine.py:154-169 / 510-513): every published x slot / mailbox word is
                                     written once, from its sentinel, by its owner PE; a violation stops the
                                     solve with SPTRSV_E_DEBUG_CHECK */
};

typedef struct sptrsv_options {
  int32_t precision;      /* SPTRSV_PRECISION_* */
  int32_t executor;       /* SPTRSV_EXECUTOR_* */
  int32_t device;         /* CUDA ordinal */
  int32_t flags;          /* SPTRSV_PLAN_* */
  double timeout_s;       /* device watchdog, SolverConfig.timeout (engine.py:75) */
  int32_t spin_initial;   /* Backoff.initial_pause (engine.py:61-66) */
  int32_t spin_max_ns;    /* Backoff.max_pause, as nanoseconds of __nanosleep */
  int32_t chain_lanes;    /* chains executor: lanes per warp task (<=32); 0 = 32 */
  int32_t probe_flags;    /* diagnostics only (tools/chains_probe.py); 0 in production */
  int32_t reserved[6];
} sptrsv_options;

typedef struct sptrsv_stats {
  double setup_ms;        /* plan creation (upload, K1, transpose, levels, schedule) */
  double solve_ms;        /* device time of the last solve (CUDA events) */
  double h2d_ms, d2h_ms;  /* host<->device copies of the last host-buffer solve */
  double kernel_ms;       /* the solve kernel alone (CUDA events around its launch) */
  int64_t spins;          /* polls that found a dependency unsolved (lock_wait_spins) */
  int64_t remote_reads;   /* dependency loads from another PE's segment */
  int64_t launches;       /* kernels launched by the last solve */
  int32_t executor;       /* executor that ran */
  int32_t n_levels;
  double e2e_ms;          /* wall time of the last host-buffer solve (copies included) */
  int32_t streamed_io;    /* 1: copies overlapped the kernel band by band; 2: zero-copy (pinned b/x read and
                           written by the kernel over PCIe); 0: copy in, solve, copy out */
  int32_t reserved_;
} sptrsv_stats;

typedef struct sptrsv_plan_info {
  int64_t n, nnz, n_offdiag;
  int32_t n_levels;
  int32_t executor;            /* executor the plan will run */
  double setup_ms;
  /* lane-chain schedule (valid when chains_ready) */
  int32_t chains_ready;
  int32_t chain_tasks;
  int64_t chain_slices, chain_stream_bytes, chain_mailboxes;
  int32_t chain_max_width, chain_lanes;
  int64_t deps_total, deps_in_task, deps_register, deps_ring, deps_mailbox;
  int64_t chain_max_task_steps;
  double schedule_ms;
} sptrsv_plan_info;

typedef struct sptrsv_plan sptrsv_plan;

/* Plan statistics (sizes, executor, schedule shape) for reports. */
int sptrsv_plan_get_info(const sptrsv_plan* plan, sptrsv_plan_info* info);

/* Fill defaults (exact, auto, device 0, 60 s, the reference Backoff(16, 512) mapped to 1024 device polls then sleeps up to 64 ns; see engine.py). */
void sptrsv_default_options(sptrsv_options* opt);

/* Upload a CSC lower-triangular L (the CscMatrix arrays, matrix.py:35-57) and
 * run validation + in-degree + transpose + level analysis on the device.
 * Replaces: column_lists + ensure_lower_triangular + Phase-1 counting of
 * solve_partitioned (engine.py:442-490) and compute_level_schedule
 * (analysis.py:43-64). On a lower-triangular violation returns
 * SPTRSV_E_{MISSING,ZERO}_DIAGONAL / STRUCTURE and stores the column in
 * *bad_col (the reference's first violation by (col, kind), matrix.py:150). */
int sptrsv_plan_create(const int64_t* col_ptr, const int64_t* row_idx, const double* values, int64_t n,
                       const sptrsv_options* opt, sptrsv_plan** out, int64_t* bad_col);

/* compute_in_degrees (analysis.py:19-27): int64[n], bit-exact. */
int sptrsv_plan_in_degrees(const sptrsv_plan* plan, int64_t* out);

/* compute_level_schedule (analysis.py:43-64): level_of int64[n]; components
 * grouped by level ascending (order int64[n], level_ptr int64[n_levels+1]). */
int sptrsv_plan_levels(const sptrsv_plan* plan, int64_t* level_of, int64_t* order, int64_t* level_ptr,
                       int64_t* n_levels);

/* Structure-only conveniences on raw CSC arrays (no plan kept). in_degree
 * accepts any structurally valid square CSC, like the reference. */
int sptrsv_in_degrees(const int64_t* col_ptr, const int64_t* row_idx, int64_t n, int32_t device, int64_t* out);

/* solve (engine.py:585-589) on host buffers: copies b in, solves, copies x
 * out. b and x are float64[n]. With the stencil executor the copies are
 * band-granular and overlap the solve (b of band t lands while earlier bands
 * solve; x of band t leaves as soon as it is stored), unless the plan was
 * created with SPTRSV_PLAN_NO_STREAMED_IO. Pinned host buffers give full
 * PCIe overlap; pageable ones are correct but serialise on the host. */
int sptrsv_solve(sptrsv_plan* plan, const double* b, double* x, sptrsv_stats* stats);

/* Device-resident solve: d_b/d_x are device pointers on the plan's device,
 * `stream` a cudaStream_t (0 = the plan's stream). Asynchronous. */
int sptrsv_solve_device_async(sptrsv_plan* plan, const double* d_b, double* d_x, void* stream);

/* The device counters of this plan's last finished solve: dependency polls
 * that found the value not yet published, and dependency loads that crossed a
 * PE boundary. After sptrsv_solve_group each PE's plan holds its own -- the
 * measured per-PE lock_wait_spins / remote_reads_issued of SolveReport.per_pe
 * (reference PeStats, engine.py:100-111). */
int sptrsv_plan_last_counters(const sptrsv_plan* plan, int64_t* spins, int64_t* remote_reads);

/* k right-hand sides, b and x laid out [k][n] (row-major: right-hand side r
 * at offset r * n). The 2D stencil executor stacks up to 16 of them into one
 * launch (its 64-band wavefront leaves most SMs idle; stacked copies fill
 * them); every other executor solves them one after another. Replaces the
 * host loop of extensions.solve_many (reference: one solve() per b). */
int sptrsv_solve_device_many_async(sptrsv_plan* plan, const double* d_b, double* d_x, int32_t k, void* stream);
int sptrsv_solve_many(sptrsv_plan* plan, const double* b, double* x, int32_t k, sptrsv_stats* stats);

/* Wait for the plan's work and report the device status of the last solve
 * (SPTRSV_E_TIMEOUT if the watchdog tripped). */
int sptrsv_synchronize(sptrsv_plan* plan, sptrsv_stats* stats);

int sptrsv_plan_destroy(sptrsv_plan* plan);

/* ---- PE partitions: the read-only inter-PE layer (solve_partitioned,
 * engine.py:438-582; Alg. 3). owner[n] is PartitionPlan.owner_arr
 * (partition.py:30-64). Each PE publishes its components' x only into its own
 * segment; other PEs read it with one-sided loads (no remote writes, no
 * collectives inside the solve).
 *   my_pe < 0 : every PE on this plan's device (one launch serves them all);
 *               solves gather x from the segments.
 *   my_pe >= 0: this process is PE my_pe only (one process per GPU); peers'
 *               segments are attached with sptrsv_plan_import_segment (CUDA
 *               IPC) or sptrsv_plan_set_peer_segment (same-process peer
 *               pointer). The caller must order consecutive solves across
 *               processes (a barrier): each solve resets the half of the
 *               parity double buffer the next solve uses, and every PE must
 *               run the same sequence of solves.
 * With the 2D stencil executor and a band-aligned owner map (whole 64-row
 * bands per PE, e.g. block_partition of lap2d-4096 over 1/2/4/8 GPUs) the
 * shared state is the stencil's mailbox array (the bottom grid row of every
 * band) instead of x segments; export/import/segment then refer to it. Other
 * owner maps fall back to the component pool. */
int sptrsv_plan_set_partition(sptrsv_plan* plan, const int32_t* owner, int32_t n_pes, int32_t my_pe);
int sptrsv_plan_export_segment(const sptrsv_plan* plan, void* ipc_handle_out);
int sptrsv_plan_import_segment(sptrsv_plan* plan, int32_t pe, const void* ipc_handle);
int sptrsv_plan_set_peer_segment(sptrsv_plan* plan, int32_t pe, void* device_ptr);
void* sptrsv_plan_segment(const sptrsv_plan* plan); /* this process's first segment (device pointer) */
/* One synchronous solve over all PEs of a partition held by ONE process
 * (replaces the reference's thread-per-PE engine run, engine.py:438-582):
 * plans[p] is PE p (set_partition(owner, n_plans, p)), peers wired with
 * sptrsv_plan_set_peer_segment (which enables P2P access when the peer lives
 * on another device). Plans may share a device or sit one per GPU; every PE's
 * kernel runs concurrently on its own stream; b and x are host arrays. */
int sptrsv_solve_group(sptrsv_plan* const* plans, int32_t n_plans, const double* b, double* x,
                       sptrsv_stats* stats);
int sptrsv_ipc_handle_size(void);

/* Matrix Market ingestion (reference mmio.py:132-144 `_coo_to_csc`): COO
 * (0-based int64 rows/cols, float64 values, nnz entries) -> CSC sorted
 * column-major, rows ascending, duplicate coordinates summed in input order
 * (bit-identical to the reference). Outputs: col_ptr int64[n+1], row_idx and
 * values sized nnz (upper bound); *nnz_out = unique entries. On the GPU. */
int sptrsv_coo_to_csc(int64_t n, const int64_t* rows, const int64_t* cols, const double* vals, int64_t nnz,
                      int32_t device, int64_t* col_ptr, int64_t* row_idx, double* values, int64_t* nnz_out);

/* Diagnostics: copy up to `count` probe timestamps (clock64) recorded by the
 * last solve when options.probe_flags asked for them. */
int sptrsv_plan_probe_read(const sptrsv_plan* plan, int64_t* out, int32_t count);

/* Last error message of this thread (empty string when none). */
const char* sptrsv_last_error(void);

/* Number of visible CUDA devices (0 without a GPU; no CUDA context is kept). */
int sptrsv_device_count(void);

int sptrsv_abi_version(void);

/* sizeof(sptrsv_options) / sizeof(sptrsv_stats) as compiled, so bindings can
 * assert their struct mirrors. */
int sptrsv_sizeof_options(void);
int sptrsv_sizeof_stats(void);

#ifdef __cplusplus
}
#endif

#endif /* SPTRSV_B200_H */
