// Internal launch interface between the C ABI (capi.cu) and the kernel files.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace sptrsv {

// ---- preprocess.cu -------------------------------------------------------
cudaError_t launch_expand_validate(const long long* cp, const long long* ri64, const double* val, int n, int* colE,
                                   int* ri32, unsigned long long* first_violation, int* structure_bad, int need_diag,
                                   cudaStream_t s);
cudaError_t launch_in_degree(const int* ri32, const int* colE, long long nnz, int* indeg, cudaStream_t s);
cudaError_t scan_exclusive(const int* in, int* out, int count, cudaStream_t s);
cudaError_t sort_pairs_stable(const int* keys_in, int* keys_out, const int* vals_in, int* vals_out, long long count,
                              int max_key, cudaStream_t s);
cudaError_t launch_transpose_keys(const int* ri32, const int* colE, const double* val, long long nnz, int n, int* key,
                                  int* entry, double* dg, cudaStream_t s);
cudaError_t launch_gather_offdiag(const int* sorted_entry, const int* colE, const double* val, long long noff, int* ci,
                                  double* cv, cudaStream_t s);
cudaError_t launch_scale_rows(const int* rp, const double* cv, const double* dg, int n, double* wv, double* rdg,
                              cudaStream_t s);
cudaError_t launch_iota(int* a, int n, cudaStream_t s);
cudaError_t launch_grid_levels(int* level, long long n, int nx, int ny, int nz, cudaStream_t s);
cudaError_t launch_widen(const int* a, long long* out, long long n, cudaStream_t s);
cudaError_t launch_level_hist(const int* level, int n, int* cnt, cudaStream_t s);
cudaError_t launch_tickets_per_level(const int* cnt, int nl, int* t, cudaStream_t s);
cudaError_t launch_pad_order(const int* by_level, const int* level, const int* level_ptr, const int* tb, int n,
                             int* padded, cudaStream_t s);

// ---- solve_rows.cu: sync-free component pool (paper Alg. 3 analogue) ------
enum RowMode : int { kModeExact = 0, kModeFast = 1, kModeLevel = 2 };

struct RowsArgs {
  int n;                    // rows in the whole matrix (global index space)
  const int* rp;            // off-diagonal CSR of the rows this launch solves (global row ids)
  const int* ci;
  const double* val;        // L_ij (exact) or -L_ij/L_ii (fast); unused for levels
  const double* dg;         // diagonal (exact)
  const double* rdg;        // 1/diagonal
  const double* b;          // right-hand side, global index
  // x segments: xseg[p] is PE p's x array (global index space; only rows p owns
  // are ever written there). For one PE xseg[0] is the whole x. For levels the
  // same slots hold int32 levels viewed through xlev.
  unsigned long long* const* xseg;
  int* const* lseg;
  const unsigned char* owner;  // owner PE of each component, nullptr when n_pes == 1
  // PEs served by this launch: block b works for PE pe_base + b % n_pe_local
  // (one PE per GPU in a multi-process run; all PEs when they share a device)
  int pe_base;
  int n_pe_local;
  int my_pe;                // set per block by the kernel
  const long long* pe_order_off;  // [n_pe_local + 1] slices of `order` per PE; nullptr: one PE, all of it
  const int* order;         // ticket slot -> row (topological order); -1 = padding
  long long order_len;      // number of slots (multiple of 32 when padded)
  int* ticket;              // pool counter(s), one per local PE, zero at launch
  DeviceStatus* status;
  int* abort_flag;
  unsigned long long timeout_ns;   // watchdog per thread from its first poll; 0 = none
  int spin_initial;         // tight polls before backing off (Backoff.initial_pause)
  int spin_max_ns;          // largest __nanosleep (Backoff.max_pause)
  int coop_long;            // 1: tickets are single-level, rows with > long_deps deps go warp-wide
  int long_deps;
  // split rows (fast mode, one PE): an order entry n + p is partial task p —
  // a slice [part_beg[p], part_end[p]) of heavy row part_heavy[p]'s entries,
  // summed by one warp and added into part_sum[h] (then part_done[h] += 1);
  // the heavy row's own ticket waits for part_done[h] == heavy_parts[h]
  const int* part_beg;
  const int* part_end;
  const int* part_heavy;
  const int* heavy_idx;     // [n]: heavy index of a split row, -1 otherwise (nullptr: no split rows)
  const int* heavy_parts;
  double* part_sum;
  int* part_done;
  long long* stamps;  // diagnostics (probe bit 512): globaltimer at each row's publish
  int debug;          // SPTRSV_PLAN_DEBUG: check owner-only, write-once publication
  int lane_loop;      // 1: a ticket's short rows complete lane by lane (solve_rows_lanes)
};

cudaError_t launch_rows(int mode, const RowsArgs& a, int blocks, cudaStream_t s);
int rows_blocks_per_sm(int mode);
int rows_lane_loop();  // SPTRSV_ROWS_LANELOOP=0 selects the per-lane spin loops (A/B)

// ---- solve_chains.cu: lane-chain lockstep executor ------------------------
struct ChainArgs;
cudaError_t launch_chains(int mode, const ChainArgs& a, int blocks, cudaStream_t s);

}  // namespace sptrsv
