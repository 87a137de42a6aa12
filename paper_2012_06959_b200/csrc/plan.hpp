// Device plan: everything resident in HBM for one matrix. One plan per
// (matrix, device); reused by every solve of that matrix.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../../include/sptrsv_b200.h"
#include "common.cuh"
#include "chains.hpp"
#include "stencil.hpp"

namespace sptrsv {

struct DevicePlan {
  sptrsv_options opt{};
  long long n = 0, nnz = 0, noff = 0;
  int device = 0;
  int num_sms = 148;
  bool structure_only = false;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;    // whole solve (resets + kernel)
  cudaEvent_t evk0 = nullptr, evk1 = nullptr;  // the solve kernel alone
  bool batch_k0 = false;  // solve_device_many: evk0 stays at the batch's first launch
  cudaError_t record_k0(cudaStream_t s) { return batch_k0 ? cudaSuccess : cudaEventRecord(evk0, s); }

  // CSR of off-diagonals + diagonal (preprocess.cu)
  int* rp = nullptr;
  int* ci = nullptr;
  double* cv = nullptr;
  double* wv = nullptr;
  double* dg = nullptr;
  double* rdg = nullptr;
  int* indeg = nullptr;

  // level analysis (K6) and the component-pool ticket order
  int* level = nullptr;
  int* by_level = nullptr;
  int* level_ptr = nullptr;
  int n_levels = 0;
  int* order = nullptr;
  long long order_len = 0;
  int coop_long = 0;
#ifndef SPTRSV_LONG_DEPS
#define SPTRSV_LONG_DEPS 32
#endif
  static constexpr int kLongDeps = SPTRSV_LONG_DEPS;  // rows with more dependencies are solved warp-wide
  static constexpr int kSplitDeps = 256;  // fast mode: rows with more are split into partial tasks
  struct SplitRows {
    int n_heavy = 0;
    int *heavy_idx = nullptr, *heavy_parts = nullptr, *part_beg = nullptr, *part_end = nullptr,
        *part_heavy = nullptr, *part_done = nullptr;
    double* part_sum = nullptr;
    void release() {
      void* ptrs[] = {heavy_idx, heavy_parts, part_beg, part_end, part_heavy, part_done, part_sum};
      for (void* p : ptrs)
        if (p) cudaFree(p);
      *this = SplitRows();
    }
  } split_rows;

  // solve scratch
  double* xbuf = nullptr;
  double* bbuf = nullptr;
  static constexpr int kCtlBlockBytes = 64;
  unsigned char* ctlblk = nullptr;   // [0,24) status, [32] ticket, [36] abort flag
  int* ticket = nullptr;             // the executors' task pool (every executor uses this one)
  DeviceStatus* status = nullptr;
  int* abort_flag = nullptr;
  cudaError_t reset_control(cudaStream_t s) { return cudaMemsetAsync(ctlblk, 0, kCtlBlockBytes, s); }
  unsigned long long** xseg_dev = nullptr;  // [1] for a single-PE plan
  int** lseg_dev = nullptr;

  ChainPlan chains;
  StencilPlan stencil;
  Stencil3Plan stencil3;
  int build_stencil3d(const std::vector<int>& h_rp, const std::vector<int>& h_ci);
  int solve_stencil3d(const double* d_b, double* d_x, cudaStream_t s, bool flags = false);
  int solve_host_streamed3d(const double* b, double* x, sptrsv_stats* st);
  // push executor (solve_push.cu): CSC of the off-diagonals + shared counters
  struct PushPlan {
    bool ready = false;
    int* cp = nullptr;
    int* ri = nullptr;
    double* v_exact = nullptr;
    double* v_fast = nullptr;
    double* left = nullptr;
    int* count = nullptr;
    void release() {
      void* ptrs[] = {cp, ri, v_exact, v_fast, left, count};
      for (void* p : ptrs)
        if (p) cudaFree(p);
      *this = PushPlan();
    }
  } push;
  int build_push();
  // band executor (solve_band.cu): dense 64-wide band columns + presence masks
  struct BandPlan {
    bool ready = false;
    double* coef = nullptr;
    unsigned long long* mask = nullptr;
    int nchunks = 0;
    void release() {
      if (coef) cudaFree(coef);
      if (mask) cudaFree(mask);
      *this = BandPlan();
    }
  } band;
  bool band_candidate(const std::vector<int>& h_rp, const std::vector<int>& h_ci) const;
  int build_band();
  int solve_band(const double* d_b, double* d_x, cudaStream_t s);
  int band_levels(int* level_out);
  bool band_narrow(const std::vector<int>& h_rp, const std::vector<int>& h_ci) const;
  // fast mode: row blocks of S rows coupled through the 64 rows above each
  // block (band_blocks.cu)
  struct BandBlocks {
    bool ready = false;
    int S = 0, nblk = 0;
    double* nt = nullptr;  // [nblk - 2] 64 x 64 coupling tails
    double* ct = nullptr;  // [nblk][64] tails of the uncoupled block solves
    double* tt = nullptr;  // [nblk][64] tails of x
    // the tail chain cut into superblocks of G steps (one PE): pp[g] = the
    // product of superblock g's coupling tails (built once per plan); per solve
    // dd[g] = g's chain run from zero, TT[g] = t at the end of g
    int G = 0, nsb = 0;
    int sb_first = -1, sb_steps = 0;  // the chain steps the superblocks cover
    double* pp = nullptr;  // [nsb] 64 x 64, K2 layout
    double* dd = nullptr;  // [nsb][64]
    double* TT = nullptr;  // [nsb][64]
    // the band's stored entries packed per column in row order (pk[off[j] ..]),
    // located through the presence mask: the sweeps stream ~half the bytes of
    // the dense 64-wide band
    double* pk = nullptr;
    int* off = nullptr;  // [n_pad + 1]
    bool pk_tma = false;  // the sweeps stream pk (k_bb_sweep_pk)
    int* reach = nullptr;  // [nblk] rows of each block the coupling reaches (K3 sweeps only those)
    // PE partition (set_partition with contiguous slabs on block boundaries):
    // this PE sweeps blocks [k0, k1) and runs their part of the tail chain;
    // the chain enters from the previous PE's last tail, read from its slot
    // (one-sided loads), and leaves through this PE's own slot
    bool part = false;
    int k0 = 0, k1 = 0, my_pe = 0, n_pes = 1;
    unsigned long long* slot = nullptr;             // own [2][64], value-is-flag, by solve parity
    const unsigned long long* prev_slot = nullptr;  // PE my_pe - 1's slot (peer mapping)
    long long solves = 0;
    void release_part() {
      if (slot) cudaFree(slot);
      slot = nullptr;
      prev_slot = nullptr;
      part = false;
      k0 = 0, k1 = nblk, my_pe = 0, n_pes = 1, solves = 0;
    }
    void release() {
      release_part();
      void* ptrs[] = {nt, ct, tt, pk, off, pp, dd, TT, reach};
      for (void* p : ptrs)
        if (p) cudaFree(p);
      *this = BandBlocks();
    }
  } bblk;
  int build_band_blocks();
  int stencil_groups(cudaStream_t s);  // stencil.cu: 1 when the band groups are in use
  int s3_zgroups(struct Stencil3Plan& P);  // stencil3d.cu: z-groups of the fast 3D wavefront
  int group_tasks_used = 0;            // tasks of the last stencil solve's band groups (0: none)
  int build_superblocks(int s_first, int nsteps, cudaStream_t st);
  int set_band_partition(const int32_t* owner, int pes, int my_pe);
  int solve_band_blocks(const double* d_b, double* d_x, cudaStream_t s);
  int solve_push(const double* d_b, double* d_x, cudaStream_t s);

  // PE partition (partition.cu): each PE owns components (PartitionPlan.owner_arr)
  // and publishes their x only into its own segment; other PEs read it.
  int n_pes = 1;          // PEs in the partition
  int n_pe_local = 1;     // PEs served by this process (all of them when they share the device)
  int pe_base = 0;        // first local PE
  unsigned char* owner_dev = nullptr;
  std::vector<unsigned long long*> local_segs;  // owned by this plan
  std::vector<void*> opened_peers;              // cudaIpcOpenMemHandle'd segments of other processes
  unsigned long long** seg_table = nullptr;     // device [2][n_pes]: half h of each PE's segment
  std::vector<unsigned long long*> host_seg_table;
  int* pe_order = nullptr;
  long long* pe_order_off = nullptr;
  int* pe_tickets = nullptr;
  int set_partition(const int32_t* owner, int pes, int my_pe);
  int solve_partitioned_rows(const double* d_b, double* d_x, cudaStream_t s);
  int sync_seg_table();
  long long part_solves = 0;  // parity of the segment double buffer
  void release_partition();
  std::vector<unsigned char> host_owner;  // owner map of the partition (empty: none)
  int grid_cap = 0;  // SMs this plan's persistent solve kernels may fill (0: all); set by group solves
  int enable_peer(const void* peer_ptr);  // P2P access to the device holding peer_ptr
  // diagnostics (probe_flags): kProbeWords int64 — per-step/chunk clock stamps
  // [0, 384), then per-task globaltimer stamps [384, 384 + 3 * 1024)
  static constexpr int kProbeWords = 6 * 64 + 3 * 1024;
  long long* probe_buf = nullptr;
  long long probe_words = kProbeWords;  // (rows executor, probe bit 512: one stamp per row)
  int executor_used = SPTRSV_EXECUTOR_ROWS;

  double setup_ms = 0.0;
  double last_solve_ms = 0.0;
  long long launches = 0;
  bool pending = false;

  int build(const int64_t* col_ptr, const int64_t* row_idx, const double* values, int64_t* bad_col);
  // levels: the component pool in (max, +1) arithmetic, or the closed form
  // x + y (+ z) when the CSR is a detected 2D / 3D lower stencil (grid = nx,
  // ny, nz; nz = 0 for 2D)
  int run_levels(const int* grid = nullptr, bool precomputed = false);
  int rows_grid(int mode) const;
  int solve_rows(const double* d_b, double* d_x, cudaStream_t s);
  int solve_chains(const double* d_b, double* d_x, cudaStream_t s);
  int build_chains(const std::vector<int>& h_rp, const std::vector<int>& h_ci);
  bool chains_preferred() const;
  int build_stencil(const std::vector<int>& h_rp, const std::vector<int>& h_ci);
  int solve_stencil(const double* d_b, double* d_x, cudaStream_t s, bool b_flags = false, bool x_flags = false,
                    int copies = 1);
  // k right-hand sides ([k][n] in d_b / d_x): one stacked launch where the
  // executor supports it (2D stencil, whole bands), else k solves in order
  int solve_device_many(const double* d_b, double* d_x, int k, cudaStream_t s);
  // host-buffer solve with band-granular H2D of b / D2H of x overlapping the
  // stencil kernel (copy streams + stream memory operations on band flags)
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  int solve_host_streamed(const double* b, double* x, sptrsv_stats* st);
  bool streamed_io_ok() const;
  int set_stencil_partition(const int32_t* owner, int pes, int my_pe);
  int stencil_sync_peers();
  int solve_device(const double* d_b, double* d_x, cudaStream_t s);
  int finish(sptrsv_stats* st);
  long long last_spins = 0, last_remote = 0;  // of the last finished solve (sptrsv_plan_last_counters)
  void release();
};

}  // namespace sptrsv
