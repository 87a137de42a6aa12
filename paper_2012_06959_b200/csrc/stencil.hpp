// Register-blocked wavefront executor for 2D five-point lower-triangular
// structure ("stencil2d"). Selected automatically when every row i = y*nx + x
// of L stores exactly the entries (i, i-nx) when y > 0 and (i, i-1) when x > 0
// besides its diagonal — the lower triangle of a 5-point operator on an
// nx-by-ny grid in natural order, with ARBITRARY coefficients. Design in
// stencil.cu.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace sptrsv {

// Block of one lane per lockstep step: kStR grid rows x kStC grid columns.
#ifndef SPTRSV_ST_R
#define SPTRSV_ST_R 2
#endif
#ifndef SPTRSV_ST_C
#define SPTRSV_ST_C 2
#endif
constexpr int kStR = SPTRSV_ST_R;
constexpr int kStC = SPTRSV_ST_C;
constexpr int kStLanes = 32;
constexpr int kStBand = kStLanes * kStR;  // grid rows per task (one CTA)
constexpr int kStBlock = kStR * kStC;     // elements per lane per step
#ifndef SPTRSV_ST_G
#define SPTRSV_ST_G 8
#endif
constexpr int kStG = SPTRSV_ST_G;         // steps per ring slot ("chunk"): the unit of every hand-over
#ifndef SPTRSV_ST_OUT_SLOTS
#define SPTRSV_ST_OUT_SLOTS 4
#endif
constexpr int kStOutSlots = SPTRSV_ST_OUT_SLOTS;  // output ring (chunks) between the compute and the store warp

// Per step, per lane: kStBlock elements; per element NF doubles:
//   fast : wu = -L[i,i-nx]/d, wl = -L[i,i-1]/d, rdg = 1/d
//   exact: wu = L[i,i-nx],   wl = L[i,i-1],    d, rdg
// stored field-major, then element pairs, then lanes, so each lane reads a
// pair of doubles with one conflict-free 16-byte shared load.
__host__ __device__ constexpr int st_fields(bool exact) { return exact ? 4 : 3; }
__host__ __device__ constexpr int st_step_bytes(bool exact) { return st_fields(exact) * kStBlock * kStLanes * 8; }
// Input ring depth in chunks: (slots - 1) * kStG steps of copies stay in flight
// (~20 steps at ~0.1 us per step covers the ~1.5 us DRAM latency).
#ifndef SPTRSV_ST_SLOTS_FAST
#define SPTRSV_ST_SLOTS_FAST 5
#endif
#ifndef SPTRSV_ST_SLOTS_EXACT
#define SPTRSV_ST_SLOTS_EXACT 4
#endif
__host__ __device__ constexpr int st_slots(bool exact) { return exact ? SPTRSV_ST_SLOTS_EXACT : SPTRSV_ST_SLOTS_FAST; }

// bands per group of the fast single-right-hand-side 2D wavefront (stencil.cu
// stencil_groups; SPTRSV_ST_GROUP overrides, 0 = one chain)
#ifndef SPTRSV_ST_GROUP_DEFAULT
#define SPTRSV_ST_GROUP_DEFAULT 1
#endif
constexpr int kStGroupDefault = SPTRSV_ST_GROUP_DEFAULT;

struct StencilPlan {
  bool ready = false;
  bool exact = true;
  int nx = 0, ny = 0;
  int n_tasks = 0;
  int steps_per_task = 0;  // nx / kStC + kStLanes - 1, rounded up to a multiple of kStG
  long long stream_bytes = 0;
  double build_ms = 0.0;
  unsigned char* stream = nullptr;     // [task][step][field][pair][lane] 16-byte pairs
  unsigned long long* mbox = nullptr;  // [n_tasks][nx] bottom grid row of each task (value-is-flag)
  // streamed host solves (sptrsv_solve): per-band b-arrived flags written by
  // the copy stream, per-band x-stored flags written by the kernel; both
  // compared against a per-solve epoch so they never need resetting
  unsigned* bflag = nullptr;  // [n_tasks]
  unsigned* xflag = nullptr;  // [n_tasks]
  unsigned epoch = 0;
  // b arrives in chunks of bands (1, 2, 4, ... up to b_chunk_max): only the
  // last band of a chunk gets a flag write, the loader derives it (0: per band)
  int b_chunk_max = 0;
  // Mailboxes are double-buffered by solve parity ([2][n_tasks][nx]): solve k
  // reads and writes half k % 2 and resets the other half for solve k + 1, so
  // a PE never resets a half a peer may still be reading (consecutive solves
  // are separated by a barrier across PEs).
  long long solves = 0;
  // several right-hand sides per launch (solve_many): mailboxes of k stacked
  // copies, [2][k * n_tasks][nx], grown on demand, with their own parity
  unsigned long long* mbox_many = nullptr;
  // band groups (fast mode, one PE, one right-hand side): groups of `grp`
  // bands run side by side, each entered through a halo task (stencil.cu);
  // decay = the plan-time error contraction per grid row (-1: not computed)
  int grp = 0, grp_tasks = 0;
  int* tband = nullptr;                    // device [grp_tasks]
  std::vector<int> grp_bands;              // the bands the groups were built for
  unsigned long long* mbox_grp = nullptr;  // [2][grp_tasks][nx]
  long long grp_solves = 0;
  double decay = -1.0;
  // fast mode, one right-hand side: b * (1/d) written by the kernel's prep
  // tasks (stencil.cu BD kernels) with per-band flags and prep counters
  double* bd = nullptr;
  unsigned* bdflag = nullptr;  // [n_tasks], compared with bd_epoch
  int* bd_done = nullptr;      // [n_tasks], zeroed per solve
  unsigned bd_epoch = 0;
  int many_k = 0;
  int many_last = 0;  // copies of the previous stacked solve (a different count re-arms every word)
  long long many_solves = 0;
  // PE partition, one PE per process (set_partition with my_pe >= 0 on a
  // band-aligned owner map): this PE solves its own bands (ascending), reads
  // the band above a PE boundary from the owning peer's mailboxes (CUDA IPC
  // mapping, one-sided .sys loads over NVLink) and publishes the bottom row
  // of a band whose successor is remote with .sys stores.
  bool part = false;
  int my_pe = -1, n_pes = 1;
  int n_my_tasks = 0;
  int* my_tasks = nullptr;                 // device [n_my_tasks]
  unsigned char* band_owner = nullptr;     // device [n_tasks]
  unsigned long long** pe_mbox = nullptr;  // device [n_pes] mailbox bases
  std::vector<unsigned long long*> host_pe_mbox;
  std::vector<int> host_band_owner, host_my_tasks;
  void release_part() {
    void* ptrs[] = {my_tasks, band_owner, pe_mbox};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    my_tasks = nullptr;
    band_owner = nullptr;
    pe_mbox = nullptr;
    host_pe_mbox.clear();
    host_band_owner.clear();
    host_my_tasks.clear();
    part = false;
    my_pe = -1;
    n_pes = 1;
    n_my_tasks = n_tasks;
  }
  void release() {
    release_part();
    void* ptrs[] = {stream, mbox, bflag, xflag, mbox_many, bd, bdflag, bd_done, tband, mbox_grp};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    stream = nullptr;
    mbox = nullptr;
    mbox_many = nullptr;
    tband = nullptr;
    mbox_grp = nullptr;
    grp = grp_tasks = 0;
    grp_bands.clear();
    grp_solves = 0;
    decay = -1.0;
    bd = nullptr;
    bdflag = nullptr;
    bd_done = nullptr;
    bd_epoch = 0;
    many_k = 0;
    many_last = 0;
    many_solves = 0;
    bflag = xflag = nullptr;
    epoch = 0;
    solves = 0;
    ready = false;
  }
};

// Structure detection on the host CSR (stencil.cu, stencil3d.cu).
int detect_stencil2d(long long n, const std::vector<int>& rp, const std::vector<int>& ci);
bool detect_stencil3d(long long n, const std::vector<int>& rp, const std::vector<int>& ci, int* dims);

// 3D seven-point lower structure (stencil3d.cu): tiles of 32 y-rows x 4
// z-planes, one CTA each, dispatched in ascending (Z, Y) order.
struct Stencil3Plan {
  bool ready = false;
  bool exact = true;
  int nx = 0, ny = 0, nz = 0, nyt = 0, nzt = 0, n_tasks = 0, steps = 0;
  long long stream_bytes = 0;
  double build_ms = 0.0;
  long long solves = 0;  // mailbox parity
  unsigned char* stream = nullptr;
  unsigned long long* ymail = nullptr;  // [2][tasks][4][nx]
  unsigned long long* zmail = nullptr;  // [2][tasks][32][nx]
  // streamed host solves: b arrives by z-slabs (k3R planes = one row of
  // tiles), flagged on the last slab of each copy; x flags per tile, raised
  // in tile order
  unsigned* bflag = nullptr;  // [nzt]
  unsigned* xflag = nullptr;  // [n_tasks]
  unsigned epoch = 0;
  int b_chunk_max = 0;
  // z-groups (fast mode, stencil3d.cu): virtual z-tiles, mailboxes sized by them
  int nztv = 0, n_vtasks = 0, zgroup = 0, zhalo = 0;
  int nytv = 0, ygrp = 0;  // y-groups: virtual y-slots (2 nyt - 1 with halo rows)
  int* zmap = nullptr;  // device [nztv]
  double decay = -1.0;  // plan-time error contraction per z-plane
  void release() {
    void* ptrs[] = {stream, ymail, zmail, bflag, xflag, zmap};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    *this = Stencil3Plan();
  }
};

// x flags raised in band order (the storer of band t waits for band t - 1's
// flag first), so the host copy stream waits once per copy, on its last band
#ifndef SPTRSV_ST_XFLAG_ORDER
#define SPTRSV_ST_XFLAG_ORDER 1
#endif

// sets f[0..n) = v with system-scope release stores (one launch)
cudaError_t stencil_release_flags(unsigned* f, int n, unsigned v, cudaStream_t s);

}  // namespace sptrsv
