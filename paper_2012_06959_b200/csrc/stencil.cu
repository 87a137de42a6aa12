// Register-blocked, warp-specialised wavefront executor for 2D five-point
// lower structure.
//
// Structure: row i = y*nx + x stores (i, i-nx) iff y > 0 and (i, i-1) iff
// x > 0 (plus the diagonal), any coefficients — detected from the CSR at plan
// time. The dependency DAG is then the nx-by-ny grid wavefront: 8191 levels
// for 4096 x 4096.
//
// Work: a task (one CTA) owns a band of kStBand = 64 grid rows. Its compute
// warp's lane l owns rows 2l, 2l+1 and, at lockstep step s, solves the 2 x kStC
// block of columns [jC, jC + C) with j = s - l. The row above comes from lane
// l-1's block of the previous step by one __shfl_up_sync, the left neighbours
// from this lane's previous block; inside the block the wavefront is resolved
// in registers. Bands depend on the band above through value-is-flag
// mailboxes (the band's bottom grid row).
//
// The compute warp is the critical path, so it only shuffles, multiplies and
// writes shared memory. Two helper warps run beside it on other SM
// sub-partitions, and every hand-over is per chunk of kStG steps:
//   * loader: per chunk, one TMA bulk copy of the coefficient stream plus a
//     16-byte cp.async gather of b (both complete on the slot's mbarrier), then
//     the band-above mailbox values of the chunk's steps (polled), st_slots()
//     chunks ahead — the compute warp never waits on global memory;
//   * storer: writes the solved blocks from a shared-memory ring to x with
//     16-byte stores.
// Hand-overs are monotone chunk counters in shared memory (release/acquire at
// CTA scope). No column indices are read: per element the solve moves 24 B of
// coefficients (fast) + 8 B b + 8 B x.
//
// Arithmetic: fast: x = wl*left + (wu*up + b/d) with pre-scaled coefficients;
// exact: s = 0 + wu*up, s = s + wl*left, x = (b - s)/d — the serial oracle's
// order (ascending columns), with absent boundary terms contributing +0, which
// leaves every partial sum unchanged, so the result stays bit-identical.
#include <vector>
#include <chrono>
#include <cstring>
#include <cstdlib>
#include <cuda.h>
#include "plan.hpp"
#include "kernels.cuh"
#include "ptx.cuh"

namespace sptrsv {

int plan_fail(int code, const char* msg);

namespace {

// b of a chunk as ONE TMA copy (kStBTma): the band's rows seen through a
// skewed 4-D tensor view of b, (q, l, r, band) with strides
// (8, (2 nx - C) * 8, nx * 8, 64 nx * 8) bytes, so that element (q, l, r) is
// b[64 band + 2 l + r][q - C l]: lane l's row pair lagging C columns per lane
// is one rectangular box {G C, 32, R, 1} at q = c G C. Columns outside
// [0, nx) of a lane read neighbouring rows of the same band (never outside
// the band; padding steps discard them) or are zero-filled past the end.
// 128-byte swizzle puts the 16-byte piece p of grid row R = 32 r + l at
// p ^ (l & 7): the compute warp's 16-byte loads are conflict-free.
constexpr bool kStBTma = kStR == 2 && kStG * kStC * 8 == 128;

// Speculative exact division (SPTRSV_ST_SPEC, default on): see compute().
// Off, every step branches on its guard (exact lap2d-4096 1.38 ms; with
// the guard ablated 0.81 ms).
#ifndef SPTRSV_ST_SPEC
#define SPTRSV_ST_SPEC 1
#endif
// x leaves interior chunks by one TMA tensor store (SPTRSV_ST_X_TMA=1, default)
// or by the storer's 16-byte stores: each warp-wide STG.128 writes 32 rows,
// 32 LSU transactions, and that storer paced the compute warp through the out
// ring (lap2d-4096 fast 0.633 -> 0.573 ms with TMA stores)
#ifndef SPTRSV_ST_X_TMA
#define SPTRSV_ST_X_TMA 1
#endif
// TMA x stores left in flight by the storer (each still reading its out slot)
#ifndef SPTRSV_ST_STORE_DEPTH
#define SPTRSV_ST_STORE_DEPTH 2
#endif
constexpr int kStStoreDepth = SPTRSV_ST_STORE_DEPTH;
static_assert(kStStoreDepth >= 0 && kStStoreDepth <= kStOutSlots - 1, "in-flight stores need free out slots");


// Thread-block clusters of kStCluster consecutive bands (SPTRSV_ST_CLUSTER,
// default 8; 1 = no clusters): inside a cluster a band hands its bottom grid
// row to the band below through distributed shared memory -- the producer's
// compute warp writes each chunk's row straight into the consumer CTA's inbox
// ring with st.async, which completes its bytes on the consumer's per-slot
// inbox mbarrier -- instead of an L2 mailbox that the consumer's poller warp
// polls. No cluster-scope fence is on the path (ptxas turns those into
// MEMBAR.GPU / CCTL.IVALL). Only the first band of each cluster polls the L2
// mailbox of the band above.
#ifndef SPTRSV_ST_CLUSTER
#define SPTRSV_ST_CLUSTER 1
#endif
constexpr int kStCluster = SPTRSV_ST_CLUSTER;

// chunk counters released before the band-below publish (see step())
#ifndef SPTRSV_ST_REL_FIRST
#define SPTRSV_ST_REL_FIRST 1
#endif
constexpr bool kStRelFirst = SPTRSV_ST_REL_FIRST;
// the band-below hand-over is done by the storer warp once the chunk's outputs
// are handed to it (SPTRSV_ST_STORER_PUB=1) instead of by the compute warp:
// the compute warp's chunk boundary is then two shared-memory stores
#ifndef SPTRSV_ST_STORER_PUB
#define SPTRSV_ST_STORER_PUB 2
#endif
// (SPTRSV_ST_STORER_PUB = 2: a fifth, dedicated warp instead: the storer's
// element-wise stores of the edge chunks delayed the first hand-overs)
constexpr bool kStStorerPub = SPTRSV_ST_STORER_PUB && kStRelFirst;
// chunk outputs handed to the storer through per-slot mbarriers (arrive /
// try_wait) instead of a polled counter (SPTRSV_ST_OUT_BAR=1)
#ifndef SPTRSV_ST_OUT_BAR
#define SPTRSV_ST_OUT_BAR 1
#endif
constexpr bool kStOutBar = SPTRSV_ST_OUT_BAR && kStRelFirst;
// inbox ring depth in chunks (the producer waits for the consumer only when it
// runs kStInbox chunks ahead)
constexpr int kStInbox = 64;

// Mailbox sentinel: a signalling NaN. FP64 arithmetic propagates NaN
// payloads but always quiets them (tools/microbench/nan_bits.cu), so no
// solved value can alias it and values are published without conversion.
// 32-bit periodic, so it is reset with one cuMemsetD32Async.
constexpr unsigned kStNotReady32 = 0xFFF40000u;
constexpr unsigned long long kStNotReady = 0xFFF40000FFF40000ull;

struct alignas(64) StArgs {
  CUtensorMap bmap;  // kStBTma and b 16-byte aligned and a full last band: b via TMA
  CUtensorMap xmap;  // the same skewed view of x: interior chunks leave by one TMA store
  const unsigned char* stream;
  unsigned long long* mbox;
  int* ticket;
  const double* b;
  double* x;
  DeviceStatus* status;
  int* abort_flag;
  unsigned long long timeout_ns;
  int spin_initial, spin_max_ns;
  int nx, ny, n_tasks, steps;
  long long* dbg;  // diagnostics (probe_flags & 16): per-chunk clock stamps of task 0, chunks [64, 128)
  int probe;       // diagnostics flags (probe_flags)
  int nap;         // helper-warp sleep between control-word polls (ns)
  int b_aligned;   // b is 16-byte aligned: gather it with 16-byte cp.async (else 8-byte)
  int x_aligned;   // x is 16-byte aligned: 16-byte stores (else 8-byte)
  // host-buffer solves with overlapped copies (null otherwise): band t's b is
  // resident once bflag[t] >= epoch; the storer sets xflag[t] = epoch once
  // band t's x is stored
  const unsigned* bflag;
  unsigned* xflag;
  unsigned epoch;
  int b_chunk_max;  // bflag is written for the last band of each doubling chunk only (0: every band)
  // PE partition (stencil.hpp): tickets index my_tasks (null: ticket = band);
  // mbox is this PE's mailbox half of this solve, peers' halves are
  // pe_mbox[owner] + mbox_half
  const int* my_tasks;
  int n_my_tasks;
  unsigned long long* const* pe_mbox;
  const unsigned char* band_owner;
  int my_pe;
  long long mbox_half;
  int b_tma_bands;  // bands [0, b_tma_bands) gather b with one TMA per chunk (0: cp.async everywhere)
  int x_tma_bands;  // bands [0, x_tma_bands) store interior chunks of x with one TMA store
  unsigned long long* mbox_next;  // the other mailbox half: the storer resets each band's row for the next solve
  int debug;                      // SPTRSV_PLAN_DEBUG: every mailbox word is written once, over its sentinel
  // several right-hand sides in one launch (solve_many): b and x are k
  // stacked [ny][nx] grids, i.e. one grid of k * ny rows whose tasks t are
  // band t % bands of right-hand side t / bands -- every copy reads the same
  // coefficient stream, and the first band of a copy has no band above
  int bands;
  // fast mode, pre-scaled right-hand side (BD kernels): the first prep_tasks
  // tickets go to prep tasks that write bd = b * (1/d) for every band in band
  // order (bd_done[t] counts the prep tasks through band t; the last one
  // raises bdflag[t] = bd_epoch); the loaders stream bd instead of b and only
  // the wu / wl fields of the coefficient stream, and the compute warp's
  // element is two FMAs (the rd field's loads and multiply leave the
  // critical step). b_in is the caller's b (also the host-copy flags' b).
  int prep_tasks;
  const double* b_in;
  double* bd;
  const double* rdg;
  unsigned* bdflag;
  int* bd_done;
  unsigned bd_epoch;
  long long n_copy;  // elements of one right-hand side (rd index = i % n_copy)
  // band groups (fast mode, one PE, one right-hand side; null otherwise):
  // task t solves band tband[t] >= 0, or is the halo task of a group
  // (tband[t] = -band - 1): that band solved from a zero row above it, its x
  // discarded, only its bottom row handed to the group's first band
  const int* tband;
  int n_bands;  // bands of the grid (the host-copy flags' range)
};
__device__ __forceinline__ int st_band(const StArgs& a, int t) {
  if (!a.tband) return t;
  const int b = a.tband[t];
  return b >= 0 ? b : -b - 1;
}
__device__ __forceinline__ bool st_halo(const StArgs& a, int t) { return a.tband && a.tband[t] < 0; }
// task t starts from a zero row above (the first band of a right-hand side or a group's halo task)
__device__ __forceinline__ bool st_no_above(const StArgs& a, int t) { return t % a.bands == 0 || st_halo(a, t); }
// task t has a band below it in the same right-hand side / group
__device__ __forceinline__ bool st_has_below(const StArgs& a, int t) {
  return t + 1 < a.n_tasks && !st_no_above(a, t + 1);
}
constexpr int kStProbeFirst = 64, kStProbeChunks = 64;
template <bool DG>
__device__ __forceinline__ long long* st_stamp(const StArgs& a, int t, int c, int lane, int slot) {
  if constexpr (!DG) return nullptr;
  // probe bit 64: stamp task 1 (a band with a band above) instead of task 0
  return (a.dbg && t == ((a.probe & 64) ? 1 : 0) && lane == 0 && c >= kStProbeFirst &&
          c < kStProbeFirst + kStProbeChunks)
             ? a.dbg + 6 * (c - kStProbeFirst) + slot
             : nullptr;
}

// diagnostics (probe bit 256): hand-over timeline in globaltimer ns for chunks
// [64, 128): slot 0 = band 1 published chunk c, slot 1 = band 2's poller
// released its inbox chunk c, slots 2 / 3 = band 2's compute warp before /
// after its wait for chunk c (band 2's chunk c needs band 1's chunk c + 4)
template <bool DG>
__device__ __forceinline__ void lag_stamp(const StArgs& a, int t, int c, int lane, int slot) {
  if constexpr (!DG) return;
  if ((a.probe & 256) && a.dbg && lane == 0 && c >= kStProbeFirst && c < kStProbeFirst + kStProbeChunks &&
      t == (slot == 0 ? 1 : 2))
    a.dbg[6 * (c - kStProbeFirst) + slot] = (long long)globaltimer_ns();
}

constexpr int kStBlkPairs = kStBlock / 2;
constexpr bool kStPubWarp = SPTRSV_ST_STORER_PUB == 2 && kStRelFirst && SPTRSV_ST_OUT_BAR;
// compute, loader, storer, poller (+ publisher) warps; the publisher shares the
// compute warp's SM sub-partition but sleeps in mbarrier.try_wait between
// chunks (~10 instructions per chunk)
constexpr int kStThreads = (kStPubWarp ? 5 : 4) * 32;
// Shared-memory rings keep 16-byte pairs lane-innermost ([...][pair][lane]) so
// every warp-wide 16-byte access touches 512 consecutive bytes (4 wavefronts,
// no bank conflicts). b pair index of grid row r, chunk step k, column pair h:
// b ring slot: [r][l][piece] 16-byte pieces, 128 bytes per grid row, piece
// p = k * (kStC / 2) + h stored at p ^ (l & 7) (the TMA 128-byte swizzle;
// the cp.async gather writes the same layout)
__host__ __device__ constexpr int st_b_piece(int r, int l, int k, int h) {
  return (r * kStLanes + l) * (kStG * kStC / 2) + ((k * (kStC / 2) + h) ^ (l & 7));
}
static_assert(kStG * kStC / 2 >= 8 || !kStBTma, "the swizzle spans eight 16-byte pieces");


__device__ __noinline__ unsigned long long st_poll(const unsigned long long* p, int* abort_flag, DeviceStatus* status,
                                                   int spin_initial, int spin_max_ns, unsigned long long deadline,
                                                   bool sys, unsigned long long& spins) {
  auto ld = [&]() { return sys ? ld_relaxed_sys_u64(p) : ld_relaxed_u64(p); };
  unsigned long long u = ld();
  int polls = 0, sleep_ns = 32;
  while (u == kStNotReady) {
    ++polls;
    if (polls > spin_initial) {
      if ((polls & 63) == 0) {
        if (ld_relaxed_s32(abort_flag)) break;
        if (deadline && globaltimer_ns() > deadline) {
          atomicExch(&status->code, 5);
          atomicExch(abort_flag, 1);
          break;
        }
      }
      __nanosleep(sleep_ns);
      if (sleep_ns < spin_max_ns) sleep_ns <<= 1;
    }
    u = ld();
  }
  spins += polls;  // added to status->spins once per task (no per-miss global atomic)
  return u;
}

// control words of one task (chunk counters)
enum {
  kCtlTask = 0, kCtlInReady = 1, kCtlInDone = 2, kCtlOutReady = 3, kCtlOutDone = 4, kCtlAbort = 5, kCtlMbReady = 6,
  kCtlGroup = 7,  // cluster rank 0: the group ticket of the current task
  kCtlPubDone = 8,  // chunks whose band-below row the publisher warp has read out of the out ring
  kCtlPrep = 9      // BD kernels: this CTA's prep task (-1: a band or nothing)
};

template <bool EXACT>
struct StSmem {
  static constexpr int kSlots = st_slots(EXACT);
  static constexpr int kStep = st_step_bytes(EXACT);
  static constexpr int kCoefChunk = kStG * kStep;
  static constexpr int kBChunk = kStLanes * kStR * kStG * kStC * 8;
  static constexpr int kCoef = 0;                                       // [kSlots][kStG][kStep]
  static constexpr int kB = kCoef + kSlots * kCoefChunk;                // [kSlots][r][k][pair][lane] f64x2
  static constexpr int kInbox = kB + kSlots * kBChunk;                  // [kStInbox][kStG][kStC] f64
  // out ring: the b slot layout ([r][l][piece], 128-byte swizzled), so a
  // whole chunk leaves with one TMA tensor store through the skewed view of x
  static constexpr int kOut = (kInbox + kStInbox * kStG * kStC * 8 + 1023) / 1024 * 1024;
  static constexpr int kOutChunk = kStG * kStLanes * kStBlock * 8;
  static constexpr int kBars = kOut + kStOutSlots * kOutChunk;
  static constexpr int kInBars = kBars + 8 * kSlots;  // [kStInbox] inbox mbarriers (cluster hand-over)
  static constexpr int kCtl = kInBars + 8 * kStInbox;
  static constexpr int kOutBars = kCtl + 64;  // [kStOutSlots] out-slot-full mbarriers (compute -> storer)
  static constexpr int kTotal = kOutBars + 8 * kStOutSlots + 1024;  // + alignment slack of the ring base
  static_assert(kB % 1024 == 0 && kBChunk % 1024 == 0, "b slots on 1024-byte boundaries (TMA swizzle)");
};

// Spin on a chunk counter; false when the task is being aborted or the
// watchdog deadline passed (the caller then aborts the task).
// Helper warps pass nap > 0: they sleep between polls so their spinning does
// not compete with the compute warp for the shared-memory pipe.
__device__ __forceinline__ bool wait_ctl(const int* ctl, int which, int need, unsigned long long deadline,
                                         int nap = 0) {
  int polls = 0;
  while (ld_acquire_cta(ctl + which) < need) {
    if (ld_acquire_cta(ctl + kCtlAbort)) return false;
    if ((++polls & 1023) == 0 && deadline && globaltimer_ns() > deadline) return false;
    if (nap) __nanosleep(nap);
  }
  return true;
}

// The compute warp's chunk-boundary wait: input slot, band-above inbox and
// output slot in one polling loop (three independent shared loads per poll
// instead of three sequential loops).
__device__ __forceinline__ bool wait_chunk(const int* ctl, int in_need, int mb_need, int out_need,
                                           unsigned long long deadline, const int* abort_flag) {
  int polls = 0;
  while (true) {
    const int i = ld_acquire_cta(ctl + kCtlInReady), m = ld_acquire_cta(ctl + kCtlMbReady),
              o = ld_acquire_cta(ctl + kCtlOutDone);
    if (i >= in_need && m >= mb_need && o >= out_need) return true;
    if (ld_acquire_cta(ctl + kCtlAbort)) return false;
    if ((++polls & 1023) == 0) {
      if (deadline && globaltimer_ns() > deadline) return false;
      if (ld_relaxed_s32(abort_flag)) return false;  // another CTA (of this cluster) gave up
    }
  }
}

// A wait failed (watchdog or a peer warp's abort): stop this task everywhere.
__device__ __forceinline__ void abort_task(const StArgs& a, int* ctl, int lane) {
  if (lane == 0) {
    atomicExch(&a.status->code, 5);
    atomicExch(a.abort_flag, 1);
    st_release_cta(ctl + kCtlAbort, 1);
  }
}

// One lane's inputs of one step, loaded a step ahead into registers.
template <bool EXACT, bool BD = false>
struct StBlk {
  double wu[kStBlock], wl[kStBlock], rd[kStBlock], dd[kStBlock], bv[kStBlock];
  double inbox[kStC];

  // step k of the chunk in input slot `slot`, inbox slot `islot`
  __device__ __forceinline__ void load(const unsigned char* smem, int slot, int islot, int k, int lane) {
    using S = StSmem<EXACT>;
    const double2* cs = reinterpret_cast<const double2*>(smem + S::kCoef + slot * S::kCoefChunk + k * S::kStep);
#pragma unroll
    for (int p = 0; p < kStBlkPairs; ++p) {
      const double2 u = cs[(0 * kStBlkPairs + p) * kStLanes + lane];
      const double2 l = cs[(1 * kStBlkPairs + p) * kStLanes + lane];
      wu[2 * p] = u.x, wu[2 * p + 1] = u.y;
      wl[2 * p] = l.x, wl[2 * p + 1] = l.y;
      if (EXACT) {
        const double2 d = cs[(2 * kStBlkPairs + p) * kStLanes + lane];
        const double2 r = cs[(3 * kStBlkPairs + p) * kStLanes + lane];
        dd[2 * p] = d.x, dd[2 * p + 1] = d.y;
        rd[2 * p] = r.x, rd[2 * p + 1] = r.y;
      } else if (!BD) {
        const double2 r = cs[(2 * kStBlkPairs + p) * kStLanes + lane];
        rd[2 * p] = r.x, rd[2 * p + 1] = r.y;
      }
    }
    const double2* bb = reinterpret_cast<const double2*>(smem + S::kB + slot * S::kBChunk);
#pragma unroll
    for (int r = 0; r < kStR; ++r) {
#pragma unroll
      for (int c = 0; c < kStC; c += 2) {
        const double2 v = bb[st_b_piece(r, lane, k, c / 2)];
        bv[r * kStC + c] = v.x, bv[r * kStC + c + 1] = v.y;
      }
    }
    const double* ib = reinterpret_cast<const double*>(smem + S::kInbox) + (islot * kStG + k) * kStC;
#pragma unroll
    for (int c = 0; c < kStC; ++c) inbox[c] = ib[c];
  }
};

// ---- warp 1: stream coefficients and b, poll the band above -----------------
// the host-copy flag that covers band t's b: the copy stream flags the last
// band of each chunk of 1, 2, 4, ... bands (b_chunk_max > 0), else every band
__device__ __forceinline__ int st_b_flag_band(const StArgs& a, int t) {
  if (a.b_chunk_max <= 0) return t;
  for (int t0b = 0, w = 1;; t0b += w, w = min(2 * w, a.b_chunk_max))
    if (t < t0b + w) return min(a.n_bands, t0b + w) - 1;
}

template <bool EXACT, bool DG, bool BD = false>
__device__ void loader(const StArgs& a, unsigned char* smem, int* ctl, int t, int lane, unsigned& phase_bits,
                       unsigned long long deadline) {
  using S = StSmem<EXACT>;
  constexpr int NB = S::kSlots;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + S::kBars);
  const int nchunks = a.steps / kStG, nblk = a.nx / kStC;
  const int band = st_band(a, t);
  const int y0 = band * kStBand + kStR * lane;
  const unsigned char* tstream = a.stream + (size_t)(band % a.bands) * a.steps * S::kStep;
  const bool b_tma = kStBTma && band < a.b_tma_bands;
  bool ok = true;
  // chunk c: its coefficient block and, per lane and grid row, the b segment of
  // column blocks [c*G - lane, c*G - lane + G) clipped to the grid
  // The coefficient block is one TMA bulk copy (lane 0, expect_tx arrival);
  // b is gathered by every lane with 16-byte cp.async (one warp instruction
  // moves 512 B; a bulk copy per grid row would queue 64 small TMA operations
  // per chunk), whose completion arrives on the same slot mbarrier (.noinc:
  // the barrier counts 1 + 32 arrivals).
  auto issue = [&](int c) {
    const int slot = c % NB;
    const int j0 = c * kStG - lane;
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      if (BD) {
        // the wu and wl fields of every step (the rd field stays behind)
        constexpr int kFields2 = 2 * kStBlkPairs * kStLanes * 16;
        mbar_expect_tx(&bars[slot], kStG * kFields2 + (b_tma ? S::kBChunk : 0));
#pragma unroll
        for (int k = 0; k < kStG; ++k)
          bulk_g2s(smem + S::kCoef + slot * S::kCoefChunk + k * S::kStep,
                   tstream + (size_t)c * S::kCoefChunk + k * S::kStep, kFields2, &bars[slot]);
      } else {
        mbar_expect_tx(&bars[slot], S::kCoefChunk + (b_tma ? S::kBChunk : 0));
        bulk_g2s(smem + S::kCoef + slot * S::kCoefChunk, tstream + (size_t)c * S::kCoefChunk, S::kCoefChunk,
                 &bars[slot]);
      }
      if (b_tma) tma_load_4d(smem + S::kB + slot * S::kBChunk, &a.bmap, c * kStG * kStC, 0, 0, band, &bars[slot]);
    }
    double2* dst = reinterpret_cast<double2*>(smem + S::kB + slot * S::kBChunk);
#pragma unroll
    for (int r = 0; r < kStR; ++r) {
      if (b_tma || y0 + r >= a.ny) continue;
      const double* src = a.b + (size_t)(y0 + r) * a.nx;
#pragma unroll
      for (int k = 0; k < kStG; ++k) {
        const int jb = j0 + k;
        if (jb < 0 || jb >= nblk) continue;
#pragma unroll
        for (int h = 0; h < kStC / 2; ++h) {
          double2* d = dst + st_b_piece(r, lane, k, h);
          const double* s = src + jb * kStC + 2 * h;
          if (a.b_aligned) {
            cp_async16(d, s);
          } else {
            cp_async8(&d->x, s);
            cp_async8(&d->y, s + 1);
          }
        }
      }
    }
    cp_async_arrive_noinc(&bars[slot]);
  };
  auto settle = [&](int c) -> bool {
    const int slot = c % NB;
    const unsigned ph = (phase_bits >> slot) & 1u;
    int polls = 0;
    while (!mbar_try_wait(&bars[slot], ph)) {
      if ((++polls & 1023) == 0 && deadline && globaltimer_ns() > deadline) return false;
    }
    phase_bits ^= 1u << slot;
    return true;
  };
  // BD: this band's bd is written by the prep tasks (which themselves wait
  // for the host copies of b)
  if (BD) {
    int polls = 0;
    while ((int)(ld_acquire_gpu_u32(a.bdflag + band) - a.bd_epoch) < 0) {
      if ((++polls & 255) == 0 && deadline && globaltimer_ns() > deadline) ok = false;
      if (!__all_sync(0xffffffffu, ok)) {
        abort_task(a, ctl, lane);
        return;
      }
      __nanosleep(64);
    }
    // generic-proxy stores of other SMs -> this SM's TMA reads
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
  // overlapped host solve: this band's b may still be on its way over PCIe
  if (a.bflag && !BD) {
    int polls = 0;
    const int flag_band = st_b_flag_band(a, band);
    while ((int)(ld_acquire_sys_u32(a.bflag + flag_band) - a.epoch) < 0) {
      if ((++polls & 255) == 0 && deadline && globaltimer_ns() > deadline) ok = false;
      if (!__all_sync(0xffffffffu, ok)) {
        abort_task(a, ctl, lane);
        return;
      }
      __nanosleep(256);
    }
  }
  // Issue as far ahead as the ring allows (bounded by the compute warp's
  // progress, never by the band above); hand chunks over in order; only the
  // hand-over waits on the band-above mailbox.
  int issued = 0;
  for (int c = 0; c < nchunks; ++c) {
    if (long long* p = st_stamp<DG>(a, t, c, lane, 2)) *p = clock64();
    const int done = ld_acquire_cta(ctl + kCtlInDone);
    while (issued < nchunks && issued < done + NB) issue(issued++);
    while (ok && issued <= c) {  // chunk c itself must be in flight: wait for its slot
      ok = wait_ctl(ctl, kCtlInDone, issued - NB + 1, deadline, a.nap);
      if (ok) issue(issued++);
    }
    if (long long* p = st_stamp<DG>(a, t, c, lane, 3)) *p = clock64();
    if (ok) ok = settle(c);
    if (ok && c * kStG < kStLanes) {
      // steps before this lane's first block: b must read as exact zeros
      // (the TMA view put neighbouring rows there, the gather left them stale)
      double2* dst = reinterpret_cast<double2*>(smem + S::kB + (c % NB) * S::kBChunk);
#pragma unroll
      for (int r = 0; r < kStR; ++r)
#pragma unroll
        for (int k = 0; k < kStG; ++k)
          if (c * kStG - lane + k < 0)
#pragma unroll
            for (int h = 0; h < kStC / 2; ++h) dst[st_b_piece(r, lane, k, h)] = make_double2(0.0, 0.0);
    }
    if (long long* p = st_stamp<DG>(a, t, c, lane, 4)) *p = clock64();
    ok = __all_sync(0xffffffffu, ok);
    if (!ok) {
      abort_task(a, ctl, lane);
      for (int r = c + 1; r < issued; ++r) settle(r);  // bounded by the deadline
      return;
    }
    if (lane == 0) st_release_cta(ctl + kCtlInReady, c + 1);
    if (long long* p = st_stamp<DG>(a, t, c, lane, 5)) *p = clock64();
  }
}

// ---- warp 3: the band above's bottom grid row -------------------------------
// Per chunk, the row-above values of lane 0's blocks of steps c*G..c*G+G-1,
// one value per lane (one L2 round trip per chunk), polled value-is-flag and
// handed over through the inbox ring. Kept apart from the loader so the
// round trip overlaps the loader's copies instead of adding to them.
template <bool EXACT, bool DG>
__device__ void poller(const StArgs& a, unsigned char* smem, int* ctl, int t, int lane, unsigned long long deadline,
                       bool above_in_cluster) {
  using S = StSmem<EXACT>;
  if (above_in_cluster) return;  // the band above pushes into our inbox itself
  if (st_no_above(a, t)) {
    // no band above: the top grid row's "row above" is zero, so the compute
    // warp's lane 0 reads zeros from the inbox like any other band (no
    // per-step has_above select)
    double* inbox = reinterpret_cast<double*>(smem + S::kInbox);
    for (int w = lane; w < kStInbox * kStG * kStC; w += kStLanes) inbox[w] = 0.0;
    __syncwarp();
    if (lane == 0) st_release_cta(ctl + kCtlMbReady, 1 << 30);
    return;
  }
  double* inbox = reinterpret_cast<double*>(smem + S::kInbox);
  // the band above on another PE: its owner's mailboxes over NVLink (.sys)
  const int up_pe = a.band_owner ? a.band_owner[t - 1] : a.my_pe;
  const bool remote = up_pe != a.my_pe;
  const unsigned long long* above = (remote ? a.pe_mbox[up_pe] + a.mbox_half : a.mbox) + (size_t)(t - 1) * a.nx;
  const int nchunks = a.steps / kStG, nblk = a.nx / kStC;
  const int k = lane / kStC, q = lane % kStC;
  unsigned long long spins = 0;
  for (int c = 0; c < nchunks; ++c) {
    // inbox slot c % kStInbox is free once the compute warp finished chunk c - kStInbox
    if (c >= kStInbox && !wait_ctl(ctl, kCtlInDone, c - kStInbox + 1, deadline, a.nap))
      return abort_task(a, ctl, lane);
    bool ok = true;
    const int j = c * kStG + k;
    if (lane < kStG * kStC && j < nblk) {
      const unsigned long long u =
          st_poll(above + j * kStC + q, a.abort_flag, a.status, a.spin_initial, a.spin_max_ns, deadline, remote,
                  spins);
      if (u == kStNotReady) ok = false;
      inbox[((c % kStInbox) * kStG + k) * kStC + q] = __longlong_as_double((long long)u);
    }
    if (!__all_sync(0xffffffffu, ok)) return abort_task(a, ctl, lane);
    if (lane == 0) st_release_cta(ctl + kCtlMbReady, c + 1);
    lag_stamp<DG>(a, t, c, lane, 1);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) spins += __shfl_xor_sync(0xffffffffu, spins, off);
  if (lane == 0 && spins) atomicAdd(&a.status->spins, spins);
  if (remote && lane == 0) atomicAdd(&a.status->remote_reads, (unsigned long long)a.nx);
}

// ---- the band-below hand-over (compute warp, or the storer with kStStorerPub)
// Per chunk, lane 31's bottom grid row as staged in the out ring goes to the
// band below: value-is-flag stores into its L2 mailbox (polled by its poller
// warp; .sys stores when it lives on another PE), or -- the band below in the
// next CTA of this cluster -- st.async straight into its inbox ring, completing
// on the consumer's per-slot inbox mbarrier. Chunk c's lane-31 blocks are
// columns j = cG - 31 .. cG - 24, i.e. the tail of the consumer's chunk c - 4
// and the head of c - 3; an inbox slot is rewritten only once the consumer
// finished the chunk kStInbox before it.
template <bool EXACT, bool PART>
struct HandDown {
  using S = StSmem<EXACT>;
  const StArgs& a;
  const unsigned char* out;
  unsigned long long* below;
  int t, nblk;
  bool below_in_cluster, below_remote;
  unsigned peer_inbox = 0, peer_ibars = 0, peer_indone = 0;
  int peer_done = 0;
  __device__ HandDown(const StArgs& args, unsigned char* smem, int* ctl, int task, unsigned crank, bool in_cluster)
      : a(args), out(smem + S::kOut), below(args.mbox + (size_t)task * args.nx), t(task), nblk(args.nx / kStC),
        below_in_cluster(in_cluster) {
    below_remote = a.band_owner && t + 1 < a.n_tasks && a.band_owner[t + 1] != a.my_pe;
    if (in_cluster) {
      peer_inbox = mapa_shared(smem + S::kInbox, crank + 1);
      peer_ibars = mapa_shared(smem + S::kInBars, crank + 1);
      peer_indone = mapa_shared(ctl + kCtlInDone, crank + 1);
    }
  }
  __device__ __forceinline__ double2 bottom(int c, int k, int h) const {
    return reinterpret_cast<const double2*>(out + (c % kStOutSlots) * S::kOutChunk)[st_b_piece(kStR - 1, kStLanes - 1,
                                                                                               k, h)];
  }
  __device__ __forceinline__ void publish(int c, int lane) const {
    constexpr int kHalves = kStC / 2;
    if (!st_has_below(a, t) || lane >= kStG * kHalves) return;
    const int k = lane / kHalves, h = lane % kHalves;
    const int jj = c * kStG + k - (kStLanes - 1);
    if (jj < 0 || jj >= nblk) return;
    const double2 v = bottom(c, k, h);
    unsigned long long* w = below + (size_t)jj * kStC + 2 * h;
    if (a.debug) {  // (engine.py:510-513: published state only moves forward)
      const unsigned long long o0 = PART && below_remote ? ld_relaxed_sys_u64(w) : ld_relaxed_u64(w);
      const unsigned long long o1 = PART && below_remote ? ld_relaxed_sys_u64(w + 1) : ld_relaxed_u64(w + 1);
      if (o0 != kStNotReady || o1 != kStNotReady) {
        if (atomicCAS(&a.status->code, 0, 10) == 0) a.status->detail = (int)(t * (long long)a.nx + jj * kStC);
        atomicExch(a.abort_flag, 1);
      }
    }
    if (PART && below_remote) {
      st_relaxed_sys_u64_if(w, as_u64(v.x), true);
      st_relaxed_sys_u64_if(w + 1, as_u64(v.y), true);
    } else {
      st_relaxed_u64_if(w, as_u64(v.x), true);
      st_relaxed_u64_if(w + 1, as_u64(v.y), true);
    }
  }
  __device__ __forceinline__ bool push(int c, int lane, unsigned long long deadline) {
    constexpr int kHalves = kStC / 2;
    const int jlo = c * kStG - (kStLanes - 1), jhi = jlo + kStG - 1;
    if (jhi >= 0 && jlo < nblk) {
      const int need = min(jhi, nblk - 1) / kStG - kStInbox + 1;
      int polls = 0;
      while (peer_done < need) {  // rare: the consumer is kStInbox chunks behind
        peer_done = ld_relaxed_cluster_s32(peer_indone);
        if ((++polls & 255) == 0 && ((deadline && globaltimer_ns() > deadline) || ld_relaxed_s32(a.abort_flag)))
          return false;
      }
      if (lane < kStG * kHalves) {
        const int k = lane / kHalves, h = lane % kHalves;
        const int jj = jlo + k;
        if (jj >= 0 && jj < nblk) {
          const double2 v = bottom(c, k, h);
          const int cc = jj / kStG, kk = jj - cc * kStG, sl = cc % kStInbox;
          st_async_f64x2(peer_inbox + (((sl * kStG + kk) * kStC + 2 * h) << 3), v.x, v.y, peer_ibars + 8 * sl);
        }
      }
    }
    return true;
  }
  __device__ __forceinline__ bool run(int c, int lane, unsigned long long deadline) {
    if (below_in_cluster) return push(c, lane, deadline);
    publish(c, lane);
    return true;
  }
};

// ---- warp 4 (kStPubWarp): the band-below hand-over ---------------------------
template <bool EXACT, bool PART, bool DG>
__device__ void publisher(const StArgs& a, unsigned char* smem, int* ctl, int t, int lane, unsigned long long deadline,
                          unsigned crank, bool below_in_cluster) {
  using S = StSmem<EXACT>;
  HandDown<EXACT, PART> hd(a, smem, ctl, t, crank, below_in_cluster);
  const int nchunks = a.steps / kStG;
  const bool any = st_has_below(a, t);
  for (int c = 0; c < nchunks; ++c) {
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + S::kOutBars) + c % kStOutSlots;
    const unsigned par = (unsigned)(c / kStOutSlots) & 1u;
    int polls = 0;
    while (!mbar_try_wait(bar, par)) {
      if (ld_acquire_cta(ctl + kCtlAbort)) return abort_task(a, ctl, lane);
      if ((++polls & 63) == 0 && deadline && globaltimer_ns() > deadline) return abort_task(a, ctl, lane);
    }
    if (any && !hd.run(c, lane, deadline)) return abort_task(a, ctl, lane);
    lag_stamp<DG>(a, t, c, lane, 0);
    __syncwarp();
    if (lane == 0) st_release_cta(ctl + kCtlPubDone, c + 1);
  }
}

// ---- warp 2: solved blocks from shared memory to x --------------------------
template <bool EXACT, bool PART, bool DG>
__device__ void storer(const StArgs& a, unsigned char* smem, int* ctl, int t, int lane, unsigned long long deadline,
                       unsigned crank, bool below_in_cluster) {
  using S = StSmem<EXACT>;
  HandDown<EXACT, PART> hd(a, smem, ctl, t, crank, below_in_cluster);
  const int nchunks = a.steps / kStG, nblk = a.nx / kStC;
  const int band = st_band(a, t);
  const bool halo = st_halo(a, t);  // a group's halo band: x is not stored
  const int y0 = band * kStBand + kStR * lane;
  // this band's row of the other mailbox half (last read by the previous
  // solve, which is complete) is reset here for the next solve: no memset
  // node between solves
  {
    ulonglong2* row = reinterpret_cast<ulonglong2*>(a.mbox_next + (size_t)t * a.nx);
    for (int w = lane; w < a.nx / 2; w += kStLanes) row[w] = make_ulonglong2(kStNotReady, kStNotReady);
  }
  const bool x_tma = kStBTma && band < a.x_tma_bands;
  // TMA stores stay in flight: after chunk c only the kStStoreDepth most recent
  // stores may still be reading their slots, so chunks <= c - kStStoreDepth
  // are handed back (edge chunks are stored synchronously and drain the rest)
  int released = 0;
  for (int c = 0; c < nchunks; ++c) {
    if (kStOutBar) {
      // the compute warp arrives on the slot's mbarrier; try_wait suspends this
      // warp in hardware until then, so it wakes without a polling interval
      unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + S::kOutBars) + c % kStOutSlots;
      const unsigned par = (unsigned)(c / kStOutSlots) & 1u;
      int polls = 0;
      while (!mbar_try_wait(bar, par)) {
        if (ld_acquire_cta(ctl + kCtlAbort)) return abort_task(a, ctl, lane);
        if ((++polls & 63) == 0 && deadline && globaltimer_ns() > deadline) return abort_task(a, ctl, lane);
      }
    } else if (!wait_ctl(ctl, kCtlOutReady, c + 1, deadline, a.nap)) {
      return abort_task(a, ctl, lane);
    }
    if (kStStorerPub && !kStPubWarp) {
      // the band below first: its hand-over is on the critical path, x is not
      if (!hd.run(c, lane, deadline)) return abort_task(a, ctl, lane);
      lag_stamp<DG>(a, t, c, lane, 0);
    }
    bool async_store = false;
    unsigned char* slot = smem + S::kOut + (c % kStOutSlots) * S::kOutChunk;
    const double2* src = reinterpret_cast<const double2*>(slot);
#ifdef SPTRSV_ST_STORE_ABL  // timing diagnostics only: hand the slot back without storing x
    if (true) {
    } else
#endif
    if (halo) {
    } else
    // interior chunk (every lane's blocks inside the row): one TMA store of
    // the whole slot; edge chunks element by element (the skewed box would
    // write padding into neighbouring rows there)
    if (x_tma && c * kStG >= kStLanes - 1 && (c + 1) * kStG <= nblk) {
      async_store = true;
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the compute warp's STS -> async proxy
        tma_store_4d(&a.xmap, c * kStG * kStC, 0, 0, band, slot);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kStStoreDepth) : "memory");
      }
    } else {
      if (x_tma && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#pragma unroll
      for (int k = 0; k < kStG; ++k) {
        const int j = c * kStG + k - lane;
        if (j >= 0 && j < nblk) {
#pragma unroll
          for (int r = 0; r < kStR; ++r) {
            if (y0 + r < a.ny) {
              double* row = a.x + (size_t)(y0 + r) * a.nx + j * kStC;
#pragma unroll
              for (int q = 0; q < kStC / 2; ++q) {
                const double2 v = src[st_b_piece(r, lane, k, q)];
                if (a.x_aligned) {
                  reinterpret_cast<double2*>(row)[q] = v;
                } else {
                  row[2 * q] = v.x;
                  row[2 * q + 1] = v.y;
                }
              }
            }
          }
        }
      }
    }
    __syncwarp();
    const int done = async_store ? c + 1 - kStStoreDepth : c + 1;
    if (done > released) {
      // the publisher warp reads the same slot (normally long done)
      if (kStPubWarp && !wait_ctl(ctl, kCtlPubDone, done, deadline, a.nap)) return abort_task(a, ctl, lane);
      released = done;
      if (lane == 0) st_release_cta(ctl + kCtlOutDone, done);
    }
  }
  if (x_tma && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
  // overlapped host solve: band t's x may now be copied to the host. Flags
  // are raised in band order (after band t - 1's), so the copy stream waits
  // on the last band of each copy only
  if (a.xflag && lane == 0 && !halo) {
    __threadfence_system();
    int polls = 0;
    while (SPTRSV_ST_XFLAG_ORDER && band > 0 && (int)(ld_acquire_sys_u32(a.xflag + band - 1) - a.epoch) < 0) {
      if (ld_relaxed_s32(a.abort_flag)) break;  // the flags are released after the kernel anyway
      if ((++polls & 255) == 0 && deadline && globaltimer_ns() > deadline) break;
      __nanosleep(64);
    }
    st_release_sys_u32(a.xflag + band, a.epoch);
  }
}

// Fast mode, 2 x 2 blocks (SPTRSV_ST_EXPAND=1, diagnostics): every element as an affine function of the four
// inputs that arrive late (the two values above, by shuffle, and the two on
// the left, from this lane's previous step), its coefficients products of
// the block's own coefficients computed off the critical path. The bottom row
// is then one (x10) and two (x11) FMAs behind the shuffle instead of two and
// four. Same operations modulo re-association (fast mode's 1e-12 contract).
#ifndef SPTRSV_ST_EXPAND
#define SPTRSV_ST_EXPAND 0
#endif
// early shuffle (default): the next step's row above is shuffled as soon as
// this step's bottom row exists and the look-ahead loads are issued at the top
// of the step, which lets ptxas software-pipeline the loads under the FMA
// chain (exact lap2d-4096: 1.46 -> 1.39 ms; fast unchanged). The expanded
// block (SPTRSV_ST_EXPAND=1) halves the chain but adds 15 DP operations per
// step and measured slower (fast 0.63 -> 0.70 ms): the step is bound by the
// warp's instruction stream, not by the FMA chain.
#ifndef SPTRSV_ST_EARLY_SHFL
#define SPTRSV_ST_EARLY_SHFL 1
#endif
constexpr bool kStExpand = SPTRSV_ST_EXPAND && kStR == 2 && kStC == 2;
// Fast mode publishes the band-below mailbox row once per chunk (one warp
// store of lane 31's staged bottom rows) instead of a predicated store per
// step: the poller below consumes whole chunks anyway, and the per-step store
// cost the compute warp ~8 instructions a step (j, bounds, predicate, address).
#ifndef SPTRSV_ST_CHUNK_PUB
#define SPTRSV_ST_CHUNK_PUB 1
#endif
constexpr bool kStChunkPub = SPTRSV_ST_CHUNK_PUB;
static_assert(kStChunkPub || kStCluster == 1, "cluster hand-overs push whole chunks");
constexpr bool kStEarlyShfl = SPTRSV_ST_EARLY_SHFL;

template <bool EXACT, bool BD>
__device__ __forceinline__ void expand_block(const StBlk<EXACT, BD>& b, const double (&up)[kStC],
                                             const double (&left)[kStR], double (&x)[kStR][kStC]) {
  if constexpr (kStR == 2 && kStC == 2) {
    const double *wu = b.wu, *wl = b.wl;
    // right-hand sides of the block's own elimination (no late inputs)
    const double k0 = __dmul_rn(b.bv[0], b.rd[0]);
    const double k1 = __fma_rn(wl[1], k0, __dmul_rn(b.bv[1], b.rd[1]));
    const double k2 = __fma_rn(wu[2], k0, __dmul_rn(b.bv[2], b.rd[2]));
    const double k3 = __fma_rn(wu[3], k1, __fma_rn(wl[3], k2, __dmul_rn(b.bv[3], b.rd[3])));
    // coefficients of (up0, up1, left0, left1)
    const double a1 = __dmul_rn(wl[1], wu[0]), c1 = __dmul_rn(wl[1], wl[0]);
    const double a2 = __dmul_rn(wu[2], wu[0]), c2 = __dmul_rn(wu[2], wl[0]);
    const double a3 = __fma_rn(wu[3], a1, __dmul_rn(wl[3], a2)), b3 = __dmul_rn(wu[3], wu[1]);
    const double c3 = __fma_rn(wu[3], c1, __dmul_rn(wl[3], c2)), d3 = __dmul_rn(wl[3], wl[2]);
    // late inputs outermost: the shuffled values last
    x[0][0] = __fma_rn(wu[0], up[0], __fma_rn(wl[0], left[0], k0));
    x[0][1] = __fma_rn(a1, up[0], __fma_rn(wu[1], up[1], __fma_rn(c1, left[0], k1)));
    x[1][0] = __fma_rn(a2, up[0], __fma_rn(c2, left[0], __fma_rn(wl[2], left[1], k2)));
    x[1][1] = __fma_rn(a3, up[0], __fma_rn(b3, up[1], __fma_rn(c3, left[0], __fma_rn(d3, left[1], k3))));
  }
}

// ---- warp 0: the lockstep wavefront -----------------------------------------
// ABL: compile-time ablations for timing experiments only (0 in production):
// 1 = no output staging, 2 = no next-step loads, 4 = no shuffle, 8 = no
// active/publish branch
template <bool EXACT, int ABL, bool PART, bool DG, bool BD = false>
__device__ void compute(const StArgs& a, unsigned char* smem, int* ctl, int t, int lane, unsigned long long deadline,
                        unsigned crank, bool below_in_cluster, bool above_in_cluster) {
  using S = StSmem<EXACT>;
  constexpr int NB = S::kSlots;
  const int nchunks = a.steps / kStG, nblk = a.nx / kStC;
  // the band below in the next CTA of this cluster: its inbox ring, inbox
  // counter and progress counter in distributed shared memory
  // consumer side: inbox slot cc % kStInbox completes chunk cc's bytes
  unsigned long long* ibars = reinterpret_cast<unsigned long long*>(smem + S::kInBars);
  auto inbox_bytes = [&](int cc) { return max(0, min(nblk, (cc + 1) * kStG) - min(nblk, cc * kStG)) * kStC * 8; };
  auto arm_inbox = [&](int cc) {  // lane 0: this phase of the slot expects chunk cc's bytes
    if (cc < nchunks) mbar_expect_tx(ibars + cc % kStInbox, inbox_bytes(cc));
  };
  // chunk cn's inputs, band-above row and a free output slot; an in-cluster
  // band above delivers through the inbox mbarrier instead of MbReady
  auto wait_in = [&](int cn, int out_need) -> bool {
    if (!above_in_cluster) return wait_chunk(ctl, cn + 1, cn + 1, out_need, deadline, a.abort_flag);
    unsigned long long* bar = ibars + cn % kStInbox;
    const unsigned par = (unsigned)(cn / kStInbox) & 1u;
    int polls = 0;
    while (true) {
      const int i = ld_acquire_cta(ctl + kCtlInReady), o = ld_acquire_cta(ctl + kCtlOutDone);
      if (i >= cn + 1 && o >= out_need && mbar_test_wait(bar, par)) break;
      if (ld_acquire_cta(ctl + kCtlAbort)) return false;
      if ((++polls & 1023) == 0) {
        if (deadline && globaltimer_ns() > deadline) return false;
        if (ld_relaxed_s32(a.abort_flag)) return false;
      }
    }
    __syncwarp();
    if (lane == 0) arm_inbox(cn + kStInbox);  // the slot's next phase (its bytes come after InDone > cn)
    return true;
  };
  unsigned long long* below = a.mbox + (size_t)t * a.nx;
  // the band below on another PE reads these over NVLink: system-scope stores
  const bool below_remote = a.band_owner && t + 1 < a.n_tasks && a.band_owner[t + 1] != a.my_pe;
  const bool publish = lane == kStLanes - 1 && st_has_below(a, t) && !below_remote;
  const bool publish_sys = lane == kStLanes - 1 && below_remote;
  const bool solo = (a.probe & 32) != 0;  // diagnostics: run without the helper warps
  constexpr bool kStSpec = EXACT && SPTRSV_ST_SPEC && kStC % 2 == 0;
  double xleft[kStR];
#pragma unroll
  for (int r = 0; r < kStR; ++r) xleft[r] = 0.0;
  double bottom[kStC], upv[kStC];
#pragma unroll
  for (int q = 0; q < kStC; ++q) bottom[q] = upv[q] = 0.0;

  // One 2 x C block. exact: Markstein division with its operand-range guards
  // folded into the returned flag (ieee: IEEE division); fast: pre-scaled FMAs.
  auto block = [&](const StBlk<EXACT, BD>& blk, const double (&top)[kStC], double (&xb)[kStR][kStC],
                   bool ieee) -> bool {
    bool bad = false;
#pragma unroll
    for (int r = 0; r < kStR; ++r) {
#pragma unroll
      for (int q = 0; q < kStC; ++q) {
        const int e = r * kStC + q;
        const double up = r == 0 ? top[q] : xb[r - 1][q];
        const double left = q == 0 ? xleft[r] : xb[r][q - 1];
        if (EXACT) {
          double acc = __dadd_rn(0.0, __dmul_rn(blk.wu[e], up));
          acc = __dadd_rn(acc, __dmul_rn(blk.wl[e], left));
          const double num = __dsub_rn(blk.bv[e], acc);
          if (ieee) {
            xb[r][q] = __ddiv_rn(num, blk.dd[e]);
          } else {
            const double qv = __dmul_rn(num, blk.rd[e]);
            // a +0 numerator is exact too (x = qv + 0 = +-0 with the IEEE
            // sign), so the zero-filled steps before a lane's first block
            // stay fast; -0 is not (qv = -0 for d > 0, but r = +0 and
            // x = +0 + -0 = +0): it takes the IEEE path
            // (bitwise, not short-circuit: no branch per element)
            const int ok = (int)markstein_ok(blk.dd[e]) &
                           (((int)(num == 0.0) & (int)(__double2hiint(num) == 0)) |
                            ((int)markstein_ok(qv) & (int)markstein_ok(num)));
            bad |= !ok;
            xb[r][q] = __fma_rn(__fma_rn(-qv, blk.dd[e], num), blk.rd[e], qv);
          }
        } else if (q == 0) {
          // left comes from the previous step (early): the late operand
          // (up, possibly straight off the shuffle) goes in the outer FMA
          xb[r][q] = __fma_rn(blk.wu[e], up, __fma_rn(blk.wl[e], left, BD ? blk.bv[e] : __dmul_rn(blk.bv[e], blk.rd[e])));
        } else {
          xb[r][q] = __fma_rn(blk.wl[e], left, __fma_rn(blk.wu[e], up, BD ? blk.bv[e] : __dmul_rn(blk.bv[e], blk.rd[e])));
        }
      }
    }
    return bad;
  };
  // A solved block: carry its right column and bottom row, stage it for the
  // storer. No select on `active`: steps before a lane's first block see zero
  // coefficients, zero b (the loader zero-fills it) and zero neighbours, so
  // they compute exact zeros -- the boundary values the first block needs;
  // steps past the last block compute garbage that only ever reaches other
  // past-the-end steps (never published, never stored).
  auto retire = [&](int c, int k, const double (&xb)[kStR][kStC]) {
#pragma unroll
    for (int r = 0; r < kStR; ++r) xleft[r] = xb[r][kStC - 1];
#pragma unroll
    for (int q = 0; q < kStC; ++q) bottom[q] = xb[kStR - 1][q];
    // early shuffle: the next step's row above enters the shared-memory
    // pipe ahead of this step's stores and the look-ahead loads
    if (kStEarlyShfl) {
#pragma unroll
      for (int q = 0; q < kStC; ++q) upv[q] = (ABL & 4) ? bottom[q] : __shfl_up_sync(0xffffffffu, bottom[q], 1);
    }
    double2* dst = reinterpret_cast<double2*>(smem + S::kOut + (c % kStOutSlots) * S::kOutChunk);
#pragma unroll
    for (int r = 0; r < kStR; ++r)
#pragma unroll
      for (int q = 0; q < kStC; q += 2)
        if (!(ABL & 1)) dst[st_b_piece(r, lane, k, q / 2)] = make_double2(xb[r][q], xb[r][q + 1]);
  };
  // Speculative exact mode (kStSpec): steps run Markstein unguarded and only
  // accumulate the guard; a chunk in which any lane's guard failed is rolled
  // back to its starting state and recomputed with IEEE division before its
  // outputs and its band-below mailbox row leave the warp. Values are
  // therefore published per chunk (one warp store from the staged outputs),
  // which is also the poller's granularity.
  bool spec_bad = false;
  double sv_xleft[kStR], sv_bottom[kStC], sv_upv[kStC];
  auto save_chunk_state = [&]() {
#pragma unroll
    for (int r = 0; r < kStR; ++r) sv_xleft[r] = xleft[r];
#pragma unroll
    for (int q = 0; q < kStC; ++q) sv_bottom[q] = bottom[q], sv_upv[q] = upv[q];
  };
  auto redo_chunk = [&](int c) {
    if ((a.probe & 128) && lane == 0) atomicAdd(&a.status->remote_reads, 1ull);  // diagnostics: count redos
#pragma unroll
    for (int r = 0; r < kStR; ++r) xleft[r] = sv_xleft[r];
#pragma unroll
    for (int q = 0; q < kStC; ++q) bottom[q] = sv_bottom[q], upv[q] = sv_upv[q];
#pragma unroll 1
    for (int k = 0; k < kStG; ++k) {
      StBlk<EXACT, BD> blk;
      blk.load(smem, c % NB, c % kStInbox, k, lane);
      double top[kStC], xb[kStR][kStC];
#pragma unroll
      for (int q = 0; q < kStC; ++q) {
        const double up = kStEarlyShfl ? upv[q] : __shfl_up_sync(0xffffffffu, bottom[q], 1);
        top[q] = lane == 0 ? blk.inbox[q] : up;
      }
      block(blk, top, xb, true);
      retire(c, k, xb);
    }
  };
  HandDown<EXACT, PART> hd(a, smem, ctl, t, crank, below_in_cluster);
  auto hand_down = [&](int c) -> bool { return kStStorerPub || hd.run(c, lane, deadline); };

  // step k of chunk c; `nxt` receives the next step's inputs
  // step k of chunk c computes from `cur` (loaded two steps earlier) and
  // loads step k + 2 into `nxt2`: a full step of slack hides the shared-memory
  // latency that a one-step lookahead leaves exposed
  auto step = [&](int c, int k, const StBlk<EXACT, BD>& cur, StBlk<EXACT, BD>& nxt2) -> bool {
    auto load_ahead = [&]() {
      if (k + 2 < kStG) {
        if (!(ABL & 2)) nxt2.load(smem, c % NB, c % kStInbox, k + 2, lane);
      } else if (c + 1 < nchunks) {
        nxt2.load(smem, (c + 1) % NB, (c + 1) % kStInbox, k + 2 - kStG, lane);
      }
    };
    // the first step that loads from chunk c + 1: make sure it is ready
    if (k == kStG - 2 && c + 1 < nchunks && !solo) {
      if (long long* p = st_stamp<DG>(a, t, c + 1, lane, 0)) *p = clock64();
      lag_stamp<DG>(a, t, c + 1, lane, 2);
      if (!wait_in(c + 1, c + 1 >= kStOutSlots ? c + 2 - kStOutSlots : 0))
        return false;
      if (long long* p = st_stamp<DG>(a, t, c + 1, lane, 1)) *p = clock64();
      lag_stamp<DG>(a, t, c + 1, lane, 3);
    }
    const int s = c * kStG + k;
    const int j = s - lane;
    const bool active = j >= 0 && j < nblk;
    if (kStEarlyShfl) load_ahead();
    double top[kStC];
#pragma unroll
    for (int q = 0; q < kStC; ++q) {
      const double up = kStEarlyShfl ? upv[q] : (ABL & 4) ? bottom[q] : __shfl_up_sync(0xffffffffu, bottom[q], 1);
      top[q] = lane == 0 ? cur.inbox[q] : up;
    }
    double xb[kStR][kStC];
    if (kStExpand && !EXACT) {
      expand_block(cur, top, xleft, xb);
    } else if (kStSpec) {
      if (k == 0) save_chunk_state();
      spec_bad |= block(cur, top, xb, false);
    } else if (block(cur, top, xb, false) && EXACT) {
      if (a.probe & 128) atomicAdd(&a.status->remote_reads, 1ull);  // diagnostics: count IEEE fallbacks
      block(cur, top, xb, true);
    }
    retire(c, k, xb);
    if (!(ABL & 8) && !kStSpec && !kStChunkPub) {
#pragma unroll
      for (int q = 0; q < kStC; ++q)
        st_relaxed_u64_if(below + j * kStC + q, as_u64(bottom[q]), publish && active);
      if (PART) {
#pragma unroll
        for (int q = 0; q < kStC; ++q)
          st_relaxed_sys_u64_if(below + j * kStC + q, as_u64(bottom[q]), publish_sys && active);
      }
    }
    if (!kStEarlyShfl) load_ahead();
    if (k == kStG - 1 && kStRelFirst) {
      // chunk boundary: hand the outputs and the input slot over BEFORE the
      // band-below publish -- the release's MEMBAR.CTA would otherwise wait
      // for the publish's global stores to be acknowledged
      if (kStSpec) {
        if (__any_sync(0xffffffffu, spec_bad)) redo_chunk(c);
        spec_bad = false;
      }
      __syncwarp();
      if (lane == 0) {
        if (kStOutBar) {
          st_release_cta(ctl + kCtlInDone, c + 1);
          mbar_arrive(reinterpret_cast<unsigned long long*>(smem + S::kOutBars) + c % kStOutSlots);
        } else {
          st_release_cta(ctl + kCtlOutReady, c + 1);
          st_release_cta(ctl + kCtlInDone, c + 1);
        }
      }
      if ((kStChunkPub || kStSpec) && !(ABL & 8) && !kStStorerPub) {
        if (!hand_down(c)) return false;
        lag_stamp<DG>(a, t, c, lane, 0);
      }
    } else if (k == kStG - 1) {
      if (kStSpec) {
        // a guard failed somewhere in this chunk: recompute it with IEEE
        // division (rare: operands outside Markstein's exponent window)
        if (__any_sync(0xffffffffu, spec_bad)) redo_chunk(c);
        spec_bad = false;
        __syncwarp();
        if (!hand_down(c)) return false;
      } else if (kStChunkPub && !(ABL & 8)) {
        __syncwarp();  // lane 31's staged bottom rows -> the lanes that store them
        if (!hand_down(c)) return false;
        lag_stamp<DG>(a, t, c, lane, 0);
      }
      // chunk boundary: hand over the outputs and the input slot
      __syncwarp();
      if (lane == 0) {
        st_release_cta(ctl + kCtlOutReady, c + 1);
        st_release_cta(ctl + kCtlInDone, c + 1);
      }
    }
    return true;
  };

  // diagnostics: per-task globaltimer stamps (start, first chunk ready, end)
  long long* tstamp = (DG && a.dbg && lane == 0 && t < 1024) ? a.dbg + 6 * kStProbeChunks + 3 * t : nullptr;
  if (tstamp) tstamp[0] = (long long)globaltimer_ns();
  StBlk<EXACT, BD> buf[3];  // step s uses buf[s % 3] (indices static after unrolling)
  if (!solo && !wait_ctl(ctl, kCtlInReady, 1, deadline)) return abort_task(a, ctl, lane);
  if (above_in_cluster && lane == 0)
    for (int cc = 0; cc < kStInbox; ++cc) arm_inbox(cc);  // first phase of every slot
  __syncwarp();
  if (!solo && !wait_in(0, 0)) return abort_task(a, ctl, lane);
  if (tstamp) tstamp[1] = (long long)globaltimer_ns();
  static_assert(kStG >= 3, "the two-step lookahead stays within one chunk boundary");
  buf[0].load(smem, 0, 0, 0, lane);
  buf[1].load(smem, 0, 0, 1, lane);
  // three chunks per iteration so that s % 3 is a compile-time constant
  for (int c0 = 0; c0 < nchunks; c0 += 3) {
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int c = c0 + u;
      if (c >= nchunks) break;
#pragma unroll
      for (int k = 0; k < kStG; ++k)
        if (!step(c, k, buf[(u * kStG + k) % 3], buf[(u * kStG + k + 2) % 3])) return abort_task(a, ctl, lane);
    }
  }
  if (tstamp) tstamp[2] = (long long)globaltimer_ns();
}

// ---- prep tasks (BD kernels): bd = b * (1/d), band by band ------------------
// Prep task p of P takes every P-th double pair of each band, bands in order,
// so every band's bd is written by all prep CTAs at once (band 0 in ~2 us)
// and the wavefront (a band every ~5.7 us) never catches up. After its share
// of band t a CTA counts itself in bd_done[t]; the last one raises
// bdflag[t]. Prep tasks wait on nothing but the host copies of b (streamed
// host solves), so handing them out before any band keeps the pool
// deadlock-free.
__device__ void prep_task(const StArgs& a, int p, unsigned long long deadline) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const long long stride = (long long)a.prep_tasks * nthr;
  // (BD kernels solve one right-hand side: rd index = element index)
  const double* __restrict__ bin = a.b_in;
  const double* __restrict__ rdg = a.rdg;
  double* __restrict__ bd = a.bd;
  const bool pairs = ((reinterpret_cast<uintptr_t>(bin) & 15) == 0) && (a.nx % 2 == 0);
  constexpr int kU = 8;  // loads in flight per thread (a loop of dependent load/store pairs paid a DRAM
                         // round trip per pair: ~7.6 us per band, slower than the wavefront)
  // (a PE partition preps only its own bands, in its ticket order)
  const int n_prep = a.my_tasks ? a.n_my_tasks : a.n_tasks;
  for (int it = 0; it < n_prep; ++it) {
    const int t = a.my_tasks ? a.my_tasks[it] : it;
    if (a.bflag) {  // streamed host solve: band t's b may still be on its way
      __shared__ int ok_s;
      if (tid == 0) {
        const int fb = st_b_flag_band(a, t);
        int polls = 0, ok = 1;
        while ((int)(ld_acquire_sys_u32(a.bflag + fb) - a.epoch) < 0) {
          if ((++polls & 255) == 0 && ((deadline && globaltimer_ns() > deadline) || ld_relaxed_s32(a.abort_flag))) {
            ok = 0;
            break;
          }
          __nanosleep(256);
        }
        ok_s = ok;
      }
      __syncthreads();
      if (!ok_s) return;
    }
    const long long e0 = (long long)t * kStBand * a.nx, e1 = min((long long)(t + 1) * kStBand, (long long)a.ny) * a.nx;
    if (pairs) {
      const double2* b2 = reinterpret_cast<const double2*>(bin);
      const double2* r2 = reinterpret_cast<const double2*>(rdg);
      double2* d2 = reinterpret_cast<double2*>(bd);
      for (long long base = e0 / 2 + (long long)p * nthr + tid; base < e1 / 2; base += kU * stride) {
        double2 bv[kU], rv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const long long e = base + u * stride;
          if (e < e1 / 2) bv[u] = __ldg(b2 + e), rv[u] = __ldg(r2 + e);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const long long e = base + u * stride;
          if (e < e1 / 2) d2[e] = make_double2(__dmul_rn(bv[u].x, rv[u].x), __dmul_rn(bv[u].y, rv[u].y));
        }
      }
    } else {
      for (long long base = e0 + (long long)p * nthr + tid; base < e1; base += kU * stride) {
        double bv[kU], rv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const long long e = base + u * stride;
          if (e < e1) bv[u] = bin[e], rv[u] = __ldg(rdg + e);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const long long e = base + u * stride;
          if (e < e1) bd[e] = __dmul_rn(bv[u], rv[u]);
        }
      }
    }
    // the CTA's stores of band t, then one fence + count by thread 0 (the
    // other threads go on with band t + 1)
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (atomicAdd(a.bd_done + t, 1) == a.prep_tasks - 1) st_release_gpu_u32(a.bdflag + t, a.bd_epoch);
    }
  }
}

template <bool EXACT, int ABL, bool PART, int CL, bool DG, bool BD = false>
__global__ void __launch_bounds__(kStThreads, 1) k_stencil2d(const __grid_constant__ StArgs a) {
  using S = StSmem<EXACT>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // the 128-byte TMA swizzle repeats every 1024 bytes: align the rings to it
  // (the same offset in every CTA, so DSMEM addresses of peers line up)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  int* ctl = reinterpret_cast<int*>(smem + S::kCtl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + S::kBars);
    for (int k = 0; k < S::kSlots; ++k) mbar_init(&bars[k], 1 + kStLanes);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  unsigned phase_bits = 0;
  const unsigned long long deadline = a.timeout_ns ? globaltimer_ns() + a.timeout_ns : 0;
  const unsigned crank = CL > 1 ? cluster_ctarank() : 0u;
  // fresh out-slot barriers per task (every arrival of the previous task was
  // consumed by its storer before the task-end __syncthreads)
  auto init_out_bars = [&]() {
    if (!kStOutBar) return;
    unsigned long long* ob = reinterpret_cast<unsigned long long*>(smem + S::kOutBars);
    for (int k = 0; k < kStOutSlots; ++k) mbar_init(&ob[k], 1);
  };
  const int n_groups = (a.n_tasks + CL - 1) / CL;
  while (true) {
    if (CL > 1) {
      // a cluster takes kStCluster consecutive bands per ticket (ascending:
      // the progress rule, engine.py:30-35); its CTAs enter and leave a task
      // together, so no CTA resets counters a peer may still write
      cluster_sync_all();
      if (threadIdx.x == 0) {
        if (crank == 0) ctl[kCtlGroup] = ld_relaxed_s32(a.abort_flag) ? n_groups : atomicAdd(a.ticket, 1);
        ctl[kCtlInReady] = ctl[kCtlInDone] = ctl[kCtlOutReady] = ctl[kCtlOutDone] = ctl[kCtlAbort] = 0;
        ctl[kCtlMbReady] = ctl[kCtlPubDone] = 0;
        init_out_bars();
        // fresh inbox barriers for this task (no st.async of the previous one is pending:
        // the band above finished it before the cluster barrier)
        unsigned long long* ib = reinterpret_cast<unsigned long long*>(smem + S::kInBars);
        for (int k = 0; k < kStInbox; ++k) mbar_init(&ib[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      cluster_sync_all();
      if (threadIdx.x == 0) {
        const int g = ld_acquire_cluster_s32(mapa_shared(ctl + kCtlGroup, 0));
        ctl[kCtlTask] = g >= n_groups ? -1 : min(g * CL + (int)crank, a.n_tasks);  // n_tasks: idle this round
      }
    } else if (threadIdx.x == 0) {
      // ascending tickets: the progress rule (engine.py:30-35); BD kernels hand
      // out their prep tasks first (they wait on nothing the bands produce)
      const int k = atomicAdd(a.ticket, 1);
#if SPTRSV_ST_BD_BANDS_FIRST  // placement experiment only (not deadlock-safe without co-residency)
      const int kb = k;
      ctl[kCtlPrep] = (BD && k >= a.n_my_tasks && k < a.n_my_tasks + a.prep_tasks) ? k - a.n_my_tasks : -1;
      ctl[kCtlTask] = kb >= a.n_my_tasks ? -1 : (a.my_tasks ? a.my_tasks[kb] : kb);
#else
      const int kb = BD ? k - a.prep_tasks : k;
      ctl[kCtlPrep] = (BD && k < a.prep_tasks) ? k : -1;
      ctl[kCtlTask] = kb >= a.n_my_tasks ? -1 : kb < 0 ? a.n_tasks : (a.my_tasks ? a.my_tasks[kb] : kb);
#endif
      ctl[kCtlInReady] = ctl[kCtlInDone] = ctl[kCtlOutReady] = ctl[kCtlOutDone] = ctl[kCtlAbort] = 0;
      ctl[kCtlMbReady] = ctl[kCtlPubDone] = 0;
      init_out_bars();
    }
    __syncthreads();
    if (BD && CL == 1 && ctl[kCtlPrep] >= 0) {
      prep_task(a, ctl[kCtlPrep], deadline);
      __syncthreads();
      continue;
    }
    const int t = ctl[kCtlTask];
    if (t < 0) break;
    if (t < a.n_tasks) {
      const bool below_in_cluster = CL > 1 && crank + 1 < (unsigned)CL && st_has_below(a, t);
      if (warp == 0)
        compute<EXACT, ABL, PART, DG, BD>(a, smem, ctl, t, lane, deadline, crank, below_in_cluster, CL > 1 && crank > 0);
      else if (a.probe & 32) {  // diagnostics: the compute warp alone, on stale shared memory
      } else if (warp == 1) loader<EXACT, DG, BD>(a, smem, ctl, t, lane, phase_bits, deadline);
      else if (warp == 2) storer<EXACT, PART, DG>(a, smem, ctl, t, lane, deadline, crank, below_in_cluster);
      else if (warp == 4) publisher<EXACT, PART, DG>(a, smem, ctl, t, lane, deadline, crank, below_in_cluster);
      else poller<EXACT, DG>(a, smem, ctl, t, lane, deadline, CL > 1 && crank > 0);
    }
    __syncthreads();
    if (CL == 1 && ctl[kCtlAbort]) break;  // (clusters leave together, through the ticket)
  }
}

// Clusters resident at once for this kernel (cudaOccupancyMaxActiveClusters), per device.
template <typename K>
int max_active_clusters(K kernel, int cl, int smem_bytes) {
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && cache[dev] > 0) return cache[dev];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cl * 32, 1, 1);
  cfg.blockDim = dim3(kStThreads, 1, 1);
  cfg.dynamicSmemBytes = smem_bytes;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kernel, &cfg) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (dev < 64 && n > 0) cache[dev] = n;
  return n;
}

template <bool EXACT, int ABL, bool PART = false, int CL = 1, bool DG = false, bool BD = false>
cudaError_t launch_stencil_v(const StArgs& a, int blocks, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  if (cudaError_t e = set_max_dyn_smem(k_stencil2d<EXACT, ABL, PART, CL, DG, BD>, StSmem<EXACT>::kTotal, attr);
      e != cudaSuccess)
    return e;
  if (CL == 1) {
    k_stencil2d<EXACT, ABL, PART, CL, DG, BD><<<blocks, kStThreads, StSmem<EXACT>::kTotal, s>>>(a);
    return cudaGetLastError();
  }
  const int groups = (a.n_tasks + CL - 1) / CL;
  const int fit = max_active_clusters(k_stencil2d<EXACT, ABL, PART, CL, DG>, CL, StSmem<EXACT>::kTotal);
  if (fit < 1) return cudaErrorLaunchOutOfResources;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CL * std::min(groups, fit), 1, 1);
  cfg.blockDim = dim3(kStThreads, 1, 1);
  cfg.dynamicSmemBytes = StSmem<EXACT>::kTotal;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_stencil2d<EXACT, ABL, PART, CL, DG>, a);
}

// probe bits 12..15 select an ablation variant of the fast kernel (timing only)
template <bool EXACT>
cudaError_t launch_stencil(const StArgs& a, int blocks, cudaStream_t s) {
  if (a.band_owner) {
    if (!EXACT && a.prep_tasks > 0) return launch_stencil_v<EXACT, 0, true, 1, false, true>(a, blocks, s);
    return launch_stencil_v<EXACT, 0, true>(a, blocks, s);
  }
  if (!EXACT) {
    switch ((a.probe >> 12) & 15) {
      case 1: return launch_stencil_v<EXACT, 1>(a, blocks, s);
      case 2: return launch_stencil_v<EXACT, 2>(a, blocks, s);
      case 3: return launch_stencil_v<EXACT, 3>(a, blocks, s);
      case 4: return launch_stencil_v<EXACT, 4>(a, blocks, s);
      case 8: return launch_stencil_v<EXACT, 8>(a, blocks, s);
      case 15: return launch_stencil_v<EXACT, 15>(a, blocks, s);
      default: break;
    }
  }
  if (!EXACT && a.prep_tasks > 0) {  // pre-scaled right-hand side (BD)
    if (a.dbg) return launch_stencil_v<EXACT, 0, false, 1, true, true>(a, blocks, s);
    return launch_stencil_v<EXACT, 0, false, 1, false, true>(a, blocks, s);
  }
  // probe bit 16: the diagnostics build of the kernel (clock / globaltimer stamps)
  if (a.dbg) {
    if (kStCluster > 1 && a.n_tasks > 1) return launch_stencil_v<EXACT, 0, false, kStCluster, true>(a, blocks, s);
    return launch_stencil_v<EXACT, 0, false, 1, true>(a, blocks, s);
  }
  if (kStCluster > 1 && a.n_tasks > 1) return launch_stencil_v<EXACT, 0, false, kStCluster>(a, blocks, s);
  return launch_stencil_v<EXACT, 0>(a, blocks, s);
}

}  // namespace

// Pack the coefficient stream [task][step][field][pair][lane] (see
// stencil.hpp) from the CSR: one thread per (task, step, lane). Row i's
// entries are (i, i - nx) when y > 0 then (i, i - 1) when x > 0 (the
// detected structure). Padding elements get zero coefficients and, in exact
// mode, d = 1/d = 1 so the Markstein guard stays on the fast path.
__global__ void k_st_pack(const int* __restrict__ rp, const double* __restrict__ val, const double* __restrict__ dg,
                          const double* __restrict__ rdg, int nx, int ny, int n_tasks, int steps, int exact,
                          unsigned char* __restrict__ out) {
  const long long items = (long long)n_tasks * steps * kStLanes;
  const int nblk = nx / kStC, NF = exact ? 4 : 3, pairs = kStBlock / 2;
  const size_t step_doubles = (size_t)NF * pairs * kStLanes * 2;
  for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < items;
       it += (long long)gridDim.x * blockDim.x) {
    const int l = (int)(it % kStLanes);
    const long long ts = it / kStLanes;
    const int sidx = (int)(ts % steps), t = (int)(ts / steps);
    const int j = sidx - l;
    double* stepbuf = reinterpret_cast<double*>(out) + (size_t)ts * step_doubles;
#pragma unroll
    for (int r = 0; r < kStR; ++r) {
      const long long y = (long long)t * kStBand + kStR * l + r;
#pragma unroll
      for (int c = 0; c < kStC; ++c) {
        const int e_ = r * kStC + c, k = e_ / 2, half = e_ % 2;
        double f[4] = {0.0, 0.0, exact ? 1.0 : 0.0, exact ? 1.0 : 0.0};
        if (j >= 0 && j < nblk && y < ny) {
          const long long i = y * nx + (long long)j * kStC + c;
          int kk = rp[i];
          const double fu = y > 0 ? val[kk++] : 0.0;
          const double fl = (j * kStC + c) > 0 ? val[kk] : 0.0;
          f[0] = fu, f[1] = fl;
          if (exact) f[2] = dg[i], f[3] = rdg[i];
          else f[2] = rdg[i];
        }
        for (int fld = 0; fld < NF; ++fld) stepbuf[((fld * pairs + k) * kStLanes + l) * 2 + half] = f[fld];
      }
    }
  }
}

// Reset `count` mailbox words to kStNotReady (cuMemsetD32Async through the
// runtime's driver entry point).
static cudaError_t fill_not_ready(unsigned long long* p, long long count, cudaStream_t s) {
  typedef CUresult (*MemsetD32)(CUdeviceptr, unsigned int, size_t, CUstream);
  static MemsetD32 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemsetD32Async", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      f = nullptr;
    }
    return reinterpret_cast<MemsetD32>(f);
  }();
  if (!fn) return cudaErrorNotSupported;
  if (count <= 0) return cudaSuccess;
  return fn((CUdeviceptr)p, kStNotReady32, (size_t)count * 2, (CUstream)s) == CUDA_SUCCESS ? cudaSuccess
                                                                                          : cudaErrorUnknown;
}

// The skewed tensor view of b (see kStBTma); returns the number of bands it
// covers (the full ones), 0 when the driver entry point or the encode fails.
static int encode_b_map(CUtensorMap* map, const double* b, int nx, int ny) {
  typedef CUresult (*Encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      f = nullptr;
    }
    return reinterpret_cast<Encode>(f);
  }();
  static const bool disabled = std::getenv("SPTRSV_NO_B_TMA") != nullptr;  // A/B diagnostics
  const int bands = ny / kStBand;
  if (!encode || disabled || bands < 1 || nx < kStLanes * kStC) return 0;
  const cuuint64_t dims[4] = {(cuuint64_t)nx + (kStLanes - 1) * kStC, (cuuint64_t)kStLanes, (cuuint64_t)kStR,
                              (cuuint64_t)bands};
  const cuuint64_t strides[3] = {(cuuint64_t)(kStR * nx - kStC) * 8, (cuuint64_t)nx * 8,
                                 (cuuint64_t)kStBand * nx * 8};
  const cuuint32_t box[4] = {kStG * kStC, kStLanes, kStR, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  if (encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(b), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 0;
  return bands;
}

// Detect the 2D five-point lower structure on the host CSR; returns nx or 0.
int detect_stencil2d(long long n, const std::vector<int>& rp, const std::vector<int>& ci) {
  if (n < 4) return 0;
  long long nx = 0;
  for (long long i = 1; i < n && !nx; ++i)
    for (int k = rp[i]; k < rp[i + 1]; ++k)
      if (i - ci[k] > 1) {
        nx = i - ci[k];
        break;
      }
  if (nx < 2 || nx % kStC != 0 || n % nx != 0 || nx > (1 << 28)) return 0;
  for (long long i = 0; i < n; ++i) {
    const long long x = i % nx, y = i / nx;
    int k = rp[i];
    if (y > 0) {
      if (k >= rp[i + 1] || ci[k] != i - nx) return 0;
      ++k;
    }
    if (x > 0) {
      if (k >= rp[i + 1] || ci[k] != i - 1) return 0;
      ++k;
    }
    if (k != rp[i + 1]) return 0;
  }
  return (int)nx;
}

int DevicePlan::build_stencil(const std::vector<int>& h_rp, const std::vector<int>& h_ci) {
  auto t0 = std::chrono::steady_clock::now();
  stencil.release();
  const int nx = detect_stencil2d(n, h_rp, h_ci);
  if (!nx) return SPTRSV_OK;
  const bool exact = opt.precision != SPTRSV_PRECISION_FAST;
  stencil.exact = exact;
  stencil.nx = nx;
  stencil.ny = (int)(n / nx);
  stencil.n_tasks = (stencil.ny + kStBand - 1) / kStBand;
  const int raw_steps = nx / kStC + kStLanes - 1;
  stencil.steps_per_task = (raw_steps + kStG - 1) / kStG * kStG;
  const int NF = st_fields(exact);
  const size_t step_bytes = st_step_bytes(exact);
  const size_t bytes = step_bytes * stencil.steps_per_task * stencil.n_tasks;
  cudaError_t e;
  auto al = [](void** p, size_t b) { return cudaMalloc(p, b < 16 ? 16 : b); };
  if ((e = al((void**)&stencil.stream, bytes)) != cudaSuccess ||
      (e = al((void**)&stencil.mbox, 2 * sizeof(unsigned long long) * (size_t)stencil.n_tasks * nx)) != cudaSuccess ||
      (e = fill_not_ready(stencil.mbox, 2ll * stencil.n_tasks * nx, 0)) != cudaSuccess ||
      (e = cudaDeviceSynchronize()) != cudaSuccess ||
      (e = al((void**)&stencil.bflag, sizeof(unsigned) * stencil.n_tasks)) != cudaSuccess ||
      (e = al((void**)&stencil.xflag, sizeof(unsigned) * stencil.n_tasks)) != cudaSuccess ||
      (e = cudaMemset(stencil.bflag, 0, sizeof(unsigned) * stencil.n_tasks)) != cudaSuccess ||
      (e = cudaMemset(stencil.xflag, 0, sizeof(unsigned) * stencil.n_tasks)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  // load the flag-release kernel now: under lazy module loading its first
  // launch would otherwise wait for the device while the solve kernel spins
  // on b flags that only later copies write (a deadlock until the watchdog)
  if ((e = stencil_release_flags(stencil.xflag, stencil.n_tasks, 0u, stream)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  // the coefficient stream is packed on the device from the CSR (one thread
  // per lane-step, no host round trip of the values)
  {
    const long long items = (long long)stencil.n_tasks * stencil.steps_per_task * kStLanes;
    const int grid = (int)std::min<long long>((items + 255) / 256, 148 * 64);
    k_st_pack<<<grid, 256, 0, stream>>>(rp, exact ? cv : wv, dg, rdg, nx, stencil.ny, stencil.n_tasks,
                                        stencil.steps_per_task, exact ? 1 : 0, stencil.stream);
    if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaStreamSynchronize(stream)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  }
  stencil.n_my_tasks = stencil.n_tasks;
  stencil.stream_bytes = (long long)bytes;
  stencil.ready = true;
  stencil.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return SPTRSV_OK;
}

// Streamed host solves: after the kernel, every band's x flag is set to the
// epoch (one launch), so a copy stream waiting on them never hangs when the
// kernel stopped early (timeout / abort); normally the storers already did.
__global__ void k_set_flags(unsigned* f, int n, unsigned v) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) st_release_sys_u32(f + i, v);
}
cudaError_t stencil_release_flags(unsigned* f, int n, unsigned v, cudaStream_t s) {
  k_set_flags<<<1, 128, 0, s>>>(f, n, v);
  return cudaGetLastError();
}

// Error contraction per grid row of the fast recurrence x = bd + a x_left +
// u x_up (a = -L[i,i-1]/L_ii, u = -L[i,i-nx]/L_ii): a solve started from a
// zero row r0 - 1 instead of the true one errs by e with
// |e_{r,c}| <= A |e_{r,c-1}| + U max|e_{r-1,.}|, e_{r,-1} = 0, so row r's
// error is at most gamma = U / (1 - A) times row r - 1's (A, U: the largest
// |a|, |u|). Device max-reduction over the pre-scaled entries.
__global__ void k_st_decay(const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ wv,
                           long long n, unsigned long long* __restrict__ amax) {
  unsigned long long ma = 0, mu = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(wv[k]));  // NaN sorts above
      if (ci[k] == i - 1) ma = max(ma, bits);
      else mu = max(mu, bits);
    }
  atomicMax(amax, ma);
  atomicMax(amax + 1, mu);
}

int DevicePlan::stencil_groups(cudaStream_t s) {
  // SPTRSV_ST_GROUP: bands per group (0: one chain of every band)
  static const int want = [] {
    const char* v = std::getenv("SPTRSV_ST_GROUP");
    return v ? std::atoi(v) : kStGroupDefault;
  }();
  const int nb = stencil.n_tasks;
  // the bands this plan solves: all of them, or this PE's under a partition
  // (whose first band is then entered through a local halo instead of the
  // peer's mailboxes: a fast PE solve reads nothing from other GPUs)
  std::vector<int> bands;
  if (stencil.part) bands = stencil.host_my_tasks;
  else for (int b = 0; b < nb; ++b) bands.push_back(b);
  if (want <= 0 || bands.empty() || (!stencil.part && nb <= want) || !wv || !rp || !ci) return 0;
  cudaError_t e;
  if (stencil.decay < 0.0) {
    unsigned long long* d = nullptr;
    unsigned long long h[2] = {0, 0};
    if ((e = cudaMalloc((void**)&d, 2 * sizeof(unsigned long long))) != cudaSuccess ||
        (e = cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), s)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e)), -1;
    k_st_decay<<<num_sms * 4, 256, 0, s>>>(rp, ci, wv, n, d);
    if ((e = cudaGetLastError()) != cudaSuccess ||
        (e = cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaStreamSynchronize(s)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e)), -1;
    cudaFree(d);
    double A, U;
    std::memcpy(&A, &h[0], 8);
    std::memcpy(&U, &h[1], 8);
    stencil.decay = (A < 1.0 && U == U) ? U / (1.0 - A) : 1e300;
  }
  // one halo band of 64 rows: the entering error is <= decay^64 |x|; groups
  // only when that is <= 2^-64 (decay <= 1/2; lap2d: 1/3, i.e. 3e-31)
  if (!(stencil.decay <= 0.5)) return 0;
  if (stencil.grp != want || stencil.grp_bands != bands) {
    // groups of up to `want` consecutive bands; a group not starting at band 0
    // is entered through a halo task (band b0 - 1 from a zero row above)
    std::vector<int> tb;
    for (size_t k = 0; k < bands.size();) {
      const int b0 = bands[k];
      if (b0 > 0) tb.push_back(-(b0 - 1) - 1);
      int len = 0;
      while (k < bands.size() && len < want && bands[k] == b0 + len) tb.push_back(bands[k++]), ++len;
    }
    if (stencil.tband) cudaFree(stencil.tband);
    if (stencil.mbox_grp) cudaFree(stencil.mbox_grp);
    stencil.tband = nullptr;
    stencil.mbox_grp = nullptr;
    const long long words = 2ll * (long long)tb.size() * stencil.nx;
    if ((e = cudaMalloc((void**)&stencil.tband, sizeof(int) * tb.size())) != cudaSuccess ||
        (e = cudaMemcpy(stencil.tband, tb.data(), sizeof(int) * tb.size(), cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMalloc((void**)&stencil.mbox_grp, sizeof(unsigned long long) * words)) != cudaSuccess ||
        (e = fill_not_ready(stencil.mbox_grp, words, s)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e)), -1;
    stencil.grp = want;
    stencil.grp_bands = bands;
    stencil.grp_tasks = (int)tb.size();
    stencil.grp_solves = 0;
  }
  return 1;
}

int DevicePlan::solve_stencil(const double* d_b, double* d_x, cudaStream_t s, bool b_flags, bool x_flags,
                              int copies) {
  if (!stencil.ready) return plan_fail(SPTRSV_E_UNSUPPORTED, "matrix is not 2D five-point lower structured");
  cudaError_t e;
  // k right-hand sides stacked into one grid of k * ny rows (full bands only)
  const bool many = copies > 1;
  if (many && (stencil.part || b_flags || x_flags || stencil.ny % kStBand != 0))
    return plan_fail(SPTRSV_E_UNSUPPORTED, "stacked right-hand sides need whole bands and a one-PE plan");
  if (many && copies > stencil.many_k) {
    if (stencil.mbox_many) cudaFree(stencil.mbox_many);
    stencil.mbox_many = nullptr;
    stencil.many_k = 0;
    const long long words = 2ll * copies * stencil.n_tasks * stencil.nx;
    if ((e = cudaMalloc((void**)&stencil.mbox_many, sizeof(unsigned long long) * words)) != cudaSuccess ||
        (e = fill_not_ready(stencil.mbox_many, words, s)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    stencil.many_k = copies;
    stencil.many_solves = 0;
    stencil.many_last = copies;
  }
  if (many && copies != stencil.many_last) {
    // each solve re-arms (for the next one) only the rows its own copies used
    if ((e = fill_not_ready(stencil.mbox_many, 2ll * stencil.many_k * stencil.n_tasks * stencil.nx, s)) !=
        cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    stencil.many_last = copies;
    stencil.many_solves = 0;
  }
  // fast mode, one right-hand side: bands in independent groups (under a PE
  // partition: this PE's bands, no peer reads)
  int grouped = 0;
  if (!stencil.exact && !many && kStCluster == 1) {
    grouped = stencil_groups(s);
    if (grouped < 0) return SPTRSV_E_CUDA;
  }
  const int n_tasks = grouped ? stencil.grp_tasks : stencil.n_tasks * (many ? copies : 1);
  unsigned long long* mbox = grouped ? stencil.mbox_grp : many ? stencil.mbox_many : stencil.mbox;
  // (the stacked mailboxes keep their halves at the allocated size)
  const long long half =
      (long long)(grouped ? stencil.grp_tasks : many ? stencil.many_k * stencil.n_tasks : stencil.n_tasks) * stencil.nx;
  const int par = (int)((grouped ? stencil.grp_solves : many ? stencil.many_solves : stencil.solves) & 1);
  if (stencil.part && !grouped) {
    for (int t : stencil.host_my_tasks)
      if (t > 0 && !stencil.host_pe_mbox[stencil.host_band_owner[t - 1]])
        return plan_fail(SPTRSV_E_INVALID_PE, "the mailboxes of a peer PE were never imported");
  }
  // this solve uses mailbox half `par` (reset by the previous solve or at
  // build); reset the other half for the next one
  if ((e = reset_control(s)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  StArgs a{};
  a.stream = stencil.stream;
  a.debug = (opt.flags & SPTRSV_PLAN_DEBUG) != 0;
  a.mbox = mbox + par * half;
  a.mbox_next = mbox + (1 - par) * half;
  a.mbox_half = par * half;
  a.ticket = ticket;
  a.n_my_tasks = n_tasks;
  a.my_pe = -1;
  if (stencil.part && !grouped) {
    a.my_tasks = stencil.my_tasks;
    a.n_my_tasks = stencil.n_my_tasks;
    a.pe_mbox = stencil.pe_mbox;
    a.band_owner = stencil.band_owner;
    a.my_pe = stencil.my_pe;
  }
  // fast mode, one right-hand side, one PE: the BD kernel (its prep tasks
  // write bd = b * (1/d) on the SMs the 64 bands leave idle; SPTRSV_NO_BD=1
  // keeps the multiply in the step, diagnostics)
  static const bool no_bd = std::getenv("SPTRSV_NO_BD") != nullptr;
  const bool bd_mode = !stencil.exact && !many && kStCluster == 1 && !no_bd && !grouped;
  if (bd_mode) {
    if (!stencil.bd) {
      if ((e = cudaMalloc((void**)&stencil.bd, sizeof(double) * (size_t)n)) != cudaSuccess ||
          (e = cudaMalloc((void**)&stencil.bdflag, sizeof(unsigned) * stencil.n_tasks)) != cudaSuccess ||
          (e = cudaMalloc((void**)&stencil.bd_done, sizeof(int) * stencil.n_tasks)) != cudaSuccess ||
          (e = cudaMemsetAsync(stencil.bdflag, 0, sizeof(unsigned) * stencil.n_tasks, s)) != cudaSuccess)
        return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    }
    if ((e = cudaMemsetAsync(stencil.bd_done, 0, sizeof(int) * stencil.n_tasks, s)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    a.b_in = d_b;
    a.bd = stencil.bd;
    a.rdg = rdg;
    a.bdflag = stencil.bdflag;
    a.bd_done = stencil.bd_done;
    a.bd_epoch = ++stencil.bd_epoch;
    if (a.bd_epoch == 0) a.bd_epoch = ++stencil.bd_epoch;  // (0 is the flags' initial value)
    a.n_copy = n;
    d_b = stencil.bd;  // the loaders stream bd (aligned) instead of b
  }
  a.b = d_b;
  a.x = d_x;
  a.status = status;
  a.abort_flag = abort_flag;
  a.timeout_ns = (unsigned long long)(opt.timeout_s * 1e9);
  a.spin_initial = opt.spin_initial;
  a.spin_max_ns = opt.spin_max_ns;
  a.nx = stencil.nx;
  a.ny = stencil.ny * (many ? copies : 1);
  a.n_tasks = n_tasks;
  // (grouped: only task 0 may be "first of a right-hand side", and the
  // coefficient stream index band % bands must not wrap for a PE's bands)
  a.bands = grouped ? std::max(n_tasks, stencil.n_tasks) : stencil.n_tasks;
  a.n_bands = stencil.n_tasks;
  a.tband = grouped ? stencil.tband : nullptr;
  a.steps = stencil.steps_per_task;
  a.probe = opt.probe_flags;
  a.b_aligned = ((uintptr_t)d_b & 15) == 0;
  a.b_tma_bands = (kStBTma && a.b_aligned) ? encode_b_map(&a.bmap, d_b, stencil.nx, a.ny) : 0;
  a.x_aligned = ((uintptr_t)d_x & 15) == 0;
  a.x_tma_bands = (SPTRSV_ST_X_TMA && kStBTma && a.x_aligned) ? encode_b_map(&a.xmap, d_x, stencil.nx, a.ny) : 0;
  if (b_flags) a.bflag = stencil.bflag;
  if (x_flags) a.xflag = stencil.xflag;
  a.epoch = stencil.epoch;
  a.b_chunk_max = b_flags ? stencil.b_chunk_max : 0;
  a.nap = (opt.probe_flags & 4) ? (opt.probe_flags >> 8) & 1023 : 64;  // probe bit 4: override the nap
  if (opt.probe_flags & 16) {
    if (!probe_buf && cudaMalloc((void**)&probe_buf, sizeof(long long) * kProbeWords) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, "probe buffer");
    cudaMemsetAsync(probe_buf, 0, sizeof(long long) * kProbeWords, s);
    a.dbg = probe_buf;
  }
  int blocks = std::max(1, std::min(a.n_my_tasks, grid_cap > 0 ? std::min(grid_cap, num_sms) : num_sms));
  if (bd_mode) {
    // the SMs the bands leave idle do the prep (at least 16 prep tasks)
    const int sms = grid_cap > 0 ? std::min(grid_cap, num_sms) : num_sms;
    a.prep_tasks = std::max(16, sms - std::min(a.n_my_tasks, sms));
    blocks = std::min(a.n_my_tasks + a.prep_tasks, std::max(sms, a.prep_tasks + 1));
  }
  ++(grouped ? stencil.grp_solves : many ? stencil.many_solves : stencil.solves);
  group_tasks_used = grouped ? stencil.grp_tasks : 0;
  if ((e = record_k0(s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  e = stencil.exact ? launch_stencil<true>(a, blocks, s) : launch_stencil<false>(a, blocks, s);
  if (e != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if ((e = cudaEventRecord(evk1, s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  launches = 1;
  return SPTRSV_OK;
}

// Band-aligned owner map, one PE per process: returns 1 when configured, 0
// when some band is split between PEs (the caller falls back to the
// component pool), < 0 on error.
int DevicePlan::set_stencil_partition(const int32_t* owner, int pes, int my_pe) {
  const long long band = (long long)kStBand * stencil.nx;
  std::vector<int> bo(stencil.n_tasks), mine;
  for (int t = 0; t < stencil.n_tasks; ++t) {
    const long long i0 = t * band, i1 = std::min(n, i0 + band);
    const int o = owner[i0];
    for (long long i = i0 + 1; i < i1; ++i)
      if (owner[i] != o) return 0;
    bo[t] = o;
    if (o == my_pe) mine.push_back(t);
  }
  stencil.release_part();
  auto al = [](void** p, size_t b) { return cudaMalloc(p, b < 16 ? 16 : b); };
  std::vector<unsigned char> bo8(bo.begin(), bo.end());
  cudaError_t e;
  if ((e = al((void**)&stencil.my_tasks, sizeof(int) * mine.size())) != cudaSuccess ||
      (e = al((void**)&stencil.band_owner, bo8.size())) != cudaSuccess ||
      (e = al((void**)&stencil.pe_mbox, sizeof(void*) * pes)) != cudaSuccess ||
      (!mine.empty() &&
       (e = cudaMemcpy(stencil.my_tasks, mine.data(), sizeof(int) * mine.size(), cudaMemcpyHostToDevice)) !=
           cudaSuccess) ||
      (e = cudaMemcpy(stencil.band_owner, bo8.data(), bo8.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  stencil.host_pe_mbox.assign(pes, nullptr);
  stencil.host_pe_mbox[my_pe] = stencil.mbox;
  stencil.host_band_owner = bo;
  stencil.host_my_tasks = mine;
  stencil.n_my_tasks = (int)mine.size();
  stencil.my_pe = my_pe;
  stencil.n_pes = pes;
  stencil.part = true;
  return stencil_sync_peers() == SPTRSV_OK ? 1 : -1;
}

int DevicePlan::stencil_sync_peers() {
  cudaError_t e = cudaMemcpy(stencil.pe_mbox, stencil.host_pe_mbox.data(), sizeof(void*) * stencil.n_pes,
                             cudaMemcpyHostToDevice);
  return e == cudaSuccess ? SPTRSV_OK : plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
}

}  // namespace sptrsv
