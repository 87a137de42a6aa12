// Fast-mode band executor by row blocks (banded-8M: bandwidth 64, ~4.7 M
// levels for 8.4 M rows).
//
// The window kernel (solve_band.cu) is one warp walking every column in order:
// a shuffle and an FMA per row on one SM, ~67 ns a row, 0.32 s for 8.4 M rows.
// Fast mode (pre-scaled rows, FMA; the 1e-12 contract) may re-associate, so
// the recurrence is cut into row blocks of S rows (k = 0 .. nblk-1, rows
// [kS, kS + S)). With bandwidth W = 64 a block depends on the blocks before
// it only through x of the W rows just above it (the previous block's tail):
//
//   x_k = c_k + N_k t_{k-1},   c_k = (I - W_kk)^{-1} (rd * b)_k,
//                              t_{k-1} = x of rows [kS - W, kS)
//
// where N_k (S x W) is how x_k responds to the W coupling values (built once
// per plan, only its W x W tail is kept). One solve is then three kernels:
//   K1  every block in parallel, one warp each: the band window sweep of the
//       block with zero coupling; keeps c of the block's tail rows;
//   K2  one CTA, nblk - 1 sequential steps: t_k = c_k^tail + N_k^tail t_{k-1}
//       (a 64 x 64 matvec per step from a TMA-fed ring) -- the only
//       sequential part, nblk steps instead of n rows;
//   K3  every block in parallel again: the same sweep, its first W rows
//       seeded with the coupling terms of t_{k-1}; writes x.
// K1 and K3 each stream the dense band once (HBM-bound); K2 is latency-bound
// at ~250 cycles per step. Exact mode keeps the column-ordered window kernel
// (the serial oracle's summation order).
#include <algorithm>
#include <cstdlib>
#include <vector>
#include "plan.hpp"
#include "kernels.cuh"
#include "ptx.cuh"

namespace sptrsv {

int plan_fail(int code, const char* msg);

namespace {

constexpr int kW = 64;           // bandwidth = window
constexpr int kBBWarps = 4;      // sweep warps per CTA (one block each)
// the sweeps read the packed band (SPTRSV_BB_PACKED=1: the stored entries
// only, located through the presence mask staged per window in shared memory
// -- half the bytes, 2.3 GB per sweep, but the data-dependent gathers made
// K1 2.14 ms against 1.13 ms on the dense band) or the dense one (default)
#ifndef SPTRSV_BB_PACKED
#define SPTRSV_BB_PACKED 0
#endif
constexpr bool kBBPacked = SPTRSV_BB_PACKED;
#ifndef SPTRSV_BB_PF
#define SPTRSV_BB_PF 16
#endif
constexpr int kPf = SPTRSV_BB_PF;  // coefficient prefetch distance (columns)
#ifndef SPTRSV_BB_TSLOTS
#define SPTRSV_BB_TSLOTS 4
#endif
constexpr int kTSlots = SPTRSV_BB_TSLOTS;  // K2 ring depth (steps)
constexpr int kTailBytes = kW * kW * 8;

// ---- setup: the packed band ------------------------------------------------
__global__ void k_bb_popc(const unsigned long long* __restrict__ mask, long long n, int* __restrict__ cnt) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x)
    cnt[j] = __popcll(mask[j]);
}
__global__ void k_bb_pack(const double* __restrict__ coef, const unsigned long long* __restrict__ mask,
                          const int* __restrict__ off, long long n, double* __restrict__ pk) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    unsigned long long m = mask[j];
    int o = off[j];
    while (m) {
      const int bit = __ffsll((long long)m) - 1;
      m &= m - 1;
      pk[o++] = coef[(size_t)j * kW + bit];
    }
  }
}

// ---- setup: N_k tail ------------------------------------------------------
// One CTA of two warps per block; lane m (of warp h) follows coupling column
// m = 32h + lane: its response N[i][m] for the block's rows i, in a window of
// 64 register accumulators (row i at slot i mod 64), pushed column by column
// exactly like the solve: N[j][m] is final when column j is reached, then
// acc[i] += w_ij N[j][m] for i = j+1 .. j+64. The band columns are staged in
// shared memory (broadcast reads). Output layout (K2's): [h][i][r] of double2
// (m = 32h + 2i + e), r = tail row.
constexpr int kNtSmem = 2 * kW * kW * 8;  // two 64-column chunks of the band

// Coupling reach (fast mode): a row whose response to every coupling value
// is <= kReachTau (2^-64) takes x = c, since the dropped N t is below
// 64 * 2^-64 |t| (~3.5e-18 of the tail's magnitude, far under the sweep's own
// rounding); reach[k] = 1 + the last row of block k above it, so K3 sweeps
// rows [0, reach[k]) of the block (rounded up to whole 64-column windows:
// the sweep writes every column of a window it enters) and K1's c stands
// beyond.
constexpr double kReachTau = 5.421010862427522e-20;  // 2^-64

__global__ void __launch_bounds__(64) k_bb_ntail(const double* __restrict__ coef, long long n, int S, int nblk,
                                                 double* __restrict__ nt, int* __restrict__ reach) {
  extern __shared__ __align__(16) double cs_raw[];
  double (*cs)[kW][kW] = reinterpret_cast<double (*)[kW][kW]>(cs_raw);
  // blocks 1 .. nblk - 2: block 0 has no coupling and the last block's tail
  // feeds no further block (it is also the only block that may be partial)
  const int k = blockIdx.x + 1;
  // the last block (launched only when it is whole: reach) feeds no tail
  if (k > nblk - 1 || (k == nblk - 1 && (long long)k * S + S > n)) return;
  const long long s0 = (long long)k * S;
  const int tid = threadIdx.x, h = tid >> 5, lane = tid & 31, m = 32 * h + lane;
  double acc[kW];
#pragma unroll
  for (int u = 0; u < kW; ++u) acc[u] = 0.0;
  const int nchunk = S / kW + 1;  // the coupling columns [s0 - 64, s0), then the block's
  auto stage = [&](int c, int buf) {
    const double2* src = reinterpret_cast<const double2*>(coef + (size_t)(s0 - kW + (long long)c * kW) * kW);
    double2* dst = reinterpret_cast<double2*>(&cs[buf][0][0]);
    for (int w = tid; w < kW * kW / 2; w += 64) dst[w] = src[w];
  };
  stage(0, 0);
  __syncthreads();
  int last = 0;  // 1 + the last row of the block whose response to coupling m exceeds kReachTau
  for (int c = 0; c < nchunk; ++c) {
    if (c + 1 < nchunk) stage(c + 1, (c + 1) & 1);
#pragma unroll
    for (int u = 0; u < kW; ++u) {
      const long long j = s0 - kW + (long long)c * kW + u;
      // coupling column s0 - 64 + m has response 1 in lane m, 0 elsewhere
      const double nj = c == 0 ? (u == m ? 1.0 : 0.0) : acc[u];
      // (NaN / inf responses compare false: keep the whole block then)
      if (c > 0 && j < n && !(fabs(nj) <= kReachTau)) last = (int)(j - s0) + 1;
      if (c > 0 && j >= s0 + S - kW && j < n) {
        const int r = (int)(j - (s0 + S - kW)), i = (m & 31) >> 1, e = m & 1;
        nt[(size_t)(k - 1) * (kTailBytes / 8) + ((h * 16 + i) * kW + r) * 2 + e] = nj;
      }
      acc[u] = 0.0;  // row j leaves the window; row j + 64 enters in its slot
      const double* cj = &cs[c & 1][u][0];
#pragma unroll
      for (int d = 1; d <= kW; ++d) acc[(u + d) & (kW - 1)] = __fma_rn(cj[d - 1], nj, acc[(u + d) & (kW - 1)]);
    }
    __syncthreads();
  }
  if (reach) atomicMax(reach + k, last);
}

// ---- K1 / K3: one warp per block, the band window sweep --------------------
struct SweepArgs {
  const double* coef;  // [n_pad][64]: w(j + d, j) at [j][d - 1] (pre-scaled, fast mode)
  const double* pk;    // packed: column j's stored entries in row order at pk[off[j] ..]
  const int* off;
  const unsigned long long* mask;  // bit d - 1 of mask[j]: (j + d, j) is stored
  const double* b;
  const double* rdg;
  const double* tt;    // K3: t_k = x of block k's tail rows, [nblk][64] (null in K1)
  double* out;         // K1: c tails [nblk][64]; K3: x
  double* x_all;       // K1: also c of every row into x (coupling reach in use), else null
  const int* reach;    // K3: rows of block k the coupling reaches (null: all)
  long long n;
  int S, nblk;
  int k_begin, k_end;  // the blocks of this PE (all blocks without a partition)
};

template <bool COUPLED>
__global__ void __launch_bounds__(32 * kBBWarps) k_bb_sweep(const __grid_constant__ SweepArgs a) {
  const int lane = threadIdx.x & 31;
  const int k = a.k_begin + blockIdx.x * kBBWarps + (threadIdx.x >> 5);
  if (k >= a.k_end) return;
  const long long s0 = (long long)k * a.S, s1 = std::min<long long>(s0 + a.S, a.n);
  // lane owns window rows 2 lane + s (s = 0, 1) of each 64-row window
  double acc[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const long long i = s0 + 2 * lane + s;
    acc[s] = i < s1 ? __dmul_rn(a.b[i], a.rdg[i]) : 0.0;
    if (COUPLED && k > 0 && i < s1) {
      // coupling terms of the previous block's tail: sum_{j in [s0-64, s0)} w_ij t_j,
      // in ascending column order
      const double* tp = a.tt + (size_t)(k - 1) * kW;
      for (int q = 0; q < kW; ++q) {
        const long long j = s0 - kW + q;
        const long long d = i - j;
        if (d >= 1 && d <= kW) acc[s] = __fma_rn(a.coef[(size_t)j * kW + d - 1], tp[q], acc[s]);
      }
    }
  }
  // next window's b * rd of the lane's rows (one iteration ahead)
  double nb[2];
  const int ncol = (int)(COUPLED && a.reach ? std::min<long long>(s1 - s0, (a.reach[k] + kW - 1) / kW * kW) : s1 - s0);
  // coefficient register ring: column j's two entries of this lane, kPf columns ahead
  double cf[kPf][2];
  // packed: the presence masks and offsets of windows w .. w + 2 staged in
  // this warp's shared-memory ring by cp.async two windows ahead, so a
  // column's entry loads do not wait on a global load of its mask
  __shared__ unsigned long long s_mask[kBBWarps][3][kW];
  __shared__ int s_off[kBBWarps][3][kW];
  const int wq = threadIdx.x >> 5;
  auto stage = [&](int w) {  // window w's masks / offsets (columns beyond n are never read)
    if (kBBPacked) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const long long col = s0 + (long long)w * kW + h * 32 + lane;
        if (col < a.n) {
          cp_async8(&s_mask[wq][w % 3][h * 32 + lane], a.mask + col);
          cp_async4(&s_off[wq][w % 3][h * 32 + lane], a.off + col);
        }
      }
      cp_async_commit();
    }
  };
  auto cload = [&](long long j, double (&dst)[2], int p) {
    if (kBBPacked) {
      // the column's presence mask and offset (broadcast shared loads), then
      // the lane's entries from the packed stream
      const int rel = (int)(j - s0), ws = (rel / kW) % 3, wi = rel % kW;
      const unsigned long long m = j < s1 ? s_mask[wq][ws][wi] : 0ull;
      const int o = j < s1 ? s_off[wq][ws][wi] : 0;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int bit = (2 * lane + s - p - 1) & (kW - 1);
        const bool present = (m >> bit) & 1ull;
        dst[s] = present ? __ldg(a.pk + o + __popcll(m & ((1ull << bit) - 1ull))) : 0.0;
      }
      return;
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int d = ((2 * lane + s - p - 1) & (kW - 1)) + 1;
      dst[s] = j < s1 ? __ldg(a.coef + (size_t)j * kW + d - 1) : 0.0;
    }
  };
  stage(0);
  stage(1);
  cp_async_wait<0>();
  __syncwarp();
#pragma unroll
  for (int u = 0; u < kPf; ++u) cload(s0 + u, cf[u], u);
  for (int c0 = 0; c0 < ncol; c0 += kW) {
    if (kBBPacked && c0 > 0) {
      // window w + 1 (staged a window ago) must have landed; window w + 2 starts
      stage(c0 / kW + 2);
      cp_async_wait<1>();
      __syncwarp();
    } else if (kBBPacked) {
      stage(2);
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const long long i = s0 + c0 + kW + 2 * lane + s;
      nb[s] = i < s1 ? __dmul_rn(__ldg(a.b + i), __ldg(a.rdg + i)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kW; ++u) {
      const long long j = s0 + c0 + u;
      const int owner = u >> 1, os = u & 1;
      double w[2] = {cf[u % kPf][0], cf[u % kPf][1]};
      cload(j + kPf, cf[u % kPf], (u + kPf) & (kW - 1));
      const double xj = __shfl_sync(0xffffffffu, os ? acc[1] : acc[0], owner);
      if (lane == owner && j < s1) {
        if (COUPLED) {
          a.out[j] = xj;
        } else {
          if (a.x_all) a.x_all[j] = xj;
          if (j >= s0 + a.S - kW)
          a.out[(size_t)k * kW + (j - (s0 + a.S - kW))] = xj;  // c of the tail rows
        }
      }
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        double v = acc[s];
        if (lane == owner && s == os) v = nb[s];  // row j leaves, row j + 64 enters
        acc[s] = __fma_rn(w[s], xj, v);
      }
    }
  }
}

// ---- K1 / K3 with the band streamed by TMA ----------------------------------
// The same sweep, but each warp's coefficient stream (its block's columns, one
// contiguous 2 MB run for S = 4096) arrives in a shared-memory ring of kRing
// chunks of kCw columns by bulk copies issued kRing chunks ahead, instead of
// a register ring of kPf columns of 8-byte global loads (~1 us of HBM latency
// against ~16 columns of sweep). Column j + 2's two entries per lane are read
// from shared memory while column j is swept.
constexpr int kCw = 8;                       // columns per chunk (4 KB)
#ifndef SPTRSV_BB_RING
#define SPTRSV_BB_RING 3
#endif
// chunks per warp ring: 3 (12 KB per warp) lets four CTAs share an SM, so the
// 2,048 blocks of banded-8M run in one wave (16 warps per SM)
constexpr int kRing = SPTRSV_BB_RING;
constexpr int kChunkBytes = kCw * kW * 8;
constexpr int kRingSmem = kBBWarps * (kRing * kChunkBytes + 8 * kRing);

template <bool COUPLED>
__global__ void __launch_bounds__(32 * kBBWarps) k_bb_sweep_tma(const __grid_constant__ SweepArgs a) {
  extern __shared__ __align__(128) unsigned char rsm[];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int k = a.k_begin + blockIdx.x * kBBWarps + wq;
  unsigned char* ring = rsm + wq * kRing * kChunkBytes;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(rsm + kBBWarps * kRing * kChunkBytes) + wq * kRing;
  if (k >= a.k_end) return;
  const long long s0 = (long long)k * a.S, s1 = std::min<long long>(s0 + a.S, a.n);
  const int ncol = (int)(COUPLED && a.reach ? std::min<long long>(s1 - s0, (a.reach[k] + kW - 1) / kW * kW) : s1 - s0);
  const int nch = (ncol + kCw - 1) / kCw;
  auto issue = [&](int c) {  // lane 0: chunk c into its slot
    if (c < nch) {
      unsigned long long* bar = bars + c % kRing;
      mbar_expect_tx(bar, kChunkBytes);
      bulk_g2s(ring + (c % kRing) * kChunkBytes, a.coef + (size_t)(s0 + (long long)c * kCw) * kW, kChunkBytes, bar);
    }
  };
  if (lane == 0) {
    for (int q = 0; q < kRing; ++q) mbar_init(bars + q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int c = 0; c < kRing; ++c) issue(c);
  }
  __syncwarp();
  auto wait_chunk_ready = [&](int c) {
    if (c < nch)
      while (!mbar_try_wait(bars + c % kRing, (unsigned)(c / kRing) & 1u)) {
      }
  };
  double acc[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const long long i = s0 + 2 * lane + s;
    acc[s] = i < s1 ? __dmul_rn(a.b[i], a.rdg[i]) : 0.0;
    if (COUPLED && k > 0 && i < s1) {
      // coupling terms in ascending column order, 16 loads in flight per batch
      // (one memory round trip per batch instead of one per column)
      const double* tp = a.tt + (size_t)(k - 1) * kW;
#pragma unroll
      for (int q0 = 0; q0 < kW; q0 += 16) {
        double cw[16], tv[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const long long j = s0 - kW + q0 + q, d = i - j;
          cw[q] = (d >= 1 && d <= kW) ? __ldg(a.coef + (size_t)j * kW + d - 1) : 0.0;
          tv[q] = __ldg(tp + q0 + q);
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          const long long d = i - (s0 - kW + q0 + q);
          if (d >= 1 && d <= kW) acc[s] = __fma_rn(cw[q], tv[q], acc[s]);
        }
      }
    }
  }
  // column rel (relative to s0): the lane's two entries from the ring
  auto sload = [&](int rel, double (&dst)[2]) {
    const double* col = reinterpret_cast<const double*>(ring + ((rel / kCw) % kRing) * kChunkBytes) + (rel % kCw) * kW;
    const int p = rel & (kW - 1);
#pragma unroll
    for (int s = 0; s < 2; ++s) dst[s] = col[(2 * lane + s - p - 1) & (kW - 1)];
  };
  double nb[2];
  double xs0 = 0.0, xs1 = 0.0;  // this lane's two columns of the current window
  double cf[4][2];  // column j at cf[j % 4] (4 divides the 64-column window), two columns ahead
  wait_chunk_ready(0);
  sload(0, cf[0]);
  if (ncol > 1) sload(1, cf[1]);
  for (int c0 = 0; c0 < ncol; c0 += kW) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const long long i = s0 + c0 + kW + 2 * lane + s;
      nb[s] = i < s1 ? __dmul_rn(__ldg(a.b + i), __ldg(a.rdg + i)) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kW; ++u) {
      const int rel = c0 + u;
      const int owner = u >> 1, os = u & 1;
      if (u % kCw == 0 && rel > 0) {
        // every read of the previous chunk has completed: refill its slot
        __syncwarp();
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(rel / kCw - 1 + kRing);
        }
      }
      if (u % kCw == kCw - 2) wait_chunk_ready(rel / kCw + 1);
      if (rel + 2 < ncol) sload(rel + 2, cf[(u + 2) % 4]);
      const double w0 = cf[u % 4][0], w1 = cf[u % 4][1];
      const double xj = __shfl_sync(0xffffffffu, os ? acc[1] : acc[0], owner);
      if (lane == owner) {  // x of the window's columns 2 lane, 2 lane + 1: stored once per window
        if (os) xs1 = xj;
        else xs0 = xj;
      }
      double v0 = acc[0], v1 = acc[1];
      if (lane == owner) {
        if (os) v1 = nb[1];
        else v0 = nb[0];
      }
      acc[0] = __fma_rn(w0, xj, v0);
      acc[1] = __fma_rn(w1, xj, v1);
    }
    // the window's x: one 16-byte store per lane (K3: x; K1: c into x when the
    // coupling reach is in use, and c of the block's tail rows)
    const long long j0 = s0 + c0 + 2 * lane;
    double* dst = COUPLED ? a.out : a.x_all;
    if (dst) {
      if (j0 + 1 < s1 && ((reinterpret_cast<uintptr_t>(dst + j0) & 15) == 0)) {
        *reinterpret_cast<double2*>(dst + j0) = make_double2(xs0, xs1);
      } else {
        if (j0 < s1) dst[j0] = xs0;
        if (j0 + 1 < s1) dst[j0 + 1] = xs1;
      }
    }
    if (!COUPLED) {
      const long long t0 = s0 + a.S - kW;
      if (j0 < s1 && j0 >= t0) a.out[(size_t)k * kW + (j0 - t0)] = xs0;
      if (j0 + 1 < s1 && j0 + 1 >= t0) a.out[(size_t)k * kW + (j0 + 1 - t0)] = xs1;
    }
  }
}

// ---- K1 / K3 on the packed band, streamed by TMA -----------------------------
// Only the stored entries (~32 of the 64 band positions per column on
// banded-8M: 2.15 GB instead of 4.3 GB per sweep). A block's entries are one
// contiguous run of `pk` (columns in order, rows ascending inside a column),
// streamed through a ring of fixed 4 KB chunks that ignore column boundaries;
// the presence masks and offsets of the current and next 64-column window sit
// in shared memory (cp.async, a window ahead). A lane finds its entry of
// column j by popcount of the mask below its bit. A chunk is refilled once
// every entry in it lies below off[j] of the column being swept (read two
// columns ago and already consumed).
constexpr int kPkChunk = 256;  // doubles per chunk (2 KB)
constexpr int kPkRing = 4;     // chunks per warp ring: entry r (relative to the block's base) at ring[r & 1023]
constexpr int kPkRingMask = kPkRing * kPkChunk - 1;
constexpr int kPkGroup = 8;    // columns per wait / refill point
constexpr int kPkWarpBytes = kPkRing * kPkChunk * 8 + 2 * kW * 8 + 2 * kW * 4;
constexpr int kPkSmem = kBBWarps * kPkWarpBytes + kBBWarps * kPkRing * 8;
constexpr int kPkPad = 2 * kPkChunk;  // doubles allocated past the last entry (whole-chunk copies)

template <bool COUPLED>
__global__ void __launch_bounds__(32 * kBBWarps, 4) k_bb_sweep_pk(const __grid_constant__ SweepArgs a) {
  extern __shared__ __align__(128) unsigned char psm[];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int k = a.k_begin + blockIdx.x * kBBWarps + wq;
  double* ring = reinterpret_cast<double*>(psm + wq * kPkWarpBytes);
  unsigned long long* smask = reinterpret_cast<unsigned long long*>(ring + kPkRing * kPkChunk);  // [2][64]
  int* soff = reinterpret_cast<int*>(smask + 2 * kW);                                          // [2][64]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(psm + kBBWarps * kPkWarpBytes) + wq * kPkRing;
  if (k >= a.k_end) return;
  const long long s0 = (long long)k * a.S, s1 = std::min<long long>(s0 + a.S, a.n);
  const int ncol = (int)(COUPLED && a.reach ? std::min<long long>(s1 - s0, (a.reach[k] + kW - 1) / kW * kW) : s1 - s0);
  const int e1 = a.off[s0 + ncol];
  const int base = a.off[s0] & ~1;  // 16-byte aligned start of the block's entries
  const int nq = (e1 - base + kPkChunk - 1) / kPkChunk;
  auto issue = [&](int q) {  // lane 0
    if (q < nq) {
      unsigned long long* bar = bars + (q & (kPkRing - 1));
      mbar_expect_tx(bar, kPkChunk * 8);
      bulk_g2s(ring + (q & (kPkRing - 1)) * kPkChunk, a.pk + base + (long long)q * kPkChunk, kPkChunk * 8, bar);
    }
  };
  // window w's masks and offsets into slot w & 1; columns past the block read
  // as empty (mask 0, offset = the block's end)
  auto stage = [&](int w) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = w * kW + h * 32 + lane, sl = (w & 1) * kW + h * 32 + lane;
      if (c < ncol) {
        cp_async8(&smask[sl], a.mask + s0 + c);
        cp_async4(&soff[sl], a.off + s0 + c);
      } else {
        smask[sl] = 0ull;
        soff[sl] = e1;
      }
    }
    cp_async_commit();
  };
  if (lane == 0) {
    for (int q = 0; q < kPkRing; ++q) mbar_init(bars + q, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int q = 0; q < kPkRing; ++q) issue(q);
  }
  stage(0);
  stage(1);
  cp_async_wait<0>();
  __syncwarp();
  int q_ready = -1, next_refill = kPkRing;
  auto slot_of = [](int rel) { return ((rel >> 6) & 1) * kW + (rel & (kW - 1)); };
  // make every chunk holding entries below off[rel_end] resident
  auto ensure = [&](int rel_end) {
    const int hi = soff[slot_of(rel_end)] - base;
    if (hi > 0) {
      const int qn = (hi - 1) / kPkChunk;
      while (q_ready < qn) {
        ++q_ready;
        while (!mbar_try_wait(bars + (q_ready & (kPkRing - 1)), (unsigned)(q_ready / kPkRing) & 1u)) {
        }
      }
    }
  };
  const int lb0 = 2 * lane - 1;  // bit of (row 2 lane + s, column at window position p) = (lb0 + s - p) & 63
  auto load_col = [&](int rel, int p, double (&dst)[2]) {
    const int sl = slot_of(rel);
    const unsigned long long m = smask[sl];
    const int o = soff[sl] - base;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int bit = (lb0 + s - p) & (kW - 1);
      const int idx = o + __popcll(m & ((1ull << bit) - 1ull));
      dst[s] = ((m >> bit) & 1ull) ? ring[idx & kPkRingMask] : 0.0;
    }
  };
  double acc[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const long long i = s0 + 2 * lane + s;
    acc[s] = i < s1 ? __dmul_rn(a.b[i], a.rdg[i]) : 0.0;
    if (COUPLED && k > 0 && i < s1) {
      const double* tp = a.tt + (size_t)(k - 1) * kW;
      for (int q = 0; q < kW; ++q) {
        const long long j = s0 - kW + q;
        const long long d = i - j;
        if (d >= 1 && d <= kW) acc[s] = __fma_rn(a.coef[(size_t)j * kW + d - 1], tp[q], acc[s]);
      }
    }
  }
  double nb[2];
  double cf[4][2];
  ensure(2);
  load_col(0, 0, cf[0]);
  load_col(1, 1, cf[1]);
  for (int c0 = 0; c0 < ncol; c0 += kW) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const long long i = s0 + c0 + kW + 2 * lane + s;
      nb[s] = i < s1 ? __dmul_rn(__ldg(a.b + i), __ldg(a.rdg + i)) : 0.0;
    }
    if (c0 > 0) {
      __syncwarp();
      stage(c0 / kW + 1);  // into the previous window's slot
    }
#pragma unroll
    for (int u = 0; u < kW; ++u) {
      const int rel = c0 + u;
      const long long j = s0 + rel;
      const int owner = u >> 1, os = u & 1;
      if (u % kPkGroup == 0) {
        if (u == kW - kPkGroup) {  // this group's lookahead reaches the next window
          cp_async_wait<0>();
          __syncwarp();
        }
        // refill the chunks wholly below off[rel] (read and consumed), then
        // wait for those the group's lookahead (columns rel + 2 .. rel + 9) reads
        const int qf = (soff[slot_of(rel)] - base) / kPkChunk;
        if (next_refill - kPkRing < qf) {
          __syncwarp();
          if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            for (int q = next_refill; q - kPkRing < qf; ++q) issue(q);
          }
          next_refill = qf + kPkRing;
        }
        ensure(rel + kPkGroup + 2);
      }
      load_col(rel + 2, (u + 2) & (kW - 1), cf[(u + 2) % 4]);
      const double w0 = cf[u % 4][0], w1 = cf[u % 4][1];
      const double xj = __shfl_sync(0xffffffffu, os ? acc[1] : acc[0], owner);
      if (lane == owner && j < s1) {
        if (COUPLED) {
          a.out[j] = xj;
        } else {
          if (a.x_all) a.x_all[j] = xj;
          if (j >= s0 + a.S - kW)
          a.out[(size_t)k * kW + (j - (s0 + a.S - kW))] = xj;
        }
      }
      double v0 = acc[0], v1 = acc[1];
      if (lane == owner) {
        if (os) v1 = nb[1];
        else v0 = nb[0];
      }
      acc[0] = __fma_rn(w0, xj, v0);
      acc[1] = __fma_rn(w1, xj, v1);
    }
  }
}

// ---- K2: the tail recurrence (one CTA) -------------------------------------
struct TailArgs {
  const double* nt;   // [nblk - 2] tails (blocks 1 .. nblk-2), K2 layout
  const double* ct;   // [nblk][64] c tails (K1)
  double* tt;         // [nblk][64] t
  int nblk;
  // PE partition: this PE's blocks [k_begin, k_end); t_{k_begin - 1} comes
  // from the previous PE's slot (value-is-flag words), t_{k_end - 1} goes to
  // this PE's slot for the next one (null: no such PE)
  int k_begin, k_end;
  const unsigned long long* prev_slot;
  unsigned long long* my_slot;
  DeviceStatus* status;
  int* abort_flag;
  unsigned long long timeout_ns;
};

struct TSmem {
  static constexpr int kN = 0;                                 // [slot] 32 KB tail of N
  static constexpr int kC = kN + kTSlots * kTailBytes;         // [slot] 512 B c tail
  static constexpr int kT = kC + kTSlots * kW * 8;             // [2][64] t double buffer
  static constexpr int kPart = kT + 2 * kW * 8;                // [64] partial sums
  static constexpr int kBars = kPart + kW * 8;                 // [slot] mbarriers
  static constexpr int kCtl = kBars + 8 * kTSlots;             // [0] steps done
  static constexpr int kTotal = kCtl + 64;
};

// threads 0..127: thread (r = tid % 64, h = tid / 64) sums the 32 terms of
// coupling columns [32h, 32h + 32) of tail row r; thread 128 (its own warp)
// streams N_k / c_k into the ring.
__global__ void __launch_bounds__(160, 1) k_bb_tail(const __grid_constant__ TailArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + TSmem::kBars);
  int* ctl = reinterpret_cast<int*>(smem + TSmem::kCtl);
  double* tb = reinterpret_cast<double*>(smem + TSmem::kT);
  double* part = reinterpret_cast<double*>(smem + TSmem::kPart);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int q = 0; q < kTSlots; ++q) mbar_init(&bars[q], 1);
    ctl[0] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const unsigned long long deadline = a.timeout_ns ? globaltimer_ns() + a.timeout_ns : 0;
  // the chain enters at block kb with t_{kb - 1}
  const int kb = a.k_begin == 0 ? 1 : a.k_begin;
  const int klast = min(a.k_end, a.nblk - 1) - 1;  // the last block whose tail is needed
  if (tid < kW) {
    double t0;
    if (a.k_begin == 0) {
      t0 = a.ct[tid];  // t_0 = c_0 tail
    } else {
      // the previous PE's last tail: one-sided loads of its slot until the
      // word is published (system scope: the slot may be a peer mapping)
      unsigned long long u = ld_relaxed_sys_u64(a.prev_slot + tid);
      int polls = 0;
      while (u == kNotReady) {
        if ((++polls & 1023) == 0 && ((deadline && globaltimer_ns() > deadline) || ld_relaxed_s32(a.abort_flag))) {
          atomicExch(&a.status->code, 5);
          atomicExch(a.abort_flag, 1);
          break;
        }
        u = ld_relaxed_sys_u64(a.prev_slot + tid);
      }
      t0 = __longlong_as_double((long long)u);
    }
    tb[((kb - 1) & 1) * kW + tid] = t0;
    a.tt[(size_t)(kb - 1) * kW + tid] = t0;
  }
  __syncthreads();
  if (tid >= 128) {
    if (tid != 128) return;
    // producer: step k (kb .. klast) uses slot (k - kb) % kTSlots
    for (int k = kb; k <= klast; ++k) {
      const int q = (k - kb) % kTSlots;
      if (k - kb >= kTSlots) {
        int polls = 0;
        while (ld_acquire_cta(ctl) < k - kb + 1 - kTSlots) {  // the slot's previous step is done
          if ((++polls & 1023) == 0 && ((deadline && globaltimer_ns() > deadline) || ld_relaxed_s32(a.abort_flag)))
            return;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bars[q], kTailBytes + kW * 8);
      bulk_g2s(smem + TSmem::kN + q * kTailBytes, a.nt + (size_t)(k - 1) * (kTailBytes / 8), kTailBytes, &bars[q]);
      bulk_g2s(smem + TSmem::kC + q * kW * 8, a.ct + (size_t)k * kW, kW * 8, &bars[q]);
    }
    return;
  }
  const int r = tid & (kW - 1), h = tid >> 6;
  unsigned phase = 0;
  // t_k for blocks kb .. klast (the last block's tail is not needed)
  for (int k = kb; k <= klast; ++k) {
    const int q = (k - kb) % kTSlots;
    int polls = 0;
    bool ok = true;
    while (!mbar_try_wait(&bars[q], (phase >> q) & 1u)) {
      if ((++polls & 1023) == 0 && deadline && globaltimer_ns() > deadline) {
        ok = false;
        break;
      }
    }
    if (!ok) {
      if (tid == 0) {
        atomicExch(&a.status->code, 5);
        atomicExch(a.abort_flag, 1);
      }
      break;  // (the producer stops at the deadline too)
    }
    phase ^= 1u << q;
    const double2* nq = reinterpret_cast<const double2*>(smem + TSmem::kN + q * kTailBytes) + h * 16 * kW + r;
    const double* tp = tb + ((k - 1) & 1) * kW + 32 * h;
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double2 w = nq[i * kW];
      s4[i & 3] = __fma_rn(w.x, tp[2 * i], s4[i & 3]);
      s4[i & 3] = __fma_rn(w.y, tp[2 * i + 1], s4[i & 3]);
    }
    const double sum = __dadd_rn(__dadd_rn(s4[0], s4[1]), __dadd_rn(s4[2], s4[3]));
    if (h == 1) part[r] = sum;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (h == 0) {
      const double* cq = reinterpret_cast<const double*>(smem + TSmem::kC + q * kW * 8);
      const double t = __dadd_rn(cq[r], __dadd_rn(sum, part[r]));
      tb[(k & 1) * kW + r] = t;
      a.tt[(size_t)k * kW + r] = t;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (tid == 0) st_release_cta(ctl, k - kb + 1);
  }
  // hand this PE's last tail to the next PE (value-is-flag words)
  if (a.my_slot && tid < kW && !ld_relaxed_s32(a.abort_flag)) {
    const int kl = a.k_end - 1;
    st_relaxed_sys_u64(a.my_slot + tid, (unsigned long long)__double_as_longlong(tb[(kl & 1) * kW + tid]));
  }
}

// ---- K2 by superblocks (one PE) --------------------------------------------
// The tail chain t_k = c_k + M_k t_{k-1} (M_k = N_k's tail) is an affine
// recurrence, so it can be cut into superblocks g of G consecutive steps:
//   d_g = g's steps run from t = 0                   (K2a, all g in parallel)
//   T_g = P_g T_{g-1} + d_g,  P_g = M_last ... M_first   (K2b, nsb steps)
//   t_k = g's steps run again from T_{g-1}            (K2c, all g in parallel)
// P_g depends on L only and is built once per plan (k_bb_prod), so a solve
// runs G + nsb + G sequential matvecs instead of nblk - 2 (2,046 for
// banded-8M: ~0.8 ms of latency -> ~0.05 ms).
__device__ __forceinline__ int k2_index(int r, int m) {  // K2 layout of element (r, m)
  return (((m >> 5) * 16 + ((m & 31) >> 1)) * kW + r) * 2 + (m & 1);
}

constexpr int kProdSmem = 2 * kW * kW * 8;
constexpr int kMinSuperSteps = 64;  // shorter chains run as one sequential chain

// setup: pp[g] = M_{s1-1} ... M_{s0} for superblock g's steps [s0, s1)
__global__ void __launch_bounds__(256) k_bb_prod(const double* __restrict__ nt, int nsteps, int G,
                                                 double* __restrict__ pp) {
  extern __shared__ __align__(16) double ps_raw[];
  double (*P)[kW] = reinterpret_cast<double (*)[kW]>(ps_raw);
  double (*M)[kW] = reinterpret_cast<double (*)[kW]>(ps_raw + kW * kW);
  const int g = blockIdx.x, tid = threadIdx.x;
  const int s0 = g * G, s1 = min(nsteps, s0 + G);
  for (int e = tid; e < kW * kW; e += 256) P[e >> 6][e & 63] = nt[(size_t)s0 * kW * kW + k2_index(e >> 6, e & 63)];
  const int r = tid >> 2, m0 = (tid & 3) * 16;
  for (int st = s0 + 1; st < s1; ++st) {
    for (int e = tid; e < kW * kW; e += 256) M[e >> 6][e & 63] = nt[(size_t)st * kW * kW + k2_index(e >> 6, e & 63)];
    __syncthreads();
    double acc[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) acc[u] = 0.0;
    for (int q = 0; q < kW; ++q) {
      const double mq = M[r][q];
#pragma unroll
      for (int u = 0; u < 16; ++u) acc[u] = __fma_rn(mq, P[q][m0 + u], acc[u]);
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) P[r][m0 + u] = acc[u];
  }
  __syncthreads();
  for (int e = tid; e < kW * kW; e += 256) pp[(size_t)g * kW * kW + k2_index(e >> 6, e & 63)] = P[e >> 6][e & 63];
}

struct TailChainArgs {
  const double* mat;    // step s: 64 x 64 at mat + s * 4096 (K2 layout)
  const double* cv;     // step s: cv + s * 64
  const double* init0;  // CTA 0's incoming t (null: zero)
  const double* init;   // CTA g > 0's incoming t: init + (g - 1) * 64 (null: zero)
  double* out_all;      // t after step s -> out_all + s * 64 (null: not kept)
  double* out_last;     // t after CTA g's last step -> out_last + g * 64 (null: not kept)
  int nsteps, G;        // CTA g runs steps [g G, min(nsteps, (g + 1) G))
  // the superblock chain of a PE (K2b, one CTA): its incoming t is the previous
  // PE's last tail, polled from that PE's slot (value-is-flag, system scope;
  // null: init0), kept at init_out; its final t goes to this PE's slot
  const unsigned long long* prev_slot;
  unsigned long long* my_slot;
  double* init_out;
  DeviceStatus* status;
  int* abort_flag;
  unsigned long long timeout_ns;
};

// One CTA per superblock, the same step as k_bb_tail: threads 0..127 sum,
// thread 128 streams the step's matrix and constant into the ring by TMA.
__global__ void __launch_bounds__(160, 1) k_bb_chain(const __grid_constant__ TailChainArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + TSmem::kBars);
  int* ctl = reinterpret_cast<int*>(smem + TSmem::kCtl);
  double* tb = reinterpret_cast<double*>(smem + TSmem::kT);
  double* part = reinterpret_cast<double*>(smem + TSmem::kPart);
  const int tid = threadIdx.x, g = blockIdx.x;
  const int s0 = g * a.G, s1 = min(a.nsteps, s0 + a.G);
  if (tid == 0) {
    for (int q = 0; q < kTSlots; ++q) mbar_init(&bars[q], 1);
    ctl[0] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const unsigned long long deadline = a.timeout_ns ? globaltimer_ns() + a.timeout_ns : 0;
  if (tid < kW) {
    const double* in = g == 0 ? a.init0 : (a.init ? a.init + (size_t)(g - 1) * kW : nullptr);
    double t0 = in ? in[tid] : 0.0;
    if (g == 0 && a.prev_slot) {
      unsigned long long u = ld_relaxed_sys_u64(a.prev_slot + tid);
      int polls = 0;
      while (u == kNotReady) {
        if ((++polls & 1023) == 0 && ((deadline && globaltimer_ns() > deadline) || ld_relaxed_s32(a.abort_flag))) {
          atomicExch(&a.status->code, 5);
          atomicExch(a.abort_flag, 1);
          break;
        }
        u = ld_relaxed_sys_u64(a.prev_slot + tid);
      }
      t0 = __longlong_as_double((long long)u);
    }
    if (g == 0 && a.init_out) a.init_out[tid] = t0;
    tb[kW + tid] = t0;  // step s reads buffer (s - s0 + 1) & 1
  }
  __syncthreads();
  if (tid >= 128) {
    if (tid != 128) return;
    for (int st = s0; st < s1; ++st) {
      const int q = (st - s0) % kTSlots;
      if (st - s0 >= kTSlots) {
        int polls = 0;
        while (ld_acquire_cta(ctl) < st - s0 + 1 - kTSlots) {
          if ((++polls & 1023) == 0 && ((deadline && globaltimer_ns() > deadline) || ld_relaxed_s32(a.abort_flag)))
            return;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bars[q], kTailBytes + kW * 8);
      bulk_g2s(smem + TSmem::kN + q * kTailBytes, a.mat + (size_t)st * (kTailBytes / 8), kTailBytes, &bars[q]);
      bulk_g2s(smem + TSmem::kC + q * kW * 8, a.cv + (size_t)st * kW, kW * 8, &bars[q]);
    }
    return;
  }
  const int r = tid & (kW - 1), h = tid >> 6;
  unsigned phase = 0;
  for (int st = s0; st < s1; ++st) {
    const int q = (st - s0) % kTSlots, cur = (st - s0) & 1;
    int polls = 0;
    bool ok = true;
    while (!mbar_try_wait(&bars[q], (phase >> q) & 1u)) {
      if ((++polls & 1023) == 0 && deadline && globaltimer_ns() > deadline) {
        ok = false;
        break;
      }
    }
    if (!ok) {
      if (tid == 0) {
        atomicExch(&a.status->code, 5);
        atomicExch(a.abort_flag, 1);
      }
      break;
    }
    phase ^= 1u << q;
    const double2* nq = reinterpret_cast<const double2*>(smem + TSmem::kN + q * kTailBytes) + h * 16 * kW + r;
    const double* tp = tb + (cur ^ 1) * kW + 32 * h;
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double2 w = nq[i * kW];
      s4[i & 3] = __fma_rn(w.x, tp[2 * i], s4[i & 3]);
      s4[i & 3] = __fma_rn(w.y, tp[2 * i + 1], s4[i & 3]);
    }
    const double sum = __dadd_rn(__dadd_rn(s4[0], s4[1]), __dadd_rn(s4[2], s4[3]));
    if (h == 1) part[r] = sum;
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (h == 0) {
      const double* cq = reinterpret_cast<const double*>(smem + TSmem::kC + q * kW * 8);
      const double t = __dadd_rn(cq[r], __dadd_rn(sum, part[r]));
      tb[cur * kW + r] = t;
      if (a.out_all) a.out_all[(size_t)st * kW + r] = t;
      if (a.out_last && st == s1 - 1) a.out_last[(size_t)g * kW + r] = t;
      if (a.my_slot && st == s1 - 1 && !ld_relaxed_s32(a.abort_flag))
        st_relaxed_sys_u64(a.my_slot + r, (unsigned long long)__double_as_longlong(t));
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (tid == 0) st_release_cta(ctl, st - s0 + 1);
  }
}

}  // namespace

// Superblocks over chain steps [s_first, s_first + nsteps) (step s computes
// t_{s+1}): G ~ sqrt(nsteps) steps each, their coupling-tail products pp.
// SPTRSV_BB_SUPER=0 keeps the single sequential chain (k_bb_tail).
int DevicePlan::build_superblocks(int s_first, int nsteps, cudaStream_t st) {
  static const bool super_on = [] {
    const char* v = std::getenv("SPTRSV_BB_SUPER");
    return !v || std::atoi(v) != 0;
  }();
  cudaError_t e;
  for (double** p : {&bblk.pp, &bblk.dd, &bblk.TT})
    if (*p) cudaFree(*p), *p = nullptr;
  bblk.G = bblk.nsb = 0;
  bblk.sb_first = s_first;
  bblk.sb_steps = nsteps;
  if (!super_on || nsteps < kMinSuperSteps) return SPTRSV_OK;
  int G = 1;
  while ((long long)G * G < nsteps) ++G;
  const int nsb = (nsteps + G - 1) / G;
  auto al = [](void** p, size_t b) { return cudaMalloc(p, b < 16 ? 16 : b); };
  if ((e = al((void**)&bblk.pp, (size_t)nsb * kTailBytes)) != cudaSuccess ||
      (e = al((void**)&bblk.dd, sizeof(double) * nsb * kW)) != cudaSuccess ||
      (e = al((void**)&bblk.TT, sizeof(double) * nsb * kW)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  static std::atomic<unsigned long long> pattr{0};
  if ((e = set_max_dyn_smem(k_bb_prod, kProdSmem, pattr)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  k_bb_prod<<<nsb, 256, kProdSmem, st>>>(bblk.nt + (size_t)s_first * (kTailBytes / 8), nsteps, G, bblk.pp);
  if ((e = cudaGetLastError()) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  bblk.G = G;
  bblk.nsb = nsb;
  return SPTRSV_OK;
}

int DevicePlan::build_band_blocks() {
  cudaError_t e;
  // rows per block: enough blocks to fill the GPU's warps, at most 4096
  long long S = kW;
  while (S < 4096 && (n + S - 1) / S > (long long)num_sms * 8) S *= 2;
  const int nblk = (int)((n + S - 1) / S);
  bblk.S = (int)S;
  bblk.nblk = nblk;
  auto al = [](void** p, size_t b) { return cudaMalloc(p, b < 16 ? 16 : b); };
  if ((e = al((void**)&bblk.nt, (size_t)std::max(nblk - 1, 1) * kTailBytes)) != cudaSuccess ||
      (e = al((void**)&bblk.ct, sizeof(double) * nblk * kW)) != cudaSuccess ||
      (e = al((void**)&bblk.tt, sizeof(double) * nblk * kW)) != cudaSuccess ||
      (e = cudaMemsetAsync(bblk.ct, 0, sizeof(double) * nblk * kW, stream)) != cudaSuccess ||
      (e = cudaMemsetAsync(bblk.nt, 0, (size_t)std::max(nblk - 1, 1) * kTailBytes, stream)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  // coupling reach per block (SPTRSV_BB_REACH=0: K3 sweeps every row): block 0
  // has no coupling (x = c), the last block is swept whole, the others are
  // raised by k_bb_ntail
  static const bool reach_on = [] {
    const char* v = std::getenv("SPTRSV_BB_REACH");
    return !v || std::atoi(v) != 0;
  }();
  if (reach_on) {
    std::vector<int> r0(nblk, 0);
    // (a whole last block gets its reach from k_bb_ntail too; a partial one is swept whole)
    r0[nblk - 1] = (n % S == 0 && nblk > 2) ? 0 : (int)S;
    if ((e = al((void**)&bblk.reach, sizeof(int) * nblk)) != cudaSuccess ||
        (e = cudaMemcpy(bblk.reach, r0.data(), sizeof(int) * nblk, cudaMemcpyHostToDevice)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  }
  if (nblk > 2) {
    static std::atomic<unsigned long long> attr{0};
    if ((e = set_max_dyn_smem(k_bb_ntail, kNtSmem, attr)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    // blocks 1 .. nblk - 2 (their tails feed the chain) and, when whole, the
    // last block (its reach only; its tail slot nt[nblk - 2] is never read)
    const int nt_blocks = (n % S == 0) ? nblk - 1 : nblk - 2;
    k_bb_ntail<<<nt_blocks, 64, kNtSmem, stream>>>(band.coef, n, (int)S, nblk, bblk.nt, bblk.reach);
    if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaStreamSynchronize(stream)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  }
  // the tail chain by superblocks (one PE: every step; a PE of a partition
  // rebuilds them over its own steps, see solve_band_blocks)
  if (nblk - 2 >= kMinSuperSteps) {
    const int rc = build_superblocks(0, nblk - 2, stream);
    if (rc != SPTRSV_OK) return rc;
    if ((e = cudaStreamSynchronize(stream)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  }
  // the packed band for the TMA sweeps (SPTRSV_BB_PK=1; measured slower than
  // the dense band on banded-8M: 1.27 / 1.11 ms per sweep at 2.3 GB against
  // 0.78 / 0.70 ms at 4.4 GB -- per column ~78 instructions and two dependent
  // shared-memory loads per entry, so the sweep stops being HBM-bound)
  static const bool pk_on = [] {
    const char* v = std::getenv("SPTRSV_BB_PK");
    return v && std::atoi(v) != 0;
  }();
  bblk.pk_tma = pk_on && !kBBPacked && noff + kPkPad < (1ll << 31);
  if (kBBPacked || bblk.pk_tma) {
    // off = exclusive scan of the per-column entry counts; pk in row order
    int* cnt = nullptr;
    if ((e = al((void**)&cnt, sizeof(int) * (n + 1))) != cudaSuccess ||
        (e = al((void**)&bblk.off, sizeof(int) * (n + 1))) != cudaSuccess ||
        (e = al((void**)&bblk.pk, sizeof(double) * (std::max<long long>(noff, 1) + kPkPad))) != cudaSuccess ||
        (e = cudaMemsetAsync(cnt, 0, sizeof(int) * (n + 1), stream)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    const int g = (int)std::min<long long>((n + 255) / 256, 148 * 32);
    k_bb_popc<<<g, 256, 0, stream>>>(band.mask, n, cnt);
    if ((e = cudaGetLastError()) != cudaSuccess || (e = scan_exclusive(cnt, bblk.off, (int)n + 1, stream)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    k_bb_pack<<<g, 256, 0, stream>>>(band.coef, band.mask, bblk.off, n, bblk.pk);
    if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaStreamSynchronize(stream)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    cudaFree(cnt);
  }
  bblk.ready = true;
  return SPTRSV_OK;
}

// PE partition: contiguous slabs in PE order whose boundaries fall on row
// blocks (multiples of S). Returns 1 when installed, 0 when the owner map does
// not fit (the caller falls back), -1 on a CUDA error.
int DevicePlan::set_band_partition(const int32_t* owner, int pes, int my_pe) {
  const long long S = bblk.S;
  std::vector<long long> r0(pes, -1), r1(pes, -1);
  for (long long i = 0; i < n; ++i) {
    const int o = owner[i];
    if (i > 0 && o < owner[i - 1]) return 0;  // not in PE order
    if (r0[o] < 0) r0[o] = i;
    else if (r1[o] != i) return 0;  // not contiguous
    r1[o] = i + 1;
  }
  for (int p = 0; p < pes; ++p) {
    if (r0[p] < 0) return 0;                  // every PE owns a slab
    if (r0[p] % S || (r1[p] % S && r1[p] != n)) return 0;  // on block boundaries
  }
  bblk.release_part();
  cudaError_t e;
  if ((e = cudaMalloc((void**)&bblk.slot, 2 * kW * sizeof(unsigned long long))) != cudaSuccess ||
      (e = cudaMemset(bblk.slot, 0xFF, 2 * kW * sizeof(unsigned long long))) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e)), -1;
  bblk.k0 = (int)(r0[my_pe] / S);
  bblk.k1 = (int)((r1[my_pe] + S - 1) / S);
  bblk.my_pe = my_pe;
  bblk.n_pes = pes;
  bblk.part = true;
  return 1;
}

int DevicePlan::solve_band_blocks(const double* d_b, double* d_x, cudaStream_t s) {
  if (!bblk.ready) return plan_fail(SPTRSV_E_UNSUPPORTED, "band blocks were not built for this plan");
  if (bblk.part && bblk.my_pe > 0 && !bblk.prev_slot)
    return plan_fail(SPTRSV_E_INVALID_PE, "the previous PE's segment was never imported");
  cudaError_t e;
  if ((e = reset_control(s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  // partition: this solve publishes into / reads slot half `par` (reset by
  // the previous solve) and resets the other half for the next one
  // (consecutive solves are separated by a barrier across PEs)
  const int par = (int)(bblk.solves & 1);
  if (bblk.part) {
    ++bblk.solves;
    if ((e = cudaMemsetAsync(bblk.slot + (1 - par) * kW, 0xFF, kW * sizeof(unsigned long long), s)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  }
  const int kb = bblk.part ? bblk.k0 : 0, ke = bblk.part ? bblk.k1 : bblk.nblk;
  SweepArgs sa{};
  sa.coef = band.coef;
  sa.pk = bblk.pk;
  sa.off = bblk.off;
  sa.mask = band.mask;
  sa.b = d_b;
  sa.rdg = rdg;
  sa.n = n;
  sa.S = bblk.S;
  sa.nblk = bblk.nblk;
  sa.k_begin = kb;
  sa.k_end = ke;
  const int grid = (ke - kb + kBBWarps - 1) / kBBWarps;
  if ((e = record_k0(s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  static const bool tma_sweep = [] {
    const char* v = std::getenv("SPTRSV_BB_TMA");
    return !v || std::atoi(v) != 0;
  }() && !kBBPacked;
  const bool pk_sweep = bblk.pk_tma && bblk.pk && bblk.off;
  if (pk_sweep) {
    static std::atomic<unsigned long long> a1{0}, a3{0};
    if ((e = set_max_dyn_smem(k_bb_sweep_pk<false>, kPkSmem, a1)) != cudaSuccess ||
        (e = set_max_dyn_smem(k_bb_sweep_pk<true>, kPkSmem, a3)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  } else if (tma_sweep) {
    static std::atomic<unsigned long long> a1{0}, a3{0};
    if ((e = set_max_dyn_smem(k_bb_sweep_tma<false>, kRingSmem, a1)) != cudaSuccess ||
        (e = set_max_dyn_smem(k_bb_sweep_tma<true>, kRingSmem, a3)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  }
  auto sweep = [&](bool coupled) {
    if (pk_sweep) {
      if (coupled) k_bb_sweep_pk<true><<<grid, 32 * kBBWarps, kPkSmem, s>>>(sa);
      else k_bb_sweep_pk<false><<<grid, 32 * kBBWarps, kPkSmem, s>>>(sa);
    } else if (tma_sweep) {
      if (coupled) k_bb_sweep_tma<true><<<grid, 32 * kBBWarps, kRingSmem, s>>>(sa);
      else k_bb_sweep_tma<false><<<grid, 32 * kBBWarps, kRingSmem, s>>>(sa);
    } else {
      if (coupled) k_bb_sweep<true><<<grid, 32 * kBBWarps, 0, s>>>(sa);
      else k_bb_sweep<false><<<grid, 32 * kBBWarps, 0, s>>>(sa);
    }
    return cudaGetLastError();
  };
  // K1: c tails (and, with the coupling reach, c of every row into x)
  sa.out = bblk.ct;
  sa.x_all = bblk.reach ? d_x : nullptr;
  if ((e = sweep(false)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  // K2: tails
  TailArgs ta{};
  ta.nt = bblk.nt;
  ta.ct = bblk.ct;
  ta.tt = bblk.tt;
  ta.nblk = bblk.nblk;
  ta.k_begin = kb;
  ta.k_end = ke;
  ta.prev_slot = bblk.part && kb > 0 ? bblk.prev_slot + par * kW : nullptr;
  ta.my_slot = bblk.part && ke < bblk.nblk ? bblk.slot + par * kW : nullptr;
  ta.status = status;
  ta.abort_flag = abort_flag;
  ta.timeout_ns = (unsigned long long)(opt.timeout_s * 1e9);
  int k2_launches = 1;
  // this PE's chain steps: t_k for k = kb2 .. klast from t_{kb2 - 1}
  const int kb2 = kb == 0 ? 1 : kb, klast = std::min(ke, bblk.nblk - 1) - 1;
  const int my_steps = klast - kb2 + 1;
  if (my_steps >= kMinSuperSteps && (bblk.sb_first != kb2 - 1 || bblk.sb_steps != my_steps)) {
    const int rc = build_superblocks(kb2 - 1, my_steps, s);  // a partition changed this PE's steps
    if (rc != SPTRSV_OK) return rc;
  }
  if (my_steps >= kMinSuperSteps && bblk.G > 0) {
    // K2a / K2b / K2c: the chain by superblocks (see k_bb_chain)
    static std::atomic<unsigned long long> cattr{0};
    if ((e = set_max_dyn_smem(k_bb_chain, TSmem::kTotal, cattr)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    TailChainArgs ca{};
    ca.status = status;
    ca.abort_flag = abort_flag;
    ca.timeout_ns = ta.timeout_ns;
    ca.mat = bblk.nt + (size_t)(kb2 - 1) * (kTailBytes / 8);  // M_k at nt[k - 1]
    ca.cv = bblk.ct + (size_t)kb2 * kW;                         // c_k
    ca.out_last = bblk.dd;
    ca.nsteps = my_steps;
    ca.G = bblk.G;
    k_bb_chain<<<bblk.nsb, 160, TSmem::kTotal, s>>>(ca);  // d_g
    if ((e = cudaGetLastError()) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    TailChainArgs cb = ca;
    cb.mat = bblk.pp;
    cb.cv = bblk.dd;
    cb.init0 = kb == 0 ? bblk.ct : nullptr;  // t_0 = c_0, or the previous PE's last tail
    cb.prev_slot = ta.prev_slot;
    cb.my_slot = ta.my_slot;
    cb.init_out = bblk.tt + (size_t)(kb2 - 1) * kW;
    cb.out_last = nullptr;
    cb.out_all = bblk.TT;
    cb.nsteps = bblk.nsb;
    cb.G = bblk.nsb;
    k_bb_chain<<<1, 160, TSmem::kTotal, s>>>(cb);  // T_g
    if ((e = cudaGetLastError()) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    TailChainArgs cc = ca;
    cc.init0 = bblk.tt + (size_t)(kb2 - 1) * kW;
    cc.init = bblk.TT;
    cc.out_last = nullptr;
    cc.out_all = bblk.tt + (size_t)kb2 * kW;
    k_bb_chain<<<bblk.nsb, 160, TSmem::kTotal, s>>>(cc);  // every t_k
    if ((e = cudaGetLastError()) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    k2_launches = 3;
  } else {
    static std::atomic<unsigned long long> attr{0};
    if ((e = set_max_dyn_smem(k_bb_tail, TSmem::kTotal, attr)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    k_bb_tail<<<1, 160, TSmem::kTotal, s>>>(ta);
    if ((e = cudaGetLastError()) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  }
  // K3: x
  sa.tt = bblk.tt;
  sa.out = d_x;
  sa.x_all = nullptr;
  sa.reach = bblk.reach;
  if ((e = sweep(true)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if ((e = cudaEventRecord(evk1, s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  launches = 2 + k2_launches;
  return SPTRSV_OK;
}

}  // namespace sptrsv
