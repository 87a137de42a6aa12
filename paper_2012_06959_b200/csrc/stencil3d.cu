// Register-blocked, warp-specialised wavefront executor for 3D seven-point
// lower structure (lap3d-128, BASELINE configs[1]).
//
// Structure: row i = (z*ny + y)*nx + x stores (i, i - nx*ny) iff z > 0,
// (i, i - nx) iff y > 0 and (i, i - 1) iff x > 0 (plus the diagonal), any
// coefficients — detected from the CSR at plan time. The DAG is the 3D
// wavefront: nx + ny + nz - 2 levels (382 for 128^3).
//
// Tiling: a task (one CTA) owns a tile of 32 grid rows in y (one per lane)
// by k3R = 4 planes in z, all nx columns. Lane l at lockstep step s solves,
// for its k3R rows (z0 + r, y0 + l), the k3C = 2 columns of block j = s - l:
//   * the y-neighbour of every row comes from lane l - 1's block of the
//     previous step (k3R * k3C values per step by __shfl_up_sync; lane 0
//     takes them from the tile above in y, polled from its y-mailbox);
//   * the z-neighbour of row r > 0 is the lane's own row r - 1 of this
//     block (registers); row 0's comes from the tile behind in z (its last
//     plane, polled from its z-mailbox);
//   * the x-neighbour is the lane's previous block.
// Tiles are dispatched in ascending (Z, Y) order, each depending only on the
// tiles at (Y-1, Z) and (Y, Z-1) — the reference's progress rule. A tile
// trails the one behind it in z by one chunk plus a mailbox round trip (not
// by the 32-step lane skew, which only separates tiles in y), so the
// critical path is ~3 y-hops + nz/k3R z-hops + nx/k3C steps.
//
// Warps: 0 compute (the only one on the critical path), 1 loader (TMA bulk
// copy of the pre-packed coefficient stream + cp.async of b), 2 storer (x
// from a shared-memory ring), 3 poller (both mailboxes into shared-memory
// inboxes). Hand-overs are monotone chunk counters at CTA scope, as in
// stencil.cu; mailboxes are value-is-flag with a signalling-NaN sentinel and
// double-buffered by solve parity.
//
// Arithmetic: fast: x = wy*y + (wz*z + (wx*left + b/d)) with pre-scaled
// coefficients; exact: s = 0 + lz*z, s += ly*y, s += lx*left, x = (b - s)/d —
// the serial oracle's ascending-column order with separate IEEE operations
// (absent boundary terms contribute +0 and leave every partial sum unchanged),
// Markstein division with a branch-free guard and an IEEE fallback.
#include <cmath>
#include <cstring>
#include <vector>
#include <chrono>
#include <cstring>
#include <algorithm>
#include "plan.hpp"
#include "kernels.cuh"
#include "ptx.cuh"

namespace sptrsv {

int plan_fail(int code, const char* msg);

namespace {

constexpr int k3R = 4, k3C = 2, k3G = 4, k3Lanes = 32;
constexpr int k3Blk = k3R * k3C;
constexpr int k3Pairs = k3Blk / 2;
constexpr int k3OutSlots = 3;
constexpr int k3Threads = 4 * 32;
constexpr unsigned k3NotReady32 = 0xFFF40000u;  // signalling NaN, as in stencil.cu
constexpr unsigned long long k3NotReady = 0xFFF40000FFF40000ull;
static_assert(k3R * k3C * k3G == 32, "the poller fetches the y-inbox of a chunk with one value per lane");

__host__ __device__ constexpr int s3_fields(bool exact) { return exact ? 5 : 4; }  // wz wy wx [d] rd
__host__ __device__ constexpr int s3_step_bytes(bool exact) { return s3_fields(exact) * k3Pairs * k3Lanes * 16; }
__host__ __device__ constexpr int s3_slots(bool exact) { return exact ? 3 : 4; }

struct S3Args {
  const unsigned char* stream;  // [task][step][field][pair][lane] f64x2
  unsigned long long* ymail;    // this solve's half: [task][k3R][nx] (lane 31's rows)
  unsigned long long* zmail;    // this solve's half: [task][32][nx] (plane z0 + k3R - 1)
  int* ticket;
  const double* b;
  double* x;
  DeviceStatus* status;
  int* abort_flag;
  unsigned long long timeout_ns;
  int spin_initial, spin_max_ns;
  int nx, ny, nz, nyt, nzt, n_tasks, steps;
  int b_aligned, x_aligned;  // 16-byte vector paths (else 8-byte halves)
  long long* dbg;            // diagnostics (probe_flags & 16): per-task globaltimer [start, ready, end]
  int probe;                 // diagnostics flags (probe_flags; 128: count exact-mode chunk redos)
  unsigned long long* ymail_next;  // the other mailbox halves: the storer resets each tile's part
  unsigned long long* zmail_next;  // for the next solve
  // streamed host solves (null otherwise): slab Z's b is resident once the
  // flag of the last slab of its copy reaches epoch; x flags per tile
  const unsigned* bflag;
  unsigned* xflag;
  unsigned epoch;
  int b_chunk_max;
  // z-groups (fast mode; null: one z-chain): virtual z-tile zv is real slab
  // zmap[zv] & 0xFFFFF, a halo tile when bit 20 is set (x discarded), the
  // first tile of its group (no z-tile behind: a zero plane) when bit 21 is
  const int* zmap;
  int nztv;  // virtual z-tiles (tasks = nytv * nztv)
  // y-groups (fast mode): every y-tile row Y >= 1 is entered through a halo
  // copy of row Y - 1 solved from a zero row above (virtual y-slots: 0 = row
  // 0, 2Y - 1 = halo of row Y - 1, 2Y = row Y); nytv = 2 nyt - 1, else nyt
  int ygrp, nytv;
};

struct S3Tile {
  int Y, Z, rt;  // tile row, real z-slab, real tile index (coefficient stream, x flags)
  bool halo, zsrc, pubz, ysrc, puby;  // halo: x discarded; ysrc / puby: y hand-over from t - 1 / to t + 1
};
__device__ __forceinline__ S3Tile s3_tile(const S3Args& a, int t) {
  S3Tile q;
  const int yv = t % a.nytv;
  const int zv = t / a.nytv;
  if (a.ygrp) {
    q.Y = (yv + 1) >> 1;  // slot 2Y: row Y; slot 2Y - 1: the halo copy of row Y - 1
    if (yv & 1) q.Y = (yv - 1) >> 1;
    q.ysrc = yv > 0 && !(yv & 1);
    q.puby = yv & 1;
  } else {
    q.Y = yv;
    q.ysrc = yv > 0;
    q.puby = yv + 1 < a.nyt;
  }
  if (!a.zmap) {
    q.Z = zv;
    q.halo = false;
    q.zsrc = zv > 0;
    q.pubz = zv + 1 < a.nzt;
  } else {
    const int m = a.zmap[zv];
    q.Z = m & 0xFFFFF;
    q.halo = (m >> 20) & 1;
    q.zsrc = !((m >> 21) & 1);
    q.pubz = zv + 1 < a.nztv && !((a.zmap[zv + 1] >> 21) & 1);
  }
  if (a.ygrp && (yv & 1)) q.halo = true;
  q.rt = q.Z * a.nyt + q.Y;
  return q;
}

template <bool EXACT>
struct S3Smem {
  static constexpr int kSlots = s3_slots(EXACT);
  static constexpr int kStep = s3_step_bytes(EXACT);
  static constexpr int kCoefChunk = k3G * kStep;
  static constexpr int kBChunk = k3R * k3G * k3Lanes * 16;     // [r][k][lane] f64x2
  static constexpr int kZChunk = k3G * k3Lanes * 16;           // [k][lane] f64x2
  static constexpr int kYChunk = k3G * k3R * k3C * 8;          // [k][r][q] f64
  static constexpr int kOutChunk = k3G * k3Pairs * k3Lanes * 16;  // [k][pair][lane] f64x2
  static constexpr int kCoef = 0;
  static constexpr int kB = kCoef + kSlots * kCoefChunk;
  static constexpr int kZ = kB + kSlots * kBChunk;
  static constexpr int kY = kZ + kSlots * kZChunk;
  static constexpr int kOut = kY + kSlots * kYChunk;
  static constexpr int kBars = kOut + k3OutSlots * kOutChunk;
  static constexpr int kCtl = kBars + 8 * kSlots;
  static constexpr int kTotal = kCtl + 64;
};

enum { kC3Task = 0, kC3InReady = 1, kC3InDone = 2, kC3OutReady = 3, kC3OutDone = 4, kC3Abort = 5, kC3MbReady = 6 };

__device__ __forceinline__ bool s3_wait(const int* ctl, int which, int need, unsigned long long deadline, int nap) {
  int polls = 0;
  while (ld_acquire_cta(ctl + which) < need) {
    if (ld_acquire_cta(ctl + kC3Abort)) return false;
    if ((++polls & 1023) == 0 && deadline && globaltimer_ns() > deadline) return false;
    if (nap) __nanosleep(nap);
  }
  return true;
}

__device__ __forceinline__ void s3_abort(const S3Args& a, int* ctl, int lane) {
  if (lane == 0) {
    atomicExch(&a.status->code, 5);
    atomicExch(a.abort_flag, 1);
    st_release_cta(ctl + kC3Abort, 1);
  }
}

// ---- warp 1: coefficient stream (TMA bulk) and b (cp.async) ----------------
template <bool EXACT>
__device__ void s3_loader(const S3Args& a, unsigned char* smem, int* ctl, int t, int lane, unsigned& phase_bits,
                          unsigned long long deadline) {
  using S = S3Smem<EXACT>;
  constexpr int NB = S::kSlots;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + S::kBars);
  const int nchunks = a.steps / k3G, nblk = a.nx / k3C;
  const S3Tile tl = s3_tile(a, t);
  const int Y = tl.Y, Z = tl.Z;
  const int y = Y * k3Lanes + lane;
  const unsigned char* tstream = a.stream + (size_t)tl.rt * a.steps * S::kStep;
  auto issue = [&](int c) {
    const int slot = c % NB;
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bars[slot], S::kCoefChunk);
      bulk_g2s(smem + S::kCoef + slot * S::kCoefChunk, tstream + (size_t)c * S::kCoefChunk, S::kCoefChunk,
               &bars[slot]);
    }
    double2* dst = reinterpret_cast<double2*>(smem + S::kB + slot * S::kBChunk) + lane;
#pragma unroll
    for (int r = 0; r < k3R; ++r) {
      const int z = Z * k3R + r;
#pragma unroll
      for (int k = 0; k < k3G; ++k) {
        const int j = c * k3G + k - lane;
        double2* d = dst + (r * k3G + k) * k3Lanes;
        if (j >= 0 && j < nblk && y < a.ny && z < a.nz) {
          const double* src = a.b + ((size_t)z * a.ny + y) * a.nx + (size_t)j * k3C;
          if (a.b_aligned) {
            cp_async16(d, src);
          } else {
            cp_async8(&d->x, src);
            cp_async8(&d->y, src + 1);
          }
        } else {
          *d = make_double2(0.0, 0.0);  // padding computes exact zeros
        }
      }
    }
    cp_async_arrive_noinc(&bars[slot]);
  };
  int issued = 0;
  bool ok = true;
  if (a.bflag) {
    // this tile's slab arrives with the copy of slabs [s0, s0 + w) (doubling w)
    int flag_slab = Z;
    for (int s0 = 0, w = 1;; s0 += w, w = min(2 * w, a.b_chunk_max))
      if (Z < s0 + w) {
        flag_slab = min(a.nzt, s0 + w) - 1;
        break;
      }
    int polls = 0;
    while ((int)(ld_acquire_sys_u32(a.bflag + flag_slab) - a.epoch) < 0) {
      if ((++polls & 255) == 0 && deadline && globaltimer_ns() > deadline) ok = false;
      if (!__all_sync(0xffffffffu, ok)) {
        s3_abort(a, ctl, lane);
        return;
      }
      __nanosleep(256);
    }
  }
  for (int c = 0; c < nchunks; ++c) {
    const int done = ld_acquire_cta(ctl + kC3InDone);
    while (issued < nchunks && issued < done + NB) issue(issued++);
    while (ok && issued <= c) {
      ok = s3_wait(ctl, kC3InDone, issued - NB + 1, deadline, 64);
      if (ok) issue(issued++);
    }
    if (ok) {
      const int slot = c % NB;
      const unsigned ph = (phase_bits >> slot) & 1u;
      int polls = 0;
      while (!mbar_try_wait(&bars[slot], ph)) {
        if ((++polls & 1023) == 0 && deadline && globaltimer_ns() > deadline) {
          ok = false;
          break;
        }
      }
      if (ok) phase_bits ^= 1u << slot;
    }
    ok = __all_sync(0xffffffffu, ok);
    if (!ok) {
      s3_abort(a, ctl, lane);
      return;
    }
    if (lane == 0) st_release_cta(ctl + kC3InReady, c + 1);
  }
}

// ---- warp 3: both mailboxes into the chunk's inboxes -----------------------
template <bool EXACT>
__device__ void s3_poller(const S3Args& a, unsigned char* smem, int* ctl, int t, int lane,
                          unsigned long long deadline) {
  using S = S3Smem<EXACT>;
  constexpr int NB = S::kSlots;
  const int nchunks = a.steps / k3G, nblk = a.nx / k3C;
  const S3Tile tl = s3_tile(a, t);
  const int Y = tl.Y;
  // z-inbox: lane l's row-0 z-neighbours = plane z0 - 1, lane l, of the tile behind
  const unsigned long long* zsrc = tl.zsrc ? a.zmail + ((size_t)(t - a.nytv) * k3Lanes + lane) * a.nx : nullptr;
  // y-inbox: lane 0's y-neighbours = lane 31's rows of the tile above; value
  // (k, r, q) of the chunk is polled by lane k * R * C + r * C + q
  const int yk = lane / (k3R * k3C), yr = (lane / k3C) % k3R, yq = lane % k3C;
  const unsigned long long* ysrc = tl.ysrc ? a.ymail + ((size_t)(t - 1) * k3R + yr) * a.nx : nullptr;
  unsigned long long spins = 0;
  for (int c = 0; c < nchunks; ++c) {
    if (c >= NB && !s3_wait(ctl, kC3InDone, c - NB + 1, deadline, 64)) return s3_abort(a, ctl, lane);
    const int slot = c % NB;
    bool ok = true;
    // the chunk's words are polled all at once: every round re-issues the
    // loads of the words still not ready as independent requests, so a
    // round costs one L2 round trip however many words it covers
    unsigned long long zw[k3G][k3C], yw = 0;
    const int jy = c * k3G + yk;  // lane 0's block at step c*G + yk
    bool zneed[k3G][k3C], yneed = ysrc && jy < nblk;
#pragma unroll
    for (int k = 0; k < k3G; ++k) {
      const int j = c * k3G + k - lane;
#pragma unroll
      for (int q = 0; q < k3C; ++q) {
        zneed[k][q] = zsrc && j >= 0 && j < nblk;
        zw[k][q] = 0ull;
      }
    }
    int polls = 0, sleep_ns = 32;
    while (true) {
      bool pending = false;
#pragma unroll
      for (int k = 0; k < k3G; ++k) {
        const int j = c * k3G + k - lane;
#pragma unroll
        for (int q = 0; q < k3C; ++q)
          if (zneed[k][q]) zw[k][q] = ld_relaxed_u64(zsrc + (size_t)j * k3C + q);
      }
      if (yneed) yw = ld_relaxed_u64(ysrc + (size_t)jy * k3C + yq);
#pragma unroll
      for (int k = 0; k < k3G; ++k)
#pragma unroll
        for (int q = 0; q < k3C; ++q) {
          zneed[k][q] = zneed[k][q] && zw[k][q] == k3NotReady;
          pending |= zneed[k][q];
        }
      yneed = yneed && yw == k3NotReady;
      pending |= yneed;
      if (!pending) break;
      ++spins;
      if (++polls > a.spin_initial) {
        if ((polls & 63) == 0 &&
            (ld_relaxed_s32(a.abort_flag) || (deadline && globaltimer_ns() > deadline))) {
          ok = false;
          break;
        }
        __nanosleep(sleep_ns);
        if (sleep_ns < a.spin_max_ns) sleep_ns <<= 1;
      }
    }
    double2* zin = reinterpret_cast<double2*>(smem + S::kZ + slot * S::kZChunk);
#pragma unroll
    for (int k = 0; k < k3G; ++k) zin[k * k3Lanes + lane] = make_double2(as_f64(zw[k][0]), as_f64(zw[k][1]));
    double* yin = reinterpret_cast<double*>(smem + S::kY + slot * S::kYChunk);
    yin[(yk * k3R + yr) * k3C + yq] = as_f64(yw);
    if (!__all_sync(0xffffffffu, ok)) return s3_abort(a, ctl, lane);
    if (lane == 0) st_release_cta(ctl + kC3MbReady, c + 1);
    if (a.dbg && lane == 0 && c == 0 && t < 192) a.dbg[2 * t] = (long long)globaltimer_ns();  // diagnostics
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) spins += __shfl_xor_sync(0xffffffffu, spins, off);
  if (lane == 0 && spins) atomicAdd(&a.status->spins, spins);
}

// ---- warp 2: solved blocks to x ---------------------------------------------
template <bool EXACT>
__device__ void s3_storer(const S3Args& a, unsigned char* smem, int* ctl, int t, int lane,
                          unsigned long long deadline) {
  using S = S3Smem<EXACT>;
  const int nchunks = a.steps / k3G, nblk = a.nx / k3C;
  const S3Tile tl = s3_tile(a, t);
  const int Y = tl.Y, Z = tl.Z;
  const int y = Y * k3Lanes + lane;
  {  // reset this tile's mailboxes in the other half for the next solve
    const ulonglong2 nr = make_ulonglong2(k3NotReady, k3NotReady);
    ulonglong2* ym = reinterpret_cast<ulonglong2*>(a.ymail_next + (size_t)t * k3R * a.nx);
    ulonglong2* zm = reinterpret_cast<ulonglong2*>(a.zmail_next + (size_t)t * k3Lanes * a.nx);
    for (int w = lane; w < k3R * a.nx / 2; w += k3Lanes) ym[w] = nr;
    for (int w = lane; w < k3Lanes * a.nx / 2; w += k3Lanes) zm[w] = nr;
  }
  for (int c = 0; c < nchunks; ++c) {
    if (!s3_wait(ctl, kC3OutReady, c + 1, deadline, 64)) return s3_abort(a, ctl, lane);
    const double2* src = reinterpret_cast<const double2*>(smem + S::kOut + (c % k3OutSlots) * S::kOutChunk);
#pragma unroll
    for (int k = 0; k < k3G; ++k) {
      const int j = c * k3G + k - lane;
      if (tl.halo || j < 0 || j >= nblk || y >= a.ny) continue;  // a halo tile's x is discarded
#pragma unroll
      for (int r = 0; r < k3R; ++r) {
        const int z = Z * k3R + r;
        if (z >= a.nz) continue;
        double* row = a.x + ((size_t)z * a.ny + y) * a.nx + (size_t)j * k3C;
        const double2 v = src[(k * k3Pairs + r) * k3Lanes + lane];
        if (a.x_aligned) {
          *reinterpret_cast<double2*>(row) = v;
        } else {
          row[0] = v.x;
          row[1] = v.y;
        }
      }
    }
    __syncwarp();
    if (lane == 0) st_release_cta(ctl + kC3OutDone, c + 1);
  }
  // streamed host solve: tile t's x may be copied once its flag is up; flags
  // go up in tile order so a copy of whole slabs waits on its last tile only
  if (a.xflag && lane == 0 && !tl.halo) {
    __threadfence_system();
    int polls = 0;
    while (tl.rt > 0 && (int)(ld_acquire_sys_u32(a.xflag + tl.rt - 1) - a.epoch) < 0) {
      if (ld_relaxed_s32(a.abort_flag)) break;  // released after the kernel anyway
      if ((++polls & 255) == 0 && deadline && globaltimer_ns() > deadline) break;
      __nanosleep(64);
    }
    st_release_sys_u32(a.xflag + tl.rt, a.epoch);
  }
}

// ---- warp 0: the lockstep wavefront -----------------------------------------
template <bool EXACT>
struct S3Blk {
  double wz[k3Blk], wy[k3Blk], wx[k3Blk], dd[k3Blk], rd[k3Blk], bv[k3Blk];
  double zin[k3C], yin[k3R][k3C];
  __device__ __forceinline__ void load(const unsigned char* smem, int slot, int k, int lane) {
    using S = S3Smem<EXACT>;
    const double2* cs = reinterpret_cast<const double2*>(smem + S::kCoef + slot * S::kCoefChunk + k * S::kStep);
#pragma unroll
    for (int p = 0; p < k3Pairs; ++p) {
      const double2 fz = cs[(0 * k3Pairs + p) * k3Lanes + lane];
      const double2 fy = cs[(1 * k3Pairs + p) * k3Lanes + lane];
      const double2 fx = cs[(2 * k3Pairs + p) * k3Lanes + lane];
      wz[2 * p] = fz.x, wz[2 * p + 1] = fz.y;
      wy[2 * p] = fy.x, wy[2 * p + 1] = fy.y;
      wx[2 * p] = fx.x, wx[2 * p + 1] = fx.y;
      if (EXACT) {
        const double2 d = cs[(3 * k3Pairs + p) * k3Lanes + lane];
        const double2 r = cs[(4 * k3Pairs + p) * k3Lanes + lane];
        dd[2 * p] = d.x, dd[2 * p + 1] = d.y;
        rd[2 * p] = r.x, rd[2 * p + 1] = r.y;
      } else {
        const double2 r = cs[(3 * k3Pairs + p) * k3Lanes + lane];
        rd[2 * p] = r.x, rd[2 * p + 1] = r.y;
      }
    }
    const double2* bb = reinterpret_cast<const double2*>(smem + S::kB + slot * S::kBChunk) + lane;
#pragma unroll
    for (int r = 0; r < k3R; ++r) {
      const double2 v = bb[(r * k3G + k) * k3Lanes];
      bv[r * k3C] = v.x, bv[r * k3C + 1] = v.y;
    }
    const double2 zz = reinterpret_cast<const double2*>(smem + S::kZ + slot * S::kZChunk)[k * k3Lanes + lane];
    zin[0] = zz.x, zin[1] = zz.y;
    const double* yy = reinterpret_cast<const double*>(smem + S::kY + slot * S::kYChunk) + k * k3R * k3C;
#pragma unroll
    for (int r = 0; r < k3R; ++r)
#pragma unroll
      for (int q = 0; q < k3C; ++q) yin[r][q] = yy[r * k3C + q];
  }
};

// early shuffle (as in stencil.cu): the next step's y-neighbours are
// shuffled right after the block and the look-ahead loads issue at the top
// of the step
#ifndef SPTRSV_S3_EARLY_SHFL
#define SPTRSV_S3_EARLY_SHFL 1
#endif
constexpr bool k3EarlyShfl = SPTRSV_S3_EARLY_SHFL;
// Fast mode can publish both mailboxes per chunk from the staged outputs too
// (SPTRSV_S3_CHUNK_PUB=1), after the chunk's counters are released, instead
// of ~10 predicated stores per step: measured lap3d-128 fast 0.209 -> 0.216 ms
// (median of 10), so the per-step stores stay the default.
#ifndef SPTRSV_S3_CHUNK_PUB
#define SPTRSV_S3_CHUNK_PUB 0
#endif
constexpr bool k3ChunkPub = SPTRSV_S3_CHUNK_PUB;
#ifndef SPTRSV_S3_SPEC
#define SPTRSV_S3_SPEC 1
#endif

template <bool EXACT>
__device__ void s3_compute(const S3Args& a, unsigned char* smem, int* ctl, int t, int lane,
                           unsigned long long deadline) {
  using S = S3Smem<EXACT>;
  constexpr int NB = S::kSlots;
  const int nchunks = a.steps / k3G, nblk = a.nx / k3C;
  const S3Tile tl = s3_tile(a, t);
  const int Y = tl.Y;
  // publish: lane 31's rows for the tile below in y, every lane's last plane
  // for the tile in front in z
  unsigned long long* ypub = a.ymail + (size_t)t * k3R * a.nx;
  unsigned long long* zpub = a.zmail + ((size_t)t * k3Lanes + lane) * a.nx;
  const bool pub_y = lane == k3Lanes - 1 && tl.puby;
  const bool pub_z = tl.pubz;
  constexpr bool k3Spec = EXACT && SPTRSV_S3_SPEC && k3C == 2;
  double xleft[k3R], prev[k3R][k3C];
#pragma unroll
  for (int r = 0; r < k3R; ++r) {
    xleft[r] = 0.0;
#pragma unroll
    for (int q = 0; q < k3C; ++q) prev[r][q] = 0.0;
  }
  // one 4 x 2 block (exact: Markstein with its guard folded into the
  // returned flag, or IEEE division; fast: pre-scaled FMAs)
  auto block = [&](const S3Blk<EXACT>& blk, const double (&yn)[k3R][k3C], double (&xb)[k3R][k3C],
                   bool ieee) -> bool {
    bool bad = false;
#pragma unroll
    for (int r = 0; r < k3R; ++r) {
#pragma unroll
      for (int q = 0; q < k3C; ++q) {
        const int e = r * k3C + q;
        const double zn = r == 0 ? blk.zin[q] : xb[r - 1][q];
        const double left = q == 0 ? xleft[r] : xb[r][q - 1];
        if (EXACT) {
          double acc = __dadd_rn(0.0, __dmul_rn(blk.wz[e], zn));
          acc = __dadd_rn(acc, __dmul_rn(blk.wy[e], yn[r][q]));
          acc = __dadd_rn(acc, __dmul_rn(blk.wx[e], left));
          const double num = __dsub_rn(blk.bv[e], acc);
          if (ieee) {
            xb[r][q] = __ddiv_rn(num, blk.dd[e]);
          } else {
            const double qv = __dmul_rn(num, blk.rd[e]);
            const int ok = (int)markstein_ok(blk.dd[e]) &
                           (((int)(num == 0.0) & (int)(__double2hiint(num) == 0)) |
                            ((int)markstein_ok(qv) & (int)markstein_ok(num)));  // +0 only: see stencil.cu
            bad |= !ok;
            xb[r][q] = __fma_rn(__fma_rn(-qv, blk.dd[e], num), blk.rd[e], qv);
          }
        } else {
          const double inner = __fma_rn(blk.wz[e], zn, __fma_rn(blk.wx[e], left, __dmul_rn(blk.bv[e], blk.rd[e])));
          xb[r][q] = __fma_rn(blk.wy[e], yn[r][q], inner);
        }
      }
    }
    return bad;
  };
  // a solved block: carry its right column and (shuffled) rows, stage it
  auto retire = [&](int c, int k, const double (&xb)[k3R][k3C]) {
#pragma unroll
    for (int r = 0; r < k3R; ++r) {
      xleft[r] = xb[r][k3C - 1];
#pragma unroll
      for (int q = 0; q < k3C; ++q)
        prev[r][q] = k3EarlyShfl ? __shfl_up_sync(0xffffffffu, xb[r][q], 1) : xb[r][q];
    }
    double2* dst = reinterpret_cast<double2*>(smem + S::kOut + (c % k3OutSlots) * S::kOutChunk) + k * k3Pairs * k3Lanes +
                   lane;
#pragma unroll
    for (int r = 0; r < k3R; ++r) dst[r * k3Lanes] = make_double2(xb[r][0], xb[r][1]);
  };
  // Speculative exact mode (as in stencil.cu): guards accumulate per chunk; a
  // chunk with a failed guard is rolled back and recomputed with IEEE
  // division before its outputs and mailbox words leave the warp, so both
  // mailboxes are published per chunk from the staged outputs.
  bool spec_bad = false;
  double sv_xleft[k3R], sv_prev[k3R][k3C];
  auto save_chunk_state = [&]() {
#pragma unroll
    for (int r = 0; r < k3R; ++r) {
      sv_xleft[r] = xleft[r];
#pragma unroll
      for (int q = 0; q < k3C; ++q) sv_prev[r][q] = prev[r][q];
    }
  };
  auto redo_chunk = [&](int c) {
    if ((a.probe & 128) && lane == 0) atomicAdd(&a.status->remote_reads, 1ull);  // diagnostics: count redos
#pragma unroll
    for (int r = 0; r < k3R; ++r) {
      xleft[r] = sv_xleft[r];
#pragma unroll
      for (int q = 0; q < k3C; ++q) prev[r][q] = sv_prev[r][q];
    }
#pragma unroll 1
    for (int k = 0; k < k3G; ++k) {
      S3Blk<EXACT> blk;
      blk.load(smem, c % NB, k, lane);
      double yn[k3R][k3C], xb[k3R][k3C];
#pragma unroll
      for (int r = 0; r < k3R; ++r)
#pragma unroll
        for (int q = 0; q < k3C; ++q) {
          const double up = k3EarlyShfl ? prev[r][q] : __shfl_up_sync(0xffffffffu, prev[r][q], 1);
          yn[r][q] = lane == 0 ? blk.yin[r][q] : up;
        }
      block(blk, yn, xb, true);
      retire(c, k, xb);
    }
  };
  auto publish_chunk = [&](int c) {
    const double2* src = reinterpret_cast<const double2*>(smem + S::kOut + (c % k3OutSlots) * S::kOutChunk);
    // y: lane 31's rows, one (step, row) per lane
    if (tl.puby && lane < k3G * k3R) {
      const int k = lane / k3R, r = lane % k3R, jj = c * k3G + k - (k3Lanes - 1);
      if (jj >= 0 && jj < nblk) {
        const double2 v = src[(k * k3Pairs + r) * k3Lanes + k3Lanes - 1];
        unsigned long long* w = ypub + (size_t)r * a.nx + (size_t)jj * k3C;
        st_relaxed_u64_if(w, as_u64(v.x), true);
        st_relaxed_u64_if(w + 1, as_u64(v.y), true);
      }
    }
    // z: every lane's last plane
    if (pub_z) {
#pragma unroll
      for (int k = 0; k < k3G; ++k) {
        const int jj = c * k3G + k - lane;
        const double2 v = src[(k * k3Pairs + k3R - 1) * k3Lanes + lane];
        st_relaxed_u64_if(zpub + (size_t)jj * k3C, as_u64(v.x), jj >= 0 && jj < nblk);
        st_relaxed_u64_if(zpub + (size_t)jj * k3C + 1, as_u64(v.y), jj >= 0 && jj < nblk);
      }
    }
  };
  auto step = [&](int c, int k, const S3Blk<EXACT>& cur, S3Blk<EXACT>& nxt) -> bool {
    const int s = c * k3G + k;
    const int j = s - lane;
    const bool active = j >= 0 && j < nblk;
    if (k3EarlyShfl && k + 1 < k3G) nxt.load(smem, c % NB, k + 1, lane);
    double yn[k3R][k3C];
#pragma unroll
    for (int r = 0; r < k3R; ++r)
#pragma unroll
      for (int q = 0; q < k3C; ++q) {
        const double up = k3EarlyShfl ? prev[r][q] : __shfl_up_sync(0xffffffffu, prev[r][q], 1);
        yn[r][q] = lane == 0 ? cur.yin[r][q] : up;
      }
    double xb[k3R][k3C];
    if (k3Spec) {
      if (k == 0) save_chunk_state();
      spec_bad |= block(cur, yn, xb, false);
    } else if (block(cur, yn, xb, false) && EXACT) {
      block(cur, yn, xb, true);
    }
    retire(c, k, xb);
    if (!k3Spec && !k3ChunkPub) {
#pragma unroll
      for (int r = 0; r < k3R; ++r)
#pragma unroll
        for (int q = 0; q < k3C; ++q)
          st_relaxed_u64_if(ypub + (size_t)r * a.nx + (size_t)j * k3C + q, as_u64(xb[r][q]), pub_y && active);
#pragma unroll
      for (int q = 0; q < k3C; ++q)
        st_relaxed_u64_if(zpub + (size_t)j * k3C + q, as_u64(xb[k3R - 1][q]), pub_z && active);
    }
    if (a.dbg && lane == 0 && c == 0 && k == k3G - 1 && t < 192) a.dbg[2 * t + 1] = (long long)globaltimer_ns();
    if (k + 1 < k3G) {
      if (!k3EarlyShfl) nxt.load(smem, c % NB, k + 1, lane);
    } else {
      if (k3Spec) {
        // a guard failed somewhere in this chunk: recompute it with IEEE division
        if (__any_sync(0xffffffffu, spec_bad)) redo_chunk(c);
        spec_bad = false;
      }
      __syncwarp();
      if (lane == 0) {
        st_release_cta(ctl + kC3OutReady, c + 1);
        st_release_cta(ctl + kC3InDone, c + 1);
      }
      // the mailboxes after the release (its MEMBAR would wait for these
      // stores); the out slot stays intact until the storer's OutDone
      if (k3Spec || k3ChunkPub) publish_chunk(c);
      if (c + 1 < nchunks) {
        if (!s3_wait(ctl, kC3InReady, c + 2, deadline, 0)) return false;
        if (!s3_wait(ctl, kC3MbReady, c + 2, deadline, 0)) return false;
        if (c + 1 >= k3OutSlots && !s3_wait(ctl, kC3OutDone, c + 2 - k3OutSlots, deadline, 0)) return false;
        nxt.load(smem, (c + 1) % NB, 0, lane);
      }
    }
    return true;
  };
  long long* ts = (a.dbg && lane == 0 && t < 1024) ? a.dbg + 6 * 64 + 3 * t : nullptr;
  if (ts) ts[0] = (long long)globaltimer_ns();
  S3Blk<EXACT> A, B;
  if (!s3_wait(ctl, kC3InReady, 1, deadline, 0) || !s3_wait(ctl, kC3MbReady, 1, deadline, 0))
    return s3_abort(a, ctl, lane);
  if (ts) ts[1] = (long long)globaltimer_ns();
  A.load(smem, 0, 0, lane);
  for (int c = 0; c < nchunks; ++c) {
    static_assert(k3G % 2 == 0, "chunks hold an even number of steps");
#pragma unroll
    for (int k = 0; k < k3G; k += 2) {
      if (!step(c, k, A, B)) return s3_abort(a, ctl, lane);
      if (!step(c, k + 1, B, A)) return s3_abort(a, ctl, lane);
    }
  }
  if (ts) ts[2] = (long long)globaltimer_ns();
}

template <bool EXACT>
__global__ void __launch_bounds__(k3Threads, 1) k_stencil3d(const __grid_constant__ S3Args a) {
  using S = S3Smem<EXACT>;
  extern __shared__ __align__(128) unsigned char smem[];
  int* ctl = reinterpret_cast<int*>(smem + S::kCtl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + S::kBars);
    for (int k = 0; k < S::kSlots; ++k) mbar_init(&bars[k], 1 + k3Lanes);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  unsigned phase_bits = 0;
  const unsigned long long deadline = a.timeout_ns ? globaltimer_ns() + a.timeout_ns : 0;
  while (true) {
    if (threadIdx.x == 0) {
      ctl[kC3Task] = atomicAdd(a.ticket, 1);  // ascending (Z, Y): the progress rule
      ctl[kC3InReady] = ctl[kC3InDone] = ctl[kC3OutReady] = ctl[kC3OutDone] = ctl[kC3Abort] = 0;
      ctl[kC3MbReady] = 0;
    }
    __syncthreads();
    const int t = ctl[kC3Task];
    if (t >= a.n_tasks) break;
    if (warp == 0) s3_compute<EXACT>(a, smem, ctl, t, lane, deadline);
    else if (warp == 1) s3_loader<EXACT>(a, smem, ctl, t, lane, phase_bits, deadline);
    else if (warp == 2) s3_storer<EXACT>(a, smem, ctl, t, lane, deadline);
    else s3_poller<EXACT>(a, smem, ctl, t, lane, deadline);
    __syncthreads();
    if (ctl[kC3Abort]) break;
  }
}

template <bool EXACT>
cudaError_t launch_s3(const S3Args& a, int blocks, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  if (cudaError_t e = set_max_dyn_smem(k_stencil3d<EXACT>, S3Smem<EXACT>::kTotal, attr); e != cudaSuccess) return e;
  k_stencil3d<EXACT><<<blocks, k3Threads, S3Smem<EXACT>::kTotal, s>>>(a);
  return cudaGetLastError();
}

static cudaError_t s3_fill_not_ready(unsigned long long* p, long long words, cudaStream_t s) {
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
  if (words <= 0) return cudaSuccess;
  return fn((CUdeviceptr)p, k3NotReady32, (size_t)words * 2, (CUstream)s) == CUDA_SUCCESS ? cudaSuccess
                                                                                         : cudaErrorUnknown;
}

}  // namespace

// Pack the 3D coefficient stream [task][step][field][pair][lane]: fields
// wz wy wx [d] rd per element (row i's entries in ascending column order:
// z, y, x neighbours); padding elements zero, exact d = 1/d = 1.
__global__ void k_s3_pack(const int* __restrict__ rp, const double* __restrict__ val, const double* __restrict__ dg,
                          const double* __restrict__ rdg, int nx, int ny, int nz, int nyt, int n_tasks, int steps,
                          int exact, unsigned char* __restrict__ out) {
  const long long items = (long long)n_tasks * steps * k3Lanes;
  const int nblk = nx / k3C, NF = exact ? 5 : 4;
  const size_t step_doubles = (size_t)NF * k3Pairs * k3Lanes * 2;
  for (long long it = blockIdx.x * (long long)blockDim.x + threadIdx.x; it < items;
       it += (long long)gridDim.x * blockDim.x) {
    const int l = (int)(it % k3Lanes);
    const long long ts = it / k3Lanes;
    const int s = (int)(ts % steps), t = (int)(ts / steps);
    const int Y = t % nyt, Z = t / nyt, j = s - l;
    const long long y = (long long)Y * k3Lanes + l;
    double* sb = reinterpret_cast<double*>(out) + (size_t)ts * step_doubles;
#pragma unroll
    for (int r = 0; r < k3R; ++r) {
      const long long z = (long long)Z * k3R + r;
#pragma unroll
      for (int q = 0; q < k3C; ++q) {
        const int e_ = r * k3C + q, pair = e_ / 2, half = e_ % 2;
        double f[5] = {0.0, 0.0, 0.0, exact ? 1.0 : 0.0, exact ? 1.0 : 0.0};
        if (j >= 0 && j < nblk && y < ny && z < nz) {
          const long long x = (long long)j * k3C + q;
          const long long i = (z * ny + y) * nx + x;
          int kk = rp[i];
          const double fz = z > 0 ? val[kk++] : 0.0;
          const double fy = y > 0 ? val[kk++] : 0.0;
          const double fx = x > 0 ? val[kk] : 0.0;
          f[0] = fz, f[1] = fy, f[2] = fx;
          if (exact) f[3] = dg[i], f[4] = rdg[i];
          else f[3] = rdg[i];
        }
        for (int fld = 0; fld < NF; ++fld) sb[((fld * k3Pairs + pair) * k3Lanes + l) * 2 + half] = f[fld];
      }
    }
  }
}

// 3D seven-point lower structure on the host CSR: returns true and (nx, ny, nz).
bool detect_stencil3d(long long n, const std::vector<int>& rp, const std::vector<int>& ci, int* dims) {
  if (n < 8) return false;
  long long nx = 0, nxy = 0;
  for (long long i = 1; i < n && (!nx || !nxy); ++i)
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const long long d = i - ci[k];
      if (d > 1 && !nx) nx = d;
      else if (nx && d > nx && !nxy) nxy = d;
    }
  if (nx < 2 || nxy < 2 * nx || nxy % nx || n % nxy || nx % k3C || nx > (1 << 24)) return false;
  const long long ny = nxy / nx, nz = n / nxy;
  if (nz < 2 || ny < 2) return false;
  for (long long i = 0; i < n; ++i) {
    const long long x = i % nx, y = (i / nx) % ny, z = i / nxy;
    int k = rp[i];
    if (z > 0) {
      if (k >= rp[i + 1] || ci[k] != i - nxy) return false;
      ++k;
    }
    if (y > 0) {
      if (k >= rp[i + 1] || ci[k] != i - nx) return false;
      ++k;
    }
    if (x > 0) {
      if (k >= rp[i + 1] || ci[k] != i - 1) return false;
      ++k;
    }
    if (k != rp[i + 1]) return false;
  }
  dims[0] = (int)nx, dims[1] = (int)ny, dims[2] = (int)nz;
  return true;
}

// Error contraction per z-plane of the fast 3D recurrence x = bd + a x_left +
// u x_up + w x_back (pre-scaled, a / u / w the x / y / z neighbours): a
// solve started from a zero plane errs by e with
// |e| <= A |e_left| + U |e_up| + W max|e_{plane behind}| and zero x / y
// boundaries, so each plane's error is at most gamma = W / (1 - A - U) times
// the one behind (A, U, W: the largest |a|, |u|, |w|).
__global__ void k_s3_decay(const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ wv,
                           long long n, int nx, unsigned long long* __restrict__ amax) {
  unsigned long long m[3] = {0, 0, 0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(wv[k]));  // NaN sorts above
      const long long d = i - ci[k];
      const int f = d == 1 ? 0 : d == nx ? 1 : 2;
      m[f] = max(m[f], bits);
    }
  for (int f = 0; f < 3; ++f) atomicMax(amax + f, m[f]);
}

// z-groups of G real z-tiles (SPTRSV_S3_ZGROUP, default 12; 0: one chain;
// lap3d-128 fast: one chain 0.225 ms, G = 16: 0.191, G = 12: 0.182),
// each after the first entered through H halo z-tiles solved from a zero
// plane, H * k3R planes enough for gamma^(H k3R) <= 2^-64 (lap3d: gamma =
// 1/4, 32 planes = 8 tiles). Returns 0 (or 1 when grouped), < 0 on error.
int DevicePlan::s3_zgroups(Stencil3Plan& P) {
  static const int want = [] {
    const char* v = std::getenv("SPTRSV_S3_ZGROUP");
    return v ? std::atoi(v) : 12;
  }();
  if (want <= 0 || !wv || !rp || !ci) return 0;
  cudaError_t e;
  unsigned long long* d = nullptr;
  unsigned long long h[3] = {0, 0, 0};
  if ((e = cudaMalloc((void**)&d, sizeof(h))) != cudaSuccess || (e = cudaMemset(d, 0, sizeof(h))) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  k_s3_decay<<<num_sms * 4, 256, 0, stream>>>(rp, ci, wv, n, P.nx, d);
  if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaStreamSynchronize(stream)) != cudaSuccess ||
      (e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  cudaFree(d);
  double A, U, W;
  std::memcpy(&A, &h[0], 8);
  std::memcpy(&U, &h[1], 8);
  std::memcpy(&W, &h[2], 8);
  P.decay = (A + U < 1.0 && W == W) ? W / (1.0 - A - U) : 1e300;
  // y-groups (SPTRSV_S3_YGROUP=1): the same bound per grid row, gamma_y =
  // U / (1 - A - W); one 32-row halo tile suffices when gamma_y^32 <= 2^-64
  // (lap3d: 1/4). Off by default: lap3d-128 0.200 ms with them against 0.181
  // without (7 y-slots instead of 4: the extra tiles cost more than the two
  // y-hops they remove)
  static const int ywant = [] {
    const char* v = std::getenv("SPTRSV_S3_YGROUP");
    return v ? std::atoi(v) : 0;
  }();
  const double gy = (A + W < 1.0 && U == U) ? U / (1.0 - A - W) : 1e300;
  if (ywant > 0 && P.nyt > 1 && gy <= 0.25) {
    P.ygrp = 1;
    P.nytv = 2 * P.nyt - 1;
  }
  if (!(P.decay < 1.0) || P.decay <= 0.0) return 0;
  const int planes = (int)std::ceil(64.0 / -std::log2(P.decay));
  const int H = (planes + k3R - 1) / k3R;
  if (H >= want || P.nzt <= want + H) return 0;  // the halo would cost more than the chain it cuts
  std::vector<int> zm;
  for (int z0 = 0; z0 < P.nzt; z0 += want) {
    if (z0 > 0)
      for (int h2 = 0; h2 < H && z0 - H + h2 >= 0; ++h2)
        zm.push_back((z0 - H + h2) | (1 << 20) | (h2 == 0 || z0 - H + h2 == 0 ? (1 << 21) : 0));
    for (int z = z0; z < std::min(P.nzt, z0 + want); ++z) zm.push_back(z | (z == 0 ? (1 << 21) : 0));
  }
  if ((e = cudaMalloc((void**)&P.zmap, sizeof(int) * zm.size())) != cudaSuccess ||
      (e = cudaMemcpy(P.zmap, zm.data(), sizeof(int) * zm.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  P.nztv = (int)zm.size();
  P.zgroup = want;
  P.zhalo = H;
  return 1;
}

int DevicePlan::build_stencil3d(const std::vector<int>& h_rp, const std::vector<int>& h_ci) {
  auto t0 = std::chrono::steady_clock::now();
  stencil3.release();
  int dims[3];
  if (!detect_stencil3d(n, h_rp, h_ci, dims)) return SPTRSV_OK;
  const bool exact = opt.precision != SPTRSV_PRECISION_FAST;
  Stencil3Plan& P = stencil3;
  P.exact = exact;
  P.nx = dims[0], P.ny = dims[1], P.nz = dims[2];
  P.nyt = (P.ny + k3Lanes - 1) / k3Lanes;
  P.nzt = (P.nz + k3R - 1) / k3R;
  P.n_tasks = P.nyt * P.nzt;
  const int nblk = P.nx / k3C;
  P.steps = (nblk + k3Lanes - 1 + k3G - 1) / k3G * k3G;
  const int NF = s3_fields(exact);
  const size_t step_doubles = s3_step_bytes(exact) / 8;
  const size_t bytes = s3_step_bytes(exact) * (size_t)P.steps * P.n_tasks;
  cudaError_t e;
  (void)step_doubles;
  (void)NF;
  auto al = [](void** p, size_t b) { return cudaMalloc(p, b < 16 ? 16 : b); };
  // fast mode: z-groups when the per-plane error contraction allows a halo
  P.nztv = P.nzt;
  P.nytv = P.nyt;
  P.ygrp = 0;
  if (!exact) {
    const int rc = s3_zgroups(P);
    if (rc < 0) return rc;
  }
  P.n_vtasks = P.nytv * P.nztv;
  const long long yw = (long long)P.n_vtasks * k3R * P.nx, zw = (long long)P.n_vtasks * k3Lanes * P.nx;
  if ((e = al((void**)&P.stream, bytes)) != cudaSuccess ||
      (e = al((void**)&P.ymail, 2 * sizeof(unsigned long long) * yw)) != cudaSuccess ||
      (e = al((void**)&P.zmail, 2 * sizeof(unsigned long long) * zw)) != cudaSuccess ||
      (e = s3_fill_not_ready(P.ymail, 2 * yw, 0)) != cudaSuccess ||
      (e = s3_fill_not_ready(P.zmail, 2 * zw, 0)) != cudaSuccess ||
      (e = al((void**)&P.bflag, sizeof(unsigned) * P.nzt)) != cudaSuccess ||
      (e = al((void**)&P.xflag, sizeof(unsigned) * P.n_tasks)) != cudaSuccess ||
      (e = cudaMemset(P.bflag, 0, sizeof(unsigned) * P.nzt)) != cudaSuccess ||
      (e = cudaMemset(P.xflag, 0, sizeof(unsigned) * P.n_tasks)) != cudaSuccess ||
      (e = cudaDeviceSynchronize()) != cudaSuccess ||
      // loaded now, not lazily while a streamed solve spins (see stencil.cu)
      (e = stencil_release_flags(P.xflag, P.n_tasks, 0u, stream)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  {  // pack the coefficient stream on the device (one thread per tile-step-lane)
    const long long items = (long long)P.n_tasks * P.steps * k3Lanes;
    const int grid = (int)std::min<long long>((items + 255) / 256, 148 * 64);
    k_s3_pack<<<grid, 256, 0, stream>>>(rp, exact ? cv : wv, dg, rdg, P.nx, P.ny, P.nz, P.nyt, P.n_tasks, P.steps,
                                        exact ? 1 : 0, P.stream);
    if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaStreamSynchronize(stream)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  }
  P.stream_bytes = (long long)bytes;
  P.ready = true;
  P.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return SPTRSV_OK;
}

int DevicePlan::solve_stencil3d(const double* d_b, double* d_x, cudaStream_t s, bool flags) {
  Stencil3Plan& P = stencil3;
  if (!P.ready) return plan_fail(SPTRSV_E_UNSUPPORTED, "matrix is not 3D seven-point lower structured");
  const long long yw = (long long)P.n_vtasks * k3R * P.nx, zw = (long long)P.n_vtasks * k3Lanes * P.nx;
  const int par = (int)(P.solves & 1);
  cudaError_t e;
  // this solve uses mailbox half `par`; reset the other half for the next one
  if ((e = reset_control(s)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  S3Args a{};
  a.stream = P.stream;
  a.ymail = P.ymail + par * yw;
  a.zmail = P.zmail + par * zw;
  a.ymail_next = P.ymail + (1 - par) * yw;
  a.zmail_next = P.zmail + (1 - par) * zw;
  a.ticket = ticket;
  a.b = d_b;
  a.x = d_x;
  a.status = status;
  a.abort_flag = abort_flag;
  a.timeout_ns = (unsigned long long)(opt.timeout_s * 1e9);
  a.probe = opt.probe_flags;
  if (flags) {
    a.bflag = stencil3.bflag;
    a.xflag = stencil3.xflag;
    a.epoch = stencil3.epoch;
    a.b_chunk_max = stencil3.b_chunk_max;
  }
  a.spin_initial = opt.spin_initial;
  a.spin_max_ns = opt.spin_max_ns;
  a.nx = P.nx, a.ny = P.ny, a.nz = P.nz, a.nyt = P.nyt, a.nzt = P.nzt;
  a.n_tasks = P.n_vtasks;
  a.zmap = P.zmap;
  a.nztv = P.nztv;
  a.ygrp = P.ygrp;
  a.nytv = P.nytv;
  a.steps = P.steps;
  a.b_aligned = ((uintptr_t)d_b & 15) == 0;
  a.x_aligned = ((uintptr_t)d_x & 15) == 0;
  if (opt.probe_flags & 16) {
    if (!probe_buf && cudaMalloc((void**)&probe_buf, sizeof(long long) * kProbeWords) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, "probe buffer");
    cudaMemsetAsync(probe_buf, 0, sizeof(long long) * kProbeWords, s);
    a.dbg = probe_buf;
  }
  const int blocks = std::max(1, std::min(P.n_vtasks, num_sms));
  ++P.solves;
  if ((e = record_k0(s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  e = P.exact ? launch_s3<true>(a, blocks, s) : launch_s3<false>(a, blocks, s);
  if (e != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if ((e = cudaEventRecord(evk1, s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  launches = 1;
  return SPTRSV_OK;
}

}  // namespace sptrsv
