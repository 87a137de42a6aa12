// Sliding-window executor for narrow-band, nearly sequential L (banded-8M:
// bandwidth 64, ~32 dependencies per row, 4.74 M levels for 8.4 M rows —
// parallelism ~1.8, so every level-synchronous or dataflow scheme pays one
// memory round trip per level; 13 s with the component pool).
//
// One warp owns a window of the next 64 rows; row r's accumulator lives in
// lane (r mod 64) / 2, slot r mod 2. For column j (in order):
//   * the owner lane of row j finishes x_j (fast: the accumulator already
//     holds b_j/l_jj + sum of pre-scaled terms; exact: (b_j - acc)/l_jj);
//   * x_j is broadcast with one __shfl_sync;
//   * every lane adds column j's band entries to its two accumulators — the
//     push / column formulation of the reference's Alg. 1 (reference.py:27-35:
//     left_sum[rid] += v * x_i in ascending column order), so exact mode
//     accumulates in the serial oracle's order, with absent band entries
//     skipped by a presence mask, and is bit-identical to solve_serial;
//   * row j's slot is recycled for row j + 64.
// Critical path per row: one shuffle + one FMA (+ the division in exact
// mode); no global round trip. A loader warp streams the band in 64-column
// chunks (one TMA bulk copy of 32 KB coefficients, plus the mask and the row
// data with cp.async) into a shared-memory ring.
#include <algorithm>
#include <vector>
#include "plan.hpp"
#include "kernels.cuh"
#include "ptx.cuh"

namespace sptrsv {

int plan_fail(int code, const char* msg);

namespace {

constexpr int kBW = 64;        // window = maximum bandwidth
constexpr int kBK = 64;        // columns per chunk
constexpr int kBSlots = 5;     // ring depth (chunks)
constexpr int kBThreads = 64;  // compute warp + loader warp

struct BandArgs {
  const double* coef;              // [n_pad][kBW]: entry (j + d, j) at [j][d - 1]
  const unsigned long long* mask;  // [n_pad]: bit d - 1 set iff (j + d, j) is stored (exact mode)
  const double* b;
  const double* dg;
  const double* rdg;
  double* x;
  DeviceStatus* status;
  int* abort_flag;
  unsigned long long timeout_ns;
  long long n;
  int nchunks;
  int exact;
};

struct BSmem {
  static constexpr int kCoef = 0;                                 // [slot][kBK][kBW] f64
  static constexpr int kCoefChunk = kBK * kBW * 8;
  static constexpr int kMask = kCoef + kBSlots * kCoefChunk;      // [slot][kBK] u64
  static constexpr int kRow = kMask + kBSlots * kBK * 8;          // [slot][3][kBK] f64: b, d, rd
  static constexpr int kRowChunk = 3 * kBK * 8;
  static constexpr int kBars = kRow + kBSlots * kRowChunk;
  static constexpr int kCtl = kBars + 8 * kBSlots;
  static constexpr int kTotal = kCtl + 64;
};
enum { kBInReady = 0, kBInDone = 1, kBAbort = 2 };

__device__ __forceinline__ bool b_wait(const int* ctl, int which, int need, unsigned long long deadline, int nap) {
  int polls = 0;
  while (ld_acquire_cta(ctl + which) < need) {
    if (ld_acquire_cta(ctl + kBAbort)) return false;
    if ((++polls & 1023) == 0 && deadline && globaltimer_ns() > deadline) return false;
    if (nap) __nanosleep(nap);
  }
  return true;
}

__device__ void band_loader(const BandArgs& a, unsigned char* smem, int* ctl, int lane, unsigned long long deadline) {
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + BSmem::kBars);
  // fast mode initialises row r's accumulator when r enters the window (while
  // column r - 64 is processed): its row data travel one window early
  const long long shift = a.exact ? 0 : kBW;
  unsigned phase = 0;
  auto issue = [&](int c) {
    const int slot = c % kBSlots;
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(&bars[slot], BSmem::kCoefChunk);
      bulk_g2s(smem + BSmem::kCoef + slot * BSmem::kCoefChunk, a.coef + (size_t)c * kBK * kBW, BSmem::kCoefChunk,
               &bars[slot]);
    }
    unsigned long long* m = reinterpret_cast<unsigned long long*>(smem + BSmem::kMask) + slot * kBK;
    double* rowd = reinterpret_cast<double*>(smem + BSmem::kRow + slot * BSmem::kRowChunk);
    for (int k = lane; k < kBK; k += 32) {
      const long long col = (long long)c * kBK + k, r = col + shift;
      cp_async8(m + k, a.mask + col);
      if (r < a.n) {
        cp_async8(rowd + k, a.b + r);
        cp_async8(rowd + kBK + k, a.dg + r);
        cp_async8(rowd + 2 * kBK + k, a.rdg + r);
      } else {
        rowd[k] = rowd[kBK + k] = 0.0;
        rowd[2 * kBK + k] = 1.0;
      }
    }
    cp_async_arrive_noinc(&bars[slot]);
  };
  int issued = 0;
  bool ok = true;
  for (int c = 0; c < a.nchunks && ok; ++c) {
    while (issued < a.nchunks && issued < c + kBSlots) {
      if (issued >= kBSlots) ok = b_wait(ctl, kBInDone, issued - kBSlots + 1, deadline, 64);
      if (!ok) break;
      issue(issued++);
    }
    if (!ok) break;
    const int slot = c % kBSlots;
    int polls = 0;
    while (!mbar_try_wait(&bars[slot], (phase >> slot) & 1u)) {
      if ((++polls & 1023) == 0 && deadline && globaltimer_ns() > deadline) {
        ok = false;
        break;
      }
    }
    phase ^= 1u << slot;
    ok = __all_sync(0xffffffffu, ok);
    if (ok && lane == 0) st_release_cta(ctl + kBInReady, c + 1);
  }
  if (!ok && lane == 0) {
    atomicExch(&a.status->code, 5);
    atomicExch(a.abort_flag, 1);
    st_release_cta(ctl + kBAbort, 1);
  }
}

template <bool EXACT>
__device__ void band_compute(const BandArgs& a, unsigned char* smem, int* ctl, int lane,
                             unsigned long long deadline) {
  // window rows 0..63: accumulators start at b*rd (fast) or 0 (exact)
  double acc[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const long long r = 2 * lane + s;
    acc[s] = (!EXACT && r < a.n) ? __dmul_rn(a.b[r], a.rdg[r]) : 0.0;
  }
  for (int c = 0; c < a.nchunks; ++c) {
    if (!b_wait(ctl, kBInReady, c + 1, deadline, 0)) return;
    const int slot = c % kBSlots;
    const double* coef = reinterpret_cast<const double*>(smem + BSmem::kCoef + slot * BSmem::kCoefChunk);
    const unsigned long long* msk = reinterpret_cast<const unsigned long long*>(smem + BSmem::kMask) + slot * kBK;
    const double* rowd = reinterpret_cast<const double*>(smem + BSmem::kRow + slot * BSmem::kRowChunk);
#pragma unroll 8
    for (int k = 0; k < kBK; ++k) {
      const long long j = (long long)c * kBK + k;
      // chunks are window-aligned (kBK == kBW), so row j's window position is
      // k itself: owner lane and slot are compile-time after unrolling
      static_assert(kBK == kBW, "window position = column index within the chunk");
      const int p = k, owner = p >> 1, os = p & 1;
      const double mine = os ? acc[1] : acc[0];
      double xj;
      if (EXACT) {
        const double num = __dsub_rn(rowd[k], mine);
        xj = div_exact(num, rowd[kBK + k], rowd[2 * kBK + k]);
      } else {
        xj = mine;
      }
      xj = __shfl_sync(0xffffffffu, xj, owner);
      if (lane == owner && j < a.n) a.x[j] = xj;
      // column j's entries for this lane's rows: row 2*lane+s+64q is j + d
      const double* cj = coef + k * kBW;
      const unsigned long long mj = EXACT ? msk[k] : 0ull;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int d = ((2 * lane + s - p - 1) & (kBW - 1)) + 1;  // 1..64 (64: the slot row j leaves)
        const double w = cj[d - 1];
        double v = acc[s];
        if (lane == owner && s == os) {
          // row j leaves the window, row j + 64 enters
          v = EXACT ? 0.0 : __dmul_rn(rowd[k], rowd[2 * kBK + k]);
        }
        if (EXACT) {
          if ((mj >> (d - 1)) & 1ull) v = __dadd_rn(v, __dmul_rn(w, xj));
        } else {
          v = __fma_rn(w, xj, v);
        }
        acc[s] = v;
      }
    }
    __syncwarp();
    if (lane == 0) st_release_cta(ctl + kBInDone, c + 1);
    if (ld_acquire_cta(ctl + kBAbort)) return;
  }
}

// Level mode (K6 for narrow bands): the same window in (max, +1) integer
// arithmetic over the presence masks — level_j = max over stored entries
// (j, i) of level_i + 1 — one shuffle per row, bit-exact by construction.
__device__ void band_levels(const BandArgs& a, unsigned char* smem, int* ctl, int lane, unsigned long long deadline) {
  int acc[2] = {0, 0};
  int* level = reinterpret_cast<int*>(a.x);
  for (int c = 0; c < a.nchunks; ++c) {
    if (!b_wait(ctl, kBInReady, c + 1, deadline, 0)) return;
    const int slot = c % kBSlots;
    const unsigned long long* msk = reinterpret_cast<const unsigned long long*>(smem + BSmem::kMask) + slot * kBK;
#pragma unroll 8
    for (int k = 0; k < kBK; ++k) {
      const long long j = (long long)c * kBK + k;
      const int p = k, owner = p >> 1, os = p & 1;
      int lv = __shfl_sync(0xffffffffu, os ? acc[1] : acc[0], owner);
      if (lane == owner && j < a.n) level[j] = lv;
      const unsigned long long mj = msk[k];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int d = ((2 * lane + s - p - 1) & (kBW - 1)) + 1;
        int v = (lane == owner && s == os) ? 0 : acc[s];  // row j + 64 enters with level 0
        if ((mj >> (d - 1)) & 1ull) v = max(v, lv + 1);
        acc[s] = v;
      }
    }
    __syncwarp();
    if (lane == 0) st_release_cta(ctl + kBInDone, c + 1);
    if (ld_acquire_cta(ctl + kBAbort)) return;
  }
}

template <int MODE>  // 0 fast, 1 exact, 2 levels
__global__ void __launch_bounds__(kBThreads, 1) k_band(const __grid_constant__ BandArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  int* ctl = reinterpret_cast<int*>(smem + BSmem::kCtl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + BSmem::kBars);
    for (int k = 0; k < kBSlots; ++k) mbar_init(&bars[k], 1 + 32);
    ctl[kBInReady] = ctl[kBInDone] = ctl[kBAbort] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const unsigned long long deadline = a.timeout_ns ? globaltimer_ns() + a.timeout_ns : 0;
  if (warp == 0) {
    if (MODE == 2) band_levels(a, smem, ctl, lane, deadline);
    else band_compute<MODE == 1>(a, smem, ctl, lane, deadline);
  }
  else band_loader(a, smem, ctl, lane, deadline);
}

template <int MODE>
cudaError_t launch_band_v(const BandArgs& a, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  if (cudaError_t e = set_max_dyn_smem(k_band<MODE>, BSmem::kTotal, attr); e != cudaSuccess) return e;
  k_band<MODE><<<1, kBThreads, BSmem::kTotal, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_band(const BandArgs& a, int mode, cudaStream_t s) {
  return mode == 2 ? launch_band_v<2>(a, s) : mode == 1 ? launch_band_v<1>(a, s) : launch_band_v<0>(a, s);
}

__global__ void k_band_scatter(const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ val,
                               int n, double* __restrict__ coef, unsigned long long* __restrict__ mask) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int k = rp[i]; k < rp[i + 1]; ++k) {
      const int c = ci[k], d = i - c;  // 1..kBW (checked on the host)
      coef[(size_t)c * kBW + d - 1] = val[k];
      atomicOr(mask + c, 1ull << (d - 1));
    }
}

}  // namespace

// Every dependency within kBW rows.
bool DevicePlan::band_narrow(const std::vector<int>& h_rp, const std::vector<int>& h_ci) const {
  if (n < 2 * kBW) return false;
  for (long long i = 0; i < n; ++i)
    if (h_rp[i] < h_rp[i + 1] && i - h_ci[h_rp[i]] > kBW) return false;
  return true;
}

// Narrow band and low parallelism (the pool wins when levels are wide).
bool DevicePlan::band_candidate(const std::vector<int>& h_rp, const std::vector<int>& h_ci) const {
  return n_levels > n / 8 && band_narrow(h_rp, h_ci);
}

int DevicePlan::build_band() {
  band.release();
  const long long n_pad = (n + kBK - 1) / kBK * kBK + kBK;
  cudaError_t e;
  auto al = [](void** p, size_t b) { return cudaMalloc(p, b < 16 ? 16 : b); };
  const bool exact = opt.precision != SPTRSV_PRECISION_FAST;
  if ((e = al((void**)&band.coef, sizeof(double) * n_pad * kBW)) != cudaSuccess ||
      (e = al((void**)&band.mask, sizeof(unsigned long long) * n_pad)) != cudaSuccess ||
      (e = cudaMemsetAsync(band.coef, 0, sizeof(double) * n_pad * kBW, stream)) != cudaSuccess ||
      (e = cudaMemsetAsync(band.mask, 0, sizeof(unsigned long long) * n_pad, stream)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  const int grid = (int)std::min<long long>((n + 255) / 256, 148 * 32);
  k_band_scatter<<<grid, 256, 0, stream>>>(rp, ci, exact ? cv : wv, (int)n, band.coef, band.mask);
  if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaStreamSynchronize(stream)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  band.nchunks = (int)((n + kBK - 1) / kBK);
  band.ready = true;
  return SPTRSV_OK;
}

int DevicePlan::solve_band(const double* d_b, double* d_x, cudaStream_t s) {
  if (!band.ready) return plan_fail(SPTRSV_E_UNSUPPORTED, "band executor was not built for this plan");
  cudaError_t e;
  if ((e = reset_control(s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  BandArgs a{};
  a.coef = band.coef;
  a.mask = band.mask;
  a.b = d_b;
  a.dg = dg;
  a.rdg = rdg;
  a.x = d_x;
  a.status = status;
  a.abort_flag = abort_flag;
  a.timeout_ns = (unsigned long long)(opt.timeout_s * 1e9);
  a.n = n;
  a.nchunks = band.nchunks;
  a.exact = opt.precision != SPTRSV_PRECISION_FAST;
  const int mode = a.exact ? 1 : 0;
  if ((e = record_k0(s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if ((e = launch_band(a, mode, s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if ((e = cudaEventRecord(evk1, s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  launches = 1;
  return SPTRSV_OK;
}

// K6 for a narrow band: levels into `level` (int32[n]) with the window kernel.
int DevicePlan::band_levels(int* level_out) {
  if (!band.ready) return plan_fail(SPTRSV_E_UNSUPPORTED, "band structure not built");
  cudaError_t e;
  if ((e = reset_control(stream)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  BandArgs a{};
  a.coef = band.coef;
  a.mask = band.mask;
  a.b = dg;  // row data are streamed but unused in level mode
  a.dg = dg;
  a.rdg = rdg;
  a.x = reinterpret_cast<double*>(level_out);
  a.status = status;
  a.abort_flag = abort_flag;
  a.timeout_ns = (unsigned long long)(std::max(opt.timeout_s, 600.0) * 1e9);
  a.n = n;
  a.nchunks = band.nchunks;
  a.exact = 1;  // loader: unshifted row data
  if ((e = launch_band(a, 2, stream)) != cudaSuccess || (e = cudaStreamSynchronize(stream)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  DeviceStatus hs{};
  if ((e = cudaMemcpy(&hs, status, sizeof(hs), cudaMemcpyDeviceToHost)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if (hs.code == SPTRSV_E_TIMEOUT) return plan_fail(SPTRSV_E_TIMEOUT, "level analysis exceeded the timeout");
  return SPTRSV_OK;
}

}  // namespace sptrsv
