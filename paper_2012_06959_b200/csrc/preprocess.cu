// Preprocessing kernels: validation, in-degree (K1), CSC->CSR transpose, level
// ordering. All integer work, bit-exact against the reference analysis
// (/root/reference/pkg/src/sptrsv/analysis.py:19-64, matrix.py:133-164).
//
// Device layout produced here (int32 indices; n, nnz < 2^31 is checked):
//   rp[n+1]    off-diagonal CSR row pointers (exclusive scan of the in-degrees)
//   ci[noff]   columns, strictly ascending per row   (the serial oracle's
//              accumulation order, reference.py:30-34)
//   cv[noff]   L values             (exact mode)
//   wv[noff]   -L_ij / L_ii         (fast mode, rows pre-scaled by 1/diag)
//   dg[n], rdg[n]  diagonal and its correctly rounded reciprocal
#include <algorithm>
#include "common.cuh"
#include "kernels.cuh"
#include <cub/cub.cuh>

namespace sptrsv {

// Expand column ids per stored entry and narrow row indices to int32.
// Also checks structure (indices in range, rows strictly increasing per column)
// and records the first lower-triangular violation as key = col*4 + kind, kind:
// 0 MissingDiagonal, 1 UpperTriangularEntry, 2 ZeroDiagonal, which is the
// reference's (col, kind-name) order (matrix.py:150).
// One warp per 32 consecutive columns: short columns (<= kShortCol entries)
// one per lane, longer ones by the whole warp in lane order afterwards -- a
// power-law column (rmat-4M's largest hold ~10^5 entries) walked by a single
// thread left the whole launch waiting on that thread (2 s of plan setup).
constexpr int kShortCol = 64;
__global__ void k_expand_validate(const long long* __restrict__ cp, const long long* __restrict__ ri64,
                                  const double* __restrict__ val, int n, int* __restrict__ colE,
                                  int* __restrict__ ri32, unsigned long long* __restrict__ first_violation,
                                  int* __restrict__ structure_bad, int need_diag) {
  const int lane = threadIdx.x & 31;
  const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w * 32 < n; w += warps) {
    const long long j0 = w * 32;
    const int j = (int)(j0 + lane);
    long long lo = 0, hi = 0;
    if (j < n) lo = cp[j], hi = cp[j + 1];
    const bool is_long = j < n && hi - lo > kShortCol;
    auto verdict = [&](int col, bool has_diag, bool upper, bool zero) {
      unsigned long long key = ~0ull;
      if (need_diag && !has_diag) key = 4ull * col + 0;
      else if (upper) key = 4ull * col + 1;
      else if (need_diag && zero) key = 4ull * col + 2;
      if (key != ~0ull) atomicMin(first_violation, key);
    };
    if (j < n && !is_long) {
      bool has_diag = false, upper = false, zero = false;
      long long prev = -1;
      for (long long k = lo; k < hi; ++k) {
        long long r = ri64[k];
        if (r < 0 || r >= n || r <= prev) { atomicExch(structure_bad, 1); }
        prev = r;
        colE[k] = j;
        ri32[k] = (int)r;
        if (r < j) upper = true;
        if (r == j) {
          has_diag = true;
          if (val != nullptr && val[k] == 0.0) zero = true;
        }
      }
      verdict(j, has_diag, upper, zero);
    }
    unsigned longs = __ballot_sync(0xffffffffu, is_long);
    while (longs) {
      const int src = __ffs(longs) - 1;
      longs &= longs - 1;
      const int col = (int)(j0 + src);
      const long long clo = __shfl_sync(0xffffffffu, lo, src), chi = __shfl_sync(0xffffffffu, hi, src);
      bool has_diag = false, upper = false, zero = false, bad = false;
      for (long long k = clo + lane; k < chi; k += 32) {
        const long long r = ri64[k];
        const long long prev = k > clo ? ri64[k - 1] : -1;
        if (r < 0 || r >= n || r <= prev) bad = true;
        colE[k] = col;
        ri32[k] = (int)r;
        if (r < col) upper = true;
        if (r == col) {
          has_diag = true;
          if (val != nullptr && val[k] == 0.0) zero = true;
        }
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicExch(structure_bad, 1);
      has_diag = __any_sync(0xffffffffu, has_diag);
      upper = __any_sync(0xffffffffu, upper);
      zero = __any_sync(0xffffffffu, zero);
      if (lane == 0) verdict(col, has_diag, upper, zero);
    }
  }
}

// K1: dep(i) = stored off-diagonal entries in row i (analysis.py:19-27).
// Stored zeros count (test_analysis.py:52-54). Upper entries count too, exactly
// as np.bincount(row_idx[row != col]) does.
__global__ void k_in_degree(const int* __restrict__ ri32, const int* __restrict__ colE, long long nnz,
                            int* __restrict__ indeg) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz; k += (long long)gridDim.x * blockDim.x) {
    int r = ri32[k];
    if (r != colE[k]) atomicAdd(&indeg[r], 1);
  }
}

// Sort keys for the CSC->CSR transpose: an off-diagonal entry sorts by its row;
// the diagonal sorts after every row (key n) and is peeled into dg[] here.
// A stable LSD radix sort keeps storage order (ascending column) inside a row.
__global__ void k_transpose_keys(const int* __restrict__ ri32, const int* __restrict__ colE,
                                 const double* __restrict__ val, long long nnz, int n, int* __restrict__ key,
                                 int* __restrict__ entry, double* __restrict__ dg) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz; k += (long long)gridDim.x * blockDim.x) {
    int r = ri32[k];
    bool diag = r == colE[k];
    key[k] = diag ? n : r;
    entry[k] = (int)k;
    if (diag) dg[r] = val ? val[k] : 1.0;
  }
}

__global__ void k_gather_offdiag(const int* __restrict__ sorted_entry, const int* __restrict__ colE,
                                 const double* __restrict__ val, long long noff, int* __restrict__ ci,
                                 double* __restrict__ cv) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < noff; k += (long long)gridDim.x * blockDim.x) {
    int e = sorted_entry[k];
    ci[k] = colE[e];
    cv[k] = val ? val[e] : 1.0;
  }
}

__global__ void k_scale_rows(const int* __restrict__ rp, const double* __restrict__ cv, const double* __restrict__ dg,
                             int n, double* __restrict__ wv, double* __restrict__ rdg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double r = __ddiv_rn(1.0, dg[i]);
    rdg[i] = r;
    for (int k = rp[i]; k < rp[i + 1]; ++k) wv[k] = -__dmul_rn(cv[k], r);
  }
}

__global__ void k_iota(int* __restrict__ a, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

__global__ void k_widen(const int* __restrict__ a, long long* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) out[i] = a[i];
}

__global__ void k_level_hist(const int* __restrict__ level, int n, int* __restrict__ cnt) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) atomicAdd(&cnt[level[i]], 1);
}

// Tickets of the component pool never straddle a level: level l starts at
// ticket tb[l]; row at rank q of level l goes to slot 32*tb[l] + q.
__global__ void k_pad_order(const int* __restrict__ by_level, const int* __restrict__ level,
                            const int* __restrict__ level_ptr, const int* __restrict__ tb, int n,
                            int* __restrict__ padded) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    int row = by_level[p];
    int l = level[row];
    padded[32 * tb[l] + (p - level_ptr[l])] = row;
  }
}

__global__ void k_tickets_per_level(const int* __restrict__ cnt, int nl, int* __restrict__ t) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nl; l += gridDim.x * blockDim.x) t[l] = (cnt[l] + 31) / 32;
}

// ---------------------------------------------------------------------------
// host-side wrappers (called from capi.cu)

static inline int grid_for(long long work, int block) {
  long long g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

cudaError_t launch_expand_validate(const long long* cp, const long long* ri64, const double* val, int n, int* colE,
                                   int* ri32, unsigned long long* first_violation, int* structure_bad, int need_diag,
                                   cudaStream_t s) {
  k_expand_validate<<<grid_for((n + 31) / 32 * 32, 256), 256, 0, s>>>(cp, ri64, val, n, colE, ri32, first_violation,
                                                                        structure_bad, need_diag);
  return cudaGetLastError();
}

cudaError_t launch_in_degree(const int* ri32, const int* colE, long long nnz, int* indeg, cudaStream_t s) {
  k_in_degree<<<grid_for(nnz, 256), 256, 0, s>>>(ri32, colE, nnz, indeg);
  return cudaGetLastError();
}

cudaError_t scan_exclusive(const int* in, int* out, int count, cudaStream_t s) {
  size_t tmp = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, count, s);
  if (e != cudaSuccess) return e;
  void* d_tmp = nullptr;
  if ((e = cudaMallocAsync(&d_tmp, tmp, s)) != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(d_tmp, tmp, in, out, count, s);
  cudaFreeAsync(d_tmp, s);
  return e;
}

static int bits_for(int n) {
  int b = 1;
  while ((1ll << b) < (long long)n + 1) ++b;
  return b;
}

cudaError_t sort_pairs_stable(const int* keys_in, int* keys_out, const int* vals_in, int* vals_out, long long count,
                              int max_key, cudaStream_t s) {
  size_t tmp = 0;
  int eb = bits_for(max_key);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys_in, keys_out, vals_in, vals_out, count, 0, eb, s);
  if (e != cudaSuccess) return e;
  void* d_tmp = nullptr;
  if ((e = cudaMallocAsync(&d_tmp, tmp, s)) != cudaSuccess) return e;
  e = cub::DeviceRadixSort::SortPairs(d_tmp, tmp, keys_in, keys_out, vals_in, vals_out, count, 0, eb, s);
  cudaFreeAsync(d_tmp, s);
  return e;
}

cudaError_t launch_transpose_keys(const int* ri32, const int* colE, const double* val, long long nnz, int n, int* key,
                                  int* entry, double* dg, cudaStream_t s) {
  k_transpose_keys<<<grid_for(nnz, 256), 256, 0, s>>>(ri32, colE, val, nnz, n, key, entry, dg);
  return cudaGetLastError();
}

cudaError_t launch_gather_offdiag(const int* sorted_entry, const int* colE, const double* val, long long noff, int* ci,
                                  double* cv, cudaStream_t s) {
  k_gather_offdiag<<<grid_for(noff, 256), 256, 0, s>>>(sorted_entry, colE, val, noff, ci, cv);
  return cudaGetLastError();
}

cudaError_t launch_scale_rows(const int* rp, const double* cv, const double* dg, int n, double* wv, double* rdg,
                              cudaStream_t s) {
  k_scale_rows<<<grid_for(n, 256), 256, 0, s>>>(rp, cv, dg, n, wv, rdg);
  return cudaGetLastError();
}

cudaError_t launch_iota(int* a, int n, cudaStream_t s) {
  k_iota<<<grid_for(n, 256), 256, 0, s>>>(a, n);
  return cudaGetLastError();
}

cudaError_t launch_widen(const int* a, long long* out, long long n, cudaStream_t s) {
  k_widen<<<grid_for(n, 256), 256, 0, s>>>(a, out, n);
  return cudaGetLastError();
}

// Closed-form levels of a 2D (nz == 0) or 3D lower stencil in natural order.
__global__ void k_grid_levels(int* __restrict__ level, long long n, int nx, int ny, int nz) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long x = i % nx, y = (i / nx) % ny, z = nz ? i / ((long long)nx * ny) : 0;
    level[i] = (int)(x + y + z);
  }
}

cudaError_t launch_grid_levels(int* level, long long n, int nx, int ny, int nz, cudaStream_t s) {
  k_grid_levels<<<grid_for((int)std::min<long long>(n, 1 << 30), 256), 256, 0, s>>>(level, n, nx, ny, nz);
  return cudaGetLastError();
}

cudaError_t launch_level_hist(const int* level, int n, int* cnt, cudaStream_t s) {
  k_level_hist<<<grid_for(n, 256), 256, 0, s>>>(level, n, cnt);
  return cudaGetLastError();
}

cudaError_t launch_tickets_per_level(const int* cnt, int nl, int* t, cudaStream_t s) {
  k_tickets_per_level<<<grid_for(nl, 256), 256, 0, s>>>(cnt, nl, t);
  return cudaGetLastError();
}

cudaError_t launch_pad_order(const int* by_level, const int* level, const int* level_ptr, const int* tb, int n,
                             int* padded, cudaStream_t s) {
  k_pad_order<<<grid_for(n, 256), 256, 0, s>>>(by_level, level, level_ptr, tb, n, padded);
  return cudaGetLastError();
}

}  // namespace sptrsv
