// Plan construction: upload the CSC arrays once, then validation, in-degree
// (K1), CSC->CSR transpose, row scaling, level analysis (K6) and — when the
// structure suits it — the lane-chain schedule. All of it is "setup" in the
// reference's vocabulary (engine.py:445-490 + analysis.py:43-64).
#include <string>
#include <algorithm>
#include "plan.hpp"
#include "kernels.cuh"

namespace sptrsv {

int plan_fail(int code, const char* msg);  // defined in capi.cu

#define P_TRY(expr)                                                    \
  do {                                                                 \
    cudaError_t _e = (expr);                                           \
    if (_e != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(_e)); \
  } while (0)

template <class T>
static cudaError_t dal(T** p, size_t count) {
  return cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
}

int DevicePlan::build(const int64_t* col_ptr, const int64_t* row_idx, const double* values, int64_t* bad_col) {
  P_TRY(cudaSetDevice(device));
  P_TRY(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device));
  P_TRY(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  P_TRY(cudaEventCreate(&ev0));
  P_TRY(cudaEventCreate(&ev1));
  P_TRY(cudaEventCreate(&evk0));
  P_TRY(cudaEventCreate(&evk1));
  const bool indeg_only = (opt.flags & 2) != 0;

  long long *d_cp = nullptr, *d_ri64 = nullptr;
  double* d_val = nullptr;
  int *colE = nullptr, *ri32 = nullptr, *sbad = nullptr;
  unsigned long long* fviol = nullptr;
  P_TRY(dal(&d_cp, n + 1));
  P_TRY(dal(&d_ri64, nnz));
  if (values) P_TRY(dal(&d_val, nnz));
  P_TRY(dal(&colE, nnz));
  P_TRY(dal(&ri32, nnz));
  P_TRY(dal(&sbad, 1));
  P_TRY(dal(&fviol, 1));
  P_TRY(cudaMemcpyAsync(d_cp, col_ptr, sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, stream));
  if (nnz) P_TRY(cudaMemcpyAsync(d_ri64, row_idx, sizeof(long long) * nnz, cudaMemcpyHostToDevice, stream));
  if (values && nnz) P_TRY(cudaMemcpyAsync(d_val, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, stream));
  P_TRY(cudaMemsetAsync(sbad, 0, sizeof(int), stream));
  P_TRY(cudaMemsetAsync(fviol, 0xFF, sizeof(unsigned long long), stream));
  P_TRY(launch_expand_validate(d_cp, d_ri64, d_val, (int)n, colE, ri32, fviol, sbad, structure_only ? 0 : 1, stream));
  int h_sbad = 0;
  unsigned long long h_fv = 0;
  P_TRY(cudaMemcpyAsync(&h_sbad, sbad, sizeof(int), cudaMemcpyDeviceToHost, stream));
  P_TRY(cudaMemcpyAsync(&h_fv, fviol, sizeof(h_fv), cudaMemcpyDeviceToHost, stream));
  P_TRY(cudaStreamSynchronize(stream));
  cudaFree(d_cp);
  cudaFree(d_ri64);
  cudaFree(sbad);
  cudaFree(fviol);
  auto cleanup = [&]() {
    cudaFree(d_val);
    cudaFree(colE);
    cudaFree(ri32);
  };
  if (h_sbad) {
    cleanup();
    return plan_fail(SPTRSV_E_STRUCTURE, "CSC structure invalid (row index out of range or rows not strictly increasing)");
  }

  // K1: in-degrees (every structurally valid matrix, like the reference)
  P_TRY(dal(&indeg, n + 1));
  P_TRY(cudaMemsetAsync(indeg, 0, sizeof(int) * (n + 1), stream));
  P_TRY(launch_in_degree(ri32, colE, nnz, indeg, stream));
  if (indeg_only) {
    P_TRY(cudaStreamSynchronize(stream));
    cleanup();
    return SPTRSV_OK;
  }
  if (h_fv != ~0ull) {
    long long col = (long long)(h_fv >> 2);
    int kind = (int)(h_fv & 3);
    if (bad_col) *bad_col = col;
    cleanup();
    if (kind == 0) return plan_fail(SPTRSV_E_MISSING_DIAGONAL, "missing diagonal");
    if (kind == 2) return plan_fail(SPTRSV_E_ZERO_DIAGONAL, "zero diagonal");
    return plan_fail(SPTRSV_E_STRUCTURE, "not lower triangular: UpperTriangularEntry");
  }

  // CSR transpose: row pointers = exclusive scan of in-degrees; entries by a
  // stable radix sort on row (ascending column kept inside each row).
  P_TRY(dal(&rp, n + 1));
  P_TRY(scan_exclusive(indeg, rp, (int)n + 1, stream));
  int h_noff = 0;
  P_TRY(cudaMemcpyAsync(&h_noff, rp + n, sizeof(int), cudaMemcpyDeviceToHost, stream));
  P_TRY(dal(&dg, n));
  int *key = nullptr, *entry = nullptr, *key_s = nullptr, *entry_s = nullptr;
  P_TRY(dal(&key, nnz));
  P_TRY(dal(&entry, nnz));
  P_TRY(dal(&key_s, nnz));
  P_TRY(dal(&entry_s, nnz));
  P_TRY(cudaMemsetAsync(dg, 0, sizeof(double) * n, stream));
  P_TRY(launch_transpose_keys(ri32, colE, d_val, nnz, (int)n, key, entry, dg, stream));
  P_TRY(sort_pairs_stable(key, key_s, entry, entry_s, nnz, (int)n, stream));
  P_TRY(cudaStreamSynchronize(stream));
  noff = h_noff;
  P_TRY(dal(&ci, noff));
  P_TRY(dal(&cv, noff));
  P_TRY(launch_gather_offdiag(entry_s, colE, d_val, noff, ci, cv, stream));
  P_TRY(cudaStreamSynchronize(stream));
  cudaFree(key);
  cudaFree(entry);
  cudaFree(key_s);
  cudaFree(entry_s);
  cleanup();

  P_TRY(dal(&wv, noff));
  P_TRY(dal(&rdg, n));
  if (!structure_only) P_TRY(launch_scale_rows(rp, cv, dg, (int)n, wv, rdg, stream));

  // solve scratch
  P_TRY(dal(&xbuf, n));
  P_TRY(dal(&bbuf, n));
  // per-solve control words in one block: one memset resets them all
  P_TRY(dal(&ctlblk, kCtlBlockBytes));
  status = reinterpret_cast<DeviceStatus*>(ctlblk);
  ticket = reinterpret_cast<int*>(ctlblk + 32);
  abort_flag = reinterpret_cast<int*>(ctlblk + 36);
  P_TRY(dal(&xseg_dev, 1));
  P_TRY(dal(&lseg_dev, 1));
  P_TRY(dal(&level, n));
  P_TRY(dal(&by_level, n));
  P_TRY(cudaMemcpyAsync(lseg_dev, &level, sizeof(int*), cudaMemcpyHostToDevice, stream));
  unsigned long long* xb = reinterpret_cast<unsigned long long*>(xbuf);
  P_TRY(cudaMemcpyAsync(xseg_dev, &xb, sizeof(xb), cudaMemcpyHostToDevice, stream));
  P_TRY(cudaStreamSynchronize(stream));

  // K6: levels (bit-exact) + level-ordered tickets for the component pool
  int rc = run_levels();
  if (rc != SPTRSV_OK) return rc;

  executor_used = SPTRSV_EXECUTOR_ROWS;
  if (!structure_only && opt.executor == SPTRSV_EXECUTOR_PUSH) {
    rc = build_push();
    if (rc != SPTRSV_OK) return rc;
    executor_used = SPTRSV_EXECUTOR_PUSH;
    return SPTRSV_OK;
  }
  if (!structure_only && opt.executor != SPTRSV_EXECUTOR_ROWS) {
    // host copy of the CSR structure for the schedulers
    std::vector<int> h_rp(n + 1), h_ci(noff);
    P_TRY(cudaMemcpy(h_rp.data(), rp, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost));
    if (noff) P_TRY(cudaMemcpy(h_ci.data(), ci, sizeof(int) * noff, cudaMemcpyDeviceToHost));
    if (opt.executor == SPTRSV_EXECUTOR_AUTO || opt.executor == SPTRSV_EXECUTOR_STENCIL) {
      rc = build_stencil(h_rp, h_ci);
      if (rc != SPTRSV_OK) return rc;
      if (stencil.ready) {
        executor_used = SPTRSV_EXECUTOR_STENCIL;
        return SPTRSV_OK;
      }
      rc = build_stencil3d(h_rp, h_ci);
      if (rc != SPTRSV_OK) return rc;
      if (stencil3.ready) {
        executor_used = SPTRSV_EXECUTOR_STENCIL;
        return SPTRSV_OK;
      }
      if (opt.executor == SPTRSV_EXECUTOR_STENCIL)
        return plan_fail(SPTRSV_E_UNSUPPORTED,
                         "stencil executor requested but L is neither 2D five-point nor 3D seven-point lower "
                         "structured");
    }
    if (opt.executor == SPTRSV_EXECUTOR_BAND || (opt.executor == SPTRSV_EXECUTOR_AUTO && band_candidate(h_rp, h_ci))) {
      if (opt.executor == SPTRSV_EXECUTOR_BAND && !band_candidate(h_rp, h_ci)) {
        bool narrow = n >= 128;
        for (long long i = 0; i < n && narrow; ++i)
          if (h_rp[i] < h_rp[i + 1] && i - h_ci[h_rp[i]] > 64) narrow = false;
        if (!narrow) return plan_fail(SPTRSV_E_UNSUPPORTED, "band executor needs every dependency within 64 rows");
      }
      rc = build_band();
      if (rc != SPTRSV_OK) return rc;
      executor_used = SPTRSV_EXECUTOR_BAND;
      return SPTRSV_OK;
    }
    rc = build_chains(h_rp, h_ci);
    if (rc != SPTRSV_OK) return rc;
    if (chains.ready && (opt.executor == SPTRSV_EXECUTOR_CHAINS || chains_preferred()))
      executor_used = SPTRSV_EXECUTOR_CHAINS;
    else if (opt.executor == SPTRSV_EXECUTOR_CHAINS)
      return plan_fail(SPTRSV_E_UNSUPPORTED, "chains schedule could not be built");
  }
  return SPTRSV_OK;
}

}  // namespace sptrsv
