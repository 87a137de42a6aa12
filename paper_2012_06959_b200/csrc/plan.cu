// Plan construction: upload the CSC arrays once, then validation, in-degree
// (K1), CSC->CSR transpose, row scaling, level analysis (K6) and — when the
// structure suits it — the lane-chain schedule. All of it is "setup" in the
// reference's vocabulary (engine.py:445-490 + analysis.py:43-64).
#include <string>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
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
  // SPTRSV_SETUP_TRACE=1: phase times of plan creation on stderr (diagnostics)
  static const bool trace = std::getenv("SPTRSV_SETUP_TRACE") != nullptr;
  auto tr0 = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!trace) return;
    cudaStreamSynchronize(stream);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[setup] %-28s %9.1f ms\n", what, std::chrono::duration<double, std::milli>(now - tr0).count());
    tr0 = now;
  };
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
  mark("upload + validate");
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
  mark("in-degree + CSR transpose");
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
  mark("scratch");
  // host copy of the CSR structure for structure detection and the schedulers
  std::vector<int> h_rp, h_ci;
  int grid_dims[3] = {0, 0, 0};
  bool grid_known = false;
  // (structure-only plans too: detection needs only the pattern, and a grid
  // stencil's levels have a closed form)
  if (!indeg_only && opt.executor != SPTRSV_EXECUTOR_ROWS && opt.executor != SPTRSV_EXECUTOR_PUSH) {
    h_rp.resize(n + 1);
    h_ci.resize(noff);
    P_TRY(cudaMemcpy(h_rp.data(), rp, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost));
    if (noff) P_TRY(cudaMemcpy(h_ci.data(), ci, sizeof(int) * noff, cudaMemcpyDeviceToHost));
    mark("CSR to host");
    if (opt.executor == SPTRSV_EXECUTOR_AUTO || opt.executor == SPTRSV_EXECUTOR_STENCIL) {
      if (const int nx = detect_stencil2d(n, h_rp, h_ci)) {
        grid_dims[0] = nx, grid_dims[1] = (int)(n / nx), grid_dims[2] = 0;
        grid_known = true;
      } else if (detect_stencil3d(n, h_rp, h_ci, grid_dims)) {
        grid_known = true;
      }
      mark("structure detection");
    }
  }
  // a narrow band: levels from the band window kernel in (max, +1) mode
  // (the pool would pay a memory round trip per level: 4.7 M levels)
  bool levels_done = false;
  if (!grid_known && !h_rp.empty() && !structure_only &&
      (opt.executor == SPTRSV_EXECUTOR_AUTO || opt.executor == SPTRSV_EXECUTOR_BAND) && band_narrow(h_rp, h_ci)) {
    int brc = build_band();
    if (brc != SPTRSV_OK) return brc;
    brc = band_levels(level);
    if (brc != SPTRSV_OK) return brc;
    levels_done = true;
    mark("band structure + levels");
  }
  int rc = run_levels(grid_known ? grid_dims : nullptr, levels_done);
  mark("levels + ticket order");
  if (rc != SPTRSV_OK) return rc;
  // keep the band (n x 64 doubles) only if the band executor will run on it
  if (band.ready && !(opt.executor == SPTRSV_EXECUTOR_BAND ||
                      (opt.executor == SPTRSV_EXECUTOR_AUTO && n_levels > n / 8)))
    band.release();
  if (rc != SPTRSV_OK) return rc;

  executor_used = SPTRSV_EXECUTOR_ROWS;
  if (!structure_only && opt.executor == SPTRSV_EXECUTOR_PUSH) {
    rc = build_push();
    if (rc != SPTRSV_OK) return rc;
    executor_used = SPTRSV_EXECUTOR_PUSH;
    return SPTRSV_OK;
  }
  if (!structure_only && opt.executor != SPTRSV_EXECUTOR_ROWS) {
    if (opt.executor == SPTRSV_EXECUTOR_AUTO || opt.executor == SPTRSV_EXECUTOR_STENCIL) {
      rc = build_stencil(h_rp, h_ci);
      if (rc != SPTRSV_OK) return rc;
      mark("stencil detect + pack");
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
      if (!band.ready) {
        rc = build_band();
        if (rc != SPTRSV_OK) return rc;
      }
      executor_used = SPTRSV_EXECUTOR_BAND;
      if (opt.precision == SPTRSV_PRECISION_FAST) {  // fast mode: the row-block formulation (band_blocks.cu)
        rc = build_band_blocks();
        if (rc != SPTRSV_OK) return rc;
        mark("band blocks (coupling tails)");
      }
      return SPTRSV_OK;
    }
    // AUTO prefers lane chains only when every row has at most 8 dependencies
    // (chains_preferred); skip building a schedule that cannot win
    int max_deps = 0;
    if (opt.executor == SPTRSV_EXECUTOR_AUTO)
      for (long long i = 0; i < n; ++i) max_deps = std::max(max_deps, h_rp[i + 1] - h_rp[i]);
    if (opt.executor == SPTRSV_EXECUTOR_AUTO && max_deps > 8) return SPTRSV_OK;
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
