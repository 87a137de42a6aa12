// C ABI (include/sptrsv_b200.h): plan lifetime, preprocessing pipeline and the
// solve entry points. Host-side runtime in C++; all compute is device kernels.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <chrono>
#include <algorithm>
#include "../../include/sptrsv_b200.h"
#include "common.cuh"
#include "kernels.cuh"
#include "plan.hpp"

using namespace sptrsv;

namespace {
thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
}  // namespace

namespace sptrsv {
int plan_fail(int code, const char* msg) { return fail(code, msg); }
}  // namespace sptrsv

namespace {

#define CUDA_TRY(expr)                                                                     \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) return fail(SPTRSV_E_CUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
  } while (0)

template <class T>
cudaError_t dalloc(T** p, size_t count) {
  return cudaMalloc((void**)p, std::max<size_t>(count, 1) * sizeof(T));
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}
}  // namespace

namespace sptrsv {

void DevicePlan::release() {
  cudaSetDevice(device);
  void* ptrs[] = {rp, ci, cv, wv, dg, rdg, indeg, level, by_level, level_ptr, order, xbuf, bbuf, ctlblk,
                  xseg_dev, lseg_dev, probe_buf};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  chains.release();
  stencil.release();
  stencil3.release();
  push.release();
  band.release();
  bblk.release();
  split_rows.release();
  release_partition();
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (evk0) cudaEventDestroy(evk0);
  if (evk1) cudaEventDestroy(evk1);
  if (stream) cudaStreamDestroy(stream);
  if (cs_in) cudaStreamDestroy(cs_in);
  if (cs_out) cudaStreamDestroy(cs_out);
}

int DevicePlan::run_levels(const int* grid, bool precomputed) {
  // K6: level_i = 1 + max(level_j) over dependencies, 0 without any; the
  // component pool in (max,+1) arithmetic over the natural (topological) order
  // — or, for a verified 2D / 3D lower stencil, its closed form: row
  // (x, y[, z]) depends exactly on (x-1, ...), (x, y-1, ...)[, (x, y, z-1)],
  // so its earliest level is x + y (+ z), the same integers.
  if (precomputed) {
    // `level` already holds the levels (the band window kernel)
  } else if (grid) {
    CUDA_TRY(launch_grid_levels(level, n, grid[0], grid[1], grid[2], stream));
  } else {
  CUDA_TRY(cudaMemsetAsync(level, 0xFF, sizeof(int) * (size_t)n, stream));
  CUDA_TRY(reset_control(stream));
  RowsArgs a{};
  a.n = (int)n;
  a.rp = rp;
  a.ci = ci;
  a.lseg = lseg_dev;
  a.xseg = xseg_dev;
  a.order = nullptr;
  a.order_len = n;
  a.ticket = ticket;
  a.status = status;
  a.abort_flag = abort_flag;
  a.timeout_ns = (unsigned long long)(std::max(opt.timeout_s, 600.0) * 1e9);  // analysis is not under the solve watchdog
  a.spin_initial = opt.spin_initial;
  a.spin_max_ns = opt.spin_max_ns;
  a.coop_long = 0;
  a.long_deps = 1 << 30;
  CUDA_TRY(launch_rows(kModeLevel, a, rows_grid(kModeLevel), stream));
  DeviceStatus hs{};
  CUDA_TRY(cudaMemcpyAsync(&hs, status, sizeof(hs), cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  if (hs.code == SPTRSV_E_TIMEOUT) return fail(SPTRSV_E_TIMEOUT, "level analysis exceeded the timeout");
  }

  // group components by level: stable sort (level, row) -> ascending rows per level
  int *iota = nullptr, *keys_out = nullptr, *cnt = nullptr, *tick = nullptr, *tb = nullptr;
  CUDA_TRY(dalloc(&iota, n));
  CUDA_TRY(dalloc(&keys_out, n));
  CUDA_TRY(launch_iota(iota, (int)n, stream));
  CUDA_TRY(sort_pairs_stable(level, keys_out, iota, by_level, n, (int)n, stream));
  int last = 0;
  if (n > 0) CUDA_TRY(cudaMemcpyAsync(&last, keys_out + n - 1, sizeof(int), cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  n_levels = n > 0 ? last + 1 : 0;
  CUDA_TRY(dalloc(&level_ptr, n_levels + 1));
  CUDA_TRY(dalloc(&cnt, n_levels + 1));
  CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int) * (n_levels + 1), stream));
  CUDA_TRY(launch_level_hist(level, (int)n, cnt, stream));
  CUDA_TRY(scan_exclusive(cnt, level_ptr, n_levels + 1, stream));
  // ticket layout for the component pool: single-level tickets when the
  // padding costs < 2x, which enables warp-wide long rows
  CUDA_TRY(dalloc(&tick, n_levels + 1));
  CUDA_TRY(dalloc(&tb, n_levels + 1));
  CUDA_TRY(cudaMemsetAsync(tick, 0, sizeof(int) * (n_levels + 1), stream));
  CUDA_TRY(launch_tickets_per_level(cnt, n_levels, tick, stream));
  CUDA_TRY(scan_exclusive(tick, tb, n_levels + 1, stream));
  int total_tickets = 0;
  CUDA_TRY(cudaMemcpyAsync(&total_tickets, tb + n_levels, sizeof(int), cudaMemcpyDeviceToHost, stream));
  CUDA_TRY(cudaStreamSynchronize(stream));
  long long padded = 32ll * total_tickets;
  // Rows with more than kLongDeps dependencies are solved warp-wide; each gets
  // a ticket of its own (after the level's short rows, packed 32 per ticket),
  // so the long rows of one level run on different warps in parallel instead
  // of one after another in the warp that drew them (power-law in-degrees:
  // rmat-4M has 2,759 rows with > 1024 dependencies in 721 levels).
  std::vector<int> h_order;
  if (n > 0 && !structure_only) {
    std::vector<int> h_by(n), h_lp(n_levels + 1), h_rp(n + 1);
    CUDA_TRY(cudaMemcpy(h_by.data(), by_level, sizeof(int) * n, cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(h_lp.data(), level_ptr, sizeof(int) * (n_levels + 1), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemcpy(h_rp.data(), rp, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost));
    h_order.reserve(padded);
    // fast mode splits rows with > kSplitDeps dependencies into partial tasks
    // of kSplitDeps entries, one warp each, placed before the level's long
    // rows: the level then costs ~one memory round trip per warp however
    // heavy its heaviest row (rmat-4M: 29,079 dependencies)
    const bool split = opt.precision == SPTRSV_PRECISION_FAST;
    std::vector<int> hv_idx, hv_parts, pt_beg, pt_end, pt_heavy;
    if (split) hv_idx.assign(n, -1);
    std::vector<int> longs;
    for (int L = 0; L < n_levels; ++L) {
      longs.clear();
      size_t in_ticket = 0;
      for (int k = h_lp[L]; k < h_lp[L + 1]; ++k) {
        const int r = h_by[k];
        if (h_rp[r + 1] - h_rp[r] > kLongDeps) {
          longs.push_back(r);
        } else {
          h_order.push_back(r);
          in_ticket = (in_ticket + 1) % 32;
        }
      }
      if (in_ticket) h_order.resize(h_order.size() + (32 - in_ticket), -1);
      for (int r : longs) {
        const int deg = h_rp[r + 1] - h_rp[r];
        if (!split || deg <= kSplitDeps) continue;
        const int h = (int)hv_parts.size();
        hv_idx[r] = h;
        hv_parts.push_back((deg + kSplitDeps - 1) / kSplitDeps);
        for (int b0 = h_rp[r]; b0 < h_rp[r + 1]; b0 += kSplitDeps) {
          h_order.push_back((int)n + (int)pt_beg.size());
          h_order.resize(h_order.size() + 31, -1);
          pt_beg.push_back(b0);
          pt_end.push_back(std::min(b0 + kSplitDeps, h_rp[r + 1]));
          pt_heavy.push_back(h);
        }
      }
      for (int r : longs) {
        h_order.push_back(r);
        h_order.resize(h_order.size() + 31, -1);
      }
    }
    padded = (long long)h_order.size();
    if (!hv_parts.empty() && (long long)n + (long long)pt_beg.size() < (1ll << 31)) {
      auto up = [&](int** d, const std::vector<int>& h) -> cudaError_t {
        cudaError_t e = dalloc(d, h.size());
        return e != cudaSuccess ? e : cudaMemcpy(*d, h.data(), sizeof(int) * h.size(), cudaMemcpyHostToDevice);
      };
      CUDA_TRY(up(&split_rows.heavy_idx, hv_idx));
      CUDA_TRY(up(&split_rows.heavy_parts, hv_parts));
      CUDA_TRY(up(&split_rows.part_beg, pt_beg));
      CUDA_TRY(up(&split_rows.part_end, pt_end));
      CUDA_TRY(up(&split_rows.part_heavy, pt_heavy));
      CUDA_TRY(dalloc(&split_rows.part_sum, hv_parts.size()));
      CUDA_TRY(dalloc(&split_rows.part_done, hv_parts.size()));
      split_rows.n_heavy = (int)hv_parts.size();
    } else if (!hv_parts.empty()) {
      // (cannot encode the partial tasks in int32: keep whole rows)
      h_order.erase(std::remove_if(h_order.begin(), h_order.end(), [&](int v) { return v >= (int)n; }),
                    h_order.end());
      padded = (long long)h_order.size();
    }
  }
  if (n > 0 && !structure_only && padded <= 8 * n) {
    CUDA_TRY(dalloc(&order, padded));
    CUDA_TRY(cudaMemcpy(order, h_order.data(), sizeof(int) * padded, cudaMemcpyHostToDevice));
    order_len = padded;
    coop_long = 1;
  } else if (n > 0 && padded <= 2 * n) {
    CUDA_TRY(dalloc(&order, padded));
    CUDA_TRY(cudaMemsetAsync(order, 0xFF, sizeof(int) * padded, stream));
    CUDA_TRY(launch_pad_order(by_level, level, level_ptr, tb, (int)n, order, stream));
    order_len = padded;
    coop_long = 1;
  } else {
    CUDA_TRY(dalloc(&order, n));
    CUDA_TRY(cudaMemcpyAsync(order, by_level, sizeof(int) * n, cudaMemcpyDeviceToDevice, stream));
    order_len = n;
    coop_long = 0;
  }
  CUDA_TRY(cudaStreamSynchronize(stream));
  cudaFree(iota);
  cudaFree(keys_out);
  cudaFree(cnt);
  cudaFree(tick);
  cudaFree(tb);
  return SPTRSV_OK;
}

int DevicePlan::rows_grid(int mode) const {
  static const int forced = [] {  // SPTRSV_ROWS_GRID: fixed block count (A/B)
    const char* v = std::getenv("SPTRSV_ROWS_GRID");
    return v ? std::atoi(v) : 0;
  }();
  if (forced > 0) return forced;
  int per_sm = rows_blocks_per_sm(mode);
  if (per_sm < 1) per_sm = 1;
  long long want = (order_len + 255) / 256;
  long long cap = (long long)num_sms * per_sm;
  if (want < 1) want = 1;
  return (int)std::min(want, cap);
}

int DevicePlan::solve_rows(const double* d_b, double* d_x, cudaStream_t s) {
  const int mode = opt.precision == SPTRSV_PRECISION_FAST ? kModeFast : kModeExact;
  CUDA_TRY(cudaMemsetAsync(d_x, 0xFF, sizeof(double) * (size_t)n, s));
  CUDA_TRY(reset_control(s));
  unsigned long long* xs = reinterpret_cast<unsigned long long*>(d_x);
  CUDA_TRY(cudaMemcpyAsync(xseg_dev, &xs, sizeof(xs), cudaMemcpyHostToDevice, s));
  RowsArgs a{};
  a.n = (int)n;
  a.rp = rp;
  a.ci = ci;
  a.val = mode == kModeFast ? wv : cv;
  a.dg = dg;
  a.rdg = rdg;
  a.b = d_b;
  a.xseg = xseg_dev;
  a.lseg = lseg_dev;
  a.order = order;
  a.order_len = order_len;
  a.ticket = ticket;
  a.status = status;
  a.abort_flag = abort_flag;
  a.timeout_ns = (unsigned long long)(opt.timeout_s * 1e9);
  a.spin_initial = opt.spin_initial;
  a.spin_max_ns = opt.spin_max_ns;
  a.coop_long = coop_long;
  a.long_deps = kLongDeps;
  a.lane_loop = rows_lane_loop();
  if (mode == kModeFast && split_rows.n_heavy) {
    CUDA_TRY(cudaMemsetAsync(split_rows.part_sum, 0, sizeof(double) * split_rows.n_heavy, s));
    CUDA_TRY(cudaMemsetAsync(split_rows.part_done, 0, sizeof(int) * split_rows.n_heavy, s));
    a.heavy_idx = split_rows.heavy_idx;
    a.heavy_parts = split_rows.heavy_parts;
    a.part_beg = split_rows.part_beg;
    a.part_end = split_rows.part_end;
    a.part_heavy = split_rows.part_heavy;
    a.part_sum = split_rows.part_sum;
    a.part_done = split_rows.part_done;
  }
  a.debug = (opt.flags & SPTRSV_PLAN_DEBUG) ? ((opt.probe_flags & 1024) ? 2 : 1) : 0;
  if (opt.probe_flags & 512) {
    // diagnostics: globaltimer of every row's publish (tools/rows_levels.py)
    if (!probe_buf || probe_words < n) {
      if (probe_buf) cudaFree(probe_buf);
      probe_buf = nullptr;
      CUDA_TRY(dalloc(&probe_buf, std::max<long long>(n, kProbeWords)));
      probe_words = std::max<long long>(n, kProbeWords);
    }
    a.stamps = probe_buf;
  }
  CUDA_TRY(record_k0(s));
  CUDA_TRY(launch_rows(mode, a, rows_grid(mode), s));
  CUDA_TRY(cudaEventRecord(evk1, s));
  launches = 1;
  return SPTRSV_OK;
}

int DevicePlan::solve_device_many(const double* d_b, double* d_x, int k, cudaStream_t s) {
  if (structure_only) return fail(SPTRSV_E_ARGUMENT, "plan was created structure-only; it cannot solve");
  if (k == 1) return solve_device(d_b, d_x, s);
  // the 2D stencil stacks up to kMaxStack right-hand sides per launch: its
  // 64 bands use 64 of the 148 SMs, so stacked copies fill the idle SMs and
  // each copy's bands start as soon as an SM frees up
  constexpr int kMaxStack = 16;
  const bool stack = executor_used == SPTRSV_EXECUTOR_STENCIL && !stencil3.ready && stencil.ready && !stencil.part &&
                     !seg_table && stencil.ny % 64 == 0;
  CUDA_TRY(cudaEventRecord(ev0, s));
  int total_launches = 0;
  for (int r = 0; r < k;) {
    const int c = stack ? std::min(kMaxStack, k - r) : 1;
    const double* b = d_b + (size_t)r * n;
    double* x = d_x + (size_t)r * n;
    int rc;
    if (stack && c > 1) rc = solve_stencil(b, x, s, false, false, c);
    else if (executor_used == SPTRSV_EXECUTOR_STENCIL)
      rc = stencil3.ready ? solve_stencil3d(b, x, s) : solve_stencil(b, x, s);
    else if (executor_used == SPTRSV_EXECUTOR_PUSH) rc = solve_push(b, x, s);
    else if (executor_used == SPTRSV_EXECUTOR_BAND) rc = bblk.ready ? solve_band_blocks(b, x, s) : solve_band(b, x, s);
    else if (executor_used == SPTRSV_EXECUTOR_CHAINS) rc = solve_chains(b, x, s);
    else rc = solve_rows(b, x, s);
    batch_k0 = true;  // the kernel events span every launch of the batch
    if (rc != SPTRSV_OK) {
      batch_k0 = false;
      return rc;
    }
    total_launches += launches;
    r += c;
  }
  launches = total_launches;
  batch_k0 = false;
  CUDA_TRY(cudaEventRecord(ev1, s));
  pending = true;
  return SPTRSV_OK;
}

int DevicePlan::solve_device(const double* d_b, double* d_x, cudaStream_t s) {
  if (structure_only) return fail(SPTRSV_E_ARGUMENT, "plan was created structure-only; it cannot solve");
  int rc;
  CUDA_TRY(cudaEventRecord(ev0, s));
  if (stencil.part) rc = solve_stencil(d_b, d_x, s);
  else if (seg_table) rc = solve_partitioned_rows(d_b, d_x, s);
  else if (executor_used == SPTRSV_EXECUTOR_STENCIL)
    rc = stencil3.ready ? solve_stencil3d(d_b, d_x, s) : solve_stencil(d_b, d_x, s);
  else if (executor_used == SPTRSV_EXECUTOR_PUSH) rc = solve_push(d_b, d_x, s);
  else if (executor_used == SPTRSV_EXECUTOR_BAND) rc = bblk.ready ? solve_band_blocks(d_b, d_x, s) : solve_band(d_b, d_x, s);
  else if (executor_used == SPTRSV_EXECUTOR_CHAINS) rc = solve_chains(d_b, d_x, s);
  else rc = solve_rows(d_b, d_x, s);
  if (rc != SPTRSV_OK) return rc;
  CUDA_TRY(cudaEventRecord(ev1, s));
  pending = true;
  return SPTRSV_OK;
}

// Stream memory operations (cuStreamWriteValue32 / cuStreamWaitValue32),
// fetched through the runtime so the library does not link libcuda.
namespace {
typedef int (*PfnValue32)(cudaStream_t, unsigned long long, unsigned, unsigned);
PfnValue32 g_write32 = nullptr, g_wait32 = nullptr;
bool stream_memops() {
  static int state = 0;  // 0 unknown, 1 available, -1 not
  if (state == 0) {
    void *w = nullptr, *t = nullptr;
    cudaDriverEntryPointQueryResult qw, qt;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &w, cudaEnableDefault, &qw) == cudaSuccess &&
        cudaGetDriverEntryPoint("cuStreamWaitValue32", &t, cudaEnableDefault, &qt) == cudaSuccess &&
        qw == cudaDriverEntryPointSuccess && qt == cudaDriverEntryPointSuccess && w && t) {
      g_write32 = reinterpret_cast<PfnValue32>(w);
      g_wait32 = reinterpret_cast<PfnValue32>(t);
      state = 1;
    } else {
      cudaGetLastError();
      state = -1;
    }
  }
  return state == 1;
}
constexpr unsigned kWaitGeq = 0;  // CU_STREAM_WAIT_VALUE_GEQ
}  // namespace

bool DevicePlan::streamed_io_ok() const {
  // a CUDA tool attached through the injection interface (Nsight Compute,
  // compute-sanitizer) serialises kernels and copies: the kernel would wait
  // for b flags that only a concurrent copy stream writes (until the watchdog)
  static const bool tool = std::getenv("CUDA_INJECTION64_PATH") != nullptr ||
                           std::getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") != nullptr ||   // ncu
                           std::getenv("NV_SANITIZER_INJECTION_TRANSPORT_TYPE") != nullptr;  // compute-sanitizer
  return !tool && executor_used == SPTRSV_EXECUTOR_STENCIL && !seg_table && !stencil.part &&
         !(opt.flags & SPTRSV_PLAN_NO_STREAMED_IO) &&
         (stencil3.ready ? stencil3.bflag != nullptr : stencil.bflag != nullptr) && stream_memops();
}

// Pinned host memory (cudaHostAlloc / cudaHostRegister under UVA): the whole
// [p, p + bytes). Only such buffers get the overlapped copies: copies from
// pageable memory block the host thread and would serialise the pipeline.
static bool device_mapped_host(const void* p, size_t bytes) {
  const void* ends[2] = {p, static_cast<const char*>(p) + bytes - 1};
  for (const void* q : ends) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, q) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (at.type != cudaMemoryTypeHost || at.devicePointer != q) return false;
  }
  return true;
}

// Host-buffer solve for the stencil executor. The kernel is launched first;
// its loader waits per band for bflag[t] >= epoch, which the input copy stream
// writes after band t's slice of b. The output stream waits per band for the
// kernel's xflag[t] >= epoch and copies that slice of x out. After the kernel
// the solve stream writes every xflag itself, so an aborted kernel (watchdog)
// can never leave the output stream waiting.
// The 3D executor's version: b in z-slabs (k3R planes, one row of tiles),
// doubling copies up to 8 slabs, flagged on their last slab; x per 2 slabs,
// each copy waiting on the flag of its last tile (flags rise in tile order).
int DevicePlan::solve_host_streamed3d(const double* b, double* x, sptrsv_stats* st) {
  auto t0 = std::chrono::steady_clock::now();
  Stencil3Plan& P = stencil3;
  const unsigned ep = ++P.epoch;
  const long long slab = 4LL * P.ny * P.nx;  // k3R planes
  static const int in_max = [] {
    const char* e = std::getenv("SPTRSV_STREAM3_IN");
    return e && std::atoi(e) > 0 ? std::atoi(e) : 8;
  }();
  static const int out_n = [] {
    const char* e = std::getenv("SPTRSV_STREAM3_OUT");
    return e && std::atoi(e) > 0 ? std::atoi(e) : 2;
  }();
  const int ns = P.nzt;
  P.b_chunk_max = in_max;
  CUDA_TRY(cudaEventRecord(ev0, stream));
  int rc = solve_stencil3d(bbuf, xbuf, stream, true);
  if (rc != SPTRSV_OK) return rc;
  CUDA_TRY(cudaEventRecord(ev1, stream));
  pending = true;
  CUDA_TRY(stencil_release_flags(P.xflag, P.n_tasks, ep, stream));
  for (int s0 = 0, w = 1; s0 < ns; s0 += w, w = std::min(2 * w, in_max)) {
    const int s1 = std::min(ns, s0 + w);
    const long long off = s0 * slab, cnt = std::min(slab * (s1 - s0), n - off);
    CUDA_TRY(cudaMemcpyAsync(bbuf + off, b + off, sizeof(double) * cnt, cudaMemcpyHostToDevice, cs_in));
    if (g_write32(cs_in, (unsigned long long)(P.bflag + s1 - 1), ep, 0) != 0)
      return fail(SPTRSV_E_CUDA, "cuStreamWriteValue32 failed");
  }
  for (int s0 = 0; s0 < ns; s0 += out_n) {
    const int s1 = std::min(ns, s0 + out_n);
    const long long off = s0 * slab, cnt = std::min(slab * (s1 - s0), n - off);
    if (g_wait32(cs_out, (unsigned long long)(P.xflag + (long long)s1 * P.nyt - 1), ep, kWaitGeq) != 0)
      return fail(SPTRSV_E_CUDA, "cuStreamWaitValue32 failed");
    CUDA_TRY(cudaMemcpyAsync(x + off, xbuf + off, sizeof(double) * cnt, cudaMemcpyDeviceToHost, cs_out));
  }
  CUDA_TRY(cudaStreamSynchronize(cs_in));
  CUDA_TRY(cudaStreamSynchronize(cs_out));
  rc = finish(st);
  if (rc != SPTRSV_OK) return rc;
  if (st) {
    st->h2d_ms = 0.0;
    st->d2h_ms = 0.0;
    st->e2e_ms = ms_since(t0);
    st->streamed_io = 1;
  }
  return SPTRSV_OK;
}

int DevicePlan::solve_host_streamed(const double* b, double* x, sptrsv_stats* st) {
  if (!cs_in) CUDA_TRY(cudaStreamCreateWithFlags(&cs_in, cudaStreamNonBlocking));
  if (!cs_out) CUDA_TRY(cudaStreamCreateWithFlags(&cs_out, cudaStreamNonBlocking));
  if (stencil3.ready) return solve_host_streamed3d(b, x, st);
  auto t0 = std::chrono::steady_clock::now();
  const unsigned ep = ++stencil.epoch;
  const long long band = (long long)kStBand * stencil.nx;
  const int nt = stencil.n_tasks;
  // Copy granularity (bands per copy): b goes in doubling chunks (1, 2, 4, 8
  // bands: the first band starts the kernel early, bigger copies keep the link
  // efficient); x comes out 2 bands at a time. Tunable by SPTRSV_STREAM_IN /
  // SPTRSV_STREAM_OUT (lap2d-4096: 3.8-4.4 ms over 1..16 bands per copy, also
  // with big x copies until the tail; the PCIe link shared by both directions
  // is the limit: 3.3 ms for the same copy pattern without the solve,
  // tools/pcie_pattern.py).
  // One stream memory operation per copy, not per band: each one costs the
  // copy stream a gap (64 flag writes + 64 waits + 64 post-kernel writes were
  // ~1 ms of a 4.3 ms solve).
  static const int in_max = [] {
    const char* e = std::getenv("SPTRSV_STREAM_IN");
    return e && std::atoi(e) > 0 ? std::atoi(e) : 8;
  }();
  static const int out_n = [] {
    const char* e = std::getenv("SPTRSV_STREAM_OUT");
    return e && std::atoi(e) > 0 ? std::atoi(e) : 2;
  }();
  stencil.b_chunk_max = in_max;
  CUDA_TRY(cudaEventRecord(ev0, stream));
  int rc = solve_stencil(bbuf, xbuf, stream, true, true);
  if (rc != SPTRSV_OK) return rc;
  CUDA_TRY(cudaEventRecord(ev1, stream));
  pending = true;
  // never leave the x copies waiting if the kernel stopped early
  CUDA_TRY(stencil_release_flags(stencil.xflag, nt, ep, stream));
  for (int t0b = 0, w = 1; t0b < nt; t0b += w, w = std::min(2 * w, in_max)) {
    const int t1b = std::min(nt, t0b + w);
    const long long off = t0b * band, cnt = std::min(band * (t1b - t0b), n - off);
    CUDA_TRY(cudaMemcpyAsync(bbuf + off, b + off, sizeof(double) * cnt, cudaMemcpyHostToDevice, cs_in));
    if (g_write32(cs_in, (unsigned long long)(stencil.bflag + t1b - 1), ep, 0) != 0)
      return fail(SPTRSV_E_CUDA, "cuStreamWriteValue32 failed");
  }
  for (int t0b = 0; t0b < nt; t0b += out_n) {
    const int t1b = std::min(nt, t0b + out_n);
    const long long off = t0b * band, cnt = std::min(band * (t1b - t0b), n - off);
    for (int t = SPTRSV_ST_XFLAG_ORDER ? t1b - 1 : t0b; t < t1b; ++t)
      if (g_wait32(cs_out, (unsigned long long)(stencil.xflag + t), ep, kWaitGeq) != 0)
        return fail(SPTRSV_E_CUDA, "cuStreamWaitValue32 failed");
    CUDA_TRY(cudaMemcpyAsync(x + off, xbuf + off, sizeof(double) * cnt, cudaMemcpyDeviceToHost, cs_out));
  }
  CUDA_TRY(cudaStreamSynchronize(cs_in));
  CUDA_TRY(cudaStreamSynchronize(cs_out));
  rc = finish(st);
  if (rc != SPTRSV_OK) return rc;
  if (st) {
    st->h2d_ms = 0.0;  // overlapped with the solve
    st->d2h_ms = 0.0;
    st->e2e_ms = ms_since(t0);
    st->streamed_io = 1;
  }
  return SPTRSV_OK;
}

int DevicePlan::finish(sptrsv_stats* st) {
  CUDA_TRY(cudaStreamSynchronize(stream));
  DeviceStatus hs{};
  CUDA_TRY(cudaMemcpy(&hs, status, sizeof(hs), cudaMemcpyDeviceToHost));
  float ms = 0.f, kms = 0.f;
  if (pending) {
    CUDA_TRY(cudaEventElapsedTime(&ms, ev0, ev1));
    CUDA_TRY(cudaEventElapsedTime(&kms, evk0, evk1));
  }
  pending = false;
  last_solve_ms = ms;
  last_spins = (long long)hs.spins;
  last_remote = (long long)hs.remote_reads;
  if (st) {
    st->setup_ms = setup_ms;
    st->solve_ms = ms;
    st->kernel_ms = kms;
    st->spins = (int64_t)hs.spins;
    st->remote_reads = (int64_t)hs.remote_reads;
    st->launches = launches;
    st->executor = executor_used;
    st->n_levels = n_levels;
  }
  if (hs.code == SPTRSV_E_TIMEOUT)
    return fail(SPTRSV_E_TIMEOUT, "solve exceeded " + std::to_string(opt.timeout_s) + "s (device watchdog)");
  if (hs.code == SPTRSV_E_DEBUG_CHECK)
    return fail(SPTRSV_E_DEBUG_CHECK, "debug check failed: publication of component " + std::to_string(hs.detail) +
                                          " was not a single owner write over its sentinel");
  return SPTRSV_OK;
}

}  // namespace sptrsv

// ---------------------------------------------------------------------------

extern "C" {

void sptrsv_default_options(sptrsv_options* opt) {
  std::memset(opt, 0, sizeof(*opt));
  opt->precision = SPTRSV_PRECISION_EXACT;
  opt->executor = SPTRSV_EXECUTOR_AUTO;
  opt->device = 0;
  opt->timeout_s = 60.0;
  opt->spin_initial = 1024;  // Backoff(16, 512) of the reference: 16 x 64 device polls, then sleeps up to 512/8 ns
  opt->spin_max_ns = 64;
  opt->chain_lanes = 32;
}

int sptrsv_abi_version(void) { return 1; }
int sptrsv_sizeof_options(void) { return (int)sizeof(sptrsv_options); }
int sptrsv_sizeof_stats(void) { return (int)sizeof(sptrsv_stats); }

const char* sptrsv_last_error(void) { return g_err.c_str(); }

int sptrsv_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return c;
}

int sptrsv_plan_create(const int64_t* col_ptr, const int64_t* row_idx, const double* values, int64_t n,
                       const sptrsv_options* opt_in, sptrsv_plan** out, int64_t* bad_col) {
  g_err.clear();
  if (!out || !col_ptr || (n > 0 && !row_idx)) return fail(SPTRSV_E_ARGUMENT, "null argument");
  *out = nullptr;
  if (bad_col) *bad_col = -1;
  sptrsv_options opt;
  if (opt_in) opt = *opt_in;
  else sptrsv_default_options(&opt);
  if (opt.chain_lanes <= 0 || opt.chain_lanes > 32) opt.chain_lanes = 32;
  const bool structure_only = (opt.flags & SPTRSV_PLAN_STRUCTURE_ONLY) != 0;
  if (!structure_only && n > 0 && !values) return fail(SPTRSV_E_ARGUMENT, "values required");
  if (n < 0) return fail(SPTRSV_E_STRUCTURE, "negative dimension");
  const long long nnz = col_ptr[n];
  if (col_ptr[0] != 0 || nnz < 0) return fail(SPTRSV_E_STRUCTURE, "malformed col_ptr");
  if (n >= (1ll << 31) - 1 || nnz >= (1ll << 31) - 1)
    return fail(SPTRSV_E_UNSUPPORTED, "n and nnz must be < 2^31 (int32 device indices)");
  for (long long j = 0; j < n; ++j)
    if (col_ptr[j + 1] < col_ptr[j]) return fail(SPTRSV_E_STRUCTURE, "col_ptr is not non-decreasing");

  auto t0 = std::chrono::steady_clock::now();
  auto* p = new DevicePlan();
  p->opt = opt;
  p->n = n;
  p->nnz = nnz;
  p->device = opt.device;
  p->structure_only = structure_only;
  int rc = p->build(col_ptr, row_idx, values, bad_col);
  if (rc != SPTRSV_OK) {
    std::string keep = g_err;
    p->release();
    delete p;
    g_err = keep;
    return rc;
  }
  p->setup_ms = ms_since(t0);
  *out = reinterpret_cast<sptrsv_plan*>(p);
  return SPTRSV_OK;
}

int sptrsv_plan_in_degrees(const sptrsv_plan* plan, int64_t* out) {
  g_err.clear();
  auto* p = reinterpret_cast<const DevicePlan*>(plan);
  if (!p || !out) return fail(SPTRSV_E_ARGUMENT, "null argument");
  CUDA_TRY(cudaSetDevice(p->device));
  long long* tmp = nullptr;
  CUDA_TRY(dalloc(&tmp, p->n));
  CUDA_TRY(launch_widen(p->indeg, tmp, p->n, p->stream));
  CUDA_TRY(cudaMemcpyAsync(out, tmp, sizeof(long long) * p->n, cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  cudaFree(tmp);
  return SPTRSV_OK;
}

int sptrsv_plan_levels(const sptrsv_plan* plan, int64_t* level_of, int64_t* order, int64_t* level_ptr,
                       int64_t* n_levels) {
  g_err.clear();
  auto* p = reinterpret_cast<const DevicePlan*>(plan);
  if (!p) return fail(SPTRSV_E_ARGUMENT, "null plan");
  CUDA_TRY(cudaSetDevice(p->device));
  if (n_levels) *n_levels = p->n_levels;
  long long* tmp = nullptr;
  CUDA_TRY(dalloc(&tmp, p->n + 1));
  if (level_of) {
    CUDA_TRY(launch_widen(p->level, tmp, p->n, p->stream));
    CUDA_TRY(cudaMemcpyAsync(level_of, tmp, sizeof(long long) * p->n, cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
  }
  if (order) {
    CUDA_TRY(launch_widen(p->by_level, tmp, p->n, p->stream));
    CUDA_TRY(cudaMemcpyAsync(order, tmp, sizeof(long long) * p->n, cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
  }
  if (level_ptr) {
    CUDA_TRY(launch_widen(p->level_ptr, tmp, p->n_levels + 1, p->stream));
    CUDA_TRY(cudaMemcpyAsync(level_ptr, tmp, sizeof(long long) * (p->n_levels + 1), cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
  }
  cudaFree(tmp);
  return SPTRSV_OK;
}

int sptrsv_in_degrees(const int64_t* col_ptr, const int64_t* row_idx, int64_t n, int32_t device, int64_t* out) {
  sptrsv_options opt;
  sptrsv_default_options(&opt);
  opt.device = device;
  opt.flags = SPTRSV_PLAN_STRUCTURE_ONLY | 2 /* in-degree only */;
  sptrsv_plan* plan = nullptr;
  int rc = sptrsv_plan_create(col_ptr, row_idx, nullptr, n, &opt, &plan, nullptr);
  if (rc != SPTRSV_OK) return rc;
  rc = sptrsv_plan_in_degrees(plan, out);
  sptrsv_plan_destroy(plan);
  return rc;
}

int sptrsv_solve(sptrsv_plan* plan, const double* b, double* x, sptrsv_stats* stats) {
  g_err.clear();
  auto* p = reinterpret_cast<DevicePlan*>(plan);
  if (!p || (p->n > 0 && (!b || !x))) return fail(SPTRSV_E_ARGUMENT, "null argument");
  CUDA_TRY(cudaSetDevice(p->device));
  if (p->n == 0) return p->finish(stats);
  if (p->structure_only) return fail(SPTRSV_E_ARGUMENT, "plan was created structure-only; it cannot solve");
  // band-granular copy overlap needs pinned buffers (pageable copies block the host)
  if (p->streamed_io_ok() && device_mapped_host(b, sizeof(double) * p->n) &&
      device_mapped_host(x, sizeof(double) * p->n))
    return p->solve_host_streamed(b, x, stats);
  auto t0 = std::chrono::steady_clock::now();
  CUDA_TRY(cudaMemcpyAsync(p->bbuf, b, sizeof(double) * p->n, cudaMemcpyHostToDevice, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  double h2d = ms_since(t0);
  int rc = p->solve_device(p->bbuf, p->xbuf, p->stream);
  if (rc != SPTRSV_OK) return rc;
  rc = p->finish(stats);
  if (rc != SPTRSV_OK) return rc;
  auto t1 = std::chrono::steady_clock::now();
  CUDA_TRY(cudaMemcpyAsync(x, p->xbuf, sizeof(double) * p->n, cudaMemcpyDeviceToHost, p->stream));
  CUDA_TRY(cudaStreamSynchronize(p->stream));
  if (stats) {
    stats->h2d_ms = h2d;
    stats->d2h_ms = ms_since(t1);
    stats->e2e_ms = ms_since(t0);
  }
  return SPTRSV_OK;
}

int sptrsv_solve_device_many_async(sptrsv_plan* plan, const double* d_b, double* d_x, int32_t k, void* stream) {
  g_err.clear();
  auto* p = reinterpret_cast<DevicePlan*>(plan);
  if (!p || k < 0) return fail(SPTRSV_E_ARGUMENT, "null plan or negative k");
  if (p->n == 0 || k == 0) return SPTRSV_OK;
  if (!d_b || !d_x) return fail(SPTRSV_E_ARGUMENT, "null argument");
  CUDA_TRY(cudaSetDevice(p->device));
  cudaStream_t s = stream ? reinterpret_cast<cudaStream_t>(stream) : p->stream;
  return p->solve_device_many(d_b, d_x, k, s);
}

int sptrsv_solve_many(sptrsv_plan* plan, const double* b, double* x, int32_t k, sptrsv_stats* stats) {
  g_err.clear();
  auto* p = reinterpret_cast<DevicePlan*>(plan);
  if (!p || k < 0) return fail(SPTRSV_E_ARGUMENT, "null plan or negative k");
  if (p->n == 0 || k == 0) return p->finish(stats);
  if (!b || !x) return fail(SPTRSV_E_ARGUMENT, "null argument");
  CUDA_TRY(cudaSetDevice(p->device));
  const size_t bytes = sizeof(double) * (size_t)p->n * k;
  double *db = nullptr, *dx = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&db, bytes, p->stream));
  CUDA_TRY(cudaMallocAsync((void**)&dx, bytes, p->stream));
  auto t0 = std::chrono::steady_clock::now();
  CUDA_TRY(cudaMemcpyAsync(db, b, bytes, cudaMemcpyHostToDevice, p->stream));
  int rc = p->solve_device_many(db, dx, k, p->stream);
  if (rc == SPTRSV_OK) rc = p->finish(stats);
  if (rc == SPTRSV_OK) {
    CUDA_TRY(cudaMemcpyAsync(x, dx, bytes, cudaMemcpyDeviceToHost, p->stream));
    CUDA_TRY(cudaStreamSynchronize(p->stream));
    if (stats) stats->e2e_ms = ms_since(t0);
  }
  cudaFreeAsync(db, p->stream);
  cudaFreeAsync(dx, p->stream);
  cudaStreamSynchronize(p->stream);
  return rc;
}

int sptrsv_solve_device_async(sptrsv_plan* plan, const double* d_b, double* d_x, void* stream) {
  g_err.clear();
  auto* p = reinterpret_cast<DevicePlan*>(plan);
  if (!p) return fail(SPTRSV_E_ARGUMENT, "null plan");
  if (p->n == 0) return SPTRSV_OK;
  CUDA_TRY(cudaSetDevice(p->device));
  cudaStream_t s = stream ? reinterpret_cast<cudaStream_t>(stream) : p->stream;
  return p->solve_device(d_b, d_x, s);
}

int sptrsv_plan_last_counters(const sptrsv_plan* plan, int64_t* spins, int64_t* remote_reads) {
  g_err.clear();
  auto* p = reinterpret_cast<const DevicePlan*>(plan);
  if (!p) return fail(SPTRSV_E_ARGUMENT, "null plan");
  if (spins) *spins = p->last_spins;
  if (remote_reads) *remote_reads = p->last_remote;
  return SPTRSV_OK;
}

int sptrsv_synchronize(sptrsv_plan* plan, sptrsv_stats* stats) {
  g_err.clear();
  auto* p = reinterpret_cast<DevicePlan*>(plan);
  if (!p) return fail(SPTRSV_E_ARGUMENT, "null plan");
  CUDA_TRY(cudaSetDevice(p->device));
  CUDA_TRY(cudaDeviceSynchronize());
  return p->finish(stats);
}

int sptrsv_plan_get_info(const sptrsv_plan* plan, sptrsv_plan_info* info) {
  g_err.clear();
  auto* p = reinterpret_cast<const DevicePlan*>(plan);
  if (!p || !info) return fail(SPTRSV_E_ARGUMENT, "null argument");
  std::memset(info, 0, sizeof(*info));
  info->n = p->n;
  info->nnz = p->nnz;
  info->n_offdiag = p->noff;
  info->n_levels = p->n_levels;
  info->executor = p->executor_used;
  info->setup_ms = p->setup_ms;
  const ChainPlan& c = p->chains;
  info->chains_ready = c.ready ? 1 : 0;
  info->chain_tasks = c.n_tasks;
  info->chain_slices = c.n_slices;
  info->chain_stream_bytes = c.stream_bytes;
  info->chain_mailboxes = c.n_mbox;
  info->chain_max_width = c.max_width;
  info->chain_lanes = c.lanes;
  info->deps_total = c.deps_total;
  info->deps_in_task = c.deps_in_task;
  info->deps_register = c.deps_reg;
  info->deps_ring = c.deps_ring;
  info->deps_mailbox = c.deps_mbox;
  info->chain_max_task_steps = c.max_task_steps;
  info->schedule_ms = c.schedule_ms;
  return SPTRSV_OK;
}

int sptrsv_plan_probe_read(const sptrsv_plan* plan, int64_t* out, int32_t count) {
  g_err.clear();
  auto* p = reinterpret_cast<const DevicePlan*>(plan);
  if (!p || !out) return fail(SPTRSV_E_ARGUMENT, "null argument");
  if (!p->probe_buf) return fail(SPTRSV_E_ARGUMENT, "no probe data: set options.probe_flags");
  CUDA_TRY(cudaSetDevice(p->device));
  CUDA_TRY(cudaMemcpy(out, p->probe_buf, sizeof(long long) * std::min<long long>(count, p->probe_words),
                      cudaMemcpyDeviceToHost));
  return SPTRSV_OK;
}

int sptrsv_plan_destroy(sptrsv_plan* plan) {
  auto* p = reinterpret_cast<DevicePlan*>(plan);
  if (!p) return SPTRSV_OK;
  p->release();
  delete p;
  return SPTRSV_OK;
}

}  // extern "C"
