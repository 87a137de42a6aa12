// Host-side scheduler for the lane-chain lockstep executor (see solve_chains.cu).
//
// 1. Tasks: contiguous row ranges [a, b) of the natural (topological) order.
//    Inside a task each row extends the chain of its largest in-task
//    dependency when that row is still a chain tail (its lane's last row);
//    otherwise it opens a new chain = a new lane. A task closes when it
//    would need more lanes than a warp has, or reaches max_rows.
// 2. Steps: ASAP lockstep list schedule, step(i) = max(step(prev in lane) + 1,
//    step(j) + 1 over in-task deps j). Every task starts with kPrefetch empty
//    steps whose only job is to launch the first prefetches.
// 3. Sources: a dependency is read from a register (chain predecessor), the
//    smem ring (same task, < kRingSteps steps old), the inbox (a value of an
//    earlier task prefetched kPrefetch steps ahead; first kMaxInbox per row)
//    or a direct mailbox poll (anything else). Mailboxes are value-is-flag.
// 4. Emit slices (one per step) packed into <= kChunkBytes chunks; rows with
//    more than kInlineDeps dependencies continue in an overflow list.
//
// Deadlock freedom: tasks are dealt in ascending order by a ticket counter and
// only wait on earlier tasks (mailboxes of rows < a) or on earlier steps of
// their own schedule — the reference's ascending-order progress rule
// (engine.py:30-35) lifted from components to tasks.
#include <vector>
#include <algorithm>
#include <cstring>
#include <chrono>
#include "plan.hpp"
#include "kernels.cuh"

namespace sptrsv {

int plan_fail(int code, const char* msg);

struct ScheduleInput {
  int n;
  const int* rp;
  const int* ci;
  const double* val;  // cv (exact) or wv (fast)
  const double* dg;
  const double* rdg;
  bool exact;
  int lanes;
  int max_rows;
};

struct ScheduleOutput {
  std::vector<unsigned char> stream;
  std::vector<long long> chunk_off;
  std::vector<int> chunk_steps;
  std::vector<int> chunk_width;
  std::vector<int> task_chunk;
  std::vector<int> ovf_src;
  std::vector<double> ovf_val;
  long long n_mbox = 0;
  int max_width = 0;
  int n_inbox = 0;
  long long deps_total = 0, deps_in_task = 0, deps_ring = 0, deps_reg = 0, deps_mbox = 0, deps_inbox = 0;
  long long n_slices = 0, max_task_steps = 0;
  bool ok = true;
};

// Dependency d of a row with nd dependencies is stored inline in its slice
// (else in the overflow list, whose mailbox reads are always direct polls).
static inline bool inline_dep(int d, int nd) { return nd <= kInlineDeps || d < kInlineDeps - 1; }

static void build_schedule(const ScheduleInput& in, ScheduleOutput& out) {
  const int n = in.n;
  const int* rp = in.rp;
  const int* ci = in.ci;
  const int L = in.lanes;
  const int P = kPrefetch;
  std::vector<int> lane_of(n), step_of(n), task_start;
  task_start.reserve(1024);

  // pass 1: tasks, lanes, steps (steps start at P: the first P are prefetch-only)
  {
    int a = 0, nl = 0;
    int tail[32], last_step[32];
    auto reset = [&]() {
      nl = 0;
      for (int q = 0; q < 32; ++q) tail[q] = -1, last_step[q] = P - 1;
    };
    reset();
    task_start.push_back(0);
    int i = 0;
    while (i < n) {
      const int lo = rp[i], hi = rp[i + 1];
      if (i - a >= in.max_rows) {
        a = i;
        reset();
        task_start.push_back(a);
      }
      int p = (hi > lo && ci[hi - 1] >= a) ? ci[hi - 1] : -1;
      int lane;
      if (p >= 0 && tail[lane_of[p]] == p) {
        lane = lane_of[p];
      } else {
        if (nl == L) {  // needs one chain more than a warp has: close the task before row i
          a = i;
          reset();
          task_start.push_back(a);
          continue;
        }
        lane = nl++;
      }
      int s = last_step[lane] + 1;
      for (int k = lo; k < hi; ++k) {
        const int j = ci[k];
        if (j >= a) s = std::max(s, step_of[j] + 1);
      }
      lane_of[i] = lane;
      step_of[i] = s;
      tail[lane] = i;
      last_step[lane] = s;
      ++i;
    }
    task_start.push_back(n);
  }
  const int n_tasks = (int)task_start.size() - 1;

  // pass 2: classify dependencies; mailboxes for rows read across tasks or
  // from too far back in the same task; inbox width of the plan
  std::vector<int> mbox_of(n, -1);
  int max_inbox = 0;
  {
    std::vector<int> prev_in_lane(32);
    for (int t = 0; t < n_tasks; ++t) {
      const int a = task_start[t], b = task_start[t + 1];
      std::fill(prev_in_lane.begin(), prev_in_lane.end(), -1);
      for (int i = a; i < b; ++i) {
        const int li = lane_of[i];
        int inbox = 0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
          const int j = ci[k];
          ++out.deps_total;
          if (j < a) {
            ++out.deps_mbox;
            if (inbox < kMaxInbox && inline_dep(k - rp[i], rp[i + 1] - rp[i])) ++inbox;
            if (mbox_of[j] < 0) mbox_of[j] = (int)out.n_mbox++;
            continue;
          }
          ++out.deps_in_task;
          if (j == prev_in_lane[li]) ++out.deps_reg;  // statistic: chain predecessor (read from the ring)
          if (step_of[i] - step_of[j] < kRingSteps) {
            ++out.deps_ring;
          } else {
            ++out.deps_mbox;
            if (mbox_of[j] < 0) mbox_of[j] = (int)out.n_mbox++;
          }
        }
        max_inbox = std::max(max_inbox, inbox);
        prev_in_lane[li] = i;
      }
    }
  }
  const int M = max_inbox;
  out.n_inbox = M;

  // pass 3: emit slices and chunks
  out.task_chunk.reserve(n_tasks + 1);
  out.chunk_off.push_back(0);
  std::vector<int> count, first, rows_by_step;
  std::vector<int> prev_in_lane(32);
  auto& st = out.stream;
  st.reserve((size_t)n * 52 + (size_t)rp[n] * 12 + 4096);
  for (int t = 0; t < n_tasks; ++t) {
    const int a = task_start[t], b = task_start[t + 1];
    out.task_chunk.push_back((int)out.chunk_steps.size());
    int nsteps = 0;
    for (int i = a; i < b; ++i) nsteps = std::max(nsteps, step_of[i] + 1);
    out.max_task_steps = std::max<long long>(out.max_task_steps, nsteps);
    count.assign(nsteps + 1, 0);
    for (int i = a; i < b; ++i) ++count[step_of[i] + 1];
    for (int s = 0; s < nsteps; ++s) count[s + 1] += count[s];
    first = count;
    rows_by_step.assign(b - a, 0);
    for (int i = a; i < b; ++i) rows_by_step[first[step_of[i]]++] = i;
    auto rows_at = [&](int s, int* row) {
      for (int q = 0; q < 32; ++q) row[q] = -1;
      if (s >= nsteps) return;
      for (int r = count[s]; r < count[s + 1]; ++r) row[lane_of[rows_by_step[r]]] = rows_by_step[r];
    };
    std::fill(prev_in_lane.begin(), prev_in_lane.end(), -1);
    // slice widths, then chunks of uniform width (the kernel computes slice
    // addresses from the chunk's width instead of loading them)
    std::vector<int> widths(nsteps, 0);
    for (int s = 0; s < nsteps; ++s)
      for (int r = count[s]; r < count[s + 1]; ++r) {
        const int i = rows_by_step[r];
        widths[s] = std::max(widths[s], std::min(rp[i + 1] - rp[i], kInlineDeps));
      }
    std::vector<int> chunk_of_step(nsteps), chunk_w;
    for (int s = 0; s < nsteps;) {
      int w = widths[s], cnt = 1;
      while (s + cnt < nsteps && (cnt + 1) * slice_bytes(std::max(w, widths[s + cnt]), M, in.exact) <= kChunkBytes) {
        w = std::max(w, widths[s + cnt]);
        ++cnt;
      }
      for (int k = 0; k < cnt; ++k) chunk_of_step[s + k] = (int)chunk_w.size();
      chunk_w.push_back(w);
      s += cnt;
    }
    int chunk_steps = 0;
    int row[32], pf[32];
    for (int s = 0; s < nsteps; ++s) {
      rows_at(s, row);
      rows_at(s + P, pf);
      const int width = chunk_w[chunk_of_step[s]];
      out.max_width = std::max(out.max_width, width);
      const int bytes = slice_bytes(width, M, in.exact);
      if (s > 0 && chunk_of_step[s] != chunk_of_step[s - 1]) {
        out.chunk_steps.push_back(chunk_steps);
        out.chunk_width.push_back(chunk_w[chunk_of_step[s - 1]]);
        out.chunk_off.push_back((long long)st.size());
        chunk_steps = 0;
      }
      const size_t base = st.size();
      st.resize(base + bytes);
      unsigned char* p = st.data() + base;
      std::memset(p, 0, bytes);
      const SliceGeom g(width, M, in.exact);
      int32_t* srow = reinterpret_cast<int32_t*>(p);
      int32_t* smbo = reinterpret_cast<int32_t*>(p + 128);
      int32_t* spf = reinterpret_cast<int32_t*>(p + 256);
      int32_t* spfm = reinterpret_cast<int32_t*>(p + g.pfm);
      double* srdg = reinterpret_cast<double*>(p + g.rdg);
      double* sdg = reinterpret_cast<double*>(p + g.dg);
      int32_t* ssrc = reinterpret_cast<int32_t*>(p + g.src);
      double* sval = reinterpret_cast<double*>(p + g.val);
      for (int q = 0; q < 32; ++q) {
        // prefetch fields for step s + P: b of that row, its inbox mailboxes
        const int f = pf[q];
        spf[q] = f;
        int m = 0;
        if (f >= 0) {
          const int fnd = rp[f + 1] - rp[f];
          for (int k = rp[f]; k < rp[f + 1] && m < M; ++k)
            if (ci[k] < a && inline_dep(k - rp[f], fnd)) spfm[m++ * 32 + q] = mbox_of[ci[k]];
        }
        for (; m < M; ++m) spfm[m * 32 + q] = -1;

        const int i = row[q];
        srow[q] = i;
        for (int d = 0; d < width; ++d) ssrc[d * 32 + q] = kSrcSkip;
        if (i < 0) {
          smbo[q] = -1;
          continue;
        }
        smbo[q] = mbox_of[i];
        srdg[q] = in.rdg ? in.rdg[i] : 0.0;
        if (in.exact) sdg[q] = in.dg ? in.dg[i] : 0.0;
        const int nd = rp[i + 1] - rp[i];
        const bool spill = nd > kInlineDeps;
        int inbox = 0;
        for (int d = 0; d < nd; ++d) {
          const int k = rp[i] + d;
          const int j = ci[k];
          int code;
          if (j < a) {
            if (inline_dep(d, nd) && inbox < M) {
              code = inbox_offset(inbox, s, q);  // prefetched kPrefetch steps ago
              ++inbox;
              ++out.deps_inbox;
            } else {
              code = kSrcDirect - mbox_of[j];
            }
          } else if (s - step_of[j] < kRingSteps) {
            code = ring_offset(step_of[j], lane_of[j]);  // includes the chain predecessor
          } else {
            code = kSrcDirect - mbox_of[j];
          }
          if (spill && d >= kInlineDeps - 1) {
            if (d == kInlineDeps - 1) {
              // slot kInlineDeps-1 points at the overflow list holding deps d..nd-1
              const long long start = (long long)out.ovf_src.size();
              const long long cnt = nd - d;
              ssrc[d * 32 + q] = kSrcOverflow;
              const long long packed = (start << 24) | cnt;
              std::memcpy(&sval[d * 32 + q], &packed, 8);
            }
            out.ovf_src.push_back(code);
            out.ovf_val.push_back(in.val ? in.val[k] : 0.0);
          } else {
            ssrc[d * 32 + q] = code;
            sval[d * 32 + q] = in.val ? in.val[k] : 0.0;
          }
        }
        prev_in_lane[q] = i;
      }
      ++chunk_steps;
      ++out.n_slices;
    }
    if (chunk_steps > 0) {
      out.chunk_steps.push_back(chunk_steps);
      out.chunk_width.push_back(chunk_w.back());
      out.chunk_off.push_back((long long)st.size());
    }
  }
  out.task_chunk.push_back((int)out.chunk_steps.size());
}

int DevicePlan::build_chains(const std::vector<int>& h_rp, const std::vector<int>& h_ci) {
  auto t0 = std::chrono::steady_clock::now();
  chains.release();
  chains.exact = opt.precision != SPTRSV_PRECISION_FAST;
  chains.lanes = opt.chain_lanes;
  // host copies of the device CSR values (the structure is passed in)
  std::vector<double> h_val(noff), h_dg(chains.exact ? n : 0), h_rdg(n);
  cudaError_t e;
  if ((noff && (e = cudaMemcpy(h_val.data(), chains.exact ? cv : wv, sizeof(double) * noff, cudaMemcpyDeviceToHost)) !=
                   cudaSuccess) ||
      (chains.exact && (e = cudaMemcpy(h_dg.data(), dg, sizeof(double) * n, cudaMemcpyDeviceToHost)) != cudaSuccess) ||
      (e = cudaMemcpy(h_rdg.data(), rdg, sizeof(double) * n, cudaMemcpyDeviceToHost)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));

  ScheduleInput in{(int)n, h_rp.data(), h_ci.data(), h_val.data(), chains.exact ? h_dg.data() : nullptr,
                   h_rdg.data(), chains.exact, chains.lanes, 1 << 22};
  ScheduleOutput out;
  build_schedule(in, out);
  chains.max_width = out.max_width;
  chains.n_inbox = out.n_inbox;
  chains.deps_total = out.deps_total;
  chains.deps_in_task = out.deps_in_task;
  chains.deps_ring = out.deps_ring;
  chains.deps_reg = out.deps_reg;
  chains.deps_mbox = out.deps_mbox;
  chains.deps_inbox = out.deps_inbox;
  if (!out.ok) {
    chains.ready = false;
    return SPTRSV_OK;
  }
  chains.n_tasks = (int)out.task_chunk.size() - 1;
  chains.n_chunks = (long long)out.chunk_steps.size();
  chains.n_slices = out.n_slices;
  chains.n_mbox = out.n_mbox;
  chains.n_overflow = (long long)out.ovf_src.size();
  chains.stream_bytes = (long long)out.stream.size();
  chains.max_task_steps = out.max_task_steps;
  auto al = [](void** p, size_t bytes) { return cudaMalloc(p, bytes < 16 ? 16 : bytes); };
  if ((e = al((void**)&chains.stream, out.stream.size())) != cudaSuccess ||
      (e = al((void**)&chains.chunk_off, sizeof(long long) * out.chunk_off.size())) != cudaSuccess ||
      (e = al((void**)&chains.chunk_steps, sizeof(int) * out.chunk_steps.size())) != cudaSuccess ||
      (e = al((void**)&chains.chunk_width, sizeof(int) * out.chunk_width.size())) != cudaSuccess ||
      (e = al((void**)&chains.task_chunk, sizeof(int) * out.task_chunk.size())) != cudaSuccess ||
      (e = al((void**)&chains.mbox, 16 * (size_t)out.n_mbox)) != cudaSuccess ||  // 16-byte slots
      (e = al((void**)&chains.ovf_src, sizeof(int) * out.ovf_src.size())) != cudaSuccess ||
      (e = al((void**)&chains.ovf_val, sizeof(double) * out.ovf_val.size())) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  cudaMemcpy(chains.stream, out.stream.data(), out.stream.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(chains.chunk_off, out.chunk_off.data(), sizeof(long long) * out.chunk_off.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(chains.chunk_steps, out.chunk_steps.data(), sizeof(int) * out.chunk_steps.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(chains.chunk_width, out.chunk_width.data(), sizeof(int) * out.chunk_width.size(), cudaMemcpyHostToDevice);
  if (!out.ovf_src.empty()) {
    cudaMemcpy(chains.ovf_src, out.ovf_src.data(), sizeof(int) * out.ovf_src.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(chains.ovf_val, out.ovf_val.data(), sizeof(double) * out.ovf_val.size(), cudaMemcpyHostToDevice);
  }
  if ((e = cudaMemcpy(chains.task_chunk, out.task_chunk.data(), sizeof(int) * out.task_chunk.size(),
                      cudaMemcpyHostToDevice)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  chains.ready = true;
  chains.schedule_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return SPTRSV_OK;
}

bool DevicePlan::chains_preferred() const {
  // Lockstep warps pay off when most dependencies stay inside a warp task and
  // rows are short; otherwise the component pool wins (RMAT, wide bands).
  return chains.ready && chains.max_width <= 8 && chains.in_task_fraction() >= 0.6;
}

}  // namespace sptrsv
