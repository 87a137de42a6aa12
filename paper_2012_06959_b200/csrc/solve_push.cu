// Push executor: the paper's shared-atomics solve (Alg. 2, /root/reference/
// PAPER.md:160-206; reference solve_shared_atomics, engine.py:324-431) on one
// B200 — the column-oriented sync-free SpTRSV the paper starts from.
//
// * A persistent grid of warps takes components (columns) in level order from
//   one ticket counter (ascending dispatch: the progress rule of
//   engine.py:30-35 — the earliest unsolved column always belongs to a running
//   warp).
// * Warp per component: lane 0 spins on the column's
//   in-degree counter s_in[j] until it equals dep(j) (lock-wait, with the
//   reference's Backoff mapped to __nanosleep), reads the accumulated left sum
//   s_ls[j], solves x_j, and the warp scatters the column: first every
//   left-sum update (fp64 atomicAdd, RED.E.ADD.F64), then one fence, then
//   every counter increment, so a consumer that sees its counter complete also
//   sees all of its left-sum contributions (the reference's update order,
//   engine.py:398-416).
// * Arithmetic: exact mode keeps the reference's form x_j = (b_j - left_j) /
//   l_jj with a correctly rounded division; fast mode pre-scales
//   (left_j accumulates -l_ij/l_ii * x_j, x_j = b_j/l_jj + left_j). Atomic
//   accumulation commutes in arbitrary order, so results match the serial
//   solve to rounding (the reference engines are likewise nondeterministic at
//   rounding level), not bit for bit.
//
// Counters and sums live in HBM and are reset by the solve; the CSC of the
// off-diagonals is built once at plan time from the CSR (stable sort by
// column keeps rows ascending inside a column).
#include <algorithm>
#include "plan.hpp"
#include "kernels.cuh"

namespace sptrsv {

int plan_fail(int code, const char* msg);

namespace {

struct PushArgs {
  int n;
  const int* cp;         // CSC of the off-diagonals: column pointers
  const int* ri;         //   row of each entry
  const double* val;     //   l_ij (exact) or -l_ij / l_ii (fast)
  const double* dg;
  const double* rdg;
  const int* indeg;      // dep(i): off-diagonals in row i
  const int* order;      // components in level order
  const double* b;
  double* x;
  double* left;          // s_ls (reset to 0 per solve)
  int* count;            // s_in (reset to 0 per solve)
  int* ticket;
  DeviceStatus* status;
  int* abort_flag;
  unsigned long long timeout_ns;
  int spin_initial, spin_max_ns;
};

__device__ __forceinline__ int ld_acquire_gpu_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_sys_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kPushBatch = 8;

// SYS: the shared state is unified (managed) memory updated with
// system-scope atomics and polled with system-scope acquires (the paper's
// Unified-Memory design; SPTRSV_PLAN_PUSH_MANAGED)
template <bool FAST, bool SYS>
__global__ void __launch_bounds__(256) k_push(PushArgs a) {
  const int lane = threadIdx.x & 31;
  const unsigned long long deadline = a.timeout_ns ? globaltimer_ns() + a.timeout_ns : 0;
  unsigned long long spins = 0;
  int t = 0, t_end = 0;
  while (true) {
    // tickets of kPushBatch consecutive components (fewer atomics on the pool)
    if (t == t_end) {
      if (lane == 0) t = atomicAdd(a.ticket, 1) * kPushBatch;
      t = __shfl_sync(0xffffffffu, t, 0);
      t_end = min(t + kPushBatch, a.n);
    }
    if (t >= a.n) break;
    const int j = a.order[t++];
    double xj = 0.0;
    int ok = 1;
    if (lane == 0) {
      // lock-wait on the in-degree counter (engine.py:497-521 / 367-380)
      const int need = a.indeg[j];
      int polls = 0, sleep_ns = 32;
      while ((SYS ? ld_acquire_sys_s32(a.count + j) : ld_acquire_gpu_s32(a.count + j)) < need) {
        ++spins;
        if (++polls > a.spin_initial) {
          if ((polls & 63) == 0) {
            if (ld_relaxed_s32(a.abort_flag)) { ok = 0; break; }
            if (deadline && globaltimer_ns() > deadline) {
              atomicExch(&a.status->code, 5);
              atomicExch(a.abort_flag, 1);
              ok = 0;
              break;
            }
          }
          __nanosleep(sleep_ns);
          if (sleep_ns < a.spin_max_ns) sleep_ns <<= 1;
        }
      }
      if (ok) {
        const double s = __ldcg(a.left + j);  // L2: the atomics' coherence point
        xj = FAST ? __dadd_rn(__dmul_rn(a.b[j], a.rdg[j]), s) : div_exact(__dsub_rn(a.b[j], s), a.dg[j], a.rdg[j]);
        a.x[j] = xj;
      }
    }
    if (!__shfl_sync(0xffffffffu, ok, 0)) break;
    xj = __shfl_sync(0xffffffffu, xj, 0);
    const int beg = a.cp[j], end = a.cp[j + 1];
    for (int k = beg + lane; k < end; k += 32) {
      if (SYS) atomicAdd_system(a.left + __ldg(a.ri + k), __ldg(a.val + k) * xj);
      else atomicAdd(a.left + __ldg(a.ri + k), __ldg(a.val + k) * xj);
    }
    __syncwarp();
    if (SYS) __threadfence_system();
    else __threadfence();  // every left-sum update before any counter increment
    for (int k = beg + lane; k < end; k += 32) {
      if (SYS) atomicAdd_system(a.count + __ldg(a.ri + k), 1);
      else atomicAdd(a.count + __ldg(a.ri + k), 1);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) spins += __shfl_xor_sync(0xffffffffu, spins, off);
  if (lane == 0 && spins) atomicAdd(&a.status->spins, spins);
}

__global__ void k_row_of_entry(const int* __restrict__ rp, int n, int* __restrict__ row) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    for (int k = rp[i]; k < rp[i + 1]; ++k) row[k] = i;
}

__global__ void k_gather_csc(const int* __restrict__ entry, const int* __restrict__ row_of,
                             const double* __restrict__ cv, const double* __restrict__ wv, long long noff,
                             int* __restrict__ ri, double* __restrict__ v_exact, double* __restrict__ v_fast) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < noff;
       k += (long long)gridDim.x * blockDim.x) {
    const int e = entry[k];
    ri[k] = row_of[e];
    v_exact[k] = cv[e];
    v_fast[k] = wv[e];
  }
}

}  // namespace

int DevicePlan::build_push() {
  auto al = [](void** p, size_t b) { return cudaMalloc(p, b < 16 ? 16 : b); };
  // the shared state: unified memory for the Unified-Memory baseline
  const bool managed = (opt.flags & SPTRSV_PLAN_PUSH_MANAGED) != 0;
  auto alm = [&](void** p, size_t b) {
    return managed ? cudaMallocManaged(p, b < 16 ? 16 : b, cudaMemAttachGlobal) : cudaMalloc(p, b < 16 ? 16 : b);
  };
  cudaError_t e;
  int *row_of = nullptr, *iota = nullptr, *keys_s = nullptr, *entry_s = nullptr;
  const int grid = (int)std::min<long long>(std::max<long long>(noff, n) / 256 + 1, 148 * 32);
  auto done = [&](cudaError_t err) {
    cudaFree(row_of);
    cudaFree(iota);
    cudaFree(keys_s);
    cudaFree(entry_s);
    return err == cudaSuccess ? SPTRSV_OK : plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(err));
  };
  if ((e = al((void**)&push.cp, sizeof(int) * (n + 1))) != cudaSuccess ||
      (e = al((void**)&push.ri, sizeof(int) * noff)) != cudaSuccess ||
      (e = al((void**)&push.v_exact, sizeof(double) * noff)) != cudaSuccess ||
      (e = al((void**)&push.v_fast, sizeof(double) * noff)) != cudaSuccess ||
      (e = alm((void**)&push.left, sizeof(double) * n)) != cudaSuccess ||
      (e = alm((void**)&push.count, sizeof(int) * n)) != cudaSuccess ||
      (e = al((void**)&row_of, sizeof(int) * noff)) != cudaSuccess ||
      (e = al((void**)&iota, sizeof(int) * noff)) != cudaSuccess ||
      (e = al((void**)&keys_s, sizeof(int) * noff)) != cudaSuccess ||
      (e = al((void**)&entry_s, sizeof(int) * noff)) != cudaSuccess)
    return done(e);
  // column counts -> CSC pointers; entries stably sorted by column
  int* ccount1 = nullptr;
  if ((e = al((void**)&ccount1, sizeof(int) * (n + 1))) != cudaSuccess) return done(e);
  if ((e = cudaMemsetAsync(ccount1, 0, sizeof(int) * (n + 1), stream)) != cudaSuccess ||
      (noff && (e = launch_level_hist(ci, (int)noff, ccount1, stream)) != cudaSuccess) ||
      (e = scan_exclusive(ccount1, push.cp, (int)n + 1, stream)) != cudaSuccess) {
    cudaFree(ccount1);
    return done(e);
  }
  if (noff) {
    k_row_of_entry<<<grid, 256, 0, stream>>>(rp, (int)n, row_of);
    if ((e = cudaGetLastError()) != cudaSuccess || (e = launch_iota(iota, (int)noff, stream)) != cudaSuccess ||
        (e = sort_pairs_stable(ci, keys_s, iota, entry_s, noff, (int)n, stream)) != cudaSuccess) {
      cudaFree(ccount1);
      return done(e);
    }
    k_gather_csc<<<grid, 256, 0, stream>>>(entry_s, row_of, cv, wv, noff, push.ri, push.v_exact, push.v_fast);
    if ((e = cudaGetLastError()) != cudaSuccess) {
      cudaFree(ccount1);
      return done(e);
    }
  }
  e = cudaStreamSynchronize(stream);
  cudaFree(ccount1);
  if (e != cudaSuccess) return done(e);
  push.ready = true;
  return done(cudaSuccess);
}

int DevicePlan::solve_push(const double* d_b, double* d_x, cudaStream_t s) {
  if (!push.ready) return plan_fail(SPTRSV_E_UNSUPPORTED, "push executor was not built for this plan");
  const bool fast = opt.precision == SPTRSV_PRECISION_FAST;
  cudaError_t e;
  if ((e = cudaMemsetAsync(push.left, 0, sizeof(double) * n, s)) != cudaSuccess ||
      (e = cudaMemsetAsync(push.count, 0, sizeof(int) * n, s)) != cudaSuccess ||
      (e = reset_control(s)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  PushArgs a{};
  a.n = (int)n;
  a.cp = push.cp;
  a.ri = push.ri;
  a.val = fast ? push.v_fast : push.v_exact;
  a.dg = dg;
  a.rdg = rdg;
  a.indeg = indeg;
  a.order = by_level;
  a.b = d_b;
  a.x = d_x;
  a.left = push.left;
  a.count = push.count;
  a.ticket = ticket;
  a.status = status;
  a.abort_flag = abort_flag;
  a.timeout_ns = (unsigned long long)(opt.timeout_s * 1e9);
  a.spin_initial = opt.spin_initial;
  a.spin_max_ns = opt.spin_max_ns;
  const bool sys = (opt.flags & SPTRSV_PLAN_PUSH_MANAGED) != 0;
  int per_sm = 0;
  if (fast) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_push<true, false>, 256, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_push<false, false>, 256, 0);
  const int blocks = std::max(1, num_sms * std::max(per_sm, 1));
  if ((e = record_k0(s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if (fast) sys ? k_push<true, true><<<blocks, 256, 0, s>>>(a) : k_push<true, false><<<blocks, 256, 0, s>>>(a);
  else sys ? k_push<false, true><<<blocks, 256, 0, s>>>(a) : k_push<false, false><<<blocks, 256, 0, s>>>(a);
  if ((e = cudaGetLastError()) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if ((e = cudaEventRecord(evk1, s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  launches = 1;
  return SPTRSV_OK;
}

}  // namespace sptrsv
