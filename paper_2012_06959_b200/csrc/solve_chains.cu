// Lane-chain lockstep executor ("chains").
//
// Why: on B200 a dependency handed between SMs through L2 costs ~800 cycles
// one way (tools/microbench: volatile ping-pong 1556 cycles round trip), a
// warp-synchronous hand-off through shared memory ~35 cycles, a register 0.
// The sync-free component pool (solve_rows.cu) pays the L2 price on every
// level; on a 2D Laplacian in natural order that is 8191 levels.
//
// How: the host scheduler (schedule.cu) cuts the rows into contiguous tasks
// of <= 32 dependency chains, gives each chain a lane and each row a lockstep
// step. One warp runs one task: at every step each lane solves its row,
// reading the chain predecessor from a register, same-task values from a
// shared-memory ring written in earlier steps, and values of earlier tasks
// from value-is-flag mailboxes in global memory (polled like the component
// pool). Tasks are dealt by an ascending ticket counter to persistent warps.
//
// Data movement: the task's schedule is a byte stream of slices (chains.hpp)
// read exactly once; lane 0 streams it into shared memory with
// cp.async.bulk (TMA bulk copies, mbarrier completion) kChunkBuffers chunks
// ahead, and every lane gathers its b values for the next chunks with
// cp.async (LDGSTS), so the lockstep loop only touches shared memory and
// registers. The next step's slice record is loaded into registers while the
// current step computes.
#include "plan.hpp"
#include "kernels.cuh"

namespace sptrsv {

int plan_fail(int code, const char* msg);

struct ChainArgs {
  const unsigned char* stream;
  const long long* chunk_off;
  const int* chunk_steps;
  const int* task_chunk;
  int n_tasks;
  unsigned long long* mbox;
  int* ticket;
  const double* b;
  double* x;
  DeviceStatus* status;
  int* abort_flag;
  unsigned long long timeout_ns;
  int spin_initial;
  int spin_max_ns;
};

namespace {

constexpr int kSmemChunks = kChunkBuffers * kChunkBytes;
constexpr int kSmemB = kChunkBuffers * kMaxChunkSteps * 32 * 8;
constexpr int kSmemRing = 32 * kRingSteps * 8;
constexpr int kSmemTotal = kSmemChunks + kSmemB + kSmemRing + 64;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned phase) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct Layout {
  int width;
  const int* row;
  const int* mbo;
  const double* rdg;
  const double* dg;
  const int* src;
  const double* val;
  int bytes;
};

template <bool EXACT>
__device__ __forceinline__ Layout slice_at(const unsigned char* p) {
  Layout s;
  s.width = *reinterpret_cast<const int*>(p);
  s.row = reinterpret_cast<const int*>(p + 16);
  s.mbo = reinterpret_cast<const int*>(p + 144);
  s.rdg = reinterpret_cast<const double*>(p + 272);
  s.dg = reinterpret_cast<const double*>(p + 528);
  const int deps = 528 + (EXACT ? 256 : 0);
  s.src = reinterpret_cast<const int*>(p + deps);
  s.val = reinterpret_cast<const double*>(p + deps + 128 * s.width);
  s.bytes = slice_bytes(s.width, EXACT);
  return s;
}

// One lane's view of one step, held in registers one step ahead (W > 0), or
// just the fixed part with deps read in the loop (W == 0).
template <int W>
struct Rec {
  int row, mbo, width;
  double rdg, dg, b;
  int code[W > 0 ? W : 1];
  double val[W > 0 ? W : 1];
};

template <bool EXACT, int W>
__device__ __forceinline__ void load_rec(Rec<W>& r, const Layout& s, const double* bslot, int lane) {
  r.width = s.width;
  r.row = s.row[lane];
  r.mbo = s.mbo[lane];
  r.rdg = s.rdg[lane];
  if (EXACT) r.dg = s.dg[lane];
  r.b = bslot[lane];
  if constexpr (W > 0) {
#pragma unroll
    for (int d = 0; d < W; ++d) {
      if (d < s.width) {
        r.code[d] = s.src[d * 32 + lane];
        r.val[d] = s.val[d * 32 + lane];
      } else {
        r.code[d] = kSrcSkip;
      }
    }
  }
}

struct Waiter {
  const ChainArgs& a;
  unsigned long long spins = 0;
  unsigned long long deadline = 0;
  __device__ explicit Waiter(const ChainArgs& args) : a(args) {
    if (a.timeout_ns) deadline = globaltimer_ns() + a.timeout_ns;
  }
  // Returns false when the launch aborts (watchdog or another warp's abort).
  __device__ __forceinline__ bool mailbox(const unsigned long long* p, double& out) {
    unsigned long long u = ld_relaxed_u64(p);
    int polls = 0, sleep_ns = 32;
    while (u == kNotReady) {
      ++spins;
      ++polls;
      if (polls > a.spin_initial) {
        if ((polls & 63) == 0) {
          if (ld_relaxed_s32(a.abort_flag)) return false;
          if (deadline && globaltimer_ns() > deadline) {
            atomicExch(&a.status->code, 5);
            atomicExch(a.abort_flag, 1);
            return false;
          }
        }
        __nanosleep(sleep_ns);
        if (sleep_ns < a.spin_max_ns) sleep_ns <<= 1;
      }
      u = ld_relaxed_u64(p);
    }
    out = as_f64(u);
    return true;
  }
};

template <bool EXACT>
__device__ __forceinline__ double fold(double acc, double v, double xj) {
  if (EXACT) return __dadd_rn(acc, __dmul_rn(v, xj));
  return __fma_rn(v, xj, acc);
}

// Issue the b gathers (cp.async) for every step of a chunk already in smem.
template <bool EXACT>
__device__ __forceinline__ void gather_b(const unsigned char* buf, int steps, double* barea, const double* b,
                                         int lane) {
  const unsigned char* p = buf;
  for (int s = 0; s < steps; ++s) {
    Layout sl = slice_at<EXACT>(p);
    int row = sl.row[lane];
    if (row >= 0) cp_async8(barea + s * 32 + lane, b + row);
    p += sl.bytes;
  }
  cp_async_commit();
}

template <bool EXACT, int W>
__global__ void __launch_bounds__(32, 1) k_chains(ChainArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* chunks = smem;
  double* barea = reinterpret_cast<double*>(smem + kSmemChunks);
  double* ring = reinterpret_cast<double*>(smem + kSmemChunks + kSmemB);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + kSmemChunks + kSmemB + kSmemRing);
  const int lane = threadIdx.x;
  if (lane == 0) {
    for (int k = 0; k < kChunkBuffers; ++k) mbar_init(&bars[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned phase_bits = 0;  // parity to wait for, per buffer
  Waiter wait(a);
  bool alive = true;

  while (alive) {
    int t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= a.n_tasks) break;
    const int c0 = a.task_chunk[t], c1 = a.task_chunk[t + 1];
    auto buf_of = [&](int c) { return chunks + (size_t)((c - c0) % kChunkBuffers) * kChunkBytes; };
    auto bar_of = [&](int c) { return &bars[(c - c0) % kChunkBuffers]; };
    auto barea_of = [&](int c) { return barea + (size_t)((c - c0) % kChunkBuffers) * kMaxChunkSteps * 32; };
    int issued_hi = c0 - 1, awaited_hi = c0 - 1;
    auto issue = [&](int c) {
      issued_hi = c;
      if (lane == 0) {
        const unsigned bytes = (unsigned)(a.chunk_off[c + 1] - a.chunk_off[c]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar_of(c), bytes);
        bulk_g2s(buf_of(c), a.stream + a.chunk_off[c], bytes, bar_of(c));
      }
    };
    auto await = [&](int c) {
      const int k = (c - c0) % kChunkBuffers;
      const unsigned ph = (phase_bits >> k) & 1u;
      while (!mbar_try_wait(&bars[k], ph)) {
      }
      phase_bits ^= 1u << k;
      awaited_hi = c;
    };
    for (int c = c0; c < c1 && c < c0 + kChunkBuffers; ++c) issue(c);
    await(c0);
    gather_b<EXACT>(buf_of(c0), a.chunk_steps[c0], barea_of(c0), a.b, lane);
    if (c0 + 1 < c1) {
      await(c0 + 1);
      gather_b<EXACT>(buf_of(c0 + 1), a.chunk_steps[c0 + 1], barea_of(c0 + 1), a.b, lane);
    }
    double xprev = 0.0;
    int step = 0;
    for (int c = c0; c < c1; ++c) {
      if (c + 1 < c1) cp_async_wait<1>();
      else cp_async_wait<0>();
      const unsigned char* p = buf_of(c);
      const double* bslot = barea_of(c);
      const int steps = a.chunk_steps[c];
      Layout cur_sl = slice_at<EXACT>(p);
      Rec<W> cur;
      load_rec<EXACT, W>(cur, cur_sl, bslot, lane);
      for (int s = 0; s < steps; ++s) {
        // prefetch next step's record (stream data is immutable in this chunk)
        Layout nxt_sl;
        Rec<W> nxt;
        const bool more = s + 1 < steps;
        if (more) {
          nxt_sl = slice_at<EXACT>(p + cur_sl.bytes);
          load_rec<EXACT, W>(nxt, nxt_sl, bslot + (s + 1) * 32, lane);
        }
        if (cur.row >= 0) {
          double acc = EXACT ? 0.0 : __dmul_rn(cur.b, cur.rdg);
          bool ok = true;
          if constexpr (W > 0) {
#pragma unroll
            for (int d = 0; d < W; ++d) {
              const int code = cur.code[d];
              if (code == kSrcSkip) break;
              double xj;
              if (code >= 0) xj = ring[code];
              else if (code == kSrcPrev) xj = xprev;
              else ok = ok && wait.mailbox(a.mbox + (-2 - code), xj);
              acc = fold<EXACT>(acc, cur.val[d], xj);
            }
          } else {
            for (int d = 0; d < cur_sl.width; ++d) {
              const int code = cur_sl.src[d * 32 + lane];
              if (code == kSrcSkip) break;
              const double v = cur_sl.val[d * 32 + lane];
              double xj;
              if (code >= 0) xj = ring[code];
              else if (code == kSrcPrev) xj = xprev;
              else ok = ok && wait.mailbox(a.mbox + (-2 - code), xj);
              acc = fold<EXACT>(acc, v, xj);
            }
          }
          if (!ok) alive = false;
          double xi = EXACT ? div_exact(__dsub_rn(cur.b, acc), cur.dg, cur.rdg) : acc;
          const unsigned long long bits = publishable(xi);
          xi = as_f64(bits);
          ring[lane * kRingSteps + (step % kRingSteps)] = xi;
          xprev = xi;
          a.x[cur.row] = xi;
          if (cur.mbo >= 0) st_relaxed_u64(a.mbox + cur.mbo, bits);
        }
        __syncwarp();
        ++step;
        if (more) {
          p += cur_sl.bytes;
          cur_sl = nxt_sl;
          cur = nxt;
        }
      }
      if (!__all_sync(0xffffffffu, alive)) {
        alive = false;
        break;
      }
      // buffer of chunk c is free: stream chunk c + kChunkBuffers into it,
      // and gather b for chunk c + 2 (its stream landed long ago)
      __syncwarp();
      if (c + kChunkBuffers < c1) issue(c + kChunkBuffers);
      if (c + 2 < c1) {
        await(c + 2);
        gather_b<EXACT>(buf_of(c + 2), a.chunk_steps[c + 2], barea_of(c + 2), a.b, lane);
      }
    }
    if (!alive) {
      // drain the bulk copies still in flight into this CTA's shared memory
      for (int c = awaited_hi + 1; c <= issued_hi; ++c) await(c);
      break;
    }
  }
  cp_async_wait<0>();
  unsigned long long sp = wait.spins;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, off);
  if (lane == 0 && sp) atomicAdd(&a.status->spins, sp);
}

template <bool EXACT, int W>
cudaError_t launch_variant(const ChainArgs& a, int blocks, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_chains<EXACT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemTotal);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  k_chains<EXACT, W><<<blocks, 32, kSmemTotal, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

int DevicePlan::solve_chains(const double* d_b, double* d_x, cudaStream_t s) {
  if (!chains.ready) return plan_fail(SPTRSV_E_UNSUPPORTED, "chains schedule not built");
  cudaError_t e;
  if ((e = cudaMemsetAsync(chains.mbox, 0xFF, sizeof(unsigned long long) * (size_t)std::max(chains.n_mbox, 1ll), s)) !=
          cudaSuccess ||
      (e = cudaMemsetAsync(chains.ticket, 0, sizeof(int), s)) != cudaSuccess ||
      (e = cudaMemsetAsync(status, 0, sizeof(DeviceStatus), s)) != cudaSuccess ||
      (e = cudaMemsetAsync(abort_flag, 0, sizeof(int), s)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  ChainArgs a{};
  a.stream = chains.stream;
  a.chunk_off = chains.chunk_off;
  a.chunk_steps = chains.chunk_steps;
  a.task_chunk = chains.task_chunk;
  a.n_tasks = chains.n_tasks;
  a.mbox = chains.mbox;
  a.ticket = chains.ticket;
  a.b = d_b;
  a.x = d_x;
  a.status = status;
  a.abort_flag = abort_flag;
  a.timeout_ns = (unsigned long long)(opt.timeout_s * 1e9);
  a.spin_initial = opt.spin_initial;
  a.spin_max_ns = opt.spin_max_ns;
  // one warp per CTA; at most 2 CTAs per SM fit the shared-memory budget
  const int blocks = std::max(1, std::min(chains.n_tasks, num_sms * 2));
  const int w = chains.max_width;
  if ((e = cudaEventRecord(evk0, s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if (chains.exact) {
    e = w <= 4 ? launch_variant<true, 4>(a, blocks, s)
               : (w <= 8 ? launch_variant<true, 8>(a, blocks, s) : launch_variant<true, 0>(a, blocks, s));
  } else {
    e = w <= 4 ? launch_variant<false, 4>(a, blocks, s)
               : (w <= 8 ? launch_variant<false, 8>(a, blocks, s) : launch_variant<false, 0>(a, blocks, s));
  }
  if (e != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if ((e = cudaEventRecord(evk1, s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  launches = 1;
  return SPTRSV_OK;
}

}  // namespace sptrsv
