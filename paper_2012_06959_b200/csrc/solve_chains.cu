// Lane-chain lockstep executor ("chains").
//
// Why: on B200 a value handed between SMs through L2 costs ~800 cycles one
// way (tools/microbench/latency.cu: volatile ping-pong 1556 cycles round
// trip), a warp-synchronous hand-off through shared memory ~35 cycles, a
// register nothing. The sync-free component pool (solve_rows.cu) pays the L2
// price on every level; a 2D Laplacian in natural order has 8191 of them.
//
// How: the host scheduler (schedule.cu) cuts the rows into contiguous tasks
// of <= 32 dependency chains, gives each chain a lane and each row a lockstep
// step. One warp runs one task: at every step each lane solves its row,
// reading the chain predecessor from a register, same-task values from a
// shared-memory ring written in earlier steps, and values of earlier tasks
// from value-is-flag mailboxes in global memory. Tasks are dealt to
// persistent warps by an ascending ticket counter.
//
// Latency hiding: every slice also names the row each lane will solve
// kPrefetch steps later and that row's cross-task mailbox slots; the lane
// issues cp.async (LDGSTS) copies of b and of those mailboxes into shared
// memory right away, so by the time the row is solved its inputs sit in
// shared memory. A copied mailbox that still held "not ready" is re-polled
// from global memory (the slow path). The schedule stream itself is read
// exactly once: lane 0 keeps kChunkBuffers chunks in flight with
// cp.async.bulk (TMA bulk copies completing on mbarriers), and the next
// step's record is loaded into registers while the current step computes.
#include "plan.hpp"
#include "kernels.cuh"

namespace sptrsv {

int plan_fail(int code, const char* msg);

struct ChainArgs {
  const unsigned char* stream;
  const long long* chunk_off;
  const int* chunk_steps;
  const int* chunk_width;
  const int* task_chunk;
  int n_tasks;
  int n_inbox;
  unsigned long long* mbox;
  const int* ovf_src;
  const double* ovf_val;
  int* ticket;
  const double* b;
  double* x;
  DeviceStatus* status;
  int* abort_flag;
  unsigned long long timeout_ns;
  int spin_initial;
  int spin_max_ns;
  int flags;            // probe variants (kProbe*), 0 in production
  long long* dbg;       // probe timestamps, nullptr unless kProbeClock
};

// Probe variants (tools/chains_probe.py): switch parts of the step off to
// attribute its cost, and record clock64 stamps of one warp's steps.
constexpr int kProbeNoB = 1, kProbeNoStoreX = 2, kProbeNoWait = 4, kProbeClock = 16;
constexpr int kProbeFirstStep = 1000, kProbeSteps = 64;

namespace {

constexpr int kSmemChunks = kChunkBuffers * kChunkBytes;
constexpr int kSmemRing = 32 * kRingSteps * 8;
constexpr int kSmemB = kPrefetch * 32 * 8;
constexpr int kSmemInbox = kMaxInbox * kPrefetch * 32 * 16;  // 16-byte slots (cp.async.cg granularity)
constexpr int kSmemSlot = kMaxInbox * kPrefetch * 32 * 4;
constexpr int kSmemTotal = kSmemChunks + kSmemRing + kSmemB + kSmemInbox + kSmemSlot + 64;

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
// b is read-only: an L1-allocating 8-byte async copy is fine.
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// Mailboxes are written during the kernel: copy them L2-only (.cg, 16 bytes),
// never from a stale L1 line. Mailbox slots are 16 bytes apart for this reason.
__device__ __forceinline__ void cp_async16_cg(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
constexpr int kMboxStride = 2;  // u64 words per mailbox slot
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Byte offsets inside a slice of a chunk whose uniform width is w: computed
// once per chunk, so loading the next step's record never waits on a load.
struct Geom {
  int sb, deps, vals, pf;
  __device__ __forceinline__ Geom(int w, int n_inbox, bool exact) {
    sb = slice_bytes(w, n_inbox, exact);
    deps = 528 + (exact ? 256 : 0);
    vals = deps + 128 * w;
    pf = deps + 384 * w;
  }
};

// One lane's view of one slice, loaded a step ahead into registers.
template <bool EXACT, int W>
struct Rec {
  int row, mbo, pf_row;
  int pf_mbox[kMaxInbox];
  double rdg, dg;
  int code[W];
  double val[W];

  __device__ __forceinline__ void load(const unsigned char* p, const Geom& g, int w, int lane, int n_inbox) {
    row = reinterpret_cast<const int*>(p + 16)[lane];
    mbo = reinterpret_cast<const int*>(p + 144)[lane];
    rdg = reinterpret_cast<const double*>(p + 272)[lane];
    if (EXACT) dg = reinterpret_cast<const double*>(p + 528)[lane];
    const int* src = reinterpret_cast<const int*>(p + g.deps);
    const double* vals = reinterpret_cast<const double*>(p + g.vals);
#pragma unroll
    for (int d = 0; d < W; ++d) {
      code[d] = d < w ? src[d * 32 + lane] : kSrcSkip;
      val[d] = d < w ? vals[d * 32 + lane] : 0.0;
    }
    const int* pf = reinterpret_cast<const int*>(p + g.pf);
    pf_row = pf[lane];
#pragma unroll
    for (int m = 0; m < kMaxInbox; ++m) pf_mbox[m] = m < n_inbox ? pf[32 + m * 32 + lane] : -1;
  }
};

// Slow path, kept out of line: poll a mailbox until it is solved. Returns its
// bits, or kNotReady when the launch is aborting (watchdog or another warp).
// Spins are added to the device status here, off the hot path.
__device__ __noinline__ unsigned long long poll_mailbox(const unsigned long long* p, int* abort_flag,
                                                        DeviceStatus* status, int spin_initial, int spin_max_ns,
                                                        unsigned long long deadline) {
  unsigned long long u = ld_relaxed_u64(p);
  int polls = 0, sleep_ns = 32;
  while (u == kNotReady) {
    ++polls;
    if (polls > spin_initial) {
      if ((polls & 63) == 0) {
        if (ld_relaxed_s32(abort_flag)) break;
        if (deadline && globaltimer_ns() > deadline) {
          atomicExch(&status->code, 5);
          atomicExch(abort_flag, 1);
          break;
        }
      }
      __nanosleep(sleep_ns);
      if (sleep_ns < spin_max_ns) sleep_ns <<= 1;
    }
    u = ld_relaxed_u64(p);
  }
  if (polls) atomicAdd(&status->spins, (unsigned long long)polls);
  return u;
}

template <bool EXACT>
__device__ __forceinline__ double fold(double acc, double v, double xj) {
  if (EXACT) return __dadd_rn(acc, __dmul_rn(v, xj));
  return __fma_rn(v, xj, acc);
}

template <bool EXACT, int W>
__global__ void __launch_bounds__(32, 1) k_chains(ChainArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* chunks = smem;
  double* ring = reinterpret_cast<double*>(smem + kSmemChunks);
  double* bring = reinterpret_cast<double*>(smem + kSmemChunks + kSmemRing);
  unsigned long long* mring = reinterpret_cast<unsigned long long*>(smem + kSmemChunks + kSmemRing + kSmemB);
  int* mslot = reinterpret_cast<int*>(smem + kSmemChunks + kSmemRing + kSmemB + kSmemInbox);
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(smem + kSmemChunks + kSmemRing + kSmemB + kSmemInbox + kSmemSlot);
  const int lane = threadIdx.x;
  const int M = a.n_inbox;
  if (lane == 0) {
    for (int k = 0; k < kChunkBuffers; ++k) mbar_init(&bars[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned phase_bits = 0;  // parity to wait for, per buffer
  const unsigned long long deadline = a.timeout_ns ? globaltimer_ns() + a.timeout_ns : 0;
  auto poll = [&](int slot, bool& ok) {
    const unsigned long long u =
        poll_mailbox(a.mbox + kMboxStride * slot, a.abort_flag, a.status, a.spin_initial, a.spin_max_ns, deadline);
    ok = ok && u != kNotReady;
    return as_f64(u);
  };
  bool alive = true;

  while (alive) {
    int t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= a.n_tasks) break;
    const int c0 = a.task_chunk[t], c1 = a.task_chunk[t + 1];
    int issued_hi = c0 - 1, awaited_hi = c0 - 1;
    auto buf_of = [&](int c) { return chunks + (size_t)((c - c0) % kChunkBuffers) * kChunkBytes; };
    auto issue = [&](int c) {
      issued_hi = c;
      if (lane == 0) {
        unsigned long long* bar = &bars[(c - c0) % kChunkBuffers];
        const unsigned bytes = (unsigned)(a.chunk_off[c + 1] - a.chunk_off[c]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar, bytes);
        bulk_g2s(buf_of(c), a.stream + a.chunk_off[c], bytes, bar);
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

    double xprev = 0.0;
    int step = 0;
    Rec<EXACT, W> cur, nxt;
    int w_next = a.chunk_width[c0], steps_next = a.chunk_steps[c0];
    for (int c = c0; c < c1 && alive; ++c) {
      const int w = w_next, steps = steps_next;
      if (c + 1 < c1) {  // scalars of the next chunk, consumed a chunk later
        w_next = a.chunk_width[c + 1];
        steps_next = a.chunk_steps[c + 1];
      }
      const Geom g(w, M, EXACT);
      await(c);
      const unsigned char* p = buf_of(c);
      cur.load(p, g, w, lane, M);
      for (int s = 0; s < steps; ++s, ++step) {
        // next record: fixed offsets, issued before this step's dependencies
        // (past the chunk's last slice it reads padding that is never used)
        nxt.load(p + (s + 1) * g.sb, g, w, lane, M);
        const bool probe = a.dbg && blockIdx.x == 0 && lane == 0 && step >= kProbeFirstStep &&
                           step < kProbeFirstStep + kProbeSteps;
        long long* stamp = probe ? a.dbg + 5 * (step - kProbeFirstStep) : nullptr;
        if (probe) stamp[0] = clock64();
        const int pslot = step % kPrefetch;
        // the copies for this step were issued kPrefetch steps ago
        if (!(a.flags & kProbeNoWait)) cp_async_wait<kPrefetch - 1>();
        if (probe) stamp[1] = clock64();
        // gather every dependency value branch-free (ring / register / inbox),
        // flag the rare ones that must be polled from global memory
        double xj[W];
        unsigned slow = 0;
#pragma unroll
        for (int d = 0; d < W; ++d) {
          const int code = cur.code[d];
          const double rv = ring[code >= 0 ? code : 0];
          const int m = kSrcInbox0 - code;
          const bool inbox = m >= 0 && m < kMaxInbox;
          const unsigned long long iu = mring[(((inbox ? m : 0) * kPrefetch + pslot) * 32 + lane) * 2];
          xj[d] = code >= 0 ? rv : (code == kSrcPrev ? xprev : as_f64(iu));
          if ((inbox && iu == kNotReady) || (code <= kSrcDirect && code != kSrcSkip)) slow |= 1u << d;
        }
        if (__any_sync(0xffffffffu, slow != 0)) {
#pragma unroll
          for (int d = 0; d < W; ++d) {
            if (slow & (1u << d)) {
              const int code = cur.code[d];
              const int m = kSrcInbox0 - code;
              const int slot = code <= kSrcDirect ? kSrcDirect - code : mslot[(m * kPrefetch + pslot) * 32 + lane];
              xj[d] = poll(slot, alive);
            }
          }
        }
        const double bi = (a.flags & kProbeNoB) ? 1.0 : bring[pslot * 32 + lane];
        double acc = EXACT ? 0.0 : __dmul_rn(bi, cur.rdg);
#pragma unroll
        for (int d = 0; d < W; ++d) {
          const double folded = fold<EXACT>(acc, cur.val[d], xj[d]);
          acc = (cur.code[d] != kSrcSkip && cur.code[d] != kSrcOverflow) ? folded : acc;
        }
        if constexpr (W == kInlineDeps) {
          // a row wider than kInlineDeps continues in the overflow list
          if (cur.code[W - 1] == kSrcOverflow) {
            const long long packed = __double_as_longlong(cur.val[W - 1]);
            const long long start = packed >> 24, cnt = packed & 0xFFFFFF;
            for (long long o = start; o < start + cnt; ++o) {
              const int oc = __ldg(a.ovf_src + o);
              const double ov = __ldg(a.ovf_val + o);
              double oj;
              if (oc >= 0) oj = ring[oc];
              else if (oc == kSrcPrev) oj = xprev;
              else oj = poll(kSrcDirect - oc, alive);
              acc = fold<EXACT>(acc, ov, oj);
            }
          }
        }
        if (probe) stamp[2] = clock64();
        if (cur.row >= 0) {
          double xi = EXACT ? div_exact(__dsub_rn(bi, acc), cur.dg, cur.rdg) : acc;
          const unsigned long long bits = publishable(xi);
          xi = as_f64(bits);
          ring[(step % kRingSteps) * 32 + lane] = xi;
          xprev = xi;
          if (!(a.flags & kProbeNoStoreX)) a.x[cur.row] = xi;
          if (cur.mbo >= 0) st_relaxed_u64(a.mbox + kMboxStride * cur.mbo, bits);
        }
        // launch the copies for step + kPrefetch into the slots just consumed
        if (cur.pf_row >= 0) {
          if (!(a.flags & kProbeNoB)) cp_async8(bring + pslot * 32 + lane, a.b + cur.pf_row);
#pragma unroll
          for (int m = 0; m < kMaxInbox; ++m) {
            const int slot = cur.pf_mbox[m];
            if (slot >= 0) {
              cp_async16_cg(mring + ((m * kPrefetch + pslot) * 32 + lane) * 2, a.mbox + kMboxStride * slot);
              mslot[(m * kPrefetch + pslot) * 32 + lane] = slot;
            }
          }
        }
        cp_async_commit();
        if (probe) stamp[3] = clock64();
        __syncwarp();
        if (probe) stamp[4] = clock64();
        cur = nxt;
      }
      if (!__all_sync(0xffffffffu, alive)) alive = false;
      __syncwarp();
      if (alive && c + kChunkBuffers < c1) issue(c + kChunkBuffers);
    }
    cp_async_wait<0>();
    if (!alive) {
      // drain the bulk copies still in flight into this CTA's shared memory
      for (int c = awaited_hi + 1; c <= issued_hi; ++c) await(c);
      break;
    }
  }
  cp_async_wait<0>();
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

template <bool EXACT>
cudaError_t launch_width(int w, const ChainArgs& a, int blocks, cudaStream_t s) {
  if (w <= 4) return launch_variant<EXACT, 4>(a, blocks, s);
  if (w <= 8) return launch_variant<EXACT, 8>(a, blocks, s);
  return launch_variant<EXACT, kInlineDeps>(a, blocks, s);
}

}  // namespace

int DevicePlan::solve_chains(const double* d_b, double* d_x, cudaStream_t s) {
  if (!chains.ready) return plan_fail(SPTRSV_E_UNSUPPORTED, "chains schedule not built");
  cudaError_t e;
  if ((e = cudaMemsetAsync(chains.mbox, 0xFF, 16 * (size_t)std::max(chains.n_mbox, 1ll), s)) !=
          cudaSuccess ||
      (e = cudaMemsetAsync(chains.ticket, 0, sizeof(int), s)) != cudaSuccess ||
      (e = cudaMemsetAsync(status, 0, sizeof(DeviceStatus), s)) != cudaSuccess ||
      (e = cudaMemsetAsync(abort_flag, 0, sizeof(int), s)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  ChainArgs a{};
  a.stream = chains.stream;
  a.chunk_off = chains.chunk_off;
  a.chunk_steps = chains.chunk_steps;
  a.chunk_width = chains.chunk_width;
  a.task_chunk = chains.task_chunk;
  a.n_tasks = chains.n_tasks;
  a.n_inbox = chains.n_inbox;
  a.mbox = chains.mbox;
  a.ovf_src = chains.ovf_src;
  a.ovf_val = chains.ovf_val;
  a.ticket = chains.ticket;
  a.b = d_b;
  a.x = d_x;
  a.status = status;
  a.abort_flag = abort_flag;
  a.timeout_ns = (unsigned long long)(opt.timeout_s * 1e9);
  a.spin_initial = opt.spin_initial;
  a.spin_max_ns = opt.spin_max_ns;
  a.flags = opt.probe_flags;
  if (opt.probe_flags & kProbeClock) {
    if (!probe_buf && cudaMalloc((void**)&probe_buf, sizeof(long long) * 5 * kProbeSteps) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, "probe buffer");
    cudaMemsetAsync(probe_buf, 0, sizeof(long long) * 5 * kProbeSteps, s);
    a.dbg = probe_buf;
  }
  // one warp per CTA, at most 2 CTAs per SM (shared-memory budget)
  const int blocks = std::max(1, std::min(chains.n_tasks, num_sms * 2));
  if ((e = cudaEventRecord(evk0, s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  e = chains.exact ? launch_width<true>(chains.max_width, a, blocks, s)
                   : launch_width<false>(chains.max_width, a, blocks, s);
  if (e != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if ((e = cudaEventRecord(evk1, s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  launches = 1;
  return SPTRSV_OK;
}

}  // namespace sptrsv
