// Lane-chain lockstep executor ("chains").
//
// Why: on B200 a value handed between SMs through L2 costs ~800 cycles one
// way (tools/microbench/latency.cu: volatile ping-pong 1556 cycles round
// trip), a warp-synchronous hand-off through shared memory ~35 cycles. The
// sync-free component pool (solve_rows.cu) pays the L2 price on every level;
// a 2D Laplacian in natural order has 8191 of them.
//
// How: the host scheduler (schedule.cu) cuts the rows into contiguous tasks
// of <= 32 dependency chains, gives each chain a lane and each row a lockstep
// step. One warp runs one task: at every step each lane solves its row,
// reading same-task values (its chain predecessor included) from a
// shared-memory ring written in earlier steps, and values of earlier tasks
// from value-is-flag mailboxes in global memory. Tasks are dealt to
// persistent warps by an ascending ticket counter.
//
// The step is one warp's critical path, so it is kept short and branch-free:
// every dependency is one shared-memory load at a byte offset the scheduler
// baked into the stream (ring slot or inbox slot); the slice addresses follow
// from the chunk's uniform width; b and cross-task mailbox values are fetched
// kPrefetch steps ahead with cp.async (LDGSTS; mailboxes L2-only .cg) into
// shared memory; a prefetched mailbox that still held "not ready" (and the
// rare direct dependency) goes through an out-of-line polling slow path. The
// schedule stream is read exactly once: lane 0 keeps kChunkBuffers chunks in
// flight with cp.async.bulk (TMA bulk copies completing on mbarriers).
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
  long long* dbg;  // probe timestamps (PROBE instantiation only)
};

// Probe (tools/chains_probe.py): clock64 stamps of block 0 lane 0 for steps
// [kProbeFirstStep, kProbeFirstStep + kProbeSteps), 5 per step.
constexpr int kProbeClock = 16;
constexpr int kProbeFirstStep = 1000, kProbeSteps = 64;

namespace {

constexpr int kMboxStride = 2;  // u64 words per mailbox slot (16-byte slots for cp.async.cg)

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
// b is read-only: an L1-allocating 8-byte async copy.
__device__ __forceinline__ void cp_async8(unsigned dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
// Mailboxes are written during the kernel: copy them L2-only (.cg, 16 bytes).
__device__ __forceinline__ void cp_async16_cg(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ double lds_f64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// Slow path, out of line: poll a mailbox until it is solved. Returns its bits,
// or kNotReady when the launch aborts (watchdog or another warp's abort).
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

// One lane's slice fields, loaded one step ahead into registers.
template <bool EXACT, int W>
struct Rec {
  int row, mbo, pf_row;
  int pf_mbox[kMaxInbox];
  double rdg, dg;
  int src[W];
  double val[W];

  __device__ __forceinline__ void load(const unsigned char* p, const SliceGeom& g, int w, int lane, int M) {
    row = reinterpret_cast<const int*>(p)[lane];
    mbo = reinterpret_cast<const int*>(p + 128)[lane];
    pf_row = reinterpret_cast<const int*>(p + 256)[lane];
#pragma unroll
    for (int m = 0; m < kMaxInbox; ++m) pf_mbox[m] = m < M ? reinterpret_cast<const int*>(p + g.pfm)[m * 32 + lane] : -1;
    rdg = reinterpret_cast<const double*>(p + g.rdg)[lane];
    if (EXACT) dg = reinterpret_cast<const double*>(p + g.dg)[lane];
#pragma unroll
    for (int d = 0; d < W; ++d) {
      src[d] = d < w ? reinterpret_cast<const int*>(p + g.src)[d * 32 + lane] : kSrcSkip;
      val[d] = d < w ? reinterpret_cast<const double*>(p + g.val)[d * 32 + lane] : 0.0;
    }
  }
};

template <bool EXACT>
__device__ __forceinline__ double fold(double acc, double v, double xj) {
  if (EXACT) return __dadd_rn(acc, __dmul_rn(v, xj));
  return __fma_rn(v, xj, acc);
}

template <bool EXACT, int W, bool PROBE>
__global__ void __launch_bounds__(32, 1) k_chains(ChainArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  const unsigned sbase = smem_u32(smem);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + kSmemBars);
  const int* mslot = reinterpret_cast<const int*>(smem + kSmemSlot);
  const int lane = threadIdx.x;
  const int M = a.n_inbox;
  if (lane == 0) {
    for (int k = 0; k < kChunkBuffers; ++k) mbar_init(&bars[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned phase_bits = 0;  // parity to wait for, per buffer
  const unsigned long long deadline = a.timeout_ns ? globaltimer_ns() + a.timeout_ns : 0;
  bool alive = true;
  auto poll = [&](int slot) {
    const unsigned long long u =
        poll_mailbox(a.mbox + kMboxStride * slot, a.abort_flag, a.status, a.spin_initial, a.spin_max_ns, deadline);
    if (u == kNotReady) alive = false;
    return as_f64(u);
  };

  while (alive) {
    int t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= a.n_tasks) break;
    const int c0 = a.task_chunk[t], c1 = a.task_chunk[t + 1];
    int issued_hi = c0 - 1, awaited_hi = c0 - 1;
    auto buf_of = [&](int c) { return smem + kSmemChunks + (size_t)((c - c0) % kChunkBuffers) * kChunkBytes; };
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

    int step = 0;
    Rec<EXACT, W> cur, nxt;
    int w_next = a.chunk_width[c0], steps_next = a.chunk_steps[c0];
    for (int c = c0; c < c1 && alive; ++c) {
      const int w = w_next, steps = steps_next;
      if (c + 1 < c1) {  // scalars of the next chunk, consumed a chunk later
        w_next = a.chunk_width[c + 1];
        steps_next = a.chunk_steps[c + 1];
      }
      const SliceGeom g(w, M, EXACT);
      await(c);
      const unsigned char* p = buf_of(c);
      cur.load(p, g, w, lane, M);
      for (int s = 0; s < steps; ++s, ++step) {
        long long* stamp = nullptr;
        if constexpr (PROBE) {
          if (blockIdx.x == 0 && lane == 0 && step >= kProbeFirstStep && step < kProbeFirstStep + kProbeSteps)
            stamp = a.dbg + 5 * (step - kProbeFirstStep);
          if (stamp) stamp[0] = clock64();
        }
        const int pslot = step % kPrefetch;
        // the b / inbox copies for this step were issued kPrefetch steps ago
        cp_async_wait<kPrefetch - 1>();
        // dependency values: one shared-memory load each, at baked offsets
        double xv[W];
#pragma unroll
        for (int d = 0; d < W; ++d) xv[d] = lds_f64(sbase + (unsigned)max(cur.src[d], 0));
        const double bi = lds_f64(sbase + kSmemB + (pslot * 32 + lane) * 8);
        // next step's record (fixed offsets; past the chunk's end it reads
        // padding that is never used)
        nxt.load(p + (s + 1) * g.sb, g, w, lane, M);
        if constexpr (PROBE) {
          if (stamp) stamp[1] = clock64();
        }
        unsigned slow = 0;
#pragma unroll
        for (int d = 0; d < W; ++d) {
          const int sc = cur.src[d];
          const bool direct = sc <= kSrcDirect;
          const bool not_ready = sc >= 0 && (unsigned long long)__double_as_longlong(xv[d]) == kNotReady;
          slow |= (direct || not_ready) ? (1u << d) : 0u;
        }
        if (__any_sync(0xffffffffu, slow != 0)) {
#pragma unroll
          for (int d = 0; d < W; ++d) {
            if (slow & (1u << d)) {
              const int sc = cur.src[d];
              const int slot = sc <= kSrcDirect ? kSrcDirect - sc : mslot[(sc - kSmemInbox) / 16];
              xv[d] = poll(slot);
            }
          }
        }
        double acc = EXACT ? 0.0 : __dmul_rn(bi, cur.rdg);
#pragma unroll
        for (int d = 0; d < W; ++d) {
          const double folded = fold<EXACT>(acc, cur.val[d], xv[d]);
          acc = (cur.src[d] >= 0 || cur.src[d] <= kSrcDirect) ? folded : acc;
        }
        if constexpr (W == kInlineDeps) {
          // a row wider than kInlineDeps continues in the overflow list
          if (cur.src[W - 1] == kSrcOverflow) {
            const long long packed = __double_as_longlong(cur.val[W - 1]);
            const long long start = packed >> 24, cnt = packed & 0xFFFFFF;
            for (long long o = start; o < start + cnt; ++o) {
              const int oc = __ldg(a.ovf_src + o);
              const double ov = __ldg(a.ovf_val + o);
              double oj = oc >= 0 ? lds_f64(sbase + (unsigned)oc) : poll(kSrcDirect - oc);
              acc = fold<EXACT>(acc, ov, oj);
            }
          }
        }
        if constexpr (PROBE) {
          if (stamp) stamp[2] = clock64();
        }
        if (cur.row >= 0) {
          double xi = EXACT ? div_exact(__dsub_rn(bi, acc), cur.dg, cur.rdg) : acc;
          const unsigned long long bits = publishable(xi);
          xi = as_f64(bits);
          *reinterpret_cast<double*>(smem + ring_offset(step, lane)) = xi;
          a.x[cur.row] = xi;
          if (cur.mbo >= 0) st_relaxed_u64(a.mbox + kMboxStride * cur.mbo, bits);
        }
        // copies for step + kPrefetch into the slots just consumed
        if (cur.pf_row >= 0) {
          cp_async8(sbase + kSmemB + (pslot * 32 + lane) * 8, a.b + cur.pf_row);
#pragma unroll
          for (int m = 0; m < kMaxInbox; ++m) {
            const int slot = cur.pf_mbox[m];
            if (slot >= 0) {
              const int idx = inbox_index(m, step, lane);
              cp_async16_cg(sbase + kSmemInbox + idx * 16, a.mbox + kMboxStride * slot);
              reinterpret_cast<int*>(smem + kSmemSlot)[idx] = slot;
            }
          }
        }
        cp_async_commit();
        if constexpr (PROBE) {
          if (stamp) stamp[3] = clock64();
        }
        __syncwarp();
        if constexpr (PROBE) {
          if (stamp) stamp[4] = clock64();
        }
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

template <bool EXACT, int W, bool PROBE>
cudaError_t launch_variant(const ChainArgs& a, int blocks, cudaStream_t s) {
  static std::atomic<unsigned long long> attr{0};
  if (cudaError_t e = set_max_dyn_smem(k_chains<EXACT, W, PROBE>, kSmemTotal, attr); e != cudaSuccess) return e;
  k_chains<EXACT, W, PROBE><<<blocks, 32, kSmemTotal, s>>>(a);
  return cudaGetLastError();
}

template <bool EXACT, bool PROBE>
cudaError_t launch_width(int w, const ChainArgs& a, int blocks, cudaStream_t s) {
  if (w <= 1) return launch_variant<EXACT, 1, PROBE>(a, blocks, s);
  if (w <= 2) return launch_variant<EXACT, 2, PROBE>(a, blocks, s);
  if (w <= 3) return launch_variant<EXACT, 3, PROBE>(a, blocks, s);
  if (w <= 4) return launch_variant<EXACT, 4, PROBE>(a, blocks, s);
  if (w <= 8) return launch_variant<EXACT, 8, PROBE>(a, blocks, s);
  return launch_variant<EXACT, kInlineDeps, PROBE>(a, blocks, s);
}

}  // namespace

int DevicePlan::solve_chains(const double* d_b, double* d_x, cudaStream_t s) {
  if (!chains.ready) return plan_fail(SPTRSV_E_UNSUPPORTED, "chains schedule not built");
  cudaError_t e;
  if ((e = cudaMemsetAsync(chains.mbox, 0xFF, 16 * (size_t)std::max(chains.n_mbox, 1ll), s)) != cudaSuccess ||
      (e = reset_control(s)) != cudaSuccess)
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
  a.ticket = ticket;
  a.b = d_b;
  a.x = d_x;
  a.status = status;
  a.abort_flag = abort_flag;
  a.timeout_ns = (unsigned long long)(opt.timeout_s * 1e9);
  a.spin_initial = opt.spin_initial;
  a.spin_max_ns = opt.spin_max_ns;
  const bool probe = (opt.probe_flags & kProbeClock) != 0;
  if (probe) {
    static_assert(6 * kProbeSteps <= kProbeWords, "probe buffer");
    if (!probe_buf && cudaMalloc((void**)&probe_buf, sizeof(long long) * kProbeWords) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, "probe buffer");
    cudaMemsetAsync(probe_buf, 0, sizeof(long long) * 5 * kProbeSteps, s);
    a.dbg = probe_buf;
  }
  // one warp per CTA, at most 2 CTAs per SM (shared-memory budget)
  const int blocks = std::max(1, std::min(chains.n_tasks, num_sms * 2));
  if ((e = record_k0(s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  const int w = chains.max_width;
  if (chains.exact) e = probe ? launch_width<true, true>(w, a, blocks, s) : launch_width<true, false>(w, a, blocks, s);
  else e = probe ? launch_width<false, true>(w, a, blocks, s) : launch_width<false, false>(w, a, blocks, s);
  if (e != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if ((e = cudaEventRecord(evk1, s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  launches = 1;
  return SPTRSV_OK;
}

}  // namespace sptrsv
