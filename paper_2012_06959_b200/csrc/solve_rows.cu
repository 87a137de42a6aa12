// Sync-free component pool: the paper's warp-per-component solve (Alg. 3,
// /root/reference/PAPER.md:339-399) restated for B200 as a pull kernel.
//
// * A persistent grid; each warp takes tickets of 32 consecutive slots of a
//   topological order (`order`) from one atomic counter — the "malleable task
//   pool". Tickets are handed out in ascending order, so the
//   earliest unsolved component always belongs to a running warp: the
//   reference's progress argument (engine.py:30-35) carries over.
// * Thread-per-component for short rows: each lane gathers its row's x_j with
//   relaxed 8-byte loads; a slot still equal to kNotReady means "not solved
//   yet" and is re-polled (lock-wait, engine.py:497-521). Loads are issued four
//   at a time so independent dependencies overlap.
// * Rows with many dependencies are solved by the whole warp when tickets are
//   single-level (coop_long): lanes poll disjoint chunks, and the partial sums
//   are folded in ascending column order (exact mode) or by a shuffle tree (fast).
// * Exact mode reproduces solve_serial bit for bit: left_sum accumulates
//   v*x_j in ascending column order with separate IEEE mul/add, then
//   x_i = (b_i - left_sum) / l_ii (reference.py:30-34).
// * Level mode runs the same dataflow over (max, +1): level_i = 1 + max level_j,
//   which is the reference's canonical earliest level (analysis.py:43-64).
#include "common.cuh"
#include "kernels.cuh"

#include <cstdlib>

#ifndef SPTRSV_LONG_UNROLL
#define SPTRSV_LONG_UNROLL 4
#endif

namespace sptrsv {

namespace {

struct Poller {
  const RowsArgs& a;
  unsigned long long spins = 0;
  unsigned long long remote = 0;
  unsigned long long deadline = 0;
  __device__ explicit Poller(const RowsArgs& args) : a(args) {
    if (a.timeout_ns) deadline = globaltimer_ns() + a.timeout_ns;
  }

  // Wait for one slot; returns false when the launch is being aborted.
  __device__ __forceinline__ bool wait_u64(const unsigned long long* p, bool sys, unsigned long long& u) {
    int polls = 0;
    int sleep_ns = 32;
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
      u = sys ? ld_relaxed_sys_u64(p) : ld_relaxed_u64(p);
    }
    return true;
  }
  __device__ __forceinline__ bool wait_s32(const int* p, int& v) {
    int polls = 0;
    int sleep_ns = 32;
    while (v < 0) {
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
      v = ld_relaxed_s32(p);
    }
    return true;
  }
};

template <int MODE>
struct Acc;

template <>
struct Acc<kModeExact> {
  double s = 0.0;
  __device__ void init(const RowsArgs&, int) { s = 0.0; }
  __device__ void add(double v, double xj) { s = __dadd_rn(s, __dmul_rn(v, xj)); }
  __device__ double finish(const RowsArgs& a, int i) const {
    return div_exact(__dsub_rn(a.b[i], s), a.dg[i], a.rdg[i]);
  }
};

template <>
struct Acc<kModeFast> {
  double s = 0.0;
  __device__ void init(const RowsArgs& a, int i) { s = __dmul_rn(a.b[i], a.rdg[i]); }
  __device__ void add(double w, double xj) { s = __fma_rn(w, xj, s); }
  __device__ double finish(const RowsArgs&, int) const { return s; }
};

template <int MODE>
__device__ __forceinline__ const unsigned long long* slot_u64(const RowsArgs& a, int j, bool& remote) {
  if (a.owner == nullptr) {
    remote = false;
    return a.xseg[0] + j;
  }
  int p = a.owner[j];
  remote = p != a.my_pe;
  return a.xseg[p] + j;
}

__device__ __forceinline__ const int* slot_s32(const RowsArgs& a, int j, bool& remote) {
  if (a.owner == nullptr) {
    remote = false;
    return a.lseg[0] + j;
  }
  int p = a.owner[j];
  remote = p != a.my_pe;
  return a.lseg[p] + j;
}

// SPTRSV_PLAN_DEBUG: the reference's debug assertions (engine.py:154-169,
// 510-513) restated for the pull protocol -- a slot is written only by the PE
// that owns the component, and only once, over its not-ready sentinel (a
// published value is final, the pull analogue of "counters never fall").
__device__ __noinline__ void debug_violation(const RowsArgs& a, int i) {
  if (atomicCAS(&a.status->code, 0, 10) == 0) a.status->detail = i;
  atomicExch(a.abort_flag, 1);
}

__device__ __forceinline__ void publish_u64(const RowsArgs& a, int i, double v) {
  unsigned long long* p = a.xseg[a.owner ? a.my_pe : 0] + i;
  if (a.debug && ((a.owner && a.owner[i] != a.my_pe) || ld_relaxed_u64(p) != kNotReady)) debug_violation(a, i);
  if (a.owner) st_relaxed_sys_u64(p, publishable(v));
  else st_relaxed_u64(p, publishable(v));
  // fault injection (probe bit 1024): row 0 published a second time -- its
  // check must find the slot already written
  if (a.debug == 2 && i == 0) {
    if (ld_relaxed_u64(p) != kNotReady) debug_violation(a, i);
    st_relaxed_u64(p, publishable(v));
  }
  if (a.stamps) a.stamps[i] = (long long)globaltimer_ns();
}

// dependencies per round of a thread's row: their column indices / values,
// then their x slots, all in flight before the first wait
#ifndef SPTRSV_ROW_GROUP
#define SPTRSV_ROW_GROUP 4
#endif
constexpr int kRowGroup = SPTRSV_ROW_GROUP;

// One lane, one row, floating point.
template <int MODE>
__device__ bool solve_row_thread(const RowsArgs& a, Poller& poll, int i) {
  Acc<MODE> acc;
  acc.init(a, i);
  int k = a.rp[i];
  const int end = a.rp[i + 1];
  const bool multi = a.owner != nullptr;
  for (; k < end; k += kRowGroup) {
    int j[kRowGroup];
    double v[kRowGroup];
    unsigned long long u[kRowGroup];
    const unsigned long long* p[kRowGroup];
    bool rem[kRowGroup];
#pragma unroll
    for (int q = 0; q < kRowGroup; ++q) {
      if (k + q < end) {
        j[q] = __ldg(a.ci + k + q);
        v[q] = __ldg(a.val + k + q);
      }
    }
#pragma unroll
    for (int q = 0; q < kRowGroup; ++q) {
      if (k + q < end) {
        p[q] = slot_u64<MODE>(a, j[q], rem[q]);
        u[q] = rem[q] ? ld_relaxed_sys_u64(p[q]) : ld_relaxed_u64(p[q]);
        if (multi && rem[q]) ++poll.remote;
      }
    }
#pragma unroll
    for (int q = 0; q < kRowGroup; ++q) {
      if (k + q < end) {
        if (!poll.wait_u64(p[q], rem[q], u[q])) return false;
        acc.add(v[q], as_f64(u[q]));
      }
    }
  }
  publish_u64(a, i, acc.finish(a, i));
  return true;
}

// The same rows, one per lane, but the warp polls them in lockstep rounds
// instead of each lane spinning inside its own row loop. With per-lane spin
// loops the lanes reconverge after every dependency group, so a row is only
// published once its 31 ticket-mates are solved too: every hop of the level
// chain then costs the slowest of ~250 dependencies plus one L2 round trip per
// group of each row. Here, per round, every unfinished lane reloads the
// not-yet-consumed part of its current window of kWin dependencies (all loads in
// flight together), folds the ready prefix in column order (so x is bitwise
// the same as the per-lane loop) and publishes its row the round its last
// dependency arrives. The next window's indices and values are prefetched while
// the current one is polled.
template <int MODE>
__device__ bool solve_rows_lanes(const RowsArgs& a, Poller& poll, int i, bool active, int lane) {
#ifndef SPTRSV_ROWS_WIN
#define SPTRSV_ROWS_WIN 4
#endif
  constexpr int kWin = SPTRSV_ROWS_WIN;
  Acc<MODE> acc;
  int k = 0, end = 0, cnt = 0, c = 0;
  int j[kWin], jn[kWin];
  double v[kWin], vn[kWin];
  if (active) {
    acc.init(a, i);
    k = a.rp[i];
    end = a.rp[i + 1];
    cnt = min(kWin, end - k);
#pragma unroll
    for (int q = 0; q < kWin; ++q) {
      j[q] = q < cnt ? __ldg(a.ci + k + q) : 0;
      v[q] = q < cnt ? __ldg(a.val + k + q) : 0.0;
      const int kn = k + kWin + q;
      jn[q] = kn < end ? __ldg(a.ci + kn) : 0;
      vn[q] = kn < end ? __ldg(a.val + kn) : 0.0;
    }
    if (cnt == 0) {
      publish_u64(a, i, acc.finish(a, i));
      active = false;
    }
  }
  int rounds = 0;
  unsigned long long deadline = poll.deadline;
  while (__any_sync(0xffffffffu, active)) {
    bool progressed = false;
    if (active) {
      unsigned long long u[kWin];
      bool rem[kWin];
#pragma unroll
      for (int q = 0; q < kWin; ++q) {
        if (q >= c && q < cnt) {
          const unsigned long long* p = slot_u64<MODE>(a, j[q], rem[q]);
          u[q] = rem[q] ? ld_relaxed_sys_u64(p) : ld_relaxed_u64(p);
        }
      }
      bool prefix = true;
#pragma unroll
      for (int q = 0; q < kWin; ++q) {
        if (q >= c && q < cnt && prefix) {
          if (u[q] == kNotReady) {
            prefix = false;
          } else {
            acc.add(v[q], as_f64(u[q]));
            if (rem[q]) ++poll.remote;  // one remote read per dependency, as the per-lane loop counts
            ++c;
            progressed = true;
          }
        }
      }
      if (c == cnt) {
        k += kWin;
        if (k >= end) {
          publish_u64(a, i, acc.finish(a, i));
          active = false;
        } else {
          cnt = min(kWin, end - k);
          c = 0;
#pragma unroll
          for (int q = 0; q < kWin; ++q) {
            j[q] = jn[q];
            v[q] = vn[q];
            const int kn = k + kWin + q;
            jn[q] = kn < end ? __ldg(a.ci + kn) : 0;
            vn[q] = kn < end ? __ldg(a.val + kn) : 0.0;
          }
        }
      }
      if (!progressed) ++poll.spins;
    }
    if (++rounds > a.spin_initial) {
      if ((rounds & 63) == 0) {
        int stop = 0;
        if (lane == 0) {
          stop = ld_relaxed_s32(a.abort_flag);
          if (!stop && deadline && globaltimer_ns() > deadline) {
            atomicExch(&a.status->code, 5);
            atomicExch(a.abort_flag, 1);
            stop = 1;
          }
        }
        if (__shfl_sync(0xffffffffu, stop, 0)) return false;
      }
      if (!__any_sync(0xffffffffu, progressed)) __nanosleep(a.spin_max_ns);
    }
  }
  return true;
}

__device__ bool level_row_thread(const RowsArgs& a, Poller& poll, int i) {
  int lv = 0;
  const int end = a.rp[i + 1];
  for (int k = a.rp[i]; k < end; k += 4) {
    int vals[4];
    const int* p[4];
    bool rem[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (k + q < end) {
        p[q] = slot_s32(a, __ldg(a.ci + k + q), rem[q]);
        vals[q] = ld_relaxed_s32(p[q]);
      }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (k + q < end) {
        if (!poll.wait_s32(p[q], vals[q])) return false;
        lv = max(lv, vals[q] + 1);
      }
  }
  st_relaxed_s32(a.lseg[a.owner ? a.my_pe : 0] + i, lv);
  return true;
}

// Whole warp, one long row. Exact mode keeps the ascending-column fold by
// letting lane 0 add the 32 products of each chunk in order.
// Warp-wide dot product of entries [beg, end) with x (fast mode), all loads
// of a round in flight before any wait. Returns false when aborting.
__device__ bool warp_dot_fast(const RowsArgs& a, Poller& poll, int beg, int end, int lane, double& part) {
  constexpr int kU = SPTRSV_LONG_UNROLL;
  for (int base = beg; base < end; base += kWarp * kU) {
    int j[kU];
    double v[kU];
    unsigned long long u[kU];
    const unsigned long long* p[kU];
    bool rem[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const int k = base + q * kWarp + lane;
      j[q] = k < end ? __ldg(a.ci + k) : -1;
      v[q] = k < end ? __ldg(a.val + k) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      if (j[q] >= 0) {
        p[q] = slot_u64<kModeFast>(a, j[q], rem[q]);
        u[q] = rem[q] ? ld_relaxed_sys_u64(p[q]) : ld_relaxed_u64(p[q]);
        if (rem[q]) ++poll.remote;
      }
    }
    bool ok = true;
#pragma unroll
    for (int q = 0; q < kU; ++q)
      if (j[q] >= 0) {
        ok = ok && poll.wait_u64(p[q], rem[q], u[q]);
        part = __fma_rn(v[q], as_f64(u[q]), part);
      }
    if (__any_sync(0xffffffffu, !ok)) return false;
  }
  return true;
}

// Partial task p of a split row: its slice of the row's dot product, added to
// the row's shared partial sum; then the row's done-count is bumped.
__device__ bool solve_part_warp(const RowsArgs& a, Poller& poll, int p, int lane) {
  double part = 0.0;
  if (!warp_dot_fast(a, poll, a.part_beg[p], a.part_end[p], lane, part)) return false;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
  if (lane == 0) {
    const int h = a.part_heavy[p];
    atomicAdd(a.part_sum + h, part);
    __threadfence();  // the sum before the count
    atomicAdd(a.part_done + h, 1);
  }
  return true;
}

__device__ __forceinline__ int ld_acquire_gpu_s32_rows(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int MODE>
__device__ bool solve_row_warp(const RowsArgs& a, Poller& poll, int i, int lane) {
  const int beg = a.rp[i], end = a.rp[i + 1];
  double s = (MODE == kModeFast) ? __dmul_rn(a.b[i], a.rdg[i]) : 0.0;
  double part = 0.0;  // fast mode: per-lane partial
  if (MODE == kModeFast && a.heavy_idx) {
    const int h = a.heavy_idx[i];
    if (h >= 0) {
      // a split row: its partial tasks (earlier tickets of the same level)
      // hold the whole dot product
      int ok = 1;
      double sum = 0.0;
      if (lane == 0) {
        const int need = a.heavy_parts[h];
        int polls = 0, sleep_ns = 32;
        while (ld_acquire_gpu_s32_rows(a.part_done + h) < need) {
          ++poll.spins;
          if (++polls > a.spin_initial) {
            if ((polls & 63) == 0) {
              if (ld_relaxed_s32(a.abort_flag)) { ok = 0; break; }
              if (poll.deadline && globaltimer_ns() > poll.deadline) {
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
          sum = __ldcg(a.part_sum + h);
          publish_u64(a, i, s + sum);
        }
      }
      return __shfl_sync(0xffffffffu, ok, 0) != 0;
    }
  }
  int base = beg;
  if (MODE == kModeFast) {
    // Very long rows (power-law in-degrees: 29,079 in rmat-4M): kLongUnroll
    // dependencies per lane per round, all loads in flight before any wait,
    // so a round costs one memory round trip for 32 * kLongUnroll entries.
    constexpr int kLongUnroll = SPTRSV_LONG_UNROLL;
    for (; base + kWarp * kLongUnroll <= end; base += kWarp * kLongUnroll) {
      int j[kLongUnroll];
      double v[kLongUnroll];
      unsigned long long u[kLongUnroll];
      const unsigned long long* p[kLongUnroll];
      bool rem[kLongUnroll];
#pragma unroll
      for (int q = 0; q < kLongUnroll; ++q) {
        j[q] = __ldg(a.ci + base + q * kWarp + lane);
        v[q] = __ldg(a.val + base + q * kWarp + lane);
      }
#pragma unroll
      for (int q = 0; q < kLongUnroll; ++q) {
        p[q] = slot_u64<MODE>(a, j[q], rem[q]);
        u[q] = rem[q] ? ld_relaxed_sys_u64(p[q]) : ld_relaxed_u64(p[q]);
        if (rem[q]) ++poll.remote;
      }
      bool ok = true;
#pragma unroll
      for (int q = 0; q < kLongUnroll; ++q) {
        ok = ok && poll.wait_u64(p[q], rem[q], u[q]);
        part = __fma_rn(v[q], as_f64(u[q]), part);
      }
      if (__any_sync(0xffffffffu, !ok)) return false;
    }
  }
  if (MODE == kModeExact) {
    // Exact: kLongUnroll rounds of 32 entries in flight at once, their products
    // v * x_j parked in this warp's shared-memory slots in entry order, then
    // lane 0 adds them one after another (the serial oracle's ascending
    // column order: the sum is inherently sequential, but one DADD chain
    // from shared memory instead of a shuffle round trip per entry and a
    // memory round trip per 32 entries)
    constexpr int kLongUnroll = SPTRSV_LONG_UNROLL;
    __shared__ double s_prod[8][kWarp * SPTRSV_LONG_UNROLL];
    double* sp = s_prod[(threadIdx.x >> 5) & 7];
    for (; base < end; base += kWarp * kLongUnroll) {
      int j[kLongUnroll];
      double v[kLongUnroll];
      unsigned long long u[kLongUnroll];
      const unsigned long long* p[kLongUnroll];
      bool rem[kLongUnroll];
#pragma unroll
      for (int q = 0; q < kLongUnroll; ++q) {
        const int k = base + q * kWarp + lane;
        j[q] = k < end ? __ldg(a.ci + k) : -1;
        v[q] = k < end ? __ldg(a.val + k) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < kLongUnroll; ++q) {
        if (j[q] >= 0) {
          p[q] = slot_u64<MODE>(a, j[q], rem[q]);
          u[q] = rem[q] ? ld_relaxed_sys_u64(p[q]) : ld_relaxed_u64(p[q]);
          if (rem[q]) ++poll.remote;
        }
      }
      bool ok = true;
#pragma unroll
      for (int q = 0; q < kLongUnroll; ++q)
        if (j[q] >= 0) {
          ok = ok && poll.wait_u64(p[q], rem[q], u[q]);
          sp[q * kWarp + lane] = __dmul_rn(v[q], as_f64(u[q]));
        }
      if (__any_sync(0xffffffffu, !ok)) return false;
      __syncwarp();
      if (lane == 0) {
        const int cnt = min(kWarp * kLongUnroll, end - base);
        for (int q = 0; q < cnt; ++q) s = __dadd_rn(s, sp[q]);
      }
      __syncwarp();  // the slots are rewritten by the next round
    }
    s = __shfl_sync(0xffffffffu, s, 0);
  }
  for (; base < end; base += kWarp) {
    int k = base + lane;
    double prod = 0.0;
    bool ok = true;
    if (k < end) {
      int j = __ldg(a.ci + k);
      double v = __ldg(a.val + k);
      bool rem;
      const unsigned long long* p = slot_u64<MODE>(a, j, rem);
      unsigned long long u = rem ? ld_relaxed_sys_u64(p) : ld_relaxed_u64(p);
      if (rem) ++poll.remote;
      ok = poll.wait_u64(p, rem, u);
      if (MODE == kModeExact) prod = __dmul_rn(v, as_f64(u));
      else part = __fma_rn(v, as_f64(u), part);
    }
    if (__any_sync(0xffffffffu, !ok)) return false;
    if (MODE == kModeExact) {
      int cnt = min(kWarp, end - base);
      for (int q = 0; q < cnt; ++q) {
        double pq = __shfl_sync(0xffffffffu, prod, q);
        s = __dadd_rn(s, pq);
      }
    }
  }
  double xi;
  if (MODE == kModeExact) {
    xi = div_exact(__dsub_rn(a.b[i], s), a.dg[i], a.rdg[i]);
  } else {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    xi = s + part;
  }
  if (lane == 0) publish_u64(a, i, xi);
  return true;
}

__device__ bool level_row_warp(const RowsArgs& a, Poller& poll, int i, int lane) {
  const int beg = a.rp[i], end = a.rp[i + 1];
  int lv = 0;
  for (int k = beg + lane; k < end; k += kWarp) {
    bool rem;
    const int* p = slot_s32(a, __ldg(a.ci + k), rem);
    int v = ld_relaxed_s32(p);
    if (!poll.wait_s32(p, v)) { lv = -1 << 30; break; }
    lv = max(lv, v + 1);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) lv = max(lv, __shfl_xor_sync(0xffffffffu, lv, off));
  if (lv < 0) return false;
  if (lane == 0) st_relaxed_s32(a.lseg[a.owner ? a.my_pe : 0] + i, lv);
  return true;
}

// resident blocks per SM the register budget is sized for (SPTRSV_ROWS_MINB):
// two blocks (2,368 warps in the pool) with 4-entry windows and 4 rounds of
// long-row loads in flight measured best on rmat-4M (fast 3.33 -> 3.13 ms,
// exact 10.4 -> 9.9 ms); one block with 8 / 8: 3.33 ms; three blocks: 3.46 ms;
// four blocks (64 registers, spilling): 5.2 ms; fewer warps (SPTRSV_ROWS_GRID
// 111 / 74 / 37 blocks of one per SM): 3.64 / 4.37 / 6.91 ms
#ifndef SPTRSV_ROWS_MINB
#define SPTRSV_ROWS_MINB 2
#endif

template <int MODE>
__global__ void __launch_bounds__(256, SPTRSV_ROWS_MINB) k_rows(RowsArgs a_in) {
  const int lane = threadIdx.x & 31;
  // the PE this block works for: its slice of the order and its ticket pool
  RowsArgs a = a_in;
  const int n_local = a_in.n_pe_local > 0 ? a_in.n_pe_local : 1;
  const int pe_local = blockIdx.x % n_local;
  a.my_pe = a_in.pe_base + pe_local;
  a.ticket = a_in.ticket + pe_local;
  if (a_in.pe_order_off) {
    const long long lo = a_in.pe_order_off[pe_local], hi = a_in.pe_order_off[pe_local + 1];
    a.order = a_in.order + lo;
    a.order_len = hi - lo;
  }
  Poller poll(a);
  while (true) {
    int t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    long long slot = (long long)t * kWarp + lane;
    if ((long long)t * kWarp >= a.order_len) break;
    int i = -1;
    if (slot < a.order_len) i = a.order ? a.order[slot] : (int)slot;
    bool is_long = false;
    if (i >= a.n) is_long = true;  // a partial task of a split row (fast mode)
    else if (i >= 0 && a.coop_long) is_long = (a.rp[i + 1] - a.rp[i]) > a.long_deps;
    bool ok = true;
    if constexpr (MODE != kModeLevel) {
      if (a.lane_loop) ok = solve_rows_lanes<MODE>(a, poll, i, i >= 0 && !is_long, lane);
      else if (i >= 0 && !is_long) ok = solve_row_thread<MODE>(a, poll, i);
    } else if (i >= 0 && !is_long) {
      ok = level_row_thread(a, poll, i);
    }
    unsigned longs = __ballot_sync(0xffffffffu, is_long);
    while (longs && __all_sync(0xffffffffu, ok)) {
      int src = __ffs(longs) - 1;
      longs &= longs - 1;
      int r = __shfl_sync(0xffffffffu, i, src);
      bool wok;
      if constexpr (MODE == kModeLevel) wok = level_row_warp(a, poll, r, lane);
      else if (MODE == kModeFast && r >= a.n) wok = solve_part_warp(a, poll, r - a.n, lane);
      else wok = solve_row_warp<MODE>(a, poll, r, lane);
      ok = ok && wok;
    }
    if (!__all_sync(0xffffffffu, ok)) break;
  }
  // fold per-thread counters
  unsigned long long sp = poll.spins, rm = poll.remote;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    sp += __shfl_xor_sync(0xffffffffu, sp, off);
    rm += __shfl_xor_sync(0xffffffffu, rm, off);
  }
  if (lane == 0 && (sp | rm)) {
    atomicAdd(&a.status->spins, sp);
    atomicAdd(&a.status->remote_reads, rm);
  }
}

}  // namespace

int rows_lane_loop() {
  static const int on = [] {
    const char* e = std::getenv("SPTRSV_ROWS_LANELOOP");
    return e ? std::atoi(e) : 1;
  }();
  return on;
}

int rows_blocks_per_sm(int mode) {
  int nb = 0;
  if (mode == kModeExact) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_rows<kModeExact>, 256, 0);
  else if (mode == kModeFast) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_rows<kModeFast>, 256, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_rows<kModeLevel>, 256, 0);
  return nb;
}

cudaError_t launch_rows(int mode, const RowsArgs& a, int blocks, cudaStream_t s) {
  if (mode == kModeExact) k_rows<kModeExact><<<blocks, 256, 0, s>>>(a);
  else if (mode == kModeFast) k_rows<kModeFast><<<blocks, 256, 0, s>>>(a);
  else k_rows<kModeLevel><<<blocks, 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace sptrsv
