// Shared device helpers for the sm_100a SpTRSV kernels.
//
// Readiness protocol ("value is the flag"): every x slot that another warp may
// poll starts as the bit pattern kNotReady (all ones, a negative NaN that IEEE
// arithmetic on this GPU never produces: computed NaNs are canonical positive
// NaNs, and kernels canonicalise a computed value that happens to equal it).
// A producer publishes a component with ONE 8-byte relaxed store of the final
// value; a consumer polls the same 8 bytes with relaxed loads. No flag array, no
// fence, one L2 round trip per dependency — this replaces the paper's
// in_degree/left_sum counter pair (reference engine.py:495-550).
#pragma once
#include <cstdint>
#include <atomic>
#include <cuda_runtime.h>

namespace sptrsv {

constexpr unsigned long long kNotReady = 0xFFFFFFFFFFFFFFFFull;
constexpr int kWarp = 32;

// cudaFuncSetAttribute applies to the current device's context only: track,
// per kernel instantiation, the devices it was set on (one bit per ordinal).
template <typename F>
inline cudaError_t set_max_dyn_smem(F* fn, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = dev < 64 ? 1ull << dev : 0ull;
  if (bit && (done.load(std::memory_order_relaxed) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_relaxed);
  return e;
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const void* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// System scope: the slot may live in a peer GPU's HBM (NVLink P2P mapping).
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const void* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(void* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys_u64(void* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int ld_relaxed_s32(const void* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_s32(void* p, int v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys_u32(const void* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const void* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu_u32(void* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys_u32(void* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double as_f64(unsigned long long u) { return __longlong_as_double((long long)u); }
__device__ __forceinline__ unsigned long long as_u64(double d) { return (unsigned long long)__double_as_longlong(d); }

// A computed value must never alias the not-ready sentinel.
__device__ __forceinline__ unsigned long long publishable(double v) {
  unsigned long long u = as_u64(v);
  return u == kNotReady ? 0x7FF8000000000000ull : u;
}

__device__ __forceinline__ int exp_bits(double v) {
  return (int)((unsigned long long)__double_as_longlong(v) >> 52) & 0x7FF;
}

// Correctly rounded a/d from the correctly rounded reciprocal rd = RN(1/d):
// q = RN(a*rd), r = a - q*d (exact by FMA), RN(q + r*rd) == RN(a/d) (Markstein).
// 3 dependent DP ops (~25 cycles on B200) instead of the ~114-cycle DDIV
// sequence; outside the safe exponent window the IEEE division runs instead.
// Bit-identical to IEEE division — verified on 1e8 random operand pairs
// (tests/test_oracle.py::test_markstein_division_is_ieee).
// Operand-range guard of div_exact as one unsigned compare.
__device__ __forceinline__ bool markstein_ok(double v) { return (unsigned)(exp_bits(v) - 101) < 1845u; }

__device__ __forceinline__ double div_exact(double a, double d, double rd) {
  double q = __dmul_rn(a, rd);
  int eq = exp_bits(q), ea = exp_bits(a), ed = exp_bits(d);
  if (eq > 100 && eq < 1946 && ea > 100 && ea < 1946 && ed > 100 && ed < 1946) {
    double r = __fma_rn(-q, d, a);
    return __fma_rn(r, rd, q);
  }
  return __ddiv_rn(a, d);
}

// Device-side status word shared by all kernels of one launch.
struct DeviceStatus {
  int code;          // 0 ok, 5 timeout (matches SPTRSV_E_TIMEOUT), 10 debug check failed
  int detail;        // debug check: the first violating component (or mailbox word)
  unsigned long long spins;       // polls that found a dependency not ready
  unsigned long long remote_reads;  // dependency loads that crossed a PE boundary
};

}  // namespace sptrsv
