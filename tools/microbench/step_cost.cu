// Cost of the pieces of one lockstep wavefront step for a single warp on B200.
// Each variant runs `iters` steps of a 2x4 register block (shfl row-above, FMA
// wavefront) and adds one more ingredient of the stencil compute warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o step_cost step_cost.cu && ./step_cost
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.s32 %0, [%1];" : "=r"(v) : "r"(su(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(int* p, int v) {
  asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(su(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_vol(const int* p) { return *(volatile const int*)p; }
__device__ __forceinline__ void st_vol(int* p, int v) { *(volatile int*)p = v; }

template <int V>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ __align__(16) double2 buf[2][12][32];
  __shared__ __align__(16) double2 obuf[8][4][32];
  __shared__ int ctl[4];
  const int lane = threadIdx.x;
  for (int i = lane; i < 2 * 12 * 32; i += 32) (&buf[0][0][0])[i] = make_double2(0.25, 0.5);
  if (lane == 0) ctl[0] = ctl[1] = 1 << 30;
  __syncwarp();
  double w[24];
#pragma unroll
  for (int i = 0; i < 24; ++i) w[i] = 0.1 * (i + 1);
  double bottom[4] = {1, 1, 1, 1}, xleft[2] = {0, 0};
  long long t0 = clk();
  for (int s = 0; s < iters; ++s) {
    double top[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) top[c] = __shfl_up_sync(0xffffffffu, bottom[c], 1);
    double xb[2][4];
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int e = r * 4 + c;
        const double up = r == 0 ? top[c] : xb[r - 1][c];
        const double left = c == 0 ? xleft[r] : xb[r][c - 1];
        xb[r][c] = __fma_rn(w[e], left, __fma_rn(w[8 + e], up, w[16 + e]));
      }
#pragma unroll
    for (int r = 0; r < 2; ++r) xleft[r] = xb[r][3];
#pragma unroll
    for (int c = 0; c < 4; ++c) bottom[c] = xb[1][c];
    if (V >= 2) {  // stage out block to shared memory
#pragma unroll
      for (int q = 0; q < 4; ++q) obuf[s & 7][q][lane] = make_double2(xb[q / 2][(q % 2) * 2], xb[q / 2][(q % 2) * 2 + 1]);
    }
    if (V >= 3) __syncwarp();
    if (V == 4 && lane == 0) st_vol(&ctl[2], s);
    if (V >= 5 && lane == 0) st_rel(&ctl[2], s);
    if (V == 6) {
      while (ld_acq(&ctl[0]) < s) {
      }
    }
    if (V >= 1) {  // load next step's 12 coefficient pairs (+ 4 b pairs)
      const double2* cs = &buf[s & 1][0][0];
#pragma unroll
      for (int i = 0; i < 12; ++i) {
        const double2 v = cs[i * 32 + lane];
        w[2 * i] = v.x;
        w[2 * i + 1] = v.y;
      }
    }
  }
  long long t1 = clk();
  if (lane == 0) cyc[V] = t1 - t0;
  out[lane] = bottom[0] + xleft[1];
}

int main() {
  double* out;
  long long* cyc;
  long long h[8];
  cudaMalloc(&out, 64 * 8);
  cudaMalloc(&cyc, 8 * 8);
  const int it = 4096;
  const char* names[] = {"shfl+fma", "+lds next", "+sts out", "+syncwarp", "+volatile ctl", "+release ctl",
                         "+acquire wait"};
  k<0><<<1, 32>>>(out, cyc, it);
  k<0><<<1, 32>>>(out, cyc, it);
  k<1><<<1, 32>>>(out, cyc, it);
  k<2><<<1, 32>>>(out, cyc, it);
  k<3><<<1, 32>>>(out, cyc, it);
  k<4><<<1, 32>>>(out, cyc, it);
  k<5><<<1, 32>>>(out, cyc, it);
  k<6><<<1, 32>>>(out, cyc, it);
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{");
  for (int v = 0; v <= 6; ++v) printf("%s\"%s\": %.1f", v ? ", " : "", names[v], h[v] / (double)it);
  printf("}\n");
  return 0;
}
