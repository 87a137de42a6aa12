// Latency floor of the 2D wavefront step for one warp on B200 (diagnostics).
// Each variant runs `iters` dependent steps and reports cycles per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain chain.cu && ./chain
//  0  dependent DFMA chain (latency of one DFMA)
//  1  dependent 64-bit __shfl_up_sync chain
//  2  the 2x2 step: row above by shuffle (lane 0 selects its inbox), 8 DFMA
//  3  the 2x2 step, row above through shared memory (STS.128 + LDS.128 of lane-1's slot)
//  4  two independent 2x2 steps interleaved (two bands in one warp)
//  5  the 2x2 step without the lane-0 select
//  6  1x2 step (one grid row per lane)
//  7  2x2 step, shuffle of the bottom row as soon as each element exists, x11 reassociated
//  8  four independent 2x2 steps interleaved
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ long long clk() {
  long long c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c));
  return c;
}

struct W {
  double wu[4], wl[4], bd[4];
};

__device__ __forceinline__ void blk(const W& w, const double (&top)[2], double (&xl)[2], double (&bot)[2]) {
  const double x00 = __fma_rn(w.wu[0], top[0], __fma_rn(w.wl[0], xl[0], w.bd[0]));
  const double x01 = __fma_rn(w.wu[1], top[1], __fma_rn(w.wl[1], x00, w.bd[1]));
  const double x10 = __fma_rn(w.wu[2], x00, __fma_rn(w.wl[2], xl[1], w.bd[2]));
  const double x11 = __fma_rn(w.wl[3], x10, __fma_rn(w.wu[3], x01, w.bd[3]));
  xl[0] = x01, xl[1] = x11;
  bot[0] = x10, bot[1] = x11;
}

template <int V>
__global__ void k(double* out, long long* cyc, int iters, double seed) {
  __shared__ __align__(16) double2 ex[2][32];
  const int lane = threadIdx.x & 31;
  W w;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    w.wu[i] = 0.1 * seed * (i + 1);
    w.wl[i] = 0.2 * seed * (i + 1);
    w.bd[i] = 0.3 * seed * (i + lane);
  }
  double inbox[2] = {seed, seed * 0.5};
  double xl[2] = {0, 0}, bot[2] = {1, 1}, xl2[2] = {0, 0}, bot2[2] = {1, 2};
  double xl3[2] = {0, 0}, bot3[2] = {1, 3}, xl4[2] = {0, 0}, bot4[2] = {1, 4};
  double acc = seed;
  __syncwarp();
  const long long t0 = clk();
  for (int s = 0; s < iters; ++s) {
    if (V == 0) {
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = __fma_rn(acc, w.wu[0], w.bd[0]);
    } else if (V == 1) {
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = __shfl_up_sync(0xffffffffu, acc, 1) + 0.0;
    } else if (V == 2 || V == 5 || V == 7) {
      double top[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double up = __shfl_up_sync(0xffffffffu, bot[q], 1);
        top[q] = (V == 5) ? up : (lane == 0 ? inbox[q] : up);
      }
      if (V == 7) {
        const double x00 = __fma_rn(w.wu[0], top[0], __fma_rn(w.wl[0], xl[0], w.bd[0]));
        const double x10 = __fma_rn(w.wu[2], x00, __fma_rn(w.wl[2], xl[1], w.bd[2]));
        const double x01 = __fma_rn(w.wu[1], top[1], __fma_rn(w.wl[1], x00, w.bd[1]));
        const double x11 = __fma_rn(w.wu[3], x01, __fma_rn(w.wl[3], x10, w.bd[3]));
        xl[0] = x01, xl[1] = x11, bot[0] = x10, bot[1] = x11;
      } else {
        blk(w, top, xl, bot);
      }
    } else if (V == 3) {
      ex[s & 1][lane] = make_double2(bot[0], bot[1]);
      __syncwarp();
      const double2 v = ex[s & 1][(lane + 31) & 31];
      double top[2] = {lane == 0 ? inbox[0] : v.x, lane == 0 ? inbox[1] : v.y};
      blk(w, top, xl, bot);
    } else if (V == 4 || V == 8) {
      double t1[2], t2[2], t3[2], t4[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double u1 = __shfl_up_sync(0xffffffffu, bot[q], 1);
        const double u2 = __shfl_up_sync(0xffffffffu, bot2[q], 1);
        t1[q] = lane == 0 ? inbox[q] : u1;
        t2[q] = lane == 0 ? inbox[q] : u2;
        if (V == 8) {
          const double u3 = __shfl_up_sync(0xffffffffu, bot3[q], 1);
          const double u4 = __shfl_up_sync(0xffffffffu, bot4[q], 1);
          t3[q] = lane == 0 ? inbox[q] : u3;
          t4[q] = lane == 0 ? inbox[q] : u4;
        }
      }
      blk(w, t1, xl, bot);
      blk(w, t2, xl2, bot2);
      if (V == 8) {
        blk(w, t3, xl3, bot3);
        blk(w, t4, xl4, bot4);
      }
    } else if (V == 6) {
      const double up = __shfl_up_sync(0xffffffffu, bot[1], 1);
      const double top = lane == 0 ? inbox[0] : up;
      const double x0 = __fma_rn(w.wu[0], top, __fma_rn(w.wl[0], xl[0], w.bd[0]));
      const double x1 = __fma_rn(w.wl[1], x0, __fma_rn(w.wu[1], bot[0], w.bd[1]));
      // (bot[0] stands in for the second column's row above, shuffled with it)
      xl[0] = x1, bot[0] = __shfl_up_sync(0xffffffffu, x0, 1), bot[1] = x1;
    }
  }
  const long long t1 = clk();
  out[blockIdx.x * 32 + lane] = acc + xl[0] + xl[1] + bot[0] + bot[1] + xl2[0] + bot2[1] + xl3[1] + bot4[0];
  if (lane == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name, int warps_per_cta = 1) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * 8 * 4);
  cudaMalloc(&cyc, 8 * 4);
  const int iters = 4096;
  k<V><<<1, 32 * warps_per_cta>>>(out, cyc, iters, 1.0);
  k<V><<<1, 32 * warps_per_cta>>>(out, cyc, iters, 1.0);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / iters / ((V == 0 || V == 1) ? 8 : 1);
  printf("{\"variant\": %d, \"name\": \"%s\", \"cycles_per_step\": %.1f}\n", V, name, per);
}

int main() {
  run<0>("dfma latency");
  run<1>("shfl f64 latency");
  run<2>("2x2 step, shfl + lane-0 select");
  run<3>("2x2 step, smem exchange");
  run<4>("2 x (2x2 step) interleaved");
  run<5>("2x2 step, no select");
  run<6>("1x2 step");
  run<7>("2x2 step, reassociated");
  run<8>("4 x (2x2 step) interleaved");
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
