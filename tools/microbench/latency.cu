// Latency microbenchmarks that size the SpTRSV critical path on B200 (sm_100a).
// Each test prints cycles per dependent hop; run once per box with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat latency.cu && ./lat
// Measures: fp64 DADD/DMUL/DFMA/DDIV dependent latency, SHFL latency,
// smem st->syncwarp->ld hop, L2 flag ping-pong between two CTAs (acquire/release),
// DSMEM push ping-pong inside a 2-CTA cluster.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ long long clk() { long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; }

__global__ void fp_lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = a;
  long long t0 = clk();
  for (int i = 0; i < iters; ++i) x = __dadd_rn(x, b);
  long long t1 = clk();
  double y = a;
  for (int i = 0; i < iters; ++i) y = __dmul_rn(y, b);
  long long t2 = clk();
  double z = a;
  for (int i = 0; i < iters; ++i) z = fma(z, b, a);
  long long t3 = clk();
  double w = a;
  for (int i = 0; i < iters; ++i) w = (w + 1.0) / b;
  long long t4 = clk();
  out[0] = x + y + z + w;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
}

__global__ void shfl_lat(double* out, long long* cyc, int iters) {
  double v = threadIdx.x;
  long long t0 = clk();
  for (int i = 0; i < iters; ++i) v = __shfl_up_sync(0xffffffffu, v, 1) + 1.0;
  long long t1 = clk();
  int u = threadIdx.x;
  for (int i = 0; i < iters; ++i) u = __shfl_up_sync(0xffffffffu, u, 1) + 1;
  long long t2 = clk();
  if (threadIdx.x == 31) { out[0] = v + u; cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}

// lane k waits for lane k-1's value written into smem, passes token along: 32-lane relay
__global__ void smem_relay(long long* cyc, int iters) {
  __shared__ volatile int slot[32];
  int lane = threadIdx.x;
  slot[lane] = -1;
  __syncwarp();
  long long t0 = clk();
  for (int it = 0; it < iters; ++it) {
    // round: lane 0 writes it, lane k waits for slot[k-1]==it, then writes slot[k]=it
    if (lane == 0) { if (it > 0) { while (slot[31] != it - 1) {} } slot[0] = it; }
    else { while (slot[lane - 1] != it) {} slot[lane] = it; }
  }
  // wait all
  while (slot[31] != iters - 1) {}
  long long t1 = clk();
  if (lane == 0) cyc[0] = t1 - t0;
}

// lockstep warp step through smem: write own slot, __syncwarp, read neighbour's slot
__global__ void smem_step(double* out, long long* cyc, int iters) {
  __shared__ double slot[2][32];
  int lane = threadIdx.x;
  double v = lane;
  long long t0 = clk();
  for (int i = 0; i < iters; ++i) {
    slot[i & 1][lane] = v;
    __syncwarp();
    v = fma(slot[i & 1][(lane + 31) & 31], 0.5, v);
  }
  long long t1 = clk();
  if (lane == 0) { out[1] = v; cyc[0] = t1 - t0; }
}

// Two CTAs ping-pong a flag through global memory (L2). Block 0 and block 1.
__global__ void l2_pingpong(int* flag, long long* cyc, int iters, unsigned* smid) {
  if (threadIdx.x != 0) return;
  unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s)); smid[blockIdx.x] = s;
  int me = blockIdx.x;
  long long t0 = clk();
  for (int i = 0; i < iters; ++i) {
    if (me == 0) {
      int v;
      asm volatile("st.release.gpu.global.s32 [%0], %1;" :: "l"(flag), "r"(2 * i + 1) : "memory");
      do { asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory"); } while (v != 2 * i + 2);
    } else {
      int v;
      do { asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory"); } while (v != 2 * i + 1);
      asm volatile("st.release.gpu.global.s32 [%0], %1;" :: "l"(flag), "r"(2 * i + 2) : "memory");
    }
  }
  long long t1 = clk();
  cyc[me] = t1 - t0;
}

// relaxed/volatile variant
__global__ void l2_pingpong_relaxed(int* flag, long long* cyc, int iters) {
  if (threadIdx.x != 0) return;
  int me = blockIdx.x;
  volatile int* f = flag;
  long long t0 = clk();
  for (int i = 0; i < iters; ++i) {
    if (me == 0) {
      *f = 2 * i + 1; while (*f != 2 * i + 2) {}
    } else {
      while (*f != 2 * i + 1) {} *f = 2 * i + 2;
    }
  }
  long long t1 = clk();
  cyc[me] = t1 - t0;
}

// DSMEM push ping-pong: CTA r writes into peer's smem slot, polls its own.
__global__ void __cluster_dims__(2, 1, 1) dsmem_pingpong(long long* cyc, int iters) {
  __shared__ int slot;
  cg::cluster_group cl = cg::this_cluster();
  if (threadIdx.x == 0) slot = -1;
  cl.sync();
  unsigned me = cl.block_rank();
  int* peer = cl.map_shared_rank(&slot, me ^ 1);
  volatile int* mine = &slot;
  long long t0 = clk();
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      if (me == 0) {
        asm volatile("st.release.cluster.s32 [%0], %1;" :: "l"(peer), "r"(2 * i + 1) : "memory");
        int v; do { asm volatile("ld.acquire.cluster.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared((void*)mine)) : "memory"); } while (v != 2 * i + 2);
      } else {
        int v; do { asm volatile("ld.acquire.cluster.shared::cta.s32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared((void*)mine)) : "memory"); } while (v != 2 * i + 1);
        asm volatile("st.release.cluster.s32 [%0], %1;" :: "l"(peer), "r"(2 * i + 2) : "memory");
      }
    }
  }
  long long t1 = clk();
  if (threadIdx.x == 0) cyc[me] = t1 - t0;
  cl.sync();
}

// global load latency (pointer chase in L2-resident buffer)
__global__ void chase(const int* nxt, long long* cyc, int iters, int* sink) {
  int p = 0;
  long long t0 = clk();
  for (int i = 0; i < iters; ++i) p = __ldcg(nxt + p);
  long long t1 = clk();
  sink[0] = p; cyc[0] = t1 - t0;
}

int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  double* dout; long long* dcyc; long long h[8]; int* dflag; unsigned* dsm; unsigned hsm[2];
  CK(cudaMalloc(&dout, 64)); CK(cudaMalloc(&dcyc, 64)); CK(cudaMalloc(&dflag, 64)); CK(cudaMalloc(&dsm, 64));
  int it = 4096;
  fp_lat<<<1, 1>>>(dout, dcyc, it, 1.0000001, 0.9999999); CK(cudaDeviceSynchronize());
  fp_lat<<<1, 1>>>(dout, dcyc, it, 1.0000001, 0.9999999); CK(cudaMemcpy(h, dcyc, 32, cudaMemcpyDeviceToHost));
  printf("{\"dadd\": %.1f, \"dmul\": %.1f, \"dfma\": %.1f, \"dadd_ddiv\": %.1f,", h[0] / (double)it, h[1] / (double)it, h[2] / (double)it, h[3] / (double)it);
  shfl_lat<<<1, 32>>>(dout, dcyc, it); shfl_lat<<<1, 32>>>(dout, dcyc, it); CK(cudaMemcpy(h, dcyc, 16, cudaMemcpyDeviceToHost));
  printf(" \"shfl_f64_plus_dadd\": %.1f, \"shfl_i32_plus_iadd\": %.1f,", h[0] / (double)it, h[1] / (double)it);
  smem_relay<<<1, 32>>>(dcyc, 256); smem_relay<<<1, 32>>>(dcyc, 256); CK(cudaMemcpy(h, dcyc, 8, cudaMemcpyDeviceToHost));
  printf(" \"smem_relay_per_hop\": %.1f,", h[0] / (256.0 * 32));
  smem_step<<<1, 32>>>(dout, dcyc, it); smem_step<<<1, 32>>>(dout, dcyc, it); CK(cudaMemcpy(h, dcyc, 8, cudaMemcpyDeviceToHost));
  printf(" \"smem_lockstep_step_plus_dfma\": %.1f,", h[0] / (double)it);
  int pit = 2000;
  CK(cudaMemset(dflag, 0, 4)); l2_pingpong<<<2, 32>>>(dflag, dcyc, pit, dsm); CK(cudaDeviceSynchronize());
  CK(cudaMemset(dflag, 0, 4)); l2_pingpong<<<2, 32>>>(dflag, dcyc, pit, dsm); CK(cudaMemcpy(h, dcyc, 16, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hsm, dsm, 8, cudaMemcpyDeviceToHost));
  printf(" \"l2_acqrel_roundtrip\": %.1f, \"smids\": [%u, %u],", h[0] / (double)pit, hsm[0], hsm[1]);
  // sweep block pairs across SMs: launch 148 blocks? use many CTAs: measure with grid 2 but occupancy spreads; also try 2 blocks placed via big grid
  CK(cudaMemset(dflag, 0, 4)); l2_pingpong_relaxed<<<2, 32>>>(dflag, dcyc, pit); CK(cudaMemcpy(h, dcyc, 16, cudaMemcpyDeviceToHost));
  printf(" \"l2_volatile_roundtrip\": %.1f,", h[0] / (double)pit);
  dsmem_pingpong<<<2, 32>>>(dcyc, pit); CK(cudaDeviceSynchronize());
  dsmem_pingpong<<<2, 32>>>(dcyc, pit); CK(cudaMemcpy(h, dcyc, 16, cudaMemcpyDeviceToHost));
  printf(" \"dsmem_roundtrip\": %.1f,", h[0] / (double)pit);
  // pointer chase, 1 MB ring with stride 257 ints
  const int N = 1 << 18; int* hn = new int[N]; for (int i = 0; i < N; ++i) hn[i] = (i + 4099) % N;
  int* dn; int* dsink; CK(cudaMalloc(&dn, N * 4)); CK(cudaMalloc(&dsink, 4)); CK(cudaMemcpy(dn, hn, N * 4, cudaMemcpyHostToDevice));
  chase<<<1, 1>>>(dn, dcyc, 4096, dsink); chase<<<1, 1>>>(dn, dcyc, 4096, dsink); CK(cudaMemcpy(h, dcyc, 8, cudaMemcpyDeviceToHost));
  printf(" \"l2_load_latency\": %.1f", h[0] / 4096.0);
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf(", \"clock_khz\": %d}\n", clk_khz);
  return 0;
}
