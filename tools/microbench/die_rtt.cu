// L2 flag round trip between the CTA on SM 0 and every other SM (B200: two
// dies; a mailbox hand-over between SMs on different dies crosses the die
// link). One CTA per SM; CTA pairs (SM 0, SM k) ping-pong 200 times through
// value-is-flag words in global memory, k = 1 .. 147 in turn.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o die_rtt die_rtt.cu && ./die_rtt
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}
__device__ __forceinline__ long long ld_vol(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_vol(long long* p, long long v) {
  asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr int kReps = 200;

__global__ void k(long long* ping, long long* pong, int* turn, int* sm_of, long long* rtt, int nsm) {
  if (threadIdx.x != 0) return;
  const int me = smid();
  sm_of[blockIdx.x] = me;
  // block with smid 0 is the hub; every other block waits for its turn
  __threadfence();
  if (me == 0) {
    for (int k = 1; k < nsm; ++k) {
      // wait until SM k's block has announced itself
      while (ld_vol((long long*)&turn[2 * k]) == 0) {}
      long long t0 = clock64();
      for (int r = 1; r <= kReps; ++r) {
        st_vol(ping + 16 * k, r);
        while (ld_vol(pong + 16 * k) != r) {}
      }
      rtt[k] = (clock64() - t0) / kReps;
    }
  } else {
    atomicExch(&turn[2 * me], 1);
    for (int r = 1; r <= kReps; ++r) {
      while (ld_vol(ping + 16 * me) != r) {}
      st_vol(pong + 16 * me, r);
    }
  }
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long long *ping, *pong, *rtt;
  int *turn, *sm_of;
  cudaMalloc(&ping, sizeof(long long) * 16 * 256);
  cudaMalloc(&pong, sizeof(long long) * 16 * 256);
  cudaMalloc(&rtt, sizeof(long long) * 256);
  cudaMalloc(&turn, sizeof(int) * 2 * 256);
  cudaMalloc(&sm_of, sizeof(int) * 256);
  cudaMemset(ping, 0, sizeof(long long) * 16 * 256);
  cudaMemset(pong, 0, sizeof(long long) * 16 * 256);
  cudaMemset(turn, 0, sizeof(int) * 2 * 256);
  cudaMemset(rtt, 0, sizeof(long long) * 256);
  // 100 KB of shared memory per block: one block per SM
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  k<<<nsm, 32, 150 * 1024>>>(ping, pong, turn, sm_of, rtt, nsm);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  long long h[256];
  cudaMemcpy(h, rtt, sizeof(long long) * 256, cudaMemcpyDeviceToHost);
  printf("{\"nsm\": %d, \"rtt_cycles_from_sm0\": [0", nsm);
  for (int s = 1; s < nsm; ++s) printf(", %lld", h[s]);
  printf("]}\n");
  return 0;
}
