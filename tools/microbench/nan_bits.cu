// Which NaN bit patterns do FP64 DFMA / DMUL / DADD / IEEE division return
// for NaN operands on this GPU? (The stencil mailbox sentinel must be a
// pattern arithmetic never produces.)
#include <cstdio>
#include <cstring>
__global__ void k(const unsigned long long* in, unsigned long long* out, int n) {
  for (int i = 0; i < n; ++i) {
    const double a = __longlong_as_double(in[i]);
    out[6 * i + 0] = __double_as_longlong(__fma_rn(a, 1.5, 2.0));
    out[6 * i + 1] = __double_as_longlong(__fma_rn(0.5, 1.5, a));
    out[6 * i + 2] = __double_as_longlong(__dmul_rn(a, 3.0));
    out[6 * i + 3] = __double_as_longlong(__dadd_rn(a, 1.0));
    out[6 * i + 4] = __double_as_longlong(__ddiv_rn(a, 3.0));
    out[6 * i + 5] = __double_as_longlong(__ddiv_rn(3.0, a));
  }
}
int main() {
  const unsigned long long h[] = {0xFFF0000000000001ull, 0x7FF0000000000001ull, 0xFFFFFFFFFFFFFFFFull,
                                  0x7FF8000000000000ull, 0xFFF8000000000123ull};
  const int n = sizeof(h) / sizeof(h[0]);
  unsigned long long *d, *o, r[6 * n];
  cudaMalloc(&d, sizeof(h));
  cudaMalloc(&o, sizeof(r));
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  k<<<1, 1>>>(d, o, n);
  cudaMemcpy(r, o, sizeof(r), cudaMemcpyDeviceToHost);
  for (int i = 0; i < n; ++i) {
    printf("in %016llx ->", h[i]);
    for (int j = 0; j < 6; ++j) printf(" %016llx", r[6 * i + j]);
    printf("\n");
  }
  return 0;
}
