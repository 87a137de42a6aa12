// COO -> CSC on the device for Matrix Market ingestion (SURVEY.md §8(f) row
// f3; reference mmio.py:132-144 `_coo_to_csc`): column-major order, rows
// ascending inside a column, duplicate coordinates summed.
//
// Keys col * n + row are radix-sorted with the entry's input position as the
// value (radix sort is stable, so duplicates keep their input order); one
// thread per unique coordinate then adds its duplicates sequentially from
// 0.0 in that order — the reference's np.bincount(group, weights) order — so
// the summed values are bit-identical. Column pointers come from a histogram
// of the unique columns and an exclusive scan.
#include <cstdint>
#include <cub/cub.cuh>
#include "../../include/sptrsv_b200.h"
#include "common.cuh"

namespace sptrsv {
int plan_fail(int code, const char* msg);
}

namespace {

__global__ void k_coo_keys(const int64_t* __restrict__ rows, const int64_t* __restrict__ cols, int64_t nnz, int64_t n,
                           unsigned long long* __restrict__ keys, int64_t* __restrict__ pos) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    keys[k] = (unsigned long long)cols[k] * (unsigned long long)n + (unsigned long long)rows[k];
    pos[k] = k;
  }
}

__global__ void k_coo_heads(const unsigned long long* __restrict__ keys, int64_t nnz, int* __restrict__ head) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
    head[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1 : 0;
}

// seg[k] = exclusive scan of head: the unique index of sorted entry k
__global__ void k_coo_starts(const int* __restrict__ head, const int* __restrict__ seg, int64_t nnz,
                             int64_t* __restrict__ start) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
    if (head[k]) start[seg[k]] = k;
}

__global__ void k_coo_reduce(const unsigned long long* __restrict__ keys, const int64_t* __restrict__ pos,
                             const double* __restrict__ vals, const int64_t* __restrict__ start, int64_t nu,
                             int64_t nnz, int64_t n, int64_t* __restrict__ row_out, double* __restrict__ val_out,
                             int* __restrict__ col_count) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nu; u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = start[u], e = u + 1 < nu ? start[u + 1] : nnz;
    double s = 0.0;
    for (int64_t k = b; k < e; ++k) s = __dadd_rn(s, vals[pos[k]]);
    const unsigned long long key = keys[b];
    row_out[u] = (int64_t)(key % (unsigned long long)n);
    val_out[u] = s;
    atomicAdd(col_count + (key / (unsigned long long)n), 1);
  }
}

__global__ void k_widen_ptr(const int* __restrict__ p, int64_t count, int64_t* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < count; k += (int64_t)gridDim.x * blockDim.x)
    out[k] = p[k];
}

int grid_of(int64_t work) { return (int)std::min<int64_t>((work + 255) / 256 + 1, 148 * 32); }

}  // namespace

using namespace sptrsv;

extern "C" int sptrsv_coo_to_csc(int64_t n, const int64_t* rows, const int64_t* cols, const double* vals, int64_t nnz,
                                 int32_t device, int64_t* col_ptr, int64_t* row_idx, double* values,
                                 int64_t* nnz_out) {
  if (n < 0 || nnz < 0 || !col_ptr || !nnz_out || (nnz && (!rows || !cols || !vals || !row_idx || !values)))
    return plan_fail(SPTRSV_E_ARGUMENT, "null argument");
  if (n >= (1ll << 31) - 1 || nnz >= (1ll << 31) - 1)
    return plan_fail(SPTRSV_E_UNSUPPORTED, "n and nnz must be < 2^31");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  cudaStream_t s;
  if ((e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  const int64_t m = nnz > 0 ? nnz : 1;
  int64_t *d_r = nullptr, *d_c = nullptr, *pos = nullptr, *pos_s = nullptr, *start = nullptr, *rout = nullptr,
          *cp64 = nullptr;
  double *d_v = nullptr, *vout = nullptr;
  unsigned long long *keys = nullptr, *keys_s = nullptr;
  int *head = nullptr, *seg = nullptr, *ccount = nullptr, *cptr = nullptr;
  void* tmp = nullptr;
  int64_t nu = 0;
  auto done = [&](cudaError_t err) -> int {
    void* ptrs[] = {d_r, d_c, pos, pos_s, start, rout, cp64, d_v, vout, keys, keys_s, head, seg, ccount, cptr, tmp};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    cudaStreamDestroy(s);
    return err == cudaSuccess ? SPTRSV_OK : plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(err));
  };
#define C_TRY(x)                   \
  do {                             \
    cudaError_t _e = (x);          \
    if (_e != cudaSuccess) return done(_e); \
  } while (0)
  C_TRY(cudaMalloc(&d_r, sizeof(int64_t) * m));
  C_TRY(cudaMalloc(&d_c, sizeof(int64_t) * m));
  C_TRY(cudaMalloc(&d_v, sizeof(double) * m));
  C_TRY(cudaMalloc(&keys, sizeof(unsigned long long) * m));
  C_TRY(cudaMalloc(&keys_s, sizeof(unsigned long long) * m));
  C_TRY(cudaMalloc(&pos, sizeof(int64_t) * m));
  C_TRY(cudaMalloc(&pos_s, sizeof(int64_t) * m));
  C_TRY(cudaMalloc(&head, sizeof(int) * m));
  C_TRY(cudaMalloc(&seg, sizeof(int) * m));
  C_TRY(cudaMalloc(&start, sizeof(int64_t) * m));
  C_TRY(cudaMalloc(&rout, sizeof(int64_t) * m));
  C_TRY(cudaMalloc(&vout, sizeof(double) * m));
  C_TRY(cudaMalloc(&ccount, sizeof(int) * (n + 1)));
  C_TRY(cudaMalloc(&cptr, sizeof(int) * (n + 1)));
  C_TRY(cudaMalloc(&cp64, sizeof(int64_t) * (n + 1)));
  C_TRY(cudaMemsetAsync(ccount, 0, sizeof(int) * (n + 1), s));
  if (nnz) {
    C_TRY(cudaMemcpyAsync(d_r, rows, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, s));
    C_TRY(cudaMemcpyAsync(d_c, cols, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, s));
    C_TRY(cudaMemcpyAsync(d_v, vals, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
    k_coo_keys<<<grid_of(nnz), 256, 0, s>>>(d_r, d_c, nnz, n, keys, pos);
    C_TRY(cudaGetLastError());
    int end_bit = 1;
    while (end_bit < 64 && ((unsigned long long)n * (unsigned long long)n >> end_bit)) ++end_bit;
    size_t tb = 0;
    C_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys_s, pos, pos_s, (int)nnz, 0, end_bit, s));
    C_TRY(cudaMalloc(&tmp, tb));
    C_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys_s, pos, pos_s, (int)nnz, 0, end_bit, s));
    k_coo_heads<<<grid_of(nnz), 256, 0, s>>>(keys_s, nnz, head);
    C_TRY(cudaGetLastError());
    cudaFree(tmp);
    tmp = nullptr;
    tb = 0;
    C_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, head, seg, (int)nnz, s));
    C_TRY(cudaMalloc(&tmp, tb));
    C_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, head, seg, (int)nnz, s));
    int last_seg = 0, last_head = 0;
    C_TRY(cudaMemcpyAsync(&last_seg, seg + nnz - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    C_TRY(cudaMemcpyAsync(&last_head, head + nnz - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    C_TRY(cudaStreamSynchronize(s));
    nu = (int64_t)last_seg + last_head;
    k_coo_starts<<<grid_of(nnz), 256, 0, s>>>(head, seg, nnz, start);
    C_TRY(cudaGetLastError());
    k_coo_reduce<<<grid_of(nu), 256, 0, s>>>(keys_s, pos_s, d_v, start, nu, nnz, n, rout, vout, ccount);
    C_TRY(cudaGetLastError());
  }
  // column pointers: exclusive scan over the n+1 counters (the last is 0)
  size_t tb2 = 0;
  C_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb2, ccount, cptr, (int)(n + 1), s));
  void* tmp2 = nullptr;
  C_TRY(cudaMalloc(&tmp2, tb2));
  cudaError_t es = cub::DeviceScan::ExclusiveSum(tmp2, tb2, ccount, cptr, (int)(n + 1), s);
  if (es == cudaSuccess) {
    k_widen_ptr<<<grid_of(n + 1), 256, 0, s>>>(cptr, n + 1, cp64);
    es = cudaGetLastError();
  }
  if (es == cudaSuccess) es = cudaMemcpyAsync(col_ptr, cp64, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s);
  if (es == cudaSuccess && nu) es = cudaMemcpyAsync(row_idx, rout, sizeof(int64_t) * nu, cudaMemcpyDeviceToHost, s);
  if (es == cudaSuccess && nu) es = cudaMemcpyAsync(values, vout, sizeof(double) * nu, cudaMemcpyDeviceToHost, s);
  if (es == cudaSuccess) es = cudaStreamSynchronize(s);
  cudaFree(tmp2);
  *nnz_out = nu;
  return done(es);
#undef C_TRY
}
