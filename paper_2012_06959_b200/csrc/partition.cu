// PE partitions: the read-only inter-PE layer (paper Alg. 3, PAPER.md:339-399;
// reference solve_partitioned, engine.py:438-582).
//
// Each PE owns the components of PartitionPlan.owner_arr and publishes their x
// only into its own segment (a full-length value-is-flag array in its HBM);
// every other PE reads that segment with one-sided loads and never writes it.
// Two deployments share this code:
//   * all PEs on one device (virtual PEs, one process): every segment is local,
//     one launch serves all PEs (block b works for PE b % n_pes) so all
//     persistent warps are co-resident;
//   * one PE per GPU (one process per GPU): the PE's own segment is local, the
//     others are peer mappings of other processes' segments opened from CUDA
//     IPC handles, read over NVLink/NVSwitch with .sys-scope relaxed loads.
// Inside the solve there is no collective and no remote write; scattering b
// and gathering x around it is the caller's (NCCL in bench.py).
#include <vector>
#include <chrono>
#include <algorithm>
#include <cstring>
#include "plan.hpp"
#include "kernels.cuh"
#include "../../include/sptrsv_b200.h"

namespace sptrsv {

int plan_fail(int code, const char* msg);

namespace {

// x[i] = segment of owner(i) at i, for the PEs of this process.
__global__ void k_gather_owned(unsigned long long* const* segs, const unsigned char* owner, int pe_base, int n_local,
                               long long n, double* x) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int p = owner[i];
    if (p >= pe_base && p < pe_base + n_local) x[i] = __longlong_as_double((long long)segs[p][i]);
  }
}

}  // namespace

void DevicePlan::release_partition() {
  stencil.release_part();
  bblk.release_part();
  for (auto* s : local_segs) cudaFree(s);
  local_segs.clear();
  for (void* p : opened_peers) cudaIpcCloseMemHandle(p);
  opened_peers.clear();
  void* ptrs[] = {owner_dev, seg_table, pe_order, pe_order_off, pe_tickets};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  owner_dev = nullptr;
  seg_table = nullptr;
  pe_order = nullptr;
  pe_order_off = nullptr;
  pe_tickets = nullptr;
  host_seg_table.clear();
  host_owner.clear();
  n_pes = 1;
  n_pe_local = 1;
  pe_base = 0;
}

int DevicePlan::set_partition(const int32_t* owner, int pes, int my_pe) {
  if (structure_only) return plan_fail(SPTRSV_E_ARGUMENT, "structure-only plan");
  if (pes < 1 || pes > 255) return plan_fail(SPTRSV_E_INVALID_PE, "need 1 <= n_pes <= 255");
  if (my_pe >= pes) return plan_fail(SPTRSV_E_INVALID_PE, "my_pe out of range");
  std::vector<unsigned char> own(n);
  for (long long i = 0; i < n; ++i) {
    if (owner[i] < 0 || owner[i] >= pes) return plan_fail(SPTRSV_E_INVALID_PE, "owner entry out of range");
    own[i] = (unsigned char)owner[i];
  }
  cudaSetDevice(device);
  release_partition();
  host_owner = own;
  if (executor_used == SPTRSV_EXECUTOR_STENCIL && stencil.ready && my_pe >= 0) {
    // band-aligned block (or band round-robin) ownership: the stencil
    // executor runs partitioned; anything else falls back to the pool
    const int rc = set_stencil_partition(owner, pes, my_pe);
    if (rc < 0) return SPTRSV_E_CUDA;
    if (rc == 1) return SPTRSV_OK;
  }
  if (executor_used == SPTRSV_EXECUTOR_BAND && bblk.ready && my_pe >= 0) {
    // contiguous slabs in PE order on row-block boundaries: the band-block
    // executor runs partitioned; anything else falls back to the pool
    const int rc = set_band_partition(owner, pes, my_pe);
    if (rc < 0) return SPTRSV_E_CUDA;
    if (rc == 1) return SPTRSV_OK;
  }
  n_pes = pes;
  pe_base = my_pe < 0 ? 0 : my_pe;
  n_pe_local = my_pe < 0 ? pes : 1;
  // per-PE ticket orders: the PE's components in level order (ascending rows per level)
  std::vector<int> h_by_level(n);
  cudaError_t e;
  if ((e = cudaMemcpy(h_by_level.data(), by_level, sizeof(int) * n, cudaMemcpyDeviceToHost)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  std::vector<long long> off(n_pe_local + 1, 0);
  for (long long k = 0; k < n; ++k) {
    const int p = own[h_by_level[k]];
    if (p >= pe_base && p < pe_base + n_pe_local) ++off[p - pe_base + 1];
  }
  for (int q = 0; q < n_pe_local; ++q) off[q + 1] += off[q];
  std::vector<int> ord(std::max<long long>(off[n_pe_local], 1));
  std::vector<long long> fill(off.begin(), off.end() - 1);
  for (long long k = 0; k < n; ++k) {
    const int r = h_by_level[k];
    const int p = own[r];
    if (p >= pe_base && p < pe_base + n_pe_local) ord[fill[p - pe_base]++] = r;
  }
  auto al = [](void** p, size_t b) { return cudaMalloc(p, b < 16 ? 16 : b); };
  if ((e = al((void**)&owner_dev, n)) != cudaSuccess ||
      (e = al((void**)&pe_order, sizeof(int) * ord.size())) != cudaSuccess ||
      (e = al((void**)&pe_order_off, sizeof(long long) * off.size())) != cudaSuccess ||
      (e = al((void**)&pe_tickets, sizeof(int) * n_pe_local)) != cudaSuccess ||
      (e = al((void**)&seg_table, 2 * sizeof(void*) * pes)) != cudaSuccess)
    return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  cudaMemcpy(owner_dev, own.data(), n, cudaMemcpyHostToDevice);
  cudaMemcpy(pe_order, ord.data(), sizeof(int) * ord.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(pe_order_off, off.data(), sizeof(long long) * off.size(), cudaMemcpyHostToDevice);
  host_seg_table.assign(pes, nullptr);
  for (int q = 0; q < n_pe_local; ++q) {
    unsigned long long* seg = nullptr;
    if ((e = al((void**)&seg, 2 * sizeof(unsigned long long) * n)) != cudaSuccess ||
        (e = cudaMemset(seg, 0xFF, 2 * sizeof(unsigned long long) * n)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    local_segs.push_back(seg);
    host_seg_table[pe_base + q] = seg;
  }
  part_solves = 0;
  if (sync_seg_table() != SPTRSV_OK) return SPTRSV_E_CUDA;
  // the read-only inter-PE layer is the component pool (warp per component,
  // value-is-flag peer loads)
  executor_used = SPTRSV_EXECUTOR_ROWS;
  return SPTRSV_OK;
}

// Device segment table [2][n_pes]: half h of PE p's segment is seg_p + h * n.
int DevicePlan::sync_seg_table() {
  std::vector<unsigned long long*> t(2 * n_pes, nullptr);
  for (int p = 0; p < n_pes; ++p)
    if (host_seg_table[p]) t[p] = host_seg_table[p], t[n_pes + p] = host_seg_table[p] + n;
  cudaError_t e = cudaMemcpy(seg_table, t.data(), sizeof(void*) * t.size(), cudaMemcpyHostToDevice);
  return e == cudaSuccess ? SPTRSV_OK : plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
}

int DevicePlan::solve_partitioned_rows(const double* d_b, double* d_x, cudaStream_t s) {
  for (int p = 0; p < n_pes; ++p)
    if (!host_seg_table[p]) return plan_fail(SPTRSV_E_INVALID_PE, "a peer segment was never imported");
  const int mode = opt.precision == SPTRSV_PRECISION_FAST ? kModeFast : kModeExact;
  // Segments are double-buffered by solve parity: this solve publishes into
  // and reads half `par` (reset by the previous solve), and resets the other
  // half for the next solve, so no PE ever resets a half a peer may still be
  // reading (consecutive solves are separated by a barrier across PEs).
  const int par = (int)(part_solves++ & 1);
  unsigned long long** table = seg_table + par * n_pes;
  cudaError_t e = cudaSuccess;
  for (auto* seg : local_segs)
    if ((e = cudaMemsetAsync(seg + (1 - par) * n, 0xFF, sizeof(unsigned long long) * n, s)) != cudaSuccess) break;
  if (e == cudaSuccess) e = cudaMemsetAsync(pe_tickets, 0, sizeof(int) * n_pe_local, s);
  if (e == cudaSuccess) e = reset_control(s);
  if (e != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  RowsArgs a{};
  a.debug = (opt.flags & SPTRSV_PLAN_DEBUG) ? ((opt.probe_flags & 1024) ? 2 : 1) : 0;
  a.n = (int)n;
  a.rp = rp;
  a.ci = ci;
  a.val = mode == kModeFast ? wv : cv;
  a.dg = dg;
  a.rdg = rdg;
  a.b = d_b;
  a.xseg = table;
  a.lseg = lseg_dev;
  a.owner = owner_dev;
  a.pe_base = pe_base;
  a.n_pe_local = n_pe_local;
  a.pe_order_off = pe_order_off;
  a.order = pe_order;
  a.order_len = 0;
  a.ticket = pe_tickets;
  a.status = status;
  a.abort_flag = abort_flag;
  a.timeout_ns = (unsigned long long)(opt.timeout_s * 1e9);
  a.spin_initial = opt.spin_initial;
  a.spin_max_ns = opt.spin_max_ns;
  a.coop_long = 0;
  a.long_deps = 1 << 30;
  a.lane_loop = rows_lane_loop();
  int per_sm = rows_blocks_per_sm(mode);
  // grid_cap: this PE's share of the SMs when several PEs' kernels share the device
  int blocks = std::max(1, (grid_cap > 0 ? std::min(grid_cap, num_sms) : num_sms) * std::max(per_sm, 1));
  blocks = std::max(n_pe_local, blocks - blocks % n_pe_local);
  if ((e = record_k0(s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if ((e = launch_rows(mode, a, blocks, s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if ((e = cudaEventRecord(evk1, s)) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if (d_x) {
    k_gather_owned<<<std::min<long long>((n + 255) / 256, 148 * 16), 256, 0, s>>>(table, owner_dev, pe_base,
                                                                                   n_pe_local, n, d_x);
    if ((e = cudaGetLastError()) != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  }
  launches = 2;
  return SPTRSV_OK;
}

// A peer pointer on another device of this process: enable P2P access from
// this plan's device to it (NVLink/NVSwitch between B200s), once.
int DevicePlan::enable_peer(const void* peer_ptr) {
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, peer_ptr);
  if (e != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  if (at.type != cudaMemoryTypeDevice || at.device == device) return SPTRSV_OK;
  int ok = 0;
  if ((e = cudaDeviceCanAccessPeer(&ok, device, at.device)) != cudaSuccess || !ok)
    return plan_fail(SPTRSV_E_CUDA, "no peer access between the plans' devices");
  cudaSetDevice(device);
  e = cudaDeviceEnablePeerAccess(at.device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    e = cudaSuccess;
  }
  return e == cudaSuccess ? SPTRSV_OK : plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
}

}  // namespace sptrsv

using namespace sptrsv;

extern "C" {

// One solve over the PEs of a partition held by this process: plans[p] is PE
// p (sptrsv_plan_set_partition(plan, owner, n_plans, p)), peers wired with
// sptrsv_plan_set_peer_segment. b is copied once per device, every PE's kernel
// is launched on its own stream (they depend on each other's published x, so
// they must run concurrently; persistent grids are capped so that the PEs of
// one device are co-resident), and x is assembled from each PE's rows.
int sptrsv_solve_group(sptrsv_plan* const* plans, int32_t n_plans, const double* b, double* x,
                       sptrsv_stats* stats) {
  if (!plans || n_plans < 1 || !b || !x) return plan_fail(SPTRSV_E_ARGUMENT, "null argument");
  std::vector<DevicePlan*> ps(n_plans);
  for (int p = 0; p < n_plans; ++p) {
    ps[p] = reinterpret_cast<DevicePlan*>(plans[p]);
    if (!ps[p]) return plan_fail(SPTRSV_E_ARGUMENT, "null plan");
    if (ps[p]->n != ps[0]->n) return plan_fail(SPTRSV_E_ARGUMENT, "plans of different matrices");
    if ((long long)ps[p]->host_owner.size() != ps[p]->n)
      return plan_fail(SPTRSV_E_INVALID_PE, "plan has no PE partition");
  }
  const long long n = ps[0]->n;
  if (n == 0) return SPTRSV_OK;
  // one b / x buffer per device: the first plan on the device lends its own
  std::vector<int> devs;
  std::vector<DevicePlan*> lead;
  std::vector<int> dev_of(n_plans), count;
  for (int p = 0; p < n_plans; ++p) {
    int k = 0;
    while (k < (int)devs.size() && devs[k] != ps[p]->device) ++k;
    if (k == (int)devs.size()) {
      devs.push_back(ps[p]->device);
      lead.push_back(ps[p]);
      count.push_back(0);
    }
    dev_of[p] = k;
    ++count[k];
  }
  auto t0 = std::chrono::steady_clock::now();
  cudaError_t e;
  for (size_t k = 0; k < devs.size(); ++k) {
    cudaSetDevice(devs[k]);
    if ((e = cudaMemcpyAsync(lead[k]->bbuf, b, sizeof(double) * n, cudaMemcpyHostToDevice, lead[k]->stream)) !=
            cudaSuccess ||
        (e = cudaStreamSynchronize(lead[k]->stream)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  }
  for (int p = 0; p < n_plans; ++p) {
    DevicePlan* d = ps[p];
    const int k = dev_of[p];
    d->grid_cap = count[k] > 1 ? std::max(1, d->num_sms / count[k]) : 0;
    cudaSetDevice(d->device);
    const int rc = d->solve_device(lead[k]->bbuf, lead[k]->xbuf, d->stream);
    if (rc != SPTRSV_OK) return rc;
  }
  double kernel_ms = 0.0;
  long long spins = 0, remote = 0, launches = 0;
  int status = SPTRSV_OK;
  for (int p = 0; p < n_plans; ++p) {
    cudaSetDevice(ps[p]->device);
    sptrsv_stats st{};
    const int rc = ps[p]->finish(&st);
    if (rc != SPTRSV_OK && status == SPTRSV_OK) status = rc;
    kernel_ms = std::max(kernel_ms, st.kernel_ms);
    spins += st.spins;
    remote += st.remote_reads;
    launches += st.launches;
  }
  if (status != SPTRSV_OK) return status;
  // every PE wrote only its own rows of its device's x buffer
  std::vector<double> tmp;
  for (size_t k = 0; k < devs.size(); ++k) {
    cudaSetDevice(devs[k]);
    double* dst = x;
    if (devs.size() > 1) {
      tmp.resize(n);
      dst = tmp.data();
    }
    if ((e = cudaMemcpy(dst, lead[k]->xbuf, sizeof(double) * n, cudaMemcpyDeviceToHost)) != cudaSuccess)
      return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    if (devs.size() > 1) {
      const std::vector<unsigned char>& own = ps[0]->host_owner;
      for (long long i = 0; i < n; ++i)
        if (dev_of[own[i]] == (int)k) x[i] = tmp[i];
    }
  }
  if (stats) {
    *stats = sptrsv_stats{};
    stats->kernel_ms = kernel_ms;
    stats->solve_ms = kernel_ms;
    stats->spins = spins;
    stats->remote_reads = remote;
    stats->launches = launches;
    stats->executor = ps[0]->executor_used;
    stats->n_levels = ps[0]->n_levels;
    stats->e2e_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return SPTRSV_OK;
}


int sptrsv_plan_set_partition(sptrsv_plan* plan, const int32_t* owner, int32_t n_pes, int32_t my_pe) {
  auto* p = reinterpret_cast<DevicePlan*>(plan);
  if (!p || !owner) return plan_fail(SPTRSV_E_ARGUMENT, "null argument");
  return p->set_partition(owner, n_pes, my_pe);
}

int sptrsv_plan_export_segment(const sptrsv_plan* plan, void* handle_out) {
  auto* p = reinterpret_cast<const DevicePlan*>(plan);
  if (!p || !handle_out) return plan_fail(SPTRSV_E_ARGUMENT, "null argument");
  if (p->stencil.part) {  // the stencil's shared state is its mailbox array
    cudaSetDevice(p->device);
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, p->stencil.mbox);
    if (e != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    std::memcpy(handle_out, &h, sizeof(h));
    return SPTRSV_OK;
  }
  if (p->bblk.part) {  // the band chain's shared state is this PE's tail slot
    cudaSetDevice(p->device);
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, p->bblk.slot);
    if (e != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
    std::memcpy(handle_out, &h, sizeof(h));
    return SPTRSV_OK;
  }
  if (p->local_segs.size() != 1) return plan_fail(SPTRSV_E_ARGUMENT, "export needs a one-PE-per-process partition");
  cudaSetDevice(p->device);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, p->local_segs[0]);
  if (e != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  std::memcpy(handle_out, &h, sizeof(h));
  return SPTRSV_OK;
}

int sptrsv_plan_import_segment(sptrsv_plan* plan, int32_t pe, const void* handle) {
  auto* p = reinterpret_cast<DevicePlan*>(plan);
  if (!p || !handle) return plan_fail(SPTRSV_E_ARGUMENT, "null argument");
  const bool st = p->stencil.part, bb = p->bblk.part;
  if (pe < 0 || pe >= (st ? p->stencil.n_pes : bb ? p->bblk.n_pes : p->n_pes))
    return plan_fail(SPTRSV_E_INVALID_PE, "pe out of range");
  if (st ? pe == p->stencil.my_pe : bb ? pe == p->bblk.my_pe : (pe >= p->pe_base && pe < p->pe_base + p->n_pe_local))
    return plan_fail(SPTRSV_E_ARGUMENT, "pe is local");
  if (bb && pe != p->bblk.my_pe - 1) return SPTRSV_OK;  // the chain reads the previous PE's slot only
  cudaSetDevice(p->device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* ptr = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return plan_fail(SPTRSV_E_CUDA, cudaGetErrorString(e));
  p->opened_peers.push_back(ptr);
  if (bb) {
    p->bblk.prev_slot = reinterpret_cast<const unsigned long long*>(ptr);
    return SPTRSV_OK;
  }
  if (st) {
    p->stencil.host_pe_mbox[pe] = reinterpret_cast<unsigned long long*>(ptr);
    return p->stencil_sync_peers();
  }
  p->host_seg_table[pe] = reinterpret_cast<unsigned long long*>(ptr);
  return p->sync_seg_table();
}

int sptrsv_plan_set_peer_segment(sptrsv_plan* plan, int32_t pe, void* device_ptr) {
  auto* p = reinterpret_cast<DevicePlan*>(plan);
  if (!p || !device_ptr) return plan_fail(SPTRSV_E_ARGUMENT, "null argument");
  if (int rc = p->enable_peer(device_ptr); rc != SPTRSV_OK) return rc;
  if (p->stencil.part) {
    if (pe < 0 || pe >= p->stencil.n_pes) return plan_fail(SPTRSV_E_INVALID_PE, "pe out of range");
    cudaSetDevice(p->device);
    p->stencil.host_pe_mbox[pe] = reinterpret_cast<unsigned long long*>(device_ptr);
    return p->stencil_sync_peers();
  }
  if (p->bblk.part) {
    if (pe < 0 || pe >= p->bblk.n_pes) return plan_fail(SPTRSV_E_INVALID_PE, "pe out of range");
    if (pe == p->bblk.my_pe - 1) p->bblk.prev_slot = reinterpret_cast<const unsigned long long*>(device_ptr);
    return SPTRSV_OK;
  }
  if (pe < 0 || pe >= p->n_pes) return plan_fail(SPTRSV_E_INVALID_PE, "pe out of range");
  cudaSetDevice(p->device);
  p->host_seg_table[pe] = reinterpret_cast<unsigned long long*>(device_ptr);
  return p->sync_seg_table();
}

void* sptrsv_plan_segment(const sptrsv_plan* plan) {
  auto* p = reinterpret_cast<const DevicePlan*>(plan);
  if (p && p->stencil.part) return p->stencil.mbox;
  if (p && p->bblk.part) return p->bblk.slot;
  if (!p || p->local_segs.empty()) return nullptr;
  return p->local_segs[0];
}

int sptrsv_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

}  // extern "C"
