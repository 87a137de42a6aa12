// Lane-chain lockstep executor ("chains"): a host-built static schedule
// streamed through shared memory by TMA bulk copies. Design in
// solve_chains.cu; the slice layout and the shared-memory map below are shared
// by the scheduler (schedule.cu), which bakes shared-memory byte offsets into
// the stream, and the kernel.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sptrsv {

// Ring of recently solved values: kRingSteps steps x 32 lanes of doubles.
constexpr int kRingSteps = 64;
// Prefetch distance in steps for b and for values of earlier tasks.
constexpr int kPrefetch = 16;
// Inbox (prefetched cross-task) dependencies per row; more become direct polls.
constexpr int kMaxInbox = 2;
// Dependencies stored inline per row; a longer row continues in the overflow list.
constexpr int kInlineDeps = 16;
// Stream chunks: the unit of one cp.async.bulk copy (bytes, multiple of 16).
constexpr int kChunkBytes = 16384;
constexpr int kChunkBuffers = 4;

// Shared-memory map of one CTA (one warp).
constexpr int kSmemChunks = 0;
constexpr int kSmemRing = kSmemChunks + kChunkBuffers * kChunkBytes;
constexpr int kSmemInbox = kSmemRing + kRingSteps * 32 * 8;   // 16-byte slots (cp.async.cg)
constexpr int kSmemB = kSmemInbox + kMaxInbox * kPrefetch * 32 * 16;
constexpr int kSmemSlot = kSmemB + kPrefetch * 32 * 8;        // mailbox id of each inbox slot
constexpr int kSmemBars = kSmemSlot + kMaxInbox * kPrefetch * 32 * 4;
constexpr int kSmemTotal = kSmemBars + 8 * kChunkBuffers;

__host__ __device__ constexpr int ring_offset(int step, int lane) { return kSmemRing + ((step % kRingSteps) * 32 + lane) * 8; }
__host__ __device__ constexpr int inbox_index(int m, int step, int lane) { return (m * kPrefetch + step % kPrefetch) * 32 + lane; }
__host__ __device__ constexpr int inbox_offset(int m, int step, int lane) { return kSmemInbox + inbox_index(m, step, lane) * 16; }

// Dependency source codes (int32 per dependency slot):
//   >= 0   shared-memory byte offset of the value (ring slot or inbox slot)
//   -1     padding, no dependency
//   -2     the rest of the row is in the overflow list (val = packed start|count)
//   <= -8  mailbox slot (-8 - code), polled directly from global memory
constexpr int kSrcSkip = -1;
constexpr int kSrcOverflow = -2;
constexpr int kSrcDirect = -8;

// Slice = one lockstep step of one warp task, 32 lanes; uniform width W inside
// a chunk, so the kernel computes every address from (chunk base, W):
//   int32  row[32]       (-1: lane idle)                     128 B
//   int32  mbox_out[32]  (-1: nobody reads it from a mailbox) 128 B
//   int32  pf_row[32]    row of this lane kPrefetch steps later (b prefetch)   128 B
//   int32  pf_mbox[M][32] its inbox mailbox slots                             128 B * M
//   f64    rdg[32]       1 / l_ii                             256 B
//   f64    dg[32]        l_ii (exact only)                    256 B
//   int32  src[W][32]                                         128 B * W
//   f64    val[W][32]                                         256 B * W
// Every array is a multiple of 128 bytes, so slices pack into 16-byte aligned
// chunks and every f64 array is 8-byte aligned.
__host__ __device__ constexpr int slice_bytes(int width, int n_inbox, bool exact) {
  return 384 + 128 * n_inbox + 256 + (exact ? 256 : 0) + 384 * width;
}
struct SliceGeom {
  int sb, pfm, rdg, dg, src, val;
  __host__ __device__ SliceGeom(int w, int n_inbox, bool exact) {
    sb = slice_bytes(w, n_inbox, exact);
    pfm = 384;
    rdg = 384 + 128 * n_inbox;
    dg = rdg + 256;
    src = rdg + 256 + (exact ? 256 : 0);
    val = src + 128 * w;
  }
};

struct ChainPlan {
  bool ready = false;
  bool exact = true;
  int n_tasks = 0;
  int lanes = 32;
  int n_inbox = 0;
  long long n_slices = 0;
  long long n_chunks = 0;
  long long n_mbox = 0;
  long long n_overflow = 0;
  long long stream_bytes = 0;
  int max_width = 0;
  long long deps_total = 0, deps_in_task = 0, deps_ring = 0, deps_reg = 0, deps_mbox = 0, deps_inbox = 0;
  long long max_task_steps = 0;
  double schedule_ms = 0.0;
  // device buffers
  unsigned char* stream = nullptr;     // slices, chunked
  long long* chunk_off = nullptr;      // [n_chunks+1] byte offsets into stream
  int* chunk_steps = nullptr;          // [n_chunks] slices per chunk
  int* chunk_width = nullptr;          // [n_chunks] dependency slots per slice (uniform in a chunk)
  int* task_chunk = nullptr;           // [n_tasks+1] first chunk of each task
  unsigned long long* mbox = nullptr;  // [n_mbox] cross-task mailboxes (value-is-flag, 16-byte slots)
  int* ovf_src = nullptr;              // overflow dependency lists (rows wider than kInlineDeps)
  double* ovf_val = nullptr;
  void release() {
    void* ptrs[] = {stream, chunk_off, chunk_steps, chunk_width, task_chunk, mbox, ovf_src, ovf_val};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    stream = nullptr;
    chunk_off = nullptr;
    chunk_steps = nullptr;
    chunk_width = nullptr;
    task_chunk = nullptr;
    mbox = nullptr;
    ovf_src = nullptr;
    ovf_val = nullptr;
    ready = false;
  }
  double in_task_fraction() const { return deps_total ? double(deps_in_task) / double(deps_total) : 1.0; }
};

}  // namespace sptrsv
