// Lane-chain lockstep executor ("chains"): a host-built static schedule
// streamed through shared memory by TMA bulk copies. Design in
// solve_chains.cu; the slice layout below is shared by the scheduler
// (schedule.cu) and the kernel.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sptrsv {

// Smem ring of recently solved values: D steps x 32 lanes of doubles.
constexpr int kRingSteps = 32;
// Prefetch distance in steps for b and for values from earlier tasks.
constexpr int kPrefetch = 16;
// Inbox (prefetched cross-task) dependencies per row; more go to direct polls.
constexpr int kMaxInbox = 2;
// Dependencies stored inline per row; a longer row continues in the overflow list.
constexpr int kInlineDeps = 16;
// Stream chunks: the unit of one cp.async.bulk copy (bytes, multiple of 16).
constexpr int kChunkBytes = 16384;
constexpr int kChunkBuffers = 4;

// Dependency source codes inside a slice.
constexpr int kSrcSkip = INT32_MIN;  // padding: no dependency in this slot
constexpr int kSrcPrev = -1;         // the lane's previous row (chain predecessor), in a register
constexpr int kSrcInbox0 = -2;       // -2 - m: inbox slot m (prefetched mailbox value), m < kMaxInbox
constexpr int kSrcOverflow = -4;     // the rest of the row is in the overflow list (val = packed start|count)
constexpr int kSrcDirect = -8;       // <= -8: mailbox slot (-8 - code), polled directly
// src >= 0: ring slot (lane * kRingSteps + step % kRingSteps)

// Slice = one lockstep step of one warp task, 32 lanes:
//   int32  width, n_inbox (+8 pad)                     16 B
//   int32  row[32]               (-1: lane idle)       128 B
//   int32  mbox_out[32]          (-1: none)            128 B
//   f64    rdg[32]               1 / l_ii              256 B
//   f64    dg[32]                l_ii (exact only)     256 B
//   int32  src[width][32]                              128 B * width
//   f64    val[width][32]                              256 B * width
//   int32  pf_row[32]            row of this lane kPrefetch steps later (b prefetch)
//   int32  pf_mbox[n_inbox][32]  its inbox mailbox slots
// Sizes are multiples of 16, so slices pack into 16-byte aligned chunks.
__host__ __device__ constexpr int slice_bytes(int width, int n_inbox, bool exact) {
  return 16 + 128 + 128 + 256 + (exact ? 256 : 0) + 384 * width + 128 + 128 * n_inbox;
}

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
  int* ticket = nullptr;
  void release() {
    void* ptrs[] = {stream, chunk_off, chunk_steps, chunk_width, task_chunk, mbox, ovf_src, ovf_val, ticket};
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
    ticket = nullptr;
    ready = false;
  }
  double in_task_fraction() const { return deps_total ? double(deps_in_task) / double(deps_total) : 1.0; }
};

}  // namespace sptrsv
