// Lane-chain lockstep executor ("chains"): a host-built static schedule
// streamed through shared memory by TMA bulk copies. Design in
// solve_chains.cu; slice layout below is shared by the scheduler
// (schedule.cu) and the kernel.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sptrsv {

// Smem ring of recently solved values: D steps x 32 lanes of doubles.
constexpr int kRingSteps = 32;
// Stream chunks: the unit of one cp.async.bulk copy (bytes, multiple of 16).
constexpr int kChunkBytes = 16384;
constexpr int kChunkBuffers = 4;
constexpr int kMaxChunkSteps = 16;  // b prefetch area per chunk buffer
// Dependency source codes inside a slice.
constexpr int kSrcSkip = INT32_MIN;  // padding: no dependency in this slot
constexpr int kSrcPrev = -1;         // the lane's previous row (chain predecessor), in a register
// src >= 0: ring slot (lane * kRingSteps + step % kRingSteps)
// src <= -2: mailbox slot (-2 - src), polled until not kNotReady

// Slice = one lockstep step of one warp task, 32 lanes:
//   int32  width                 (+12 bytes pad)   16 B
//   int32  row[32]               (-1: lane idle)   128 B
//   int32  mbox_out[32]          (-1: none)        128 B
//   f64    rdg[32]               1 / l_ii          256 B
//   f64    dg[32]                l_ii (exact only) 256 B
//   int32  src[width][32]                          128 B * width
//   f64    val[width][32]                          256 B * width
// Sizes are multiples of 16, so slices pack into 16-byte aligned chunks.
__host__ __device__ constexpr int slice_bytes(int width, bool exact) {
  return 16 + 128 + 128 + 256 + (exact ? 256 : 0) + 384 * width;
}

struct ChainPlan {
  bool ready = false;
  bool exact = true;
  int n_tasks = 0;
  int lanes = 32;
  long long n_slices = 0;
  long long n_chunks = 0;
  long long n_mbox = 0;
  long long stream_bytes = 0;
  int max_width = 0;
  long long deps_total = 0, deps_in_task = 0, deps_ring = 0, deps_reg = 0, deps_mbox = 0;
  long long max_task_steps = 0;
  double schedule_ms = 0.0;
  // device buffers
  unsigned char* stream = nullptr;     // slices, chunked
  long long* chunk_off = nullptr;      // [n_chunks+1] byte offsets into stream
  int* chunk_steps = nullptr;          // [n_chunks] slices per chunk
  int* task_chunk = nullptr;           // [n_tasks+1] first chunk of each task
  unsigned long long* mbox = nullptr;  // [n_mbox] cross-task mailboxes (value-is-flag)
  int* ticket = nullptr;
  void release() {
    void* ptrs[] = {stream, chunk_off, chunk_steps, task_chunk, mbox, ticket};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    stream = nullptr;
    chunk_off = nullptr;
    chunk_steps = nullptr;
    task_chunk = nullptr;
    mbox = nullptr;
    ticket = nullptr;
    ready = false;
  }
  double in_task_fraction() const { return deps_total ? double(deps_in_task) / double(deps_total) : 1.0; }
};

}  // namespace sptrsv
