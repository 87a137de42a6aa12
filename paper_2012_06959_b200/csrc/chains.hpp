// Lane-chain lockstep executor ("chains"): host-built static schedule.
// See solve_chains.cu for the design; this header only carries the device
// buffers the plan owns.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sptrsv {

struct ChainPlan {
  bool ready = false;
  int n_tasks = 0;
  long long n_slices = 0;
  long long n_chunks = 0;
  long long n_mbox = 0;
  long long stream_bytes = 0;
  int max_width = 0;
  double in_task_fraction = 0.0;  // share of dependencies resolved inside a warp task
  // device buffers
  unsigned char* stream = nullptr;   // slices, chunked, 16-byte aligned chunks
  long long* chunk_off = nullptr;    // [n_chunks+1] byte offsets into stream
  int* chunk_steps = nullptr;        // [n_chunks] slices (steps) per chunk
  int* task_chunk = nullptr;         // [n_tasks+1] first chunk of each task
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
};

}  // namespace sptrsv
