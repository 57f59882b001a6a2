// host_io.hpp — host<->device transfers of caller-owned (pageable) arrays for
// the stateless C-ABI calls.
//
// The reference API takes and returns plain host arrays (std::vector / span,
// SURVEY §8(b)), so every im_update_volume / im_deform call moves the mesh
// across PCIe.  A pageable cudaMemcpy runs at ~17 GB/s on the B200 box
// (driver-internal single-threaded staging); here the copy is split into
// ~1 MiB chunks that a small host thread pool stages through pinned buffers,
// each chunk's DMA issued as soon as its staging copy lands, so host memcpy
// bandwidth (several threads) and the ~53 GB/s pinned DMA overlap.  The
// staging pass also gives callers a free look at the bytes (the planar
// z == 0 check of im_update_volume).  Downloads mirror it: chunked DMA into
// pinned memory with an event per chunk, workers copying (and widening
// uint32 node ids to size_t) into the caller's arrays as chunks complete.
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "runtime.hpp"

namespace imb {

// Fixed set of worker threads; run() executes fn(0..n-1) on the workers and
// the calling thread and returns when all tasks finished (first exception
// rethrown).
class HostPool {
 public:
  explicit HostPool(int threads);
  ~HostPool();
  HostPool(const HostPool&) = delete;
  HostPool& operator=(const HostPool&) = delete;
  int size() const { return (int)th_.size() + 1; }
  void run(int n, const std::function<void(int)>& fn);

 private:
  void worker();
  void drain(const std::function<void(int)>& fn, int n);
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0;
  std::atomic<int> next_{0};
  int finished_ = 0;
  unsigned long long gen_ = 0;
  bool stop_ = false;
  std::exception_ptr err_;
};

struct H2DJob {
  void* dst;        // device
  const void* src;  // host (pageable or pinned)
  size_t bytes;
};

// Per-chunk hook on the staged bytes: (job, host chunk pointer, byte offset in
// the job, length).  Chunks of a job start at multiples of `align` bytes.
using ChunkScan = std::function<void(int, const unsigned char*, size_t, size_t)>;

// Uploads all jobs on `stream` (default ctx.stream; asynchronously w.r.t. the
// device: the copies are enqueued when this returns).  align: chunk alignment
// in bytes.
void staged_h2d(Context& ctx, const H2DJob* jobs, int n_jobs, size_t align = 192,
                const ChunkScan& scan = {}, cudaStream_t stream = nullptr);

// page-locked (cudaHostAlloc / cudaHostRegister) host memory
bool host_is_pinned(const void* p);
HostPool& host_pool(Context& ctx);
// the context's pinned download staging buffer (grow-only; callers must not
// overlap two users)
unsigned char* pinned_out(Context& ctx, size_t bytes);

struct D2HJob {
  const void* src;  // device
  void* dst;        // host
  size_t count;     // elements
  int src_size;     // bytes per device element
  bool widen_u32;   // device uint32 -> host uint64 (src_size must be 4)
};

// Downloads all jobs (enqueued after the work already on ctx.stream) and
// returns when the host arrays are filled.
void staged_d2h(Context& ctx, const D2HJob* jobs, int n_jobs);

}  // namespace imb
