// Process-wide host-side resources of the host-buffer executor
// (moa_product_rows_host, host_exec.cu):
//
//  * pooled per-call queue sets (streams + reusable events + small cached
//    device buffers), checked out by one call and returned at its end, so the
//    number of streams is bounded by peak concurrency, not by the number of
//    threads that ever called (the reference's execute_parallel builds a new
//    thread pool per call, parallel.py:37-41);
//  * a private device memory pool per GPU with a bounded release threshold
//    for the large block buffers (other cudaMallocAsync users are unaffected);
//  * page-locked staging slots per GPU plus a small pool of host copy
//    threads, so PAGEABLE host buffers (plain numpy arrays) move at link speed:
//    a copy thread packs rows into a slot while the copy engine drains the
//    previous one (the CUDA driver's own pageable path runs at 11-22 GB/s on
//    B200 hosts, profiles/r02_host_probe.json).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <functional>
#include <vector>

namespace moa::host {

// Run fn(0..n-1) on the copy threads and the calling thread; returns when all
// are done.
void parallel_for(int n, const std::function<void(int)>& fn);
int copy_threads();

struct Queues {
  int device = -1;
  cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
  cudaStream_t s_aux[3] = {nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> events;  // reused across calls
  size_t events_used = 0;
  static constexpr int kCached = 5;
  void* cached[kCached] = {};        // small device buffers kept with the queues
  size_t cached_bytes[kCached] = {};

  cudaEvent_t event(cudaError_t& err);            // a fresh-for-this-call event
  // cached device buffer i (from `pool`, ordered on `st`), or nullptr when
  // `bytes` is too large to keep
  void* cached_buffer(int i, size_t bytes, cudaMemPool_t pool, cudaStream_t st, cudaError_t& err);
};

// Exclusive use of one queue set of `device` (the device must be current).
Queues* checkout(int device, cudaError_t& err);
// Return it; all work the caller enqueued on it must be complete.
void checkin(Queues* q);

// Private stream-ordered pool of `device` (release threshold
// $MOA_HOST_POOL_KEEP_BYTES, default 16 GiB).
cudaMemPool_t device_pool(int device, cudaError_t& err);

// Is host memory at p page-locked (pinned or registered with CUDA)?
bool is_pinned(const void* p);

// The device address of page-locked host memory at p (its mapping into the
// device's address space; the same address under unified addressing), or
// nullptr when p is not page-locked or not mapped.
void* device_view(void* p);

// rows x width bytes, host (pitch hpitch) -> device (pitch dpitch), on `st`.
// Page-locked host memory: one asynchronous 2-D copy.  Pageable: packed
// through staging slots by the copy threads; returns once every chunk is
// issued (the copies complete in stream order on `st`).
cudaError_t h2d(int device, void* dst, size_t dpitch, const void* src, size_t hpitch,
                size_t width, size_t rows, bool pinned, cudaStream_t st);
// device (pitch dpitch) -> host (pitch hpitch), after everything already
// enqueued on `st`.  Page-locked: asynchronous.  Pageable: staged, and
// returns when the host rows hold the data.
cudaError_t d2h(int device, void* dst, size_t hpitch, const void* src, size_t dpitch,
                size_t width, size_t rows, bool pinned, cudaStream_t st);

}  // namespace moa::host
