// Host-side launch interface shared by the kernel translation units and the
// C ABI (capi.cu).  One Problem is the 2-D view the host plan collapses to:
// C[M x N] (ldc) = fold_k reduce(combine(A[M x K] (lda), B[K x N] (ldb))).
#pragma once

#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

namespace moa {

struct Problem {
  int dtype;  // MOA_DTYPE_*
  void* c;
  const void* a;
  const void* b;
  int64_t M, K, N;
  int64_t lda, ldb, ldc;
  int combine, reduce;
  bool accumulate;
  cudaStream_t stream;
};

// launched-kernel counter (moa_launch_count)
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
// SMs of the current device (cached per device index)
inline int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
  int v = cache[dev].load(std::memory_order_relaxed);
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

// K == 1 (every outer product, plan_outer kernel.py:95-108, and K=1 inner
// products): write-streaming kernel.  outer.cu
cudaError_t launch_outer(const Problem& p);
// K == 0: fill with the reduce identity (the empty fold).  outer.cu
cudaError_t launch_fill(const Problem& p);
// (multiply, add) on float64: FP64 tensor-core (DMMA) kernel.  dmma.cu
cudaError_t launch_dmma(const Problem& p);
// the same product with TMA-staged operands (dmma_tma.cu); bitwise identical
bool dmma_tma_eligible(const Problem& p);
cudaError_t launch_dmma_tma(const Problem& p);
// ... and its 16x32-tile form for problems below one wave of 64x64 tiles
cudaError_t launch_dmma_tma_tiny(const Problem& p);
// everything else: CUDA-core semiring kernel (exact compare-select fold, plus
// the device-checked FMNMX3 fast loop for add/subtract x min/max).  semiring.cu
cudaError_t launch_semiring(const Problem& p);
bool semiring_fast_candidate(int dtype, int combine, int reduce, bool accumulate);

}  // namespace moa
