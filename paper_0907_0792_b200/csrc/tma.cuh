// TMA + mbarrier helpers shared by the TMA-staged kernels (dmma_tma.cu,
// tropical.cuh): 2-D bulk tensor loads that complete on a shared-memory
// mbarrier (SASS UTMALDG / SYNCS.*).  Host side: tensor-map encoding through
// the driver entry point (tma.cu), so the library needs no -lcuda.
#pragma once

#include <cuda.h>
#include <cstdint>

namespace moa {

// row-major rows x cols matrix of elem_bytes elements, row stride ld
// (elements), box box_rows x box_cols, optional 128-byte swizzle; false when
// the driver entry point is missing or the encoder rejects the layout
bool make_tensor_map_2d(CUtensorMap* map, const void* ptr, int elem_bytes, int64_t rows,
                        int64_t cols, int64_t ld, int box_rows, int box_cols, bool swizzle128);
bool tensor_maps_available();

namespace tma {

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// A consumer's release of a stage that TMA (the async proxy) will overwrite:
// every lane orders its shared-memory reads of the stage before the async
// proxy's next writes (fence.proxy.async), the warp converges, and one lane
// arrives on the stage's `empty` barrier.  Without the fence ptxas may hoist the
// arrive above the slab's last fragment loads, so the producer's refill can
// land before they read — seen as intermittent corruption of a few warps'
// results (tests/test_gpu_parity.py::test_dmma_accumulate_launches_repeat_bitwise).
__device__ __forceinline__ void release_stage(uint64_t* empty_bar, int lane) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) mbar_arrive(empty_bar);
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// box at (c0 = column, c1 = row) of the map into dst, completing on bar
__device__ __forceinline__ void load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar))
      : "memory");
}
// first 1024-byte aligned byte of a dynamic shared buffer (the 128-byte
// swizzle needs it); derived by offset so loads stay in the shared space
__device__ __forceinline__ unsigned char* align1k(unsigned char* raw) {
  return raw + ((1024u - (smem_addr(raw) & 1023u)) & 1023u);
}

}  // namespace tma
}  // namespace moa
