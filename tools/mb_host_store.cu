// Kernel stores into page-locked (mapped) host memory: which store form gets
// closest to the copy engine's ~56 GB/s device->host rate?  Each variant
// writes the same bytes (a 2-D tile layout like the DMMA epilogues': tiles of
// 16 rows x 32 doubles, 256-byte row runs) into host memory:
//   0: per-thread 16-byte stores straight from registers (the production
//      DMMA tiny epilogue: 64-byte runs per warp instruction)
//   1: tile staged in shared memory, then 16 threads per 256-byte row
//   2: tile staged in shared memory, then one cp.async.bulk (TMA bulk copy)
//      per 256-byte row, issued by one thread
//   3: 32-byte streaming stores, whole rows per warp (the outer kernel's form)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_host_store tools/mb_host_store.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int TM = 16, TN = 32;  // tile rows x doubles

template <int V>
__global__ void __launch_bounds__(128) store_tiles(double* __restrict__ c, int M, int N) {
  __shared__ __align__(128) double tile[TM][TN];
  const int tiles_n = N / TN;
  const int m0 = (blockIdx.x / tiles_n) * TM, n0 = (blockIdx.x % tiles_n) * TN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  // the values a DMMA warp would hold: rows g, g+8; columns 8*warp + 2t, +1
  double v[4];
#pragma unroll
  for (int q = 0; q < 4; q++) v[q] = (double)(m0 + g + 8 * (q >> 1)) * 1e-3 + n0 + 8 * warp + 2 * t + (q & 1);
  if (V == 0) {
#pragma unroll
    for (int h = 0; h < 2; h++)
      *reinterpret_cast<double2*>(c + (size_t)(m0 + g + 8 * h) * N + n0 + 8 * warp + 2 * t) =
          make_double2(v[2 * h], v[2 * h + 1]);
    return;
  }
#pragma unroll
  for (int h = 0; h < 2; h++) {
    tile[g + 8 * h][8 * warp + 2 * t] = v[2 * h];
    tile[g + 8 * h][8 * warp + 2 * t + 1] = v[2 * h + 1];
  }
  __syncthreads();
  if (V == 1) {
    // 16 threads x 16 B per row: one warp instruction covers two rows
#pragma unroll
    for (int i = 0; i < 2; i++) {
      const int r = (tid >> 4) + 8 * i, cc = (tid & 15) * 2;
      *reinterpret_cast<double2*>(c + (size_t)(m0 + r) * N + n0 + cc) =
          *reinterpret_cast<const double2*>(&tile[r][cc]);
    }
  } else if (V == 2) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid < TM) {
      const unsigned src = (unsigned)__cvta_generic_to_shared(&tile[tid][0]);
      double* dst = c + (size_t)(m0 + tid) * N + n0;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   :: "l"(dst), "r"(src), "n"(TN * 8) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else if (V == 3) {
    // 32-byte stores: 8 threads per 256-byte row, 4 rows per warp instruction
#pragma unroll
    for (int i = 0; i < 1; i++) {
      const int r = tid >> 3, cc = (tid & 7) * 4;
      const double4 x = *reinterpret_cast<const double4*>(&tile[r][cc]);
      double* d = c + (size_t)(m0 + r) * N + n0 + cc;
      asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};"
                   :: "l"(d), "d"(x.x), "d"(x.y), "d"(x.z), "d"(x.w) : "memory");
    }
  }
}

template <int V>
double run(double* c, int M, int N, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  const int blocks = (M / TM) * (N / TN);
  store_tiles<V><<<blocks, 128>>>(c, M, N);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    CK(cudaEventRecord(a));
    store_tiles<V><<<blocks, 128>>>(c, M, N);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  printf("{\"unit\": \"GB/s into page-locked host memory (best of reps, CUDA events)\"");
  for (int M : {256, 4096, 65536}) {
    const int N = M == 65536 ? 2048 : 256 * (M == 4096 ? 8 : 1);
    const size_t bytes = (size_t)M * N * 8;
    double* h;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
    double* dev = nullptr;
    CK(cudaHostGetDevicePointer(&dev, h, 0));
    const int reps = M == 65536 ? 3 : 50;
    const double t0 = run<0>(dev, M, N, reps), t1 = run<1>(dev, M, N, reps);
    const double t2 = run<2>(dev, M, N, reps), t3 = run<3>(dev, M, N, reps);
    double* d;
    CK(cudaMalloc(&d, bytes));
    const double td = run<0>(d, M, N, reps);
    printf(", \"%dx%d (%zu KiB)\": {\"regs_16B\": %.1f, \"smem_rows_16B\": %.1f, \"tma_bulk_rows\": %.1f, "
           "\"smem_rows_32B_cs\": %.1f, \"device_memory_regs_16B_us\": %.2f, \"regs_16B_us\": %.2f}",
           M, N, bytes >> 10, bytes / t0 / 1e6, bytes / t1 / 1e6, bytes / t2 / 1e6, bytes / t3 / 1e6,
           td * 1e3, t0 * 1e3);
    // check the TMA variant wrote the right values
    const int r = M / 2 + 3, col = N / 2 + 5;
    const double want = (double)r * 1e-3 + col;
    if (h[(size_t)r * N + col] != want) printf(", \"check\": \"mismatch %g vs %g\"", h[(size_t)r * N + col], want);
    CK(cudaFree(d));
    CK(cudaFreeHost(h));
  }
  printf("}\n");
  return 0;
}
