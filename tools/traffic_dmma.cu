// One c4-sized launch per rasterisation group size, for
//   ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
// (tools; not part of the library).
#include "../paper_0907_0792_b200/csrc/dmma.cu"

#include <cstdio>

std::atomic<uint64_t> moa::g_launches{0};

__global__ void fill(double* p, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = (double)(((i + 1) * 0x9E3779B97F4A7C15ull ^ seed) >> 11) * 0x1.0p-53;
}

int main() {
  const int64_t n = 16384;
  double *a, *b, *c;
  cudaMalloc(&a, n * n * 8); cudaMalloc(&b, n * n * 8); cudaMalloc(&c, n * n * 8);
  fill<<<1184, 256>>>(a, n * n, 1); fill<<<1184, 256>>>(b, n * n, 2);
  moa::Problem p{MOA_DTYPE_F64, c, a, b, n, n, n, n, n, n, 2, 0, false, 0};
  using namespace moa;
  dmma_dispatch<DmmaCfg<64, 128, 32, 32, 4, 16, 2, false, 8>>(p);
  dmma_dispatch<DmmaCfg<64, 128, 32, 32, 4, 16, 2, false, 16>>(p);
  dmma_dispatch<DmmaCfg<64, 128, 32, 32, 4, 16, 2, false, 32>>(p);
  cudaError_t e = cudaDeviceSynchronize();
  printf("traffic_dmma: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
