// DMMA (mma.sync m16n8k4 f64) dependent-chain latency and per-warp issue rate,
// measured with clock64 in one warp (tools; not part of the library).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_dmma_latency tools/mb_dmma_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void chain(double* out, long long* cycles, int iters) {
  double d[CHAINS][4];
  for (int c = 0; c < CHAINS; c++)
    for (int q = 0; q < 4; q++) d[c][q] = threadIdx.x * 1e-3 + c;
  const double a0 = 1.0000001, a1 = 0.9999999, b0 = 1.0000002;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int c = 0; c < CHAINS; c++)
      asm volatile(
          "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5}, {%6}, "
          "{%0, %1, %2, %3};"
          : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
          : "d"(a0), "d"(a1), "d"(b0));
  }
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < CHAINS; c++)
    for (int q = 0; q < 4; q++) s += d[c][q];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cycles = t1 - t0;
}

template <int CHAINS>
void run(double* out, long long* dc) {
  const int iters = 4096;
  chain<CHAINS><<<1, 32>>>(out, dc, iters);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  printf("{\"chains\": %d, \"cycles_per_mma_step\": %.2f, \"cycles_per_mma\": %.2f}\n", CHAINS,
         (double)c / iters, (double)c / iters / CHAINS);
}

int main() {
  double* out;
  long long* dc;
  cudaMalloc(&out, 32 * 8);
  cudaMalloc(&dc, 8);
  run<1>(out, dc); run<1>(out, dc);
  run<2>(out, dc);
  run<4>(out, dc);
  run<8>(out, dc);
  run<16>(out, dc);
  return 0;
}
