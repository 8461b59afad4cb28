// Issue rate of the DPX add-then-min (VIADDMNMX) for the int32 tropical loop:
// acc[j] = min(a + b[j], acc[j]) with a shared (operand-reuse candidate) vs a
// different a per instruction, and the 3-input VIMNMX3 for comparison
// (tools; not part of the library).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_viaddmnmx tools/mb_viaddmnmx.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int NA = 16;

template <int MODE, int ITERS>
__global__ void mix(int* out, int seed) {
  __shared__ int av[64];
  if (threadIdx.x < 64) av[threadIdx.x] = seed * threadIdx.x - 1000;
  __syncthreads();
  int acc[NA], b[NA], a[NA];
#pragma unroll
  for (int i = 0; i < NA; i++) { acc[i] = 1 << 30; b[i] = seed * i + threadIdx.x; a[i] = seed + i; }
  int a0 = 0;
  for (int it = 0; it < ITERS; it++) {
    a0 = av[it & 63];  // opaque to the compiler: no algebra across iterations
#pragma unroll
    for (int i = 0; i < NA; i++) a[i] = av[(it + i) & 63];
#pragma unroll
    for (int i = 0; i < NA; i++) {
      if (MODE == 0) acc[i] = __viaddmin_s32(a0, b[i], acc[i]);       // shared a
      if (MODE == 1) acc[i] = __viaddmin_s32(a[i], b[i], acc[i]);     // distinct a
      if (MODE == 2) acc[i] = __vimin3_s32(acc[i], b[i], a0);         // 3-input min
      if (MODE == 3) acc[i] = min(acc[i], b[i] + a0);                 // IADD + IMNMX
    }
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < NA; i++) s += acc[i];
  if (s == 12345) out[0] = s;
}

template <typename F>
float timeit(F f, int reps) {
  cudaEvent_t x, y; CK(cudaEventCreate(&x)); CK(cudaEventCreate(&y));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    CK(cudaEventRecord(x)); f(); CK(cudaEventRecord(y)); CK(cudaEventSynchronize(y));
    float ms; CK(cudaEventElapsedTime(&ms, x, y)); if (ms < best) best = ms;
  }
  return best;
}

template <int MODE>
void run(const char* name, int* d, int sms, int warps_per_sm) {
  constexpr int IT = 4096;
  const int threads = 256, blocks = sms * warps_per_sm * 32 / threads;
  float ms = timeit([&] { mix<MODE, IT><<<blocks, threads>>>(d, 7); }, 5);
  const double winstr = (double)blocks * threads / 32 * IT * NA;
  printf(", \"%s_w%d_winstr_per_clk_sm\": %.3f", name, warps_per_sm,
         winstr / (ms * 1e-3) / sms / 1.965e9);
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int* d; CK(cudaMalloc(&d, 1 << 20));
  printf("{\"sms\": %d", sms);
  for (int w : {16, 32}) {
    run<0>("viaddmnmx_shared_a", d, sms, w);
    run<1>("viaddmnmx_distinct_a", d, sms, w);
    run<2>("vimnmx3", d, sms, w);
    run<3>("iadd_imnmx_pairs", d, sms, w);
  }
  printf("}\n");
  return 0;
}
