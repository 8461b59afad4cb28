// Variants of the float32 tropical TMA kernel (csrc/tropical.cuh) on the c5
// data distribution (uniform [0, 100) with 5% +inf), timed with CUDA events
// and checked bit for bit against the production variant.  Prints JSON lines.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//   -I paper_0907_0792_b200/csrc -I include -o tools/tune_tropical tools/tune_tropical.cu \
//   paper_0907_0792_b200/csrc/tma.cu paper_0907_0792_b200/csrc/host_runtime.cu
// Usage: tools/tune_tropical [N=16384] [reps=3] [which=0: all variants, 1: bm128 only, 2: int32 DPX bm64 vs bm128, 3: unrolled quad loop, 4: scalar-FADD form]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "semiring_impl.cuh"

namespace moa {
std::atomic<uint64_t> g_launches{0};
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

using namespace moa;

__global__ void fill_c5(float* x, int64_t n, unsigned seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    h ^= h >> 31;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 29;
    const float u = (float)(h >> 40) * (1.0f / 16777216.0f);
    x[i] = ((h & 0xff) < 13) ? __int_as_float(0x7f800000) : u * 100.0f;
  }
}

template <typename F>
double time_ms(F f, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(f());
  CK(cudaDeviceSynchronize());
  double best = 1e30;
  for (int r = 0; r < reps; r++) {
    CK(cudaEventRecord(a));
    CK(f());
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  return best;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 16384;
  const int reps = argc > 2 ? atoi(argv[2]) : 3;
  float *a, *b, *c0, *c1;
  unsigned* special;
  CK(cudaMalloc(&a, n * n * 4));
  CK(cudaMalloc(&b, n * n * 4));
  CK(cudaMalloc(&c0, n * n * 4));
  CK(cudaMalloc(&c1, n * n * 4));
  CK(cudaMalloc(&special, 16));
  fill_c5<<<1184, 256>>>(a, n * n, 1);
  fill_c5<<<1184, 256>>>(b, n * n, 2);
  CK(cudaMemset(special, 0, 16));
  launch_scan<float>(a, n, n, n, special, 0);
  launch_scan<float>(b, n, n, n, special + 1, 0);
  CK(cudaDeviceSynchronize());
  Problem p{};
  p.dtype = 1;
  p.a = a;
  p.b = b;
  p.M = p.N = p.K = n;
  p.lda = p.ldb = p.ldc = n;
  p.combine = C_ADD;
  p.reduce = R_MIN;
  p.accumulate = false;
  p.stream = 0;
  const double pairs = (double)n * n * n;
  auto report = [&](const char* name, float* c, double ms) {
    std::vector<unsigned> h0(n * n), h1(n * n);
    CK(cudaMemcpy(h0.data(), c0, n * n * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h1.data(), c, n * n * 4, cudaMemcpyDeviceToHost));
    int64_t diffs = 0;
    for (int64_t i = 0; i < n * n; i++) diffs += h0[i] != h1[i];
    printf("{\"kernel\": \"%s\", \"N\": %lld, \"ms\": %.3f, \"Gpairs_s\": %.1f, \"bit_diffs\": %lld}\n",
           name, (long long)n, ms, pairs / ms / 1e6, (long long)diffs);
    fflush(stdout);
  };
  if (argc > 3 && atoi(argv[3]) == 2) {  // int32 (add, min) on the DPX route: bm64 vs bm128
    p.dtype = 2;
    p.c = c0;
    report("int32_bm64_quad_refill1", c0, time_ms([&] { return tropical_tma_launch<C_ADD, R_MIN, 3, false, 3, 1, true, 64, 1>(p, nullptr); }, reps));
    p.c = c1;
    CK(cudaMemset(c1, 0, n * n * 4));
    report("int32_bm128_quad_refill1", c1, time_ms([&] { return tropical_tma_launch<C_ADD, R_MIN, 3, false, 2, 1, true, 128, 1>(p, nullptr); }, reps));
    return 0;
  }
  p.c = c0;
  double ms = time_ms([&] { return tropical_tma_launch<C_ADD, R_MIN, 2, false, 3, 1, true, 64, 1>(p, special); }, reps);
  report("production_bm64_quad_refill1", c0, ms);
  p.c = c1;
  auto variant = [&](const char* name, auto launch) {
    CK(cudaMemset(c1, 0, n * n * 4));
    report(name, c1, time_ms(launch, reps));
  };
  const int which = argc > 3 ? atoi(argv[3]) : 0;
  if (which == 0 || which == 1)
    variant("bm128_quad_refill1", [&] { return tropical_tma_launch<C_ADD, R_MIN, 2, false, 2, 1, true, 128, 1, 0>(p, special); });
  if (which == 4) {  // scalar-FADD form on both tile shapes (ncu target)
    variant("bm128_quad_form2", [&] { return tropical_tma_launch<C_ADD, R_MIN, 2, false, 2, 1, true, 128, 1, 2>(p, special); });
    variant("bm64_quad_form2", [&] { return tropical_tma_launch<C_ADD, R_MIN, 2, false, 3, 1, true, 64, 1, 2>(p, special); });
  }
  if (which == 3) {
    variant("bm128_quad_unroll2", [&] { return tropical_tma_launch<C_ADD, R_MIN, 2, false, 2, 2, true, 128, 1, 0>(p, special); });
    variant("bm64_quad_unroll2", [&] { return tropical_tma_launch<C_ADD, R_MIN, 2, false, 3, 2, true, 64, 1, 0>(p, special); });
  }
  if (which == 0) {
    variant("bm64_quad_refill1_form1_swapped", [&] { return tropical_tma_launch<C_ADD, R_MIN, 2, false, 3, 1, true, 64, 1, 1>(p, special); });
    variant("bm64_quad_refill1_form2_scalar_fadd", [&] { return tropical_tma_launch<C_ADD, R_MIN, 2, false, 3, 1, true, 64, 1, 2>(p, special); });
    variant("bm128_quad_refill1_form1_swapped", [&] { return tropical_tma_launch<C_ADD, R_MIN, 2, false, 2, 1, true, 128, 1, 1>(p, special); });
  }
  return 0;
}
