// Small-problem K1 comparison (tools; not part of the library): the cp.async
// tiny/small tiles of dmma.cu against the TMA 16x32 tiles of dmma_tma.cu on
// problems below one wave of 64x64 tiles, L2 flushed before every timed launch,
// with a bit comparison against the cp.async tiny tiles.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -I include -o tools/tune_dmma_tiny tools/tune_dmma_tiny.cu
#include "../paper_0907_0792_b200/csrc/dmma.cu"
#include "../paper_0907_0792_b200/csrc/dmma_tma.cu"
#include "../paper_0907_0792_b200/csrc/tma.cu"

#include <cstdio>
#include <functional>

std::atomic<uint64_t> moa::g_launches{0};

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__global__ void fill_uniform(double* p, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    p[i] = (double)(x >> 11) * 0x1.0p-53 * 2.0 - 1.0;
  }
}
__global__ void count_diff(const double* a, const double* b, size_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    c += (__double_as_longlong(a[i]) != __double_as_longlong(b[i]));
  atomicAdd(out, c);
}

struct Shape { int64_t M, K, N; };
__global__ void empty_kernel(double* p) { if (p == nullptr && threadIdx.x == 1024) p[0] = 0; }

int main() {
  const Shape shapes[] = {{256, 256, 256}, {128, 256, 256}, {256, 1000, 256}, {300, 301, 702},
                          {512, 512, 512}, {1024, 256, 512}, {64, 4096, 64}, {256, 2048, 256}};
  const size_t cap = 8 << 20;  // doubles per operand
  double *A, *B, *C, *Cref, *flush;
  unsigned long long* cnt;
  CK(cudaMalloc(&A, cap * 8)); CK(cudaMalloc(&B, cap * 8)); CK(cudaMalloc(&C, cap * 8));
  CK(cudaMalloc(&Cref, cap * 8)); CK(cudaMalloc(&flush, 256 << 20)); CK(cudaMalloc(&cnt, 8));
  fill_uniform<<<1184, 256>>>(A, cap, 11); fill_uniform<<<1184, 256>>>(B, cap, 12);
  cudaEvent_t s, e;
  CK(cudaEventCreate(&s)); CK(cudaEventCreate(&e));
  for (const Shape& sh : shapes) {
    moa::Problem p{MOA_DTYPE_F64, Cref, A, B, sh.M, sh.K, sh.N, sh.K, sh.N, sh.N, 2, 0, false, 0};
    CK(moa::dmma_dispatch<moa::CfgTiny>(p));
    CK(cudaDeviceSynchronize());
    p.c = C;
    const bool tma_ok = moa::dmma_tma_eligible(p);
    auto run = [&](const char* name, std::function<cudaError_t()> fn, bool warm = false) {
      CK(fn()); CK(cudaDeviceSynchronize());
      float best = 1e30f, sum = 0.f;
      const int reps = 30;
      for (int r = 0; r < reps; r++) {
        if (!warm) CK(cudaMemsetAsync(flush, r & 1, 256 << 20));
        CK(cudaEventRecord(s)); CK(fn()); CK(cudaEventRecord(e));
        CK(cudaEventSynchronize(e));
        float ms; CK(cudaEventElapsedTime(&ms, s, e)); best = ms < best ? ms : best; sum += ms;
      }
      CK(cudaMemset(cnt, 0, 8));
      count_diff<<<592, 256>>>(C, Cref, (size_t)sh.M * sh.N, cnt);
      unsigned long long d; CK(cudaMemcpy(&d, cnt, 8, cudaMemcpyDeviceToHost));
      CK(cudaMemset(C, 0, (size_t)sh.M * sh.N * 8));
      printf("{\"kernel\": \"%s\", \"M\": %lld, \"K\": %lld, \"N\": %lld, \"us_best\": %.2f, "
             "\"us_mean\": %.2f, \"TFLOPs_best\": %.3f, \"bit_diffs\": %llu, \"l2\": \"%s\"}\n", name,
             (long long)sh.M, (long long)sh.K, (long long)sh.N, best * 1e3, sum / reps * 1e3,
             2.0 * sh.M * sh.N * sh.K / (best * 1e-3) / 1e12, d, warm ? "warm" : "flushed");
      fflush(stdout);
    };
    run("cpasync_tiny_16x32", [&] { return moa::dmma_dispatch<moa::CfgTiny>(p); });
    run("cpasync_small_32x32", [&] { return moa::dmma_dispatch<moa::CfgSmall>(p); });
    if (tma_ok) {
      run("tma_tiny_16x32_s8", [&] { return moa::dmma_tiny_tma_launch<8>(p); });
      run("tma_tiny_16x32_s8", [&] { return moa::dmma_tiny_tma_launch<8>(p); }, true);
      run("tma_tiny_16x32_s4", [&] { return moa::dmma_tiny_tma_launch<4>(p); });
      run("tma_main_64x64", [&] { return moa::launch_dmma_tma(p); });
    }
    run("cpasync_tiny_16x32", [&] { return moa::dmma_dispatch<moa::CfgTiny>(p); }, true);
    if (&sh == &shapes[0]) {
      run("empty_kernel_128x128", [&] { empty_kernel<<<128, 128>>>(C); return cudaGetLastError(); });
      run("empty_kernel_128x128", [&] { empty_kernel<<<128, 128>>>(C); return cudaGetLastError(); }, true);
    }
  }
  return 0;
}
