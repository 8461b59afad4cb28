// Register-tile / occupancy sweep of the exact semiring kernel for float64
// routes (tools; not part of the library).  Checks identical bits across tiles.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -o tools/tune_semiring_f64 tools/tune_semiring_f64.cu
#include "../paper_0907_0792_b200/csrc/semiring_impl.cuh"
#include "../paper_0907_0792_b200/csrc/tma.cu"

#include <cstdio>

std::atomic<uint64_t> moa::g_launches{0};

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__global__ void fill(double* p, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    p[i] = (double)(x >> 11) * 0x1.0p-53 * 100.0 - 30.0;
  }
}
__global__ void count_diff(const double* a, const double* b, size_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    c += (__double_as_longlong(a[i]) != __double_as_longlong(b[i]));
  atomicAdd(out, c);
}

template <int C, int R, int TM, int TN, int MINB>
void trial(const char* route, const moa::Problem& p0, double* out, double* ref, unsigned long long* cnt,
           bool is_ref) {
  moa::Problem p = p0;
  p.c = is_ref ? ref : out;
  p.combine = C; p.reduce = R;
  cudaEvent_t s, e;
  CK(cudaEventCreate(&s)); CK(cudaEventCreate(&e));
  CK((moa::semiring_launch<double, C, R, false, -1, TM, TN, MINB>(p, nullptr)));
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 3; r++) {
    CK(cudaEventRecord(s));
    CK((moa::semiring_launch<double, C, R, false, -1, TM, TN, MINB>(p, nullptr)));
    CK(cudaEventRecord(e)); CK(cudaEventSynchronize(e));
    float ms; CK(cudaEventElapsedTime(&ms, s, e)); best = ms < best ? ms : best;
  }
  unsigned long long diff = 0;
  if (!is_ref) {
    CK(cudaMemset(cnt, 0, 8));
    count_diff<<<1184, 256>>>(out, ref, (size_t)p.M * p.N, cnt);
    CK(cudaMemcpy(&diff, cnt, 8, cudaMemcpyDeviceToHost));
  }
  const double pairs = (double)p.M * p.N * p.K;
  printf("{\"route\": \"%s\", \"tile\": \"%dx%d_minb%d\", \"ms\": %.3f, \"Gpairs_s\": %.1f, \"bit_diffs\": %llu}\n",
         route, TM, TN, MINB, best, pairs / (best * 1e-3) / 1e9, diff);
  fflush(stdout);
}

template <int C, int R>
void sweep(const char* route, const moa::Problem& p, double* c, double* ref, unsigned long long* cnt) {
  trial<C, R, 8, 8, 1>(route, p, c, ref, cnt, true);
  trial<C, R, 8, 4, 2>(route, p, c, ref, cnt, false);
  trial<C, R, 4, 8, 2>(route, p, c, ref, cnt, false);
  trial<C, R, 4, 4, 3>(route, p, c, ref, cnt, false);
  trial<C, R, 4, 4, 4>(route, p, c, ref, cnt, false);
}

int main() {
  const int64_t n = 4096;
  double *a, *b, *c, *ref;
  unsigned long long* cnt;
  CK(cudaMalloc(&a, n * n * 8)); CK(cudaMalloc(&b, n * n * 8));
  CK(cudaMalloc(&c, n * n * 8)); CK(cudaMalloc(&ref, n * n * 8)); CK(cudaMalloc(&cnt, 8));
  fill<<<1184, 256>>>(a, n * n, 1); fill<<<1184, 256>>>(b, n * n, 2);
  moa::Problem p{MOA_DTYPE_F64, ref, a, b, n, n, n, n, n, n, 0, 0, false, 0};
  sweep<2, 0>("mul_add_exact", p, c, ref, cnt);
  sweep<0, 0>("add_add", p, c, ref, cnt);
  sweep<0, 2>("add_min", p, c, ref, cnt);
  sweep<2, 3>("mul_max", p, c, ref, cnt);
  sweep<4, 2>("min_min", p, c, ref, cnt);
  return 0;
}
