// The TMA-staged DMMA kernel (csrc/dmma_tma.cu): one tile per CTA vs the
// persistent form (one CTA per resident slot) and 2 / 4 consecutive tiles per
// CTA, each CTA streaming its tiles' k-slabs back to back, across K, CUDA-event times (best of reps) and bit-equality.
// Prints JSON lines.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//   -I paper_0907_0792_b200/csrc -I include -o tools/tune_dmma_persist tools/tune_dmma_persist.cu \
//   paper_0907_0792_b200/csrc/tma.cu -lcuda
#include <cstdio>
#include <array>
#include <cstring>
#include <vector>

#include "dmma_tma.cu"

namespace moa {
std::atomic<uint64_t> g_launches{0};
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

using namespace moa;

__global__ void fill_u(double* x, int64_t n, unsigned seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t h = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 29;
    x[i] = (double)(h >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
}

template <int TPC>
double run(Problem p, int reps) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  CK((dmma_tma_launch<TmaMain, TPC>(p)));
  CK(cudaDeviceSynchronize());
  double best = 1e30;
  for (int r = 0; r < reps; r++) {
    CK(cudaEventRecord(a)); CK((dmma_tma_launch<TmaMain, TPC>(p))); CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); best = ms < best ? ms : best;
  }
  return best;
}

int main(int argc, char** argv) {
  std::vector<std::array<int64_t, 3>> shapes = {{32768, 256, 4096}, {32768, 64, 4096}, {32768, 512, 4096},
                                                {8192, 1024, 8192}, {4096, 4096, 4096}, {2048, 2048, 2048},
                                                {16384, 16384, 16384}};
  const bool acc = argc > 1 && atoi(argv[1]) == 1;
  if (argc > 2) shapes.resize(atoi(argv[2]));  // first n shapes only
  for (auto& s : shapes) {
    const int64_t M = s[0], K = s[1], N = s[2];
    double *a, *b, *c0, *c1;
    CK(cudaMalloc(&a, M * K * 8)); CK(cudaMalloc(&b, K * N * 8));
    CK(cudaMalloc(&c0, M * N * 8)); CK(cudaMalloc(&c1, M * N * 8));
    fill_u<<<1184, 256>>>(a, M * K, 1); fill_u<<<1184, 256>>>(b, K * N, 2);
    fill_u<<<1184, 256>>>(c0, M * N, 3); fill_u<<<1184, 256>>>(c1, M * N, 3);
    Problem p{}; p.dtype = 0; p.a = a; p.b = b; p.M = M; p.N = N; p.K = K;
    p.lda = K; p.ldb = N; p.ldc = N; p.combine = 2; p.reduce = 0; p.stream = 0;
    p.accumulate = acc;
    const int reps = argc > 3 ? atoi(argv[3]) : acc ? 1 : (M * N * K > (int64_t)1 << 40 ? 3 : 20);
    p.c = c0; double t0 = run<1>(p, reps);
    std::vector<double> h0(M * N), h1(M * N);
    CK(cudaMemcpy(h0.data(), c0, M * N * 8, cudaMemcpyDeviceToHost));
    const double fl = 2.0 * M * N * K;
    printf("{\"M\": %lld, \"K\": %lld, \"N\": %lld, \"accumulate\": %d, \"tiles_per_cta\": 1, \"ms\": %.4f, \"TF\": %.2f}\n",
           (long long)M, (long long)K, (long long)N, (int)acc, t0, fl / t0 / 1e9);
    auto other = [&](int tpc, double t1) {
      CK(cudaMemcpy(h1.data(), c1, M * N * 8, cudaMemcpyDeviceToHost));
      int64_t diffs = 0;
      for (int64_t i = 0; i < M * N; i++) diffs += memcmp(&h0[i], &h1[i], 8) != 0;
      printf("{\"M\": %lld, \"K\": %lld, \"N\": %lld, \"accumulate\": %d, \"tiles_per_cta\": %d, \"ms\": %.4f, \"TF\": %.2f, \"bit_diffs\": %lld}\n",
             (long long)M, (long long)K, (long long)N, (int)acc, tpc, t1, fl / t1 / 1e9, (long long)diffs);
      fflush(stdout);
    };
    p.c = c1; CK(cudaMemcpy(c1, c0, 0, cudaMemcpyDeviceToDevice));
    if (acc) fill_u<<<1184, 256>>>(c1, M * N, 3);
    other(0, run<0>(p, reps));
    if (acc) fill_u<<<1184, 256>>>(c1, M * N, 3);
    other(2, run<2>(p, reps));
    if (acc) fill_u<<<1184, 256>>>(c1, M * N, 3);
    other(4, run<4>(p, reps));
    CK(cudaFree(a)); CK(cudaFree(b)); CK(cudaFree(c0)); CK(cudaFree(c1));
  }
  return 0;
}
