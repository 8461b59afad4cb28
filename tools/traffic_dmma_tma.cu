// c4-sized launches of the TMA DMMA kernel, one per raster group size GM, for
//   ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
// plus an event-timed best-of-3 per GM and a bit comparison against GM=8
// (tools; not part of the library).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -I include -o tools/traffic_dmma_tma tools/traffic_dmma_tma.cu -lcuda
#include "../paper_0907_0792_b200/csrc/dmma_tma.cu"
#include "../paper_0907_0792_b200/csrc/tma.cu"

#include <cstdio>
#include <cstdlib>

std::atomic<uint64_t> moa::g_launches{0};

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__global__ void fill(double* p, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = (double)(((i + 1) * 0x9E3779B97F4A7C15ull ^ seed) >> 11) * 0x1.0p-53;
}
__global__ void count_diff(const double* a, const double* b, size_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    c += (__double_as_longlong(a[i]) != __double_as_longlong(b[i]));
  atomicAdd(out, c);
}

template <int GM>
void trial(moa::Problem p, const double* cref, unsigned long long* cnt, int reps) {
  using Cfg = moa::TmaCfg<64, 64, 32, 32, 4, 3, GM>;
  cudaEvent_t s, e;
  CK(cudaEventCreate(&s)); CK(cudaEventCreate(&e));
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    CK(cudaEventRecord(s)); CK(moa::dmma_tma_launch<Cfg>(p)); CK(cudaEventRecord(e));
    CK(cudaEventSynchronize(e));
    float ms; CK(cudaEventElapsedTime(&ms, s, e)); best = ms < best ? ms : best;
  }
  unsigned long long diff = 0;
  if (cref) {
    CK(cudaMemset(cnt, 0, 8));
    count_diff<<<1184, 256>>>(static_cast<const double*>(p.c), cref, (size_t)p.M * p.N, cnt);
    CK(cudaMemcpy(&diff, cnt, 8, cudaMemcpyDeviceToHost));
  }
  const double tf = 2.0 * p.M * p.N * p.K / (best * 1e-3) / 1e12;
  printf("{\"GM\": %d, \"M\": %lld, \"ms\": %.3f, \"TFLOPs\": %.2f, \"bit_diffs_vs_gm8\": %llu}\n", GM,
         (long long)p.M, best, tf, diff);
  fflush(stdout);
}

int main(int argc, char** argv) {
  const int64_t n = 16384;
  const int reps = argc > 1 ? atoi(argv[1]) : 3;
  double *a, *b, *c, *cref;
  unsigned long long* cnt;
  CK(cudaMalloc(&a, n * n * 8)); CK(cudaMalloc(&b, n * n * 8));
  CK(cudaMalloc(&c, n * n * 8)); CK(cudaMalloc(&cref, n * n * 8)); CK(cudaMalloc(&cnt, 8));
  fill<<<1184, 256>>>(a, n * n, 1); fill<<<1184, 256>>>(b, n * n, 2);
  moa::Problem pr{MOA_DTYPE_F64, cref, a, b, n, n, n, n, n, n, 2, 0, false, 0};
  CK((moa::dmma_tma_launch<moa::TmaCfg<64, 64, 32, 32, 4, 3, 8>>(pr)));
  CK(cudaDeviceSynchronize());
  moa::Problem p = pr;
  p.c = c;
  trial<8>(p, cref, cnt, reps);
  trial<16>(p, cref, cnt, reps);
  trial<24>(p, cref, cnt, reps);
  trial<32>(p, cref, cnt, reps);
  trial<48>(p, cref, cnt, reps);
  trial<64>(p, cref, cnt, reps);
  CK(cudaDeviceSynchronize());
  return 0;
}
