// Tile-shape sweep for the FP64 DMMA kernel (tools; not part of the library).
// Includes the kernel translation unit so every DmmaCfg can be instantiated;
// times each config on the BASELINE shapes and checks that every config gives
// bit-identical results (the determinism argument in dmma.cu).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -I include -o tools/tune_dmma tools/tune_dmma.cu
#include "../paper_0907_0792_b200/csrc/dmma.cu"
#include "../paper_0907_0792_b200/csrc/dmma_tma.cu"
#include "../paper_0907_0792_b200/csrc/tma.cu"

#include <cstdio>
#include <vector>

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

struct Shape { const char* name; int64_t M, K, N; };

template <class Cfg>
double run_cfg(const moa::Problem& p, int reps) {
  cudaEvent_t s, e;
  CK(cudaEventCreate(&s)); CK(cudaEventCreate(&e));
  CK(moa::dmma_dispatch<Cfg>(p));
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    CK(cudaEventRecord(s)); CK(moa::dmma_dispatch<Cfg>(p)); CK(cudaEventRecord(e));
    CK(cudaEventSynchronize(e));
    float ms; CK(cudaEventElapsedTime(&ms, s, e)); best = ms < best ? ms : best;
  }
  return best;
}

template <class Cfg>
void trial_tma(const char* name, const Shape& sh, double* A, double* B, double* C, double* Cref,
               unsigned long long* d_cnt) {
  moa::Problem p{MOA_DTYPE_F64, C, A, B, sh.M, sh.K, sh.N, sh.K, sh.N, sh.N, 2, 0, false, 0};
  if (!moa::dmma_tma_eligible(p)) { printf("{\"cfg\": \"tma\", \"eligible\": false}\n"); return; }
  cudaEvent_t s, e;
  CK(cudaEventCreate(&s)); CK(cudaEventCreate(&e));
  CK(moa::dmma_tma_launch<Cfg>(p));
  CK(cudaDeviceSynchronize());
  const int reps = sh.M * sh.N * sh.K > (1ll << 36) ? 2 : 10;
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    CK(cudaEventRecord(s)); CK(moa::dmma_tma_launch<Cfg>(p)); CK(cudaEventRecord(e));
    CK(cudaEventSynchronize(e));
    float ms; CK(cudaEventElapsedTime(&ms, s, e)); best = ms < best ? ms : best;
  }
  unsigned long long diff = 0;
  CK(cudaMemset(d_cnt, 0, 8));
  count_diff<<<1184, 256>>>(C, Cref, (size_t)sh.M * sh.N, d_cnt);
  CK(cudaMemcpy(&diff, d_cnt, 8, cudaMemcpyDeviceToHost));
  const double tf = 2.0 * sh.M * sh.N * sh.K / (best * 1e-3) / 1e12;
  printf("{\"shape\": \"%s\", \"cfg\": \"tma_%s\", \"ms\": %.4f, \"tflops\": %.2f, "
         "\"frac_of_36.96\": %.4f, \"bit_diffs_vs_first\": %llu}\n", sh.name, name, best, tf, tf / 36.96, diff);
  fflush(stdout);
}

template <class Cfg>
void trial(const char* cname, const Shape& sh, double* A, double* B, double* C, double* Cref,
           unsigned long long* d_cnt, bool first) {
  moa::Problem p{MOA_DTYPE_F64, first ? Cref : C, A, B, sh.M, sh.K, sh.N, sh.K, sh.N, sh.N,
                 2, 0, false, 0};
  const int reps = sh.M * sh.N * sh.K > (1ll << 36) ? 2 : 10;
  double ms = run_cfg<Cfg>(p, reps);
  unsigned long long diff = 0;
  if (!first) {
    CK(cudaMemset(d_cnt, 0, 8));
    count_diff<<<1184, 256>>>(C, Cref, (size_t)sh.M * sh.N, d_cnt);
    CK(cudaMemcpy(&diff, d_cnt, 8, cudaMemcpyDeviceToHost));
  }
  const double tf = 2.0 * sh.M * sh.N * sh.K / (ms * 1e-3) / 1e12;
  printf("{\"shape\": \"%s\", \"cfg\": \"%s\", \"threads\": %d, \"smem\": %zu, \"ms\": %.4f, "
         "\"tflops\": %.2f, \"frac_of_36.96\": %.4f, \"bit_diffs_vs_first\": %llu}\n",
         sh.name, cname, Cfg::THREADS, Cfg::SMEM, ms, tf, tf / 36.96, diff);
  fflush(stdout);
}

int main() {
  std::vector<Shape> shapes = {{"c1", 256, 256, 256}, {"m1k", 1024, 1024, 1024},
                               {"c3", 32768, 256, 4096}, {"c4", 16384, 16384, 16384}};
  for (const Shape& sh : shapes) {
    double *A, *B, *C, *Cref;
    unsigned long long* d_cnt;
    CK(cudaMalloc(&A, sh.M * sh.K * 8)); CK(cudaMalloc(&B, sh.K * sh.N * 8));
    CK(cudaMalloc(&C, sh.M * sh.N * 8)); CK(cudaMalloc(&Cref, sh.M * sh.N * 8));
    CK(cudaMalloc(&d_cnt, 8));
    fill_uniform<<<1184, 256>>>(A, sh.M * sh.K, 1); fill_uniform<<<1184, 256>>>(B, sh.K * sh.N, 2);
    using namespace moa;
    // reference bits: the cp.async large tile; every other config must match them
    trial<DmmaCfg<64, 128, 32, 32, 4, 16, 2, false, 16>>("cp_64x128_s4_2cta_g16", sh, A, B, C, Cref, d_cnt, true);
    trial<DmmaCfg<64, 64, 32, 32, 3, 16, 3>>("cp_64x64_medium", sh, A, B, C, Cref, d_cnt, false);
    trial<DmmaCfg<32, 32, 16, 16, 3, 32, 1>>("cp_32x32_small", sh, A, B, C, Cref, d_cnt, false);
    trial<DmmaCfg<16, 32, 16, 8, 8, 32, 1>>("cp_16x32_tiny_s8", sh, A, B, C, Cref, d_cnt, false);
    trial_tma<moa::TmaMain>("64x64_s4_3cta", sh, A, B, C, Cref, d_cnt);
    trial_tma<moa::TmaCfg<64, 128, 32, 32, 4, 2, 16>>("64x128_s4_2cta", sh, A, B, C, Cref, d_cnt);
    CK(cudaFree(A)); CK(cudaFree(B)); CK(cudaFree(C)); CK(cudaFree(Cref)); CK(cudaFree(d_cnt));
  }
  return 0;
}
