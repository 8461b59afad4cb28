// Register-tile sweep for the float32 tropical fast loop (VIMNMX3 mode) at BASELINE
// config 5's shape (tools; not part of the library).  Times each thread-tile
// shape of semiring_kernel and checks that all give identical bits.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        -o tools/tune_semiring tools/tune_semiring.cu
#include "../paper_0907_0792_b200/csrc/semiring_impl.cuh"
#include "../paper_0907_0792_b200/csrc/tma.cu"

#include <cstdio>

std::atomic<uint64_t> moa::g_launches{0};

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__global__ void fill_tropical(float* p, size_t n, unsigned long long seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long x = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    const float u = (float)(x >> 40) * 0x1.0p-24f;
    p[i] = ((x & 0xff) < 13) ? __int_as_float(0x7f800000) : u * 100.0f;  // ~5% +inf
  }
}
__global__ void count_diff(const float* a, const float* b, size_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    c += (__float_as_int(a[i]) != __float_as_int(b[i]));
  atomicAdd(out, c);
}

void trial_tropical(const moa::Problem& p0, float* out, float* ref, unsigned* special,
                    unsigned long long* cnt) {
  moa::Problem p = p0;
  p.c = out;
  cudaEvent_t s, e;
  CK(cudaEventCreate(&s)); CK(cudaEventCreate(&e));
  CK((moa::tropical_launch<0, 2, 2, false>(p, special)));
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 2; r++) {
    CK(cudaEventRecord(s));
    CK((moa::tropical_launch<0, 2, 2, false>(p, special)));
    CK(cudaEventRecord(e)); CK(cudaEventSynchronize(e));
    float ms; CK(cudaEventElapsedTime(&ms, s, e)); best = ms < best ? ms : best;
  }
  unsigned long long diff = 0;
  CK(cudaMemset(cnt, 0, 8));
  count_diff<<<1184, 256>>>(out, ref, (size_t)p.M * p.N, cnt);
  CK(cudaMemcpy(&diff, cnt, 8, cudaMemcpyDeviceToHost));
  const double pairs = (double)p.M * p.N * p.K;
  printf("{\"kernel\": \"tropical\", \"ms\": %.3f, \"Gpairs_s\": %.1f, \"frac_of_24475\": %.4f, \"bit_diffs\": %llu}\n",
         best, pairs / (best * 1e-3) / 1e9, pairs / (best * 1e-3) / 1e9 / 24475.4, diff);
  fflush(stdout);
}

template <int MINB, int UNR, bool QUAD = false, int BMT = 128>
void trial_tma(const moa::Problem& p0, float* out, float* ref, unsigned* special,
               unsigned long long* cnt) {
  moa::Problem p = p0;
  p.c = out;
  if (!moa::tropical_tma_eligible(p)) { printf("{\"kernel\": \"tropical_tma\", \"eligible\": false}\n"); return; }
  cudaEvent_t s, e;
  CK(cudaEventCreate(&s)); CK(cudaEventCreate(&e));
  CK(cudaMemset(out, 0, (size_t)p.M * p.N * 4));
  CK((moa::tropical_tma_launch<0, 2, 2, false, MINB, UNR, QUAD, BMT>(p, special)));
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 2; r++) {
    CK(cudaEventRecord(s));
    CK((moa::tropical_tma_launch<0, 2, 2, false, MINB, UNR, QUAD, BMT>(p, special)));
    CK(cudaEventRecord(e)); CK(cudaEventSynchronize(e));
    float ms; CK(cudaEventElapsedTime(&ms, s, e)); best = ms < best ? ms : best;
  }
  unsigned long long diff = 0;
  CK(cudaMemset(cnt, 0, 8));
  count_diff<<<1184, 256>>>(out, ref, (size_t)p.M * p.N, cnt);
  CK(cudaMemcpy(&diff, cnt, 8, cudaMemcpyDeviceToHost));
  const double pairs = (double)p.M * p.N * p.K;
  printf("{\"kernel\": \"tropical_tma_bm%d_minb%d_unr%d%s\", \"M\": %ld, \"K\": %ld, \"N\": %ld, \"ms\": %.3f, \"Gpairs_s\": %.1f, \"frac_of_24475\": %.4f, \"bit_diffs\": %llu}\n",
         BMT, MINB, UNR, QUAD ? "_quad" : "", (long)p.M, (long)p.K, (long)p.N, best, pairs / (best * 1e-3) / 1e9, pairs / (best * 1e-3) / 1e9 / 24475.4, diff);
  fflush(stdout);
}

template <int TM, int TN, int MINB>
void trial(const moa::Problem& p0, float* out, float* ref, unsigned* special, unsigned long long* cnt) {
  moa::Problem p = p0;
  p.c = out;
  cudaEvent_t s, e;
  CK(cudaEventCreate(&s)); CK(cudaEventCreate(&e));
  CK((moa::semiring_launch<float, 0, 2, false, -1, TM, TN, MINB>(p, special)));
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 2; r++) {
    CK(cudaEventRecord(s));
    CK((moa::semiring_launch<float, 0, 2, false, -1, TM, TN, MINB>(p, special)));
    CK(cudaEventRecord(e)); CK(cudaEventSynchronize(e));
    float ms; CK(cudaEventElapsedTime(&ms, s, e)); best = ms < best ? ms : best;
  }
  unsigned long long diff = 0;
  if (out != ref) {
    CK(cudaMemset(cnt, 0, 8));
    count_diff<<<1184, 256>>>(out, ref, (size_t)p.M * p.N, cnt);
    CK(cudaMemcpy(&diff, cnt, 8, cudaMemcpyDeviceToHost));
  }
  const double pairs = (double)p.M * p.N * p.K;
  printf("{\"tile\": \"%dx%d_%dcta\", \"ms\": %.3f, \"Gpairs_s\": %.1f, \"frac_of_24475\": %.4f, \"bit_diffs\": %llu}\n",
         TM, TN, MINB, best, pairs / (best * 1e-3) / 1e9, pairs / (best * 1e-3) / 1e9 / 24475.4, diff);
  fflush(stdout);
}

int main() {
  const int64_t n = 16384;
  float *a, *b, *c, *ref;
  unsigned* special;
  unsigned long long* cnt;
  CK(cudaMalloc(&a, n * n * 4)); CK(cudaMalloc(&b, n * n * 4));
  CK(cudaMalloc(&c, n * n * 4)); CK(cudaMalloc(&ref, n * n * 4));
  CK(cudaMalloc(&special, 8)); CK(cudaMalloc(&cnt, 8));
  fill_tropical<<<1184, 256>>>(a, n * n, 11); fill_tropical<<<1184, 256>>>(b, n * n, 12);
  unsigned flags[2] = {moa::S_PINF | moa::S_PZERO, moa::S_PINF | moa::S_PZERO};  // mode 2 data
  CK(cudaMemcpy(special, flags, 8, cudaMemcpyHostToDevice));
  moa::Problem p{MOA_DTYPE_F32, ref, a, b, n, n, n, n, n, n, 0, 2, false, 0};
  trial<8, 8, 2>(p, ref, ref, special, cnt);  // exact loop: the reference bits
  trial_tma<3, 1, true, 64>(p, c, ref, special, cnt);
  trial_tma<2, 1, true, 64>(p, c, ref, special, cnt);
  trial_tma<2, 2, true, 64>(p, c, ref, special, cnt);
  trial_tma<3, 1, true, 64>(p, c, ref, special, cnt);
  // ragged shape: K odd (lone-k tail), M/N not tile multiples
  moa::Problem q{MOA_DTYPE_F32, ref, a, b, 1000, 1001, 1004, 1004, 1004, 1004, 0, 2, false, 0};
  CK((moa::semiring_launch<float, 0, 2, false, -1>(q, special)));
  trial_tma<2, 1>(q, c, ref, special, cnt);
  trial_tma<2, 1, true>(q, c, ref, special, cnt);
  trial_tma<3, 1, true, 64>(q, c, ref, special, cnt);
  moa::Problem q2{MOA_DTYPE_F32, ref, a, b, 1000, 1002, 1004, 1004, 1004, 1004, 0, 2, false, 0};
  CK((moa::semiring_launch<float, 0, 2, false, -1>(q2, special)));
  trial_tma<2, 1, true>(q2, c, ref, special, cnt);
  trial_tma<3, 1, true, 64>(q2, c, ref, special, cnt);
  moa::Problem q3{MOA_DTYPE_F32, ref, a, b, 1000, 1003, 1004, 1004, 1004, 1004, 0, 2, false, 0};
  CK((moa::semiring_launch<float, 0, 2, false, -1>(q3, special)));
  trial_tma<2, 1, true>(q3, c, ref, special, cnt);
  trial_tma<3, 1, true, 64>(q3, c, ref, special, cnt);
  return 0;
}
