// Microbenchmarks that pin the roofline denominators MEASURED_PEAKS.json lacks:
// FP64 DMMA (mma.sync f64 -> DMMA.8x8x4), FP64 DFMA, the f32 (add,min) semiring
// instruction mix (FADD2 + FMNMX3) and write-only HBM streaming.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks tools/peaks.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <int ITERS>
__global__ void dmma_m8n8k4(double* out, double seed) {
  double a = seed + threadIdx.x, b = seed * 0.5 + threadIdx.x;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; i++) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; i++) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int ITERS>
__global__ void dmma_m16n8k16(double* out, double seed) {
  double a[8], b[4];
  for (int i = 0; i < 8; i++) a[i] = seed + i + threadIdx.x;
  for (int i = 0; i < 4; i++) b[i] = seed * 0.5 + i;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) c[i][j] = 0.0;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int i = 0; i < 4; i++) for (int j = 0; j < 4; j++) s += c[i][j];
  if (s == 12345.0) out[0] = s;
}

template <int ITERS>
__global__ void dfma_loop(double* out, double seed) {
  double x[16];
  double m = seed * 1e-9, ad = seed;
#pragma unroll
  for (int i = 0; i < 16; i++) x[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) x[i] = fma(x[i], m, ad);
  }
  double s = 0; for (int i = 0; i < 16; i++) s += x[i];
  if (s == 12345.0) out[0] = s;
}

// (add,min) f32 fast mix: per 2 contraction steps one FADD2 and one 3-input min.
template <int ITERS>
__global__ void minplus_f32x2(float* out, float seed) {
  float acc[16];
  float ax = seed + threadIdx.x, ay = seed * 2.f;
#pragma unroll
  for (int i = 0; i < 16; i++) acc[i] = 1e30f;
  unsigned long long bb[16];
#pragma unroll
  for (int i = 0; i < 16; i++) {
    float lo = i * 0.25f, hi = i * 0.5f;
    bb[i] = ((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo);
  }
  unsigned long long av = ((unsigned long long)__float_as_uint(ay) << 32) | __float_as_uint(ax);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) {
      unsigned long long s;
      asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(s) : "l"(av), "l"(bb[i]));
      float s0 = __uint_as_float((unsigned)s), s1 = __uint_as_float((unsigned)(s >> 32));
      asm volatile("min.f32 %0, %0, %1, %2;" : "+f"(acc[i]) : "f"(s0), "f"(s1));
    }
    av += 0x0000000100000001ull;
  }
  float s = 0; for (int i = 0; i < 16; i++) s += acc[i];
  if (s == 12345.f) out[0] = s;
}

// scalar mix: FADD + FMNMX per pair
template <int ITERS>
__global__ void minplus_f32(float* out, float seed) {
  float acc[16], b[16];
  float a = seed + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 16; i++) { acc[i] = 1e30f; b[i] = i * 0.25f; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) {
      float s;
      asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(s) : "f"(a), "f"(b[i]));
      asm volatile("min.f32 %0, %0, %1;" : "+f"(acc[i]) : "f"(s));
    }
    a += 1.0f;
  }
  float s = 0; for (int i = 0; i < 16; i++) s += acc[i];
  if (s == 12345.f) out[0] = s;
}

// reference-exact compare/select fold: acc = (acc < s) ? acc : s
template <int ITERS>
__global__ void minplus_f32_sel(float* out, float seed) {
  float acc[16], b[16];
  float a = seed + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 16; i++) { acc[i] = 1e30f; b[i] = i * 0.25f; }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < 16; i++) {
      float s;
      asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(s) : "f"(a), "f"(b[i]));
      asm volatile("{ .reg .pred p; setp.lt.f32 p, %0, %1; selp.f32 %0, %0, %1, p; }" : "+f"(acc[i]) : "f"(s));
    }
    a += 1.0f;
  }
  float s = 0; for (int i = 0; i < 16; i++) s += acc[i];
  if (s == 12345.f) out[0] = s;
}

__global__ void write_v4(double* __restrict__ p, size_t n4, double v) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    double* q = p + 4 * i;
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(q), "d"(v), "d"(v), "d"(v), "d"(v) : "memory");
  }
}
__global__ void write_v2(double* __restrict__ p, size_t n2, double v) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += stride) {
    double2 w = make_double2(v, v);
    __stcs(reinterpret_cast<double2*>(p) + i, w);
  }
}

template <typename F>
float timeit(F f, int reps) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; r++) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("{\"sms\": %d, \"clock_khz_attr\": %d", sms, clk);
  double* d; CK(cudaMalloc(&d, 1 << 20));
  const int IT = 4096;
  for (int wpb : {4, 8, 16}) {
    int blocks = sms * 2, threads = 32 * wpb;
    float ms = timeit([&] { dmma_m8n8k4<IT><<<blocks, threads>>>(d, 1.0); }, 5);
    double flop = 2.0 * blocks * wpb * (double)IT * 8 * 256;
    printf(", \"dmma_m8n8k4_w%d_tflops\": %.2f", wpb, flop / ms / 1e9);
  }
  for (int wpb : {4, 8, 16}) {
    int blocks = sms * 2, threads = 32 * wpb;
    float ms = timeit([&] { dmma_m16n8k16<IT / 8><<<blocks, threads>>>(d, 1.0); }, 5);
    double flop = 2.0 * blocks * wpb * (double)(IT / 8) * 4 * 2048;
    printf(", \"dmma_m16n8k16_w%d_tflops\": %.2f", wpb, flop / ms / 1e9);
  }
  for (int wpb : {8, 16, 32}) {
    int blocks = sms * 2, threads = 32 * wpb;
    float ms = timeit([&] { dfma_loop<IT><<<blocks, threads>>>(d, 1.0); }, 5);
    double flop = 2.0 * blocks * threads * (double)IT * 16;
    printf(", \"dfma_w%d_tflops\": %.2f", wpb, flop / ms / 1e9);
  }
  for (int wpb : {8, 16, 32}) {
    int blocks = sms * 2, threads = 32 * wpb;
    float ms = timeit([&] { minplus_f32x2<IT><<<blocks, threads>>>((float*)d, 1.0f); }, 5);
    double pairs = 2.0 * blocks * threads * (double)IT * 16;
    printf(", \"minplus_fadd2_fmnmx3_w%d_Tpairs\": %.2f", wpb, pairs / ms / 1e9);
    ms = timeit([&] { minplus_f32<IT><<<blocks, threads>>>((float*)d, 1.0f); }, 5);
    pairs = 1.0 * blocks * threads * (double)IT * 16;
    printf(", \"minplus_fadd_fmnmx_w%d_Tpairs\": %.2f", wpb, pairs / ms / 1e9);
    ms = timeit([&] { minplus_f32_sel<IT><<<blocks, threads>>>((float*)d, 1.0f); }, 5);
    printf(", \"minplus_fadd_setp_selp_w%d_Tpairs\": %.2f", wpb, pairs / ms / 1e9);
  }
  size_t bytes = 1ull << 30;
  double* w; CK(cudaMalloc(&w, bytes));
  for (int mult : {1, 2, 4, 8}) {
    int blocks = sms * mult;
    float ms = timeit([&] { write_v4<<<blocks, 512>>>(w, bytes / 32, 1.0); }, 10);
    printf(", \"write_v4_cs_b%dx_GBs\": %.1f", mult, bytes / ms / 1e6);
    ms = timeit([&] { write_v2<<<blocks, 512>>>(w, bytes / 16, 1.0); }, 10);
    printf(", \"write_v2_cs_b%dx_GBs\": %.1f", mult, bytes / ms / 1e6);
  }
  float ms = timeit([&] { CK(cudaMemsetAsync(w, 0, bytes)); }, 10);
  printf(", \"memset_GBs\": %.1f", bytes / ms / 1e6);
  printf("}\n");
  return 0;
}
