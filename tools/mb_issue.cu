// Where does the float32 (add, min) instruction mix stop?  Issue-rate probes
// for the c5 tropical loop (FADD2 on the FMA pipe + VIMNMX3 on the ALU pipe):
// each variant runs NA independent accumulator chains per thread and reports
// warp-instructions issued per clock per SM sub-partition (SMSP) at the
// measured clock, for several warps-per-SMSP counts.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_issue tools/mb_issue.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

using u64 = unsigned long long;
constexpr int NA = 16;

__device__ __forceinline__ u64 fadd2(u64 a, u64 b) {
  u64 r;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float fadd(float a, float b) {
  float r;
  asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ unsigned vmin3(unsigned a, unsigned b, unsigned c) {
  return __vimin3_u32(a, b, c);  // VIMNMX3.U32
}
__device__ __forceinline__ unsigned lop(unsigned a, unsigned b) {
  unsigned r;
  asm volatile("xor.b32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ unsigned imin(unsigned a, unsigned b) {
  unsigned r;
  asm volatile("min.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}

// V: 0 FADD2 | 1 VIMNMX3 | 2 FADD2+VIMNMX3 (the c5 unit) | 3 FADD2+LOP3 |
//    4 2xFADD+VIMNMX3 | 5 FADD | 6 LOP3 | 7 IMNMX (2-input) | 8 FADD2+IMNMX |
//    9 VIMNMX3+LOP3 | 10 FADD2 + VIMNMX3 on independent inputs (no FADD2->min dependency)
template <int V, int ITERS>
__global__ void mix(unsigned* out, unsigned seed) {
  u64 x[NA];
  unsigned acc[NA];
  float f[NA];
  const u64 inc = 0x0000000100000001ull * (seed | 1);
#pragma unroll
  for (int i = 0; i < NA; i++) {
    x[i] = (u64)(seed + i) * 0x9E3779B97F4A7C15ull;
    acc[i] = seed * (i + 3);
    f[i] = __uint_as_float(0x3f800000u + i + threadIdx.x);
  }
  const float fa = __uint_as_float(0x3f000000u + seed);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NA; i++) {
      if (V == 0) x[i] = fadd2(x[i], inc);
      if (V == 1) acc[i] = vmin3(acc[i], (unsigned)x[i], (unsigned)(x[i] >> 32));
      if (V == 2) {
        const u64 s = fadd2(x[i], inc);
        acc[i] = vmin3(acc[i], (unsigned)s, (unsigned)(s >> 32));
      }
      if (V == 3) {
        x[i] = fadd2(x[i], inc);
        acc[i] = lop(acc[i], (unsigned)x[i]);
      }
      if (V == 4) {
        const float s0 = fadd(f[i], fa), s1 = fadd(f[(i + 1) % NA], fa);
        acc[i] = vmin3(acc[i], __float_as_uint(s0), __float_as_uint(s1));
      }
      if (V == 5) f[i] = fadd(f[i], fa);
      if (V == 6) acc[i] = lop(acc[i], (unsigned)x[i]);
      if (V == 7) acc[i] = imin(acc[i], (unsigned)x[i] + it);
      if (V == 8) {
        x[i] = fadd2(x[i], inc);
        acc[i] = imin(acc[i], (unsigned)x[i]);
      }
      if (V == 9) {
        acc[i] = vmin3(acc[i], (unsigned)x[i], (unsigned)(x[i] >> 32));
        x[i] = (x[i] & 0xffffffff00000000ull) | lop((unsigned)x[i], acc[i]);
      }
      if (V == 10) {
        x[i] = fadd2(x[i], inc);
        acc[i] = vmin3(acc[i], (unsigned)x[(i + 7) % NA], (unsigned)(x[(i + 11) % NA] >> 32));
      }
    }
  }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < NA; i++) s += acc[i] + (unsigned)x[i] + __float_as_uint(f[i]);
  if (s == 0x12345u) out[0] = s;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  int sms, khz;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0));
  unsigned* d;
  CK(cudaMalloc(&d, 1024));
  const char* names[] = {"fadd2", "vimnmx3", "fadd2+vimnmx3", "fadd2+lop3", "2fadd+vimnmx3",
                         "fadd", "lop3", "imnmx", "fadd2+imnmx", "vimnmx3+lop3",
                         "fadd2+vimnmx3_indep"};
  const int per_iter[] = {1, 1, 2, 2, 3, 1, 1, 1, 2, 2, 2};  // warp-instructions per (it, i)
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"units\": \"warp-instr per clock per SMSP\"", sms,
         khz / 1e3);
  constexpr int IT = 2048;
  auto run = [&](int v, auto kern) {
    printf(", \"%s\": {", names[v]);
    for (int wps : {1, 2, 3, 4, 8, 16}) {  // warps per SMSP
      const int threads = 128 * wps > 1024 ? 1024 : 128 * wps;
      const int blocks = sms * (128 * wps / threads);
      float ms = timeit([&] { kern<<<blocks, threads>>>(d, 7u); });
      const double winstr = (double)blocks * threads / 32 * IT * NA * per_iter[v];
      const double per_smsp_clk = winstr / (ms * 1e-3) / (sms * 4.0) / (khz * 1e3);
      printf("%s\"w%d\": %.3f", wps == 1 ? "" : ", ", wps, per_smsp_clk);
    }
    printf("}");
  };
  run(0, mix<0, IT>);
  run(1, mix<1, IT>);
  run(2, mix<2, IT>);
  run(3, mix<3, IT>);
  run(4, mix<4, IT>);
  run(5, mix<5, IT>);
  run(6, mix<6, IT>);
  run(7, mix<7, IT>);
  run(8, mix<8, IT>);
  run(9, mix<9, IT>);
  run(10, mix<10, IT>);
  printf("}\n");
  return 0;
}
