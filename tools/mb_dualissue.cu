// Issue-slot probe for the c5 tropical loop: how many issue cycles does one
// FADD2 (packed float32 add, FMA pipe) take, and does it pair with an ALU-pipe
// instruction (VIMNMX3 / LOP3 / IMNMX) in the same cycles?
// Each variant runs NA independent register chains per thread (no loads, no
// dependencies between the paired instructions), so the only limits are issue
// and pipe throughput.  Reports warp-instructions per clock per SM
// sub-partition (SMSP) at the device's max clock, for several warps per SMSP.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_dualissue tools/mb_dualissue.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

using u64 = unsigned long long;
constexpr int NA = 8;

__device__ __forceinline__ void fadd2(u64& x, u64 c) {
  asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(c));
}
__device__ __forceinline__ void fadd2_bcast(u64& x, float a) {  // FADD2 R, R.F32x2, R.F32
  asm volatile("{\n\t.reg .b64 t;\n\tmov.b64 t, {%1, %1};\n\tadd.rn.f32x2 %0, %0, t;\n\t}" : "+l"(x) : "f"(a));
}
__device__ __forceinline__ void fadd(float& x, float c) { asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x) : "f"(c)); }
__device__ __forceinline__ void ffma(float& x, float c) { asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(x) : "f"(c)); }
__device__ __forceinline__ void lop3(unsigned& x, unsigned c) { asm volatile("xor.b32 %0, %0, %1;" : "+r"(x) : "r"(c)); }
__device__ __forceinline__ void vmin3(unsigned& x, unsigned p, unsigned q) {
  x = __vimin3_u32(x, p, q);  // VIMNMX3.U32; the empty asm keeps each one live
  asm volatile("" : "+r"(x));
}
__device__ __forceinline__ void imin(unsigned& x, unsigned p) { asm volatile("min.u32 %0, %0, %1;" : "+r"(x) : "r"(p)); }

// V: 0 FADD2 | 1 FADD2 (scalar broadcast operand) | 2 LOP3 | 3 VIMNMX3 | 4 FADD
//    5 FADD2 + LOP3 | 6 FADD2 + VIMNMX3 | 7 FADD + VIMNMX3 | 8 FADD + LOP3
//    9 FADD2 + IMNMX | 10 FADD2(bcast) + VIMNMX3 | 11 FFMA | 12 FFMA + VIMNMX3
//    13 2 FADD + VIMNMX3 | 14 FADD2 + 2 LOP3 | 15 FADD2 + 2 FADD + 2 VIMNMX3
//    16 FADD2 + FADD + VIMNMX3 | 17 2 FADD2 + 2 FADD + 3 VIMNMX3
template <int V, int ITERS>
__global__ void mix(unsigned* out, unsigned seed) {
  u64 x[NA];
  float f[NA];
  unsigned acc[NA];
  const u64 inc = 0x3f8000003f800000ull + seed;
  const float fa = __uint_as_float(0x3f000000u + seed);
  const unsigned p = seed * 7 + 1, q = seed * 13 + 5;
#pragma unroll
  for (int i = 0; i < NA; i++) {
    x[i] = (u64)(seed + i) * 0x9E3779B97F4A7C15ull;
    f[i] = __uint_as_float(0x3f800000u + i + threadIdx.x);
    acc[i] = seed * (i + 3) + threadIdx.x;
  }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NA; i++) {
      if (V == 0) fadd2(x[i], inc);
      if (V == 1) fadd2_bcast(x[i], fa);
      if (V == 2) lop3(acc[i], acc[(i + 1) % NA]);
      if (V == 3) vmin3(acc[i], p, q);
      if (V == 4) fadd(f[i], fa);
      if (V == 5) { fadd2(x[i], inc); lop3(acc[i], acc[(i + 1) % NA]); }
      if (V == 6) { fadd2(x[i], inc); vmin3(acc[i], p, q); }
      if (V == 7) { fadd(f[i], fa); vmin3(acc[i], p, q); }
      if (V == 8) { fadd(f[i], fa); lop3(acc[i], acc[(i + 1) % NA]); }
      if (V == 9) { fadd2(x[i], inc); imin(acc[i], p); asm volatile("" : "+r"(acc[i])); }
      if (V == 10) { fadd2_bcast(x[i], fa); vmin3(acc[i], p, q); }
      if (V == 11) ffma(f[i], fa);
      if (V == 12) { ffma(f[i], fa); vmin3(acc[i], p, q); }
      if (V == 13) { fadd(f[i], fa); fadd(f[(i + 1) % NA], fa); vmin3(acc[i], p, q); }
      if (V == 15) {  // 1 FADD2 + 2 FADD (128 adds) + 2 VIMNMX3 per (it, i): 2 c5 units in 5 instructions
        fadd2(x[i], inc); fadd(f[i], fa); fadd(f[(i + 1) % NA], fa);
        vmin3(acc[i], p, q); vmin3(acc[(i + 1) % NA], q, p);
      }
      if (V == 16) {  // 1 FADD2 + 1 FADD + 1 VIMNMX3 (no pairing constraint): FMA/ALU mix probe
        fadd2(x[i], inc); fadd(f[i], fa); vmin3(acc[i], p, q);
      }
      if (V == 17) {  // 2 FADD2 + 2 FADD + 3 VIMNMX3: 3 units in 7 instructions
        fadd2(x[i], inc); fadd(f[i], fa); vmin3(acc[i], p, q); fadd2(x[(i + 1) % NA], inc);
        fadd(f[(i + 1) % NA], fa); vmin3(acc[(i + 1) % NA], q, p); vmin3(acc[(i + 2) % NA], p, p);
      }
      if (V == 14) { fadd2(x[i], inc); lop3(acc[i], acc[(i + 1) % NA]); lop3(acc[(i + 3) % NA], acc[(i + 5) % NA]); }
    }
  }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < NA; i++) s += acc[i] + (unsigned)x[i] + (unsigned)(x[i] >> 32) + __float_as_uint(f[i]);
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
  const char* names[] = {"fadd2", "fadd2_bcast", "lop3", "vimnmx3", "fadd",
                         "fadd2+lop3", "fadd2+vimnmx3", "fadd+vimnmx3", "fadd+lop3", "fadd2+imnmx",
                         "fadd2_bcast+vimnmx3", "ffma", "ffma+vimnmx3", "2fadd+vimnmx3", "fadd2+2lop3",
                         "fadd2+2fadd+2vimnmx3", "fadd2+fadd+vimnmx3", "2fadd2+2fadd+3vimnmx3"};
  const int per_iter[] = {1, 1, 1, 1, 1, 2, 2, 2, 2, 2, 2, 1, 2, 3, 3, 5, 3, 7};  // warp-instructions per (it, i)
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"units\": \"warp-instr per clock per SMSP\"", sms,
         khz / 1e3);
  constexpr int IT = 4096;
  auto run = [&](int v, auto kern) {
    printf(", \"%s\": {", names[v]);
    for (int wps : {2, 4, 8, 16}) {  // warps per SMSP
      const int threads = 128 * wps > 1024 ? 1024 : 128 * wps;
      const int blocks = sms * (128 * wps / threads);
      float ms = timeit([&] { kern<<<blocks, threads>>>(d, 7u); });
      const double winstr = (double)blocks * threads / 32 * IT * NA * per_iter[v];
      const double per_smsp_clk = winstr / (ms * 1e-3) / (sms * 4.0) / (khz * 1e3);
      printf("%s\"w%d\": %.3f", wps == 2 ? "" : ", ", wps, per_smsp_clk);
    }
    printf("}");
    fflush(stdout);
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
  run(11, mix<11, IT>);
  run(12, mix<12, IT>);
  run(13, mix<13, IT>);
  run(14, mix<14, IT>);
  run(15, mix<15, IT>);
  run(16, mix<16, IT>);
  run(17, mix<17, IT>);
  printf("}\n");
  return 0;
}
