// Instruction-mix microbenchmarks for the float32 (add, min) semiring loop:
// which pipe bounds FADD2 + FMNMX3, and what the alternatives cost.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/peaks_minplus tools/peaks_minplus.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

constexpr int NA = 16;
using u64 = unsigned long long;

__device__ __forceinline__ u64 fadd2(u64 a, u64 b) { u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ float lo(u64 x) { return __uint_as_float((unsigned)x); }
__device__ __forceinline__ float hi(u64 x) { return __uint_as_float((unsigned)(x >> 32)); }
__device__ __forceinline__ float min3(float a, float b, float c) { float r; asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
__device__ __forceinline__ float min2(float a, float b) { float r; asm volatile("min.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float fadd(float a, float b) { float r; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ u64 pack(float a, float b) { return ((u64)__float_as_uint(b) << 32) | __float_as_uint(a); }

// mode 0: FMNMX3 only      mode 1: FADD2 only        mode 2: FADD2 + FMNMX3
// mode 3: 2xFADD + FMNMX3  mode 4: FADD2 + 2xFMNMX   mode 5: FMNMX only
// mode 6: FADD only        mode 7: FADD2 + FMNMX3, 2 k-pairs per acc (4 sums -> 2 FMNMX3)
template <int MODE, int ITERS>
__global__ void mix(float* out, float seed) {
  float acc[NA];
  u64 av = pack(seed + threadIdx.x, seed * 2.f), av2 = pack(seed * 3.f, seed + 1.f);
  u64 bb[NA];
#pragma unroll
  for (int i = 0; i < NA; i++) { acc[i] = 1e30f + i; bb[i] = pack(i * 0.25f, i * 0.5f); }
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < NA; i++) {
      if (MODE == 0) { acc[i] = min3(acc[i], lo(bb[i]), hi(av)); }
      if (MODE == 1) { bb[i] = fadd2(bb[i], av); }
      if (MODE == 2) { u64 s = fadd2(av, bb[i]); acc[i] = min3(acc[i], lo(s), hi(s)); }
      if (MODE == 3) { float s0 = fadd(lo(av), lo(bb[i])), s1 = fadd(hi(av), hi(bb[i])); acc[i] = min3(acc[i], s0, s1); }
      if (MODE == 4) { u64 s = fadd2(av, bb[i]); acc[i] = min2(min2(acc[i], lo(s)), hi(s)); }
      if (MODE == 5) { acc[i] = min2(acc[i], lo(bb[i]) + (float)it); }
      if (MODE == 6) { acc[i] = fadd(acc[i], lo(bb[i])); }
      if (MODE == 8) { acc[i] = __uint_as_float(__vimin3_u32(__float_as_uint(acc[i]), (unsigned)bb[i], (unsigned)av)); }
      if (MODE == 9) { u64 s = fadd2(av, bb[i]); acc[i] = __uint_as_float(__vimin3_u32(__float_as_uint(acc[i]), (unsigned)s, (unsigned)(s >> 32))); }
      if (MODE == 10) { u64 s = fadd2(av, bb[i]);
        if (i & 1) acc[i] = __uint_as_float(__vimin3_u32(__float_as_uint(acc[i]), (unsigned)s, (unsigned)(s >> 32)));
        else acc[i] = min3(acc[i], lo(s), hi(s)); }
      if (MODE == 11) { u64 s = fadd2(av, bb[i]);
        if ((i & 3) == 0) acc[i] = __uint_as_float(__vimin3_u32(__float_as_uint(acc[i]), (unsigned)s, (unsigned)(s >> 32)));
        else acc[i] = min3(acc[i], lo(s), hi(s)); }
      if (MODE == 7) { u64 s = fadd2(av, bb[i]); u64 t = fadd2(av2, bb[i]); acc[i] = min3(min3(acc[i], lo(s), hi(s)), lo(t), hi(t)); }
    }
    av += 0x0000000100000001ull;
    av2 += 0x0000000100000001ull;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < NA; i++) s += acc[i] + lo(bb[i]);
  if (s == 12345.f) out[0] = s;
}

// register-tile microkernel: TI x TJ accumulators fed by TI a-pairs and TJ
// b-pairs (the semiring kernel's inner loop without shared memory)
template <int TI, int TJ, int ITERS>
__global__ void tile(float* out, float seed) {
  u64 ap[TI], bp[TJ];
  float acc[TI][TJ];
#pragma unroll
  for (int i = 0; i < TI; i++) ap[i] = pack(seed + i + threadIdx.x, seed * i);
#pragma unroll
  for (int j = 0; j < TJ; j++) bp[j] = pack(j * 0.5f, j * 0.25f + seed);
#pragma unroll
  for (int i = 0; i < TI; i++)
#pragma unroll
    for (int j = 0; j < TJ; j++) acc[i][j] = 1e30f;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int i = 0; i < TI; i++)
#pragma unroll
      for (int j = 0; j < TJ; j++) {
        u64 s = fadd2(ap[i], bp[j]);
        acc[i][j] = __uint_as_float(__vimin3_u32(__float_as_uint(acc[i][j]), (unsigned)s, (unsigned)(s >> 32)));
      }
#pragma unroll
    for (int i = 0; i < TI; i++) ap[i] += 0x0000000100000001ull;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < TI; i++)
#pragma unroll
    for (int j = 0; j < TJ; j++) s += acc[i][j];
  if (s == 12345.f) out[0] = s;
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

template <int MODE>
void run(const char* name, double instr_per_iter, float* d, int sms) {
  constexpr int IT = 4096;
  const int blocks = sms * 2, threads = 1024;
  float ms = timeit([&] { mix<MODE, IT><<<blocks, threads>>>(d, 1.0f); }, 5);
  // warp-instructions of the measured kind per clock per SM at 1965 MHz
  const double warps = blocks * threads / 32.0;
  const double winstr = warps * IT * NA * instr_per_iter;
  printf(", \"%s_winstr_per_clk_sm\": %.3f", name, winstr / (ms * 1e-3) / sms / 1.965e9);
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float* d; CK(cudaMalloc(&d, 1 << 20));
  printf("{\"sms\": %d", sms);
  run<0>("fmnmx3", 1, d, sms);
  run<1>("fadd2", 1, d, sms);
  run<2>("fadd2_fmnmx3_pairs", 1, d, sms);     // per pair-of-pairs: report as (FADD2+FMNMX3) units
  run<3>("2fadd_fmnmx3", 1, d, sms);
  run<4>("fadd2_2fmnmx", 1, d, sms);
  run<5>("fmnmx", 1, d, sms);
  run<6>("fadd", 1, d, sms);
  run<7>("2fadd2_2fmnmx3", 1, d, sms);
  run<8>("vimnmx3", 1, d, sms);
  run<9>("fadd2_vimnmx3_units", 1, d, sms);
  run<10>("fadd2_half_fmnmx3_half_vimnmx3_units", 1, d, sms);
  run<11>("fadd2_3q_fmnmx3_1q_vimnmx3_units", 1, d, sms);
  {
    constexpr int IT = 1024;
    auto tile_run = [&](const char* name, auto kern, int ti, int tj, int blocks, int threads) {
      float ms = timeit([&] { kern<<<blocks, threads>>>(d, 1.0f); }, 5);
      const double pairs = 2.0 * blocks * threads * (double)IT * ti * tj;
      printf(", \"%s_Tpairs\": %.2f", name, pairs / (ms * 1e-3) / 1e12);
    };
    tile_run("tile8x8_16w", tile<8, 8, IT>, 8, 8, sms * 2, 256);
    tile_run("tile8x8_8w", tile<8, 8, IT>, 8, 8, sms * 1, 256);
    tile_run("tile4x8_32w", tile<4, 8, IT>, 4, 8, sms * 4, 256);
    tile_run("tile4x8_16w", tile<4, 8, IT>, 4, 8, sms * 2, 256);
    tile_run("tile4x4_64w", tile<4, 4, IT>, 4, 4, sms * 8, 256);
    tile_run("tile4x4_32w", tile<4, 4, IT>, 4, 4, sms * 4, 256);
    tile_run("tile8x4_32w", tile<8, 4, IT>, 8, 4, sms * 4, 256);
  }
  printf("}\n");
  return 0;
}
