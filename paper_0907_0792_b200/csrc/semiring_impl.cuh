// K2: the CUDA-core semiring kernel — every (combine, reduce) pair other than
// the tensor-core (multiply, add) float64 path.
//
// Reference loop (_ckernel.pyx:55-72, generic; :37-52 for (multiply, add)):
//     for i in rows: for l < rowsinred: av = a[l + i*lstride]
//         for j < elsinop: res[i*restride+j] = reduce(res[..], combine(av, b[l*rstride+j]))
// Every result element is an l-ascending fold from the identity.  Rows (and
// elements) are independent, so the GPU tiles C into (16*TM) x (16*TN) blocks
// of 16x16 threads with a TM x TN register tile each; each thread folds its
// elements over l in ascending order with the reference's exact operations,
// which makes the result bit-identical to the reference for every pair (the
// "exact" loop).
//
// For combine in {add, subtract} with reduce in {min, max} on float32 — the
// tropical semirings, BASELINE config 5 — the exact loop costs a FADD, FSETP
// and FSEL per pair; the fast loops of tropical.cuh add two contraction steps
// at once with a packed FADD2 and fold both sums with one 3-input min/max
// (VIMNMX3 on the bit patterns when every combine result is a non-negative
// float, FMNMX3 when no combine result can be NaN or -0.0, moa_common.cuh).
// A pre-scan kernel here records which special values occur in A and B; the
// host launches one kernel per fold mode (this file's MODEK = 0 exact
// specialisation among them) and all but the one the device flags select
// return at once, so there is no host synchronisation and the result never
// depends on the choice.
//
// Shared-memory layout: both tiles are stored as k-PAIRS, As[kp][m] =
// (A[m][2kp], A[m][2kp+1]) and Bs[kp][n] = (B[2kp][n], B[2kp+1][n]).  Thread
// (ty, tx) owns rows ty*TM..ty*TM+TM-1 and columns 16j + tx; A reads are
// warp-broadcasts and a warp's B reads per j cover one contiguous span.
// Global->shared staging is element-wise cp.async (3 stages).
#pragma once

#include <type_traits>

#include "host_runtime.h"
#include "moa_common.cuh"
#include "moa_kernels.h"
#include "../../include/moa_b200.h"

namespace moa {

namespace {

constexpr int SNT = 256, GROUP_M = 8;  // 16 x 16 threads per CTA

template <typename T> struct alignas(2 * sizeof(T)) KPair { T x, y; };

template <typename T, int C, int R, int TM_, int TN_, int MINB_>
struct SemiringShape {
  static constexpr bool F4 = sizeof(typename AccType<T, C, R>::type) == 4;
  static constexpr int TM = TM_, TN = TN_;
  static constexpr int BM = 16 * TM, BN = 16 * TN;
  // k per stage (one barrier per BK): 32 for 4-byte accumulators and for
  // float64 data (4096^3 exact (multiply, add) 10.06 -> 9.74 ms, sums -3%,
  // compare-select -1..-2%; profiles/r02_tune_semiring_kunroll.jsonl); 16 for
  // float32 data summed in float64, int64, and division, whose staged divisor
  // tables would not fit three 32-deep stages
  static constexpr int BK = F4 ? 32 : (std::is_same<T, double>::value && C != C_DIV) ? 32 : 16;
  static constexpr int KP = BK / 2;             // k-pairs per stage
  static constexpr int STAGES = 3;
  static constexpr int A_STAGE = KP * BM;       // pairs
  static constexpr int B_STAGE = KP * BN;       // pairs
  static constexpr size_t SMEM = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(KPair<T>);
  // element-wise loader: thread t copies A elements (row t/BK + (SNT/BK)*q, k t%BK)
  // and B elements (k t/BN + (SNT/BN)*q, column t%BN)
  static constexpr int QA = BM * BK / SNT, A_RSTEP = SNT / BK;
  static constexpr int QB = BK * BN / SNT, B_KSTEP = SNT / BN;
  static_assert(QA <= 32 && B_KSTEP % 2 == 0 && TM % 2 == 0 && TN % 2 == 0, "tile layout");
  static_assert(SNT % BN == 0 && SNT % BK == 0 && (BM * BK) % SNT == 0,
                "the element-wise loaders cover whole tiles only when BN and BK divide the CTA");
};

// Default tiles: float32 min/max (c5): 8x8 per thread, two CTAs per SM
// (tools/tune_semiring.cu); float64 or float64-accumulated: 8x8, one CTA.
// Unroll of the exact loop's k steps: 4 lets ptxas hoist the next steps'
// shared loads over the current FP64 work — 4096^3 float64 (add, min) 16.43 ->
// 14.46 ms, (multiply, max) 15.98 -> 14.35, exact (multiply, add) 10.54 ->
// 10.06, (min, min) 20.29 -> 18.96, float32 and int32 routes 1-4% faster, all
// bit-identical — but division (staged reciprocals / multipliers), int64 and
// the float64 / int32 (min|max, add|multiply) pairs run slower unrolled (f64
// divide 8.23 -> 9.53 ms, int32 (min, add) -14%), so they keep 1
// (profiles/r02_tune_semiring_kunroll.jsonl, r02_route_sweep_4096.jsonl,
// tools/tune_semiring_kunroll.cu, tools/route_sweep.py).
#ifndef MOA_SEMIRING_KUNROLL
#define MOA_SEMIRING_KUNROLL 4
#endif
constexpr int KUNROLL = MOA_SEMIRING_KUNROLL;

template <typename T, int C, int R> struct DefaultTile {
  static constexpr bool F4 = sizeof(typename AccType<T, C, R>::type) == 4;
  static constexpr int TM = 8, TN = 8, MINB = F4 ? 2 : 1;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
template <int BYTES>
__device__ __forceinline__ void cp_async_elem(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(smem_u32(dst)), "l"(src),
               "n"(BYTES), "r"(valid ? BYTES : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// 3-input fold of the tropical fast loops (tropical.cuh)
template <int R, bool INTFOLD>
__device__ __forceinline__ float fold3(float acc, float s0, float s1) {
  if (INTFOLD) {  // non-negative floats: unsigned order == float order
    const unsigned x = __float_as_uint(acc), y = __float_as_uint(s0), z = __float_as_uint(s1);
    return __uint_as_float(R == R_MIN ? __vimin3_u32(x, y, z) : __vimax3_u32(x, y, z));
  }
  float r;
  if (R == R_MIN)
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(acc), "f"(s0), "f"(s1));
  else
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(acc), "f"(s0), "f"(s1));
  return r;
}

// MODEK: -1 = exact fold only (no pre-scan); 0 = the exact specialisation of a
// tropical candidate, which returns at once unless the device-side pre-scan
// selected the exact loop (modes 1 and 2 are the kernels of tropical.cuh).
template <typename T, int C, int R, bool ACC, int MODEK, int TM, int TN, int MINB>
__global__ void __launch_bounds__(SNT, MINB)
    semiring_kernel(T* __restrict__ c, const T* __restrict__ a, const T* __restrict__ b,
                    int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc,
                    const unsigned* special, int64_t tiles_m, int64_t tiles_n) {
  using A = typename AccType<T, C, R>::type;
  using Shape = SemiringShape<T, C, R, TM, TN, MINB>;
  constexpr int STAGES = Shape::STAGES, BM = Shape::BM, BN = Shape::BN;
  constexpr int BK = Shape::BK, KP = Shape::KP;
  if constexpr (MODEK >= 0) {
    if (tropical_mode_of<ACC>(C, R, special) != MODEK) return;
  }
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KPair<T>* As = reinterpret_cast<KPair<T>*>(smem_raw);
  KPair<T>* Bs = As + STAGES * Shape::A_STAGE;
  // division: RN(1/b) of the current B stage, [BK][BN], NaN where b is
  // outside the reciprocal path's range (so every proof using it fails); for
  // integers the same slots hold each divisor's multiplier and shifts
  // (div_magic; 8 bytes for int32, 16 for int64).
  constexpr bool RCP = C == C_DIV && std::is_same<A, double>::value;
  constexpr bool MAGIC = C == C_DIV && std::is_integral<A>::value;  // staged multipliers
  double* Ys = reinterpret_cast<double*>(Bs + STAGES * Shape::B_STAGE);

  // grouped rasterisation: GROUP_M row tiles sweep the column tiles together
  const int64_t pid = blockIdx.x;
  const int64_t width = GROUP_M * tiles_n;
  const int64_t first_m = (pid / width) * GROUP_M;
  const int64_t gsize = (tiles_m - first_m) < GROUP_M ? (tiles_m - first_m) : GROUP_M;
  const int64_t m0 = (first_m + (pid % width) % gsize) * BM;
  const int64_t n0 = ((pid % width) / gsize) * BN;

  const int tid = threadIdx.x;
  const int ty = tid >> 4, tx = tid & 15;
  // Thread (ty, tx) owns columns 16j + tx: a warp's 16 B loads per j hit one
  // contiguous run of k-pairs (a 32g + 2tx mapping puts them 2 pairs apart:
  // 4-way bank conflicts for double, 2-way for float).
  // (int64 multiply keeps the paired mapping: with 16j + tx ptxas shuffles the 64-bit
  // multiply-add accumulators, 2.7 -> 2.2 T pairs/s for (multiply, add))
  constexpr bool PAIRED = std::is_same<T, int64_t>::value && C == C_MUL;
  auto col_of = [&](int j) { return PAIRED ? 32 * (j >> 1) + 2 * tx + (j & 1) : 16 * j + tx; };

  // ---- accumulators: rows ty*TM+i, columns col_of(j) ----
  A acc[TM][TN];
  {
    // Under ACCUMULATE the seeds come from C through opaque copies of its
    // origin: otherwise the compiler keeps these addresses and bounds tests
    // alive through the main loop for the epilogue and spills them.
    int64_t om0 = m0, on0 = n0;
    const T* oc = c;
    if (ACC) asm volatile("" : "+l"(om0), "+l"(on0), "+l"(oc));
#pragma unroll
    for (int i = 0; i < TM; i++)
#pragma unroll
      for (int j = 0; j < TN; j++) {
        const int64_t row = om0 + ty * TM + i;
        const int64_t col = on0 + col_of(j);
        if (ACC && row < M && col < N)
          acc[i][j] = A(oc[row * ldc + col]);
        else
          acc[i][j] = ReduceOp<R>::template identity<A>();
      }
  }
  // ---- element-wise async copies into the k-pair layouts (zero-filled outside) ----
  // Per-thread bases are fixed for the whole kernel; a stage only adds k0.
  const int a_kk = tid % BK, a_r = tid / BK;
  const int b_n = tid % BN, b_kk = tid / BN;
  const T* a_src = a + (m0 + a_r) * lda + a_kk;
  const int64_t a_qstep = (int64_t)Shape::A_RSTEP * lda;
  const T* b_src = b + (int64_t)b_kk * ldb + n0 + b_n;
  const int64_t b_qstep = (int64_t)Shape::B_KSTEP * ldb;
  unsigned a_rows_ok = 0;
#pragma unroll
  for (int q = 0; q < Shape::QA; q++)
    if (m0 + a_r + q * Shape::A_RSTEP < M) a_rows_ok |= 1u << q;
  const bool b_col_ok = n0 + b_n < N;
  const int a_dst = 2 * ((a_kk >> 1) * BM + a_r) + (a_kk & 1);             // T elements
  const int b_dst = 2 * ((b_kk >> 1) * BN + b_n) + (b_kk & 1);             // T elements
  auto load_stage = [&](int stage, int64_t k0) {
    T* as = reinterpret_cast<T*>(As + stage * Shape::A_STAGE) + a_dst;
    T* bs = reinterpret_cast<T*>(Bs + stage * Shape::B_STAGE) + b_dst;
    const bool a_k_ok = k0 + a_kk < K;
    const T* pa = a_src + k0;
#pragma unroll
    for (int q = 0; q < Shape::QA; q++) {
      const bool ok = a_k_ok && ((a_rows_ok >> q) & 1u);
      cp_async_elem<sizeof(T)>(as + 2 * Shape::A_RSTEP * q,
                               ok ? pa + q * a_qstep : a, ok);
    }
    const T* pb = b_src + k0 * ldb;
#pragma unroll
    for (int q = 0; q < Shape::QB; q++) {
      const bool ok = b_col_ok && (k0 + b_kk + Shape::B_KSTEP * q < K);
      cp_async_elem<sizeof(T)>(bs + Shape::B_KSTEP * BN * q,
                               ok ? pb + q * b_qstep : b, ok);
    }
  };

  const int64_t KT = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; s++) {
    if (s < KT) load_stage(s, (int64_t)s * BK);
    cp_async_commit();
  }

  for (int64_t kt = 0; kt < KT; kt++) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int64_t nk = kt + STAGES - 1;
      if (nk < KT) load_stage((int)(nk % STAGES), nk * BK);
      cp_async_commit();
    }
    const KPair<T>* as = As + (int)(kt % STAGES) * Shape::A_STAGE;
    const KPair<T>* bs = Bs + (int)(kt % STAGES) * Shape::B_STAGE;
    const int64_t krem = K - kt * BK;
    const int kend = krem < BK ? (int)krem : BK;
    if constexpr (RCP) {
      // the previous stage's readers passed the barrier above, so Ys is free
#pragma unroll
      for (int q = 0; q < BK * BN / SNT; q++) {
        const int e = tid + q * SNT, k = e / BN, n = e % BN;
        const double bval = double(reinterpret_cast<const T*>(bs + (k >> 1) * BN + n)[k & 1]);
        Ys[k * BN + n] = rcp_range(bval) ? rcp_rn(bval) : __longlong_as_double(0x7ff8000000000000ll);
      }
      __syncthreads();
    }
    if constexpr (MAGIC) {
      using G = decltype(div_magic(A(0)));
      G* Gs = reinterpret_cast<G*>(Ys);
#pragma unroll
      for (int q = 0; q < BK * BN / SNT; q++) {
        const int e = tid + q * SNT, k = e / BN, n = e % BN;
        Gs[k * BN + n] = div_magic(A(reinterpret_cast<const T*>(bs + (k >> 1) * BN + n)[k & 1]));
      }
      __syncthreads();
    }

    {
      // exact loop: the reference's fold, k ascending, k beyond K skipped.
      // A elements are warp-broadcast loads; the B elements of columns
      // 16j + tx sit one k-pair apart, so a warp's 16 loads per j span 128
      // (float) or 256 (double) contiguous bytes.
      constexpr bool MINMAX_SUM = (C == C_MIN || C == C_MAX) && (R == R_ADD || R == R_MUL) &&
                                  !std::is_same<T, float>::value;
      constexpr int KU = (C == C_DIV || std::is_same<T, int64_t>::value || MINMAX_SUM) ? 1 : KUNROLL;
#pragma unroll KU
      for (int kk = 0; kk < kend; kk++) {
        const T* ak = reinterpret_cast<const T*>(as + (kk >> 1) * BM + ty * TM) + (kk & 1);
        const T* bk = reinterpret_cast<const T*>(bs + (kk >> 1) * BN + (PAIRED ? 2 * tx : tx)) + (kk & 1);
        A av[TM], bv[TN];
#pragma unroll
        for (int i = 0; i < TM; i++) av[i] = A(ak[2 * i]);
#pragma unroll
        for (int j = 0; j < TN; j++) bv[j] = A(bk[2 * (PAIRED ? 32 * (j >> 1) + (j & 1) : 16 * j)]);
        if constexpr (MAGIC) {
          using G = decltype(div_magic(A(0)));
          using U = typename IntTraits<A>::U;
          const G* Gs = reinterpret_cast<const G*>(Ys);
          G gv[TN];
#pragma unroll
          for (int j = 0; j < TN; j++) gv[j] = Gs[kk * BN + col_of(j)];
#pragma unroll
          for (int i = 0; i < TM; i++) {
            const U nx = av[i] < 0 ? U(0) - U(av[i]) : U(av[i]);
#pragma unroll
            for (int j = 0; j < TN; j++)
              acc[i][j] = ReduceOp<R>::f(acc[i][j], idiv_magic(av[i], nx, bv[j], gv[j]));
          }
        } else if constexpr (RCP) {
          // each row's TN quotients from the staged reciprocals, proven
          // together (div_candidate); a failed proof redoes the row exactly
          double yv[TN];
#pragma unroll
          for (int j = 0; j < TN; j++) yv[j] = Ys[kk * BN + col_of(j)];
#pragma unroll
          for (int i = 0; i < TM; i++) {
            A q[TN];
            bool ok = rcp_range(av[i]);
#pragma unroll
            for (int j = 0; j < TN; j++) q[j] = div_candidate(av[i], bv[j], yv[j], ok);
            if (!ok) {
#pragma unroll
              for (int j = 0; j < TN; j++) q[j] = CombineOp<C_DIV>::f(av[i], bv[j]);
            }
#pragma unroll
            for (int j = 0; j < TN; j++) acc[i][j] = ReduceOp<R>::f(acc[i][j], q[j]);
          }
        } else if constexpr (std::is_same<T, float>::value && C == C_MUL && R == R_ADD) {
          // float32 data accumulated in float64: the product of two floats is
          // exact in float64, so RN(acc + RN(a*b)) = RN(acc + a*b) = DFMA
          // (one FP64 instruction per pair instead of two, same bits)
#pragma unroll
          for (int i = 0; i < TM; i++)
#pragma unroll
            for (int j = 0; j < TN; j++) acc[i][j] = __fma_rn(av[i], bv[j], acc[i][j]);
        } else if constexpr (std::is_same<A, int32_t>::value && (C == C_ADD || C == C_SUB) &&
                             (R == R_MIN || R == R_MAX)) {
          // int32 tropical: one DPX add-then-min/max (VIADDMNMX) per pair;
          // the add wraps like wrap_add and subtract adds the wrapped negation
#pragma unroll
          for (int j = 0; j < TN; j++)
            if (C == C_SUB) bv[j] = wrap_sub(int32_t(0), bv[j]);
#pragma unroll
          for (int i = 0; i < TM; i++)
#pragma unroll
            for (int j = 0; j < TN; j++)
              acc[i][j] = R == R_MIN ? __viaddmin_s32(av[i], bv[j], acc[i][j])
                                     : __viaddmax_s32(av[i], bv[j], acc[i][j]);
        } else {
#pragma unroll
          for (int i = 0; i < TM; i++)
#pragma unroll
            for (int j = 0; j < TN; j++)
              acc[i][j] = ReduceOp<R>::f(acc[i][j], CombineOp<C>::f(av[i], bv[j]));
        }
      }
    }
  }
  cp_async_wait<0>();

  // ---- epilogue ----
#pragma unroll
  for (int i = 0; i < TM; i++) {
    const int64_t row = m0 + ty * TM + i;
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; j++) {
      const int64_t col = n0 + col_of(j);
      if (col < N) c[row * ldc + col] = convert<T, A>(acc[i][j]);
    }
  }
}

// Special-value flags of one float32 value, branch-free on its bit pattern
__device__ __forceinline__ unsigned special_bits(unsigned u) {
  const unsigned mag = u & 0x7fffffffu;
  unsigned f = (u >> 31) ? S_NEG : 0u;
  f |= mag > 0x7f800000u ? S_NAN : 0u;
  f |= u == 0x7f800000u ? S_PINF : 0u;
  f |= u == 0xff800000u ? S_NINF : 0u;
  f |= u == 0u ? S_PZERO : 0u;
  f |= u == 0x80000000u ? S_NZERO : 0u;
  return f;
}

// OR of special_bits over x[0, n), strided over `nthr` threads starting at
// `tid`: scalar head up to 16-byte alignment, then four 16-byte loads in
// flight per thread per step (the scan is a pure HBM stream, so the loads in
// flight set its speed), then a scalar tail
__device__ __forceinline__ unsigned scan_segment(const float* __restrict__ x, int64_t n,
                                                 int64_t tid, int64_t nthr) {
  unsigned bits = 0;
  int64_t head = (int64_t)((16u - (reinterpret_cast<uintptr_t>(x) & 15u)) & 15u) / 4;
  if (head > n) head = n;
  if (tid < head) bits |= special_bits(__float_as_uint(__ldg(x + tid)));
  const uint4* v = reinterpret_cast<const uint4*>(x + head);
  const int64_t nv = (n - head) / 4;
  constexpr int U = 4;
  int64_t i = tid;
  for (; i + (U - 1) * nthr < nv; i += U * nthr) {
    uint4 q[U];
#pragma unroll
    for (int u = 0; u < U; u++) q[u] = __ldcs(v + i + u * nthr);
#pragma unroll
    for (int u = 0; u < U; u++)
      bits |= special_bits(q[u].x) | special_bits(q[u].y) | special_bits(q[u].z) |
              special_bits(q[u].w);
  }
  for (; i < nv; i += nthr) {
    const uint4 q = __ldcs(v + i);
    bits |= special_bits(q.x) | special_bits(q.y) | special_bits(q.z) | special_bits(q.w);
  }
  const int64_t tail0 = head + nv * 4;
  if (tail0 + tid < n) bits |= special_bits(__float_as_uint(__ldg(x + tail0 + tid)));
  return bits;
}

// Device pre-scan of a rows x cols float32 matrix (row stride ld): the OR of
// its values' special-value flags into *out.  Contiguous matrices are one
// segment over the whole grid; strided ones give each block row its own rows.
__global__ void __launch_bounds__(256) scan_special_kernel(const float* __restrict__ x, int64_t rows,
                                                           int64_t cols, int64_t ld,
                                                           unsigned* __restrict__ out) {
  unsigned bits = 0;
  if (ld == cols || rows == 1) {
    const int64_t nthr = (int64_t)gridDim.x * gridDim.y * blockDim.x;
    const int64_t tid = ((int64_t)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;
    bits = scan_segment(x, rows * cols, tid, nthr);
  } else {
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) bits |= scan_segment(x + r * ld, cols, tid, nthr);
  }
  bits = __reduce_or_sync(0xffffffffu, bits);
  if ((threadIdx.x & 31) == 0 && bits) atomicOr(out, bits);
}

template <typename T>
void launch_scan(const T* x, int64_t rows, int64_t cols, int64_t ld, unsigned* out,
                 cudaStream_t s) {
  static_assert(std::is_same<T, float>::value, "the pre-scan serves the float32 fast folds");
  if (rows <= 0 || cols <= 0) return;
  const unsigned bx = 256;
  int64_t gx, gy;
  if (ld == cols || rows == 1) {
    gx = (int64_t)kNumSMs * 8;  // eight 256-thread blocks per SM stream the whole matrix
    const int64_t need = (rows * cols / 16 + bx - 1) / bx;  // >= 16 floats per thread
    if (gx > need) gx = need < 1 ? 1 : need;
    gy = 1;
  } else {
    gx = (cols / 16 + bx - 1) / bx;
    if (gx < 1) gx = 1;
    if (gx > 64) gx = 64;
    gy = ((int64_t)kNumSMs * 8 + gx - 1) / gx;
    if (gy > rows) gy = rows;
    if (gy > 65535) gy = 65535;
  }
  scan_special_kernel<<<dim3((unsigned)gx, (unsigned)gy), bx, 0, s>>>(x, rows, cols, ld, out);
  count_launch();
}

template <typename T, int C, int R, bool ACC, int MODEK, int TM = DefaultTile<T, C, R>::TM,
          int TN = DefaultTile<T, C, R>::TN, int MINB = DefaultTile<T, C, R>::MINB>
cudaError_t semiring_launch(const Problem& p, const unsigned* special) {
  using Shape = SemiringShape<T, C, R, TM, TN, MINB>;
  auto kern = semiring_kernel<T, C, R, ACC, MODEK, TM, TN, MINB>;
  using Acc = typename AccType<T, C, R>::type;
  // staged reciprocals (float64) or multipliers (integers) for division
  constexpr size_t stage_elem = C != C_DIV ? 0
                                : std::is_same<Acc, double>::value ? sizeof(double)
                                : std::is_same<Acc, int64_t>::value ? sizeof(DivMagic64)
                                : std::is_same<Acc, int32_t>::value ? sizeof(DivMagic32) : 0;
  const size_t smem = Shape::SMEM + (size_t)Shape::BK * Shape::BN * stage_elem;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t tiles_m = (p.M + Shape::BM - 1) / Shape::BM;
  const int64_t tiles_n = (p.N + Shape::BN - 1) / Shape::BN;
  const int64_t tiles = tiles_m * tiles_n;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  kern<<<(unsigned)tiles, SNT, smem, p.stream>>>(
      static_cast<T*>(p.c), static_cast<const T*>(p.a), static_cast<const T*>(p.b), p.M, p.N, p.K,
      p.lda, p.ldb, p.ldc, special, tiles_m, tiles_n);
  count_launch();
  return cudaGetLastError();
}

}  // namespace
}  // namespace moa

#include "tropical.cuh"

namespace moa {
namespace {

// float32 tropical pair ((add|sub|mul) x (min|max); multiply only with the
// unsigned-order fold): pre-scan A (M x K, lda), B (K x N, ldb) and, when
// accumulating, C (M x N, ldc) for NaN / +-inf / +-0 / sign, then launch one
// specialisation per fold mode; all but the one the flags select exit at once.
//
// The 12-byte flags buffer comes from the library's private device pool
// (host_runtime.cu), which keeps its memory mapped: from the device's default
// pool (release threshold 0) every launch re-mapped a fresh chunk after the
// previous one had been unmapped at a synchronisation, and those mapping
// operations intermittently blocked the host for tens of ms while kernels
// were in flight — the k-chunked accumulate schedule of c5's first block took
// 42-136 ms from one repetition to the next (tools/c5_repeat_device.py).
template <int C, int R, bool ACC>
cudaError_t tropical_candidate(const Problem& p) {
  unsigned* special = nullptr;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  cudaMemPool_t pool = e == cudaSuccess ? host::device_pool(dev, e) : nullptr;
  if (pool == nullptr) return e != cudaSuccess ? e : cudaErrorMemoryAllocation;
  e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&special), 3 * sizeof(unsigned), pool,
                              p.stream);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(special, 0, 3 * sizeof(unsigned), p.stream);
  if (e == cudaSuccess) {
    launch_scan<float>(static_cast<const float*>(p.a), p.M, p.K, p.lda, special, p.stream);
    launch_scan<float>(static_cast<const float*>(p.b), p.K, p.N, p.ldb, special + 1, p.stream);
    if (ACC) launch_scan<float>(static_cast<const float*>(p.c), p.M, p.N, p.ldc, special + 2, p.stream);
    if constexpr (C == C_ADD || C == C_MUL) e = tropical_launch<C, R, 2, ACC>(p, special);
    if constexpr (C != C_MUL) {
      if (e == cudaSuccess) e = tropical_launch<C, R, 1, ACC>(p, special);
    }
    if (e == cudaSuccess) e = semiring_launch<float, C, R, ACC, 0>(p, special);
  }
  cudaError_t e2 = cudaFreeAsync(special, p.stream);
  return e != cudaSuccess ? e : e2;
}

template <typename T, int C, int R>
cudaError_t semiring_acc(const Problem& p) {
  constexpr bool cand = std::is_same<T, float>::value && (C == C_ADD || C == C_SUB || C == C_MUL) &&
                        (R == R_MIN || R == R_MAX);
  // int32 (add|subtract, min|max): exact integer arithmetic, so the TMA
  // tropical kernel (four-k step; 128x128 tiles from 256 of them, 64x128
  // below, as for float32: 250.4 vs 250.9 ms at 16384^3, 0.157 vs 0.099 ms at
  // 1000^3, profiles/r02_tune_tropical_bm128.jsonl) runs it with one DPX
  // VIADDMNMX per pair and no pre-scan whenever rows are 16-byte aligned
  constexpr bool i32trop = std::is_same<T, int32_t>::value && (C == C_ADD || C == C_SUB) &&
                           (R == R_MIN || R == R_MAX);
  if constexpr (cand) {
    return p.accumulate ? tropical_candidate<C, R, true>(p) : tropical_candidate<C, R, false>(p);
  } else if constexpr (i32trop) {
    if (tropical_tma_eligible(p) && tropical_big_tiles(p))
      return p.accumulate ? tropical_tma_launch<C, R, 3, true, 2, 1, true, 128, 1>(p, nullptr)
                          : tropical_tma_launch<C, R, 3, false, 2, 1, true, 128, 1>(p, nullptr);
    if (tropical_tma_eligible(p))
      return p.accumulate ? tropical_tma_launch<C, R, 3, true, 3, 1, true, 64, 1>(p, nullptr)
                          : tropical_tma_launch<C, R, 3, false, 3, 1, true, 64, 1>(p, nullptr);
    return p.accumulate ? semiring_launch<T, C, R, true, -1>(p, nullptr)
                        : semiring_launch<T, C, R, false, -1>(p, nullptr);
  } else {
    return p.accumulate ? semiring_launch<T, C, R, true, -1>(p, nullptr)
                        : semiring_launch<T, C, R, false, -1>(p, nullptr);
  }
}

template <typename T, int C>
cudaError_t semiring_red(const Problem& p) {
  switch (p.reduce) {
    case R_ADD: return semiring_acc<T, C, R_ADD>(p);
    case R_MUL: return semiring_acc<T, C, R_MUL>(p);
    case R_MIN: return semiring_acc<T, C, R_MIN>(p);
    default: return semiring_acc<T, C, R_MAX>(p);
  }
}

template <typename T>
cudaError_t semiring_comb(const Problem& p) {
  switch (p.combine) {
    case C_ADD: return semiring_red<T, C_ADD>(p);
    case C_SUB: return semiring_red<T, C_SUB>(p);
    case C_MUL: return semiring_red<T, C_MUL>(p);
    case C_DIV: return semiring_red<T, C_DIV>(p);
    case C_MIN: return semiring_red<T, C_MIN>(p);
    default: return semiring_red<T, C_MAX>(p);
  }
}

}  // namespace
}  // namespace moa
