// K2 fast loops for the float32 tropical semirings — combine in {add, subtract}
// (BASELINE config 5) or multiply (max-times / min-times, non-negative data
// only), reduce in {min, max} — in their own kernels.
//
// Two kernels share the loop: tropical_tma_kernel (16-byte aligned rows:
// TMA-staged tiles, mbarrier pipeline, no block barrier in the main loop;
// 128x128 C tiles of 256 threads, two CTAs per SM, for large outputs and 64x128
// tiles of 128 threads, three CTAs per SM, below that; four k per step) and
// tropical_kernel (any alignment: cp.async into padded A[BM][BK+4],
// B[BK][BN+4]; 128x128 tiles).  Operands stay in their natural row-major
// layouts; a thread owns 8 rows and columns 64g + 4tx + c (g < 2, c < 4) of
// its C tile.
// For each k-pair (k, k+1) it forms, per row i and
// column pair (j, j+1),
//     s  = FADD2((B[k][j],   B[k][j+1]),   a[i][k]   broadcast)
//     s' = FADD2((B[k+1][j], B[k+1][j+1]), a[i][k+1] broadcast)
//     acc[i][j]   = min3(acc[i][j],   s.x, s'.x)
//     acc[i][j+1] = min3(acc[i][j+1], s.y, s'.y)
// i.e. one packed add and one 3-input fold per two (a, b) pairs, with the B
// operand straight from a 64-bit shared load.  The fold is VIMNMX3 on the bit
// patterns (mode 2: every combine result is a non-negative float) or FMNMX3
// (mode 1: no combine result can be NaN or -0.0); see tropical_fold_mode.
// Both are exact (bit-identical to the reference's compare-select fold) under
// their conditions, which the device pre-scan establishes; the kernel returns
// at once when the pre-scan selected another mode.
#pragma once

#include "moa_common.cuh"
#include "tma.cuh"

namespace moa {
namespace {

constexpr int TBM = 128, TBN = 128, TBK = 32, TSTAGES = 3, TNT = 256;
constexpr int TLDA = TBK + 4, TLDB = TBN + 4;  // floats; rows stay 16-byte aligned
constexpr int TA_STAGE = TBM * TLDA, TB_STAGE = TBK * TLDB;
constexpr size_t TSMEM = (size_t)TSTAGES * (TA_STAGE + TB_STAGE) * sizeof(float);

__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(bytes)
               : "memory");
}

// (x0 op a, x1 op a) with the scalar a broadcast to both lanes
template <int C>
__device__ __forceinline__ unsigned long long pair_op_bcast(float x0, float x1, float a) {
  unsigned long long r;
  if (C == C_SUB)  // combine(a, b) = a - b, A element first (_ckernel.pyx:71)
    asm("{\n\t.reg .b64 ta, tb;\n\tmov.b64 ta, {%1, %1};\n\tmov.b64 tb, {%2, %3};\n\t"
        "sub.rn.f32x2 %0, ta, tb;\n\t}"
        : "=l"(r) : "f"(a), "f"(x0), "f"(x1));
  else if (C == C_MUL)
    asm("{\n\t.reg .b64 ta, tb;\n\tmov.b64 ta, {%1, %1};\n\tmov.b64 tb, {%2, %3};\n\t"
        "mul.rn.f32x2 %0, tb, ta;\n\t}"
        : "=l"(r) : "f"(a), "f"(x0), "f"(x1));
  else
    asm("{\n\t.reg .b64 ta, tb;\n\tmov.b64 ta, {%1, %1};\n\tmov.b64 tb, {%2, %3};\n\t"
        "add.rn.f32x2 %0, tb, ta;\n\t}"
        : "=l"(r) : "f"(a), "f"(x0), "f"(x1));
  return r;
}
// MODE 3 (int32 data through the same kernel, bit patterns carried as floats):
// acc = reduce(acc, combine(a, b)) as one DPX add-then-min/max (VIADDMNMX),
// two's-complement wraparound; subtract adds b's wrapped negation
template <int C, int R>
__device__ __forceinline__ float iaddmnmx(float a, float b, float acc) {
  const int x = __float_as_int(a), y = C == C_SUB ? -__float_as_int(b) : __float_as_int(b);
  const int z = __float_as_int(acc);
  return __int_as_float(R == R_MIN ? __viaddmin_s32(x, y, z) : __viaddmax_s32(x, y, z));
}

__device__ __forceinline__ float lo32(unsigned long long v) { return __uint_as_float((unsigned)v); }
__device__ __forceinline__ float hi32(unsigned long long v) {
  return __uint_as_float((unsigned)(v >> 32));
}

// Accumulators of a thread owning rows r0 + rstep*i (i < 8) and columns
// 64g + 4tx + cc (acc[i][4g + cc]).  From the identity — or, for the
// unsigned-order max fold, from +0: every combine result is >= +0 there and
// K >= 1, so the max is unchanged while -inf's sign bit would break the
// order — or from C's previous contents under MOA_FLAG_ACCUMULATE (whose
// values the fold mode has already checked).
template <int R, bool INTFOLD, bool ACC, bool I32 = false>
__device__ __forceinline__ void init_acc(float (&acc)[8][8], const float* c, int64_t M, int64_t N,
                                         int64_t ldc, int64_t m0, int64_t n0, int r0, int rstep,
                                         int tx) {
  const float init = I32 ? __int_as_float(ReduceOp<R>::template identity<int32_t>())
                     : (INTFOLD && R == R_MAX) ? 0.0f : ReduceOp<R>::template identity<float>();
  // opaque copies of C's origin: otherwise the compiler keeps these addresses
  // and bounds tests alive through the main loop for the epilogue and spills
  if (ACC) asm volatile("" : "+l"(m0), "+l"(n0), "+l"(c));
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) {
      acc[i][j] = init;
      if (ACC) {
        const int64_t row = m0 + r0 + rstep * i, col = n0 + 64 * (j >> 2) + 4 * tx + (j & 3);
        if (row < M && col < N) {
          const float v = c[row * ldc + col];
          // unsigned-order max: a negative seed never wins against results >= +0
          acc[i][j] = (INTFOLD && !I32 && R == R_MAX && (__float_as_uint(v) >> 31)) ? 0.0f : v;
        }
      }
    }
}

template <int C, int R, int MODE, bool ACC, bool VEC>
__global__ void __launch_bounds__(TNT, 2)
    tropical_kernel(float* __restrict__ c, const float* __restrict__ a, const float* __restrict__ b,
                    int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc,
                    const unsigned* special, int64_t tiles_m, int64_t tiles_n) {
  static_assert(MODE == 1 || MODE == 2, "fast modes only");
  constexpr bool INTFOLD = MODE == 2;
  if (tropical_mode_of<ACC>(C, R, special) != MODE) return;
  extern __shared__ __align__(16) float tsm[];
  float* As = tsm;
  float* Bs = tsm + TSTAGES * TA_STAGE;

  const int64_t pid = blockIdx.x;
  constexpr int GM = 8;
  const int64_t width = GM * tiles_n;
  const int64_t first_m = (pid / width) * GM;
  const int64_t gsize = (tiles_m - first_m) < GM ? (tiles_m - first_m) : GM;
  const int64_t m0 = (first_m + (pid % width) % gsize) * TBM;
  const int64_t n0 = ((pid % width) / gsize) * TBN;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;

  float acc[8][8];
  init_acc<R, INTFOLD, ACC>(acc, c, M, N, ldc, m0, n0, ty * 8, 1, tx);

  // ---- loaders: 16-byte chunks (VEC) or single elements, zero-filled outside ----
  auto load_stage = [&](int stage, int64_t k0) {
    float* as = As + stage * TA_STAGE;
    float* bs = Bs + stage * TB_STAGE;
    if constexpr (VEC) {
#pragma unroll
      for (int q = 0; q < TBM * TBK / 4 / TNT; q++) {  // 4 chunks per thread
        const int ch = tid + q * TNT, r = ch >> 3, kc = (ch & 7) * 4;
        const int64_t gm = m0 + r, gk = k0 + kc;
        int64_t rem = gm < M ? K - gk : 0;
        rem = rem < 0 ? 0 : (rem > 4 ? 4 : rem);
        cp_async16_zfill(as + r * TLDA + kc, rem ? a + gm * lda + gk : a, (int)rem * 4);
      }
#pragma unroll
      for (int q = 0; q < TBK * TBN / 4 / TNT; q++) {  // 4 chunks per thread
        const int ch = tid + q * TNT, r = ch >> 5, nc = (ch & 31) * 4;
        const int64_t gk = k0 + r, gn = n0 + nc;
        int64_t rem = gk < K ? N - gn : 0;
        rem = rem < 0 ? 0 : (rem > 4 ? 4 : rem);
        cp_async16_zfill(bs + r * TLDB + nc, rem ? b + gk * ldb + gn : b, (int)rem * 4);
      }
    } else {
#pragma unroll
      for (int q = 0; q < TBM * TBK / TNT; q++) {
        const int e = tid + q * TNT, r = e / TBK, kk = e % TBK;
        const int64_t gm = m0 + r, gk = k0 + kk;
        const bool ok = gm < M && gk < K;
        cp_async_elem<4>(as + r * TLDA + kk, ok ? a + gm * lda + gk : a, ok);
      }
#pragma unroll
      for (int q = 0; q < TBK * TBN / TNT; q++) {
        const int e = tid + q * TNT, r = e / TBN, nn = e % TBN;
        const int64_t gk = k0 + r, gn = n0 + nn;
        const bool ok = gk < K && gn < N;
        cp_async_elem<4>(bs + r * TLDB + nn, ok ? b + gk * ldb + gn : b, ok);
      }
    }
  };

  const int64_t KT = (K + TBK - 1) / TBK;
#pragma unroll
  for (int s = 0; s < TSTAGES - 1; s++) {
    if (s < KT) load_stage(s, (int64_t)s * TBK);
    cp_async_commit();
  }

  for (int64_t kt = 0; kt < KT; kt++) {
    cp_async_wait<TSTAGES - 2>();
    __syncthreads();
    {
      const int64_t nk = kt + TSTAGES - 1;
      if (nk < KT) load_stage((int)(nk % TSTAGES), nk * TBK);
      cp_async_commit();
    }
    const float* as = As + (int)(kt % TSTAGES) * TA_STAGE + (ty * 8) * TLDA;
    const float* bs = Bs + (int)(kt % TSTAGES) * TB_STAGE + 4 * tx;
    const int64_t krem = K - kt * TBK;
    const int kend = krem < TBK ? (int)krem : TBK;

    // one k-pair (k, k+1): B rows k and k+1 as 16-byte loads, A pair per row as
    // one 8-byte (broadcast) load
    auto kpair = [&](int k) {
      float4 b0[2], b1[2];
#pragma unroll
      for (int g = 0; g < 2; g++) {
        b0[g] = *reinterpret_cast<const float4*>(bs + k * TLDB + 64 * g);
        b1[g] = *reinterpret_cast<const float4*>(bs + (k + 1) * TLDB + 64 * g);
      }
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const float2 av = *reinterpret_cast<const float2*>(as + i * TLDA + k);
#pragma unroll
        for (int g = 0; g < 2; g++) {
#pragma unroll
          for (int p = 0; p < 2; p++) {
            const float x0 = p ? b0[g].z : b0[g].x, x1 = p ? b0[g].w : b0[g].y;
            const float y0 = p ? b1[g].z : b1[g].x, y1 = p ? b1[g].w : b1[g].y;
            const unsigned long long s = pair_op_bcast<C>(x0, x1, av.x);
            const unsigned long long t = pair_op_bcast<C>(y0, y1, av.y);
            const int j = 4 * g + 2 * p;
            acc[i][j] = fold3<R, INTFOLD>(acc[i][j], lo32(s), lo32(t));
            acc[i][j + 1] = fold3<R, INTFOLD>(acc[i][j + 1], hi32(s), hi32(t));
          }
        }
      }
    };
    const int npairs = kend >> 1;
#pragma unroll 1
    for (int kp = 0; kp < npairs; kp++) kpair(2 * kp);
    {
      const int k4 = 2 * npairs;
      if (k4 < kend) {  // lone last k: scalar combine + 2-input fold
#pragma unroll
        for (int i = 0; i < 8; i++) {
          const float av = as[i * TLDA + k4];
#pragma unroll
          for (int g = 0; g < 2; g++)
#pragma unroll
            for (int cc = 0; cc < 4; cc++)
              acc[i][4 * g + cc] =
                  ReduceOp<R>::f(acc[i][4 * g + cc], CombineOp<C>::f(av, bs[k4 * TLDB + 64 * g + cc]));
        }
      }
    }
  }
  cp_async_wait<0>();

  const bool vec_store = (ldc % 4 == 0) && (reinterpret_cast<uintptr_t>(c) % 16 == 0);
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const int64_t row = m0 + ty * 8 + i;
    if (row >= M) continue;
#pragma unroll
    for (int g = 0; g < 2; g++) {
      const int64_t col = n0 + 64 * g + 4 * tx;
      if (vec_store && col + 3 < N) {
        *reinterpret_cast<float4*>(c + row * ldc + col) =
            make_float4(acc[i][4 * g], acc[i][4 * g + 1], acc[i][4 * g + 2], acc[i][4 * g + 3]);
      } else {
#pragma unroll
        for (int cc = 0; cc < 4; cc++)
          if (col + cc < N) c[row * ldc + col + cc] = acc[i][4 * g + cc];
      }
    }
  }
}

// ---- TMA-staged variant ------------------------------------------------------
// The same fold with both tiles brought in by TMA and no block-wide barrier in
// the main loop (full/empty mbarrier pair per stage, one thread issuing), so
// the 256 compute threads run only shared loads, FADD2 and the 3-input fold.
//   A stage: one box of 128 rows x 32 k (128 B per row), 128-byte swizzle:
//            element (r, k) at r*128 + (((k>>2) ^ r) & 7)*16 + (k&3)*4.
//   B stage: one box of 32 k x 128 columns, unswizzled (512 B rows): a warp
//            reads one 256-byte run of a row, already conflict-free.
// Thread (ty, tx) owns rows ty + 16i (i < 8), so the two A rows a warp reads
// per load differ in (r & 7) and sit in different banks, and the swizzle term
// ((k>>2) ^ ty) & 7 is the same for all eight rows.
// (BMT = 64: 64 x 128 CTA tiles of 128 threads, rows ty + 8i, three CTAs per
// SM with up to 168 registers per thread instead of 128.)
template <int BMT>
struct TropTma {
  static constexpr int BM = BMT, THREADS = 2 * BMT, ROW_STEP = BMT / 8;
  static constexpr int A_BYTES = BMT * TBK * 4, B_BYTES = TBK * TBN * 4;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = (size_t)TSTAGES * STAGE_BYTES + 1024 + 64;
  static_assert(ROW_STEP % 8 == 0, "rows ty + ROW_STEP*i keep the swizzle term ty & 7");
};
constexpr int TT_A_BYTES = TropTma<128>::A_BYTES, TT_B_BYTES = TropTma<128>::B_BYTES;
constexpr int TT_STAGE_BYTES = TropTma<128>::STAGE_BYTES;
constexpr size_t TT_SMEM = TropTma<128>::SMEM;

// FORM (the FADD2/fold pairing; all bit-identical): 0 = row k's and row k+1's
// column pairs folded lo with lo, hi with hi (production); 1 = row k+1's pair
// swapped inside its FADD2 (.LO_HI operand) so each fold reads one even and
// one odd register; 2 = scalar FADDs.  1 and 2 measured slower at c5 (213.6
// and 246.3 vs 211.2 ms, profiles/r02_tune_tropical_form.jsonl).
// REFILL 0: thread 0 refills the slab consumed one iteration earlier once
// every warp has released it (empty mbarrier), i.e. warp 0 waits for the
// slowest warp each k-slab; REFILL 1: the LAST warp to finish a slab refills
// its stage at once (a shared counter per stage), so no warp ever waits on
// another's progress except for data.
template <int C, int R, int MODE, bool ACC, int MINB = 2, int UNR = 1, bool QUAD = false,
          int BMT = 128, int REFILL = 0, int FORM = 0>
__global__ void __launch_bounds__(TropTma<BMT>::THREADS, MINB)
    tropical_tma_kernel(float* __restrict__ c, int64_t M, int64_t N, int64_t K, int64_t ldc,
                        const unsigned* special, int64_t tiles_m, int64_t tiles_n,
                        const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_b) {
  static_assert(MODE == 1 || MODE == 2 || MODE == 3, "fast modes only");
  static_assert(MODE != 3 || C == C_ADD || C == C_SUB, "int32 mode: add/subtract combines");
  using TT = TropTma<BMT>;
  constexpr bool INTFOLD = MODE == 2, I32 = MODE == 3;
  if constexpr (!I32) {  // float modes: the device pre-scan picks the fold
    if (tropical_mode_of<ACC>(C, R, special) != MODE) return;
  }
  extern __shared__ __align__(16) unsigned char tt_raw[];
  unsigned char* base = tma::align1k(tt_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + TSTAGES * TT::STAGE_BYTES);
  uint64_t* empty = full + TSTAGES;
  unsigned* done_warps = reinterpret_cast<unsigned*>(empty + TSTAGES);  // REFILL 1

  const int64_t pid = blockIdx.x;
  constexpr int GM = 8;
  const int64_t width = GM * tiles_n;
  const int64_t first_m = (pid / width) * GM;
  const int64_t gsize = (tiles_m - first_m) < GM ? (tiles_m - first_m) : GM;
  const int64_t m0 = (first_m + (pid % width) % gsize) * TT::BM;
  const int64_t n0 = ((pid % width) / gsize) * TBN;
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15, lane = tid & 31;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < TSTAGES; s++) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], TT::THREADS / 32);
      done_warps[s] = 0;
    }
    tma::mbar_init_fence();
  }
  __syncthreads();

  const int64_t KT = (K + TBK - 1) / TBK;
  auto issue = [&](int stage, int64_t kt) {  // one thread
    unsigned char* st = base + stage * TT::STAGE_BYTES;
    tma::mbar_expect_tx(&full[stage], TT::STAGE_BYTES);
    tma::load_2d(st, &map_a, (int)(kt * TBK), (int)m0, &full[stage]);
    tma::load_2d(st + TT::A_BYTES, &map_b, (int)n0, (int)(kt * TBK), &full[stage]);
  };
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < TSTAGES; s++)
      if (s < KT) issue(s, s);
  }

  float acc[8][8];
  init_acc<R, INTFOLD, ACC, I32>(acc, c, M, N, ldc, m0, n0, ty, TT::ROW_STEP, tx);

  for (int64_t kt = 0; kt < KT; kt++) {
    const int stage = (int)(kt % TSTAGES);
    tma::mbar_wait(&full[stage], (unsigned)((kt / TSTAGES) & 1));
    const unsigned char* as = base + stage * TT::STAGE_BYTES + ty * 128;
    const float* bs = reinterpret_cast<const float*>(base + stage * TT::STAGE_BYTES + TT::A_BYTES) +
                      4 * tx;
    const int64_t krem = K - kt * TBK;
    const int kend = krem < TBK ? (int)krem : TBK;
    // k-pair (k, k+1) of row i with A values (a0, a1) and B rows k, k+1
    auto fold_pair = [&](int i, float a0, float a1, const float4 (&b0)[2], const float4 (&b1)[2]) {
#pragma unroll
      for (int g = 0; g < 2; g++) {
#pragma unroll
        for (int p = 0; p < 2; p++) {
          const float x0 = p ? b0[g].z : b0[g].x, x1 = p ? b0[g].w : b0[g].y;
          const float y0 = p ? b1[g].z : b1[g].x, y1 = p ? b1[g].w : b1[g].y;
          const int j = 4 * g + 2 * p;
          if constexpr (I32) {  // k then k+1, as the exact loop folds them
            acc[i][j] = iaddmnmx<C, R>(a1, y0, iaddmnmx<C, R>(a0, x0, acc[i][j]));
            acc[i][j + 1] = iaddmnmx<C, R>(a1, y1, iaddmnmx<C, R>(a0, x1, acc[i][j + 1]));
          } else if constexpr (FORM == 2) {
            // scalar adds (FADD: one issue slot per pair, as FADD2 costs two)
            acc[i][j] = fold3<R, INTFOLD>(acc[i][j], CombineOp<C>::f(a0, x0), CombineOp<C>::f(a1, y0));
            acc[i][j + 1] = fold3<R, INTFOLD>(acc[i][j + 1], CombineOp<C>::f(a0, x1), CombineOp<C>::f(a1, y1));
          } else if constexpr (FORM == 1) {
            // row k+1's pair enters its FADD2 swapped (free: the .LO_HI operand
            // form), so each 3-input fold reads one even and one odd register
            const unsigned long long s = pair_op_bcast<C>(x0, x1, a0);
            const unsigned long long t = pair_op_bcast<C>(y1, y0, a1);
            acc[i][j] = fold3<R, INTFOLD>(acc[i][j], lo32(s), hi32(t));
            acc[i][j + 1] = fold3<R, INTFOLD>(acc[i][j + 1], hi32(s), lo32(t));
          } else {
            const unsigned long long s = pair_op_bcast<C>(x0, x1, a0);
            const unsigned long long t = pair_op_bcast<C>(y0, y1, a1);
            acc[i][j] = fold3<R, INTFOLD>(acc[i][j], lo32(s), lo32(t));
            acc[i][j + 1] = fold3<R, INTFOLD>(acc[i][j + 1], hi32(s), hi32(t));
          }
        }
      }
    };
    auto kpair = [&](int k) {
      const int aoff = ((((k >> 2) ^ ty) & 7) << 4) + ((k & 3) << 2);
      float4 b0[2], b1[2];
#pragma unroll
      for (int g = 0; g < 2; g++) {
        b0[g] = *reinterpret_cast<const float4*>(bs + k * TBN + 64 * g);
        b1[g] = *reinterpret_cast<const float4*>(bs + (k + 1) * TBN + 64 * g);
      }
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const float2 av = *reinterpret_cast<const float2*>(as + i * TT::ROW_STEP * 128 + aoff);
        fold_pair(i, av.x, av.y, b0, b1);
      }
    };
    int kdone = 0;
    if constexpr (QUAD) {
      // four k per step: B rows k..k+3 held in registers, one 16-byte A load
      // (k..k+3 are one swizzle chunk) per row — 16 shared loads per 256
      // (a, b) pairs instead of 24
      const int nquads = kend >> 2;
#pragma unroll UNR
      for (int kq = 0; kq < nquads; kq++) {
        const int k = 4 * kq;
        const int aoff = ((kq ^ ty) & 7) << 4;
        float4 bq[4][2];
#pragma unroll
        for (int r = 0; r < 4; r++)
#pragma unroll
          for (int g = 0; g < 2; g++)
            bq[r][g] = *reinterpret_cast<const float4*>(bs + (k + r) * TBN + 64 * g);
#pragma unroll
        for (int i = 0; i < 8; i++) {
          const float4 av = *reinterpret_cast<const float4*>(as + i * TT::ROW_STEP * 128 + aoff);
          fold_pair(i, av.x, av.y, bq[0], bq[1]);
          fold_pair(i, av.z, av.w, bq[2], bq[3]);
        }
      }
      kdone = 4 * nquads;
      if (kend - kdone >= 2) {
        kpair(kdone);
        kdone += 2;
      }
    } else {
      const int npairs = kend >> 1;
#pragma unroll UNR
      for (int kp = 0; kp < npairs; kp++) kpair(2 * kp);
      kdone = 2 * npairs;
    }
    if (kdone < kend) {  // lone last k: scalar combine + 2-input fold
      const int k = kend - 1;
      const int aoff = ((((k >> 2) ^ ty) & 7) << 4) + ((k & 3) << 2);
#pragma unroll
      for (int i = 0; i < 8; i++) {
        const float av = *reinterpret_cast<const float*>(as + i * TT::ROW_STEP * 128 + aoff);
#pragma unroll
        for (int g = 0; g < 2; g++)
#pragma unroll
          for (int cc = 0; cc < 4; cc++) {
            if constexpr (I32)
              acc[i][4 * g + cc] = iaddmnmx<C, R>(av, bs[k * TBN + 64 * g + cc], acc[i][4 * g + cc]);
            else
              acc[i][4 * g + cc] = ReduceOp<R>::f(acc[i][4 * g + cc],
                                                  CombineOp<C>::f(av, bs[k * TBN + 64 * g + cc]));
          }
      }
    }
    if constexpr (REFILL == 1) {
      // this warp's reads of the stage before the async proxy's refill, then
      // count the warp out; the last one (acq_rel: every other warp's reads
      // happen-before) refills the stage with slab kt + TSTAGES
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        unsigned before;
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(before)
                     : "r"(tma::smem_addr(&done_warps[stage]))
                     : "memory");
        if (before == TT::THREADS / 32 - 1) {
          // reset before the refill's expect_tx arrive (a release), which the
          // warps' next wait on this stage acquires
          done_warps[stage] = 0;
          if (kt + TSTAGES < KT) issue(stage, kt + TSTAGES);
        }
      }
    } else {
      tma::release_stage(&empty[stage], lane);
      // refill the slab consumed one iteration ago (its readers are long done)
      if (tid == 0 && kt >= 1 && kt - 1 + TSTAGES < KT) {
        const int ps = (int)((kt - 1) % TSTAGES);
        tma::mbar_wait(&empty[ps], (unsigned)(((kt - 1) / TSTAGES) & 1));
        issue(ps, kt - 1 + TSTAGES);
      }
    }
  }

  const bool vec_store = (ldc % 4 == 0) && (reinterpret_cast<uintptr_t>(c) % 16 == 0);
#pragma unroll
  for (int i = 0; i < 8; i++) {
    const int64_t row = m0 + ty + TT::ROW_STEP * i;
    if (row >= M) continue;
#pragma unroll
    for (int g = 0; g < 2; g++) {
      const int64_t col = n0 + 64 * g + 4 * tx;
      if (vec_store && col + 3 < N) {
        *reinterpret_cast<float4*>(c + row * ldc + col) =
            make_float4(acc[i][4 * g], acc[i][4 * g + 1], acc[i][4 * g + 2], acc[i][4 * g + 3]);
      } else {
#pragma unroll
        for (int cc = 0; cc < 4; cc++)
          if (col + cc < N) c[row * ldc + col + cc] = acc[i][4 * g + cc];
      }
    }
  }
}

// TMA needs 16-byte aligned bases and row strides and 32-bit coordinates
inline bool tropical_tma_eligible(const Problem& p) {
  return p.lda % 4 == 0 && p.ldb % 4 == 0 && reinterpret_cast<uintptr_t>(p.a) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(p.b) % 16 == 0 && p.M < (int64_t(1) << 31) &&
         p.N < (int64_t(1) << 31) && p.K < (int64_t(1) << 31) && p.lda < (int64_t(1) << 36) &&
         p.ldb < (int64_t(1) << 36) && tensor_maps_available();
}

template <int C, int R, int MODE, bool ACC, int MINB = 2, int UNR = 1, bool QUAD = false,
          int BMT = 128, int REFILL = 0, int FORM = 0>
cudaError_t tropical_tma_launch(const Problem& p, const unsigned* special) {
  using TT = TropTma<BMT>;
  CUtensorMap map_a, map_b;
  if (!make_tensor_map_2d(&map_a, p.a, 4, p.M, p.K, p.lda, TT::BM, TBK, true) ||
      !make_tensor_map_2d(&map_b, p.b, 4, p.K, p.N, p.ldb, TBK, TBN, false))
    return cudaErrorInvalidValue;
  auto kern = tropical_tma_kernel<C, R, MODE, ACC, MINB, UNR, QUAD, BMT, REFILL, FORM>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TT::SMEM);
  if (e != cudaSuccess) return e;
  const int64_t tiles_m = (p.M + TT::BM - 1) / TT::BM, tiles_n = (p.N + TBN - 1) / TBN;
  const int64_t tiles = tiles_m * tiles_n;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  kern<<<(unsigned)tiles, TT::THREADS, TT::SMEM, p.stream>>>(
      static_cast<float*>(p.c), p.M, p.N, p.K, p.ldc, special, tiles_m, tiles_n, map_a, map_b);
  count_launch();
  return cudaGetLastError();
}

// 128 x 128 CTA tiles once there are >= 256 of them (see tropical_launch)
inline bool tropical_big_tiles(const Problem& p) {
  return ((p.M + 127) / 128) * ((p.N + 127) / 128) >= 256;
}

template <int C, int R, int MODE, bool ACC>
cudaError_t tropical_launch(const Problem& p, const unsigned* special) {
  // TMA-staged kernel when the layout allows it (the first TMA version: 19.5
  // vs 18.6 T pairs/s at c5, profiles/r01_tune_tropical_tma.jsonl); bit-identical
  // 64 x 128 CTA tiles of 128 threads, three per SM (up to 168 registers per
  // thread), stepping four k at a time (B rows in registers, 16-byte A loads):
  // c5 217.9 ms vs 222.4 ms for 128 x 128 tiles of 256 threads (two per SM,
  // 128 registers) and 228.7 ms for those with the two-k step; 1000^3
  // 0.089 vs 0.146 ms (twice the CTAs) — profiles/r01_tune_tropical_quad.jsonl,
  // r01_tune_tropical_bm64.jsonl
  // Each stage is refilled by the last warp to release it (REFILL 1: c5 218.3
  // -> 211.2 ms, bit-identical, profiles/r02_tune_tropical_refill.jsonl).
  // With the last-warp refill, 128 x 128 tiles of 256 threads (two CTAs and
  // 16 warps per SM at 128 registers) overtake the 64 x 128 ones from 256 such
  // tiles up: c5 206.7 vs 211.2 ms, 2048^3 0.484 vs 0.516 ms, 1000^3 0.136 vs
  // 0.083 ms (profiles/r02_tune_tropical_bm128.jsonl).
  if (tropical_tma_eligible(p)) {
    if (tropical_big_tiles(p)) return tropical_tma_launch<C, R, MODE, ACC, 2, 1, true, 128, 1>(p, special);
    return tropical_tma_launch<C, R, MODE, ACC, 3, 1, true, 64, 1>(p, special);
  }
  const bool vec = (p.lda % 4 == 0) && (p.ldb % 4 == 0) &&
                   (reinterpret_cast<uintptr_t>(p.a) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(p.b) % 16 == 0);
  auto kern = vec ? tropical_kernel<C, R, MODE, ACC, true> : tropical_kernel<C, R, MODE, ACC, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TSMEM);
  if (e != cudaSuccess) return e;
  const int64_t tiles_m = (p.M + TBM - 1) / TBM, tiles_n = (p.N + TBN - 1) / TBN;
  const int64_t tiles = tiles_m * tiles_n;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  kern<<<(unsigned)tiles, TNT, TSMEM, p.stream>>>(
      static_cast<float*>(p.c), static_cast<const float*>(p.a), static_cast<const float*>(p.b),
      p.M, p.N, p.K, p.lda, p.ldb, p.ldc, special, tiles_m, tiles_n);
  count_launch();
  return cudaGetLastError();
}

}  // namespace
}  // namespace moa
