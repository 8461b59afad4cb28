// K1: the (multiply, add) float64 inner product on the FP64 tensor cores.
//
// Reference: _ckernel.pyx:37-52 (_rows_mul_add), the paper's row-of-C loop
// (PAPER.md:505-518): each row of B is scaled by one element of A and
// accumulated into the result row.  On B200 the FP64 tensor-core instruction
// is the warp-level mma.sync f64 (SASS DMMA.8x8x4, 64 FMA/clk/SM, measured
// 36.96 TFLOP/s in tools/peaks.cu); tcgen05 has no f64 kind, so this is the
// tensor-core path.  The kernel keeps the paper's formulation at tile scale:
// a 16-deep slab of A columns and the matching 16 rows of B are staged in
// shared memory and every B row of the slab is scaled and accumulated into
// the warp's register-resident block of C rows.
//
// Tiling: CTA tile BM x BN, warp tile WM x WN built from m16n8k4 MMAs (each a
// DMMA.8x8x4 pair); BK = 16 or 32; STAGES-deep cp.async pipeline (LDGSTS, 16-byte
// when rows are 16-byte aligned, else 8-byte), OOB elements zero-filled by
// the copy's src-size so edges need no branches in the main loop.
// Shared layouts are padded so every fragment LDS.64 is conflict-free:
//   A: row-major [BM][BK+4]  (A frag (g,t) -> slot 4g+t mod 16)
//   B: row-major [BK][BN+4]  (B frag (t,g) -> slot 4t+g mod 16)
//
// Determinism: every output element accumulates k in ascending 4-wide DMMA
// steps starting from k = 0 whatever the tile shape or the row range, so all
// tile configurations (and any row sharding across GPUs) give identical bits.
#include "moa_common.cuh"
#include "moa_kernels.h"
#include "../../include/moa_b200.h"

namespace moa {

namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5}, {%6}, "
      "{%0, %1, %2, %3};"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

template <int BM_, int BN_, int WM_, int WN_, int STAGES_, int BK_ = 16, int MINB_ = 1,
          bool PF_ = false, int GM_ = 8>
struct DmmaCfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_;
  static constexpr int DBK = BK_, MIN_BLOCKS = MINB_;
  static constexpr bool PREFETCH = PF_;  // load the next k4 step's fragments before the MMAs
  static constexpr int GROUP_M = GM_;    // row tiles per rasterisation group
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
  static constexpr int MI = WM / 16, NI = WN / 8;
  static constexpr int LDA_S = DBK + 4;  // doubles
  static constexpr int LDB_S = BN + 4;   // doubles
  static constexpr int A_STAGE = BM * LDA_S, B_STAGE = DBK * LDB_S;
  static constexpr size_t SMEM = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);
  static_assert(LDA_S % 16 == 4 && LDB_S % 16 == 4, "conflict-free padding");
};

template <class Cfg, bool VEC16, bool ACC>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MIN_BLOCKS)
    dmma_kernel(double* __restrict__ c, const double* __restrict__ a, const double* __restrict__ b,
                int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb, int64_t ldc,
                int64_t tiles_m, int64_t tiles_n) {
  constexpr int BM = Cfg::BM, BN = Cfg::BN, WM = Cfg::WM, WN = Cfg::WN, STAGES = Cfg::STAGES;
  constexpr int MI = Cfg::MI, NI = Cfg::NI, LDA_S = Cfg::LDA_S, LDB_S = Cfg::LDB_S;
  constexpr int THREADS = Cfg::THREADS, DBK = Cfg::DBK;
  extern __shared__ __align__(16) double dsm[];
  double* As = dsm;
  double* Bs = dsm + STAGES * Cfg::A_STAGE;

  const int64_t pid = blockIdx.x;
  constexpr int GM = Cfg::GROUP_M;
  const int64_t width = GM * tiles_n;
  const int64_t first_m = (pid / width) * GM;
  const int64_t gsize = (tiles_m - first_m) < GM ? (tiles_m - first_m) : GM;
  const int64_t m0 = (first_m + (pid % width) % gsize) * BM;
  const int64_t n0 = ((pid % width) / gsize) * BN;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / Cfg::WARPS_N) * WM, wn0 = (warp % Cfg::WARPS_N) * WN;
  const int g = lane >> 2, t = lane & 3;

  // ---- async tile copy (zero-filled outside M x K / K x N) ----
  auto load_stage = [&](int stage, int64_t k0) {
    double* as = As + stage * Cfg::A_STAGE;
    double* bs = Bs + stage * Cfg::B_STAGE;
    constexpr int EPC = VEC16 ? 2 : 1;  // elements per copy
    constexpr int A_CHUNKS = BM * DBK / EPC, B_CHUNKS = DBK * BN / EPC;
#pragma unroll
    for (int it = 0; it < (A_CHUNKS + THREADS - 1) / THREADS; it++) {
      const int ch = tid + it * THREADS;
      if (A_CHUNKS % THREADS == 0 || ch < A_CHUNKS) {
        const int r = ch / (DBK / EPC), kc = (ch % (DBK / EPC)) * EPC;
        const int64_t gm = m0 + r, gk = k0 + kc;
        int64_t rem = (gm < M) ? (K - gk) : 0;
        rem = rem < 0 ? 0 : (rem > EPC ? EPC : rem);
        const double* src = rem > 0 ? a + gm * lda + gk : a;
        if (VEC16) cp_async16(as + r * LDA_S + kc, src, (int)rem * 8);
        else cp_async8(as + r * LDA_S + kc, src, (int)rem * 8);
      }
    }
#pragma unroll
    for (int it = 0; it < (B_CHUNKS + THREADS - 1) / THREADS; it++) {
      const int ch = tid + it * THREADS;
      if (B_CHUNKS % THREADS == 0 || ch < B_CHUNKS) {
        const int r = ch / (BN / EPC), nc = (ch % (BN / EPC)) * EPC;
        const int64_t gk = k0 + r, gn = n0 + nc;
        int64_t rem = (gk < K) ? (N - gn) : 0;
        rem = rem < 0 ? 0 : (rem > EPC ? EPC : rem);
        const double* src = rem > 0 ? b + gk * ldb + gn : b;
        if (VEC16) cp_async16(bs + r * LDB_S + nc, src, (int)rem * 8);
        else cp_async8(bs + r * LDB_S + nc, src, (int)rem * 8);
      }
    }
  };

  double acc[MI][NI][4];
#pragma unroll
  for (int mi = 0; mi < MI; mi++)
#pragma unroll
    for (int ni = 0; ni < NI; ni++)
#pragma unroll
      for (int q = 0; q < 4; q++) {
        if (ACC) {
          const int64_t row = m0 + wm0 + mi * 16 + g + (q >> 1) * 8;
          const int64_t col = n0 + wn0 + ni * 8 + 2 * t + (q & 1);
          acc[mi][ni][q] = (row < M && col < N) ? c[row * ldc + col] : 0.0;
        } else {
          acc[mi][ni][q] = 0.0;
        }
      }

  const int64_t KT = (K + DBK - 1) / DBK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; s++) {
    if (s < KT) load_stage(s, (int64_t)s * DBK);
    cp_async_commit();
  }

  for (int64_t kt = 0; kt < KT; kt++) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int64_t nk = kt + STAGES - 1;
      if (nk < KT) load_stage((int)(nk % STAGES), nk * DBK);
      cp_async_commit();
    }
    const double* as = As + (int)(kt % STAGES) * Cfg::A_STAGE + (wm0 + g) * LDA_S + t;
    const double* bs = Bs + (int)(kt % STAGES) * Cfg::B_STAGE + t * LDB_S + wn0 + g;
    if constexpr (!Cfg::PREFETCH) {
#pragma unroll
      for (int kk = 0; kk < DBK; kk += 4) {
        double af[MI][2], bf[NI];
#pragma unroll
        for (int mi = 0; mi < MI; mi++) {
          af[mi][0] = as[(mi * 16) * LDA_S + kk];
          af[mi][1] = as[(mi * 16 + 8) * LDA_S + kk];
        }
#pragma unroll
        for (int ni = 0; ni < NI; ni++) bf[ni] = bs[kk * LDB_S + ni * 8];
#pragma unroll
        for (int mi = 0; mi < MI; mi++)
#pragma unroll
          for (int ni = 0; ni < NI; ni++) dmma_16x8x4(acc[mi][ni], af[mi][0], af[mi][1], bf[ni]);
      }
    } else {
      // software-pipelined fragments: step kk's MMAs issue while kk+4's loads fly
      double af[2][MI][2], bf[2][NI];
#pragma unroll
      for (int mi = 0; mi < MI; mi++) {
        af[0][mi][0] = as[(mi * 16) * LDA_S];
        af[0][mi][1] = as[(mi * 16 + 8) * LDA_S];
      }
#pragma unroll
      for (int ni = 0; ni < NI; ni++) bf[0][ni] = bs[ni * 8];
#pragma unroll
      for (int kk = 0; kk < DBK; kk += 4) {
        const int cur = (kk / 4) & 1, nxt = cur ^ 1;
        if (kk + 4 < DBK) {
#pragma unroll
          for (int mi = 0; mi < MI; mi++) {
            af[nxt][mi][0] = as[(mi * 16) * LDA_S + kk + 4];
            af[nxt][mi][1] = as[(mi * 16 + 8) * LDA_S + kk + 4];
          }
#pragma unroll
          for (int ni = 0; ni < NI; ni++) bf[nxt][ni] = bs[(kk + 4) * LDB_S + ni * 8];
        }
#pragma unroll
        for (int mi = 0; mi < MI; mi++)
#pragma unroll
          for (int ni = 0; ni < NI; ni++)
            dmma_16x8x4(acc[mi][ni], af[cur][mi][0], af[cur][mi][1], bf[cur][ni]);
      }
    }
  }
  cp_async_wait<0>();

  // ---- epilogue: each thread holds (g, 2t..2t+1) and (g+8, 2t..2t+1) of every 16x8 block
  const bool pair_ok = (ldc % 2 == 0) && (reinterpret_cast<uintptr_t>(c) % 16 == 0);
#pragma unroll
  for (int mi = 0; mi < MI; mi++)
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int64_t row = m0 + wm0 + mi * 16 + g + h * 8;
      if (row >= M) continue;
      double* crow = c + row * ldc;
#pragma unroll
      for (int ni = 0; ni < NI; ni++) {
        const int64_t col = n0 + wn0 + ni * 8 + 2 * t;
        if (pair_ok && col + 1 < N) {
          *reinterpret_cast<double2*>(crow + col) =
              make_double2(acc[mi][ni][2 * h], acc[mi][ni][2 * h + 1]);
        } else {
          if (col < N) crow[col] = acc[mi][ni][2 * h];
          if (col + 1 < N) crow[col + 1] = acc[mi][ni][2 * h + 1];
        }
      }
    }
}

template <class Cfg, bool VEC16, bool ACC>
cudaError_t dmma_launch(const Problem& p) {
  auto kern = dmma_kernel<Cfg, VEC16, ACC>;
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
  if (e != cudaSuccess) return e;
  const int64_t tiles_m = (p.M + Cfg::BM - 1) / Cfg::BM, tiles_n = (p.N + Cfg::BN - 1) / Cfg::BN;
  const int64_t tiles = tiles_m * tiles_n;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  kern<<<(unsigned)tiles, Cfg::THREADS, Cfg::SMEM, p.stream>>>(
      static_cast<double*>(p.c), static_cast<const double*>(p.a), static_cast<const double*>(p.b),
      p.M, p.N, p.K, p.lda, p.ldb, p.ldc, tiles_m, tiles_n);
  count_launch();
  return cudaGetLastError();
}

// Tile configurations (tools/tune_dmma.cu sweep, profiles/r01_tune_dmma*.jsonl):
// large: 64x128 CTA, 8 warps of 32x32, 4 stages, 2 CTAs/SM  -> 88.9% of peak at c4;
//        groups of 16 row tiles (tools/traffic_dmma.cu: 83 GB of DRAM reads per c4
//        launch vs 94 GB for 8, same time)
// medium: 64x64 CTA, 4 warps of 32x32, 3 stages, 3 CTAs/SM
// small: 32x32 CTA, 4 warps of 16x16, BK=32 (few k-tile round trips)
// tiny: 16x32 CTA, 4 warps of 16x8: the most warps for problems that give
//       fewer than 148 small tiles (c1: 8.7 vs 10.8 us; one warp already
//       saturates its sub-partition's DMMA pipe, tools/mb_dmma_latency.cu);
//       8 stages keep a whole 256-deep K in flight (cold-cache ncu: 7.0 vs
//       8.0 us at c1)
using CfgLarge = DmmaCfg<64, 128, 32, 32, 4, 16, 2, false, 16>;
using CfgMedium = DmmaCfg<64, 64, 32, 32, 3, 16, 3>;
using CfgSmall = DmmaCfg<32, 32, 16, 16, 3, 32, 1>;
using CfgTiny = DmmaCfg<16, 32, 16, 8, 8, 32, 1>;

template <class Cfg>
cudaError_t dmma_dispatch(const Problem& p) {
  const bool vec16 = (p.lda % 2 == 0) && (p.ldb % 2 == 0) &&
                     (reinterpret_cast<uintptr_t>(p.a) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(p.b) % 16 == 0);
  if (vec16)
    return p.accumulate ? dmma_launch<Cfg, true, true>(p) : dmma_launch<Cfg, true, false>(p);
  return p.accumulate ? dmma_launch<Cfg, false, true>(p) : dmma_launch<Cfg, false, false>(p);
}

}  // namespace

cudaError_t launch_dmma(const Problem& p) {
  // all configurations give identical bits (k order is fixed), so the choice
  // only has to fill the 148 SMs
  auto tiles = [&](int bm, int bn) { return ((p.M + bm - 1) / bm) * ((p.N + bn - 1) / bn); };
  // TMA-staged 64x64 kernel (dmma_tma.cu) once it fills the SMs: 96.9% of the
  // DMMA peak at c4 vs 88.9% for the cp.async kernels
  // (profiles/r01_tune_dmma_tma_cfgs.jsonl); below that its 16x32-tile form
  // (more CTAs; profiles/r01_tune_dmma_tiny.jsonl: at or below the cp.async
  // tiny/small tiles on every shape tried)
  if (dmma_tma_eligible(p))
    return tiles(64, 64) >= kNumSMs ? launch_dmma_tma(p) : launch_dmma_tma_tiny(p);
  // unaligned operands: per-thread cp.async tiles
  if (tiles(64, 128) >= 2 * kNumSMs) return dmma_dispatch<CfgLarge>(p);
  if (tiles(64, 64) >= kNumSMs) return dmma_dispatch<CfgMedium>(p);
  if (tiles(32, 32) >= kNumSMs) return dmma_dispatch<CfgSmall>(p);
  return dmma_dispatch<CfgTiny>(p);
}

}  // namespace moa
