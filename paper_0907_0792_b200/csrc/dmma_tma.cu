// K1 with TMA staging: the (multiply, add) float64 kernel of dmma.cu with its
// operand tiles brought in by the Tensor Memory Accelerator
// (cp.async.bulk.tensor, SASS UTMALDG) instead of per-thread cp.async.
//
// One elected thread issues, per 16-deep k-slab, one 2-D TMA box of A
// (64 rows x 16 doubles) and eight boxes of B (16 rows x 16 doubles), all
// completing on one mbarrier per pipeline stage; the other threads only wait
// on that barrier and run DMMA.  TMA zero-fills everything outside M x K and
// K x N, so edges need no code at all.
//
// Boxes land with the 128-byte swizzle (16-byte chunk c of 128-byte line r
// stored at chunk c ^ (r & 7)).  The m16n8k4 fragment pattern would still hit
// the same banks four times per half-warp, so the MMA rows and columns are
// relabelled instead of the data: MMA row g of a 16-row block reads tile row
// sigma(g) = 2(g&3) + ((g>>2)&1) + 8(g>>3), and MMA column g of the n8 block
// pair (2q, 2q+1) reads tile column 16q + pi(g) with pi = {0,1,8,9,2,3,10,11}
// / {4,5,12,13,6,7,14,15}.  Every fragment LDS.64 is then conflict-free, and
// the epilogue writes each accumulator pair to the relabelled (still
// contiguous) positions.  Each C element still accumulates k in ascending
// 4-wide DMMA steps from k = 0, so the bits equal every dmma.cu configuration.
#include "moa_common.cuh"
#include "tma.cuh"
#include "moa_kernels.h"
#include "../../include/moa_b200.h"

namespace moa {

namespace {

// BM x BN CTA tile of (BM/WM)*(BN/WN) warps, WM x WN warp tiles (multiples of
// 16: the relabelling works on 16-row blocks and pairs of n8 blocks), 16-deep
// slabs in STAGES pipeline stages, MINB CTAs per SM, GM-row-tile raster groups
// REFILL 0: thread 0 refills a stage once every warp has released it (an
// `empty` mbarrier per stage: warp 0 waits for the slowest warp); REFILL 1: the
// last warp to finish with a stage refills it at once (a shared counter).
template <int BM_, int BN_, int WM_, int WN_, int STAGES_, int MINB_, int GM_, int REFILL_ = 0>
struct TmaCfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int GM = GM_, BK = 16, REFILL = REFILL_;
  static constexpr int WARPS = (BM / WM) * (BN / WN), THREADS = 32 * WARPS;
  static constexpr int MI = WM / 16, NI = WN / 8;
  static constexpr int A_BYTES = BM * BK * 8, B_BYTES = BK * BN * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 /*align*/ + 20 * STAGES;
  static_assert(WM % 16 == 0 && WN % 16 == 0 && BM % WM == 0 && BN % WN == 0, "tile shape");
  static_assert(BM <= 256, "one TMA box of A per slab");
};
// 4 warps of 32x32, three CTAs per SM: 96.9% of the DMMA peak at c4 and 94.9%
// at c3 (vs 93.4% / 92.6% for 64x128 with 8 warps), profiles/r01_tune_dmma_tma_cfgs.jsonl;
// last-warp refill: c4 246.2 -> 243.6 ms (97.7%), c3 unchanged, bit-identical
// (profiles/r02_tune_dmma_refill.jsonl)
using TmaMain = TmaCfg<64, 64, 32, 32, 4, 3, 8, 1>;

using tma::load_2d;
using tma::mbar_arrive;
using tma::mbar_expect_tx;
using tma::mbar_init;
using tma::mbar_wait;

__device__ __forceinline__ void dmma_step(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5}, {%6}, "
      "{%0, %1, %2, %3};"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// tile row of MMA row g (0..15) inside a 16-row block; tile column offset of
// MMA column g (0..7) for the even (h=0) / odd (h=1) n8 block of a pair
__device__ __forceinline__ int sigma(int g) { return 2 * (g & 3) + ((g >> 2) & 1) + 8 * (g >> 3); }
__device__ __forceinline__ int pi_col(int g, int h) {
  return ((g >> 1) & 1) * 8 + (g & 1) + 2 * (g >> 2) + 4 * h;
}
// byte offset of element (r, k) in a swizzled A stage (BM lines of 128 B)
__device__ __forceinline__ int a_off(int r, int k) {
  return r * 128 + ((((k >> 1) ^ r) & 7) << 4) + ((k & 1) << 3);
}
// byte offset of element (k, n) in a swizzled B stage (8 boxes of 16 lines x 128 B)
__device__ __forceinline__ int b_off(int k, int n) {
  return (n >> 4) * 2048 + k * 128 + (((((n & 15) >> 1) ^ k) & 7) << 4) + ((n & 1) << 3);
}

// TPC (tiles per CTA): 1 = one tile per CTA (production); 0 = persistent,
// gridDim.x <= tiles CTAs (one per resident slot) taking tiles blockIdx.x,
// blockIdx.x + gridDim.x, ...; n >= 2 = tiles n*blockIdx.x .. n*blockIdx.x+n-1.
// A CTA with several tiles streams their k-slabs back to back: the refills
// run ahead into the next tile's first slabs while this tile's last slabs and
// epilogue run, so a short-K tile pays no TMA round trip at its start.
template <class Cfg, bool ACC, int TPC = 1>
__global__ void __launch_bounds__(Cfg::THREADS, Cfg::MINB)
    dmma_tma_kernel(double* __restrict__ c, int64_t M, int64_t N, int64_t K, int64_t ldc,
                    int64_t tiles_m, int64_t tiles_n, const __grid_constant__ CUtensorMap map_a,
                    const __grid_constant__ CUtensorMap map_b) {
  static_assert(TPC == 1 || Cfg::REFILL == 1, "a multi-tile slab stream refills from the last warp");
  constexpr bool MULTI = TPC != 1;
  extern __shared__ __align__(16) unsigned char tm_raw[];
  // swizzle-128B destinations must be 1024-byte aligned
  // (offset from tm_raw rather than integer rounding of the pointer, so the
  // compiler keeps the shared address space: LDS, not generic LD)
  unsigned char* base = tma::align1k(tm_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;  // one arrival per warp when it is done with a slab
  unsigned* done_warps = reinterpret_cast<unsigned*>(empty + Cfg::STAGES);  // REFILL 1

  // origin of this CTA's local tile `lt` (row-tile raster groups of GM); the
  // launcher keeps tile indices below 2^31, so 32-bit divisions suffice
  auto origin = [&](int64_t lt, int64_t& m0, int64_t& n0) {
    const uint32_t pid = TPC == 0   ? blockIdx.x + (uint32_t)lt * gridDim.x
                         : TPC == 1 ? blockIdx.x
                                    : blockIdx.x * (uint32_t)TPC + (uint32_t)lt;
    const uint32_t width = Cfg::GM * (uint32_t)tiles_n;
    const uint32_t first_m = (pid / width) * Cfg::GM;
    const uint32_t gsize = ((uint32_t)tiles_m - first_m) < Cfg::GM ? ((uint32_t)tiles_m - first_m) : Cfg::GM;
    const uint32_t r = pid % width;
    m0 = (int64_t)(first_m + r % gsize) * Cfg::BM;
    n0 = (int64_t)(r / gsize) * Cfg::BN;
  };
  int64_t my_tiles = 1;
  if constexpr (TPC == 0) {
    my_tiles = (tiles_m * tiles_n - (int64_t)blockIdx.x + gridDim.x - 1) / gridDim.x;
  } else if constexpr (TPC > 1) {
    const int64_t rest = tiles_m * tiles_n - (int64_t)blockIdx.x * TPC;
    my_tiles = rest < TPC ? rest : TPC;
  }

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / (Cfg::BN / Cfg::WN)) * Cfg::WM, wn0 = (warp % (Cfg::BN / Cfg::WN)) * Cfg::WN;
  const int g = lane >> 2, t = lane & 3;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < Cfg::STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::WARPS);
      done_warps[s] = 0;
    }
    tma::mbar_init_fence();
  }
  __syncthreads();

  // slab s of the CTA's stream: k-slab s % KT of local tile s / KT
  const int64_t KT = (K + Cfg::BK - 1) / Cfg::BK;
  const int64_t total = my_tiles * KT;
  auto issue = [&](int stage, int64_t s) {  // one thread
    int64_t tm0 = 0, tn0 = 0;
    // (MULTI: the launcher keeps each CTA's slab count below 2^31)
    origin(MULTI ? (uint32_t)s / (uint32_t)KT : 0, tm0, tn0);
    const int64_t kt = MULTI ? (uint32_t)s % (uint32_t)KT : s;
    unsigned char* st = base + stage * Cfg::STAGE_BYTES;
    mbar_expect_tx(&full[stage], Cfg::STAGE_BYTES);
    load_2d(st, &map_a, (int)(kt * Cfg::BK), (int)tm0, &full[stage]);
#pragma unroll
    for (int j = 0; j < Cfg::BN / 16; j++)
      load_2d(st + Cfg::A_BYTES + j * 2048, &map_b, (int)(tn0 + 16 * j), (int)(kt * Cfg::BK),
                  &full[stage]);
  };
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < Cfg::STAGES; s++)
      if (s < total) issue(s, s);
  }

  // per-thread fragment offsets (bytes within a stage), fixed for the kernel
  int a_row[Cfg::MI][2];
#pragma unroll
  for (int mi = 0; mi < Cfg::MI; mi++) {
    a_row[mi][0] = wm0 + mi * 16 + sigma(g);
    a_row[mi][1] = wm0 + mi * 16 + sigma(g + 8);
  }
  int b_col[Cfg::NI];
#pragma unroll
  for (int ni = 0; ni < Cfg::NI; ni++) b_col[ni] = wn0 + 16 * (ni >> 1) + pi_col(g, ni & 1);
  const bool pair_ok = (ldc % 2 == 0) && (reinterpret_cast<uintptr_t>(c) % 16 == 0);

#pragma unroll 1
  for (int64_t lt = 0; lt < my_tiles; lt++) {
    int64_t m0, n0;
    origin(lt, m0, n0);
    // accumulator (mi, ni, q) is C element (a_row[mi][q>>1], pi(2t + (q&1)))
    double acc[Cfg::MI][Cfg::NI][4];
#pragma unroll
    for (int mi = 0; mi < Cfg::MI; mi++)
#pragma unroll
      for (int ni = 0; ni < Cfg::NI; ni++)
#pragma unroll
        for (int q = 0; q < 4; q++) {
          if (ACC) {
            const int64_t row = m0 + a_row[mi][q >> 1];
            const int64_t col = n0 + wn0 + 16 * (ni >> 1) + pi_col(2 * t, ni & 1) + (q & 1);
            acc[mi][ni][q] = (row < M && col < N) ? c[row * ldc + col] : 0.0;
          } else {
            acc[mi][ni][q] = 0.0;
          }
        }

    // No block-wide barrier in the main loop: warps release a slab through its
    // `empty` mbarrier (REFILL 0: thread 0 refills the slab consumed one
    // iteration earlier) or the last warp out refills it (REFILL 1), keeping
    // up to STAGES slabs in flight ahead.
    for (int64_t kt = 0; kt < KT; kt++) {
      const int64_t s = lt * KT + kt;
      const int stage = (int)(s % Cfg::STAGES);
      mbar_wait(&full[stage], (unsigned)((s / Cfg::STAGES) & 1));
      const unsigned char* as = base + stage * Cfg::STAGE_BYTES;
      const unsigned char* bs = as + Cfg::A_BYTES;
#pragma unroll
      for (int kk = 0; kk < Cfg::BK; kk += 4) {
        double af[Cfg::MI][2], bf[Cfg::NI];
#pragma unroll
        for (int mi = 0; mi < Cfg::MI; mi++) {
          af[mi][0] = *reinterpret_cast<const double*>(as + a_off(a_row[mi][0], kk + t));
          af[mi][1] = *reinterpret_cast<const double*>(as + a_off(a_row[mi][1], kk + t));
        }
#pragma unroll
        for (int ni = 0; ni < Cfg::NI; ni++)
          bf[ni] = *reinterpret_cast<const double*>(bs + b_off(kk + t, b_col[ni]));
#pragma unroll
        for (int mi = 0; mi < Cfg::MI; mi++)
#pragma unroll
          for (int ni = 0; ni < Cfg::NI; ni++) dmma_step(acc[mi][ni], af[mi][0], af[mi][1], bf[ni]);
      }
      if constexpr (Cfg::REFILL == 1) {
        // count this warp out of the stage (its reads ordered before the async
        // proxy's refill); the last warp out refills it with slab s + STAGES
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          unsigned before;
          asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                       : "=r"(before)
                       : "r"(tma::smem_addr(&done_warps[stage]))
                       : "memory");
          if (before == Cfg::WARPS - 1) {
            done_warps[stage] = 0;  // before the refill's expect_tx arrive (a release)
            if (s + Cfg::STAGES < total) issue(stage, s + Cfg::STAGES);
          }
        }
      } else {
        tma::release_stage(&empty[stage], lane);
        // refill the slab of iteration s-1 with slab s-1+STAGES
        if (tid == 0 && s >= 1 && s - 1 + Cfg::STAGES < total) {
          const int ps = (int)((s - 1) % Cfg::STAGES);
          mbar_wait(&empty[ps], (unsigned)(((s - 1) / Cfg::STAGES) & 1));
          issue(ps, s - 1 + Cfg::STAGES);
        }
      }
    }

    // ---- epilogue: accumulator (q&1) of MMA column 2t -> tile columns pi(2t), pi(2t+1)
#pragma unroll
    for (int mi = 0; mi < Cfg::MI; mi++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int64_t row = m0 + a_row[mi][h];
        if (row >= M) continue;
        double* crow = c + row * ldc;
#pragma unroll
        for (int ni = 0; ni < Cfg::NI; ni++) {
          const int64_t col = n0 + wn0 + 16 * (ni >> 1) + pi_col(2 * t, ni & 1);
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
}

template <class Cfg, int TPC = 1>
cudaError_t dmma_tma_launch(const Problem& p) {
  CUtensorMap map_a, map_b;
  if (!make_tensor_map_2d(&map_a, p.a, 8, p.M, p.K, p.lda, Cfg::BM, 16, true) ||
      !make_tensor_map_2d(&map_b, p.b, 8, p.K, p.N, p.ldb, Cfg::BK, 16, true))
    return cudaErrorInvalidValue;
  auto kern = p.accumulate ? dmma_tma_kernel<Cfg, true, TPC> : dmma_tma_kernel<Cfg, false, TPC>;
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM);
  if (e != cudaSuccess) return e;
  const int64_t tiles_m = (p.M + Cfg::BM - 1) / Cfg::BM, tiles_n = (p.N + Cfg::BN - 1) / Cfg::BN;
  const int64_t tiles = tiles_m * tiles_n;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  int64_t grid = tiles;
  if constexpr (TPC == 0) {
    const int64_t slots = (int64_t)sm_count() * Cfg::MINB;
    grid = tiles < slots ? tiles : slots;
  } else if constexpr (TPC > 1) {
    grid = (tiles + TPC - 1) / TPC;
  }
  if (TPC != 1) {
    const int64_t per_cta = (tiles + grid - 1) / grid * ((p.K + Cfg::BK - 1) / Cfg::BK);
    if (per_cta >= (int64_t(1) << 31)) return cudaErrorInvalidConfiguration;
  }
  kern<<<(unsigned)grid, Cfg::THREADS, Cfg::SMEM, p.stream>>>(
      static_cast<double*>(p.c), p.M, p.N, p.K, p.ldc, tiles_m, tiles_n, map_a, map_b);
  count_launch();
  return cudaGetLastError();
}

// ---- tiny problems (fewer than one wave of 64x64 tiles, e.g. BASELINE c1) ----
// 16 x 32 CTA tiles of four 16 x 8 warps: one DMMA chain per warp, the most
// warps such a problem gives (one warp already saturates its sub-partition's
// DMMA pipe, tools/mb_dmma_latency.cu).  The cp.async version of this tile
// spends ~35 issue slots per DMMA on per-thread copy addressing and
// bounds arithmetic with one warp per scheduler (ncu: 2209 instructions per
// warp for 64 DMMAs, every slot ~4 cycles apart); here one thread issues two
// TMA boxes per 32-deep slab and the warps only wait, load fragments and MMA.
// No swizzle: the boxes are four doubles wider than the slab (A: 16 x 36,
// B: 32 x 36 — the extra columns are the neighbouring slab/tile, or TMA's zero
// fill, and are never read), so rows sit 288 bytes apart and every m16n8k4
// fragment LDS.64 (A[g][k+t], B[k+t][g]) covers each bank once per half-warp.
// Plain MMA rows/columns, k ascending in 4-wide DMMA steps from k = 0: the
// bits equal every other K1 configuration.
struct TinyCfg {
  static constexpr int BM = 16, BN = 32, BK = 32, PAD = 4, WARPS = BN / 8, THREADS = 32 * WARPS;
  static constexpr int A_PITCH = BK + PAD, B_PITCH = BN + PAD;  // doubles
  static constexpr int A_BYTES = BM * A_PITCH * 8, B_BYTES = BK * B_PITCH * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static_assert(A_BYTES % 128 == 0 && STAGE_BYTES % 128 == 0, "TMA destinations 128-byte aligned");
};

template <int STAGES, bool ACC>
__global__ void __launch_bounds__(TinyCfg::THREADS, 1)
    dmma_tiny_tma_kernel(double* __restrict__ c, int64_t M, int64_t N, int64_t K, int64_t ldc,
                         int64_t tiles_n, const __grid_constant__ CUtensorMap map_a,
                         const __grid_constant__ CUtensorMap map_b) {
  using T = TinyCfg;
  extern __shared__ __align__(128) unsigned char tt_raw[];
  unsigned char* base = tt_raw + ((128u - (tma::smem_addr(tt_raw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * T::STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  const int64_t m0 = (blockIdx.x / tiles_n) * T::BM, n0 = (blockIdx.x % tiles_n) * T::BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3, wn0 = 8 * warp;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], T::WARPS);
    }
    tma::mbar_init_fence();
  }
  __syncthreads();

  const int64_t KT = (K + T::BK - 1) / T::BK;
  auto issue = [&](int stage, int64_t kt) {  // one thread
    unsigned char* st = base + stage * T::STAGE_BYTES;
    mbar_expect_tx(&full[stage], T::STAGE_BYTES);
    load_2d(st, &map_a, (int)(kt * T::BK), (int)m0, &full[stage]);
    load_2d(st + T::A_BYTES, &map_b, (int)n0, (int)(kt * T::BK), &full[stage]);
  };
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < STAGES; s++)
      if (s < KT) issue(s, s);
  }

  double acc[4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    if (ACC) {
      const int64_t row = m0 + g + (q >> 1) * 8, col = n0 + wn0 + 2 * t + (q & 1);
      acc[q] = (row < M && col < N) ? c[row * ldc + col] : 0.0;
    } else {
      acc[q] = 0.0;
    }
  }

  for (int64_t kt = 0; kt < KT; kt++) {
    const int stage = (int)(kt % STAGES);
    mbar_wait(&full[stage], (unsigned)((kt / STAGES) & 1));
    const double* as = reinterpret_cast<const double*>(base + stage * T::STAGE_BYTES);
    const double* bs = reinterpret_cast<const double*>(base + stage * T::STAGE_BYTES + T::A_BYTES);
    const double* a0p = as + g * T::A_PITCH + t;
    const double* a1p = a0p + 8 * T::A_PITCH;
    const double* bp = bs + t * T::B_PITCH + wn0 + g;
#pragma unroll
    for (int kk = 0; kk < T::BK; kk += 4)
      dmma_step(acc, a0p[kk], a1p[kk], bp[kk * T::B_PITCH]);
    tma::release_stage(&empty[stage], lane);
    if (tid == 0 && kt >= 1 && kt - 1 + STAGES < KT) {
      const int ps = (int)((kt - 1) % STAGES);
      mbar_wait(&empty[ps], (unsigned)(((kt - 1) / STAGES) & 1));
      issue(ps, kt - 1 + STAGES);
    }
  }

  const bool pair_ok = (ldc % 2 == 0) && (reinterpret_cast<uintptr_t>(c) % 16 == 0);
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int64_t row = m0 + g + 8 * h, col = n0 + wn0 + 2 * t;
    if (row >= M) continue;
    double* crow = c + row * ldc;
    if (pair_ok && col + 1 < N) {
      *reinterpret_cast<double2*>(crow + col) = make_double2(acc[2 * h], acc[2 * h + 1]);
    } else {
      if (col < N) crow[col] = acc[2 * h];
      if (col + 1 < N) crow[col + 1] = acc[2 * h + 1];
    }
  }
}

// 8 stages keep a whole 256-deep K (c1) in flight
template <int STAGES = 8>
cudaError_t dmma_tiny_tma_launch(const Problem& p) {
  using T = TinyCfg;
  CUtensorMap map_a, map_b;
  if (!make_tensor_map_2d(&map_a, p.a, 8, p.M, p.K, p.lda, T::BM, T::A_PITCH, false) ||
      !make_tensor_map_2d(&map_b, p.b, 8, p.K, p.N, p.ldb, T::BK, T::B_PITCH, false))
    return cudaErrorInvalidValue;
  auto kern = p.accumulate ? dmma_tiny_tma_kernel<STAGES, true> : dmma_tiny_tma_kernel<STAGES, false>;
  const size_t smem = (size_t)STAGES * T::STAGE_BYTES + 128 + 16 * STAGES;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t tiles_m = (p.M + T::BM - 1) / T::BM, tiles_n = (p.N + T::BN - 1) / T::BN;
  const int64_t tiles = tiles_m * tiles_n;
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  kern<<<(unsigned)tiles, T::THREADS, smem, p.stream>>>(static_cast<double*>(p.c), p.M, p.N, p.K,
                                                        p.ldc, tiles_n, map_a, map_b);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

bool dmma_tma_eligible(const Problem& p) {
  // TMA: 16-byte aligned bases and row strides, 32-bit coordinates.  The
  // tensor map's global strides must also be below 2^40 bytes.
  return p.lda % 2 == 0 && p.ldb % 2 == 0 &&
         reinterpret_cast<uintptr_t>(p.a) % 16 == 0 && reinterpret_cast<uintptr_t>(p.b) % 16 == 0 &&
         p.M < (int64_t(1) << 31) && p.N < (int64_t(1) << 31) && p.K < (int64_t(1) << 31) &&
         p.lda < (int64_t(1) << 36) && p.ldb < (int64_t(1) << 36) && tensor_maps_available();
}

cudaError_t launch_dmma_tma(const Problem& p) { return dmma_tma_launch<TmaMain>(p); }

// 8 stages (110 KB, whole K of c1 in flight) while the grid fits one CTA per
// SM; beyond that 4 stages, so four CTAs share an SM
// (profiles/r01_tune_dmma_tiny.jsonl: c1 8.2 vs 9.0 us; 1024x256x512 16.4 vs 20.5 us)
cudaError_t launch_dmma_tma_tiny(const Problem& p) {
  const int64_t tiles = ((p.M + TinyCfg::BM - 1) / TinyCfg::BM) * ((p.N + TinyCfg::BN - 1) / TinyCfg::BN);
  return tiles <= kNumSMs ? dmma_tiny_tma_launch<8>(p) : dmma_tiny_tma_launch<4>(p);
}

}  // namespace moa
