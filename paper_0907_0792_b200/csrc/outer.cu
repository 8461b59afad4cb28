// K3: the write-streaming outer-product kernel, and the identity fill.
//
// The outer product is the rowsinred = 1 case of the reference's unified loop
// (kernel.py:95-108; _ckernel.pyx:45-52 / 64-72 with l = 0 only):
//     res[i*restride + j] = reduce(res[i*restride + j], combine(a[i*lstride], b[j]))
// with res prefilled by the identity (kernel.py:149).  Here the identity lives
// in a register, so the kernel never reads C: per element it is one combine,
// one reduce against the identity (which keeps the reference's +0.0 for an add
// reduce of a -0.0 combine result) and one streaming store.  The roofline is
// the HBM write bandwidth; A (one value per row) and B (one row) are tiny and
// stay in L1/L2, B in registers.
//
// Layout: thread x of the grid owns a fixed 32-byte column chunk of every row
// (4 doubles / 8 floats), loads its B chunk once, then walks its block's run
// of consecutive rows issuing one 256-bit st.global.cs per row
// (STG.E.EF.ENL2.256).  A warp writes 1 KiB of contiguous row per store.
#include <type_traits>

#include "moa_common.cuh"
#include "moa_kernels.h"
#include "../../include/moa_b200.h"

namespace moa {

namespace {

__device__ __forceinline__ void st_stream_32B(double* p, const double (&v)[4]) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v[0]), "d"(v[1]),
               "d"(v[2]), "d"(v[3])
               : "memory");
}
__device__ __forceinline__ void st_stream_32B(float* p, const float (&v)[8]) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]),
               "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
__device__ __forceinline__ void st_stream_32B(int64_t* p, const int64_t (&v)[4]) {
  asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v[0]), "l"(v[1]),
               "l"(v[2]), "l"(v[3])
               : "memory");
}
__device__ __forceinline__ void st_stream_32B(int32_t* p, const int32_t (&v)[8]) {
  asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void ld_32B(const int64_t* p, int64_t (&v)[4]) {
  asm volatile("ld.global.v4.b64 {%0, %1, %2, %3}, [%4];"
               : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3])
               : "l"(p));
}
__device__ __forceinline__ void ld_32B(const int32_t* p, int32_t (&v)[8]) {
  asm volatile("ld.global.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                 "=r"(v[6]), "=r"(v[7])
               : "l"(p));
}
__device__ __forceinline__ void ld_32B(const double* p, double (&v)[4]) {
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3])
               : "l"(p));
}
__device__ __forceinline__ void ld_32B(const float* p, float (&v)[8]) {
  asm volatile("ld.global.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
                 "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}

// one result element: reduce(init, combine(a, b)) in the accumulation type
template <typename T, int C, int R>
__device__ __forceinline__ T outer_elem(T av, T bv, T init) {
  using A = typename AccType<T, C, R>::type;
  A v = CombineOp<C>::f(A(av), A(bv));
  return convert<T, A>(ReduceOp<R>::f(A(init), v));
}

template <typename T, int C, int R, bool ACC>
__global__ void __launch_bounds__(256) outer_vec_kernel(T* __restrict__ c, const T* __restrict__ a,
                                                        const T* __restrict__ b, int64_t M,
                                                        int64_t NV, int64_t lda, int64_t ldc,
                                                        int64_t rows_per_block) {
  constexpr int V = 32 / sizeof(T);
  const int64_t jv = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (jv >= NV) return;
  T bv[V];
#pragma unroll
  for (int q = 0; q < V; q++) bv[q] = __ldg(b + jv * V + q);
  const T ident = ReduceOp<R>::template identity<T>();
  T* cp = c + jv * V;
  const int64_t r0 = blockIdx.y * rows_per_block;
  const int64_t r1 = (r0 + rows_per_block) < M ? (r0 + rows_per_block) : M;
  using A = typename AccType<T, C, R>::type;
  if constexpr (C == C_DIV && std::is_integral<A>::value) {
    // the thread's V divisors serve every row of its run: one multiplier each
    // (div_magic / idiv_magic, moa_common.cuh)
    using G = decltype(div_magic(A(0)));
    using U = typename IntTraits<A>::U;
    G gv[V];
#pragma unroll
    for (int q = 0; q < V; q++) gv[q] = div_magic(A(bv[q]));
#pragma unroll 2
    for (int64_t i = r0; i < r1; i++) {
      const A av = A(__ldg(a + i * lda));
      const U nx = av < 0 ? U(0) - U(av) : U(av);
      T out[V];
      if (ACC) ld_32B(cp + i * ldc, out);
#pragma unroll
      for (int q = 0; q < V; q++)
        out[q] = convert<T, A>(ReduceOp<R>::f(A(ACC ? out[q] : ident), idiv_magic(av, nx, A(bv[q]), gv[q])));
      st_stream_32B(cp + i * ldc, out);
    }
  } else if constexpr (C == C_DIV && std::is_same<A, double>::value) {
    // the thread's V divisors are reused by every row of its run: one
    // reciprocal each (div_candidate, moa_common.cuh)
    double yv[V];
#pragma unroll
    for (int q = 0; q < V; q++) {
      const double bd = double(A(bv[q]));
      yv[q] = rcp_range(bd) ? rcp_rn(bd) : __longlong_as_double(0x7ff8000000000000ll);
    }
#pragma unroll 2
    for (int64_t i = r0; i < r1; i++) {
      const A av = A(__ldg(a + i * lda));
      A quo[V];
      bool ok = rcp_range(av);
#pragma unroll
      for (int q = 0; q < V; q++) quo[q] = div_candidate(av, A(bv[q]), yv[q], ok);
      if (!ok) {
#pragma unroll
        for (int q = 0; q < V; q++) quo[q] = CombineOp<C_DIV>::f(av, A(bv[q]));
      }
      T out[V];
      if (ACC) ld_32B(cp + i * ldc, out);
#pragma unroll
      for (int q = 0; q < V; q++)
        out[q] = convert<T, A>(ReduceOp<R>::f(A(ACC ? out[q] : ident), quo[q]));
      st_stream_32B(cp + i * ldc, out);
    }
  } else {
#pragma unroll 4
  for (int64_t i = r0; i < r1; i++) {
    const T av = __ldg(a + i * lda);
    T out[V];
    if (ACC) {
      ld_32B(cp + i * ldc, out);
#pragma unroll
      for (int q = 0; q < V; q++) out[q] = outer_elem<T, C, R>(av, bv[q], out[q]);
    } else {
#pragma unroll
      for (int q = 0; q < V; q++) out[q] = outer_elem<T, C, R>(av, bv[q], ident);
    }
    st_stream_32B(cp + i * ldc, out);
  }
  }
}

// any N / ldc / alignment: one column per thread, rows strided over gridDim.y
template <typename T, int C, int R, bool ACC>
__global__ void __launch_bounds__(256) outer_scalar_kernel(T* __restrict__ c, const T* __restrict__ a,
                                                           const T* __restrict__ b, int64_t M,
                                                           int64_t N, int64_t lda, int64_t ldc) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= N) return;
  const T bv = __ldg(b + j);
  const T ident = ReduceOp<R>::template identity<T>();
#pragma unroll 4
  for (int64_t i = blockIdx.y; i < M; i += gridDim.y) {
    T* cp = c + i * ldc + j;
    *cp = outer_elem<T, C, R>(__ldg(a + i * lda), bv, ACC ? *cp : ident);
  }
}

// narrow rows (N < 64): flat grid-stride over all M*N elements
template <typename T, int C, int R, bool ACC>
__global__ void __launch_bounds__(256) outer_flat_kernel(T* __restrict__ c, const T* __restrict__ a,
                                                         const T* __restrict__ b, int64_t M,
                                                         int64_t N, int64_t lda, int64_t ldc) {
  const T ident = ReduceOp<R>::template identity<T>();
  const int64_t total = M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / N, j = idx - i * N;
    T* cp = c + i * ldc + j;
    *cp = outer_elem<T, C, R>(__ldg(a + i * lda), __ldg(b + j), ACC ? *cp : ident);
  }
}

template <typename T, int R>
__global__ void __launch_bounds__(256) fill_kernel(T* __restrict__ c, int64_t M, int64_t N,
                                                   int64_t ldc) {
  const T ident = ReduceOp<R>::template identity<T>();
  for (int64_t i = blockIdx.y; i < M; i += gridDim.y)
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N;
         j += (int64_t)gridDim.x * blockDim.x)
      c[i * ldc + j] = ident;
}

inline unsigned clamp_grid_y(int64_t want, int64_t M) {
  int64_t g = want < M ? want : M;
  if (g > 65535) g = 65535;
  if (g < 1) g = 1;
  return (unsigned)g;
}

template <typename T, int C, int R, bool ACC>
cudaError_t outer_typed(const Problem& p) {
  T* c = static_cast<T*>(p.c);
  const T* a = static_cast<const T*>(p.a);
  const T* b = static_cast<const T*>(p.b);
  constexpr int V = 32 / sizeof(T);
  const bool vec = (p.N % V == 0) && (p.ldc % V == 0) &&
                   (reinterpret_cast<uintptr_t>(c) % 32 == 0) && p.N >= 64;
  const int64_t target_blocks = (int64_t)kNumSMs * 8;  // 8 x 256 threads per SM
  if (vec) {
    // each block streams a short run of consecutive rows (16 by default): the
    // write front then advances through memory in dense runs (tools/tune_outer.cu:
    // 6.89 TB/s vs 6.0 for rows strided over the grid)
    const int64_t NV = p.N / V;
    const unsigned bx = NV >= 256 ? 256u : (unsigned)(((NV + 31) / 32) * 32);
    const int64_t gx = (NV + bx - 1) / bx;
    int64_t rpb = 16;
    if ((p.M + rpb - 1) / rpb > 65535) rpb = (p.M + 65534) / 65535;
    const int64_t gy = (p.M + rpb - 1) / rpb;
    dim3 grid((unsigned)gx, (unsigned)(gy < 1 ? 1 : gy));
    outer_vec_kernel<T, C, R, ACC><<<grid, bx, 0, p.stream>>>(c, a, b, p.M, NV, p.lda, p.ldc, rpb);
  } else if (p.N >= 64) {
    const unsigned bx = p.N >= 256 ? 256u : (unsigned)(((p.N + 31) / 32) * 32);
    const int64_t gx = (p.N + bx - 1) / bx;
    dim3 grid((unsigned)gx, clamp_grid_y((target_blocks + gx - 1) / gx, p.M));
    outer_scalar_kernel<T, C, R, ACC><<<grid, bx, 0, p.stream>>>(c, a, b, p.M, p.N, p.lda, p.ldc);
  } else {
    const int64_t total = p.M * p.N;
    int64_t blocks = (total + 255) / 256;
    if (blocks > target_blocks) blocks = target_blocks;
    if (blocks < 1) blocks = 1;
    outer_flat_kernel<T, C, R, ACC><<<(unsigned)blocks, 256, 0, p.stream>>>(c, a, b, p.M, p.N, p.lda,
                                                                          p.ldc);
  }
  count_launch();
  return cudaGetLastError();
}

template <typename T, int C, int R>
cudaError_t outer_acc(const Problem& p) {
  return p.accumulate ? outer_typed<T, C, R, true>(p) : outer_typed<T, C, R, false>(p);
}

template <typename T, int C>
cudaError_t outer_red(const Problem& p) {
  switch (p.reduce) {
    case R_ADD: return outer_acc<T, C, R_ADD>(p);
    case R_MUL: return outer_acc<T, C, R_MUL>(p);
    case R_MIN: return outer_acc<T, C, R_MIN>(p);
    default: return outer_acc<T, C, R_MAX>(p);
  }
}

template <typename T>
cudaError_t outer_comb(const Problem& p) {
  switch (p.combine) {
    case C_ADD: return outer_red<T, C_ADD>(p);
    case C_SUB: return outer_red<T, C_SUB>(p);
    case C_MUL: return outer_red<T, C_MUL>(p);
    case C_DIV: return outer_red<T, C_DIV>(p);
    case C_MIN: return outer_red<T, C_MIN>(p);
    default: return outer_red<T, C_MAX>(p);
  }
}

template <typename T>
cudaError_t fill_typed(const Problem& p) {
  T* c = static_cast<T*>(p.c);
  const unsigned bx = p.N >= 256 ? 256u : (unsigned)(((p.N + 31) / 32) * 32);
  int64_t gx = (p.N + bx - 1) / bx;
  if (gx > 65535) gx = 65535;
  dim3 grid((unsigned)gx, clamp_grid_y(((int64_t)kNumSMs * 8 + gx - 1) / gx, p.M));
  switch (p.reduce) {
    case R_ADD: fill_kernel<T, R_ADD><<<grid, bx, 0, p.stream>>>(c, p.M, p.N, p.ldc); break;
    case R_MUL: fill_kernel<T, R_MUL><<<grid, bx, 0, p.stream>>>(c, p.M, p.N, p.ldc); break;
    case R_MIN: fill_kernel<T, R_MIN><<<grid, bx, 0, p.stream>>>(c, p.M, p.N, p.ldc); break;
    default: fill_kernel<T, R_MAX><<<grid, bx, 0, p.stream>>>(c, p.M, p.N, p.ldc); break;
  }
  count_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_outer(const Problem& p) {
  switch (p.dtype) {
    case MOA_DTYPE_F64: return outer_comb<double>(p);
    case MOA_DTYPE_F32: return outer_comb<float>(p);
    case MOA_DTYPE_I32: return outer_comb<int32_t>(p);
    default: return outer_comb<int64_t>(p);
  }
}

cudaError_t launch_fill(const Problem& p) {
  switch (p.dtype) {
    case MOA_DTYPE_F64: return fill_typed<double>(p);
    case MOA_DTYPE_F32: return fill_typed<float>(p);
    case MOA_DTYPE_I32: return fill_typed<int32_t>(p);
    default: return fill_typed<int64_t>(p);
  }
}

}  // namespace moa
