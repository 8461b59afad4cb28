// Shared device definitions: the operation codes of the reference
// (ops.py:52-66, _ckernel.pyx:11-34) as compile-time functors, the
// accumulation type rule for float32 storage, and launch helpers.
#pragma once

#include <cstdint>
#include <type_traits>

#include <cuda_runtime.h>

namespace moa {

enum Combine : int { C_ADD = 0, C_SUB = 1, C_MUL = 2, C_DIV = 3, C_MIN = 4, C_MAX = 5 };
enum Reduce : int { R_ADD = 0, R_MUL = 1, R_MIN = 2, R_MAX = 3 };

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------------------
// Integer element types (the reference is float64 only): exact
// two's-complement arithmetic.  add/sub/mul wrap modulo 2^bits (computed on
// the unsigned type, so there is no undefined behaviour); divide truncates
// toward zero with x/0 = 0 and MIN/-1 = MIN.  On integer-valued data whose
// partial results stay below 2^53 in magnitude this equals the reference's
// float64 result exactly, which is what the parity tests pin (divide excepted).
// ---------------------------------------------------------------------------
template <typename T> struct IntTraits;
template <> struct IntTraits<int32_t> {
  using U = uint32_t;
  static constexpr int32_t kMax = 2147483647, kMin = -2147483647 - 1;
};
template <> struct IntTraits<int64_t> {
  using U = uint64_t;
  static constexpr int64_t kMax = 9223372036854775807LL, kMin = -9223372036854775807LL - 1;
};
template <typename T> __host__ __device__ constexpr bool is_int() {
  return std::is_same<T, int32_t>::value || std::is_same<T, int64_t>::value;
}
template <typename T> __device__ __forceinline__ T wrap_add(T x, T y) {
  using U = typename IntTraits<T>::U;
  return T(U(x) + U(y));
}
template <typename T> __device__ __forceinline__ T wrap_sub(T x, T y) {
  using U = typename IntTraits<T>::U;
  return T(U(x) - U(y));
}
template <typename T> __device__ __forceinline__ T wrap_mul(T x, T y) {
  using U = typename IntTraits<T>::U;
  return T(U(x) * U(y));
}
template <typename T> __device__ __forceinline__ T safe_div(T x, T y) {
  if (y == 0) return T(0);
  if (y == T(-1)) return wrap_sub(T(0), x);  // MIN / -1 wraps to MIN
  return x / y;
}

// ---------------------------------------------------------------------------
// combine(x, y) with the reference's operand order (_ckernel.pyx:71: combine
// gets the A element first).  Every arithmetic op is an explicit _rn intrinsic
// so nvcc can never contract a combine with a following reduce into an FMA
// (the reference is built with -ffp-contract=off, setup.py:14).
// min/max are the reference's compare-and-select (ops.py:42-47), NOT fmin/fmax:
// x if x < y else y keeps the second operand on NaN and on a +-0 tie.
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Division by a reused divisor.  In the inner product every B element divides
// a whole column of A elements, so the kernels take y = RN(1/b) once per B
// element and form each quotient as
//     q0 = RN(a*y), r0 = a - b*q0 (FMA), q1 = RN(q0 + r0*y), r1 = a - b*q1 (FMA, exact)
// and ACCEPT q1 only when the exact residual proves it is the correctly
// rounded quotient: |a - b*q1| < |b| * ulp(q1)/2, q1 not a power of two (whose
// lower rounding interval is half as wide).  No midpoint can be a quotient of
// two floating-point numbers, so the test is exact; operands whose exponents
// could under/overflow any step (|a|, |b| outside [2^-400, 2^400)), zeros,
// infinities and NaNs take the IEEE division.  (float32 keeps __fdiv_rn: its
// IEEE division is already cheap.)
// Either way the result is RN(a/b), bit for bit (tests/test_gpu_parity.py).
// Kernels prove a whole row of quotients at once and redo the row with the
// IEEE division when any proof fails, so the common case has no branches.
__device__ __forceinline__ double rcp_rn(double b) { return __drcp_rn(b); }

// operand exponent within the reciprocal path's range
__device__ __forceinline__ bool rcp_range(double x) {
  return ((unsigned)(__double_as_longlong(x) >> 52) & 0x7ffu) - 623u < 800u;  // [2^-400, 2^400)
}
// candidate quotient for in-range a, b with y = RN(1/b); ok &= proof that it
// is RN(a/b).  Out-of-range operands give garbage and must not be used.
__device__ __forceinline__ double div_candidate(double a, double b, double y, bool& ok) {
  const double q0 = __dmul_rn(a, y);
  const double r0 = __fma_rn(-b, q0, a);
  const double q1 = __fma_rn(r0, y, q0);
  const double r1 = __fma_rn(-b, q1, a);
  const unsigned long long uq = __double_as_longlong(q1);
  const unsigned eq = (unsigned)(uq >> 52) & 0x7ffu;  // >= 223 in range
  const double half_ulp_b = fabs(b) * __longlong_as_double((unsigned long long)(eq - 53u) << 52);
  ok = ok && (uq & 0xfffffffffffffull) != 0 && fabs(r1) < half_ulp_b;
  return q1;
}

// int32 division by a reused divisor with a per-divisor multiplier
// (Granlund & Montgomery 1994, round-up variant, on magnitudes): for d = |y|,
// l = ceil(log2 d), m = floor(2^32 (2^l - d) / d) + 1, and every 32-bit n,
// floor(n / d) = (t + ((n - t) >> min(l, 1))) >> max(l - 1, 0) with
// t = mulhi(m, n).  The sign is applied after (truncating division), |MIN|
// = 2^31 is a valid n, MIN / -1 wraps to MIN like safe_div, and y = 0 gives 0.
struct DivMagic32 {
  uint32_t m;
  uint32_t sh;  // sh1 | sh2 << 8 | (y == 0) << 16
};
__device__ __forceinline__ DivMagic32 div_magic(int32_t y) {
  const uint32_t d = y < 0 ? 0u - uint32_t(y) : uint32_t(y);
  if (d == 0) return DivMagic32{0u, 1u << 16};
  const uint32_t l = d == 1 ? 0u : 32u - __clz(d - 1u);
  const uint32_t m = uint32_t(((((uint64_t)1 << l) - d) << 32) / d) + 1u;
  const uint32_t sh1 = l < 1u ? l : 1u, sh2 = l > 0u ? l - 1u : 0u;
  return DivMagic32{m, sh1 | (sh2 << 8)};
}
__device__ __forceinline__ int32_t idiv_magic(int32_t x, uint32_t nx, int32_t y, DivMagic32 g) {
  const uint32_t t = __umulhi(g.m, nx);
  const uint32_t q = (t + ((nx - t) >> (g.sh & 0xffu))) >> ((g.sh >> 8) & 0xffu);
  const uint32_t neg = uint32_t((x ^ y) >> 31);  // all ones when the signs differ
  const int32_t r = int32_t((q ^ neg) - neg);
  return (g.sh >> 16) ? 0 : r;
}

// The same for int64 (64-bit multiplier, 128-bit set-up division per divisor).
struct DivMagic64 {
  uint64_t m;
  uint32_t sh;  // sh1 | sh2 << 8 | (y == 0) << 16
};
__device__ __forceinline__ DivMagic64 div_magic(int64_t y) {
  const uint64_t d = y < 0 ? 0ull - uint64_t(y) : uint64_t(y);
  if (d == 0) return DivMagic64{0ull, 1u << 16};
  const uint32_t l = d == 1 ? 0u : 64u - (uint32_t)__clzll((long long)(d - 1ull));
  const unsigned __int128 num = ((((unsigned __int128)1) << l) - d) << 64;
  const uint64_t m = uint64_t(num / d) + 1ull;
  const uint32_t sh1 = l < 1u ? l : 1u, sh2 = l > 0u ? l - 1u : 0u;
  return DivMagic64{m, sh1 | (sh2 << 8)};
}
__device__ __forceinline__ int64_t idiv_magic(int64_t x, uint64_t nx, int64_t y, DivMagic64 g) {
  const uint64_t t = __umul64hi(g.m, nx);
  const uint64_t q = (t + ((nx - t) >> (g.sh & 0xffu))) >> ((g.sh >> 8) & 0xffu);
  const uint64_t neg = uint64_t((x ^ y) >> 63);
  const int64_t r = int64_t((q ^ neg) - neg);
  return (g.sh >> 16) ? 0 : r;
}

template <int C> struct CombineOp;
template <> struct CombineOp<C_ADD> {
  static __device__ __forceinline__ double f(double x, double y) { return __dadd_rn(x, y); }
  static __device__ __forceinline__ float f(float x, float y) { return __fadd_rn(x, y); }
  static __device__ __forceinline__ int32_t f(int32_t x, int32_t y) { return wrap_add(x, y); }
  static __device__ __forceinline__ int64_t f(int64_t x, int64_t y) { return wrap_add(x, y); }
};
template <> struct CombineOp<C_SUB> {
  static __device__ __forceinline__ double f(double x, double y) { return __dsub_rn(x, y); }
  static __device__ __forceinline__ float f(float x, float y) { return __fsub_rn(x, y); }
  static __device__ __forceinline__ int32_t f(int32_t x, int32_t y) { return wrap_sub(x, y); }
  static __device__ __forceinline__ int64_t f(int64_t x, int64_t y) { return wrap_sub(x, y); }
};
template <> struct CombineOp<C_MUL> {
  static __device__ __forceinline__ double f(double x, double y) { return __dmul_rn(x, y); }
  static __device__ __forceinline__ float f(float x, float y) { return __fmul_rn(x, y); }
  static __device__ __forceinline__ int32_t f(int32_t x, int32_t y) { return wrap_mul(x, y); }
  static __device__ __forceinline__ int64_t f(int64_t x, int64_t y) { return wrap_mul(x, y); }
};
template <> struct CombineOp<C_DIV> {
  static __device__ __forceinline__ double f(double x, double y) { return __ddiv_rn(x, y); }
  static __device__ __forceinline__ float f(float x, float y) { return __fdiv_rn(x, y); }
  static __device__ __forceinline__ int32_t f(int32_t x, int32_t y) { return safe_div(x, y); }
  static __device__ __forceinline__ int64_t f(int64_t x, int64_t y) { return safe_div(x, y); }
};
template <> struct CombineOp<C_MIN> {
  template <typename T> static __device__ __forceinline__ T f(T x, T y) { return x < y ? x : y; }
};
template <> struct CombineOp<C_MAX> {
  template <typename T> static __device__ __forceinline__ T f(T x, T y) { return x > y ? x : y; }
};

// reduce(acc, v): _ckernel.pyx:26-34 / ops.py:61-66; acc is the left operand.
// Integer identities: 0, 1, and the type's max / min for the +inf / -inf of min / max.
template <int R> struct ReduceOp;
template <> struct ReduceOp<R_ADD> {
  static __device__ __forceinline__ double f(double x, double y) { return __dadd_rn(x, y); }
  static __device__ __forceinline__ float f(float x, float y) { return __fadd_rn(x, y); }
  static __device__ __forceinline__ int32_t f(int32_t x, int32_t y) { return wrap_add(x, y); }
  static __device__ __forceinline__ int64_t f(int64_t x, int64_t y) { return wrap_add(x, y); }
  template <typename T> static __host__ __device__ constexpr T identity() { return T(0); }
};
template <> struct ReduceOp<R_MUL> {
  static __device__ __forceinline__ double f(double x, double y) { return __dmul_rn(x, y); }
  static __device__ __forceinline__ float f(float x, float y) { return __fmul_rn(x, y); }
  static __device__ __forceinline__ int32_t f(int32_t x, int32_t y) { return wrap_mul(x, y); }
  static __device__ __forceinline__ int64_t f(int64_t x, int64_t y) { return wrap_mul(x, y); }
  template <typename T> static __host__ __device__ constexpr T identity() { return T(1); }
};
template <> struct ReduceOp<R_MIN> {
  template <typename T> static __device__ __forceinline__ T f(T x, T y) { return x < y ? x : y; }
  template <typename T> static __host__ __device__ T identity() {
    if constexpr (is_int<T>()) return IntTraits<T>::kMax;
    else return T(__builtin_huge_val());
  }
};
template <> struct ReduceOp<R_MAX> {
  template <typename T> static __device__ __forceinline__ T f(T x, T y) { return x > y ? x : y; }
  template <typename T> static __host__ __device__ T identity() {
    if constexpr (is_int<T>()) return IntTraits<T>::kMin;
    else return T(-__builtin_huge_val());
  }
};

// ---------------------------------------------------------------------------
// Arithmetic type for a storage type.  The reference upcasts every operand to
// float64 (arrays.py:77-78), so a float32 product must equal the float64
// result rounded once to float32.  For a min/max reduce float32 arithmetic
// already gives that (add/sub/mul/div of two floats rounded to float32 equals
// the float64 op rounded to float32 — 53 >= 2*24+2 makes double rounding
// innocuous — and a compare-select fold commutes with a monotone rounding), so
// it stays in float32.  Sums and products of many terms do not commute with
// rounding, so add/multiply reduces on float32 storage run in float64.
// ---------------------------------------------------------------------------
// Accumulation/computation type.  float32 data reproduces the reference's
// float64 arithmetic rounded once: sums and products of the fold need float64;
// a min/max fold can stay in float32 (rounding is monotone) only when no
// combine result that is nonzero in float64 can round to a signed zero in
// float32 — true for add/subtract/min/max, not for multiply/divide, whose
// underflow would turn max(-tiny, +0) = +0 into a -0/+0 tie.
template <typename T, int C, int R> struct AccType { using type = T; };
template <int C> struct AccType<float, C, R_ADD> { using type = double; };
template <int C> struct AccType<float, C, R_MUL> { using type = double; };
template <> struct AccType<float, C_MUL, R_MIN> { using type = double; };
template <> struct AccType<float, C_MUL, R_MAX> { using type = double; };
template <> struct AccType<float, C_DIV, R_MIN> { using type = double; };
template <> struct AccType<float, C_DIV, R_MAX> { using type = double; };

template <typename To, typename From> __device__ __forceinline__ To convert(From x) { return To(x); }
template <> __device__ __forceinline__ float convert<float, double>(double x) { return __double2float_rn(x); }

// ---------------------------------------------------------------------------
// operand special-value flags from the device pre-scan (semiring fast path)
// ---------------------------------------------------------------------------
enum SpecialBits : unsigned {
  S_NAN = 1u, S_PINF = 2u, S_NINF = 4u, S_NZERO = 8u, S_PZERO = 16u,
  S_NEG = 32u  // sign bit set (any negative value, -0.0 or -inf)
};

// Whether a fold with the hardware 3-input min/max (FMNMX3, which prefers the
// non-NaN operand and may order +-0 arbitrarily) is bit-identical to the
// reference's compare-select fold, given the special values that occur in A
// and in B.  True iff no combine result can be NaN or -0.0: then the fold is
// an exact min/max over ordered values and any association order gives the
// same bits.
__host__ __device__ inline bool fast_fold_is_exact(int combine, unsigned fa, unsigned fb) {
  if ((fa | fb) & S_NAN) return false;
  if (combine == C_ADD) {
    // a+b is NaN only for inf + -inf; -0 only for -0 + -0 (round-to-nearest).
    if (((fa & S_PINF) && (fb & S_NINF)) || ((fa & S_NINF) && (fb & S_PINF))) return false;
    if ((fa & S_NZERO) && (fb & S_NZERO)) return false;
    return true;
  }
  if (combine == C_SUB) {
    // a-b is NaN only for inf - inf of equal sign; -0 only for -0 - +0.
    if (((fa & S_PINF) && (fb & S_PINF)) || ((fa & S_NINF) && (fb & S_NINF))) return false;
    if ((fa & S_NZERO) && (fb & S_PZERO)) return false;
    return true;
  }
  return false;
}

// Fold mode for the float32 tropical loops: 0 = exact compare-select,
// 1 = FMNMX3 on floats, 2 = VIMNMX3 on the bit patterns.  Mode 2 needs every
// combine result to be a non-negative, non-NaN float, for which unsigned
// integer order equals float order (and +-0 ties cannot occur): true for
// add of two sign-clear, NaN-free operands (and for multiply, below).
// VIMNMX3 issues faster beside FADD2 than FMNMX3 does
// (profiles/r01_minplus_mix2.json).
__host__ __device__ inline int tropical_fold_mode(int combine, unsigned fa, unsigned fb) {
  if (combine == C_MUL) {
    // max-times / min-times: only the unsigned-order fold, for sign-clear,
    // NaN-free operands without a 0 x inf pair (every product is then a
    // non-negative non-NaN float; underflow gives +0)
    constexpr unsigned Z = S_PZERO | S_NZERO, I = S_PINF | S_NINF;
    if ((fa | fb) & (S_NAN | S_NEG)) return 0;
    if (((fa & Z) && (fb & I)) || ((fa & I) && (fb & Z))) return 0;
    return 2;
  }
  if (!fast_fold_is_exact(combine, fa, fb)) return 0;
  if (combine == C_ADD && !((fa | fb) & (S_NAN | S_NEG))) return 2;
  return 1;
}

// With MOA_FLAG_ACCUMULATE the result's previous contents are folded too:
// they must hold no NaN or -0.0 for any fast mode (fc = C's scan flags).  The
// unsigned-order fold also needs sign-clear seeds, except for max: there every
// combine result is >= +0 and K >= 1, so a negative seed (the -inf identity
// the reference prefills, say) never wins and is replaced by +0 (init_acc).
// A min fold with negative seeds drops to FMNMX3 for add/subtract and to the
// exact loop for multiply, which has no FMNMX3 kernel.
__host__ __device__ inline int tropical_fold_mode_acc(int combine, int reduce, unsigned fa,
                                                      unsigned fb, unsigned fc) {
  const int m = tropical_fold_mode(combine, fa, fb);
  if (fc & (S_NAN | S_NZERO)) return 0;
  if (m == 2 && (fc & S_NEG) && reduce != R_MAX) return combine == C_MUL ? 0 : 1;
  return m;
}
template <bool ACC>
__device__ __forceinline__ int tropical_mode_of(int combine, int reduce, const unsigned* special) {
  return ACC ? tropical_fold_mode_acc(combine, reduce, __ldg(special), __ldg(special + 1),
                                      __ldg(special + 2))
             : tropical_fold_mode(combine, __ldg(special), __ldg(special + 1));
}

}  // namespace moa
