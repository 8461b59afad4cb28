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
// could under/overflow any step (|a|, |b| outside [2^-400, 2^400) for double,
// [2^-40, 2^40) for float), zeros, infinities and NaNs take the IEEE division.
// Either way the result is RN(a/b), bit for bit (tests/test_gpu_parity.py).
// Kernels prove a whole row of quotients at once and redo the row with the
// IEEE division when any proof fails, so the common case has no branches.
__device__ __forceinline__ double rcp_rn(double b) { return __drcp_rn(b); }
__device__ __forceinline__ float rcp_rn(float b) { return __frcp_rn(b); }

// operand exponent within the reciprocal path's range
__device__ __forceinline__ bool rcp_range(double x) {
  return ((unsigned)(__double_as_longlong(x) >> 52) & 0x7ffu) - 623u < 800u;  // [2^-400, 2^400)
}
__device__ __forceinline__ bool rcp_range(float x) {
  return ((__float_as_uint(x) >> 23) & 0xffu) - 87u < 80u;  // [2^-40, 2^40)
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
__device__ __forceinline__ float div_candidate(float a, float b, float y, bool& ok) {
  const float q0 = __fmul_rn(a, y);
  const float r0 = __fmaf_rn(-b, q0, a);
  const float q1 = __fmaf_rn(r0, y, q0);
  const float r1 = __fmaf_rn(-b, q1, a);
  const unsigned uq = __float_as_uint(q1);
  const unsigned eq = (uq >> 23) & 0xffu;  // >= 47 in range
  const float half_ulp_b = fabsf(b) * __uint_as_float((eq - 24u) << 23);
  ok = ok && (uq & 0x7fffffu) != 0 && fabsf(r1) < half_ulp_b;
  return q1;
}

// Integer division by a reused divisor through yr = RN(1/double(y)).
// q = trunc(x*yr) is exact or, when x/y is an integer, one unit short: for
// int32 the estimate's error (< |x/y| 2^-51) is below the distance 1/|y| from
// any non-integer x/y to the next integer.  int64 operands lose bits in the
// conversion, so the remainder gets one more estimate (|error| < 2^13 after
// the first).  The last unit is fixed from the exact remainder (truncating
// division: r = 0 or sign(r) = sign(x) with |r| < |y|), and y = 0, y = -1
// keep safe_div's results.
template <typename T>
__device__ __forceinline__ T idiv_by_rcp(T x, double xd, T y, double yr) {
  using U = typename IntTraits<T>::U;
  T q;
  if constexpr (sizeof(T) == 8) q = T(__double2ll_rz(xd * yr));
  else q = T(__double2int_rz(xd * yr));
  T r = wrap_sub(x, wrap_mul(q, y));
  if constexpr (sizeof(T) == 8) {
    q = wrap_add(q, T(__double2ll_rz(double(r) * yr)));
    r = wrap_sub(x, wrap_mul(q, y));
  }
  const T s = ((x ^ y) < 0) ? T(-1) : T(1);
  const U ar = r < 0 ? U(0) - U(r) : U(r), ay = y < 0 ? U(0) - U(y) : U(y);
  if (r != 0 && ((r < 0) != (x < 0))) q = wrap_sub(q, s);
  else if (ar >= ay) q = wrap_add(q, s);
  return y == 0 ? T(0) : (y == T(-1) ? wrap_sub(T(0), x) : q);
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
template <typename T, int R> struct AccType { using type = T; };
template <> struct AccType<float, R_ADD> { using type = double; };
template <> struct AccType<float, R_MUL> { using type = double; };

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
// add of two sign-clear, NaN-free operands.  VIMNMX3 issues faster beside
// FADD2 than FMNMX3 does (profiles/r01_minplus_mix2.json).
__host__ __device__ inline int tropical_fold_mode(int combine, unsigned fa, unsigned fb) {
  if (!fast_fold_is_exact(combine, fa, fb)) return 0;
  if (combine == C_ADD && !((fa | fb) & (S_NAN | S_NEG))) return 2;
  return 1;
}

// With MOA_FLAG_ACCUMULATE the result's previous contents are folded too:
// they must hold no NaN or -0.0 for any fast mode (fc = C's scan flags) and
// be sign-clear for the unsigned-order fold.
__host__ __device__ inline int tropical_fold_mode_acc(int combine, unsigned fa, unsigned fb,
                                                      unsigned fc) {
  const int m = tropical_fold_mode(combine, fa, fb);
  if (fc & (S_NAN | S_NZERO)) return 0;
  return (m == 2 && (fc & S_NEG)) ? 1 : m;
}
template <bool ACC>
__device__ __forceinline__ int tropical_mode_of(int combine, const unsigned* special) {
  return ACC ? tropical_fold_mode_acc(combine, __ldg(special), __ldg(special + 1), __ldg(special + 2))
             : tropical_fold_mode(combine, __ldg(special), __ldg(special + 1));
}

}  // namespace moa
