// The C ABI (include/moa_b200.h): the B200 replacement for the reference's
// backend hot-loop entry _ckernel.product_rows (_ckernel.pyx:75-88).
//
// The reference dispatches on the op codes ((2,0) -> _rows_mul_add, else
// _rows_generic, _ckernel.pyx:82-88) and walks rows start, start+step, ...
// Here the row set becomes a plain 2-D problem: rows start + t*step are A rows
// at stride lstride*step and C rows at stride restride*step, so one launch
// covers any (start, step) with no gather.  Kernel choice:
//   rowsinred == 0      -> identity fill (the empty fold; nothing in ACCUMULATE)
//   rowsinred == 1      -> K3 write-streaming outer kernel (outer.cu)
//   (multiply, add) f64 -> K1 DMMA tensor-core kernel (dmma.cu), unless EXACT or
//                          rowsinred < kDmmaMinK
//   otherwise           -> K2 semiring kernel (semiring.cu)
//
// Below one DMMA k-step group (rowsinred < 8) a (multiply, add) product is
// bound by writing C, not by arithmetic: the exact fold's two FP64
// instructions per pair (DMUL, DADD: <= 14 per element) issue faster than HBM
// absorbs the 8-byte result, so it runs at the DMMA route's speed and returns
// the reference's bits (_ckernel.pyx:37-52), as the reference's own
// element-wise tolerance for small random cases expects (tests/
// test_acceptance.py:34-53, rtol 1e-12).  The rule depends on rowsinred only,
// so row sharding never changes the route, and k-chunked accumulation keeps
// every chunk at >= 16 (distributed.k_chunks, host_exec k_chunks).
#include <cstdio>
#include <string>

#include "moa_common.cuh"
#include "moa_kernels.h"
#include "../../include/moa_b200.h"

namespace {
thread_local std::string t_last_error;
}

namespace moa {
std::atomic<uint64_t> g_launches{0};
void set_last_error(const std::string& msg) { t_last_error = msg; }
}

namespace {

int fail(int code, const std::string& msg) {
  t_last_error = msg;
  return code;
}

enum class Route { None, Fill, Outer, Dmma, SemiringExact, SemiringFast, SemiringDpx };

constexpr int64_t kDmmaMinK = 8;

Route route(int dtype, int64_t rows, int64_t K, int64_t N, int comb, int red, uint32_t flags) {
  if (rows <= 0 || N <= 0) return Route::None;
  const bool acc = (flags & MOA_FLAG_ACCUMULATE) != 0;
  if (K == 0) return acc ? Route::None : Route::Fill;
  if (K == 1) return Route::Outer;
  if (dtype == MOA_DTYPE_F64 && comb == moa::C_MUL && red == moa::R_ADD && !(flags & MOA_FLAG_EXACT) &&
      K >= kDmmaMinK)
    return Route::Dmma;
  if (moa::semiring_fast_candidate(dtype, comb, red, acc)) return Route::SemiringFast;
  if (dtype == MOA_DTYPE_I32 && (comb == moa::C_ADD || comb == moa::C_SUB) &&
      (red == moa::R_MIN || red == moa::R_MAX))
    return Route::SemiringDpx;
  return Route::SemiringExact;
}

const char* route_name(Route r) {
  switch (r) {
    case Route::Fill: return "fill";
    case Route::Outer: return "outer";
    case Route::Dmma: return "dmma";
    case Route::SemiringExact: return "semiring_exact";
    case Route::SemiringFast: return "semiring_fast";
    case Route::SemiringDpx: return "semiring_dpx";
    default: return "none";
  }
}

}  // namespace

extern "C" {

int moa_abi_version(void) { return 101; }

int moa_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return n;
}

const char* moa_last_error(void) { return t_last_error.c_str(); }

uint64_t moa_launch_count(void) { return moa::g_launches.load(std::memory_order_relaxed); }

const char* moa_plan_kernel(int dtype, int64_t noproc, int64_t rowsinred, int64_t elsinop,
                            int combine_code, int reduce_code, uint32_t flags) {
  return route_name(route(dtype, noproc, rowsinred, elsinop, combine_code, reduce_code, flags));
}

int moa_product_rows(int dtype, void* res, const void* a, const void* b, int64_t noproc,
                     int64_t rowsinred, int64_t elsinop, int64_t lstride, int64_t rstride,
                     int64_t restride, int combine_code, int reduce_code, int64_t start,
                     int64_t step, uint32_t flags, void* stream) {
  t_last_error.clear();
  if (dtype < MOA_DTYPE_F64 || dtype > MOA_DTYPE_I64)
    return fail(MOA_E_DTYPE, "unknown dtype code " + std::to_string(dtype));
  if (combine_code < 0 || combine_code > 5)
    return fail(MOA_E_OPCODE, "unknown combine code " + std::to_string(combine_code));
  if (reduce_code < 0 || reduce_code > 3)
    return fail(MOA_E_OPCODE, "unknown reduce code " + std::to_string(reduce_code));
  if (noproc < 0 || rowsinred < 0 || elsinop < 0 || lstride < 0 || rstride < 0 || restride < 0)
    return fail(MOA_E_BOUNDS, "negative loop bound or stride");
  if (step < 1) return fail(MOA_E_BOUNDS, "step must be >= 1, got " + std::to_string(step));
  if (start < 0) return fail(MOA_E_BOUNDS, "start must be >= 0, got " + std::to_string(start));
  if (start >= noproc || elsinop == 0) return 0;  // surplus worker / empty rows: no work

  const int64_t rows = (noproc - start + step - 1) / step;
  const Route r = route(dtype, rows, rowsinred, elsinop, combine_code, reduce_code, flags);
  if (r == Route::None) return 0;
  if (res == nullptr || (rowsinred > 0 && (a == nullptr || b == nullptr)))
    return fail(MOA_E_NULL, "null operand pointer");

  const size_t esz = (dtype == MOA_DTYPE_F64 || dtype == MOA_DTYPE_I64) ? 8 : 4;
  moa::Problem p;
  p.dtype = dtype;
  p.c = static_cast<char*>(res) + (size_t)(start * restride) * esz;
  p.a = a ? static_cast<const char*>(a) + (size_t)(start * lstride) * esz : nullptr;
  p.b = b;
  p.M = rows;
  p.K = rowsinred;
  p.N = elsinop;
  p.lda = lstride * step;
  p.ldb = rstride;
  p.ldc = restride * step;
  p.combine = combine_code;
  p.reduce = reduce_code;
  p.accumulate = (flags & MOA_FLAG_ACCUMULATE) != 0;
  p.stream = static_cast<cudaStream_t>(stream);

  // the launchers check cudaGetLastError(); drop a stale, non-sticky error an
  // earlier call of this library left in this thread's runtime state
  (void)cudaGetLastError();
  cudaError_t e = cudaSuccess;
  switch (r) {
    case Route::Fill: e = moa::launch_fill(p); break;
    case Route::Outer: e = moa::launch_outer(p); break;
    case Route::Dmma: e = moa::launch_dmma(p); break;
    default: e = moa::launch_semiring(p); break;
  }
  if (e != cudaSuccess)
    return fail((int)e, std::string(route_name(r)) + " launch failed: " + cudaGetErrorString(e));
  return 0;
}

}  // extern "C"
