// K2 dispatch: the semiring kernel templates live in semiring_impl.cuh and are
// instantiated per element type in semiring_<type>.cu (compiled in parallel).
#include "moa_common.cuh"
#include "moa_kernels.h"
#include "../../include/moa_b200.h"

namespace moa {

cudaError_t launch_semiring_f64(const Problem& p);
cudaError_t launch_semiring_f32(const Problem& p);
cudaError_t launch_semiring_i32(const Problem& p);
cudaError_t launch_semiring_i64(const Problem& p);

bool semiring_fast_candidate(int dtype, int combine, int reduce, bool accumulate) {
  (void)accumulate;  // accumulate folds C's contents too; the pre-scan covers them
  return dtype == MOA_DTYPE_F32 && (combine == C_ADD || combine == C_SUB || combine == C_MUL) &&
         (reduce == R_MIN || reduce == R_MAX);
}

cudaError_t launch_semiring(const Problem& p) {
  switch (p.dtype) {
    case MOA_DTYPE_F64: return launch_semiring_f64(p);
    case MOA_DTYPE_F32: return launch_semiring_f32(p);
    case MOA_DTYPE_I32: return launch_semiring_i32(p);
    default: return launch_semiring_i64(p);
  }
}

}  // namespace moa
