// K2 semiring kernels instantiated for int64_t elements (see semiring_impl.cuh).
#include "semiring_impl.cuh"

namespace moa {
cudaError_t launch_semiring_i64(const Problem& p) { return semiring_comb<int64_t>(p); }
}  // namespace moa
