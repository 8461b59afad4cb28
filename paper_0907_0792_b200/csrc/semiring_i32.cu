// K2 semiring kernels instantiated for int32_t elements (see semiring_impl.cuh).
#include "semiring_impl.cuh"

namespace moa {
cudaError_t launch_semiring_i32(const Problem& p) { return semiring_comb<int32_t>(p); }
}  // namespace moa
