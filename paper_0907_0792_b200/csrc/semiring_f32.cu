// K2 semiring kernels instantiated for float elements (see semiring_impl.cuh).
#include "semiring_impl.cuh"

namespace moa {
cudaError_t launch_semiring_f32(const Problem& p) { return semiring_comb<float>(p); }
}  // namespace moa
