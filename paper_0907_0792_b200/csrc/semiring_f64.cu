// K2 semiring kernels instantiated for double elements (see semiring_impl.cuh).
#include "semiring_impl.cuh"

namespace moa {
cudaError_t launch_semiring_f64(const Problem& p) { return semiring_comb<double>(p); }
}  // namespace moa
