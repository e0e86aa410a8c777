// Fused OMP solver instantiations for c64 data.
#include "fmp_omp_impl.cuh"

namespace fmp {
cudaError_t launch_omp_c64(const OmpArgs& a, cudaStream_t st) {
  return a.op->kind == HADAMARD ? launch_omp_v<float2, true>(a, st) : launch_omp_v<float2, false>(a, st);
}
}  // namespace fmp
