// Fused OMP solver instantiations for f32 data.
#include "fmp_omp_impl.cuh"

namespace fmp {
cudaError_t launch_omp_f32(const OmpArgs& a, cudaStream_t st) {
  return launch_omp_v<float, true>(a, st);
}
}  // namespace fmp
