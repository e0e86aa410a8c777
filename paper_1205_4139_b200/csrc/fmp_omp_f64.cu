// Fused OMP solver instantiations for f64 data.
#include "fmp_omp_impl.cuh"

namespace fmp {
cudaError_t launch_omp_f64(const OmpArgs& a, cudaStream_t st) {
  return launch_omp_v<double, true>(a, st);
}
}  // namespace fmp
