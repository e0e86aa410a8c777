// Fused OMP solver instantiations for f64 data.
#include "fmp_omp_impl.cuh"

namespace fmp {
cudaError_t launch_omp_f64(const OmpArgs& a, cudaStream_t st) {
  return launch_omp_v<double, true>(a, st);
}
void omp_info_f64(const DevOp& op, int64_t batch, int64_t T, int* out4) {
  omp_info_v<double, true>(op, batch, T, out4);
}
}  // namespace fmp
