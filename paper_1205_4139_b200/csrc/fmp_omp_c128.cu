// Fused OMP solver instantiations for c128 data.
#include "fmp_omp_impl.cuh"

namespace fmp {
cudaError_t launch_omp_c128(const OmpArgs& a, cudaStream_t st) {
  return a.op->kind == HADAMARD ? launch_omp_v<double2, true>(a, st) : launch_omp_v<double2, false>(a, st);
}
int omp_ctas_c128(const DevOp& op, int64_t batch, int64_t T) {
  return op.kind == HADAMARD ? 1 : omp_ctas_v<double2, false>(op, batch, T);
}
void omp_info_c128(const DevOp& op, int64_t batch, int64_t T, int* out4) {
  if (op.kind == HADAMARD) omp_info_v<double2, true>(op, batch, T, out4);
  else omp_info_v<double2, false>(op, batch, T, out4);
}
}  // namespace fmp
