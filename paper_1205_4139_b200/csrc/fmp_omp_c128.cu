// Fused OMP solver instantiations for c128 data.
#include "fmp_omp_impl.cuh"

namespace fmp {
cudaError_t launch_omp_c128(const OmpArgs& a, cudaStream_t st) {
  return a.op->kind == HADAMARD ? launch_omp_v<double2, true>(a, st) : launch_omp_v<double2, false>(a, st);
}
// the two-CTA solver runs the F16 conventional rows (fmp_omp_impl.cuh)
int omp_f16_c128(const DevOp& op, int64_t batch, int64_t T) {
  return op.kind != HADAMARD && f16_ok<double2, false>(op) && !omp_f16_off() &&
         omp_ctas_v<double2, false>(op, batch, T) == 2;
}
int omp_ctas_c128(const DevOp& op, int64_t batch, int64_t T) {
  return op.kind == HADAMARD ? 1 : omp_ctas_v<double2, false>(op, batch, T);
}
void omp_info_c128(const DevOp& op, int64_t batch, int64_t T, int* out4) {
  if (op.kind == HADAMARD) omp_info_v<double2, true>(op, batch, T, out4);
  else omp_info_v<double2, false>(op, batch, T, out4);
}
}  // namespace fmp
