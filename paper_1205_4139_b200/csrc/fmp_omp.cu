// Fused OMP solver: launch dispatch (the kernel is fmp_omp_impl.cuh; each
// element type is instantiated in its own translation unit).
#include "fmp_kcommon.cuh"

namespace fmp {
cudaError_t launch_omp_c128(const OmpArgs& a, cudaStream_t st);
cudaError_t launch_omp_c64(const OmpArgs& a, cudaStream_t st);
cudaError_t launch_omp_f64(const OmpArgs& a, cudaStream_t st);
cudaError_t launch_omp_f32(const OmpArgs& a, cudaStream_t st);

int omp_grid(const DevOp&, int, int64_t batch, int64_t) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(batch, (int64_t)OMP_CTAS * num_sms()));
}

cudaError_t launch_omp(const OmpArgs& a, cudaStream_t st) {
  g_launches = 0;
  if (a.op->kind == HADAMARD && !a.op->glat) return cudaErrorInvalidValue;
  switch (a.dtype) {
    case C128: return launch_omp_c128(a, st);
    case C64: return launch_omp_c64(a, st);
    case F64: return a.op->kind == HADAMARD ? launch_omp_f64(a, st) : cudaErrorInvalidValue;
    case F32: return a.op->kind == HADAMARD ? launch_omp_f32(a, st) : cudaErrorInvalidValue;
  }
  return cudaErrorInvalidValue;
}
}  // namespace fmp
