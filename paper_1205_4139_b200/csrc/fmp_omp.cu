// Fused OMP solver: launch dispatch (the kernel is fmp_omp_impl.cuh; each
// element type is instantiated in its own translation unit).
#include "fmp_kcommon.cuh"

namespace fmp {
cudaError_t launch_omp_c128(const OmpArgs& a, cudaStream_t st);
cudaError_t launch_omp_c64(const OmpArgs& a, cudaStream_t st);
cudaError_t launch_omp_f64(const OmpArgs& a, cudaStream_t st);
cudaError_t launch_omp_f32(const OmpArgs& a, cudaStream_t st);
int omp_ctas_c128(const DevOp& op, int64_t batch, int64_t T);
int omp_f16_c128(const DevOp& op, int64_t batch, int64_t T);
int omp_ctas_c64(const DevOp& op, int64_t batch, int64_t T);

void omp_info_c128(const DevOp& op, int64_t batch, int64_t T, int* out4);
void omp_info_c64(const DevOp& op, int64_t batch, int64_t T, int* out4);
void omp_info_f64(const DevOp& op, int64_t batch, int64_t T, int* out4);
void omp_info_f32(const DevOp& op, int64_t batch, int64_t T, int* out4);

void omp_info(const DevOp& op, int dtype, int64_t batch, int64_t T, int* out4) {
  switch (dtype) {
    case C128: omp_info_c128(op, batch, T, out4); break;
    case C64: omp_info_c64(op, batch, T, out4); break;
    case F64: omp_info_f64(op, batch, T, out4); break;
    default: omp_info_f32(op, batch, T, out4); break;
  }
}

int omp_ctas(const DevOp& op, int dtype, int64_t batch, int64_t T) {
  switch (dtype) {
    case C128: return omp_ctas_c128(op, batch, T);
    case C64: return omp_ctas_c64(op, batch, T);
  }
  return 1;
}

int omp_grid(const DevOp& op, int dtype, int64_t batch, int64_t T) {
  const int64_t slots = (int64_t)omp_ctas(op, dtype, batch, T) * num_sms();
  return (int)std::max<int64_t>(1, std::min<int64_t>(batch, slots));
}

int omp_gpu_fast_until(const DevOp& op, int dtype, int64_t batch, int64_t T) {
  // measured on B200 (bench.py --mode custom:T sweeps): a Fourier transform
  // iteration of the one-CTA solver costs about as much as 8 log2(N) / 3
  // fast-update atoms, of the two-CTA solver (kernel table read through L1)
  // 4 log2(N) / 3; the Hadamard FWHT needs no twiddles
  const int64_t logn = op.log2n;
  if (op.kind == HADAMARD) return (int)(2 * logn);
  // the two-CTA solver's F16 conventional rows (kernel table through L1):
  // 2 log2(N) / 3 (config 2: custom:8 measured fastest of 1..16, 307 k/s)
  if (dtype == C128 && omp_f16_c128(op, batch, T)) return (int)(2 * logn / 3);
  return (int)((omp_ctas(op, dtype, batch, T) == 2 ? 4 : 8) * logn / 3);
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
