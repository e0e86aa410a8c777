// IncrementalQR (solvers.hpp:90-109, solvers.cpp:222-274) on the device:
// a thin QR of a growing column set, Q (rows x t, column-major, fp64
// complex) resident in HBM.  push_column runs two Gram-Schmidt passes -- all
// t projections of a pass at once (classical Gram-Schmidt with
// reorthogonalisation), rather than the reference's column-by-column
// modified Gram-Schmidt -- then rejects the column when the remainder is at
// most 1e-10 of its norm, as the reference does.
#include "fmp_kcommon.cuh"

namespace fmp {
namespace {

constexpr int QR_THREADS = 256;

// out[i * nb + b] = partial of q_i^H v over block b's row range
__global__ void __launch_bounds__(QR_THREADS) k_qr_dots(const double2* __restrict__ Q, int64_t rows,
                                                        const double2* __restrict__ v,
                                                        double2* __restrict__ part) {
  __shared__ double red[32];
  const int i = blockIdx.y, nb = gridDim.x;
  const int64_t chunk = (rows + nb - 1) / nb;
  const int64_t r0 = (int64_t)blockIdx.x * chunk, r1 = min(rows, r0 + chunk);
  const double2* q = Q + (size_t)i * rows;
  double sr = 0.0, si = 0.0;
  for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
    const double2 a = q[r], b = v[r];
    sr = fma(a.x, b.x, fma(a.y, b.y, sr));  // conj(a) b
    si = fma(a.x, b.y, fma(-a.y, b.x, si));
  }
  sr = block_sum(sr, red);
  si = block_sum(si, red);
  if (threadIdx.x == 0) part[(size_t)i * nb + blockIdx.x] = make_double2(sr, si);
}

// s_i = sum of the nb partials (fixed order); acc_i += s_i
__global__ void k_qr_reduce(const double2* __restrict__ part, int nb, int t, double2* __restrict__ s,
                            double2* __restrict__ acc) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= t) return;
  double2 z = make_double2(0.0, 0.0);
  for (int b = 0; b < nb; ++b) {
    const double2 p = part[(size_t)i * nb + b];
    z.x += p.x;
    z.y += p.y;
  }
  s[i] = z;
  acc[i].x += z.x;
  acc[i].y += z.y;
}

// v[r] -= sum_i q_i[r] s_i
__global__ void __launch_bounds__(QR_THREADS) k_qr_update(const double2* __restrict__ Q, int64_t rows,
                                                          int t, const double2* __restrict__ s,
                                                          double2* __restrict__ v) {
  extern __shared__ double2 ss[];
  for (int i = threadIdx.x; i < t; i += blockDim.x) ss[i] = s[i];
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    double2 a = v[r];
    for (int i = 0; i < t; ++i) {
      const double2 q = Q[(size_t)i * rows + r], c = ss[i];
      a.x -= q.x * c.x - q.y * c.y;
      a.y -= q.x * c.y + q.y * c.x;
    }
    v[r] = a;
  }
}

// per-block partial ||v||^2
__global__ void __launch_bounds__(QR_THREADS) k_qr_norm(const double2* __restrict__ v, int64_t rows,
                                                        double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    s += mag2(v[r]);
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void k_qr_sum(const double* __restrict__ part, int cnt, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) s += part[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

__global__ void k_qr_store(double2* __restrict__ qnew, const double2* __restrict__ v, int64_t rows,
                           double inv) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (int64_t)gridDim.x * blockDim.x)
    qnew[r] = make_double2(v[r].x * inv, v[r].y * inv);
}

}  // namespace

int qr_dot_blocks(int64_t rows) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(num_sms() * 2, (rows + 4095) / 4096));
}

cudaError_t launch_qr_project(const double2* Q, int64_t rows, int t, double2* v, double2* part,
                              double2* s, double2* acc, cudaStream_t st) {
  if (t == 0) return cudaSuccess;
  const int nb = qr_dot_blocks(rows);
  k_qr_dots<<<dim3(nb, t), QR_THREADS, 0, st>>>(Q, rows, v, part);
  k_qr_reduce<<<(t + 127) / 128, 128, 0, st>>>(part, nb, t, s, acc);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(num_sms() * 8, (rows + QR_THREADS - 1) / QR_THREADS));
  k_qr_update<<<grid, QR_THREADS, (size_t)t * sizeof(double2), st>>>(Q, rows, t, s, v);
  g_launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_qr_norm(const double2* v, int64_t rows, double* part, double* out, cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(num_sms() * 4, (rows + QR_THREADS - 1) / QR_THREADS));
  k_qr_norm<<<grid, QR_THREADS, 0, st>>>(v, rows, part);
  k_qr_sum<<<1, 256, 0, st>>>(part, grid, out);
  g_launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_qr_store(double2* qnew, const double2* v, int64_t rows, double inv, cudaStream_t st) {
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(num_sms() * 8, (rows + QR_THREADS - 1) / QR_THREADS));
  k_qr_store<<<grid, QR_THREADS, 0, st>>>(qnew, v, rows, inv);
  ++g_launches;
  return cudaGetLastError();
}

// z_i = q_i^H rhs for the t columns (partials then the fixed-order sum)
cudaError_t launch_qr_dots(const double2* Q, int64_t rows, int t, const double2* rhs, double2* part,
                           double2* z, double2* scratch, cudaStream_t st) {
  if (t == 0) return cudaSuccess;
  const int nb = qr_dot_blocks(rows);
  k_qr_dots<<<dim3(nb, t), QR_THREADS, 0, st>>>(Q, rows, rhs, part);
  cudaMemsetAsync(scratch, 0, (size_t)t * sizeof(double2), st);
  k_qr_reduce<<<(t + 127) / 128, 128, 0, st>>>(part, nb, t, z, scratch);
  g_launches += 2;
  return cudaGetLastError();
}

}  // namespace fmp
