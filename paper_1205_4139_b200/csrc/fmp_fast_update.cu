// Batched fast correlation update h = h0 - sum_tau x_tau P_{lambda_tau} c
// (kernel.cpp:209-303) with an optional fused band argmax.
#include "fmp_kcommon.cuh"

namespace fmp {
namespace {
// ----------------------------------------------------------- fast update
template <class V, bool HAD, int RPT, bool GSM>
__global__ void __launch_bounds__(FU_THREADS) k_fast_update(
    DevOp op, const V* __restrict__ h0, const uint32_t* __restrict__ support,
    const V* __restrict__ coeffs, int t, int64_t batch, V* __restrict__ hout,
    uint64_t* __restrict__ amax, double* __restrict__ mag_ws, int chunk) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[32];
  __shared__ unsigned redu[32];
  const int n = (int)op.n;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5,
            nw = nth >> 5;
  // staged kernel table, then the atom chunk (lambda, -x or -x/N)
  const V* gF = fourier_table<V>(op);
  const uint16_t* gH = op.glat;
  size_t goff = 0;
  if constexpr (GSM) {
    if constexpr (!HAD) {
      V* s = reinterpret_cast<V*>(smem_raw);
      for (int i = tid; i < n; i += nth) s[i] = gF[i];
      gF = s;
      goff = (size_t)n * sizeof(V);
    } else {
      uint16_t* s = reinterpret_cast<uint16_t*>(smem_raw);
      const int* src = reinterpret_cast<const int*>(op.glat);
      int* dst = reinterpret_cast<int*>(s);
      for (int i = tid; i < n / 2; i += nth) dst[i] = src[i];
      if ((n & 1) && tid == 0) s[n - 1] = op.glat[n - 1];
      gH = s;
      goff = (((size_t)n * 2 + 15) / 16) * 16;
    }
  }
  V* s_xn = reinterpret_cast<V*>(smem_raw + goff);
  unsigned* s_lam = reinterpret_cast<unsigned*>(s_xn + chunk);
  const double xscale = HAD ? -1.0 / (double)n : -1.0;
  double* msc = mag_ws + (size_t)blockIdx.x * n;

  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    const V* hb = h0 + b * n;
    V* ob = hout ? hout + b * n : nullptr;
    double best = 0.0;
    // outputs are produced tile by tile; the atom list is consumed in chunks
    const int ntiles = n >= 32 * RPT ? n / (32 * RPT) : 0;
    for (int c0 = 0; c0 < t || c0 == 0; c0 += chunk) {
      const int cn = min(chunk, t - c0);
      __syncthreads();
      for (int j = tid; j < cn; j += nth) {
        s_lam[j] = support[b * t + c0 + j];
        s_xn[j] = scale(coeffs[b * t + c0 + j], xscale);
      }
      __syncthreads();
      const bool first = c0 == 0, last = c0 + chunk >= t;
      const V* src = first ? hb : ob;  // later chunks continue from the partial h
      if (ntiles) {
        for (int tile = warp; tile < ntiles; tile += nw) {
          const int i0 = tile * 32 * RPT;
          V acc[RPT];
#pragma unroll
          for (int r = 0; r < RPT; ++r) acc[r] = src[i0 + lane + 32 * r];
          fast_tile<V, HAD, RPT>(acc, i0, lane, n, gF, gH, s_lam, s_xn, cn);
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const int i = i0 + lane + 32 * r;
            if (ob) ob[i] = acc[r];
            if (last) {
              const double mm = mag2(acc[r]);
              msc[i] = mm;
              best = fmax(best, mm);
            }
          }
        }
      } else {
        for (int i = tid; i < n; i += nth) {
          V acc = src[i];
          fast_point<V, HAD>(acc, i, n, gF, gH, s_lam, s_xn, cn);
          if (ob) ob[i] = acc;
          if (last) {
            const double mm = mag2(acc);
            msc[i] = mm;
            best = fmax(best, mm);
          }
        }
      }
      if (t == 0) break;
    }
    if (amax) {
      best = block_max(best, red);
      const double cut = best * (1.0 - kTieBandRel);
      unsigned firsti = 0xffffffffu;
      for (int k = tid; k < n; k += nth)
        if (msc[k] >= cut) { firsti = (unsigned)k; break; }
      firsti = block_min_u(firsti, redu);
      if (tid == 0) amax[b] = (firsti == 0xffffffffu ? 0u : firsti) + 1;  // 1-based
    }
  }
}

template <class V, bool HAD, int RPT>
cudaError_t launch_fu_t(const FastUpdateArgs& a, cudaStream_t st) {
  const DevOp& op = *a.op;
  const int n = (int)op.n;
  const size_t gbytes = HAD ? (((size_t)n * 2 + 15) / 16) * 16 : (size_t)n * sizeof(V);
  int chunk = (int)std::min<int64_t>(std::max<int64_t>(a.t, 1), 1024);
  const size_t small = (size_t)chunk * (sizeof(V) + 4) + 16;
  const bool gsm = gbytes + small <= (size_t)smem_optin() - 2048;
  const size_t smem = (gsm ? gbytes : 0) + small;
  const int grid = std::max(1, a.grid);
  if (gsm) {
    auto k = k_fast_update<V, HAD, RPT, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, FU_THREADS, smem, st>>>(op, (const V*)a.h0, a.support, (const V*)a.coeffs,
                                       (int)a.t, a.batch, (V*)a.h_out, a.argmax_out,
                                       a.mag_ws, chunk);
  } else {
    auto k = k_fast_update<V, HAD, RPT, false>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, FU_THREADS, smem, st>>>(op, (const V*)a.h0, a.support, (const V*)a.coeffs,
                                       (int)a.t, a.batch, (V*)a.h_out, a.argmax_out,
                                       a.mag_ws, chunk);
  }
  ++g_launches;
  return cudaGetLastError();
}

template <class V, bool HAD>
cudaError_t launch_fu_v(const FastUpdateArgs& a, cudaStream_t st) {
  const int64_t n = a.op->n;
  if (n >= 32 * 8 * 16) return launch_fu_t<V, HAD, 8>(a, st);
  return launch_fu_t<V, HAD, 2>(a, st);
}

}  // namespace

int fast_update_grid(const DevOp&, int, int64_t batch) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(batch, num_sms()));
}

cudaError_t launch_fast_update(const FastUpdateArgs& a, cudaStream_t st) {
  g_launches = 0;
  const bool had = a.op->kind == HADAMARD;
  if (had && !a.op->glat) return cudaErrorInvalidValue;
  switch (a.dtype) {
    case C128: return had ? launch_fu_v<double2, true>(a, st) : launch_fu_v<double2, false>(a, st);
    case C64: return had ? launch_fu_v<float2, true>(a, st) : launch_fu_v<float2, false>(a, st);
    case F64: return had ? launch_fu_v<double, true>(a, st) : cudaErrorInvalidValue;
    case F32: return had ? launch_fu_v<float, true>(a, st) : cudaErrorInvalidValue;
  }
  return cudaErrorInvalidValue;
}

}  // namespace fmp
