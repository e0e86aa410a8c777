// Batched fast correlation update h = h0 - sum_tau x_tau P_{lambda_tau} c
// (kernel.cpp:209-303) with an optional fused band argmax.
#include "fmp_kcommon.cuh"

namespace fmp {
namespace {
// --------------------------------------- real Hadamard: quad-lane lattice
// Each lane owns 4 consecutive outputs per 128-output group, so one 8-byte
// shared-memory load brings the 4 lattice entries it needs for an atom: for
// output i = i0 + 128 r + 4 lane + q the entry i XOR l sits in group r ^ lr,
// lane slot lane ^ ll, position q ^ lq (lr, ll, lq fields of l, uniform over
// the warp).  The group permutation lives in the load addresses, the
// position permutation lq is a branch to a fixed register mapping; each entry becomes an exact float / double by one byte permute
// (PRMT) into a magic-number pattern and one bias subtraction, and the
// multiply-adds run packed (FFMA2 / FADD2) for f32.  Same operations and
// order per output as fast_point / fast_tile, so results are unchanged.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
// entry s (0..3) of the 4-entry group held in w as an exact lattice value k
template <int S>
__device__ __forceinline__ float quad_f(uint2 w) {
  const uint32_t word = (S >> 1) ? w.y : w.x;
  return __uint_as_float(prmt(word, 0x4B000000u, (S & 1) ? 0x7632u : 0x7610u));  // 2^23 + u
}
template <int S>
__device__ __forceinline__ double quad_d(uint2 w) {
  const uint32_t word = (S >> 1) ? w.y : w.x;
  const uint32_t u = prmt(word, 0u, (S & 1) ? 0x4432u : 0x4410u);
  return __hiloint2double(0x43300000, (int)u) - 4503599627403264.0;  // 2^52 + 2^15
}

template <int RPT, int LQ>
__device__ __forceinline__ void quad_mac(float2 (&acc)[RPT][2], float x, const uint2 (&w)[RPT]) {
  const float2 xx = make_float2(x, x);
  const float2 bias = make_float2(-8421376.0f, -8421376.0f);  // -(2^23 + 2^15)
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const uint2 ww = w[r];
    const float2 g01 = __fadd2_rn(make_float2(quad_f<0 ^ LQ>(ww), quad_f<1 ^ LQ>(ww)), bias);
    const float2 g23 = __fadd2_rn(make_float2(quad_f<2 ^ LQ>(ww), quad_f<3 ^ LQ>(ww)), bias);
    acc[r][0] = __ffma2_rn(xx, g01, acc[r][0]);
    acc[r][1] = __ffma2_rn(xx, g23, acc[r][1]);
  }
}
template <int RPT, int LQ>
__device__ __forceinline__ void quad_mac(double (&acc)[RPT][4], double x, const uint2 (&w)[RPT]) {
#pragma unroll
  for (int r = 0; r < RPT; ++r) {
    const uint2 ww = w[r];
    acc[r][0] = fma(x, quad_d<0 ^ LQ>(ww), acc[r][0]);
    acc[r][1] = fma(x, quad_d<1 ^ LQ>(ww), acc[r][1]);
    acc[r][2] = fma(x, quad_d<2 ^ LQ>(ww), acc[r][2]);
    acc[r][3] = fma(x, quad_d<3 ^ LQ>(ww), acc[r][3]);
  }
}
template <int RPT, class A, class T>
__device__ __forceinline__ void quad_mac_q(A& acc, T x, const uint2 (&w)[RPT], int lq) {
  switch (lq) {
    case 0: quad_mac<RPT, 0>(acc, x, w); break;
    case 1: quad_mac<RPT, 1>(acc, x, w); break;
    case 2: quad_mac<RPT, 2>(acc, x, w); break;
    default: quad_mac<RPT, 3>(acc, x, w); break;
  }
}

// accumulator tile of one lane: RPT groups of 4 consecutive outputs
template <class T, int RPT> struct QuadAcc;
template <int RPT> struct QuadAcc<float, RPT> {
  float2 a[RPT][2];
  __device__ __forceinline__ void load(const float* p) {
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const float4 v = *reinterpret_cast<const float4*>(p + 128 * r);
      a[r][0] = make_float2(v.x, v.y);
      a[r][1] = make_float2(v.z, v.w);
    }
  }
  __device__ __forceinline__ float get(int r, int q) const { return (q & 1) ? a[r][q >> 1].y : a[r][q >> 1].x; }
  __device__ __forceinline__ void store(float* p) const {
#pragma unroll
    for (int r = 0; r < RPT; ++r)
      *reinterpret_cast<float4*>(p + 128 * r) = make_float4(a[r][0].x, a[r][0].y, a[r][1].x, a[r][1].y);
  }
};
template <int RPT> struct QuadAcc<double, RPT> {
  double a[RPT][4];
  __device__ __forceinline__ void load(const double* p) {
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      const double2 v0 = *reinterpret_cast<const double2*>(p + 128 * r);
      const double2 v1 = *reinterpret_cast<const double2*>(p + 128 * r + 2);
      a[r][0] = v0.x; a[r][1] = v0.y; a[r][2] = v1.x; a[r][3] = v1.y;
    }
  }
  __device__ __forceinline__ double get(int r, int q) const { return a[r][q]; }
  __device__ __forceinline__ void store(double* p) const {
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
      *reinterpret_cast<double2*>(p + 128 * r) = make_double2(a[r][0], a[r][1]);
      *reinterpret_cast<double2*>(p + 128 * r + 2) = make_double2(a[r][2], a[r][3]);
    }
  }
};

template <class T, int RPT>
__device__ __forceinline__ void fast_tile_quad(QuadAcc<T, RPT>& acc, int i0, int lane,
                                               const uint16_t* __restrict__ gH,
                                               const unsigned* lam, const T* xn, int t) {
  if (t <= 0) return;
  int l_nx = (int)lam[0];
  T x_nx = xn[0];
  for (int tau = 0; tau < t; ++tau) {
    const int l = l_nx;
    const T x = x_nx;
    if (tau + 1 < t) {
      l_nx = (int)lam[tau + 1];
      x_nx = xn[tau + 1];
    }
    // group k of the tile reads entry group ((i0 + 128 k) ^ l) >> 7
    const uint16_t* pb = gH + 4 * (lane ^ ((l >> 2) & 31));
    const int gx = (i0 ^ l) & ~127;
    uint2 w[RPT];
#pragma unroll
    for (int k = 0; k < RPT; ++k) w[k] = *reinterpret_cast<const uint2*>(pb + (gx ^ (128 * k)));
    quad_mac_q<RPT>(acc.a, x, w, l & 3);
  }
}

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
    // real Hadamard with a staged lattice: quad-lane tiles of 128 RPT/4 outputs
    constexpr bool QUAD = HAD && GSM && (sizeof(V) == 4 || sizeof(V) == 8) && RPT >= 4;
    // 8 (f64) or 16 (f32) groups of 128 outputs per warp tile: the per-atom
    // work (atom fetch, address bases, the lq branch) spread over more MACs
    constexpr int QR = sizeof(typename scal<V>::T) == 4 ? 16 : 8;
    const int qtiles = n / (128 * QR);
    const bool quad = QUAD && qtiles >= nw;  // every warp owns a tile
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
      if (quad) {
        using T = typename scal<V>::T;
        for (int tile = warp; tile < qtiles; tile += nw) {
          const int i0 = tile * 128 * QR;
          QuadAcc<T, QR> acc;
          acc.load(reinterpret_cast<const T*>(src) + i0 + 4 * lane);
          fast_tile_quad<T, QR>(acc, i0, lane, gH, s_lam, reinterpret_cast<const T*>(s_xn), cn);
          if (ob) acc.store(reinterpret_cast<T*>(ob) + i0 + 4 * lane);
          if (last && amax) {
#pragma unroll
            for (int r = 0; r < QR; ++r)
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const int i = i0 + 128 * r + 4 * lane + q;
                const double mm = mag2(acc.get(r, q));
                msc[i] = mm;
                best = fmax(best, mm);
              }
          }
        }
      } else if (ntiles) {
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
            if (last && amax) {
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
          if (last && amax) {
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
