// Device building blocks for the OMP correlation path on sm_100a.
//
// Element types: complex data is double2 (c128) or float2 (c64); real
// (Hadamard with real data) is double (f64) or float (f32).  Atom and row
// indices are 0-based on the device (the C ABI converts from the reference's
// 1-based convention, proj/include/fastmp/transform.hpp:32-34).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fmp {

constexpr double kTieBandRel = 1e-9;  // solvers.cpp:40

// ------------------------------------------------------------ element ops
template <class T> struct vec2;
template <> struct vec2<double> { using type = double2; };
template <> struct vec2<float> { using type = float2; };

template <class T, bool CPLX> struct elem { using V = typename vec2<T>::type; };
template <class T> struct elem<T, false> { using V = T; };

__device__ __forceinline__ double2 zero_of(double2) { return make_double2(0.0, 0.0); }
__device__ __forceinline__ float2 zero_of(float2) { return make_float2(0.f, 0.f); }
__device__ __forceinline__ double zero_of(double) { return 0.0; }
__device__ __forceinline__ float zero_of(float) { return 0.f; }

__device__ __forceinline__ double2 add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 add(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double add(double a, double b) { return a + b; }
__device__ __forceinline__ float add(float a, float b) { return a + b; }
__device__ __forceinline__ double2 sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 sub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double sub(double a, double b) { return a - b; }
__device__ __forceinline__ float sub(float a, float b) { return a - b; }

__device__ __forceinline__ double2 scale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ float2 scale(float2 a, double s) { return make_float2(a.x * (float)s, a.y * (float)s); }
__device__ __forceinline__ double scale(double a, double s) { return a * s; }
__device__ __forceinline__ float scale(float a, double s) { return a * (float)s; }

// |z|^2 evaluated in fp64 (float products are exact in double)
__device__ __forceinline__ double mag2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double mag2(float2 a) { return (double)a.x * a.x + (double)a.y * a.y; }
__device__ __forceinline__ double mag2(double a) { return a * a; }
__device__ __forceinline__ double mag2(float a) { return (double)a * a; }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 conj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ float2 conj(float2 a) { return make_float2(a.x, -a.y); }

// to/from the fp64 complex the least-squares state is kept in
__device__ __forceinline__ void from_c128(double2 v, double2& o) { o = v; }
__device__ __forceinline__ void from_c128(double2 v, float2& o) { o = make_float2((float)v.x, (float)v.y); }
__device__ __forceinline__ void from_c128(double2 v, double& o) { o = v.x; }
__device__ __forceinline__ void from_c128(double2 v, float& o) { o = (float)v.x; }
__device__ __forceinline__ double2 to_c128(double2 v) { return v; }
__device__ __forceinline__ double2 to_c128(float2 v) { return make_double2(v.x, v.y); }
__device__ __forceinline__ double2 to_c128(double v) { return make_double2(v, 0.0); }
__device__ __forceinline__ double2 to_c128(float v) { return make_double2(v, 0.0); }

// acc -= x * g, with x complex (xn = -x pre-negated) and g complex or real
__device__ __forceinline__ void msub(double2& acc, double2 xn, double2 g) {
  acc.x = fma(xn.x, g.x, acc.x);
  acc.x = fma(-xn.y, g.y, acc.x);
  acc.y = fma(xn.x, g.y, acc.y);
  acc.y = fma(xn.y, g.x, acc.y);
}
__device__ __forceinline__ void msub(float2& acc, float2 xn, float2 g) {
  acc.x = fmaf(xn.x, g.x, acc.x);
  acc.x = fmaf(-xn.y, g.y, acc.x);
  acc.y = fmaf(xn.x, g.y, acc.y);
  acc.y = fmaf(xn.y, g.x, acc.y);
}
__device__ __forceinline__ void msub(double2& acc, double2 xn, double g) {
  acc.x = fma(xn.x, g, acc.x);
  acc.y = fma(xn.y, g, acc.y);
}
__device__ __forceinline__ void msub(float2& acc, float2 xn, float g) {
  acc.x = fmaf(xn.x, g, acc.x);
  acc.y = fmaf(xn.y, g, acc.y);
}
__device__ __forceinline__ void msub(double& acc, double xn, double g) { acc = fma(xn, g, acc); }
__device__ __forceinline__ void msub(float& acc, float xn, float g) { acc = fmaf(xn, g, acc); }

// ------------------------------------------------------ transform passes
//
// In-place transforms on a buffer laid out with one pad slot every RMAX
// elements (conflict-free strided smem access for every pass).  The Fourier
// transform is a decimation-in-time FFT that consumes bit-reversed input and
// produces natural order (the same factorisation as the reference's radix-2
// DIT, transform.cpp:60-84, grouped into radix-R passes); callers scatter
// their input straight to bit-reversed slots, so no permutation pass exists.
// The Hadamard transform (transform.cpp:86-100) runs on natural order.

__host__ __device__ constexpr double c16(int k) {  // cos(2 pi k / 16)
  return (k & 15) == 0 ? 1.0
       : (k & 15) == 1 ? 0.92387953251128675613
       : (k & 15) == 2 ? 0.70710678118654752440
       : (k & 15) == 3 ? 0.38268343236508977173
       : (k & 15) == 4 ? 0.0
       : (k & 15) == 5 ? -0.38268343236508977173
       : (k & 15) == 6 ? -0.70710678118654752440
       : (k & 15) == 7 ? -0.92387953251128675613
       : (k & 15) == 8 ? -1.0
       : (k & 15) == 9 ? -0.92387953251128675613
       : (k & 15) == 10 ? -0.70710678118654752440
       : (k & 15) == 11 ? -0.38268343236508977173
       : (k & 15) == 12 ? 0.0
       : (k & 15) == 13 ? 0.38268343236508977173
       : (k & 15) == 14 ? 0.70710678118654752440
       : 0.92387953251128675613;
}

// v * W_len^j, W = exp(-2 pi i / len) (conjugated when INV); len <= 16
template <bool INV, class V>
__device__ __forceinline__ V mul_wconst(V v, int len, int j) {
  if (j == 0) return v;
  const int k = j * (16 / len);  // W_16^k
  if (k == 4) {  // -i (forward) / +i (inverse)
    V o;
    if (INV) { o.x = -v.y; o.y = v.x; } else { o.x = v.y; o.y = -v.x; }
    return o;
  }
  const double c = c16(k), s = INV ? c16(k - 4) : -c16(k - 4);  // W = c + i s
  V w;
  w.x = (decltype(v.x))c;
  w.y = (decltype(v.x))s;
  return cmul(v, w);
}

// R-point DFT in registers, input in bit-reversed order, output natural.
// Stages are template-recursive so every register index is a compile-time
// constant (a runtime-indexed v[] would be placed in local memory).
template <int R, bool INV, int LEN, class V>
__device__ __forceinline__ void dft_stage(V (&v)[R]) {
  if constexpr (LEN <= R) {
#pragma unroll
    for (int base = 0; base < R; base += LEN) {
#pragma unroll
      for (int j = 0; j < LEN / 2; ++j) {
        const V t = mul_wconst<INV>(v[base + j + LEN / 2], LEN, j);
        const V u = v[base + j];
        v[base + j] = add(u, t);
        v[base + j + LEN / 2] = sub(u, t);
      }
    }
    dft_stage<R, INV, LEN * 2>(v);
  }
}

template <int R, bool INV, class V>
__device__ __forceinline__ void dft_reg(V (&v)[R]) {
  dft_stage<R, INV, 2>(v);
}

// R-point Walsh-Hadamard in registers (natural order)
template <int R, int HALF, class V>
__device__ __forceinline__ void wht_stage(V (&v)[R]) {
  if constexpr (HALF < R) {
#pragma unroll
    for (int base = 0; base < R; base += 2 * HALF) {
#pragma unroll
      for (int j = 0; j < HALF; ++j) {
        const V a = v[base + j], b = v[base + j + HALF];
        v[base + j] = add(a, b);
        v[base + j + HALF] = sub(a, b);
      }
    }
    wht_stage<R, HALF * 2>(v);
  }
}

template <int R, class V>
__device__ __forceinline__ void wht_reg(V (&v)[R]) {
  wht_stage<R, 1>(v);
}

template <int LOGR>
__device__ __forceinline__ int padx(int p) { return p + (p >> LOGR); }

__device__ __forceinline__ unsigned brev_n(unsigned x, int log2n) {
  return log2n ? (__brev(x) >> (32 - log2n)) : 0u;
}

template <int R>
__host__ __device__ constexpr int brev_small(int j) {
  int r = 0;
  for (int b = 1, rb = R >> 1; b < R; b <<= 1, rb >>= 1)
    if (j & b) r |= rb;
  return r;
}

// j with brev_small<R>(j) == q (bit reversal is an involution)
template <int R>
__host__ __device__ constexpr int brev_inv(int q) { return brev_small<R>(q); }

template <int R> struct log2_of { static constexpr int v = R <= 1 ? 0 : 1 + log2_of<R / 2>::v; };
template <> struct log2_of<1> { static constexpr int v = 0; };

// Twiddle providers: tw(k) = exp(-2 pi i k / 2^log2tab) for k < 2^log2tab.
template <class V>
struct TwTable {  // full table (global memory, L1/L2 cached); direct lookups
  static constexpr bool kPowers = false;
  const V* __restrict__ p;
  __device__ __forceinline__ V operator()(int k) const { return p[k]; }
};
template <class V>
struct TwTwoLevel {  // W^k = lo[k mod 2^a] * hi[k >> a]; both tiny, in smem
  // a pass needs W^(rho step) for rho < R: one lookup, then products
  // (at most 4 roundings deep), which keeps smem traffic to the data itself
  static constexpr bool kPowers = true;
  const V* lo;  // padded: entry i at i + i/8 (pass indices are strided by 8)
  const V* hi;
  int a;
  __device__ __forceinline__ static int pad(int i) { return i + (i >> 3); }
  __device__ __forceinline__ V operator()(int k) const {
    return cmul(lo[pad(k & ((1 << a) - 1))], hi[pad(k >> a)]);
  }
};

// One radix-R sub-problem u of the pass over sub-blocks of span S = 2^logS
// (see file comment); the twiddle table has 2^log2tab entries (it may be
// longer than the vector).
template <int R, int LOGP, bool INV, bool HAD, class V, class TW>
__device__ __forceinline__ void pass_one(V* buf, int log2n, int logS, int log2tab,
                                         const TW& tw, int u) {
  constexpr int LOGR = log2_of<R>::v;
  const int S = 1 << logS;
  const int o = u & (S - 1);
  const int base = ((u >> logS) << (logS + LOGR)) + o;
  V v[R];
#pragma unroll
  for (int j = 0; j < R; ++j) v[j] = buf[padx<LOGP>(base + j * S)];
  if constexpr (HAD) {
    wht_reg<R>(v);
  } else {
    if (logS > 0) {
      // twiddle index brev(j) * o * 2^log2tab / (R S)
      const int step = o << (log2tab - logS - LOGR);
      if constexpr (TW::kPowers) {
        // powers w^q applied as they are formed; only w, w^2, w^4, w^8 stay
        // live (register pressure at 64 registers per thread)
        V w1 = tw(step);
        if (INV) w1.y = -w1.y;
        V p2 = w1, p4 = w1, p8 = w1;
#pragma unroll
        for (int q = 1; q < R; ++q) {
          V wq;
          if (q == 1) wq = w1;
          else if (q == 2) wq = p2 = cmul(w1, w1);
          else if (q == 4) wq = p4 = cmul(p2, p2);
          else if (q == 8) wq = p8 = cmul(p4, p4);
          else {
            wq = (q & 8) ? p8 : ((q & 4) ? p4 : p2);
            const int rest = q & ((q & 8) ? 7 : ((q & 4) ? 3 : 1));
            if (rest & 4) wq = cmul(wq, p4);
            if (rest & 2) wq = cmul(wq, p2);
            if (rest & 1) wq = cmul(wq, w1);
          }
          v[brev_inv<R>(q)] = cmul(v[brev_inv<R>(q)], wq);
        }
      } else {
#pragma unroll
        for (int j = 1; j < R; ++j) {
          V w = tw(brev_small<R>(j) * step);
          if (INV) w.y = -w.y;
          v[j] = cmul(v[j], w);
        }
      }
    }
    dft_reg<R, INV>(v);
  }
#pragma unroll
  for (int j = 0; j < R; ++j) buf[padx<LOGP>(base + j * S)] = v[j];
}

template <int R, int LOGP, bool INV, bool HAD, class V, class TW>
__device__ __forceinline__ void transform_pass(V* buf, int log2n, int logS, const TW& tw,
                                               int tid, int nth, int log2tab) {
  constexpr int LOGR = log2_of<R>::v;
  const int nsub = 1 << (log2n - LOGR);
  for (int u = tid; u < nsub; u += nth)
    pass_one<R, LOGP, INV, HAD>(buf, log2n, logS, log2tab, tw, u);
}

// Whole in-place transform of one vector held by the calling block, radix
// RMAX passes then one smaller remainder pass; padding period RMAX.
// Ends with a __syncthreads().
// pass 0 of a transform whose input is produced on the fly: LOAD(slot)
// returns the input element at (unpadded) slot, so the buffer needs no
// zero-fill or scatter beforehand
template <int R, int LOGP, bool INV, bool HAD, class V, class LOAD>
__device__ __forceinline__ void first_pass_loaded(V* buf, int log2n, const LOAD& load, int tid,
                                                  int nth) {
  const int nsub = 1 << (log2n - log2_of<R>::v);
  for (int u = tid; u < nsub; u += nth) {
    V v[R];
#pragma unroll
    for (int j = 0; j < R; ++j) v[j] = load(u * R + j);
    if constexpr (HAD) wht_reg<R>(v);
    else dft_reg<R, INV>(v);
#pragma unroll
    for (int j = 0; j < R; ++j) buf[padx<LOGP>(u * R + j)] = v[j];
  }
}

// first pass driven by a slot map (int16, -1 = zero slot): each thread
// fetches its R = 8 map entries with one 16-byte load (consecutive threads,
// consecutive 16-byte words: no bank conflicts), then the values it maps to
template <int LOGP, bool INV, bool HAD, class V, class VAL>
__device__ __forceinline__ void first_pass_map8(V* buf, int log2n, const int16_t* map, const VAL& val,
                                                int tid, int nth) {
  const int nsub = 1 << (log2n - 3);
  const int4* m4 = reinterpret_cast<const int4*>(map);
  for (int u = tid; u < nsub; u += nth) {
    const int4 w = m4[u];
    const int packed[4] = {w.x, w.y, w.z, w.w};
    V v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int q = (int)(int16_t)((packed[j >> 1] >> (16 * (j & 1))) & 0xFFFF);
      v[j] = val(q);
    }
    if constexpr (HAD) wht_reg<8>(v);
    else dft_reg<8, INV>(v);
#pragma unroll
    for (int j = 0; j < 8; ++j) buf[padx<LOGP>(u * 8 + j)] = v[j];
  }
}

// log2tab: size of the twiddle table (defaults to the vector); a block that
// runs the first stages of a longer transform passes the full length.
template <int RMAX, bool INV, bool HAD, class V, class TW>
__device__ void block_transform(V* buf, int log2n, const TW& tw, int tid, int nth,
                                int log2tab = -1, int s = 0) {
  constexpr int LOGP = log2_of<RMAX>::v;
  if (log2tab < 0) log2tab = log2n;
  for (; log2n - s >= LOGP; s += LOGP) {
    transform_pass<RMAX, LOGP, INV, HAD>(buf, log2n, s, tw, tid, nth, log2tab);
    __syncthreads();
  }
  switch (log2n - s) {
    case 1: transform_pass<2, LOGP, INV, HAD>(buf, log2n, s, tw, tid, nth, log2tab); __syncthreads(); break;
    case 2: transform_pass<4, LOGP, INV, HAD>(buf, log2n, s, tw, tid, nth, log2tab); __syncthreads(); break;
    case 3: if constexpr (RMAX > 8) {
              transform_pass<8, LOGP, INV, HAD>(buf, log2n, s, tw, tid, nth, log2tab); __syncthreads();
            }
            break;
    default: break;
  }
}

// ------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ unsigned warp_min_u(unsigned v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// reductions of the per-warp partials held by lanes 0..NWC-1 (the other
// lanes hold the identity): log2(NWC) butterfly rounds then a broadcast of
// lane 0, bitwise the same result as the full five-round butterfly (the
// extra rounds only combine identities).  NWC = 0: unknown, full butterfly.
template <int NWC>
__device__ __forceinline__ double xsum_nw(double v) {
  if constexpr (NWC <= 0 || NWC >= 32) {
    return warp_sum(v);
  } else {
#pragma unroll
    for (int o = NWC / 2; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return __shfl_sync(0xffffffffu, v, 0);
  }
}
template <int NWC>
__device__ __forceinline__ double xmax_nw(double v) {
  if constexpr (NWC <= 0 || NWC >= 32) {
    return warp_max(v);
  } else {
#pragma unroll
    for (int o = NWC / 2; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return __shfl_sync(0xffffffffu, v, 0);
  }
}
template <int NWC>
__device__ __forceinline__ unsigned xmin_u_nw(unsigned v) {
  if constexpr (NWC <= 0 || NWC >= 32) {
    return warp_min_u(v);
  } else {
#pragma unroll
    for (int o = NWC / 2; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return __shfl_sync(0xffffffffu, v, 0);
  }
}

// block-wide reductions; `red` needs 32 doubles of shared scratch.  Every
// thread receives the result.  Contains two __syncthreads(); LEAD = false
// drops the leading one when the caller knows `red` is not being read.
// NWC: the block's warp count when known at compile time.
template <bool LEAD = true, int NWC = 0>
__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  if (LEAD) __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double r = lane < nw ? red[lane] : 0.0;
  return xmax_nw<NWC>(r);
}
template <int NWC = 0>
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double r = lane < nw ? red[lane] : 0.0;
  return xsum_nw<NWC>(r);
}
// three sums at once; `red` needs 96 doubles
__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  c = warp_sum(c);
  __syncthreads();
  if (lane == 0) {
    red[w] = a;
    red[32 + w] = b;
    red[64 + w] = c;
  }
  __syncthreads();
  a = warp_sum(lane < nw ? red[lane] : 0.0);
  b = warp_sum(lane < nw ? red[32 + lane] : 0.0);
  c = warp_sum(lane < nw ? red[64 + lane] : 0.0);
}
template <bool LEAD = true, int NWC = 0>
__device__ __forceinline__ unsigned block_min_u(unsigned v, unsigned* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_min_u(v);
  if (LEAD) __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  unsigned r = lane < nw ? red[lane] : 0xffffffffu;
  return xmin_u_nw<NWC>(r);
}

}  // namespace fmp
