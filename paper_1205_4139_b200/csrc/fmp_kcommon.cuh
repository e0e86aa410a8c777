// Internal helpers shared by the kernel translation units.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "fmp_device.cuh"
#include "fmp_kernels.cuh"

namespace fmp {
extern thread_local int g_launches;
}  // namespace fmp

namespace fmp {

namespace {

// streamed input: spin (acquire) until the copy stream has flagged the
// chunk.  Returns false instead when the host raised the abort word (a
// page-locked, device-mapped int the host sets on an error path, so no CUDA
// call is needed to release the kernel) or after 60 s without the flag; the
// caller then marks its problems failed and the host reports FMP_ECUDA.  No
// trap: the context survives.
__device__ __forceinline__ bool wait_ready(const int* flag, const volatile int* abort_word) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  // the abort word lives in host memory: a read crosses PCIe and competes
  // with the input copies, so it is polled once per millisecond of waiting
  unsigned long long next_poll = t0 + 1000000ull;
  for (;;) {
    int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
    if (v) return true;
    __nanosleep(500);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t >= next_poll) {
      if (abort_word && *abort_word) return false;
      if (t - t0 > 60000000000ull) return false;
      next_poll = t + 1000000ull;
    }
  }
}
// aborted[] value of a problem whose streamed input never arrived
constexpr int kInputLost = 2;

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 1;
  }
  return sms;
}

int smem_optin() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (v <= 0) v = 48 * 1024;
  }
  return v;
}

template <class V> struct scal;
template <> struct scal<double2> { using T = double; };
template <> struct scal<float2> { using T = float; };
template <> struct scal<double> { using T = double; };
template <> struct scal<float> { using T = float; };

template <class V> __device__ __forceinline__ const V* twiddles(const DevOp& op);
template <> __device__ __forceinline__ const double2* twiddles<double2>(const DevOp& op) { return op.tw64; }
template <> __device__ __forceinline__ const float2* twiddles<float2>(const DevOp& op) { return op.tw32; }
template <> __device__ __forceinline__ const double* twiddles<double>(const DevOp&) { return nullptr; }
template <> __device__ __forceinline__ const float* twiddles<float>(const DevOp&) { return nullptr; }

template <class V> __device__ __forceinline__ const V* fourier_table(const DevOp& op);
template <> __device__ __forceinline__ const double2* fourier_table<double2>(const DevOp& op) { return op.g64; }
template <> __device__ __forceinline__ const float2* fourier_table<float2>(const DevOp& op) { return op.g32; }
template <> __device__ __forceinline__ const double* fourier_table<double>(const DevOp&) { return nullptr; }
template <> __device__ __forceinline__ const float* fourier_table<float>(const DevOp&) { return nullptr; }

constexpr int RMAX = 16;
constexpr int LOGP = 4;
#ifndef FMP_OMP_THREADS
#define FMP_OMP_THREADS 512
#endif
constexpr int OMP_THREADS = FMP_OMP_THREADS;
constexpr int FU_THREADS = 512;

__device__ __forceinline__ double inv_sqrt_n(int n) { return 1.0 / sqrt((double)n); }

// slot of logical input position p for the in-place transform
template <bool HAD>
__device__ __forceinline__ int in_slot(unsigned p, int log2n) {
  return padx<LOGP>(HAD ? (int)p : (int)brev_n(p, log2n));
}

// ------------------------------------------------------------ fast tile
// acc[r] (outputs i0 + lane + 32 r) -= sum_tau xn-scaled kernel entries.
// Fourier: source (i - lambda) mod n (kernel.cpp:247-255, map_index
// kernel.cpp:111-118); Hadamard: i XOR lambda on the integer lattice N*c
// (kernel.cpp:227-238), xn = -x/N so that xn * k == -x * c exactly.
// Exact conversion of a biased lattice entry u = k + 32768 to k in T without
// the (slow, XU-pipe) integer conversion: 2^52 + u (2^23 + u for float) is
// assembled from its bit pattern and the bias subtracted, both exact.
__device__ __forceinline__ void lat_to(unsigned u, double& o) {
  o = __hiloint2double(0x43300000, (int)u) - 4503599627403264.0;  // 2^52 + 2^15
}
__device__ __forceinline__ void lat_to(unsigned u, float& o) {
  o = __int_as_float(0x4B000000 | (int)u) - 8421376.0f;  // 2^23 + 2^15
}

// acc -= x * conj(g) with xn = -x
__device__ __forceinline__ void msub_conj(double2& acc, double2 xn, double2 g) {
  acc.x = fma(xn.x, g.x, acc.x);
  acc.x = fma(xn.y, g.y, acc.x);
  acc.y = fma(xn.y, g.x, acc.y);
  acc.y = fma(-xn.x, g.y, acc.y);
}
__device__ __forceinline__ void msub_conj(float2& acc, float2 xn, float2 g) {
  acc.x = fmaf(xn.x, g.x, acc.x);
  acc.x = fmaf(xn.y, g.y, acc.x);
  acc.y = fmaf(xn.y, g.x, acc.y);
  acc.y = fmaf(-xn.x, g.y, acc.y);
}
template <class V>
__device__ __forceinline__ void msub_conj(V&, V, V) {}

// acc[r] -= x gk[r ^ lr] for a warp-uniform lr < RPT (fixed register maps)
template <int RPT, int LR, class V, class T>
__device__ __forceinline__ void lattice_mac_fixed(V (&acc)[RPT], V x, const T (&gk)[RPT]) {
#pragma unroll
  for (int r = 0; r < RPT; ++r) msub(acc[r], x, gk[r ^ LR]);
}
template <int RPT, class V, class T>
__device__ __forceinline__ void lattice_mac(V (&acc)[RPT], V x, const T (&gk)[RPT], int lr) {
  switch (lr) {
    case 0: lattice_mac_fixed<RPT, 0>(acc, x, gk); break;
    case 1: if constexpr (RPT > 1) lattice_mac_fixed<RPT, 1 % RPT>(acc, x, gk); break;
    case 2: if constexpr (RPT > 2) lattice_mac_fixed<RPT, 2 % RPT>(acc, x, gk); break;
    case 3: if constexpr (RPT > 3) lattice_mac_fixed<RPT, 3 % RPT>(acc, x, gk); break;
    case 4: if constexpr (RPT > 4) lattice_mac_fixed<RPT, 4 % RPT>(acc, x, gk); break;
    case 5: if constexpr (RPT > 5) lattice_mac_fixed<RPT, 5 % RPT>(acc, x, gk); break;
    case 6: if constexpr (RPT > 6) lattice_mac_fixed<RPT, 6 % RPT>(acc, x, gk); break;
    default: if constexpr (RPT > 7) lattice_mac_fixed<RPT, 7 % RPT>(acc, x, gk); break;
  }
}

// HALFG: the Fourier kernel is stored as its conjugate-symmetric half,
// c[0..n/2] (c[n-j] = conj(c[j]), kernel.cpp:35-45); windows that stay on one
// side of n/2 read it forwards (lower) or mirrored and conjugated (upper).
template <class V, bool HAD, int RPT, bool HALFG = false>
__device__ __forceinline__ void fast_tile(V (&acc)[RPT], int i0, int lane, int n,
                                          const V* __restrict__ gF,
                                          const uint16_t* __restrict__ gH,
                                          const unsigned* lam, const V* xn, int t) {
  using T = typename scal<V>::T;
  const int mask = n - 1;
  if (t <= 0) return;
  // the atom list is read one step ahead so its smem latency overlaps the
  // previous atom's kernel loads and FMAs
  int l_nx = (int)lam[0];
  V x_nx = xn[0];
  if constexpr (!HAD) {
    for (int tau = 0; tau < t; ++tau) {
      const int l = l_nx;
      const V x = x_nx;
      if (tau + 1 < t) {
        l_nx = (int)lam[tau + 1];
        x_nx = xn[tau + 1];
      }
      const int w0 = (i0 - l) & mask;
      if constexpr (!HALFG) {
        if (w0 + 32 * RPT <= n) {
          const V* p = gF + w0 + lane;
          V gv[RPT];
#pragma unroll
          for (int r = 0; r < RPT; ++r) gv[r] = p[32 * r];
#pragma unroll
          for (int r = 0; r < RPT; ++r) msub(acc[r], x, gv[r]);
        } else {
#pragma unroll
          for (int r = 0; r < RPT; ++r) msub(acc[r], x, gF[(w0 + lane + 32 * r) & mask]);
        }
      } else {
        const int half = n >> 1;
        if (w0 + 32 * RPT <= half + 1) {
          const V* p = gF + w0 + lane;
          V gv[RPT];
#pragma unroll
          for (int r = 0; r < RPT; ++r) gv[r] = p[32 * r];
#pragma unroll
          for (int r = 0; r < RPT; ++r) msub(acc[r], x, gv[r]);
        } else if (w0 > half && w0 + 32 * RPT <= n) {
          const V* p = gF + (n - w0 - lane);
          V gv[RPT];
#pragma unroll
          for (int r = 0; r < RPT; ++r) gv[r] = p[-32 * r];
#pragma unroll
          for (int r = 0; r < RPT; ++r) msub_conj(acc[r], x, gv[r]);
        } else {
#pragma unroll
          for (int r = 0; r < RPT; ++r) {
            const int j = (w0 + lane + 32 * r) & mask;
            if (j <= half) msub(acc[r], x, gF[j]);
            else msub_conj(acc[r], x, gF[n - j]);
          }
        }
      }
    }
  } else {
    for (int tau = 0; tau < t; ++tau) {
      const int l = l_nx;
      const V x = x_nx;
      if (tau + 1 < t) {
        l_nx = (int)lam[tau + 1];
        x_nx = xn[tau + 1];
      }
      // output i0 + lane + 32 r reads entry (i0 + lane + 32 r) XOR l: the 32
      // RPT block is permuted row-wise by lr = (l >> 5) mod RPT, which is
      // uniform over the warp, so the loads use compile-time offsets from
      // one base and the permutation is a branch to a fixed register mapping
      const uint16_t* pb = gH + (i0 ^ (l & ~(32 * RPT - 1))) + (lane ^ (l & 31));
      const int lr = (l >> 5) & (RPT - 1);
      T gk[RPT];
#pragma unroll
      for (int k = 0; k < RPT; ++k) lat_to((unsigned)pb[32 * k], gk[k]);
      lattice_mac<RPT>(acc, x, gk, lr);
    }
  }
}

// single output (small n): h0 value in acc
template <class V, bool HAD, bool HALFG = false>
__device__ __forceinline__ void fast_point(V& acc, int i, int n, const V* __restrict__ gF,
                                           const uint16_t* __restrict__ gH,
                                           const unsigned* lam, const V* xn, int t) {
  using T = typename scal<V>::T;
  for (int tau = 0; tau < t; ++tau) {
    const int l = (int)lam[tau];
    if constexpr (!HAD) {
      const int j = (i - l) & (n - 1);
      if (!HALFG || j <= (n >> 1)) msub(acc, xn[tau], gF[j]);
      else msub_conj(acc, xn[tau], gF[n - j]);
    }
    else {
      T gv;
      lat_to((unsigned)gH[i ^ l], gv);
      msub(acc, xn[tau], gv);
    }
  }
}

// ----------------------------------------------------------------- argmax
template <class V>
__global__ void __launch_bounds__(512) k_argmax(const V* __restrict__ h, int64_t n,
                                                int64_t batch, uint64_t* __restrict__ out) {
  __shared__ double red[32];
  __shared__ unsigned redu[32];
  const int tid = threadIdx.x, nth = blockDim.x;
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    const V* hb = h + b * n;
    double best = 0.0;
    for (int64_t k = tid; k < n; k += nth) best = fmax(best, mag2(hb[k]));
    best = block_max(best, red);
    const double cut = best * (1.0 - kTieBandRel);
    unsigned first = 0xffffffffu;
    for (int64_t k = tid; k < n; k += nth)
      if (mag2(hb[k]) >= cut) { first = (unsigned)k; break; }
    first = block_min_u(first, redu);
    if (tid == 0) out[b] = (first == 0xffffffffu ? 0u : first) + 1;  // 1-based
    __syncthreads();
  }
}

}  // namespace
}  // namespace fmp
