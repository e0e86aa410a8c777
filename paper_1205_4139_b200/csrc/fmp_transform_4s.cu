// Large-N structured transforms in two passes over HBM ("four-step"):
// N = N1 N2, x viewed as an N1 x N2 row-major matrix, x[N2 n1 + n2].
//
//   Fourier:  X[k1 + N1 k2] = sum_n2 W_N2^(n2 k2) W_N^(n2 k1) sum_n1 x[N2 n1 + n2] W_N1^(n1 k1)
//   Hadamard: X[N2 k1 + k2] = sum_n2 H_N2(k2, n2) sum_n1 H_N1(k1, n1) x[N2 n1 + n2]
//
// Pass A transforms C adjacent columns per CTA tile (strided loads of C
// consecutive elements = one 32-byte sector per row), applies the inter-pass
// twiddle and writes Y[k1][n2] row-major; pass B transforms C rows per tile
// and writes X (C consecutive outputs per k2 for Fourier, whole rows for
// Hadamard).  Each pass moves N elements in and out once, against
// log16(N) read+write passes of the global radix-16 path.
//
// The Omega ends never touch a dense vector: the adjoint's input (m values
// at Omega) is scattered per column tile from a list sorted by column, the
// forward's output is gathered per row tile from a list sorted by row, and
// a sparse input (the support of the current estimate) is placed per tile.
// Reference semantics: transform.cpp:60-152, sensing.cpp:93-109.
#include <type_traits>

#include "fmp_kcommon.cuh"

namespace fmp {
namespace {

constexpr int FS_THREADS = 512;
constexpr int FS_U = 16;   // tile loads in flight per thread
constexpr int FS_SKEW = 4;  // elements added to the per-vector stride (bank skew)
constexpr int FS_R = 16;   // radix of the in-smem passes (64 registers per thread at 1024 threads)

// One radix-R sub-problem of a decimation-in-frequency pass: the transpose
// of pass_one's DIT step (same index sets and twiddles; the R-point DFT
// first, the twiddles on its outputs after).  Running the DIT passes'
// transposes from the widest span down turns natural-order input into
// bit-reversed-order output, so the tile loads store into smem in order.
template <int R, bool INV, bool HAD, class V, class TW>
__device__ __forceinline__ void pass_dif(V* buf, int logS, int log2tab, const TW& tw, int u) {
  constexpr int LOGR = log2_of<R>::v;
  const int S = 1 << logS;
  const int o = u & (S - 1);
  const int base = ((u >> logS) << (logS + LOGR)) + o;
  // padx(base + j S) = padx(base) + j (S + S / 2^LOGP) when S is a multiple
  // of the padding period, or S = 1 with base a multiple of it (R >= 2^LOGP):
  // one pointer and a constant step instead of a shift and add per element
  const bool lin = logS >= LOGP || (logS == 0 && LOGR >= LOGP);
  V* const p = buf + padx<LOGP>(base);
  const int sp = S + (S >> LOGP);
  auto at = [&](int j) -> V& { return lin ? p[j * sp] : buf[padx<LOGP>(base + j * S)]; };
  V v[R];
#pragma unroll
  for (int j = 0; j < R; ++j) v[j] = at(j);
  if constexpr (HAD) {
    wht_reg<R>(v);
  } else {
    // the DIT pass applies (F_R P_R) D; its transpose is D (P_R F_R), and
    // dft_reg computes F_R P_R, so F_R v = dft_reg(P_R v), then P_R again
    // (compile-time register renaming)
    {
      V t[R];
#pragma unroll
      for (int j = 0; j < R; ++j) t[j] = v[brev_small<R>(j)];
      dft_reg<R, INV>(t);
#pragma unroll
      for (int j = 0; j < R; ++j) v[j] = t[brev_small<R>(j)];
    }
    if (logS > 0) {
      const int step = o << (log2tab - logS - LOGR);
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
    }
  }
#pragma unroll
  for (int j = 0; j < R; ++j) at(j) = v[j];
}

// C vectors of length 2^L (stride `stride` apart, padded layout) transformed
// in place, natural order in, bit-reversed order out (Fourier; Hadamard is
// natural both ways); ends with a barrier
template <class V, bool INV, bool HAD, int C, class TW>
__device__ void multi_transform(V* buf, int stride, int L, int log2tab, const TW& tw, int tid,
                                int nth) {
  auto run = [&](auto rtag, int s) {
    constexpr int R = decltype(rtag)::value;
    constexpr int LOGR = log2_of<R>::v;
    const int nsub = 1 << (L - LOGR);
    for (int u = tid; u < C * nsub; u += nth) {
      const int v = u >> (L - LOGR);
      pass_dif<R, INV, HAD>(buf + v * stride, s, log2tab, tw, u & (nsub - 1));
    }
    __syncthreads();
  };
  constexpr int LOGF = log2_of<FS_R>::v;
  // the DIT schedule is full passes at s = 0, LOGF, ... then a remainder on
  // top; the DIF runs it backwards
  const int full = L / LOGF, rem = L - full * LOGF;
  switch (rem) {
    case 1: run(std::integral_constant<int, 2>{}, full * LOGF); break;
    case 2: run(std::integral_constant<int, 4>{}, full * LOGF); break;
    case 3: if constexpr (FS_R > 8) run(std::integral_constant<int, 8>{}, full * LOGF); break;
    default: break;
  }
  for (int p = full - 1; p >= 0; --p) run(std::integral_constant<int, FS_R>{}, p * LOGF);
}

struct FsArgs {
  DevOp op;
  int L1, L2;          // N1 = 2^L1 rows, N2 = 2^L2 columns
  int64_t batch;
  // pass A input: mode 0 dense (batch x n), 1 Omega (batch x m, list A),
  // 2 sparse (cnt entries (lam, xs) of ONE vector)
  int in_mode;
  const void* in;
  const uint32_t* lam;
  const double2* xs;
  int cnt;
  void* mid;           // batch x n
  // pass B output: mode 0 dense (batch x n), 1 Omega gather (batch x m, list B)
  int out_mode;
  void* out;
  int tw_smem;         // two-level twiddles staged in smem (else the global table)
};

template <class V>
struct TwSel {  // the staged two-level table, or the global one
  TwTwoLevel<V> s;
  TwTable<V> g;
  bool sm;
  __device__ __forceinline__ V operator()(int k) const { return sm ? s(k) : g(k); }
};

template <class V, bool HAD>
__device__ __forceinline__ V load_cast(const double2& x) {
  V v;
  from_c128(x, v);
  return v;
}

// stage lo[k] = W^k (k < 2^a) and hi[k] = W^(k 2^a) in smem
template <class V>
__device__ TwTwoLevel<V> stage_twiddles(unsigned char* p, const DevOp& op, int a, int tid,
                                        int nth) {
  V* lo = reinterpret_cast<V*>(p);
  V* hi = lo + TwTwoLevel<V>::pad(1 << a) + 1;
  const V* full = twiddles<V>(op);
  for (int k = tid; k < (1 << a); k += nth) lo[TwTwoLevel<V>::pad(k)] = full[k];
  for (int k = tid; k < (int)(op.n >> a); k += nth) hi[TwTwoLevel<V>::pad(k)] = full[(int64_t)k << a];
  return TwTwoLevel<V>{lo, hi, a};
}

template <class V, bool INV, bool HAD, int C>
__global__ void __launch_bounds__(FS_THREADS, 1) k_fs_a(FsArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const DevOp& op = a.op;
  const int L1 = a.L1, L2 = a.L2, L = L1 + L2;
  const int N1 = 1 << L1, N2 = 1 << L2;
  const int64_t n = op.n;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int stride = N1 + (N1 >> LOGP) + FS_SKEW;  // columns of a row in different banks
  V* buf = reinterpret_cast<V*>(sm);
  TwSel<V> tw{};
  if constexpr (!HAD) {
    tw.sm = a.tw_smem != 0;
    tw.g = TwTable<V>{twiddles<V>(op)};
    if (tw.sm)
      tw.s = stage_twiddles<V>(sm + ((sizeof(V) * (size_t)C * stride + 15) / 16) * 16, op,
                               min(L1, L2), tid, nth);
  }
  const V zv = zero_of(V{});
  const int tiles = N2 / C;
  const V* in = reinterpret_cast<const V*>(a.in);
  V* mid = reinterpret_cast<V*>(a.mid);
  for (int64_t tile = blockIdx.x; tile < a.batch * tiles; tile += gridDim.x) {
    const int64_t b = tile / tiles;
    const int c0 = (int)(tile - b * tiles) * C;
    auto slot = [&](int n1) { return padx<LOGP>(n1); };  // natural order (DIF)
    if (a.in_mode == 0) {
      // FS_U independent loads in flight per thread before the smem stores
      for (int e0 = tid; e0 < N1 * C; e0 += nth * FS_U) {
        V v[FS_U];
#pragma unroll
        for (int u = 0; u < FS_U; ++u) {
          const int e = e0 + u * nth;
          if (e < N1 * C) {
            const int n1 = e / C, c = e - n1 * C;
            v[u] = in[b * n + ((int64_t)n1 << L2) + c0 + c];
          }
        }
#pragma unroll
        for (int u = 0; u < FS_U; ++u) {
          const int e = e0 + u * nth;
          if (e < N1 * C) {
            const int n1 = e / C, c = e - n1 * C;
            buf[c * stride + slot(n1)] = v[u];
          }
        }
      }
    } else {
      for (int e = tid; e < C * stride; e += nth) buf[e] = zv;
      __syncthreads();
      if (a.in_mode == 1) {
        const uint32_t e0 = op.fs_aoff[c0], e1 = op.fs_aoff[c0 + C];
        for (uint32_t eb = e0 + tid; eb < e1; eb += nth * 4) {
          uint32_t pos[4];
          V v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t e = eb + u * nth;
            if (e < e1) {
              pos[u] = op.fs_apos[e];
              v[u] = in[b * op.m + op.fs_arow[e]];
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t e = eb + u * nth;
            if (e < e1) {
              const int n1 = (int)(pos[u] >> L2), c = (int)(pos[u] & (N2 - 1)) - c0;
              buf[c * stride + slot(n1)] = v[u];
            }
          }
        }
      } else {
        int placed = 0;
        for (int e = tid; e < a.cnt; e += nth) {
          const uint32_t pos = a.lam[e];
          if (pos == 0xffffffffu) continue;  // entry not in this transform (sharded solver)
          const int c = (int)(pos & (N2 - 1)) - c0;
          if (c >= 0 && c < C) {
            buf[c * stride + slot((int)(pos >> L2))] = load_cast<V, HAD>(a.xs[e]);
            placed = 1;
          }
        }
        // a sparse input (the current estimate, |support| << N2) leaves most
        // column tiles empty: their transform is zero, so store zeros and
        // skip the passes (the barrier of __syncthreads_or covers the fill)
        if (!__syncthreads_or(placed)) {
          for (int e = tid; e < N1 * C; e += nth) {
            const int q = e / C, c = e - q * C;
            mid[b * n + ((int64_t)q << L2) + c0 + c] = zv;
          }
          continue;
        }
      }
    }
    __syncthreads();
    multi_transform<V, INV, HAD, C>(buf, stride, L1, L, tw, tid, nth);
    if constexpr (HAD) {
      for (int e = tid; e < N1 * C; e += nth) {
        const int q = e / C, c = e - q * C;
        mid[b * n + ((int64_t)q << L2) + c0 + c] = buf[c * stride + padx<LOGP>(q)];
      }
    } else {
      // thread (q0, c): slots q = q0 + r 2^bq hold k1 = K0 + brev(r), K0 =
      // brev(q0); visiting r in bit-reversed order walks k1 = K0 + m, so the
      // inter-pass twiddle W_N^(n2 k1) is one lookup every 8 outputs and a
      // multiplication by W_N^n2 in between
      constexpr int QS = FS_THREADS / C;  // slots per round
      constexpr int BQ = log2_of<QS>::v;
      const int c = tid % C, q0 = tid / C;
      const int n2 = c0 + c;
      const int lr = L1 - BQ;  // log2 rounds
      const int K0 = (int)brev_n((unsigned)q0, L1);
      V wstep = tw(n2);
      if (INV) wstep.y = -wstep.y;
      V w = wstep;
      for (int mm = 0; mm < (1 << lr); ++mm) {
        const int r = (int)brev_n((unsigned)mm, lr);
        const int q = q0 + (r << BQ);
        const int k1 = K0 + mm;
        if ((mm & 7) == 0) {
          w = tw(n2 * k1);
          if (INV) w.y = -w.y;
        } else {
          w = cmul(w, wstep);
        }
        mid[b * n + ((int64_t)k1 << L2) + n2] = cmul(buf[c * stride + padx<LOGP>(q)], w);
      }
    }
    __syncthreads();
  }
}

template <class V, bool INV, bool HAD, int C>
__global__ void __launch_bounds__(FS_THREADS, 1) k_fs_b(FsArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const DevOp& op = a.op;
  const int L1 = a.L1, L2 = a.L2, L = L1 + L2;
  const int N1 = 1 << L1, N2 = 1 << L2;
  const int64_t n = op.n;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int stride = N2 + (N2 >> LOGP) + FS_SKEW;
  V* buf = reinterpret_cast<V*>(sm);
  TwSel<V> tw{};
  if constexpr (!HAD) {
    tw.sm = a.tw_smem != 0;
    tw.g = TwTable<V>{twiddles<V>(op)};
    if (tw.sm)
      tw.s = stage_twiddles<V>(sm + ((sizeof(V) * (size_t)C * stride + 15) / 16) * 16, op,
                               min(L1, L2), tid, nth);
  }
  const double sc = 1.0 / sqrt((double)n);
  const int tiles = N1 / C;
  const V* mid = reinterpret_cast<const V*>(a.mid);
  V* out = reinterpret_cast<V*>(a.out);
  for (int64_t tile = blockIdx.x; tile < a.batch * tiles; tile += gridDim.x) {
    const int64_t b = tile / tiles;
    const int r0 = (int)(tile - b * tiles) * C;
    for (int e0 = tid; e0 < C * N2; e0 += nth * FS_U) {
      V v[FS_U];
#pragma unroll
      for (int u = 0; u < FS_U; ++u) {
        const int e = e0 + u * nth;
        if (e < C * N2) v[u] = mid[b * n + ((int64_t)(r0 + (e >> L2)) << L2) + (e & (N2 - 1))];
      }
#pragma unroll
      for (int u = 0; u < FS_U; ++u) {
        const int e = e0 + u * nth;
        if (e < C * N2) {
          const int c = e >> L2, n2 = e & (N2 - 1);
          buf[c * stride + padx<LOGP>(n2)] = v[u];
        }
      }
    }
    __syncthreads();
    multi_transform<V, INV, HAD, C>(buf, stride, L2, L, tw, tid, nth);
    if (a.out_mode == 0) {
      if constexpr (HAD) {
        for (int e = tid; e < C * N2; e += nth) {
          const int c = e >> L2, k2 = e & (N2 - 1);
          out[b * n + ((int64_t)(r0 + c) << L2) + k2] = scale(buf[c * stride + padx<LOGP>(k2)], sc);
        }
      } else {
        for (int e = tid; e < C * N2; e += nth) {
          const int q = e / C, c = e - q * C;  // slot q holds k2 = brev(q)
          const int k2 = (int)brev_n((unsigned)q, L2);
          out[b * n + r0 + c + ((int64_t)k2 << L1)] = scale(buf[c * stride + padx<LOGP>(q)], sc);
        }
      }
    } else {
      const uint32_t e0 = op.fs_boff[r0], e1 = op.fs_boff[r0 + C];
      for (uint32_t e = e0 + tid; e < e1; e += nth) {
        const uint32_t pos = op.fs_bpos[e];
        int c, k2;
        if constexpr (HAD) {
          c = (int)(pos >> L2) - r0;
          k2 = (int)(pos & (N2 - 1));
        } else {
          c = (int)(pos & (N1 - 1)) - r0;
          k2 = (int)(pos >> L1);
        }
        const int q = HAD ? k2 : (int)brev_n((unsigned)k2, L2);
        out[b * op.m + op.fs_brow[e]] = scale(buf[c * stride + padx<LOGP>(q)], sc);
      }
    }
    __syncthreads();
  }
}

template <class V>
constexpr int fs_cols() { return 32 / (int)sizeof(V) < 2 ? 2 : 32 / (int)sizeof(V); }

template <class V, bool INV, bool HAD>
cudaError_t launch_fs(const FsTransform& t, cudaStream_t st) {
  constexpr int C = fs_cols<V>();
  const DevOp& op = *t.op;
  FsArgs a{};
  a.op = op;
  a.L1 = op.fs_l1;
  a.L2 = op.log2n - op.fs_l1;
  a.batch = t.batch;
  a.in_mode = t.in_mode;
  a.in = t.in;
  a.lam = t.lam;
  a.xs = t.xs;
  a.cnt = t.cnt;
  a.mid = t.mid;
  a.out_mode = t.out_mode;
  a.out = t.out;
  const int Lmax = a.L1 > a.L2 ? a.L1 : a.L2;
  const int amin = a.L1 < a.L2 ? a.L1 : a.L2;
  const size_t bufb =
      ((sizeof(V) * (size_t)C * ((1 << Lmax) + ((1 << Lmax) >> LOGP) + FS_SKEW) + 15) / 16) * 16;
  auto tpad = [](int i) { return i + (i >> 3); };  // TwTwoLevel::pad (device-only)
  const size_t twb = HAD ? 0
                         : sizeof(V) * (size_t)(tpad(1 << amin) + 1 + tpad(1 << (op.log2n - amin)) + 1);
  const size_t cap = (size_t)smem_optin() - 1024;
  if (bufb > cap) return cudaErrorInvalidConfiguration;
  a.tw_smem = !HAD && bufb + twb <= cap;
  const size_t smem = bufb + (a.tw_smem ? twb : 0);
  const int64_t tiles_a = t.batch * ((1 << a.L2) / C), tiles_b = t.batch * ((1 << a.L1) / C);
  if (t.in_mode == 2 && t.batch != 1) return cudaErrorInvalidValue;
  auto fa = k_fs_a<V, INV, HAD, C>;
  auto fb = k_fs_b<V, INV, HAD, C>;
  cudaFuncSetAttribute(fa, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(fb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  fa<<<(unsigned)std::min<int64_t>(tiles_a, num_sms()), FS_THREADS, smem, st>>>(a);
  fb<<<(unsigned)std::min<int64_t>(tiles_b, num_sms()), FS_THREADS, smem, st>>>(a);
  g_launches += 2;
  return cudaGetLastError();
}

template <class V, bool HAD>
cudaError_t launch_fs_v(const FsTransform& t, cudaStream_t st) {
  return t.inverse ? launch_fs<V, true, HAD>(t, st) : launch_fs<V, false, HAD>(t, st);
}

}  // namespace

// row split of the two-pass transform, or 0 when it does not apply
int fs_split(int log2n) {
  if (log2n < 18 || log2n > 24) return 0;
  return log2n / 2;  // N1 = 2^(L/2) rows, N2 = 2^(L - L/2) columns
}

cudaError_t launch_transform_fs(const FsTransform& t, cudaStream_t st) {
  g_launches = 0;
  if (!t.op->fs_l1 || !t.op->fs_aoff) return cudaErrorInvalidValue;
  const bool had = t.op->kind == HADAMARD;
  switch (t.dtype) {
    case C128: return had ? launch_fs_v<double2, true>(t, st) : launch_fs_v<double2, false>(t, st);
    case C64: return had ? launch_fs_v<float2, true>(t, st) : launch_fs_v<float2, false>(t, st);
    case F64: return had ? launch_fs_v<double, true>(t, st) : cudaErrorInvalidValue;
    case F32: return had ? launch_fs_v<float, true>(t, st) : cudaErrorInvalidValue;
  }
  return cudaErrorInvalidValue;
}

}  // namespace fmp
