// Kernels of the sharded single-signal solver (config 5: one N = 2^24 signal
// over the whole GPU, or P GPUs).  Shard p of P owns the correlation entries
// k = p + P k' (cyclic), so that
//   * the fast update of a shard reads the kernel class c = (p - lambda) mod P,
//     stored class-major (gcm[c][j'] = c[c + P j']), contiguously, and
//   * the band argmax reduces per shard to (best |h|^2) and (first index in
//     the band), exchanged between shards (solvers.cpp:90-101).
// Least squares is replicated on every shard with deterministic reductions,
// so all shards hold bit-identical coefficients.
#include "fmp_kcommon.cuh"

namespace fmp {
namespace {

constexpr int LG_THREADS = 256;
constexpr int LG_RPT = 4;
constexpr int LG_CHUNK = 1024;

// h[k'] = h0[k'] - sum_tau x_tau c[(p + P k' - lambda_tau) mod N] over this
// shard; per-CTA max |h|^2 into blkmax
template <class V>
__global__ void __launch_bounds__(LG_THREADS) k_lg_fast(const V* __restrict__ h0s, V* __restrict__ hs,
                                                        const V* __restrict__ gcm, int64_t np, int P,
                                                        int p, int64_t n, const uint32_t* __restrict__ lam,
                                                        const V* __restrict__ xn, int s,
                                                        double* __restrict__ blkmax) {
  __shared__ unsigned s_lam[LG_CHUNK];
  __shared__ V s_x[LG_CHUNK];
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t tile = (int64_t)32 * LG_RPT;
  const int64_t ntiles = (np + tile - 1) / tile;
  const int nwarps = LG_THREADS / 32;
  double best = 0.0;
  for (int64_t tb = (int64_t)blockIdx.x * nwarps; tb < ntiles; tb += (int64_t)gridDim.x * nwarps) {
    const int64_t t0 = tb + warp;
    const int64_t k0 = t0 * tile;
    V acc[LG_RPT];
#pragma unroll
    for (int r = 0; r < LG_RPT; ++r) {
      const int64_t k = k0 + lane + 32 * r;
      acc[r] = (t0 < ntiles && k < np) ? h0s[k] : zero_of(V{});
    }
    for (int c0 = 0; c0 < s; c0 += LG_CHUNK) {
      const int cn = min(LG_CHUNK, s - c0);
      __syncthreads();
      for (int j = tid; j < cn; j += LG_THREADS) {
        s_lam[j] = lam[c0 + j];
        s_x[j] = xn[c0 + j];
      }
      __syncthreads();
      if (t0 < ntiles) {
        for (int tau = 0; tau < cn; ++tau) {
          const int64_t d = ((int64_t)p + n - (int64_t)s_lam[tau]) % n;  // (p - lambda) mod N
          const int64_t cls = d % P, off = d / P;
          const V* g = gcm + cls * np;
          const V x = s_x[tau];
          int64_t j = k0 + lane + off;
          if (j >= np) j -= np;
#pragma unroll
          for (int r = 0; r < LG_RPT; ++r) {
            int64_t jj = j + 32 * r;
            if (jj >= np) jj -= np;
            msub(acc[r], x, __ldg(g + jj));
          }
        }
      }
    }
    if (t0 < ntiles) {
      double tm = 0.0;
#pragma unroll
      for (int r = 0; r < LG_RPT; ++r) {
        const int64_t k = k0 + lane + 32 * r;
        if (k < np) {
          hs[k] = acc[r];
          tm = fmax(tm, mag2(acc[r]));
        }
      }
      tm = warp_max(tm);
      if (lane == 0) blkmax[gridDim.x + t0] = tm;  // the tile's maximum (k_lg_first)
      best = fmax(best, tm);
    }
  }
  best = block_max(best, red);
  if (tid == 0) blkmax[blockIdx.x] = best;
}

// max |v|^2 of a strided view v[k'] = base[off + stride k'], k' < cnt: per
// tile of 32 LG_RPT positions into tilemax = blkmax + gridDim.x (the tiles
// of k_lg_fast), per CTA into blkmax
template <class V>
__global__ void __launch_bounds__(LG_THREADS) k_lg_max(const V* __restrict__ base, int64_t off,
                                                       int64_t stride, int64_t cnt,
                                                       double* __restrict__ blkmax) {
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = LG_THREADS / 32;
  const int64_t tile = 32 * LG_RPT, ntiles = (cnt + tile - 1) / tile;
  double best = 0.0;
  // TU tiles per warp per round, all loads issued before the reductions
  // (one tile at a time leaves each warp waiting on HBM latency per tile)
  constexpr int TU = 4;
  const int64_t step = (int64_t)gridDim.x * nwarps;
  for (int64_t t0 = (int64_t)blockIdx.x * nwarps + warp; t0 < ntiles; t0 += TU * step) {
    V v[TU][LG_RPT];
#pragma unroll
    for (int u = 0; u < TU; ++u)
#pragma unroll
      for (int r = 0; r < LG_RPT; ++r) {
        const int64_t k = (t0 + u * step) * tile + lane + 32 * r;
        v[u][r] = k < cnt ? base[off + stride * k] : zero_of(V{});
      }
#pragma unroll
    for (int u = 0; u < TU; ++u) {
      const int64_t t = t0 + u * step;
      double tm = 0.0;
#pragma unroll
      for (int r = 0; r < LG_RPT; ++r) tm = fmax(tm, mag2(v[u][r]));
      tm = warp_max(tm);
      if (t < ntiles) {
        if (lane == 0) blkmax[gridDim.x + t] = tm;
        best = fmax(best, tm);
      }
    }
  }
  best = block_max(best, red);
  if (threadIdx.x == 0) blkmax[blockIdx.x] = best;
}

__global__ void k_lg_reduce_max(const double* __restrict__ part, int cnt, double* __restrict__ out) {
  __shared__ double red[32];
  double b = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) b = fmax(b, part[i]);
  b = block_max(b, red);
  if (threadIdx.x == 0) *out = b;
}

// first index in the band: stage 1 finds the first tile whose maximum
// reaches the cut (every tile maximum is read once, in parallel; atomicMin),
// stage 2 the first position >= cut inside it.  A tile's maximum reaches the
// cut iff one of its entries does (same |v|^2 arithmetic), so the result is
// the smallest k' with |v|^2 >= cut.
// cut_best: the best |h|^2 on the device (one shard: no host round trip);
// same double arithmetic as the host's best * (1 - 1e-9)
__global__ void __launch_bounds__(LG_THREADS) k_lg_first_tile(const double* __restrict__ tilemax,
                                                              int64_t ntiles, double cut,
                                                              const double* __restrict__ cut_best,
                                                              unsigned long long* __restrict__ first_tile) {
  if (cut_best) cut = *cut_best * (1.0 - 1e-9);
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles;
       t += (int64_t)gridDim.x * blockDim.x)
    if (tilemax[t] >= cut) {
      atomicMin(first_tile, (unsigned long long)t);
      break;  // later t of this thread are larger
    }
}

template <class V>
__global__ void k_lg_first_elem(const V* __restrict__ base, int64_t off, int64_t stride, int64_t cnt,
                                double cut, const double* __restrict__ cut_best,
                                const unsigned long long* __restrict__ first_tile,
                                unsigned long long* __restrict__ first) {
  if (cut_best) cut = *cut_best * (1.0 - 1e-9);
  const unsigned long long t = *first_tile;
  if (t == ~0ull) return;
  const int64_t k = (int64_t)t * (32 * LG_RPT) + threadIdx.x;
  if (k < cnt && mag2(base[off + stride * k]) >= cut) atomicMin(first, (unsigned long long)k);
}

// the pick record [best, first (as a double, exact below 2^53), h0 re, h0 im]
template <class V>
__global__ void k_lg_pick(const double* __restrict__ best, const unsigned long long* __restrict__ first,
                          const V* __restrict__ h0s, double* __restrict__ rec) {
  const unsigned long long k = *first;
  rec[0] = *best;
  rec[1] = k == ~0ull ? -1.0 : (double)k;
  double2 h = make_double2(0.0, 0.0);
  if (k != ~0ull) h = to_c128(h0s[k]);
  rec[2] = h.x;
  rec[3] = h.y;
}

// ---- replicated least squares (same arithmetic as k_omp, deterministic)
struct LgLs {
  double2* W;        // column-major packed, capacity T
  double2* x;        // T
  double2* z;        // T
  double2* l;        // T
  uint32_t* lam;     // T, 0-based atoms
  void* xn;          // T (data dtype): -x for the fast update
  double* part;      // block partials (3 per block)
  double* scal;      // [0] gamma [1] yy [2] zz [3] d [4] znew.x [5] znew.y [6] aborted
  int T;
};

__device__ __forceinline__ int lg_wofs(int T, int i, int j) {
  return j * T - (j * (j - 1)) / 2 + (i - j);
}

template <bool HAD>
__device__ __forceinline__ double2 lg_gram(const DevOp& op, unsigned a, unsigned b) {
  if constexpr (HAD) return make_double2(op.gr64[a ^ b], 0.0);
  else return op.g64[(a - b) & (unsigned)(op.n - 1)];
}

// l = W a (a_j = G(lambda_j, pick)), one warp per row (lanes over j),
// per-block partials of |l|^2 and l^H z (fixed order: identical on every shard)
template <bool HAD>
__global__ void __launch_bounds__(LG_THREADS) k_lg_ls_a(DevOp op, LgLs L, int s, unsigned pick) {
  __shared__ double red[3][LG_THREADS / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * (LG_THREADS / 32) + w;
  double ll = 0.0, lzr = 0.0, lzi = 0.0;
  if (i < s) {
    double ar = 0.0, ai = 0.0;
    for (int j = lane; j <= i; j += 32) {
      const double2 wv = L.W[lg_wofs(L.T, i, j)], v = lg_gram<HAD>(op, L.lam[j], pick);
      ar = fma(wv.x, v.x, fma(-wv.y, v.y, ar));
      ai = fma(wv.x, v.y, fma(wv.y, v.x, ai));
    }
    ar = warp_sum(ar);
    ai = warp_sum(ai);
    if (lane == 0) {
      L.l[i] = make_double2(ar, ai);
      const double2 zc = L.z[i];
      ll = ar * ar + ai * ai;
      lzr = ar * zc.x + ai * zc.y;
      lzi = ar * zc.y - ai * zc.x;
    }
  }
  if (lane == 0) {
    red[0][w] = ll;
    red[1][w] = lzr;
    red[2][w] = lzi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (int q = 0; q < LG_THREADS / 32; ++q) {
      a += red[0][q];
      b += red[1][q];
      c += red[2][q];
    }
    L.part[3 * blockIdx.x] = a;
    L.part[3 * blockIdx.x + 1] = b;
    L.part[3 * blockIdx.x + 2] = c;
  }
}

// d, z_s (single thread, fixed order: identical on every shard)
__global__ void k_lg_ls_b(LgLs L, int nblk, double2 bnew) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double ll = 0.0, lzr = 0.0, lzi = 0.0;
  for (int b = 0; b < nblk; ++b) {
    ll += L.part[3 * b];
    lzr += L.part[3 * b + 1];
    lzi += L.part[3 * b + 2];
  }
  const double gamma = L.scal[0];
  const double d2 = gamma - ll;
  if (!(d2 > 1e-12 * gamma)) {  // solvers.cpp:32,144
    L.scal[6] = 1.0;
    return;
  }
  const double d = sqrt(d2);
  L.scal[3] = d;
  L.scal[4] = (bnew.x - lzr) / d;
  L.scal[5] = (bnew.y - lzi) / d;
  L.scal[6] = 0.0;
}

// new row of W and x = W^H z, one warp per column; appends the atom
template <class V>
__global__ void __launch_bounds__(LG_THREADS) k_lg_ls_c(LgLs L, int s, unsigned pick, double xscale) {
  const int lane = threadIdx.x & 31;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (L.scal[6] != 0.0) return;
  const double d = L.scal[3];
  const double2 znew = make_double2(L.scal[4], L.scal[5]);
  V* xn = reinterpret_cast<V*>(L.xn);
  if (j < s) {
    double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
    for (int i = j + lane; i < s; i += 32) {
      const double2 l = L.l[i], w = L.W[lg_wofs(L.T, i, j)], zc = L.z[i];
      ar += l.x * w.x + l.y * w.y;
      ai += l.x * w.y - l.y * w.x;
      br += w.x * zc.x + w.y * zc.y;
      bi += w.x * zc.y - w.y * zc.x;
    }
    ar = warp_sum(ar);
    ai = warp_sum(ai);
    br = warp_sum(br);
    bi = warp_sum(bi);
    if (lane == 0) {
      const double2 wn = make_double2(-ar / d, -ai / d);
      L.W[lg_wofs(L.T, s, j)] = wn;
      const double xr = br + wn.x * znew.x + wn.y * znew.y;
      const double xi = bi + wn.x * znew.y - wn.y * znew.x;
      L.x[j] = make_double2(xr, xi);
      from_c128(make_double2(xr * xscale, xi * xscale), xn[j]);
    }
  } else if (j == s && lane == 0) {
    L.W[lg_wofs(L.T, s, s)] = make_double2(1.0 / d, 0.0);
    L.z[s] = znew;
    L.lam[s] = pick;
    const double2 xs = make_double2(znew.x / d, znew.y / d);
    L.x[s] = xs;
    from_c128(make_double2(xs.x * xscale, xs.y * xscale), xn[s]);
    L.scal[2] += znew.x * znew.x + znew.y * znew.y;  // zz
  }
}

// dense sparse-estimate vector for the forward transform: out[lambda_j] = x_j
template <class V>
__global__ void k_lg_scatter_x(V* __restrict__ out, const uint32_t* __restrict__ lam,
                               const double2* __restrict__ x, int s) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < s) from_c128(x[j], out[lam[j]]);
}

// r = y - Phi x (Phi x given at the rows), per-block partial ||r||^2
template <class V>
__global__ void __launch_bounds__(LG_THREADS) k_lg_resid(const V* __restrict__ y,
                                                         const V* __restrict__ ax, V* __restrict__ r,
                                                         int64_t m, double* __restrict__ part) {
  __shared__ double red[32];
  double r2 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const V v = sub(y[i], ax[i]);
    r[i] = v;
    r2 += mag2(v);
  }
  r2 = block_sum(r2, red);
  if (threadIdx.x == 0) part[blockIdx.x] = r2;
}

// one block, fixed order (strided per-thread sums, then the shuffle tree):
// identical on every shard
__global__ void k_lg_sum(const double* __restrict__ part, int cnt, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) s += part[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

// shard view of a full vector: dst[k'] = src[p + P k']
template <class V>
__global__ void k_lg_take(const V* __restrict__ src, V* __restrict__ dst, int64_t np, int P, int p) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < np;
       k += (int64_t)gridDim.x * blockDim.x)
    dst[k] = src[p + (int64_t)P * k];
}

// class-major kernel: gcm[c][j'] = c[c + P j']
template <class V>
__global__ void k_lg_classmajor(const V* __restrict__ g, V* __restrict__ gcm, int64_t n, int P) {
  const int64_t np = n / P;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / np, j = i - c * np;
    gcm[i] = g[c + (int64_t)P * j];
  }
}

}  // namespace

int lg_grid() { return num_sms() * 4; }

cudaError_t lg_launch_fast(int dtype, const void* h0s, void* hs, const void* gcm, int64_t np, int P,
                           int p, int64_t n, const uint32_t* lam, const void* xn, int s,
                           double* blkmax, cudaStream_t st) {
  const int grid = lg_grid();
  if (dtype == C128)
    k_lg_fast<double2><<<grid, LG_THREADS, 0, st>>>((const double2*)h0s, (double2*)hs, (const double2*)gcm,
                                                    np, P, p, n, lam, (const double2*)xn, s, blkmax);
  else
    k_lg_fast<float2><<<grid, LG_THREADS, 0, st>>>((const float2*)h0s, (float2*)hs, (const float2*)gcm,
                                                   np, P, p, n, lam, (const float2*)xn, s, blkmax);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_launch_max(int dtype, const void* base, int64_t off, int64_t stride, int64_t cnt,
                          double* blkmax, double* out, cudaStream_t st) {
  const int grid = lg_grid();
  if (dtype == C128)
    k_lg_max<double2><<<grid, LG_THREADS, 0, st>>>((const double2*)base, off, stride, cnt, blkmax);
  else
    k_lg_max<float2><<<grid, LG_THREADS, 0, st>>>((const float2*)base, off, stride, cnt, blkmax);
  k_lg_reduce_max<<<1, 1024, 0, st>>>(blkmax, grid, out);
  g_launches += 2;
  return cudaGetLastError();
}

cudaError_t lg_launch_reduce_max(double* blkmax, double* out, cudaStream_t st) {
  k_lg_reduce_max<<<1, 1024, 0, st>>>(blkmax, lg_grid(), out);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_launch_first(int dtype, const void* base, int64_t off, int64_t stride, int64_t cnt,
                            double cut, const double* cut_best, const double* blkmax,
                            unsigned long long* first, cudaStream_t st) {
  // blkmax: the per-CTA maxima followed by the tile maxima of the last
  // k_lg_max / k_lg_fast over this view; first[1] is scratch for the tile
  const int grid = lg_grid();
  const int64_t ntiles = (cnt + 32 * LG_RPT - 1) / (32 * LG_RPT);
  cudaMemsetAsync(first, 0xff, 16, st);
  k_lg_first_tile<<<(unsigned)std::min<int64_t>(grid, (ntiles + LG_THREADS - 1) / LG_THREADS), LG_THREADS, 0,
                    st>>>(blkmax + grid, ntiles, cut, cut_best, first + 1);
  if (dtype == C128)
    k_lg_first_elem<double2><<<1, 32 * LG_RPT, 0, st>>>((const double2*)base, off, stride, cnt, cut,
                                                       cut_best, first + 1, first);
  else
    k_lg_first_elem<float2><<<1, 32 * LG_RPT, 0, st>>>((const float2*)base, off, stride, cnt, cut,
                                                      cut_best, first + 1, first);
  g_launches += 2;
  return cudaGetLastError();
}

cudaError_t lg_launch_ls(int dtype, const DevOp& op, double2* W, double2* x, double2* z, double2* l,
                         uint32_t* lam, void* xn, double* part, double* scal, int T, int s,
                         unsigned pick, double2 bnew, cudaStream_t st) {
  LgLs L{W, x, z, l, lam, xn, part, scal, T};
  const int nblk = std::max(1, (s + LG_THREADS / 32 - 1) / (LG_THREADS / 32));
  if (op.kind == HADAMARD) k_lg_ls_a<true><<<nblk, LG_THREADS, 0, st>>>(op, L, s, pick);
  else k_lg_ls_a<false><<<nblk, LG_THREADS, 0, st>>>(op, L, s, pick);
  k_lg_ls_b<<<1, 32, 0, st>>>(L, nblk, bnew);
  const int warps = s + 1, cblk = (warps * 32 + LG_THREADS - 1) / LG_THREADS;
  const double xscale = op.kind == HADAMARD ? -1.0 / (double)op.n : -1.0;
  if (dtype == C128) k_lg_ls_c<double2><<<cblk, LG_THREADS, 0, st>>>(L, s, pick, xscale);
  else k_lg_ls_c<float2><<<cblk, LG_THREADS, 0, st>>>(L, s, pick, xscale);
  g_launches += 3;
  return cudaGetLastError();
}

cudaError_t lg_launch_pick(int dtype, const double* best, const unsigned long long* first,
                           const void* h0s, double* rec, cudaStream_t st) {
  if (dtype == C128) k_lg_pick<double2><<<1, 1, 0, st>>>(best, first, (const double2*)h0s, rec);
  else k_lg_pick<float2><<<1, 1, 0, st>>>(best, first, (const float2*)h0s, rec);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_launch_scatter_x(int dtype, void* out, const uint32_t* lam, const double2* x, int s,
                                cudaStream_t st) {
  const int blocks = std::max(1, (s + 255) / 256);
  if (dtype == C128) k_lg_scatter_x<double2><<<blocks, 256, 0, st>>>((double2*)out, lam, x, s);
  else k_lg_scatter_x<float2><<<blocks, 256, 0, st>>>((float2*)out, lam, x, s);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_launch_resid(int dtype, const void* y, const void* ax, void* r, int64_t m,
                            double* part, double* out, cudaStream_t st) {
  const int grid = lg_grid();
  if (dtype == C128)
    k_lg_resid<double2><<<grid, LG_THREADS, 0, st>>>((const double2*)y, (const double2*)ax, (double2*)r, m, part);
  else
    k_lg_resid<float2><<<grid, LG_THREADS, 0, st>>>((const float2*)y, (const float2*)ax, (float2*)r, m, part);
  k_lg_sum<<<1, 256, 0, st>>>(part, grid, out);
  g_launches += 2;
  return cudaGetLastError();
}

cudaError_t lg_launch_sum(const double* part, int cnt, double* out, cudaStream_t st) {
  k_lg_sum<<<1, 256, 0, st>>>(part, cnt, out);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_launch_take(int dtype, const void* src, void* dst, int64_t np, int P, int p,
                           cudaStream_t st) {
  const int grid = lg_grid();
  if (dtype == C128) k_lg_take<double2><<<grid, 256, 0, st>>>((const double2*)src, (double2*)dst, np, P, p);
  else k_lg_take<float2><<<grid, 256, 0, st>>>((const float2*)src, (float2*)dst, np, P, p);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_launch_classmajor(int dtype, const void* g, void* gcm, int64_t n, int P,
                                 cudaStream_t st) {
  const int grid = lg_grid();
  if (dtype == C128) k_lg_classmajor<double2><<<grid, 256, 0, st>>>((const double2*)g, (double2*)gcm, n, P);
  else k_lg_classmajor<float2><<<grid, 256, 0, st>>>((const float2*)g, (float2*)gcm, n, P);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace fmp
