// Kernels of the sharded single-signal solver (config 5: one N = 2^24 signal
// over one GPU or P GPUs).  Shard p of P owns the correlation entries
// k = p + P k' (cyclic), k' < np = N / P, so that
//   * the fast update of a shard reads the kernel class c = (p - lambda) mod P,
//     stored class-major (gcm[c][j'] = c[c + P j']), contiguously;
//   * the conventional row of a shard is an np-point transform: the residual
//     folded into np bins (z[j] = sum over rows with omega = j mod np of
//     r_m W_N^(-omega_m p)), so no shard transforms all N entries;
//   * the residual r = y - Phi x is a sum over shards of np-point forward
//     transforms of each shard's atoms (one all-reduce of the M-vector).
// Identification follows the reference's band rule (solvers.cpp:90-101) on
// fp64 values: every shard lists the entries whose working-precision |h|
// lies within twice the rounding bound of its maximum, re-evaluates them as
// h_j = h0_j - sum_tau x_tau c[(j - lambda_tau) mod N] in fp64 from the
// replicated fp64 h0 and kernel (kernel.cpp:246-261), and the records of all
// shards are merged identically everywhere: the maximum fp64 |h|^2 and the
// smallest index within 1e-9 of it.  These values do not depend on P or on
// the transforms, so picks and coefficients are bitwise the same for every
// shard count.  Least squares is replicated with deterministic reductions.
#include "fmp_kcommon.cuh"

namespace fmp {
namespace {

constexpr int LG_THREADS = 256;
constexpr int LG_RPT = 4;
constexpr int LG_TILE = 32 * LG_RPT;
constexpr int LG_CHUNK = 1024;

__device__ __forceinline__ bool prev_flagged(const LgShard& S, int prev) {
  return prev >= 0 && S.pick[prev].flags != 0;
}

// h[k'] = h0[k'] - sum_tau x_tau c[(p + P k' - lambda_tau) mod N] over this
// shard; per-tile and per-CTA maxima of |h|^2 into blkmax
template <class V>
__global__ void __launch_bounds__(LG_THREADS) k_lg_fast(LgShard S, int s) {
  __shared__ unsigned s_cls[LG_CHUNK];
  __shared__ unsigned s_off[LG_CHUNK];
  __shared__ V s_x[LG_CHUNK];
  __shared__ double red[32];
  const V* __restrict__ h0s = reinterpret_cast<const V*>(S.h0s);
  V* __restrict__ hs = reinterpret_cast<V*>(S.hs);
  const V* __restrict__ gcm = reinterpret_cast<const V*>(S.gcm);
  const V* __restrict__ xn = reinterpret_cast<const V*>(S.xn);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned np = (unsigned)S.np, nmask = (unsigned)S.n - 1u, pmask = (unsigned)S.P - 1u;
  const unsigned ntiles = (np + LG_TILE - 1) / LG_TILE;
  const int nwarps = LG_THREADS / 32;
  double best = 0.0;
  for (unsigned tb = blockIdx.x * nwarps; tb < ntiles; tb += gridDim.x * nwarps) {
    const unsigned t0 = tb + warp;
    const unsigned k0 = t0 * LG_TILE;
    V acc[LG_RPT];
#pragma unroll
    for (int r = 0; r < LG_RPT; ++r) {
      const unsigned k = k0 + lane + 32 * r;
      acc[r] = (t0 < ntiles && k < np) ? h0s[k] : zero_of(V{});
    }
    for (int c0 = 0; c0 < s; c0 += LG_CHUNK) {
      const int cn = min(LG_CHUNK, s - c0);
      __syncthreads();
      // per atom: source class and offset of (p - lambda) mod N, once per CTA
      for (int j = tid; j < cn; j += LG_THREADS) {
        const unsigned d = ((unsigned)S.p - S.lam[c0 + j]) & nmask;
        s_cls[j] = d & pmask;
        s_off[j] = d >> S.log2P;
        s_x[j] = xn[c0 + j];
      }
      __syncthreads();
      if (t0 < ntiles) {
        for (int tau = 0; tau < cn; ++tau) {
          const V* g = gcm + (size_t)s_cls[tau] * np;
          const V x = s_x[tau];
          const unsigned j = k0 + lane + s_off[tau];
#pragma unroll
          for (int r = 0; r < LG_RPT; ++r) msub(acc[r], x, __ldg(g + ((j + 32 * r) & (np - 1))));
        }
      }
    }
    if (t0 < ntiles) {
      double tm = 0.0;
#pragma unroll
      for (int r = 0; r < LG_RPT; ++r) {
        const unsigned k = k0 + lane + 32 * r;
        if (k < np) {
          hs[k] = acc[r];
          tm = fmax(tm, mag2(acc[r]));
        }
      }
      tm = warp_max(tm);
      if (lane == 0) S.blkmax[gridDim.x + t0] = tm;  // the tile's maximum
      best = fmax(best, tm);
    }
  }
  best = block_max(best, red);
  if (tid == 0) S.blkmax[blockIdx.x] = best;
}

// per-tile (128 positions) and per-CTA maxima of |h|^2 over np entries
template <class V>
__global__ void __launch_bounds__(LG_THREADS) k_lg_max(const V* __restrict__ h, int64_t cnt,
                                                       double* __restrict__ blkmax) {
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = LG_THREADS / 32;
  const int64_t ntiles = (cnt + LG_TILE - 1) / LG_TILE;
  double best = 0.0;
  // TU tiles per warp per round, all loads issued before the reductions
  constexpr int TU = 4;
  const int64_t step = (int64_t)gridDim.x * nwarps;
  for (int64_t t0 = (int64_t)blockIdx.x * nwarps + warp; t0 < ntiles; t0 += TU * step) {
    V v[TU][LG_RPT];
#pragma unroll
    for (int u = 0; u < TU; ++u)
#pragma unroll
      for (int r = 0; r < LG_RPT; ++r) {
        const int64_t k = (t0 + u * step) * LG_TILE + lane + 32 * r;
        v[u][r] = k < cnt ? h[k] : zero_of(V{});
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

__global__ void k_lg_best(const double* __restrict__ blkmax, int cnt, LgRec* __restrict__ rec) {
  __shared__ double red[32];
  double b = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) b = fmax(b, blkmax[i]);
  b = block_max(b, red);
  if (threadIdx.x == 0) rec->best32 = b;
}

// candidates: entries whose |h| is within 2E of this shard's maximum, E the
// working-precision rounding bound ecoef (hy + goff sum|x| + gamma max|x|)
// (ecoef a multiple of 2^-24 or 2^-53 per transform level).  Only a tile
// whose maximum reaches the cut is scanned.
template <class V>
__global__ void __launch_bounds__(LG_THREADS) k_lg_cands(LgShard S, const V* __restrict__ h,
                                                         double ecoef, int prev, int grid) {
  if (prev_flagged(S, prev)) return;
  const double best = S.rec_send->best32;
  if (best == 0.0) return;  // nothing here can reach a non-zero band
  const double e = ecoef * (S.scal[10] + S.op.goff * S.scal[7] + S.scal[0] * S.scal[8]);
  const double lo = sqrt(best) * (1.0 - kTieBandRel) - 2.0 * e;
  const double cut = lo > 0.0 ? lo * lo : -1.0;
  const int64_t ntiles = (S.np + LG_TILE - 1) / LG_TILE;
  const double* tilemax = S.blkmax + grid;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (!(tilemax[t] >= cut)) continue;
    const int64_t k1 = S.np < (t + 1) * LG_TILE ? S.np : (t + 1) * LG_TILE;
    for (int64_t k = t * LG_TILE; k < k1; ++k)
      if (mag2(h[k]) >= cut) {
        const unsigned c = atomicAdd(S.ccount, 1u);
        if (c < (unsigned)LG_LCAP) S.cand[c] = (uint32_t)k;
      }
  }
}

// the candidate count of an identification; kept when the previous pick is
// flagged, so that its candidates survive for the exact fallback
__global__ void k_lg_reset(LgShard S, int prev) {
  if (!prev_flagged(S, prev)) *S.ccount = 0u;
}

// fp64 correlation of each candidate, one CTA per candidate (fixed-order
// reduction: the value depends only on the candidate, not on P)
__global__ void __launch_bounds__(LG_THREADS) k_lg_eval(LgShard S, int s, int prev) {
  __shared__ double red[2][LG_THREADS / 32];
  if (prev_flagged(S, prev)) return;
  const unsigned cnt = min(*S.ccount, (unsigned)LG_LCAP);
  const unsigned nmask = (unsigned)S.n - 1u;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (unsigned c = blockIdx.x; c < cnt; c += gridDim.x) {
    const unsigned j = (unsigned)S.p + ((unsigned)S.cand[c] << S.log2P);
    double ar = 0.0, ai = 0.0;
    for (int q = threadIdx.x; q < s; q += LG_THREADS) {
      const double2 xv = S.x[q];
      const double2 g = S.op.g64[(j - S.lam[q]) & nmask];
      ar = fma(xv.x, g.x, fma(-xv.y, g.y, ar));
      ai = fma(xv.x, g.y, fma(xv.y, g.x, ai));
    }
    ar = warp_sum(ar);
    ai = warp_sum(ai);
    if (lane == 0) {
      red[0][w] = ar;
      red[1][w] = ai;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double sr = 0.0, si = 0.0;
      for (int q = 0; q < LG_THREADS / 32; ++q) {
        sr += red[0][q];
        si += red[1][q];
      }
      const double2 h0 = S.h0x[j];
      const double hr = h0.x - sr, hi = h0.y - si;
      S.cval[c] = hr * hr + hi * hi;
    }
    __syncthreads();
  }
}

__global__ void k_lg_record(LgShard S, int prev) {
  if (prev_flagged(S, prev)) return;
  const unsigned cnt = *S.ccount;
  if (threadIdx.x == 0) S.rec_send->count = cnt;
  for (unsigned c = threadIdx.x; c < min(cnt, (unsigned)LG_RC); c += blockDim.x) {
    LgCand e;
    e.j = (uint64_t)S.p + ((uint64_t)S.cand[c] << S.log2P);
    e.m64 = S.cval[c];
    S.rec_send->c[c] = e;
  }
}

// the band rule over the gathered records (host twin: lg_merge_host)
__host__ __device__ inline void merge_records(const LgRec* recs, int P, const uint32_t* selbits,
                                              LgPick* out) {
  LgPick pk{};
  pk.j = ~0ull;
  for (int q = 0; q < P; ++q) {
    if (recs[q].count > (uint32_t)LG_LCAP) pk.flags |= LG_TOOMANY;
    if (recs[q].count > (uint32_t)LG_RC) pk.flags |= LG_OVERFLOW;
  }
  if (pk.flags) {
    *out = pk;
    return;
  }
  double best = 0.0;
  for (int q = 0; q < P; ++q)
    for (uint32_t c = 0; c < recs[q].count; ++c) best = best > recs[q].c[c].m64 ? best : recs[q].c[c].m64;
  pk.best64 = best;
  if (best == 0.0) {
    pk.flags = LG_ZERO;
    *out = pk;
    return;
  }
  const double cut = best * (1.0 - kTieBandRel);
  for (int q = 0; q < P; ++q)
    for (uint32_t c = 0; c < recs[q].count; ++c)
      if (recs[q].c[c].m64 >= cut && recs[q].c[c].j < pk.j) pk.j = recs[q].c[c].j;
  if (selbits && ((selbits[pk.j >> 5] >> (pk.j & 31)) & 1u)) pk.flags = LG_STAGNANT;
  *out = pk;
}

__global__ void k_lg_merge(LgShard S, int cur, int prev) {
  if (prev_flagged(S, prev)) return;
  LgPick pk;
  merge_records(S.rec_all, S.P, S.selbits, &pk);
  if (!pk.flags) pk.b = S.h0x[pk.j];
  S.pick[cur] = pk;
}

// ---- fallback after an overflowing record: exact maximum and first in band
__global__ void k_lg_fb_best(LgShard S) {
  __shared__ double red[32];
  const unsigned cnt = min(*S.ccount, (unsigned)LG_LCAP);
  double b = 0.0;
  for (unsigned c = threadIdx.x; c < cnt; c += blockDim.x) b = fmax(b, S.cval[c]);
  b = block_max(b, red);
  if (threadIdx.x == 0) S.fb[0] = b;
}

__global__ void k_lg_fb_first(LgShard S) {
  __shared__ unsigned long long red[32];
  const unsigned cnt = min(*S.ccount, (unsigned)LG_LCAP);
  const double cut = S.fb[1] * (1.0 - kTieBandRel);
  unsigned long long f = ~0ull;
  for (unsigned c = threadIdx.x; c < cnt; c += blockDim.x)
    if (S.cval[c] >= cut) f = min(f, (unsigned long long)S.p + ((unsigned long long)S.cand[c] << S.log2P));
#pragma unroll
  for (int o = 16; o; o >>= 1) f = min(f, __shfl_xor_sync(0xffffffffu, f, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = f;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) f = min(f, red[w]);
    f = min(f, red[0]);
    reinterpret_cast<unsigned long long*>(S.fb)[2] = f;
  }
}

__global__ void k_lg_fb_pick(LgShard S, int cur) {
  LgPick pk{};
  pk.best64 = S.fb[1];
  pk.j = reinterpret_cast<const unsigned long long*>(S.fb)[3];
  if (pk.best64 == 0.0 || pk.j == ~0ull) pk.flags = LG_ZERO;
  else if ((S.selbits[pk.j >> 5] >> (pk.j & 31)) & 1u) pk.flags = LG_STAGNANT;
  else pk.b = S.h0x[pk.j];
  S.pick[cur] = pk;
}

// ---- replicated least squares (the fused solver's arithmetic, k_omp)
__device__ __forceinline__ int lg_wofs(int T, int i, int j) {
  return j * T - (j * (j - 1)) / 2 + (i - j);
}

// l = W a (a_j = G(lambda_j, pick)), one warp per row (lanes over j),
// per-block partials of |l|^2 and l^H z (fixed order: identical on every shard)
__global__ void __launch_bounds__(LG_THREADS) k_lg_ls_a(LgShard S, int s, int cur) {
  __shared__ double red[3][LG_THREADS / 32];
  if (S.pick[cur].flags) return;
  const unsigned pick = (unsigned)S.pick[cur].j, nmask = (unsigned)S.n - 1u;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * (LG_THREADS / 32) + w;
  double ll = 0.0, lzr = 0.0, lzi = 0.0;
  if (i < s) {
    double ar = 0.0, ai = 0.0;
    for (int j = lane; j <= i; j += 32) {
      const double2 wv = S.W[lg_wofs(S.T, i, j)], v = S.op.g64[(S.lam[j] - pick) & nmask];
      ar = fma(wv.x, v.x, fma(-wv.y, v.y, ar));
      ai = fma(wv.x, v.y, fma(wv.y, v.x, ai));
    }
    ar = warp_sum(ar);
    ai = warp_sum(ai);
    if (lane == 0) {
      S.l[i] = make_double2(ar, ai);
      const double2 zc = S.z[i];
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
    S.part[3 * blockIdx.x] = a;
    S.part[3 * blockIdx.x + 1] = b;
    S.part[3 * blockIdx.x + 2] = c;
  }
}

// d, z_s (single thread, fixed order)
__global__ void k_lg_ls_b(LgShard S, int nblk, int cur) {
  if (threadIdx.x != 0 || blockIdx.x != 0 || S.pick[cur].flags) return;
  double ll = 0.0, lzr = 0.0, lzi = 0.0;
  for (int b = 0; b < nblk; ++b) {
    ll += S.part[3 * b];
    lzr += S.part[3 * b + 1];
    lzi += S.part[3 * b + 2];
  }
  const double gamma = S.scal[0];
  const double d2 = gamma - ll;
  if (!(d2 > 1e-12 * gamma)) {  // solvers.cpp:32,144
    S.scal[6] = 1.0;
    return;
  }
  const double2 bnew = S.pick[cur].b;
  const double d = sqrt(d2);
  S.scal[3] = d;
  S.scal[4] = (bnew.x - lzr) / d;
  S.scal[5] = (bnew.y - lzi) / d;
}

// new row of W and x = W^H z, one warp per column; appends the atom
template <class V>
__global__ void __launch_bounds__(LG_THREADS) k_lg_ls_c(LgShard S, int s, int cur, double xscale) {
  if (S.pick[cur].flags || S.scal[6] != 0.0) return;
  const int lane = threadIdx.x & 31;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const double d = S.scal[3];
  const double2 znew = make_double2(S.scal[4], S.scal[5]);
  V* xn = reinterpret_cast<V*>(S.xn);
  if (j < s) {
    double ar = 0.0, ai = 0.0, br = 0.0, bi = 0.0;
    for (int i = j + lane; i < s; i += 32) {
      const double2 l = S.l[i], w = S.W[lg_wofs(S.T, i, j)], zc = S.z[i];
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
      S.W[lg_wofs(S.T, s, j)] = wn;
      const double xr = br + wn.x * znew.x + wn.y * znew.y;
      const double xi = bi + wn.x * znew.y - wn.y * znew.x;
      S.x[j] = make_double2(xr, xi);
      from_c128(make_double2(xr * xscale, xi * xscale), xn[j]);
    }
  } else if (j == s && lane == 0) {
    const unsigned pick = (unsigned)S.pick[cur].j;
    S.W[lg_wofs(S.T, s, s)] = make_double2(1.0 / d, 0.0);
    S.z[s] = znew;
    S.lam[s] = pick;
    atomicOr(S.selbits + (pick >> 5), 1u << (pick & 31));
    const double2 xs = make_double2(znew.x / d, znew.y / d);
    S.x[s] = xs;
    from_c128(make_double2(xs.x * xscale, xs.y * xscale), xn[s]);
    S.scal[2] += znew.x * znew.x + znew.y * znew.y;  // zz
  }
}

// sum |x| and max |x| over the s + 1 coefficients (the next rounding bound)
__global__ void k_lg_xstats(LgShard S, int cnt, int cur) {
  __shared__ double red[32];
  if (S.pick[cur].flags || S.scal[6] != 0.0) return;
  double a = 0.0, mx = 0.0;
  for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
    const double2 v = S.x[j];
    const double m = sqrt(v.x * v.x + v.y * v.y);
    a += m;
    mx = fmax(mx, m);
  }
  a = block_sum(a, red);
  mx = block_max(mx, red);
  if (threadIdx.x == 0) {
    S.scal[7] = a;
    S.scal[8] = mx;
  }
}

// ---- residual
__global__ void k_lg_class_pos(LgShard S, int cnt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= cnt) return;
  const unsigned l = S.lam[j];
  S.lamc[j] = (int)(l & (unsigned)(S.P - 1)) == S.p ? l >> S.log2P : 0xffffffffu;
}

template <class V>
__global__ void k_lg_scatter(LgShard S, V* __restrict__ out, int cnt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < cnt && S.lamc[j] != 0xffffffffu) from_c128(S.x[j], out[S.lamc[j]]);
}

template <class V> __device__ __forceinline__ V tw_at(const DevOp& op, unsigned k);
template <> __device__ __forceinline__ double2 tw_at<double2>(const DevOp& op, unsigned k) { return op.tw64[k]; }
template <> __device__ __forceinline__ float2 tw_at<float2>(const DevOp& op, unsigned k) { return op.tw32[k]; }

// this shard's part of Phi x at every row: X_p[omega mod np] W_N^(omega p) / sqrt(P)
template <class V>
__global__ void k_lg_partial(LgShard S, const V* __restrict__ X, V* __restrict__ out) {
  const double isp = 1.0 / sqrt((double)S.P);
  const unsigned nmask = (unsigned)S.n - 1u, npm = (unsigned)S.np - 1u;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < S.m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned w = S.op.omega[i];
    out[i] = scale(cmul(X[w & npm], tw_at<V>(S.op, (w * (unsigned)S.p) & nmask)), isp);
  }
}

// r = y - ax (stored when r != null), per-block partial ||r||^2
template <class V>
__global__ void __launch_bounds__(LG_THREADS) k_lg_resid(const V* __restrict__ y, const V* __restrict__ ax,
                                                         V* __restrict__ r, int64_t m, double* __restrict__ part) {
  __shared__ double red[32];
  double r2 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const V v = sub(y[i], ax[i]);
    if (r) r[i] = v;
    r2 += mag2(v);
  }
  r2 = block_sum(r2, red);
  if (threadIdx.x == 0) part[blockIdx.x] = r2;
}

// one block, fixed order: identical on every shard
__global__ void k_lg_sum(const double* __restrict__ part, int cnt, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) s += part[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

// z[j] = (1 / sqrt(P)) sum over rows with omega = j mod np of r_m conj(W_N^(omega p))
template <class V>
__global__ void k_lg_fold(LgShard S) {
  const V* r = reinterpret_cast<const V*>(S.r);
  V* z = reinterpret_cast<V*>(S.fold);
  const double isp = 1.0 / sqrt((double)S.P);
  const unsigned nmask = (unsigned)S.n - 1u;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < S.np;
       j += (int64_t)gridDim.x * blockDim.x) {
    V acc = zero_of(V{});
    for (uint32_t e = S.bin_off[j]; e < S.bin_off[j + 1]; ++e) {
      const uint32_t row = S.bin_row[e];
      const unsigned w = S.op.omega[row];
      acc = add(acc, cmul(r[row], conj(tw_at<V>(S.op, (w * (unsigned)S.p) & nmask))));
    }
    z[j] = scale(acc, isp);
  }
}

template <class V>
__global__ void k_lg_sum_partials(const V* const* __restrict__ src, int P, V* __restrict__ dst, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    V a = src[0][i];
    for (int q = 1; q < P; ++q) a = add(a, src[q][i]);
    dst[i] = a;
  }
}

template <class V>
__global__ void k_lg_take_narrow(LgShard S) {
  V* h0s = reinterpret_cast<V*>(S.h0s);
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < S.np;
       k += (int64_t)gridDim.x * blockDim.x)
    from_c128(S.h0x[(int64_t)S.p + ((int64_t)k << S.log2P)], h0s[k]);
}

template <class V>
__global__ void k_lg_classmajor(const V* __restrict__ g, V* __restrict__ gcm, int64_t n, int P) {
  const int64_t np = n / P;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / np, j = i - c * np;
    gcm[i] = g[c + (int64_t)P * j];
  }
}

__global__ void k_lg_reduce_f64(const double* __restrict__ src, int P, int op_max, double* __restrict__ dst) {
  if (threadIdx.x || blockIdx.x) return;
  double a = src[0];
  for (int q = 1; q < P; ++q) a = op_max ? fmax(a, src[q]) : a + src[q];
  *dst = a;
}

__global__ void k_lg_reduce_u64_min(const unsigned long long* __restrict__ src, int P,
                                    unsigned long long* __restrict__ dst) {
  if (threadIdx.x || blockIdx.x) return;
  unsigned long long a = src[0];
  for (int q = 1; q < P; ++q) a = min(a, src[q]);
  *dst = a;
}

int blocks_for(int64_t cnt, int per = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((cnt + per - 1) / per, 8 * num_sms()));
}

}  // namespace

int lg_grid() { return num_sms() * 4; }

cudaError_t lg_fast(const LgShard& S, int s, cudaStream_t st) {
  const int grid = lg_grid();
  if (S.dtype == C128) k_lg_fast<double2><<<grid, LG_THREADS, 0, st>>>(S, s);
  else k_lg_fast<float2><<<grid, LG_THREADS, 0, st>>>(S, s);
  k_lg_best<<<1, 1024, 0, st>>>(S.blkmax, grid, S.rec_send);
  g_launches += 2;
  return cudaGetLastError();
}

cudaError_t lg_max(const LgShard& S, const void* h, cudaStream_t st) {
  const int grid = lg_grid();
  if (S.dtype == C128) k_lg_max<double2><<<grid, LG_THREADS, 0, st>>>((const double2*)h, S.np, S.blkmax);
  else k_lg_max<float2><<<grid, LG_THREADS, 0, st>>>((const float2*)h, S.np, S.blkmax);
  k_lg_best<<<1, 1024, 0, st>>>(S.blkmax, grid, S.rec_send);
  g_launches += 2;
  return cudaGetLastError();
}

cudaError_t lg_identify(const LgShard& S, const void* h, int s, double ecoef, int prev, cudaStream_t st) {
  k_lg_reset<<<1, 1, 0, st>>>(S, prev);
  ++g_launches;
  const int grid = lg_grid();
  const int64_t ntiles = (S.np + LG_TILE - 1) / LG_TILE;
  const int cb = blocks_for(ntiles, LG_THREADS);
  if (S.dtype == C128) k_lg_cands<double2><<<cb, LG_THREADS, 0, st>>>(S, (const double2*)h, ecoef, prev, grid);
  else k_lg_cands<float2><<<cb, LG_THREADS, 0, st>>>(S, (const float2*)h, ecoef, prev, grid);
  k_lg_eval<<<grid, LG_THREADS, 0, st>>>(S, s, prev);
  k_lg_record<<<1, 64, 0, st>>>(S, prev);
  g_launches += 3;
  return cudaGetLastError();
}

cudaError_t lg_merge(const LgShard& S, int cur, int prev, cudaStream_t st) {
  k_lg_merge<<<1, 1, 0, st>>>(S, cur, prev);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_fb_local_best(const LgShard& S, cudaStream_t st) {
  k_lg_fb_best<<<1, 1024, 0, st>>>(S);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_fb_local_first(const LgShard& S, cudaStream_t st) {
  k_lg_fb_first<<<1, 1024, 0, st>>>(S);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_fb_pick(const LgShard& S, int cur, cudaStream_t st) {
  k_lg_fb_pick<<<1, 1, 0, st>>>(S, cur);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_ls(const LgShard& S, int s, int cur, cudaStream_t st) {
  const int nblk = std::max(1, (s + LG_THREADS / 32 - 1) / (LG_THREADS / 32));
  k_lg_ls_a<<<nblk, LG_THREADS, 0, st>>>(S, s, cur);
  k_lg_ls_b<<<1, 32, 0, st>>>(S, nblk, cur);
  const int warps = s + 1, cblk = (warps * 32 + LG_THREADS - 1) / LG_THREADS;
  const double xscale = -1.0;  // Fourier: xn = -x
  if (S.dtype == C128) k_lg_ls_c<double2><<<cblk, LG_THREADS, 0, st>>>(S, s, cur, xscale);
  else k_lg_ls_c<float2><<<cblk, LG_THREADS, 0, st>>>(S, s, cur, xscale);
  k_lg_xstats<<<1, 1024, 0, st>>>(S, s + 1, cur);
  g_launches += 4;
  return cudaGetLastError();
}

cudaError_t lg_class_positions(const LgShard& S, int cnt, cudaStream_t st) {
  if (cnt <= 0) return cudaSuccess;
  k_lg_class_pos<<<(cnt + 255) / 256, 256, 0, st>>>(S, cnt);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_scatter_dense(const LgShard& S, int dtype, void* out, int64_t len, int cnt, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, (size_t)len * elem_bytes(dtype), st);
  if (e != cudaSuccess || cnt <= 0) return e;
  if (dtype == C128) k_lg_scatter<double2><<<(cnt + 255) / 256, 256, 0, st>>>(S, (double2*)out, cnt);
  else k_lg_scatter<float2><<<(cnt + 255) / 256, 256, 0, st>>>(S, (float2*)out, cnt);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_partial(const LgShard& S, int dtype, const void* X, void* out, cudaStream_t st) {
  const int b = blocks_for(S.m);
  if (dtype == C128) k_lg_partial<double2><<<b, 256, 0, st>>>(S, (const double2*)X, (double2*)out);
  else k_lg_partial<float2><<<b, 256, 0, st>>>(S, (const float2*)X, (float2*)out);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_resid(const LgShard& S, int dtype, const void* ax, cudaStream_t st) {
  const int grid = lg_grid();
  if (dtype == C128) {
    // (for fp32 data this is the fp64 residual norm only: r stays the fp32 one)
    double2* r = S.dtype == C128 ? (double2*)S.r : nullptr;
    k_lg_resid<double2><<<grid, LG_THREADS, 0, st>>>(S.y64, (const double2*)ax, r, S.m, S.part);
  } else {
    k_lg_resid<float2><<<grid, LG_THREADS, 0, st>>>((const float2*)S.y, (const float2*)ax, (float2*)S.r,
                                                    S.m, S.part);
  }
  k_lg_sum<<<1, 256, 0, st>>>(S.part, grid, S.scal + 9);
  g_launches += 2;
  return cudaGetLastError();
}

cudaError_t lg_fold(const LgShard& S, cudaStream_t st) {
  const int b = blocks_for(S.np);
  if (S.dtype == C128) k_lg_fold<double2><<<b, 256, 0, st>>>(S);
  else k_lg_fold<float2><<<b, 256, 0, st>>>(S);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_sum_partials(int dtype, const void* const* src, int P, void* dst, int64_t m, cudaStream_t st) {
  const int b = blocks_for(m);
  if (dtype == C128)
    k_lg_sum_partials<double2><<<b, 256, 0, st>>>((const double2* const*)src, P, (double2*)dst, m);
  else
    k_lg_sum_partials<float2><<<b, 256, 0, st>>>((const float2* const*)src, P, (float2*)dst, m);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_take_narrow(const LgShard& S, cudaStream_t st) {
  const int b = blocks_for(S.np);
  if (S.dtype == C128) k_lg_take_narrow<double2><<<b, 256, 0, st>>>(S);
  else k_lg_take_narrow<float2><<<b, 256, 0, st>>>(S);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_classmajor(int dtype, const void* g, void* gcm, int64_t n, int P, cudaStream_t st) {
  const int grid = lg_grid();
  if (dtype == C128) k_lg_classmajor<double2><<<grid, 256, 0, st>>>((const double2*)g, (double2*)gcm, n, P);
  else k_lg_classmajor<float2><<<grid, 256, 0, st>>>((const float2*)g, (float2*)gcm, n, P);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_reduce_f64(const double* src, int P, int op_max, double* dst, cudaStream_t st) {
  k_lg_reduce_f64<<<1, 1, 0, st>>>(src, P, op_max, dst);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t lg_reduce_u64_min(const unsigned long long* src, int P, unsigned long long* dst, cudaStream_t st) {
  k_lg_reduce_u64_min<<<1, 1, 0, st>>>(src, P, dst);
  ++g_launches;
  return cudaGetLastError();
}

void lg_merge_host(const LgRec* recs, int P, const uint32_t* selbits, LgPick* out) {
  merge_records(recs, P, selbits, out);
}

}  // namespace fmp
