// CoSaMP (solvers.cpp:413-544) as one fused persistent kernel, one problem per
// CTA at a time.  Per iteration: correlation (the fast update on the current
// K-atom estimate, kernel.cpp:209-303, or U^H scatter(r)), the 2K largest
// |h|^2 with the reference's band tie rule (select_largest, solvers.cpp:62-86:
// an exact radix select of the count-th largest value on the order-preserving
// bit patterns of |h|^2, then "clear the band outright, then smallest
// positions inside it"), the union with the current support, least squares
// by Cholesky of the Gram lookups with the normal-equations pivot floor
// (solvers.cpp:120-177), pruning to the K largest coefficients with the same
// band rule, and the explicit residual by one forward transform.
#include "fmp_kcommon.cuh"

namespace fmp {
namespace {

constexpr int CS_THREADS = 512;
constexpr int CRMAX = 8;
constexpr int CLOGP = 3;

struct CosK {
  DevOp op;
  const void* y;
  const double* tol;
  int64_t batch;
  int T, K;
  int fast;                 // fast updates (t >= 2) vs conventional
  uint64_t* support;        // batch x K (final, ascending, 1-based)
  double2* coeffs;          // batch x K
  uint64_t* size;           // batch
  uint64_t* iters;
  double* resid;
  int32_t* aborted;
  uint64_t* hist_sup;       // batch x T x K (supports after each iteration), optional
  uint64_t* hist_size;      // batch x T, optional
  void* hist;               // batch x T x n correlation history, optional
  // workspace per CTA
  double* mag_ws;           // n
  void* h0_ws;              // n
  double2* L_ws;            // (3K)^2
  void* r_ws;               // m
  int* queue;
};

__device__ __forceinline__ unsigned long long dkey(double v) {
  return (unsigned long long)__double_as_longlong(v);  // v >= 0: monotone
}

// the count-th largest of m[0..len) (multiplicity counted): radix select on
// the 64-bit patterns, 8 bits per round, histogram in smem.  All threads
// return the same value.  `hist` needs 256 ints, `ctl` 4 ints.
__device__ double kth_largest(const double* m, int len, int count, int* hist, unsigned long long* ctl) {
  const int tid = threadIdx.x, nth = blockDim.x;
  unsigned long long prefix = 0, mask = 0;
  int need = count;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += nth) hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < len; i += nth) {
      const unsigned long long k = dkey(m[i]);
      if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255], 1);
    }
    __syncthreads();
    if (tid == 0) {
      int acc = 0, d = 255;
      for (; d > 0; --d) {
        if (acc + hist[d] >= need) break;
        acc += hist[d];
      }
      ctl[0] = (unsigned long long)d;
      ctl[1] = (unsigned long long)(need - acc);
    }
    __syncthreads();
    prefix |= ctl[0] << shift;
    mask |= 255ull << shift;
    need = (int)ctl[1];
    __syncthreads();
  }
  return __longlong_as_double((long long)prefix);
}

// exclusive prefix of v over the block (thread order); total optional.
// `tmp` needs 33 ints.
__device__ int block_scan_excl(int v, int* tmp, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) tmp[w] = x;
  __syncthreads();
  if (w == 0) {
    int z = lane < nw ? tmp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    if (lane < nw) tmp[lane] = z;  // inclusive warp totals
    if (lane == 31) tmp[32] = z;
  }
  __syncthreads();
  const int before = (w ? tmp[w - 1] : 0) + x - v;
  if (total) *total = tmp[32];
  return before;
}

template <class V, bool HAD>
__global__ void __launch_bounds__(CS_THREADS, 1) k_cosamp(CosK a) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ double red[32];
  __shared__ unsigned redu[32];
  __shared__ int s_hist[256];
  __shared__ unsigned long long s_ctl[4];
  __shared__ int s_prob, s_cnt[4];
  const DevOp& op = a.op;
  const int n = (int)op.n, m = (int)op.m, log2n = op.log2n, T = a.T, K = a.K;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int nbuf = n + (n >> CLOGP);
  const V zv = zero_of(V{});
  const double sc = 1.0 / sqrt((double)n);
  const double xscale = HAD ? -1.0 / (double)n : -1.0;
  const int C2 = min(2 * K, n), C3 = 3 * K;

  V* buf = reinterpret_cast<V*>(sm);
  unsigned char* p = sm + ((sizeof(V) * (size_t)nbuf + 15) / 16) * 16;
  unsigned* s_sup = reinterpret_cast<unsigned*>(p); p += 4 * (size_t)C3;   // current support
  unsigned* s_mrg = reinterpret_cast<unsigned*>(p); p += 4 * (size_t)C3;   // merged atoms
  unsigned* s_pick = reinterpret_cast<unsigned*>(p); p += 4 * (size_t)C3;  // picked / kept
  p = sm + (((size_t)(p - sm) + 15) / 16) * 16;
  double2* s_x = reinterpret_cast<double2*>(p); p += 16 * (size_t)C3;      // coefficients
  double2* s_b = reinterpret_cast<double2*>(p); p += 16 * (size_t)C3;      // LS solution
  V* s_xn = reinterpret_cast<V*>(p); p += ((sizeof(V) * (size_t)C3 + 15) / 16) * 16;
  double* s_mg = reinterpret_cast<double*>(p); p += 8 * (size_t)C3;        // |b|^2 (C3)
  unsigned* s_bits = reinterpret_cast<unsigned*>(p);                         // support bitmap (n bits)

  double* msc = a.mag_ws + (size_t)blockIdx.x * n;
  V* h0w = reinterpret_cast<V*>(a.h0_ws) + (size_t)blockIdx.x * n;
  double2* L = a.L_ws + (size_t)blockIdx.x * C3 * C3;
  V* rs = reinterpret_cast<V*>(a.r_ws) + (size_t)blockIdx.x * m;
  const V* gF = fourier_table<V>(op);
  const uint16_t* gH = op.glat;
  const V* twt = twiddles<V>(op);
  auto gram = [&](unsigned ga, unsigned gb) -> double2 {
    if constexpr (HAD) return make_double2(op.gr64[ga ^ gb], 0.0);
    else return op.g64[(ga - gb) & (unsigned)(n - 1)];
  };

  for (;;) {
    __syncthreads();
    if (tid == 0) s_prob = atomicAdd(a.queue, 1);
    __syncthreads();
    const int64_t prob = s_prob;
    if (prob >= a.batch) break;
    const V* y = reinterpret_cast<const V*>(a.y) + prob * m;
    const double tol = a.tol[prob];
    double yy = 0.0;
    for (int j = tid; j < m; j += nth) yy += mag2(y[j]);
    yy = block_sum(yy, red);
    double rn = sqrt(yy);
    int s = 0, iters = 0, aborted = 0;
    for (int i = tid; i < (n + 31) / 32; i += nth) s_bits[i] = 0u;
    if (!(K == 0 || rn <= tol)) {
      for (int t = 1; t <= T; ++t) {
        // ---- correlation
        V* hrow = a.hist ? reinterpret_cast<V*>(a.hist) + ((size_t)prob * T + (t - 1)) * n : nullptr;
        if (t == 1 || !a.fast) {
          const V* r = t == 1 ? y : rs;
          for (int i = tid; i < nbuf; i += nth) buf[i] = zv;
          __syncthreads();
          for (int j = tid; j < m; j += nth)
            buf[padx<CLOGP>(HAD ? (int)op.omega[j] : (int)brev_n(op.omega[j], log2n))] = r[j];
          __syncthreads();
          block_transform<CRMAX, true, HAD>(buf, log2n, TwTable<V>{twt}, tid, nth);
          for (int k = tid; k < n; k += nth) {
            const V v = scale(buf[padx<CLOGP>(k)], sc);
            if (t == 1) h0w[k] = v;
            if (hrow) hrow[k] = v;
            msc[k] = mag2(v);
          }
        } else {
          for (int i = tid; i < n; i += nth) {
            V acc = h0w[i];
            fast_point<V, HAD>(acc, i, n, gF, gH, s_sup, s_xn, s);
            if (hrow) hrow[i] = acc;
            msc[i] = mag2(acc);
          }
        }
        __syncthreads();
        // ---- the C2 largest (top_atoms, solvers.cpp:105-118 -> select_largest)
        //      united with the support (std::set_union): one index-ordered
        //      compaction of "sure, or among the first tied, or in the support"
        {
          double hi = INFINITY, lo = INFINITY;
          if (C2 < n) {
            const double bnd = kth_largest(msc, n, C2, s_hist, s_ctl);
            hi = bnd * (1.0 + kTieBandRel);
            lo = bnd * (1.0 - kTieBandRel);
          }
          const int per = (n + nth - 1) / nth, i0 = tid * per, i1 = min(n, i0 + per);
          int nsure = 0, ntied = 0;
          if (C2 < n)
            for (int i = i0; i < i1; ++i) {
              const double v = msc[i];
              nsure += v > hi;
              ntied += v <= hi && v >= lo;
            }
          int tot_sure;
          const int tied_before = block_scan_excl(ntied, s_hist, nullptr);
          block_scan_excl(nsure, s_hist, &tot_sure);
          const int cap = C2 - tot_sure;  // tied positions taken, in index order
          int nsel = 0, tr = tied_before;
          for (int i = i0; i < i1; ++i) {
            const double v = msc[i];
            bool sel = C2 >= n || v > hi;
            if (!sel && v <= hi && v >= lo) sel = tr++ < cap;
            sel = sel || (s_bits[i >> 5] >> (i & 31) & 1u);
            nsel += sel;
          }
          int total;
          int o = block_scan_excl(nsel, s_hist, &total);
          tr = tied_before;
          for (int i = i0; i < i1; ++i) {
            const double v = msc[i];
            bool sel = C2 >= n || v > hi;
            if (!sel && v <= hi && v >= lo) sel = tr++ < cap;
            sel = sel || (s_bits[i >> 5] >> (i & 31) & 1u);
            if (sel) s_mrg[o++] = (unsigned)i;
          }
          if (tid == 0) s_cnt[3] = total;
          __syncthreads();
        }
        const int sm_ = s_cnt[3];
        if (tid == 0) s_cnt[1] = s;
        // ---- least squares on merged: Cholesky of the Gram lookups
        for (int e = tid; e < sm_ * sm_; e += nth) {
          const int i = e / sm_, j = e % sm_;
          if (i >= j) L[i * sm_ + j] = gram(s_mrg[i], s_mrg[j]);
        }
        for (int i = tid; i < sm_; i += nth) s_b[i] = to_c128(h0w[s_mrg[i]]);  // phi_i^H y
        __syncthreads();
        int bad = 0;
        for (int j = 0; j < sm_; ++j) {
          // column j: pivot (one thread), then the rows below (all threads)
          if (tid == 0) {
            const double diag = gram(s_mrg[j], s_mrg[j]).x;
            double d = L[j * sm_ + j].x;
            for (int k = 0; k < j; ++k) d -= mag2(L[j * sm_ + k]);
            if (!(d > 1e-12 * diag)) s_cnt[0] = -1;
            else {
              s_cnt[0] = 0;
              L[j * sm_ + j] = make_double2(sqrt(d), 0.0);
            }
          }
          __syncthreads();
          if (s_cnt[0] < 0) { bad = 1; break; }
          const double ljj = L[j * sm_ + j].x;
          for (int i = j + 1 + tid; i < sm_; i += nth) {
            double2 v = L[i * sm_ + j];
            for (int k = 0; k < j; ++k) {
              const double2 pp = L[i * sm_ + k], q = L[j * sm_ + k];
              v.x -= pp.x * q.x + pp.y * q.y;
              v.y -= pp.y * q.x - pp.x * q.y;
            }
            L[i * sm_ + j] = make_double2(v.x / ljj, v.y / ljj);
          }
          __syncthreads();
        }
        if (bad) { aborted = 1; break; }
        if (tid == 0) {
          for (int i = 0; i < sm_; ++i) {  // L z = b
            double2 v = s_b[i];
            for (int k = 0; k < i; ++k) {
              const double2 pp = L[i * sm_ + k], q = s_b[k];
              v.x -= pp.x * q.x - pp.y * q.y;
              v.y -= pp.x * q.y + pp.y * q.x;
            }
            const double l = L[i * sm_ + i].x;
            s_b[i] = make_double2(v.x / l, v.y / l);
          }
          for (int i = sm_ - 1; i >= 0; --i) {  // L^H x = z
            double2 v = s_b[i];
            for (int k = i + 1; k < sm_; ++k) {
              const double2 pp = L[k * sm_ + i], q = s_b[k];
              v.x -= pp.x * q.x + pp.y * q.y;
              v.y -= pp.x * q.y - pp.y * q.x;
            }
            const double l = L[i * sm_ + i].x;
            s_b[i] = make_double2(v.x / l, v.y / l);
          }
          // ---- prune to the K largest |b|^2 (select_largest, band rule)
          const int keep = min(K, sm_);
          for (int i = 0; i < sm_; ++i) s_mg[i] = mag2(s_b[i]);
          int ns = 0, nt = 0;
          if (keep < sm_) {
            // count-th largest by selection (sm_ <= 3K is small)
            double bnd = 0.0;
            {
              int done = 0;
              double prev = INFINITY;
              while (done < keep) {
                double best = -1.0;
                int mult = 0;
                for (int i = 0; i < sm_; ++i)
                  if (s_mg[i] < prev) {
                    if (s_mg[i] > best) { best = s_mg[i]; mult = 1; }
                    else if (s_mg[i] == best) ++mult;
                  }
                bnd = best;
                done += mult;
                prev = best;
              }
            }
            const double hi = bnd * (1.0 + kTieBandRel), lo = bnd * (1.0 - kTieBandRel);
            for (int i = 0; i < sm_; ++i)
              if (s_mg[i] > hi) s_pick[ns++] = (unsigned)i;
            for (int i = 0; i < sm_ && ns + nt < keep; ++i)
              if (s_mg[i] <= hi && s_mg[i] >= lo) { s_pick[ns + nt] = (unsigned)i; ++nt; }
            // kept positions ascending (positions order == atom order)
            for (int i = 1; i < keep; ++i) {
              const unsigned v = s_pick[i];
              int j = i - 1;
              while (j >= 0 && s_pick[j] > v) { s_pick[j + 1] = s_pick[j]; --j; }
              s_pick[j + 1] = v;
            }
          } else {
            for (int i = 0; i < sm_; ++i) s_pick[i] = (unsigned)i;
          }
          for (int i = 0; i < s_cnt[1]; ++i) s_bits[s_sup[i] >> 5] &= ~(1u << (s_sup[i] & 31));
          for (int i = 0; i < keep; ++i) {
            s_bits[s_mrg[s_pick[i]] >> 5] |= 1u << (s_mrg[s_pick[i]] & 31);
            s_sup[i] = s_mrg[s_pick[i]];
            s_x[i] = s_b[s_pick[i]];
            from_c128(make_double2(s_x[i].x * xscale, s_x[i].y * xscale), s_xn[i]);
          }
          s_cnt[0] = keep;
        }
        __syncthreads();
        s = s_cnt[0];
        // ---- residual r = y - Phi_S x (one forward transform)
        for (int i = tid; i < nbuf; i += nth) buf[i] = zv;
        __syncthreads();
        for (int j = tid; j < s; j += nth) {
          V xv;
          from_c128(s_x[j], xv);
          buf[padx<CLOGP>(HAD ? (int)s_sup[j] : (int)brev_n(s_sup[j], log2n))] = xv;
        }
        __syncthreads();
        block_transform<CRMAX, false, HAD>(buf, log2n, TwTable<V>{twt}, tid, nth);
        double r2 = 0.0;
        for (int j = tid; j < m; j += nth) {
          const V rv = sub(y[j], scale(buf[padx<CLOGP>((int)op.omega[j])], sc));
          rs[j] = rv;
          r2 += mag2(rv);
        }
        rn = sqrt(block_sum(r2, red));
        iters = t;
        if (a.hist_sup && tid == 0) {
          uint64_t* hs = a.hist_sup + ((size_t)prob * T + (t - 1)) * K;
          for (int j = 0; j < K; ++j) hs[j] = j < s ? (uint64_t)s_sup[j] + 1 : 0;
          a.hist_size[prob * T + (t - 1)] = (uint64_t)s;
        }
        if (rn <= tol) break;
      }
    }
    uint64_t* sup = a.support + prob * K;
    double2* co = a.coeffs + prob * K;
    for (int j = tid; j < K; j += nth) {
      sup[j] = j < s ? (uint64_t)s_sup[j] + 1 : 0;
      co[j] = j < s ? s_x[j] : make_double2(0.0, 0.0);
    }
    if (tid == 0) {
      a.size[prob] = (uint64_t)s;
      a.iters[prob] = (uint64_t)iters;
      a.resid[prob] = rn;
      a.aborted[prob] = aborted;
    }
  }
}

template <class V, bool HAD>
cudaError_t launch_cos(const CosArgs& c, cudaStream_t st) {
  const DevOp& op = *c.op;
  const int64_t n = op.n;
  const int C3 = 3 * (int)c.k;
  const size_t smem = ((sizeof(V) * (size_t)(n + (n >> CLOGP)) + 15) / 16) * 16 + 12 * (size_t)C3 + 16 +
                      16 * 2 * (size_t)C3 + ((sizeof(V) * (size_t)C3 + 15) / 16) * 16 + 8 * (size_t)C3 +
                      4 * (size_t)((n + 31) / 32) + 64;
  if (smem > (size_t)smem_optin() - 4096) return cudaErrorInvalidConfiguration;
  CosK k{};
  k.op = op;
  k.y = c.y;
  k.tol = c.tol;
  k.batch = c.batch;
  k.T = (int)c.max_iter;
  k.K = (int)c.k;
  k.fast = c.fast;
  k.support = c.support;
  k.coeffs = c.coeffs;
  k.size = c.size;
  k.iters = c.iters;
  k.resid = c.resid;
  k.aborted = c.aborted;
  k.hist_sup = c.hist_sup;
  k.hist_size = c.hist_size;
  k.hist = c.hist;
  k.mag_ws = c.mag_ws;
  k.h0_ws = c.h0_ws;
  k.L_ws = c.L_ws;
  k.r_ws = c.r_ws;
  k.queue = c.queue;
  auto f = k_cosamp<V, HAD>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  f<<<std::max(1, c.grid), CS_THREADS, smem, st>>>(k);
  ++g_launches;
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_cosamp(const CosArgs& c, cudaStream_t st) {
  g_launches = 0;
  const bool had = c.op->kind == HADAMARD;
  if (had && !c.op->glat) return cudaErrorInvalidValue;
  switch (c.dtype) {
    case C128: return had ? launch_cos<double2, true>(c, st) : launch_cos<double2, false>(c, st);
    case C64: return had ? launch_cos<float2, true>(c, st) : launch_cos<float2, false>(c, st);
    case F64: return had ? launch_cos<double, true>(c, st) : cudaErrorInvalidValue;
    case F32: return had ? launch_cos<float, true>(c, st) : cudaErrorInvalidValue;
  }
  return cudaErrorInvalidValue;
}

}  // namespace fmp
