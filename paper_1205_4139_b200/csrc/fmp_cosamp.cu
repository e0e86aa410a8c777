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
  int s_cap;                // merged sizes whose packed L fits the smem region
  int region;               // bytes of the transform-buffer / L region
  uint64_t* support;        // batch x K (final, ascending, 1-based)
  double2* coeffs;          // batch x K
  uint64_t* size;           // batch
  uint64_t* iters;
  double* resid;
  int32_t* aborted;
  uint64_t* hist_sup;       // batch x T x K (supports after each iteration), optional
  void* hist;               // batch x T x n correlation history, optional
  // workspace per CTA
  double* mag_ws;           // n
  void* h0_ws;              // n
  double2* L_ws;            // (3K)^2
  void* r_ws;               // m
  int* queue;
  unsigned long long* phase_ws;  // optional cycles per phase (conv, fast, identify, ls, resid, other)
  const int* ready;              // optional streamed-input flags
  int64_t ready_chunk;
  const volatile int* abort_word;
};

__device__ __forceinline__ unsigned long long dkey(double v) {
  return (unsigned long long)__double_as_longlong(v);  // v >= 0: monotone
}

// the count-th largest of m[0..len) (multiplicity counted): radix select on
// the 64-bit patterns, 8 bits per round; the digit holding the count-th
// largest is found by a parallel suffix scan of the 256-bin histogram.
// All threads return the same value.  `hist` needs 256 ints, `ctl` 2; the
// block must have >= 256 threads.
__device__ double kth_largest(const double* m, int len, int count, int* hist, unsigned long long* ctl) {
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, w = tid >> 5;
  __shared__ int wsum[8];
  unsigned long long prefix = 0, mask = 0;
  int need = count;
  for (int shift = 56; shift >= 0; shift -= 8) {
    if (tid < 256) hist[tid] = 0;
    __syncthreads();
    for (int i = tid; i < len; i += nth) {
      const unsigned long long k = dkey(m[i]);
      if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 255], 1);
    }
    __syncthreads();
    // suffix sums: thread d (< 256) owns digit 255 - d, so an inclusive
    // prefix over d is the count of candidates with digit >= 255 - d
    int v = 0, incl = 0;
    if (tid < 256) {
      v = hist[255 - tid];
      incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) wsum[w] = incl;
    }
    __syncthreads();
    if (tid < 256) {
      for (int q = 0; q < w; ++q) incl += wsum[q];
      const int before = incl - v;  // candidates with a larger digit
      if (before < need && incl >= need) {
        ctl[0] = (unsigned long long)(255 - tid);
        ctl[1] = (unsigned long long)(need - before);
      }
    }
    __syncthreads();
    prefix |= ctl[0] << shift;
    mask |= 255ull << shift;
    need = (int)ctl[1];
  }
  __syncthreads();
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

// select_largest (solvers.cpp:62-86) as ascending positions: the `count`
// largest of vals[0..len) -- everything above the band around the
// count-th largest value, then the smallest positions inside the band --
// united with the positions set in `bits` (optional).  One index-ordered
// compaction, so `out` comes out sorted.  Returns the number written.
__device__ int select_band(const double* vals, int len, int count, const unsigned* bits,
                           unsigned* out, int* s_hist, unsigned long long* s_ctl) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const bool all = count >= len;
  double hi = INFINITY, lo = INFINITY;
  if (!all) {
    const double bnd = kth_largest(vals, len, count, s_hist, s_ctl);
    hi = bnd * (1.0 + kTieBandRel);
    lo = bnd * (1.0 - kTieBandRel);
  }
  const int per = (len + nth - 1) / nth, i0 = tid * per, i1 = min(len, i0 + per);
  int nsure = 0, ntied = 0;
  if (!all)
    for (int i = i0; i < i1; ++i) {
      const double v = vals[i];
      nsure += v > hi;
      ntied += v <= hi && v >= lo;
    }
  int tot_sure = 0;
  const int tied_before = block_scan_excl(ntied, s_hist, nullptr);
  block_scan_excl(nsure, s_hist, &tot_sure);
  const int cap = count - tot_sure;  // tied positions taken, in index order
  auto chosen = [&](int i, int& tr) {
    const double v = vals[i];
    bool sel = all || v > hi;
    if (!sel && v <= hi && v >= lo) sel = tr++ < cap;
    if (bits) sel = sel || ((bits[i >> 5] >> (i & 31)) & 1u);
    return sel;
  };
  int nsel = 0, tr = tied_before;
  for (int i = i0; i < i1; ++i) nsel += chosen(i, tr);
  int total;
  int o = block_scan_excl(nsel, s_hist, &total);
  tr = tied_before;
  for (int i = i0; i < i1; ++i)
    if (chosen(i, tr)) out[o++] = (unsigned)i;
  __syncthreads();
  return total;
}

template <class V, bool HAD>
__global__ void __launch_bounds__(CS_THREADS, 1) k_cosamp(CosK a) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ double red[32];
  __shared__ int s_hist[256];
  __shared__ unsigned long long s_ctl[4];
  __shared__ int s_prob, s_lost;
  const DevOp& op = a.op;
  const int n = (int)op.n, m = (int)op.m, log2n = op.log2n, T = a.T, K = a.K;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nth >> 5;
  const int nbuf = n + (n >> CLOGP);
  const V zv = zero_of(V{});
  const double sc = 1.0 / sqrt((double)n);
  const double xscale = HAD ? -1.0 / (double)n : -1.0;
  const int C2 = min(2 * K, n), C3 = 3 * K;

  V* buf = reinterpret_cast<V*>(sm);  // shared with L (packed) during least squares
  unsigned char* p = sm + a.region;
  unsigned* s_sup = reinterpret_cast<unsigned*>(p); p += 4 * (size_t)C3;   // current support
  unsigned* s_mrg = reinterpret_cast<unsigned*>(p); p += 4 * (size_t)C3;   // merged atoms
  unsigned* s_pick = reinterpret_cast<unsigned*>(p); p += 4 * (size_t)C3;  // kept positions
  p = sm + (((size_t)(p - sm) + 15) / 16) * 16;
  double2* s_x = reinterpret_cast<double2*>(p); p += 16 * (size_t)C3;      // coefficients / z
  double2* s_b = reinterpret_cast<double2*>(p); p += 16 * (size_t)C3;      // rhs (eliminated)
  double2* s_t = reinterpret_cast<double2*>(p); p += 16 * (size_t)C3;      // LS solution
  double2* s_c2 = reinterpret_cast<double2*>(p); p += 16 * (size_t)C3;     // column cache (LDL^H)
  V* s_xn = reinterpret_cast<V*>(p); p += ((sizeof(V) * (size_t)C3 + 15) / 16) * 16;
  double* s_mg = reinterpret_cast<double*>(p); p += 8 * (size_t)C3;        // |b|^2
  unsigned* s_bits = reinterpret_cast<unsigned*>(p);                         // support bitmap

  double* msc = a.mag_ws + (size_t)blockIdx.x * n;
  V* h0w = reinterpret_cast<V*>(a.h0_ws) + (size_t)blockIdx.x * n;
  double2* Lg = a.L_ws + (size_t)blockIdx.x * C3 * (C3 + 1) / 2;  // packed lower triangle
  V* rs = reinterpret_cast<V*>(a.r_ws) + (size_t)blockIdx.x * m;
  const V* gF = fourier_table<V>(op);
  const uint16_t* gH = op.glat;
  const V* twt = twiddles<V>(op);
  // Gram entry phi_a^H phi_b from the kernel (kernel.cpp:113-140)
  auto gram = [&](unsigned ga, unsigned gb) -> double2 {
    if constexpr (HAD) return make_double2(op.gr64[ga ^ gb], 0.0);
    else return op.g64[(ga - gb) & (unsigned)(n - 1)];
  };

  // opt-in phase profile (thread 0's clock between barrier-terminated phases)
  unsigned long long ph[6] = {0, 0, 0, 0, 0, 0};
  unsigned long long ph_last = clock64();
  auto mark = [&](int phase) {
    if (a.phase_ws && tid == 0) {
      const unsigned long long now = clock64();
      ph[phase] += now - ph_last;
      ph_last = now;
    }
  };

  // s_lost: streamed input abandoned (host abort or timeout), sticky: the
  // CTA fails every later problem without waiting again
  if (tid == 0) s_lost = 0;
  for (;;) {
    __syncthreads();
    if (tid == 0) {
      s_prob = atomicAdd(a.queue, 1);
      if (!s_lost && a.ready && s_prob < a.batch &&
          !wait_ready(a.ready + s_prob / a.ready_chunk, a.abort_word))
        s_lost = 1;
    }
    __syncthreads();
    const int64_t prob = s_prob;
    if (prob >= a.batch) break;
    if (s_lost) {
      if (tid == 0) {
        a.size[prob] = 0;
        a.iters[prob] = 0;
        a.resid[prob] = 0.0;
        a.aborted[prob] = kInputLost;
      }
      continue;
    }
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
        // ---- correlation: U^H scatter(r) (t = 1 or conventional) or the
        //      fast update on the current estimate (kernel.cpp:209-303)
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
        mark(t == 1 || !a.fast ? 0 : 1);
        // ---- merged = sorted(support) U top_atoms(h, 2K) (solvers.cpp:105-118, 471-478)
        const int sm_ = select_band(msc, n, C2, s_bits, s_mrg, s_hist, s_ctl);
        // ---- normal equations on merged (solvers.cpp:120-177): Cholesky,
        //      left-looking like the reference, one warp per row dot
        mark(2);
        // Right-looking LDL^H of the Gram on merged (entries looked up in the
        // kernel), the rhs phi^H y = h0[merged] eliminated in the same sweep:
        // one barrier per column.  Pivot j is g_jj - sum_k |l_jk|^2 with the
        // terms subtracted in the reference's order (solvers.cpp:148-160).
        const double diag = gram(0u, 0u).x;
        auto row = [](int i) { return (size_t)i * (i + 1) / 2; };
        // rows [r0, sm_) of the packed triangle in the shared-memory region,
        // rows [0, r0) in global memory: row i is rewritten at every one of
        // its i steps, so the long bottom rows take the fast memory and the
        // rarely touched top rows spill (r0 = 0 when the whole triangle fits)
        int r0 = 0;
        if (sm_ > a.s_cap) {
          const size_t cap = (size_t)a.region / 16, tot = row(sm_);
          while (tot - row(r0) > cap) ++r0;
        }
        double2* const Ls = reinterpret_cast<double2*>(sm);
        const size_t base0 = row(r0);
        auto Lrow = [&](int i) -> double2* { return i < r0 ? Lg + row(i) : Ls + (row(i) - base0); };
        __syncthreads();  // buf is free
        // column j of the factor, double-buffered in smem (s_t is free until
        // the back substitution): the update of step j reads column j from
        // one buffer and writes column j + 1, as it finalises, into the other
        double2* colb[2] = {s_t, s_c2};
        for (int i = warp; i < sm_; i += nw) {
          const unsigned li = s_mrg[i];
          double2* Li = Lrow(i);
          for (int l = lane; l <= i; l += 32) {
            const double2 g = gram(li, s_mrg[l]);
            Li[l] = g;
            if (l == 0) colb[0][i] = g;
          }
          if (lane == 0) s_b[i] = to_c128(h0w[li]);
        }
        __syncthreads();
        bool bad = false;
        for (int j = 0; j < sm_; ++j) {
          const double2* cj = colb[j & 1];
          double2* cn = colb[(j + 1) & 1];
          const double d = cj[j].x;
          if (!(d > 1e-12 * diag)) { bad = true; break; }
          const double inv = 1.0 / d;
          const double2 bj = s_b[j];
          for (int i = j + 1 + warp; i < sm_; i += nw) {
            double2* Li = Lrow(i);
            const double2 aij = cj[i];
            const double2 u = make_double2(aij.x * inv, aij.y * inv);  // a_ij / d_j
            for (int l = j + 1 + lane; l <= i; l += 32) {
              const double2 alj = cj[l];
              double2 v = Li[l];
              v.x -= u.x * alj.x + u.y * alj.y;  // a_il -= a_ij conj(a_lj) / d_j
              v.y -= u.y * alj.x - u.x * alj.y;
              Li[l] = v;
              if (l == j + 1) cn[i] = v;
            }
            if (lane == 0) {
              s_b[i].x -= u.x * bj.x - u.y * bj.y;
              s_b[i].y -= u.x * bj.y + u.y * bj.x;
            }
          }
          __syncthreads();
        }
        if (bad) { aborted = 1; break; }
        // back substitution of D L'^H x = b' (column-oriented; x into s_t):
        // x_i = (b'_i - sum_{k>i} conj(a_ki) x_k) / d_i
        for (int i = sm_ - 1; i >= 0; --i) {
          const double2* Li = Lrow(i);
          const double d = Li[i].x;
          const double2 xi = make_double2(s_b[i].x / d, s_b[i].y / d);
          for (int q = tid; q < i; q += nth) {
            const double2 pp = Li[q];
            s_b[q].x -= pp.x * xi.x + pp.y * xi.y;
            s_b[q].y -= pp.x * xi.y - pp.y * xi.x;
          }
          if (tid == 0) s_t[i] = xi;
          __syncthreads();
        }
        mark(3);
        for (int i = tid; i < sm_; i += nth) s_mg[i] = mag2(s_t[i]);
        for (int i = tid; i < s; i += nth) atomicAnd(&s_bits[s_sup[i] >> 5], ~(1u << (s_sup[i] & 31)));
        __syncthreads();
        const int keep = select_band(s_mg, sm_, min(K, sm_), nullptr, s_pick, s_hist, s_ctl);
        for (int i = tid; i < keep; i += nth) {
          const unsigned atom = s_mrg[s_pick[i]];
          const double2 xv = s_t[s_pick[i]];
          atomicOr(&s_bits[atom >> 5], 1u << (atom & 31));
          s_sup[i] = atom;
          s_x[i] = xv;
          from_c128(make_double2(xv.x * xscale, xv.y * xscale), s_xn[i]);
        }
        s = keep;
        __syncthreads();
        mark(2);
        // ---- residual r = y - Phi_S x (one forward transform)
        for (int i = tid; i < nbuf; i += nth) buf[i] = zv;  // (after the barrier above)
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
        mark(4);
        iters = t;
        if (a.hist_sup) {
          uint64_t* hs = a.hist_sup + ((size_t)prob * T + (t - 1)) * K;
          for (int j = tid; j < K; j += nth) hs[j] = j < s ? (uint64_t)s_sup[j] + 1 : 0;
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
    mark(5);
  }
  if (a.phase_ws && tid == 0)
    for (int i = 0; i < 6; ++i) atomicAdd(a.phase_ws + i, ph[i]);
}

template <class V, bool HAD>
cudaError_t launch_cos(const CosArgs& c, cudaStream_t st) {
  const DevOp& op = *c.op;
  const int64_t n = op.n;
  const int C3 = 3 * (int)c.k;
  const size_t small = 12 * (size_t)C3 + 16 + 16 * 4 * (size_t)C3 +
                       ((sizeof(V) * (size_t)C3 + 15) / 16) * 16 + 8 * (size_t)C3 +
                       4 * (size_t)((n + 31) / 32) + 64;
  const size_t bufb = ((sizeof(V) * (size_t)(n + (n >> CLOGP)) + 15) / 16) * 16;
  const size_t avail = (size_t)smem_optin() - 4096 - small;
  const size_t want = 16 * (size_t)C3 * (C3 + 1) / 2;
  const size_t region = std::max(bufb, std::min(want, avail) / 16 * 16);
  int s_cap = 0;
  while (s_cap < C3 && 16 * (size_t)(s_cap + 1) * (s_cap + 2) / 2 <= region) ++s_cap;
  const size_t smem = region + small;
  if (smem > (size_t)smem_optin() - 4096) return cudaErrorInvalidConfiguration;
  CosK k{};
  k.op = op;
  k.y = c.y;
  k.tol = c.tol;
  k.batch = c.batch;
  k.T = (int)c.max_iter;
  k.K = (int)c.k;
  k.fast = c.fast;
  k.s_cap = s_cap;
  k.region = (int)region;
  k.support = c.support;
  k.coeffs = c.coeffs;
  k.size = c.size;
  k.iters = c.iters;
  k.resid = c.resid;
  k.aborted = c.aborted;
  k.hist_sup = c.hist_sup;
  k.hist = c.hist;
  k.mag_ws = c.mag_ws;
  k.h0_ws = c.h0_ws;
  k.L_ws = c.L_ws;
  k.r_ws = c.r_ws;
  k.queue = c.queue;
  k.phase_ws = c.phase_ws;
  k.ready = c.ready;
  k.ready_chunk = c.ready_chunk;
  k.abort_word = c.abort_word;
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
