// Fused persistent OMP solver (solvers.cpp:296-411).
//
// One CTA owns one recovery problem at a time and pulls the next from a work
// counter, so problems that halt early (config 4's noise tolerance) free their
// SM at once.  Per problem, everything lives in shared memory:
//
//   buf  the transform buffer (n + n/8 slots); during fast iterations it holds
//        h0 = Phi^H y, so the shifted-kernel accumulate reads only smem
//   g    the correlation kernel c (Fourier: n complex; Hadamard: int16 lattice
//        N*c), staged once per CTA and shared by every problem it solves
//   W    the inverse Cholesky factor L^{-1} of the Gram matrix of the selected
//        columns, column-major packed (global workspace when it does not fit)
//   r    the residual (conventional iterations only)
//
// Iteration t (solvers.cpp:335-403): correlation h_t (t = 1 and conventional
// rows: U^H scatter(r) by a radix-8 FFT/FWHT; fast rows: h0 - sum x g shifted),
// band argmax (first index within 1e-9 of the max), stagnation stops, one Gram
// row appended to W (entries are lookups c[(a-b) mod N] / c[a^b]), z = W b with
// b = h0[Lambda], x = W^H z, then the residual: ||r||^2 = ||y||^2 - ||z||^2
// while that identity is well away from the tolerance, else an explicit
// r = y - Phi_Lambda x by one forward transform of the sparse estimate.
#pragma once
#include <atomic>
#include <type_traits>

#include "fmp_kcommon.cuh"

namespace fmp {
namespace {


// Radix of the in-kernel transform passes and the matching padding period
// of the transform buffer (one pad slot per radix).  Elements of <= 8 bytes
// (c64, f64, f32) hold a radix-16 sub-problem in <= 32 registers: config 4
// c64 (n = 2^14) runs 16 16 16 4 instead of 8 8 8 8 4 (31.3 k -> 36.3 k
// recoveries/s); c128 stays at radix 8 (radix 16 spills at 128 registers;
// its config-2 solver has the F16 rows instead).
template <class V> __host__ __device__ constexpr int ormax_v() { return sizeof(V) <= 8 ? 16 : 8; }
template <class V> __host__ __device__ constexpr int ologp_v() { return sizeof(V) <= 8 ? 4 : 3; }
// least-squares passes: LSG threads per row / column, LSU loads per thread
// issued together.  W in L2 or 512 threads: 8 / 4 (measured best, round 1);
// the F16 plan (256 threads, W in smem, T <= 64 rows in one sweep): 4 / 4
#ifndef FMP_LSGG
#define FMP_LSGG 8
#endif
#ifndef FMP_LSUG
#define FMP_LSUG 4
#endif
#ifndef FMP_LSG16
#define FMP_LSG16 4
#endif
#ifndef FMP_LSU16
#define FMP_LSU16 4
#endif

struct OmpK {
  DevOp op;
  const void* y;
  const double* tol;
  int64_t batch;
  int T;
  int64_t fast_until;
  uint64_t* support;  // 1-based, batch x T
  double2* coeffs;
  uint64_t* size;
  uint64_t* iters;
  uint64_t* hlen;
  double* resid;
  int32_t* aborted;
  uint8_t* modes;
  void* hist;
  double2* w_ws;
  void* h0_ws;
  double* mag_ws;
  void* r_ws;
  void* ys_ws;  // grid x m: y in transform-slot order (plans without smem maps)
  int* queue;
  // shared-memory plan
  void* buf_ws;  // grid x (n + n/8) when the buffer lives in global memory
  int r_smem, w_smem, map_smem;
  int w_rows;  // F16: leading rows of W (row-major packed) kept in shared memory
  int off_g, off_r, off_w, off_tw, off_small, off_map;
  int tw_a;       // two-level twiddle split
  double margin;  // relative slack on the residual identity
  unsigned long long* phase_ws;  // optional: cycles per phase (conv, fast, argmax, ls, resid, other)
  const int* ready;              // optional streamed-input flags (OmpArgs)
  int64_t ready_chunk;
  const volatile int* abort_word;  // host-raised abort of the streamed input (OmpArgs)
  // fp32 data (REFINE): fp64 h0 = Phi^H y per problem (batch x n, c128 / f64),
  // the error-bound coefficient and max_{k != 0} |c_k| (DevOp::goff)
  const void* h0x;
  double ecoef;
  double goff;
  unsigned long long* rstats;  // optional: identifications, candidates, overflows
};

// candidates re-evaluated in fp64 per identification (fp32 data) before the
// block falls back to evaluating every qualifying element thread-serially
constexpr int RCAP = 64;

template <class V> struct wide_t { using T = double2; };
template <> struct wide_t<double> { using T = double; };
template <> struct wide_t<float> { using T = double; };

template <bool HAD>
__device__ __forceinline__ double2 gram(const DevOp& op, unsigned a, unsigned b) {
  // (Phi^H Phi)_{ab} = c[(a - b) mod N] (Fourier) or c[a XOR b] (Hadamard)
  if constexpr (HAD) return make_double2(op.gr64[a ^ b], 0.0);
  else return op.g64[(a - b) & (unsigned)(op.n - 1)];
}

// column-major packed lower triangle with capacity T: W(i, j), i >= j
__device__ __forceinline__ int wofs(int T, int i, int j) {
  return j * T - (j * (j - 1)) / 2 + (i - j);
}

// ---------------------------------------------------------------- F16 path
// Config 2's two-CTA solver (Fourier, n = 4096 = 16^3, 256 threads): every
// transform of a conventional row or residual is three radix-16 passes with
// one 16-point sub-problem per thread, and both ends stay in registers:
//   * thread u ends the residual's forward transform holding X[u + 256 j]
//     (natural order, j = 0..15), forms r at the rows of Omega among them and
//     keeps those 16 values in registers; the next adjoint's first pass needs
//     exactly them, because DIT group g = brev8(u) holds the bit-reversed rows
//     brev12(16 g + j) = u + 256 brev4(j);
//   * the adjoint's last pass leaves h[u + 256 j] in registers, where the
//     identification reads |h|^2 (no store, no re-read);
//   * the sparse estimate enters the forward transform from per-group lists
//     of atoms (head / next, appended as atoms are selected): no zero-fill.
// Shared memory moves 64 + 128 + 64 KB per transform instead of the radix-8
// path's zero-fill, scatter, four read-write passes and gathers.  Padding:
// p + p/16 + p/512 keeps every pass (and the brev8 store) bank-conflict free.
__device__ __forceinline__ int pad16(int p) { return p + (p >> 4) + (p >> 9); }
__device__ __forceinline__ int brev8(int x) { return (int)(__brev((unsigned)x) >> 24); }

// F16 twiddle tables in shared memory: lo[k] = W^k (k < 64), hi[k] = W^(64 k)
// (k < 4): W^k = lo[k & 63] hi[k >> 6]
template <class V>
struct TwF16 {
  const V* lo;
  const V* hi;
};

// twiddles of a radix-16 DIT sub-problem (offset o in a span 2^LOGS of the
// 4096-point transform): W^(o 2^(8 - LOGS)) from the two-level table, its
// powers by products (the power scheme of pass_one: <= 4 roundings per
// twiddle), then the 16-point DFT
template <bool INV, int LOGS, class V>
__device__ __forceinline__ void r16_step(V (&v)[16], int o, const TwF16<V>& tw) {
  if constexpr (LOGS > 0) {
    const int k = o << (8 - LOGS);
    V w1 = cmul(tw.lo[k & 63], tw.hi[k >> 6]);
    if (INV) w1.y = -w1.y;
    V p2 = w1, p4 = w1, p8 = w1;
#pragma unroll
    for (int q = 1; q < 16; ++q) {
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
      v[brev_inv<16>(q)] = cmul(v[brev_inv<16>(q)], wq);
    }
  }
  dft_reg<16, INV>(v);
}

// passes 2 and 3 of the 4096-point transform (pass 1 stored by the caller;
// the leading barrier publishes it); v returns X[tid + 256 j].
// WARP1: pass 1 was stored by group = thread (the forward transform's atom
// lists), so the 16 groups a middle-pass thread reads come from its own
// half-warp and a warp barrier publishes them
template <bool INV, bool WARP1, class V>
__device__ __forceinline__ void f16_passes23(V* buf, V (&v)[16], const TwF16<V>& tw, int tid) {
  if (WARP1) __syncwarp();
  else __syncthreads();
  {
    const int o = tid & 15, base = ((tid >> 4) << 8) + o;
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = buf[pad16(base + 16 * j)];
    r16_step<INV, 4>(v, o, tw);
#pragma unroll
    for (int j = 0; j < 16; ++j) buf[pad16(base + 16 * j)] = v[j];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = buf[pad16(tid + 256 * j)];
  r16_step<INV, 8>(v, tid, tw);
}

// GMODE: kernel table source (0 global, 1 smem full, 2 smem conjugate half,
// Fourier only); BUFG: transform buffer in global memory (n beyond smem);
// NT threads per CTA, CT CTAs resident per SM (launch bounds)
// F16: the register-resident radix-16 conventional rows (see above)
template <class V, bool HAD, int RPT, int GMODE, bool BUFG, int NT, int CT, bool F16 = false>
__global__ void __launch_bounds__(NT, CT) k_omp(OmpK a) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ double red[96];
  __shared__ unsigned redu[32];
  __shared__ double red2[F16 ? 32 : 1];  // F16: the residual norm's partials
  __shared__ int s_prob, s_lost;
  constexpr int NW = NT / 32;  // warps per CTA (block reductions)
  constexpr int ORMAX = ormax_v<V>(), OLOGP = ologp_v<V>();
  // (c64: 4 threads per row, 8 loads per sweep - config 4's long rows of W
  // in L2: 38.5 k -> 39.3 k recoveries/s)
  constexpr bool LS48 = std::is_same<V, float2>::value;
  constexpr int LSG = F16 ? FMP_LSG16 : (LS48 ? 4 : FMP_LSGG), LSU = F16 ? FMP_LSU16 : (LS48 ? 8 : FMP_LSUG);
  const DevOp& op = a.op;
  const int n = (int)op.n, m = (int)op.m, log2n = op.log2n, T = a.T;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5,
            nw = nth >> 5;
  const int nbuf = n + (n >> OLOGP);
  const V zv = zero_of(V{});
  const double sc = 1.0 / sqrt((double)n);
  const double xscale = HAD ? -1.0 / (double)n : -1.0;

  V* buf = BUFG ? reinterpret_cast<V*>(a.buf_ws) + (size_t)blockIdx.x * nbuf
                : reinterpret_cast<V*>(sm);
  const V* gF = fourier_table<V>(op);
  const uint16_t* gH = op.glat;
  if constexpr (GMODE == 1 || GMODE == 2) {
    if constexpr (!HAD) {
      V* s = reinterpret_cast<V*>(sm + a.off_g);
      const int cnt = GMODE == 2 ? n / 2 + 1 : n;
      for (int i = tid; i < cnt; i += nth) s[i] = gF[i];
      gF = s;
    } else {
      uint16_t* s = reinterpret_cast<uint16_t*>(sm + a.off_g);
      for (int i = tid; i < n; i += nth) s[i] = op.glat[i];
      gH = s;
    }
  }
  // two-level twiddles (Fourier): lo[k] = W^k, hi[k] = W^(k 2^a)
  TwTwoLevel<V> tw{nullptr, nullptr, a.tw_a};
  TwF16<V> tw16{nullptr, nullptr};
  if constexpr (F16) {
    V* lo = reinterpret_cast<V*>(sm + a.off_tw);
    V* hi = lo + 64;
    const V* full = twiddles<V>(op);
    for (int k = tid; k < 64; k += nth) lo[k] = full[k];
    for (int k = tid; k < 4; k += nth) hi[k] = full[64 * k];
    tw16.lo = lo;
    tw16.hi = hi;
  } else if constexpr (!HAD) {
    V* lo = reinterpret_cast<V*>(sm + a.off_tw);
    V* hi = lo + TwTwoLevel<V>::pad(1 << a.tw_a) + 1;
    const V* full = twiddles<V>(op);
    for (int k = tid; k < (1 << a.tw_a); k += nth) lo[TwTwoLevel<V>::pad(k)] = full[k];
    for (int k = tid; k < (n >> a.tw_a); k += nth) hi[TwTwoLevel<V>::pad(k)] = full[k << a.tw_a];
    tw.lo = lo;
    tw.hi = hi;
  }
  V* rs = a.r_smem ? reinterpret_cast<V*>(sm + a.off_r)
                   : reinterpret_cast<V*>(a.r_ws) + (size_t)blockIdx.x * m;
  double2* W = a.w_smem ? reinterpret_cast<double2*>(sm + a.off_w)
                       : a.w_ws + (size_t)blockIdx.x * ((size_t)T * (T + 1) / 2);
  // F16: W row-major packed (row i at i (i + 1) / 2), split by rows: the
  // first R0 in shared memory, the later (shorter-lived) ones in the CTA's
  // global workspace.  R0 is a multiple of 8 or covers every row, so the 8
  // rows a warp takes in the first least-squares pass lie on one side.
  double2* const Ws = reinterpret_cast<double2*>(sm + a.off_w);
  double2* const Wg = a.w_ws + (size_t)blockIdx.x * ((size_t)T * (T + 1) / 2);
  const int R0 = a.w_rows;
  auto tri = [](int i) { return (i * (i + 1)) >> 1; };
  unsigned char* p = sm + a.off_small;
  double2* s_x = reinterpret_cast<double2*>(p); p += 16 * (size_t)T;
  double2* s_z = reinterpret_cast<double2*>(p); p += 16 * (size_t)T;
  double2* s_l = reinterpret_cast<double2*>(p); p += 16 * (size_t)T;
  V* s_xn = reinterpret_cast<V*>(p); p += ((sizeof(V) * (size_t)T + 15) / 16) * 16;
  unsigned* s_lam = reinterpret_cast<unsigned*>(p); p += ((4 * (size_t)T + 15) / 16) * 16;
  unsigned* s_sel = reinterpret_cast<unsigned*>(p);  // n bits: atoms selected so far
  p += ((4 * (size_t)((n + 31) / 32) + 15) / 16) * 16;
  // REFINE: identification candidates (index, fp64 |h|^2) and their count
  double* s_cval = reinterpret_cast<double*>(p); p += 8 * RCAP;
  unsigned* s_cand = reinterpret_cast<unsigned*>(p); p += 4 * RCAP;
  int* s_ncand = reinterpret_cast<int*>(p);
  // F16 (never REFINE, same region): per 16-slot group the first selected
  // atom (-1: none) and, per atom, the next one in its group
  int16_t* s_head = reinterpret_cast<int16_t*>(s_cval);
  int16_t* s_next = s_head + (F16 ? n / 16 : 0);
  constexpr bool REFINE = sizeof(typename scal<V>::T) == 4;
  static_assert(!(F16 && REFINE), "F16 is the fp64 path");
  using X = typename wide_t<V>::T;
  const X* h0x_all = reinterpret_cast<const X*>(a.h0x);

  // slot -> row map of the Omega scatter (-1: zero slot), so the adjoint's
  // first pass reads r directly
  int16_t* s_map = a.map_smem ? reinterpret_cast<int16_t*>(sm + a.off_map) : nullptr;
  // slot -> support position of the sparse estimate (forward transform input)
  int16_t* s_xmap = a.map_smem ? s_map + ((n + 7) / 8) * 8 : nullptr;
  if (s_map) {
    for (int i = tid; i < n; i += nth) s_map[i] = -1;
    __syncthreads();
    for (int j = tid; j < m; j += nth)
      s_map[HAD ? (int)op.omega[j] : (int)brev_n(op.omega[j], log2n)] = (int16_t)j;
  }
  V* h0w = reinterpret_cast<V*>(a.h0_ws) + (size_t)blockIdx.x * n;
  double* msc = a.mag_ws + (size_t)blockIdx.x * n;  // used only when a warp owns > 1 tile
  const double gamma = HAD ? op.gr64[0] : op.g64[0].x;  // c(1) = M/N
  // Gram entry (Phi^H Phi)_{ab}: from the staged kernel when it is exact fp64
  // (c128 table, or the Hadamard integer lattice), else the fp64 table
  auto gram_of = [&](unsigned ga, unsigned gb) -> double2 {
    if constexpr ((GMODE == 1 || GMODE == 2) && HAD) {
      return make_double2((double)((int)gH[ga ^ gb] - 32768) / (double)n, 0.0);
    } else if constexpr (GMODE == 1 && sizeof(V) == 16) {
      return to_c128(gF[(ga - gb) & (unsigned)(n - 1)]);
    } else if constexpr (GMODE == 2 && sizeof(V) == 16) {
      const unsigned j = (ga - gb) & (unsigned)(n - 1);
      return j <= (unsigned)(n >> 1) ? to_c128(gF[j]) : to_c128(conj(gF[n - j]));
    } else {
      return gram<HAD>(op, ga, gb);
    }
  };
  // index of transform slot i in buf (padded layouts)
  auto bp = [](int i) { return F16 ? pad16(i) : padx<OLOGP>(i); };
  const int ntiles = n >= 32 * RPT ? n / (32 * RPT) : 0;
  const bool regs_only = ntiles > 0 && ntiles <= nw;  // every thread owns <= 1 tile

  // opt-in phase profile (thread 0's clock between phase boundaries, which
  // all end in a block-wide barrier)
  // (added straight to the global totals: a per-thread array here would
  // live in local memory, and its loads / stores ran on every call)
  unsigned long long ph_last = clock64();
  auto mark = [&](int phase) {
    if (a.phase_ws && tid == 0) {
      const unsigned long long now = clock64();
      atomicAdd(a.phase_ws + phase, now - ph_last);
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
        if (a.hlen) a.hlen[prob] = 0;
      }
      continue;
    }
    const V* y = reinterpret_cast<const V*>(a.y) + prob * m;
    // no smem maps: y and r are kept in transform-slot order (ys_ws, r_ws)
    V* ysl = (!F16 && !s_map && a.ys_ws) ? reinterpret_cast<V*>(a.ys_ws) + (size_t)blockIdx.x * m : nullptr;
    // F16: the measurements of this thread's rows (tid + 256 j in Omega) in
    // thread order (DevOp::f16_omt / f16_yidx)
    V* yc = F16 ? (a.r_smem ? rs : reinterpret_cast<V*>(a.ys_ws) + (size_t)blockIdx.x * m) : nullptr;
    // F16: first pass of the adjoint from r of this thread's rows (rr[j]: row
    // tid + 256 j), stored to DIT group brev8(tid)
    auto adj_pass1 = [&](V (&rr)[16]) {
      if constexpr (F16) {
        const int g = brev8(tid);
        V v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = rr[brev_small<16>(j)];
        dft_reg<16, true>(v);
#pragma unroll
        for (int j = 0; j < 16; ++j) buf[pad16(16 * g + j)] = v[j];
      }
    };
    if constexpr (F16) {
      for (int g = tid; g < n / 16; g += nth) s_head[g] = -1;
      for (int j = tid; j < m; j += nth) yc[op.f16_yidx[j]] = y[j];
    }
    const double tol = a.tol[prob];
    const X* h0x = REFINE ? h0x_all + prob * n : nullptr;

    for (int i = tid; i < (n + 31) / 32; i += nth) s_sel[i] = 0u;
    if (s_xmap)
      for (int i = tid; i < n; i += nth) s_xmap[i] = -1;
    double yy = 0.0;
    for (int j = tid; j < m; j += nth) yy += mag2(y[j]);
    yy = block_sum<NW>(yy, red);
    double rn = sqrt(yy);
    double zz = 0.0;
    int s = 0, iters = 0, aborted = 0, tlast = 0;
    bool rn_explicit = true;
    bool buf_h0 = false;  // buf currently holds h0 in padded layout

    // explicit residual r = y - Phi_Lambda x by one forward transform of the
    // sparse estimate (replaces update_residual, solvers.cpp:180-192)
    auto residual_explicit = [&](int cnt) -> double {
      if constexpr (F16) {
        // (every earlier read of buf - fast rows, the identification scan -
        // is followed by a block-wide barrier on every path that gets here)
        {
          // pass 1 from the atom lists: thread tid owns group tid (slots
          // 16 tid + j, atom q at slot brev12(lambda_q))
          V v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = zv;
          for (int q = s_head[tid]; q >= 0; q = s_next[q]) {
            const int jj = (int)(brev_n(s_lam[q], log2n) & 15u);
            V xv;
            from_c128(s_x[q], xv);
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (j == jj) v[j] = xv;
          }
          dft_reg<16, false>(v);
#pragma unroll
          for (int j = 0; j < 16; ++j) buf[pad16(16 * tid + j)] = v[j];
        }
        V v[16];
        f16_passes23<false, true>(buf, v, tw16, tid);
        // r = y - Phi x at this thread's rows of Omega (ascending j); the
        // next conventional row's first pass follows at once (after the
        // norm's barriers, which also end every read of this transform), so
        // r never leaves registers
        const uint32_t om = op.f16_omt[tid];
        int c = (int)(om >> 16);
        double r2 = 0.0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {  // v[j] becomes r of row tid + 256 j
          if ((om >> j) & 1u) {
            v[j] = sub(yc[c], scale(v[j], sc));
            ++c;
            r2 += mag2(v[j]);
          } else {
            v[j] = zv;
          }
        }
        buf_h0 = false;
        (void)cnt;
        // one barrier: it ends every read of this transform's buffer before
        // the next first pass overwrites it, and publishes the norm's
        // per-warp partials
        r2 = warp_sum(r2);
        if (lane == 0) red2[warp] = r2;
        __syncthreads();
        const double rn_ = sqrt(xsum_nw<NW>(lane < NW ? red2[lane] : 0.0));
        adj_pass1(v);
        return rn_;
      }
      if (s_xmap && log2n >= 3) {
        __syncthreads();
        first_pass_map8<OLOGP, false, HAD>(
            buf, log2n, s_xmap,
            [&](int q) {
              V xv = zv;
              if (q >= 0) from_c128(s_x[q], xv);
              return xv;
            },
            tid, nth);
        __syncthreads();
        block_transform<ORMAX, false, HAD>(buf, log2n, tw, tid, nth, -1, 3);  // (the mapped pass did 3 bits)
      } else {
        for (int i = tid; i < nbuf; i += nth) buf[i] = zv;
        __syncthreads();
        for (int j = tid; j < cnt; j += nth) {
          V xv;
          from_c128(s_x[j], xv);
          buf[padx<OLOGP>(HAD ? (int)s_lam[j] : (int)brev_n(s_lam[j], log2n))] = xv;
        }
        __syncthreads();
        block_transform<ORMAX, false, HAD>(buf, log2n, tw, tid, nth);
      }
      double r2 = 0.0;
      if (ysl) {
        // slot order: r[k] belongs to the row in transform slot scat_pos[k],
        // y was stored in that order at t = 1; the next conventional row
        // reads r with coalesced loads (no dependent index -> value chains)
        for (int k = tid; k < m; k += nth) {
          const unsigned p = op.scat_pos[k];
          const int w = HAD ? (int)p : (int)brev_n(p, log2n);
          const V rv = sub(ysl[k], scale(buf[padx<OLOGP>(w)], sc));
          rs[k] = rv;
          r2 += mag2(rv);
        }
      } else {
        for (int j = tid; j < m; j += nth) {
          const V rv = sub(y[j], scale(buf[padx<OLOGP>((int)op.omega[j])], sc));
          rs[j] = rv;
          r2 += mag2(rv);
        }
      }
      buf_h0 = false;
      return sqrt(block_sum<NW>(r2, red));
    };

    // REFINE: the fp64 residual norm ||y - Phi_Lambda x|| (solvers.cpp:388-389)
    // summed directly over the cnt atoms, O(M t), with fp64 entries of Phi
    // (entry(), transform.cpp:154-163): halting decisions near the tolerance
    // and the reported residual_norm do not depend on fp32 rounding
    auto residual64 = [&](int cnt) -> double {
      double r2 = 0.0;
      for (int j = tid; j < m; j += nth) {
        const unsigned w = op.omega[j];
        double ar = 0.0, ai = 0.0;
        for (int q = 0; q < cnt; ++q) {
          const double2 xv = s_x[q];
          const unsigned l = s_lam[q];
          if constexpr (HAD) {
            const double sg = (__popc(w & l) & 1) ? -1.0 : 1.0;
            ar = fma(sg, xv.x, ar);
            ai = fma(sg, xv.y, ai);
          } else {
            const double2 e = op.tw64[(w * l) & (unsigned)(n - 1)];
            ar = fma(xv.x, e.x, fma(-xv.y, e.y, ar));
            ai = fma(xv.x, e.y, fma(xv.y, e.x, ai));
          }
        }
        const double2 yv = to_c128(y[j]);
        const double rr = yv.x - ar * sc, ri = yv.y - ai * sc;
        r2 += rr * rr + ri * ri;
      }
      return sqrt(block_sum<NW>(r2, red));
    };
    // REFINE: fp64 correlation h_j = h0_j - sum_tau x_tau c[(j - lambda_tau)
    // mod N] (or c[j ^ lambda_tau]), the reference's fast_update value
    // (kernel.cpp:227-261) from the fp64 h0 and kernel, one thread
    auto h64_serial = [&](unsigned j) -> double {
      double2 acc = to_c128(h0x[j]);
      for (int q = 0; q < s; ++q) {
        const double2 xv = s_x[q];
        const double2 g = gram<HAD>(op, j, s_lam[q]);
        acc.x -= xv.x * g.x - xv.y * g.y;
        acc.y -= xv.x * g.y + xv.y * g.x;
      }
      return acc.x * acc.x + acc.y * acc.y;
    };
    // |h0_j| <= ||phi_j|| ||y|| = sqrt(M/N) ||y|| bounds every correlation
    const double hy = sqrt((double)m / (double)n * yy);

    if (!(rn <= tol)) {
      for (int t = 1; t <= T; ++t) {
        const bool fast_row = t >= 2 && (int64_t)t <= a.fast_until;
        tlast = t;
        // booked like the reference's cost rows: t = 1 counts under the plan
        // (solvers.cpp:336-340) although it always runs the transform
        if (a.modes && tid == 0) a.modes[prob * T + (t - 1)] = (int64_t)t <= a.fast_until ? 1 : 0;
        V* hrow = a.hist ? reinterpret_cast<V*>(a.hist) + ((size_t)prob * T + (t - 1)) * n
                         : nullptr;
        double best = 0.0;
        double m2[RPT];
        if (REFINE && tid == 0) *s_ncand = 0;  // read after the barriers below
        mark(5);
        if (F16 && !fast_row) {
          // conventional correlation: U^H scatter(r) (sensing.cpp:102-109),
          // r in registers (t = 1: y)
          if constexpr (F16) {
            // (t >= 2: the first pass ran at the end of the previous
            // iteration's residual)
            if (t == 1) {
              const uint32_t om = op.f16_omt[tid];
              int c = (int)(om >> 16);
              V rr[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                if ((om >> j) & 1u) rr[j] = yc[c++];
                else rr[j] = zv;
              }
              __syncthreads();  // yc was written by other threads; buf may still be read
              adj_pass1(rr);
            }
            V v[16];
            f16_passes23<true, false>(buf, v, tw16, tid);
            if (t != 1 && !hrow) {
              // |h|^2 into the slot's first 8 bytes, re-read by the
              // identification scan; 1/sqrt N = 2^-6 here, so scaling |v|^2
              // by 1/N gives bitwise the |h|^2 of the scaled h
              const double s2 = sc * sc;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const double mm = mag2(v[j]) * s2;
                reinterpret_cast<double*>(buf)[2 * pad16(tid + 256 * j)] = mm;
                best = fmax(best, mm);
              }
            } else {
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                // own slots: h0 (t = 1, kept for the fast rows), else |h|^2
                const int k = tid + 256 * j;
                const V hv = scale(v[j], sc);
                const double mm = mag2(hv);
                if (t == 1) {
                  buf[pad16(k)] = hv;
                  h0w[k] = hv;
                } else {
                  reinterpret_cast<double*>(buf)[2 * pad16(k)] = mm;
                }
                if (hrow) hrow[k] = hv;
                best = fmax(best, mm);
              }
            }
            buf_h0 = t == 1;
          }
        } else if (!fast_row) {
          // conventional correlation: U^H scatter(r) (sensing.cpp:102-109)
          const V* r = t == 1 ? y : rs;
          if (s_map && log2n >= 3) {
            __syncthreads();  // buf may still be read (previous argmax / h0)
            first_pass_map8<OLOGP, true, HAD>(
                buf, log2n, s_map, [&](int q) { return q >= 0 ? r[q] : zv; }, tid, nth);
            __syncthreads();
            block_transform<ORMAX, true, HAD>(buf, log2n, tw, tid, nth, -1, 3);
          } else {
            for (int i = tid; i < nbuf; i += nth) buf[i] = zv;
            __syncthreads();
            // rows in transform-slot order (op.scat_pos ascending): the lanes'
            // stores land on increasing slots instead of bit-reversed ones
            if (!ysl) {
              for (int k = tid; k < m; k += nth) buf[padx<OLOGP>((int)op.scat_pos[k])] = r[op.scat_row[k]];
            } else if (t == 1) {
              for (int k = tid; k < m; k += nth) {
                const V v = y[op.scat_row[k]];
                ysl[k] = v;
                buf[padx<OLOGP>((int)op.scat_pos[k])] = v;
              }
            } else {
              for (int k = tid; k < m; k += nth) buf[padx<OLOGP>((int)op.scat_pos[k])] = rs[k];
            }
            __syncthreads();
            block_transform<ORMAX, true, HAD>(buf, log2n, tw, tid, nth);
          }
          if (t == 1) {
            // h0 = Phi^H y stays in buf (scaled, padded) for the fast rows
            for (int i = tid; i < nbuf; i += nth) buf[i] = scale(buf[i], sc);
            __syncthreads();
          }
          const double scv = t == 1 ? 1.0 : sc;
          for (int k = tid; k < n; k += nth) {
            const V v = scale(buf[padx<OLOGP>(k)], scv);
            if (t == 1) h0w[k] = v;
            if (hrow) hrow[k] = v;
            best = fmax(best, mag2(v));
          }
          buf_h0 = t == 1;
        } else {
          // fast correlation (kernel.cpp:209-303) from h0 and the staged c
          if (!buf_h0) {
            __syncthreads();
            for (int k = tid; k < n; k += nth) buf[bp(k)] = h0w[k];
            buf_h0 = true;
            __syncthreads();
          }
          if (ntiles) {
            for (int tile = warp; tile < ntiles; tile += nw) {
              const int i0 = tile * 32 * RPT;
              V acc[RPT];
#pragma unroll
              for (int r = 0; r < RPT; ++r) acc[r] = buf[bp(i0 + lane + 32 * r)];
              fast_tile<V, HAD, RPT, GMODE == 2>(acc, i0, lane, n, gF, gH, s_lam, s_xn, s);
#pragma unroll
              for (int r = 0; r < RPT; ++r) {
                const int i = i0 + lane + 32 * r;
                m2[r] = mag2(acc[r]);
                if (!regs_only) msc[i] = m2[r];
                best = fmax(best, m2[r]);
                if (hrow) hrow[i] = acc[r];
              }
            }
            if (regs_only && warp >= ntiles) {
#pragma unroll
              for (int r = 0; r < RPT; ++r) m2[r] = -1.0;
            }
          } else {
            for (int i = tid; i < n; i += nth) {
              V acc = buf[bp(i)];
              fast_point<V, HAD, GMODE == 2>(acc, i, n, gF, gH, s_lam, s_xn, s);
              const double mm = mag2(acc);
              msc[i] = mm;
              best = fmax(best, mm);
              if (hrow) hrow[i] = acc;
            }
          }
        }
        // identification with the tie band (solvers.cpp:90-101, :362-367)
        // `red` was last read before the least-squares pass-2 barrier (or the
        // transform's barriers at t = 1): no leading barrier needed
        const double my_best = best;  // this thread's own maximum
        best = block_max<false, NW>(best, red);
        mark(fast_row ? 1 : 0);
        if (!REFINE && best == 0.0) break;
        double cut = best * (1.0 - kTieBandRel);
        if constexpr (REFINE) {
          // fp32 correlations decide nothing by themselves: every index whose
          // fp32 |h| is within twice the rounding bound E of the fp32 maximum
          // is a candidate, re-evaluated below in fp64.  E bounds |h32 - h64|
          // by ecoef (a multiple of 2^-24 (log2 N + 2)) times the largest
          // magnitude any term of the accumulation can reach: |h0_j| <= hy,
          // the off-diagonal kernel terms goff * sum|x|, the diagonal one
          // gamma * max|x| (identical in every warp: same shuffle tree)
          double xs1 = 0.0, xmx = 0.0;
          for (int q = lane; q < s; q += 32) {
            const double2 xv = s_x[q];
            const double ax = sqrt(xv.x * xv.x + xv.y * xv.y);
            xs1 += ax;
            xmx = fmax(xmx, ax);
          }
          xs1 = warp_sum(xs1);
          xmx = warp_max(xmx);
          const double e = a.ecoef * (hy + a.goff * xs1 + gamma * xmx);
          const double lo = sqrt(best) * (1.0 - kTieBandRel) - 2.0 * e;
          cut = lo > 0.0 ? lo * lo : -1.0;  // -1: every element qualifies
        }
        // own elements with |h|^2 >= cut, ascending index; f(k) returns true to stop
        auto scan = [&](auto&& f) {
          if (!fast_row) {
            // only a thread whose own maximum (over these same indices k) reaches
            // the band can hold the pick
            const double scv = t == 1 ? 1.0 : sc;
            if (my_best >= cut)
              for (int k = tid; k < n; k += nth)
                if (mag2(scale(buf[padx<OLOGP>(k)], scv)) >= cut && f((unsigned)k)) return;
          } else if (regs_only) {
#pragma unroll
            for (int r = 0; r < RPT; ++r)
              if (warp < ntiles && m2[r] >= cut && f((unsigned)(warp * 32 * RPT + lane + 32 * r)))
                return;
          } else if (ntiles) {
            // several tiles per warp: only a thread whose own maximum reaches
            // the band re-reads its own entries, in ascending index order
            if (my_best >= cut)
              for (int tile = warp; tile < ntiles; tile += nw)
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                  const int i = tile * 32 * RPT + lane + 32 * r;
                  if (msc[i] >= cut && f((unsigned)i)) return;
                }
          } else {
            for (int k = tid; k < n; k += nth)
              if (msc[k] >= cut && f((unsigned)k)) return;
          }
        };
        unsigned pick;
        if constexpr (!REFINE) {
          unsigned first = 0xffffffffu;
          if (F16 && !fast_row) {
            if constexpr (F16) {
              if (my_best >= cut)
                for (int j = 0; j < 16; ++j) {
                  const int q = pad16(tid + 256 * j);
                  const double mm = t == 1 ? mag2(buf[q]) : reinterpret_cast<const double*>(buf)[2 * q];
                  if (mm >= cut) { first = (unsigned)(tid + 256 * j); break; }
                }
            }
          } else if (!fast_row) {
            // only a thread whose own maximum (over these same indices k) reaches
            // the band can hold the pick
            const double scv = t == 1 ? 1.0 : sc;
            if (my_best >= cut)
              for (int k = tid; k < n; k += nth)
                if (mag2(scale(buf[padx<OLOGP>(k)], scv)) >= cut) { first = (unsigned)k; break; }
          } else if (regs_only) {
#pragma unroll
            for (int r = RPT - 1; r >= 0; --r)
              if (m2[r] >= cut) first = (unsigned)(warp * 32 * RPT + lane + 32 * r);
          } else if (ntiles) {
            // several tiles per warp: only a thread whose own maximum reaches
            // the band re-reads its own entries, in ascending index order
            if (my_best >= cut)
              for (int tile = warp; tile < ntiles && first == 0xffffffffu; tile += nw)
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                  const int i = tile * 32 * RPT + lane + 32 * r;
                  if (msc[i] >= cut) { first = (unsigned)i; break; }
                }
          } else {
            for (int k = tid; k < n; k += nth)
              if (msc[k] >= cut) { first = (unsigned)k; break; }
          }
          pick = block_min_u<false, NW>(first, redu);  // redu: only used here
        } else {
          scan([&](unsigned k) {
            const int c = atomicAdd(s_ncand, 1);
            if (c < RCAP) s_cand[c] = k;
            return false;
          });
          __syncthreads();
          const int nc = *s_ncand;
          double best64;
          if (nc == 1) {
            // a single candidate is the pick: every index whose fp64 |h| is
            // within the band of the fp64 maximum passes the candidate cut
            pick = s_cand[0];
            best64 = best;  // (only its sign is used below)
          } else if (nc <= RCAP) {
            // one warp per candidate, lanes over the atoms (fixed shuffle tree)
            for (int c = warp; c < nc; c += nw) {
              const unsigned j = s_cand[c];
              double ar = 0.0, ai = 0.0;
              for (int q = lane; q < s; q += 32) {
                const double2 xv = s_x[q];
                const double2 g = gram<HAD>(op, j, s_lam[q]);
                ar = fma(xv.x, g.x, fma(-xv.y, g.y, ar));
                ai = fma(xv.x, g.y, fma(xv.y, g.x, ai));
              }
              ar = warp_sum(ar);
              ai = warp_sum(ai);
              if (lane == 0) {
                const double2 h0j = to_c128(h0x[j]);
                const double hr = h0j.x - ar, hi = h0j.y - ai;
                s_cval[c] = hr * hr + hi * hi;
              }
            }
            __syncthreads();
            // the reference's rule on the fp64 values (solvers.cpp:90-101):
            // every warp reduces the same list
            double b = 0.0;
            for (int c = lane; c < nc; c += 32) b = fmax(b, s_cval[c]);
            best64 = warp_max(b);
            const double cut64 = best64 * (1.0 - kTieBandRel);
            unsigned f = 0xffffffffu;
            for (int c = lane; c < nc; c += 32)
              if (s_cval[c] >= cut64) f = min(f, s_cand[c]);
            pick = warp_min_u(f);
          } else {
            // more candidates than the list holds: every thread evaluates its
            // own qualifying elements serially (max, then first in band)
            double b = 0.0;
            scan([&](unsigned k) { b = fmax(b, h64_serial(k)); return false; });
            best64 = block_max<true, NW>(b, red);
            const double cut64 = best64 * (1.0 - kTieBandRel);
            unsigned f = 0xffffffffu;
            scan([&](unsigned k) {
              if (h64_serial(k) >= cut64) { f = k; return true; }
              return false;
            });
            pick = block_min_u<true, NW>(f, redu);
          }
          if (a.rstats && tid == 0) {
            atomicAdd(a.rstats, 1ull);
            atomicAdd(a.rstats + 1, (unsigned long long)nc);
            if (nc > RCAP) atomicAdd(a.rstats + 2, 1ull);
          }
          if (best64 == 0.0) break;
        }
        if (pick >= (unsigned)n) break;  // no candidate (cannot happen: the maximum is in band)
        // stagnation guard (solvers.cpp:365-367): selected-atom bitmap, no barrier
        if ((s_sel[pick >> 5] >> (pick & 31)) & 1u) break;
        // b_s = h0[pick], read early so its latency hides behind the row pass
        // (REFINE: the fp64 h0)
        const V bpre = REFINE ? zv : (buf_h0 ? buf[bp((int)pick)] : h0w[pick]);
        const double2 bpre64 = REFINE ? to_c128(h0x[pick]) : make_double2(0.0, 0.0);
        mark(2);

        // ---- least squares: append one Gram row to W = L^{-1} (G = L L^H).
        // l = W a with a_j = G(lambda_j, pick) looked up in c.  Eight threads
        // per row (lane group q = tid % 8 sums j = q, q+8, ...), reduced with
        // three shuffles, so all 512 threads share the O(s^2) work; the same
        // pass accumulates |l|^2 and l^H z into per-warp partials
        double ll = 0.0, lzr = 0.0, lzi = 0.0;
        for (int base = 0; base < s; base += nth / LSG) {
          const int i = base + tid / LSG, q = tid % LSG;
          double ar = 0.0, ai = 0.0;
          // wat(j) = W(i, j)
          auto dot_row = [&](auto&& wat) {
            for (int j0 = q; j0 <= i; j0 += LSG * LSU) {
              // fixed-size predicated chunk: all loads issue before the FMAs
              double2 w[LSU], v[LSU];
#pragma unroll
              for (int u = 0; u < LSU; ++u) {
                const int j = j0 + LSG * u;
                if (j <= i) {
                  w[u] = wat(j);
                  v[u] = gram_of(s_lam[j], pick);
                } else {
                  w[u] = make_double2(0.0, 0.0);
                  v[u] = w[u];
                }
              }
#pragma unroll
              for (int u = 0; u < LSU; ++u) {
                ar = fma(w[u].x, v[u].x, fma(-w[u].y, v[u].y, ar));
                ai = fma(w[u].x, v[u].y, fma(w[u].y, v[u].x, ai));
              }
            }
          };
          if (i < s) {
            if constexpr (F16) {
              // (two call sites: shared and global loads stay distinct)
              if (i < R0) {
                const double2* Wr = Ws + tri(i);
                dot_row([&](int j) { return Wr[j]; });
              } else {
                const double2* Wr = Wg + tri(i);
                dot_row([&](int j) { return Wr[j]; });
              }
            } else {
              dot_row([&](int j) { return W[wofs(T, i, j)]; });
            }
          }
#pragma unroll
          for (int o = LSG / 2; o; o >>= 1) {
            ar += __shfl_xor_sync(0xffffffffu, ar, o);
            ai += __shfl_xor_sync(0xffffffffu, ai, o);
          }
          if (i < s && q == 0) {
            s_l[i] = make_double2(ar, ai);
            const double2 zc = s_z[i];
            ll += ar * ar + ai * ai;
            lzr += ar * zc.x + ai * zc.y;  // conj(l) z
            lzi += ar * zc.y - ai * zc.x;
          }
        }
        ll = warp_sum(ll);
        lzr = warp_sum(lzr);
        lzi = warp_sum(lzi);
        if (lane == 0) {
          red[warp] = ll;
          red[32 + warp] = lzr;
          red[64 + warp] = lzi;
        }
        __syncthreads();  // publishes s_l and the partials
        // every warp reduces the nw partials with the same shuffle tree, so
        // every thread holds the bitwise-same sums
        ll = lane < nw ? red[lane] : 0.0;
        lzr = lane < nw ? red[32 + lane] : 0.0;
        lzi = lane < nw ? red[64 + lane] : 0.0;
        ll = xsum_nw<NW>(ll);
        lzr = xsum_nw<NW>(lzr);
        lzi = xsum_nw<NW>(lzi);
        const double d2 = gamma - ll;
        // pivot floor as the reference's normal-equations path
        // (solvers.cpp:32,144); see DESIGN.md for the QR criterion
        if (!(d2 > 1e-12 * gamma)) { aborted = 1; break; }
        // one reciprocal square root instead of a sqrt and per-element
        // divisions (fp64 division / sqrt are long software sequences)
        const double invd = rsqrt(d2);
        const double2 bnew = REFINE ? bpre64 : to_c128(bpre);
        const double2 znew = make_double2((bnew.x - lzr) * invd, (bnew.y - lzi) * invd);
        // new row of W, one pass per column j < s (eight threads each; column
        // j of the packed W is contiguous): W_sj = -(1/d) sum_{i=j}^{s-1}
        // conj(l_i) W_ij.  Older rows never change, so x = W^H z only gains
        // the new term: x_j += conj(W_sj) z_s
        for (int base = 0; base < s; base += nth / LSG) {
          const int j = base + tid / LSG, q = tid % LSG;
          double ar = 0.0, ai = 0.0;
          if (j < s) {
            const double2* Wc = W + wofs(T, j, j);
            for (int i0 = j + q; i0 < s; i0 += LSG * LSU) {
              double2 l[LSU], w[LSU];
#pragma unroll
              for (int u = 0; u < LSU; ++u) {
                const int i = i0 + LSG * u;
                if (i < s) {
                  l[u] = s_l[i];
                  if constexpr (F16) {
                    if (i < R0) w[u] = Ws[tri(i) + j];
                    else w[u] = Wg[tri(i) + j];
                  } else {
                    w[u] = Wc[i - j];
                  }
                } else {
                  l[u] = make_double2(0.0, 0.0);
                  w[u] = l[u];
                }
              }
#pragma unroll
              for (int u = 0; u < LSU; ++u) {
                ar = fma(l[u].x, w[u].x, fma(l[u].y, w[u].y, ar));  // conj(l) w
                ai = fma(l[u].x, w[u].y, fma(-l[u].y, w[u].x, ai));
              }
            }
          }
#pragma unroll
          for (int o = LSG / 2; o; o >>= 1) {
            ar += __shfl_xor_sync(0xffffffffu, ar, o);
            ai += __shfl_xor_sync(0xffffffffu, ai, o);
          }
          if (j < s && q == 0) {
            const double2 wn = make_double2(-ar * invd, -ai * invd);
            if constexpr (F16) (s < R0 ? Ws : Wg)[tri(s) + j] = wn;
            else W[wofs(T, s, j)] = wn;
            const double2 xo = s_x[j];
            const double xr = xo.x + wn.x * znew.x + wn.y * znew.y;
            const double xi = xo.y + wn.x * znew.y - wn.y * znew.x;
            s_x[j] = make_double2(xr, xi);
            from_c128(make_double2(xr * xscale, xi * xscale), s_xn[j]);
          }
        }
        if (tid == 0) {
          if constexpr (F16) (s < R0 ? Ws : Wg)[tri(s) + s] = make_double2(invd, 0.0);
          else W[wofs(T, s, s)] = make_double2(invd, 0.0);
          s_z[s] = znew;
          s_lam[s] = pick;
          s_sel[pick >> 5] |= 1u << (pick & 31);
          if (s_xmap) s_xmap[HAD ? (int)pick : (int)brev_n(pick, log2n)] = (int16_t)s;
          if constexpr (F16) {
            const int g = (int)(brev_n(pick, log2n) >> 4);
            s_next[s] = s_head[g];
            s_head[g] = (int16_t)s;
          }
          const double2 xs = make_double2(znew.x * invd, znew.y * invd);
          s_x[s] = xs;
          from_c128(make_double2(xs.x * xscale, xs.y * xscale), s_xn[s]);
        }
        zz += znew.x * znew.x + znew.y * znew.y;
        ++s;
        __syncthreads();
        iters = t;
        mark(3);

        // ---- residual and halting (solvers.cpp:388-402)
        const bool next_conv = t < T && !((int64_t)(t + 1) <= a.fast_until);
        const double r2id = yy - zz;  // ||y||^2 - ||P y||^2
        if constexpr (REFINE) {
          // halting on fp64 values: the identity (b = fp64 h0, LS in fp64)
          // unless it is within 1e-10 ||y||^2 of tol^2, then the direct fp64
          // residual; an fp32 r is formed only to feed a conventional row
          if (next_conv) residual_explicit(s);
          bool halt;
          rn_explicit = fabs(r2id - tol * tol) <= 1e-10 * yy;  // (rn64 of this state)
          if (rn_explicit) {
            rn = residual64(s);
            halt = rn <= tol;
          } else {
            halt = r2id <= tol * tol;
          }
          mark(4);
          if (halt) break;
        } else {
          const bool near = !(r2id > tol * tol + a.margin * yy);
          if (next_conv || near) {
            rn = residual_explicit(s);
            rn_explicit = true;
          } else {
            rn = sqrt(fmax(r2id, 0.0));
            rn_explicit = false;
          }
          mark(4);
          if (rn_explicit && rn <= tol) break;
        }
      }
      if (REFINE) {
        // the fp64 identity where it resolves ||r|| to ~1e-10 relative, else
        // the direct fp64 residual
        const double r2id = yy - zz;
        if (!rn_explicit) rn = r2id > 1e-6 * yy ? sqrt(r2id) : residual64(s);
      } else if (!rn_explicit) {
        rn = residual_explicit(s);
      }
      mark(4);
    }
    // ---- results (RecoveryResult, solvers.hpp:53-64)
    uint64_t* sup = a.support + prob * T;
    double2* co = a.coeffs + prob * T;
    for (int j = tid; j < T; j += nth) {
      sup[j] = j < s ? (uint64_t)s_lam[j] + 1 : 0;
      co[j] = j < s ? s_x[j] : make_double2(0.0, 0.0);
      if (a.modes && j >= tlast) a.modes[prob * T + j] = 0;  // rows never run
    }
    if (tid == 0) {
      a.size[prob] = (uint64_t)s;
      a.iters[prob] = (uint64_t)iters;
      a.resid[prob] = rn;
      a.aborted[prob] = aborted;
      if (a.hlen) a.hlen[prob] = (uint64_t)tlast;
    }
  }
}

struct OmpPlan {
  size_t total;
  int gmode;
  bool rsm, wsm, bufg, msm;
  int wrows;  // F16: rows of W in shared memory (wsm: at least one)
  int off_g, off_r, off_w, off_tw, off_small, off_map, tw_a;
};

// the F16 conventional rows apply (config 2's two-CTA solver)
template <class V, bool HAD>
constexpr bool f16_type() { return !HAD && sizeof(V) == 16; }
template <class V, bool HAD>
bool f16_ok(const DevOp& op) {
  return !HAD && sizeof(V) == 16 && op.n == 4096 && op.f16_omt && op.f16_yidx;
}

template <class V, bool HAD>
OmpPlan omp_plan(const DevOp& op, int64_t T, int ctas, bool f16 = false, bool conv_heavy = false) {
  OmpPlan p{};
  const int64_t n = op.n, m = op.m;
  auto al = [](size_t b) { return ((b + 15) / 16) * 16; };
  const size_t buf = f16 ? al((size_t)(n + n / 16 + n / 512) * sizeof(V))
                         : al((size_t)(n + (n >> ologp_v<V>())) * sizeof(V));
  const size_t gfull = al(HAD ? (size_t)n * 2 : (size_t)n * sizeof(V));
  const size_t ghalf = al((size_t)(n / 2 + 1) * sizeof(V));
  const size_t r = al((size_t)m * sizeof(V));
  const size_t w = al((size_t)T * (T + 1) / 2 * 16);
  p.tw_a = (op.log2n + 1) / 2;
  // two-level twiddle tables, each padded i + i/8 (TwTwoLevel)
  const size_t lo_n = ((size_t)1 << p.tw_a) + ((size_t)1 << p.tw_a) / 8 + 1;
  const size_t hi_n = ((size_t)n >> p.tw_a) + ((size_t)n >> p.tw_a) / 8 + 1;
  // (F16: 64 + 4 two-level entries, unpadded)
  const size_t tw = HAD ? 0 : (f16 ? al((size_t)68 * sizeof(V)) : al((lo_n + hi_n) * sizeof(V)));
  const size_t small = al(3 * 16 * (size_t)T) + al(sizeof(V) * (size_t)T) + al(4 * (size_t)T) +
                       al(4 * (size_t)((n + 31) / 32)) +
                       (sizeof(typename scal<V>::T) == 4 ? (size_t)12 * RCAP + 16 : 0) +
                       (f16 ? al(2 * (size_t)(n / 16)) + al(2 * (size_t)T) : 0);
  // ctas > 1: the SM's shared memory (optin + 1 KB) split between the CTAs,
  // less each CTA's 1 KB reservation and the kernel's static shared memory
  // (1936 bytes; omp_ctas_v confirms the residency with the occupancy API)
  const size_t cap = ctas == 1 ? (size_t)smem_optin() - 2048
                               : ((size_t)smem_optin() + 1024) / ctas - 1024 - 1952;
  size_t tot = tw + small;
  // the transform buffer has first claim on smem (a global-memory buffer
  // sends every transform pass through L2); the kernel table follows and
  // falls back to global memory (GMODE 0) when it does not fit beside it
  const size_t gmin = HAD ? gfull : ghalf;
  p.bufg = tot + buf > cap;
  if (!p.bufg) tot += buf;
  // W next: the least-squares phase is latency bound.  F16 leaves the kernel
  // table in global memory (read through L1 by the fast rows and the Gram
  // lookups); the problem's measurements (16 KB, read by every residual)
  // come first and W takes what is left, by rows: the leading rows - read by
  // every later iteration - in shared memory, the last ones in the CTA's
  // global workspace (config 2: rows 0..47 of 64).  Measured on config 2:
  // y in smem / W in L2 308 k, W in smem / y in L2 322 k recoveries/s (the
  // residual then waits ~10 % of the time on its measurements)
  const char* gs = getenv("FMP_F16_GSMEM");
  const bool f16g = f16 && !(gs && atoi(gs) == 1);  // F16 with the table in global memory
  size_t wbytes = w;
  p.wrows = 0;
  if (f16g) {
    p.rsm = tot + r <= cap;
    if (p.rsm) tot += r;
    int R = (int)T;
    auto trib = [&](int rr) { return al((size_t)rr * (rr + 1) / 2 * 16); };
    if (tot + trib(R) > cap) {
      R &= ~7;
      while (R > 0 && tot + trib(R) > cap) R -= 8;
    }
    const char* wr = getenv("FMP_F16_WROWS");  // timing tools: cap the rows kept in smem
    if (wr && atoi(wr) >= 0 && atoi(wr) < R) R = atoi(wr) & ~7;
    p.wrows = R;
    p.wsm = R > 0;
    wbytes = trib(R);
  } else {
    p.wsm = tot + w + gmin <= cap;
  }
  if (p.wsm) tot += wbytes;
  p.gmode = 0;
  // A solve that is mostly conventional rows (fast rows for fewer than half
  // of its iterations) gets the slot maps before the kernel table and r:
  // its rows then skip the zero fill and the scatter / gather through L2
  // (config 4 c64: table 36.4 k, r 37.3 k, maps 38.4 k recoveries/s).
  // FMP_OMP_PLAN (timing tools): "g" the table first whatever the mode, "r"
  // no table (room for r), "m" neither (room for the maps)
  const char* pe = getenv("FMP_OMP_PLAN");
  const size_t mapb = 2 * al((size_t)((n + 7) / 8) * 8 * 2);  // row map + support map
  const bool maps_ok = !f16 && !p.bufg && m <= 32767 && T <= 32767;
  const bool maps_first = maps_ok && tot + mapb <= cap &&
                          ((conv_heavy && !(pe && (pe[0] == 'g' || pe[0] == 'r'))) || (pe && pe[0] == 'm'));
  p.msm = maps_first;
  if (p.msm) tot += mapb;
  const bool no_g = pe && (pe[0] == 'r' || pe[0] == 'm'), no_r = pe && pe[0] == 'm';
  if (!(HAD && !op.glat) && !f16g && !no_g) {
    if (tot + gfull <= cap) { p.gmode = 1; tot += gfull; }
    else if (!HAD && tot + ghalf <= cap) { p.gmode = 2; tot += ghalf; }
    // several CTAs per SM: the conjugate half stays in global memory, where
    // the L1 left beside the CTAs' shared memory keeps it resident
  }
  if (!f16g) {
    p.rsm = !no_r && tot + r <= cap;
    if (p.rsm) tot += r;
  }
  if (!p.msm) {
    p.msm = maps_ok && tot + mapb <= cap;
    if (p.msm) tot += mapb;
  }
  p.total = tot;
  size_t off = p.bufg ? 0 : buf;
  p.off_tw = (int)off; off += tw;
  p.off_w = (int)off; if (p.wsm) off += wbytes;
  p.off_g = (int)off; off += p.gmode == 1 ? gfull : (p.gmode == 2 ? ghalf : 0);
  p.off_r = (int)off; if (p.rsm) off += r;
  p.off_map = (int)off; if (p.msm) off += mapb;
  p.off_small = (int)off;
  return p;
}

template <class V, bool HAD, int RPT, int GMODE, bool BUFG, int NT, int CT, bool F16 = false>
void launch_k(const OmpK& k, int grid, size_t smem, cudaStream_t st) {
  auto f = k_omp<V, HAD, RPT, GMODE, BUFG, NT, CT, F16>;
  // the attribute is per device and only grows: set it when a launch needs
  // more than this instantiation was last given (saves a driver call per
  // launch in the latency regime)
  static std::atomic<int> set_smem[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& cur = set_smem[dev & 63];
  if ((int)smem > cur.load(std::memory_order_relaxed)) {
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cur.store((int)smem, std::memory_order_relaxed);
  }
  f<<<grid, NT, smem, st>>>(k);
}

template <class V, bool HAD, int RPT, bool BUFG, int NT, int CT, bool F16 = false>
void launch_g(const OmpK& k, int gmode, int grid, size_t smem, cudaStream_t st) {
  if (gmode == 1) launch_k<V, HAD, RPT, 1, BUFG, NT, CT, F16>(k, grid, smem, st);
  else if (!HAD && gmode == 2) launch_k<V, HAD, RPT, 2, BUFG, NT, CT, F16>(k, grid, smem, st);
  else launch_k<V, HAD, RPT, 0, BUFG, NT, CT, F16>(k, grid, smem, st);
}

template <class V, bool HAD, int RPT, int NT, int CT, bool F16 = false>
cudaError_t launch_omp_t(const OmpArgs& a, cudaStream_t st) {
  const DevOp& op = *a.op;
  const OmpPlan p = omp_plan<V, HAD>(op, a.max_iter, CT, F16, a.fast_until * 2 < a.max_iter);
  if (p.total > (size_t)smem_optin() - 2048) return cudaErrorInvalidConfiguration;
  OmpK k{};
  k.op = op;
  k.y = a.y;
  k.tol = a.tol;
  k.batch = a.batch;
  k.T = (int)a.max_iter;
  k.fast_until = a.fast_until;
  k.support = a.support;
  k.coeffs = a.coeffs;
  k.size = a.size;
  k.iters = a.iters;
  k.hlen = a.hlen;
  k.resid = a.resid;
  k.aborted = a.aborted;
  k.modes = a.modes;
  k.hist = a.hist;
  k.w_ws = a.w_ws;
  k.h0_ws = a.h0_ws;
  k.mag_ws = a.mag_ws;
  k.r_ws = a.r_ws;
  k.ys_ws = p.msm ? nullptr : a.ys_ws;
  k.queue = a.queue;
  k.r_smem = p.rsm;
  k.w_smem = p.wsm;
  k.w_rows = p.wrows;
  k.map_smem = p.msm;
  k.off_map = p.off_map;
  k.buf_ws = a.buf_ws;
  if (p.bufg && !a.buf_ws) return cudaErrorInvalidValue;
  k.off_g = p.off_g;
  k.off_r = p.off_r;
  k.off_w = p.off_w;
  k.off_tw = p.off_tw;
  k.off_small = p.off_small;
  k.tw_a = p.tw_a;
  k.margin = is_double(a.dtype) ? 1e-10 : 1e-5;
  k.phase_ws = a.phase_ws;
  k.ready = a.ready;
  k.ready_chunk = a.ready_chunk;
  k.abort_word = a.abort_word;
  k.h0x = a.h0x;
  k.goff = op.goff;
  k.rstats = a.rstats;
  if (sizeof(typename scal<V>::T) == 4) {
    if (!a.h0x) return cudaErrorInvalidValue;
    // fp32 rounding bound coefficient: 8 x 2^-24 per transform level (+2)
    k.ecoef = 8.0 * 0x1p-24 * (double)(op.log2n + 2);
  }
  const int grid = std::max(1, a.grid);
  if constexpr (CT == 1) {
    if (p.bufg) launch_g<V, HAD, RPT, true, NT, CT>(k, p.gmode, grid, p.total, st);
    else launch_g<V, HAD, RPT, false, NT, CT>(k, p.gmode, grid, p.total, st);
  } else {
    if (p.bufg) return cudaErrorInvalidConfiguration;
    if constexpr (F16) {
      if (!a.ys_ws || p.msm) return cudaErrorInvalidValue;
      k.ys_ws = a.ys_ws;
    }
    launch_g<V, HAD, RPT, false, NT, CT, F16>(k, p.gmode, grid, p.total, st);
  }
  ++g_launches;
  return cudaGetLastError();
}

// Two resident CTAs of 256 threads per SM (two problems in flight: one's
// latency-bound identification / least-squares phases overlap the other's
// transforms) when both transform buffers fit in shared memory and the batch
// fills them; measured on config 2 (B200): 239 k against 227 k recoveries/s at
// the best switch point of each.  Fourier only (the Hadamard lattice path
// keeps its kernel table in shared memory).
// FMP_OMP_F16=0: the radix-8 conventional rows in the two-CTA solver too
// (timing comparisons)
inline bool omp_f16_off() {
  const char* e = getenv("FMP_OMP_F16");
  return e && atoi(e) == 0;
}

template <class V, bool HAD>
int omp_ctas_v(const DevOp& op, int64_t batch, int64_t T) {
  const char* e = getenv("FMP_OMP_CTAS");
  if (e && atoi(e) == 1) return 1;
  if (HAD || sizeof(V) < 8 || op.n < 32 * 8 * 8) return 1;
  if (batch < 2 * (int64_t)num_sms()) return 1;
  const bool f16 = f16_ok<V, HAD>(op) && !omp_f16_off();
  const OmpPlan p = omp_plan<V, HAD>(op, T, 2, f16);
  if (p.bufg) return 1;
  // the plan must really leave two CTAs resident
  int occ = 0;
  auto f = p.gmode == 2 ? k_omp<V, HAD, 8, 2, false, 256, 2> : k_omp<V, HAD, 8, 0, false, 256, 2>;
  if constexpr (f16_type<V, HAD>())
    if (f16) f = p.gmode == 2 ? k_omp<V, HAD, 8, 2, false, 256, 2, true> : k_omp<V, HAD, 8, 0, false, 256, 2, true>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.total);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f, 256, p.total);
  return occ >= 2 ? 2 : 1;
}

// the configuration launch_omp_v picks: CTAs per SM, threads per CTA, kernel
// table mode (0 global, 1 smem full, 2 smem conjugate half), buffer in global
template <class V, bool HAD>
void omp_info_v(const DevOp& op, int64_t batch, int64_t T, int* out4) {
  int ctas = 1;
  if constexpr (!HAD && sizeof(V) >= 8) ctas = omp_ctas_v<V, HAD>(op, batch, T);
  int nt = ctas == 2 ? 256 : OMP_THREADS;
  const char* e = getenv("FMP_OMP_NT");
  if (ctas == 1 && op.n == 32 * 8 * 4 && batch <= num_sms() && !(e && atoi(e) == 512)) nt = 128;
  const OmpPlan p = omp_plan<V, HAD>(op, T, ctas, ctas == 2 && f16_ok<V, HAD>(op) && !omp_f16_off());
  out4[0] = ctas;
  out4[1] = nt;
  out4[2] = p.gmode;
  out4[3] = p.bufg ? 1 : 0;
}

template <class V, bool HAD>
cudaError_t launch_omp_v(const OmpArgs& a, cudaStream_t st) {
  if constexpr (!HAD && sizeof(V) >= 8) {
    if (omp_ctas_v<V, HAD>(*a.op, a.batch, a.max_iter) == 2) {
      if constexpr (f16_type<V, HAD>())
        if (f16_ok<V, HAD>(*a.op) && !omp_f16_off()) return launch_omp_t<V, HAD, 8, 256, 2, true>(a, st);
      return launch_omp_t<V, HAD, 8, 256, 2>(a, st);
    }
  }
  // latency regime (no more problems than SMs) at n = 1024: one 4-warp CTA
  // per problem, whose block-wide barriers and reductions are cheaper than
  // those of 16 warps (config 1: 75.8 -> 65.9 us per recovery)
  if (a.op->n == 32 * 8 * 4 && a.batch <= num_sms()) {
    // FMP_OMP_NT=512 / 256: the 16- / 8-warp CTA (timing tools)
    const char* e = getenv("FMP_OMP_NT");
    if (e && atoi(e) == 256) return launch_omp_t<V, HAD, 4, 256, 1>(a, st);
    if (!(e && atoi(e) == 512)) return launch_omp_t<V, HAD, 8, 128, 1>(a, st);
  }
  // lanes own RPT outputs; pick RPT so that one tile per warp covers n
  constexpr int NW = OMP_THREADS / 32;
  if (a.op->n >= 32 * 8 * NW && OMP_THREADS <= 512) return launch_omp_t<V, HAD, 8, OMP_THREADS, 1>(a, st);
  if (a.op->n >= 32 * 4 * NW) return launch_omp_t<V, HAD, 4, OMP_THREADS, 1>(a, st);
  return launch_omp_t<V, HAD, 2, OMP_THREADS, 1>(a, st);
}

}  // namespace
}  // namespace fmp
