// Kernel launch interface shared by the C ABI (fmp_capi.cu) and the kernels
// (fmp_kernels.cu).  Plain structs of device pointers; no torch types.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fmp {

enum Kind { FOURIER = 0, HADAMARD = 1 };
enum DType { C128 = 0, C64 = 1, F64 = 2, F32 = 3 };

inline int elem_bytes(int dt) { return dt == C128 ? 16 : (dt == F32 ? 4 : 8); }
inline bool is_complex(int dt) { return dt == C128 || dt == C64; }
inline bool is_double(int dt) { return dt == C128 || dt == F64; }

// Device-resident operator Phi = S_Omega U (sensing.hpp:39-66) plus its
// correlation kernel c = Phi^H Phi e_1 (kernel.hpp:31-40) in every storage
// form the kernels read.
struct DevOp {
  int kind = 0;
  int log2n = 0;
  int64_t n = 0, m = 0;
  uint32_t* omega = nullptr;  // m, 0-based rows, ascending
  double2* tw64 = nullptr;    // n twiddles exp(-2 pi i k / n) (Fourier)
  float2* tw32 = nullptr;
  double2* g64 = nullptr;     // c, n entries, fp64 (Fourier: exact conj symmetry)
  float2* g32 = nullptr;      // c rounded to c64 (Fourier)
  double* gr64 = nullptr;     // c real part (Hadamard), exact k/N
  uint16_t* glat = nullptr;   // Hadamard lattice N*c + 32768 (|N c| <= M); null if M > 32767
  double goff = 0.0;          // max over k != 0 of |c_k| (fp32 rounding bounds)
  // Omega scatter sorted by transform slot (slot = brev(row) Fourier, row
  // Hadamard): the large-n transform's blocks find their rows by bisection
  uint32_t* scat_pos = nullptr;  // m, ascending slots
  uint32_t* scat_row = nullptr;  // m, index into the m-vector for each slot
  uint32_t* scat_off = nullptr;  // n/256 + 1: number of slots below 256 i (n >= 256)
  // the fused solver's F16 rows (Fourier, n = 4096; fmp_omp_impl.cuh): per
  // thread u < 256 the rows u + 256 j in Omega (mask) and the count of such
  // rows of threads < u (off << 16), and each row's place in that order
  uint32_t* f16_omt = nullptr;   // 256
  uint16_t* f16_yidx = nullptr;  // m
  // two-pass transform (n = N1 N2, N1 = 2^fs_l1; fmp_transform_4s.cu), n >= 2^18:
  // Omega sorted by column (pos mod N2) for the pass-A scatter and by output
  // row k1 for the pass-B gather, each with per-column / per-row offsets
  int fs_l1 = 0;
  uint32_t* fs_aoff = nullptr;  // N2 + 1
  uint32_t* fs_apos = nullptr;  // m
  uint32_t* fs_arow = nullptr;  // m
  uint32_t* fs_boff = nullptr;  // N1 + 1
  uint32_t* fs_bpos = nullptr;  // m
  uint32_t* fs_brow = nullptr;  // m
  // one-pass Hadamard adjoint for n beyond one CTA (fmp_transform_fold.cu):
  // for block size B = 2^(11+q), Omega's rows ordered by (row g of 32 within
  // the block, position j in the row, input block ih), packed
  // m | ih << 20 | j << 26, with B/32 + 1 per-row offsets; null if unused
  uint32_t* fold_tab[4] = {};
  uint32_t* fold_off[4] = {};
  // Hadamard, n >= 2^12: Omega as a bitmap with running counts, per word w of
  // 32 positions {mask of the positions in Omega, number of Omega's rows
  // below 32 w}: a row of 32 inputs is r[rank .. rank + popc(mask)) (Omega is
  // ascending), which the register fold walks without any table
  uint2* om_wr = nullptr;  // n / 32
};

struct TransformArgs {
  const DevOp* op;  // host copy of the device op (pointers are device)
  int dtype;
  int inverse;      // 1: adjoint U^H, 0: forward U
  int in_omega;     // 1: input is m values scattered at Omega, 0: dense n
  int out_omega;    // 1: output gathered at Omega (m values), 0: dense n
  const void* in;
  void* out;        // may be null when only the argmax is wanted
  int64_t batch;
  uint64_t* argmax_out;  // optional: band argmax of |out|^2 per vector (dense out only)
  void* work;            // batch x n scratch, required when n > transform_max_n(dtype)
  int* sync;             // 32 + batch ints of scratch (job-queue path), optional
};

// two-pass transform of `batch` vectors (see fmp_transform_4s.cu)
struct FsTransform {
  const DevOp* op;
  int dtype;
  int inverse;
  int in_mode;              // 0 dense n, 1 m values at Omega, 2 sparse (lam, xs; batch 1)
  const void* in;
  const uint32_t* lam;      // in_mode 2: 0-based positions
  const double2* xs;        // in_mode 2: values (fp64); positions 0xffffffff are skipped
  int cnt;
  void* mid;                // batch x n scratch
  int out_mode;             // 0 dense n, 1 gathered at Omega (m)
  void* out;
  int64_t batch;
};

struct FastUpdateArgs {
  const DevOp* op;
  int dtype;
  const void* h0;           // batch x n
  const uint32_t* support;  // batch x t, 0-based atoms
  const void* coeffs;       // batch x t, data dtype
  int64_t t;
  int64_t batch;
  void* h_out;              // optional batch x n
  uint64_t* argmax_out;     // optional batch
  double* mag_ws;           // workspace (grid x n doubles) for the argmax
  int grid;
};

struct ArgmaxArgs {
  int dtype;
  const void* h;
  int64_t n, batch;
  uint64_t* out;
};

struct OmpArgs {
  const DevOp* op;
  int dtype;
  const void* y;            // batch x m (data dtype)
  const double* tol;        // batch absolute tolerances
  int64_t batch;
  int64_t max_iter;         // T
  int64_t fast_until;       // iterations t <= fast_until (t >= 2) use the fast update
  // outputs
  uint64_t* support;        // batch x T, 1-based atoms in selection order, 0 padded
  double2* coeffs;          // batch x T
  uint64_t* iters;          // batch (iterations_run)
  uint64_t* size;           // batch (support size)
  uint64_t* hlen;           // batch (correlation vectors computed), optional
  double* resid;            // batch
  int32_t* aborted;         // batch
  uint8_t* modes;           // batch x T (1 fast, 0 conventional), optional
  void* hist;               // batch x T x n (data dtype), optional
  // workspace, per resident CTA
  double2* w_ws;            // grid x T(T+1)/2
  void* h0_ws;              // grid x n (data dtype)
  double* mag_ws;           // grid x n
  void* r_ws;               // grid x m (data dtype) when r is not in smem
  void* ys_ws;              // grid x m (data dtype): y in transform-slot order (no smem maps)
  void* buf_ws;             // grid x (n + n/8) (data dtype): transform buffer when n exceeds smem
  int* queue;               // work counter (zeroed before launch)
  int grid;
  unsigned long long* phase_ws;  // optional per-phase cycle totals (6)
  // streamed input (optional): problem b may be read once ready[b / ready_chunk]
  // != 0 (set by the copy stream after the chunk's host-to-device copy)
  const int* ready;
  int64_t ready_chunk;
  const volatile int* abort_word;  // device view of the host's abort word (streamed input)
  // fp32 data: fp64 h0 = Phi^H y per problem (batch x n, c128 / f64; the
  // identification and the least-squares right-hand side are decided in fp64)
  const void* h0x;
  unsigned long long* rstats;  // optional: identifications, candidates, overflows
};

struct CosArgs {
  const DevOp* op;
  int dtype;
  const void* y;            // batch x m
  const double* tol;        // batch
  int64_t batch, max_iter, k;
  int fast;
  uint64_t* support;        // batch x k
  double2* coeffs;          // batch x k
  uint64_t* size;
  uint64_t* iters;
  double* resid;
  int32_t* aborted;
  uint64_t* hist_sup;       // batch x T x k, optional
  void* hist;               // batch x T x n, optional
  double* mag_ws;           // grid x n
  void* h0_ws;              // grid x n
  double2* L_ws;            // grid x (3k)^2
  void* r_ws;               // grid x m
  int* queue;
  int grid;
  unsigned long long* phase_ws;
  const int* ready;         // optional streamed-input flags (as OmpArgs)
  int64_t ready_chunk;
  const volatile int* abort_word;
};

// launchers (return cudaError_t); all async on `stream`
cudaError_t launch_transform(const TransformArgs& a, cudaStream_t stream);
cudaError_t launch_transform_fs(const FsTransform& t, cudaStream_t stream);
// Hadamard adjoint of m values at Omega, n beyond one CTA: one pass, no
// intermediate (fmp_transform_fold.cu); cudaErrorNotSupported if not applicable
cudaError_t launch_wht_fold(const TransformArgs& a, cudaStream_t stream);
int fs_split(int log2n);  // N1 = 2^fs_split rows of the two-pass transform, 0: not used
cudaError_t launch_fast_update(const FastUpdateArgs& a, cudaStream_t stream);
cudaError_t launch_argmax(const ArgmaxArgs& a, cudaStream_t stream);
cudaError_t launch_kernel_finish(const DevOp& op, cudaStream_t stream);
// max over k != 0 of |c_k| into *out (zeroed by the launcher)
cudaError_t launch_gmax_off(const DevOp& op, unsigned long long* out, cudaStream_t stream);
// widen fp32 values to fp64 (count scalars)
cudaError_t launch_widen(const float* in, double* out, int64_t count, cudaStream_t stream);
cudaError_t launch_twiddles(const DevOp& op, cudaStream_t stream);
cudaError_t launch_omp(const OmpArgs& a, cudaStream_t stream);
cudaError_t launch_cosamp(const CosArgs& a, cudaStream_t stream);
// resident CTA count the OMP launcher will use (sizes the workspaces)
int omp_grid(const DevOp& op, int dtype, int64_t batch, int64_t max_iter);
// resident fused-solver CTAs per SM for this launch (1 or 2) and the switch
// point of FMP_MODE_GPU for it
int omp_ctas(const DevOp& op, int dtype, int64_t batch, int64_t max_iter);
int omp_gpu_fast_until(const DevOp& op, int dtype, int64_t batch, int64_t max_iter);
// {CTAs per SM, threads per CTA, kernel-table mode, buffer in global memory}
void omp_info(const DevOp& op, int dtype, int64_t batch, int64_t max_iter, int* out4);
int fast_update_grid(const DevOp& op, int dtype, int64_t batch);
// largest n the smem-resident transform handles for this element size
int64_t transform_max_n(int dtype);
// least squares for a fixed support (batch problems, s atoms each, 0-based):
// x (batch x s), bad[b] = dependent position or -1; L scratch grid x s x s
cudaError_t launch_least_squares(const DevOp& op, int dtype, const void* y, const uint32_t* sup,
                                 int s, int64_t batch, double2* x, int64_t* bad, double2* L,
                                 int grid, cudaStream_t st);
// ---- sharded single-signal solver (fmp_large.cu; config 5).  Shard p of P
// owns the correlation entries k = p + P k' (cyclic), k' < np = n / P.
constexpr int LG_RC = 64;         // candidates per shard carried in an exchange record
constexpr int LG_LCAP = 1 << 16;  // candidates a shard evaluates in fp64 per identification
struct LgCand {
  uint64_t j;    // global 0-based atom
  double m64;    // fp64 |h_j|^2 = |h0_j - sum_tau x_tau c[(j - lambda_tau) mod N]|^2
};
// one shard's identification record (exchanged by all-gather)
struct LgRec {
  double best32;       // this shard's maximum of the working-precision |h|^2
  uint32_t count;      // candidates found (may exceed LG_RC: overflow)
  uint32_t pad;
  LgCand c[LG_RC];
};
enum LgFlag { LG_ZERO = 1, LG_STAGNANT = 2, LG_OVERFLOW = 4, LG_TOOMANY = 8 };
// the merged pick (identical on every shard)
struct LgPick {
  uint64_t j;    // global 0-based atom
  double best64;
  double2 b;     // fp64 h0 at j (least-squares right-hand side)
  int32_t flags;
  int32_t pad;
};
// device state of one shard (pointers into its GPU's memory)
struct LgShard {
  DevOp op;                 // full operator: omega, tw64 / tw32, g64, ...
  int dtype;                // C64 or C128 (working precision of h and r)
  int P, p, log2P, T;
  int64_t n, m, np;
  const void* gcm;          // kernel, class-major gcm[c][j'] = c[c + P j'] (dtype)
  void* h0s;                // own class of h0 (dtype)
  void* hs;                 // own class of the current correlation (dtype)
  const double2* h0x;       // fp64 h0 = Phi^H y, all n entries (replicated)
  double* blkmax;           // per-CTA maxima, then one per 128-position tile
  uint32_t* cand;           // LG_LCAP local candidates k'
  double* cval;             // their fp64 |h|^2
  unsigned* ccount;         // [0] candidates found
  LgRec* rec_send;          // this shard's record
  LgRec* rec_all;           // the P gathered records
  LgPick* pick;             // [2]: picks of alternate iterations
  double* fb;               // fallback scratch: [0] local best64, [1] global best64; u64 [2] first, [3] global first
  // least squares (replicated)
  double2 *W, *x, *z, *l;
  uint32_t* lam;            // T atoms, 0-based
  void* xn;                 // T, dtype: -x for the fast update
  double* part;
  double* scal;             // [0] gamma [1] yy [2] zz [3] d [4..5] znew [6] abort [7] sum|x| [8] max|x| [9] r2 [10] hy
  uint32_t* selbits;        // n bits: atoms selected
  // residual
  const void* y;            // m (dtype)
  const double2* y64;       // m, fp64 (fp32 data widened; = y for c128)
  void* r;                  // m (dtype)
  void* ax;                 // m (dtype or c128): Phi x at Omega, or this shard's partial
  void* axsum;              // m: sum of the partials over shards (P > 1)
  uint32_t* lamc;           // T: this shard's atoms as k' (0xffffffff: other class)
  void* fold;               // np (dtype): folded residual (P > 1)
  const uint32_t* bin_off;  // np + 1: rows by bin omega mod np (P > 1)
  const uint32_t* bin_row;  // m
};
int lg_grid();
// correlation rows and the local identification record
cudaError_t lg_fast(const LgShard& S, int s, cudaStream_t st);                 // hs, tile maxima, best32
cudaError_t lg_max(const LgShard& S, const void* h, cudaStream_t st);          // tile maxima, best32 of h
cudaError_t lg_identify(const LgShard& S, const void* h, int s, double ecoef, int prev, cudaStream_t st);
cudaError_t lg_merge(const LgShard& S, int cur, int prev, cudaStream_t st);     // rec_all -> pick[cur]
// fallback when a record overflowed: exact max / first over every candidate
cudaError_t lg_fb_local_best(const LgShard& S, cudaStream_t st);               // fb[0]
cudaError_t lg_fb_local_first(const LgShard& S, cudaStream_t st);              // u64 fb[2] (reads fb[1])
cudaError_t lg_fb_pick(const LgShard& S, int cur, cudaStream_t st);             // pick[cur] from fb[1], fb[3]
// least squares for pick[cur] (skipped when it is flagged), sum|x|, max|x|
cudaError_t lg_ls(const LgShard& S, int s, int cur, cudaStream_t st);
// residual pieces
cudaError_t lg_class_positions(const LgShard& S, int cnt, cudaStream_t st);    // lamc
cudaError_t lg_scatter_dense(const LgShard& S, int dtype, void* out, int64_t len, int cnt, cudaStream_t st);
cudaError_t lg_partial(const LgShard& S, int dtype, const void* X, void* out, cudaStream_t st);
cudaError_t lg_resid(const LgShard& S, int dtype, const void* ax, cudaStream_t st);  // r (dtype runs), scal[9]
cudaError_t lg_fold(const LgShard& S, cudaStream_t st);                         // fold <- r
cudaError_t lg_sum_partials(int dtype, const void* const* src, int P, void* dst, int64_t m, cudaStream_t st);
// setup
cudaError_t lg_take_narrow(const LgShard& S, cudaStream_t st);                  // h0s <- h0x
cudaError_t lg_classmajor(int dtype, const void* g, void* gcm, int64_t n, int P, cudaStream_t st);
cudaError_t lg_reduce_f64(const double* src, int P, int op_max, double* dst, cudaStream_t st);
cudaError_t lg_reduce_u64_min(const unsigned long long* src, int P, unsigned long long* dst, cudaStream_t st);
// the merge rule on host records (tests): returns the pick as a LgPick
void lg_merge_host(const LgRec* recs, int P, const uint32_t* selbits, LgPick* out);

// FMA-pipe throughput (FMAs per second) measured by a calibration kernel
cudaError_t fma_peak(int is_double, double* fma_per_s);
// number of kernel launches issued by the last launch_* call on this thread
int last_launch_count();
// IncrementalQR helpers (fmp_qr.cu): Q column-major rows x t, fp64 complex
int qr_dot_blocks(int64_t rows);
cudaError_t launch_qr_project(const double2* Q, int64_t rows, int t, double2* v, double2* part,
                              double2* s, double2* acc, cudaStream_t st);
cudaError_t launch_qr_norm(const double2* v, int64_t rows, double* part, double* out, cudaStream_t st);
cudaError_t launch_qr_store(double2* qnew, const double2* v, int64_t rows, double inv, cudaStream_t st);
cudaError_t launch_qr_dots(const double2* Q, int64_t rows, int t, const double2* rhs, double2* part,
                           double2* z, double2* scratch, cudaStream_t st);

// seeded instance generation on the device (fmp_gen.cu)
cudaError_t gen_batch(const DevOp& op, int64_t k, double noise_stddev, int real, uint64_t base,
                      uint64_t first, int64_t batch, double* y_out, double* x_out, double* nn_out,
                      uint64_t* fixups, cudaStream_t st);
void dd_eval_host(int fn, const double* x, int64_t cnt, double* out, double* frac);
cudaError_t dd_eval_dev(int fn, const double* x, int64_t cnt, double* out, double* frac, cudaStream_t st);

}  // namespace fmp
