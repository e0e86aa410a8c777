/*
 * fmp.h — C ABI of the B200 OMP correlation path (libfmp_cuda.so).
 *
 * This is the drop-in boundary for the reference library's correlation / OMP
 * interface, /root/reference/proj/include/fastmp (a C++20 library with no FFI
 * of its own).  Each entry point names the reference interface it replaces;
 * the C++ facade include/fastmp_b200/fastmp.hpp re-exposes those signatures
 * on top of this ABI, and INTEGRATION.md shows the bindings.
 *
 * Conventions
 *   - plain pointers and sizes only; no C++ or torch types
 *   - complex vectors are interleaved (re, im); `dtype` selects the element:
 *       FMP_C128 complex double, FMP_C64 complex float,
 *       FMP_F64 / FMP_F32 real (Hadamard operators with real data only)
 *   - atom and row indices are 1-based, as in the reference
 *     (transform.hpp:32-34); supports are in selection order
 *   - batched calls process `batch` independent vectors laid out back to back
 *   - functions without a `_dev` suffix take HOST buffers, copy in, compute
 *     on the context's GPU and copy out before returning (the reference's
 *     value semantics);  `_dev` variants take DEVICE pointers and enqueue on
 *     `stream` (NULL = the context stream) without synchronising
 *   - every call returns a status; fmp_last_error() describes the last
 *     failure on the calling thread.  Status codes map 1:1 onto the
 *     reference's exceptions: FMP_EINVAL = std::invalid_argument
 *     (kernel.cpp:213-222, sensing.cpp:94,104, transform.cpp:121,138),
 *     FMP_ERANK = RankDeficientError (solvers.hpp:42-51)
 *   - handles are re-entrant per handle; use one context per host thread
 *     for concurrent work.  A context's device workspaces are shared by its
 *     calls, so calls on one context are ordered on the device: a `_dev`
 *     call enqueued on another stream than the previous call first waits
 *     (cudaStreamWaitEvent) for that call's work.  Independent solves that
 *     should overlap on the device need separate contexts.
 *   - results of the fused solvers are deterministic for a given launch
 *     configuration but not bitwise batch-invariant: the solver's CTA shape
 *     depends on the batch (fmp_omp_plan_info), and block reductions over a
 *     different number of warps round differently (supports are unaffected
 *     beyond the reference's own 1e-9 tie band)
 */
#ifndef FMP_H
#define FMP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum fmp_status {
  FMP_OK = 0,
  FMP_EINVAL = 1,       /* std::invalid_argument in the reference */
  FMP_ERANK = 2,        /* RankDeficientError */
  FMP_ECUDA = 3,        /* CUDA runtime / launch failure */
  FMP_ENOMEM = 4,       /* device allocation failed */
  FMP_EUNSUPPORTED = 5, /* shape outside what the GPU path implements */
  FMP_ENCCL = 6         /* collective failure (sharded solve) */
};

enum fmp_kind { FMP_FOURIER = 0, FMP_HADAMARD = 1 };       /* TransformKind, types.hpp:28 */
enum fmp_dtype { FMP_C128 = 0, FMP_C64 = 1, FMP_F64 = 2, FMP_F32 = 3 };
/* CorrelationMode (cost_model.hpp:58); FMP_MODE_CUSTOM uses fast_until */
enum fmp_mode {
  FMP_MODE_CONVENTIONAL = 0,
  FMP_MODE_FAST = 1,
  FMP_MODE_ADAPTIVE = 2,
  FMP_MODE_CUSTOM = 3,
  FMP_MODE_GPU = 4     /* Adaptive with the B200-calibrated switch point */
};

typedef struct fmp_ctx_s* fmp_ctx;
typedef struct fmp_op_s* fmp_op;

int fmp_version(void);
/* number of CUDA devices visible to this process (0 without a GPU) */
int fmp_device_count(int* out);
/* page-locked host memory (cudaHostAlloc, portable across devices): host
 * buffers from here let the host-buffer solves overlap their copies with
 * the solve (see fmp_omp_solve) */
int fmp_host_alloc(size_t bytes, void** out);
int fmp_host_free(void* p);
/* calibrate the FMA pipe of the context's GPU: FMAs per second (fp64 when
 * is_double, else fp32) — the roofline denominator of the accumulate path */
int fmp_fma_peak(fmp_ctx ctx, int is_double, double* fma_per_s);
const char* fmp_last_error(void);
/* number of kernel launches the last call on this thread issued */
int fmp_last_launch_count(void);

/* ---------------------------------------------------------------- context */
int fmp_ctx_create(int device, fmp_ctx* out);
int fmp_ctx_destroy(fmp_ctx ctx);
/* cudaStream_t to enqueue on (NULL restores the context-owned stream) */
int fmp_ctx_set_stream(fmp_ctx ctx, void* stream);
void* fmp_ctx_stream(fmp_ctx ctx);
int fmp_ctx_synchronize(fmp_ctx ctx);

/* --------------------------------------------------------------- operator */
/* SensingOperator(StructuredUnitary(kind, n), make_row_selection(n, rows))
 * (sensing.hpp:39-44, sensing.cpp:72-80 validation): rows are 1-based,
 * distinct, in [1, n]; they are sorted here as the reference does.  Builds
 * the correlation kernel c = Phi^H Phi e_1 on the device
 * (compute_kernel, kernel.hpp:42-43).  n must be a power of two. */
int fmp_operator_create(fmp_ctx ctx, int kind, uint64_t n, const uint64_t* rows_1based,
                        uint64_t m, fmp_op* out);
int fmp_operator_destroy(fmp_op op);
int fmp_operator_info(fmp_op op, int* kind, uint64_t* n, uint64_t* m);
/* CorrelationKernel readback (kernel.hpp:31-40): c (2n doubles); Hadamard
 * also the sorted distinct values (up to m+1) and value_index (n); Fourier
 * sets *nvalues = 0.  values / value_index may be NULL. */
int fmp_operator_kernel(fmp_op op, double* c_out, double* values_out,
                        uint32_t* value_index_out, uint64_t* nvalues);
/* crossover_iteration (cost_model.hpp:76): the Adaptive switch point */
uint64_t fmp_crossover_iteration(int kind, uint64_t n);
/* the same switch point measured for this GPU path (FMP_MODE_GPU): fast
 * updates while t <= this, transforms afterwards — for the one-CTA-per-SM
 * solver (small batches, the sharded config-5 solver) */
uint64_t fmp_gpu_crossover(int kind, uint64_t n);
/* the switch point FMP_MODE_GPU uses for a batched solve of `batch` problems
 * of `dtype` with max_iterations T on op (the solver's configuration depends
 * on the batch: two CTAs per SM when both fit) */
uint64_t fmp_gpu_crossover_for(fmp_op op, int dtype, uint64_t batch, uint64_t max_iterations);
/* the fused solver's configuration for such a solve (tests / tools):
 * out4 = {CTAs per SM, threads per CTA, kernel table (0 global memory,
 * 1 shared full, 2 shared conjugate half), transform buffer in global memory} */
int fmp_omp_plan_info(fmp_op op, int dtype, uint64_t batch, uint64_t max_iterations, int* out4);

/* ------------------------------------------------------ transforms (batched) */
/* SensingOperator::apply, Phi x (sensing.cpp:93-100): x batch x n -> y batch x m */
int fmp_apply(fmp_op op, int dtype, const void* x, uint64_t batch, void* y_out);
int fmp_apply_dev(fmp_op op, int dtype, const void* x, uint64_t batch, void* y_out, void* stream);
/* SensingOperator::apply_adjoint, Phi^H r (sensing.cpp:102-109) — the
 * conventional correlation: r batch x m -> h batch x n.  argmax_out
 * (optional, batch) receives the 1-based band argmax of |h| (solvers.cpp:90-101)
 * and h_out may then be NULL. */
int fmp_apply_adjoint(fmp_op op, int dtype, const void* r, uint64_t batch, void* h_out,
                      uint64_t* argmax_out);
int fmp_apply_adjoint_dev(fmp_op op, int dtype, const void* r, uint64_t batch, void* h_out,
                          uint64_t* argmax_out, void* stream);
/* StructuredUnitary::forward / adjoint (transform.hpp:46-47), dense n -> n */
int fmp_unitary_forward(fmp_op op, int dtype, const void* v, uint64_t batch, void* out);
int fmp_unitary_adjoint(fmp_op op, int dtype, const void* v, uint64_t batch, void* out);

/* --------------------------------------------------- fast update (batched) */
/* fast_update (kernel.hpp:95-98): h = h0 - sum_tau coeffs[tau] P_{support[tau]} c
 * for `batch` problems, each with t atoms: h0 batch x n, support batch x t
 * (1-based, distinct per problem), coeffs batch x t.  h_out (batch x n) and/or
 * argmax_out (batch, 1-based band argmax) may be NULL (not both). */
int fmp_fast_update(fmp_op op, int dtype, const void* h0, const uint64_t* support,
                    const void* coeffs, uint64_t t, uint64_t batch, void* h_out,
                    uint64_t* argmax_out);
int fmp_fast_update_dev(fmp_op op, int dtype, const void* h0, const uint32_t* support0,
                        const void* coeffs, uint64_t t, uint64_t batch, void* h_out,
                        uint64_t* argmax_out, void* stream);

/* argmax_magnitude with the 1e-9 tie band (solvers.cpp:90-101): 1-based */
int fmp_argmax_band(fmp_ctx ctx, int dtype, const void* h, uint64_t n, uint64_t batch,
                    uint64_t* idx_out);

/* least_squares (solvers.hpp:82-85) in its normal-equations form
 * (solvers.cpp:120-177) for `batch` problems sharing the support size s:
 * y batch x m, support batch x s (1-based), coeffs_out batch x s complex fp64.
 * A numerically dependent column gives FMP_ERANK with *position (0-based
 * position within that problem's support; the first failing problem). */
int fmp_least_squares(fmp_op op, int dtype, const void* y, const uint64_t* support, uint64_t s,
                      uint64_t batch, double* coeffs_out, int64_t* position);

/* ----------------------------------------------------------- OMP (batched) */
typedef struct {
  uint64_t max_iterations;     /* SolveConfig::max_iterations (>= 1) */
  double tolerance;            /* residual_tolerance used when tolerances == NULL */
  const double* tolerances;    /* optional per-problem tolerances (batch) */
  int mode;                    /* fmp_mode */
  uint64_t fast_until;         /* FMP_MODE_CUSTOM: t <= fast_until use the fast update */
  int record_correlations;     /* keep every correlation vector (history) */
} fmp_omp_config;

typedef struct {
  uint64_t* support;      /* batch x max_iterations, 1-based, selection order, 0 padded */
  double* coeffs;         /* batch x max_iterations complex (always fp64) */
  uint64_t* support_size; /* batch */
  uint64_t* iterations;   /* batch: iterations_run */
  double* residual;       /* batch: residual_norm */
  int32_t* aborted;       /* batch: rank_deficient_abort */
  uint8_t* modes;         /* optional batch x max_iterations: 1 fast, 0 conventional */
  uint64_t* history_len;  /* optional batch: correlation vectors recorded */
  void* history;          /* optional batch x max_iterations x n (dtype) */
} fmp_omp_result;

/* omp_solve (solvers.hpp:70-71) over `batch` measurement vectors y (batch x m)
 * sharing one operator.  Selected supports follow the reference's
 * identification rule exactly; least squares runs in fp64. */
int fmp_omp_solve(fmp_op op, int dtype, const void* y, uint64_t batch,
                  const fmp_omp_config* cfg, fmp_omp_result* out);
int fmp_omp_solve_dev(fmp_op op, int dtype, const void* y, uint64_t batch,
                      const fmp_omp_config* cfg, fmp_omp_result* out, void* stream);
/* The same over several GPUs: ops[i] is the operator built on GPU i's
 * context (one fmp_operator_create per device, the same kind, n and rows).
 * The batch is split into nops contiguous blocks (the first batch % nops
 * one problem larger), each solved by fmp_omp_solve on its device from a
 * host thread of its own; results land in `out` at their global positions.
 * The problems are independent: no collective.  This is the multi-device
 * form of the reference's solve-per-worker pool (fastmp_cli.cpp:276-303);
 * the seeded command-line driver paper_1205_4139_b200/host/fmp_driver.cpp
 * runs over it.  The first failing block's status and message are
 * returned.  Page-locked y and result buffers (fmp_host_alloc) take the
 * streamed path of fmp_omp_solve. */
int fmp_omp_solve_multi(const fmp_op* ops, int nops, int dtype, const void* y, uint64_t batch,
                        const fmp_omp_config* cfg, fmp_omp_result* out);

/* ------------------------------------------------------- CoSaMP (batched) */
/* cosamp_solve (solvers.hpp:73-78, solvers.cpp:413-544) with sparsity k over
 * `batch` measurement vectors.  cfg as for OMP: max_iterations, tolerance(s),
 * record_correlations; mode CONVENTIONAL / FAST / ADAPTIVE (the reference's
 * adaptive_cosamp_uses_fast, cost_model.cpp:91-96; GPU and CUSTOM behave as
 * FAST).  Supports come out ascending like the reference's.  Merge, band
 * selection and pruning follow select_largest (solvers.cpp:62-86) exactly;
 * least squares is the normal-equations Cholesky in fp64. */
typedef struct {
  uint64_t* support;          /* batch x k, ascending 1-based atoms, 0 padded */
  double* coeffs;             /* batch x k complex (fp64) */
  uint64_t* support_size;     /* batch */
  uint64_t* iterations;       /* batch */
  double* residual;           /* batch */
  int32_t* aborted;           /* batch: rank_deficient_abort */
  uint64_t* support_history;  /* optional batch x max_iterations x k (0 padded) */
  void* history;              /* optional batch x max_iterations x n (dtype) */
} fmp_cosamp_result;
int fmp_cosamp_solve(fmp_op op, int dtype, const void* y, uint64_t batch, uint64_t k,
                     const fmp_omp_config* cfg, fmp_cosamp_result* out);
int fmp_cosamp_solve_dev(fmp_op op, int dtype, const void* y, uint64_t batch, uint64_t k,
                         const fmp_omp_config* cfg, fmp_cosamp_result* out, void* stream);

/* ------------------------------------------------------------ IncrementalQR */
/* IncrementalQR (solvers.hpp:90-109): thin QR of a growing column set, Q
 * resident on the device.  push_column returns *accepted = 0 (and leaves the
 * factorisation unchanged) when the column's remainder after two
 * Gram-Schmidt passes is at most 1e-10 of its norm (solvers.cpp:244).
 * Columns / rhs / x are host arrays of interleaved complex fp64. */
typedef struct fmp_qr_s* fmp_qr;
int fmp_qr_create(fmp_ctx ctx, uint64_t rows, uint64_t capacity, fmp_qr* out);
int fmp_qr_destroy(fmp_qr qr);
int fmp_qr_push_column(fmp_qr qr, const double* col, int* accepted);
int fmp_qr_solve(fmp_qr qr, const double* rhs, double* x_out);
uint64_t fmp_qr_cols(fmp_qr qr);

/* profiling aid: when enabled, each fused solve accumulates SM cycles per
 * phase (conventional correlation, fast correlation, identification, least
 * squares, residual, other), summed over CTAs, readable afterwards */
int fmp_set_phase_profiling(int enabled);
int fmp_phase_cycles(fmp_ctx ctx, double* out6);
/* with phase profiling on, the fp32 solves (c64 / f32) also count, over the
 * last solve: identifications, fp64-re-evaluated candidates, and
 * identifications whose candidates overflowed the per-CTA list */
int fmp_refine_stats(fmp_ctx ctx, double* out3);

/* ------------------------------------------- sharded single-signal solver */
/* omp_solve (solvers.cpp:296-411) for ONE large signal spread over `nshards`
 * shards, one per GPU (config 5).  Shard p owns the correlation entries
 * k = p + nshards * k' (1-based atom k + 1): its fast rows read its class of
 * the kernel, its conventional rows are (N / nshards)-point transforms of the
 * residual folded into its class, and the residual is the sum over shards of
 * their atoms' forward transforms.  Per iteration the shards exchange one
 * identification record (all-gather of at most 64 candidates re-evaluated in
 * fp64; fmp_large_merge_records is the rule) and, before a conventional row,
 * one M-vector (all-reduce sum); least squares is replicated bit-identically.
 * Picks and coefficients do not depend on nshards.  Fourier only.
 *
 * Exchanges run on the device: through NCCL when every shard of the group
 * has a communicator (one rank per shard: fmp_comm_init_rank across
 * processes, fmp_comm_init_all for several GPUs in one process), else
 * between shards of one process on one GPU (emulation: all nshards shards
 * passed to one fmp_large_group_solve call).  The host synchronises once per
 * iteration on the previous iteration's decisions (halting, rank deficiency)
 * while the device already computes the next correlation. */
typedef struct fmp_comm_s* fmp_comm;
/* NCCL (libnccl.so.2, loaded at first use): a 128-byte unique id made on one
 * rank and shared with the others (any transport), then one communicator
 * per rank on `device` */
int fmp_comm_unique_id(void* id128);
int fmp_comm_init_rank(int device, int nranks, int rank, const void* id128, fmp_comm* out);
/* n communicators of one process, rank i on devices[i] */
int fmp_comm_init_all(const int* devices, int n, fmp_comm* out);
int fmp_comm_destroy(fmp_comm comm);

typedef struct fmp_large_s* fmp_large;
/* comm: this shard's communicator, or NULL (nshards == 1, or emulation) */
int fmp_large_create(fmp_op op, int dtype, uint64_t shard, uint64_t nshards,
                     const fmp_omp_config* cfg, fmp_comm comm, fmp_large* out);
int fmp_large_destroy(fmp_large lg);
/* solve with the `count` shards of this process (all nshards for emulation or
 * one process over several GPUs, one per process with NCCL across
 * processes); y: m values (host), tol: absolute residual tolerance */
int fmp_large_group_solve(fmp_large* shards, int count, const void* y, double tol);
int fmp_large_result(fmp_large lg, uint64_t* support, double* coeffs, uint64_t* support_size,
                     uint64_t* iterations, double* residual, int32_t* aborted);
/* the whole solve on one GPU (nshards = 1) */
int fmp_large_solve(fmp_op op, int dtype, const void* y, const fmp_omp_config* cfg,
                    fmp_omp_result* out);
/* the record merge every shard runs after the all-gather (host twin of the
 * device kernel, for tests): `recs` = nshards records of
 * fmp_large_record_size() bytes, `selbits` the selected-atom bitmap (or
 * NULL); out4 = {atom (0-based, as double), best |h|^2, flags, 0} with flags
 * 1 zero correlation, 2 stagnation, 4 a record overflowed (exact fallback),
 * 8 more candidates than a shard evaluates */
int fmp_large_record_size(void);
int fmp_large_merge_records(const void* recs, int nshards, const uint32_t* selbits, double* out4);

/* ------------------------------------------------------ instance generation */
/* seeded synthetic problems for the bench / parity harness, following the
 * reference's make_row_selection / make_instance recipes (sensing.cpp:61-70,
 * :119-153) with its Rng (random.cpp).  y is synthesised directly from the
 * K nonzeros (identical up to rounding to op.apply(x)). real != 0 draws
 * real N(0,1) nonzeros.  Host memory; threads 0 = all cores. */
int fmp_make_row_selection(uint64_t n, uint64_t m, uint64_t seed, uint64_t* rows_out);
int fmp_make_batch(int kind, uint64_t n, const uint64_t* rows_1based, uint64_t m, uint64_t k,
                   double noise_stddev, int real, uint64_t base_seed, uint64_t first,
                   uint64_t batch, int threads, double* y_out, double* x_out,
                   double* noise_norm_out);
uint64_t fmp_derive_seed(uint64_t base, uint64_t index);
/* make_instance's draws for one seed (sensing.cpp:132-147): x (n complex)
 * and noise (m complex); the caller forms y = apply(x) + noise */
int fmp_draw_instance(uint64_t n, uint64_t m, uint64_t k, double noise_stddev, uint64_t seed,
                      double* x_out, double* noise_out);

/* GPU-side generation of the same batch: fmp_make_batch's
 * draws computed on the device of `op` (Omega = op's rows) and bit-identical
 * to it: the mt19937_64 stream, the Fisher-Yates support, the Gaussians and
 * y in the host's summation order.  log / cos / sin are evaluated in
 * double-double arithmetic and rounded; values whose exact result lies
 * within 0.025 ulp of a rounding midpoint (where glibc may round the other
 * way, its measured error reaching 0.515 ulp) are recomputed on the host with
 * glibc -- *fixups_out (optional) counts them.  Device buffers: y_out
 * batch x m complex128 (interleaved), x_out batch x n complex128 or NULL,
 * noise_norm_out batch doubles or NULL.  Synchronises `stream` (NULL = the
 * context's) once, for the host recomputation.  Replaces, for the harness,
 * make_instance (sensing.cpp:119-153) with Rng (random.cpp:34-67). */
int fmp_make_batch_dev(fmp_op op, uint64_t k, double noise_stddev, int real, uint64_t base_seed,
                       uint64_t first, uint64_t batch, double* y_out, double* x_out,
                       double* noise_norm_out, uint64_t* fixups_out, void* stream);
/* the device generator's double-double log (fn 0) / cos (1) / sin (2) run on
 * the host (tests): out = the correctly rounded value, frac (optional) = the
 * exact result's distance from it towards its neighbour, in ulps (0..0.5) */
int fmp_dd_eval(int fn, const double* x, uint64_t count, double* out, double* frac);
/* the same on the device (device buffers; frac required), on `stream` */
int fmp_dd_eval_dev(int fn, const double* x, uint64_t count, double* out, double* frac, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FMP_H */
