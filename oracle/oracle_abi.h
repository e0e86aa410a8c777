/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the OMP correlation path.
 *
 * Two libraries export exactly this ABI:
 *   oracle/_build/libfmp_oracle.so  C restatement of the reference algorithm
 *                                   (oracle/fmp_oracle.c, every function cites
 *                                   the reference file:line it follows)
 *   oracle/_ref/libfmp_ref.so       the UNMODIFIED reference sources under
 *                                   /root/reference/proj/src compiled by
 *                                   oracle/Makefile, reached through the thin
 *                                   wrapper oracle/ref_capi.cpp
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load these.  The product path (paper_1205_4139_b200) never does.
 *
 * Conventions (mirroring proj/include/fastmp): complex vectors are interleaved
 * (re, im) doubles; atom / row indices are 1-based; kind 0 = Fourier,
 * 1 = Hadamard; mode 0 = Conventional, 1 = Fast, 2 = Adaptive; ls 0 =
 * IncrementalQR, 1 = NormalEquations.  Status: 0 ok, 1 invalid argument,
 * 2 rank deficient (position in *aux), 9 other exception.
 */
#ifndef FMP_ORACLE_ABI_H
#define FMP_ORACLE_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t fmpo_splitmix64(uint64_t x);
uint64_t fmpo_derive_seed(uint64_t base, uint64_t index);
/* first `count` raw mt19937_64 outputs for `seed` */
void fmpo_rng_u64(uint64_t seed, uint64_t count, uint64_t* out);
/* `count` complex gaussians from a fresh Rng(seed) */
void fmpo_rng_complex_gaussian(uint64_t seed, uint64_t count, double* out);
int fmpo_rng_sample(uint64_t seed, uint64_t n, uint64_t m, uint64_t* out);

int fmpo_make_row_selection(uint64_t n, uint64_t m, uint64_t seed,
                            uint64_t* omega_out);
/* make_instance (sensing.cpp:119-153): x_true (2n), y (2m), noise (2m) */
int fmpo_make_instance(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                       uint64_t k, double noise_stddev, uint64_t seed,
                       double* x_out, double* y_out, double* noise_out);
/* harness rule for real N(0,1) nonzeros: support from
 * Rng(seed).sample_one_based(n,k), x = sqrt(2)*Re(next_complex_gaussian()),
 * y = op.apply(x) */
int fmpo_make_real_instance(int kind, uint64_t n, const uint64_t* omega,
                            uint64_t m, uint64_t k, uint64_t seed,
                            double* x_out, double* y_out);

int fmpo_forward(int kind, uint64_t n, const double* v, double* out);
int fmpo_adjoint(int kind, uint64_t n, const double* v, double* out);
int fmpo_apply(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
               const double* x, double* y_out);
int fmpo_apply_adjoint(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                       const double* r, double* h_out);
int fmpo_column(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                uint64_t j, double* out);
int fmpo_entry(int kind, uint64_t n, uint64_t row, uint64_t col, double* out2);

/* compute_kernel: c (2n); Hadamard: values (<= n) and value_index (n) and
 * *nvalues; Fourier: *nvalues = 0 */
int fmpo_compute_kernel(int kind, uint64_t n, const uint64_t* omega,
                        uint64_t m, double* c_out, double* values_out,
                        uint32_t* value_index_out, uint64_t* nvalues);
int fmpo_fast_update(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                     const double* h0, const uint64_t* support,
                     const double* coeffs, uint64_t t, int symmetry,
                     double* h_out);
uint64_t fmpo_crossover_iteration(int kind, uint64_t n);
/* 0-based argmax with the 1e-9 tie band (solvers.cpp:90-101); restatement
 * only (the reference keeps it in an anonymous namespace) */
uint64_t fmpo_argmax_magnitude(const double* h, uint64_t n);

int fmpo_least_squares(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                       const uint64_t* support, uint64_t s, const double* y,
                       int ls_method, double* coeffs_out, uint64_t* aux);

typedef struct {
  uint64_t max_iterations;
  double residual_tolerance;
  int mode;
  int ls_method;
  int fourier_symmetry;
  int record_correlations;
} fmpo_solve_config;

typedef struct {
  uint64_t* support;      /* max_iterations, selection order, 1-based */
  double* coeffs;         /* 2 * max_iterations */
  uint64_t support_size;
  uint64_t iterations_run;
  double residual_norm;
  int rank_deficient_abort;
  uint64_t history_len;   /* number of recorded correlation vectors */
  double* correlation_history; /* max_iterations * 2n, or NULL */
  int* mode_used;         /* max_iterations, or NULL: 1 fast, 0 conventional */
} fmpo_solve_result;

int fmpo_omp_solve(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                   const double* y, const fmpo_solve_config* cfg,
                   fmpo_solve_result* out);

/* Batched OMP over `batch` measurement vectors (y: batch x 2m) on `threads`
 * host threads (0 = hardware_concurrency); outputs are batch-major arrays
 * (support: batch x max_iterations, coeffs: batch x 2 max_iterations,
 * iterations / residual / aborted: batch).  Used for the CPU baseline. */
int fmpo_omp_solve_batch(int kind, uint64_t n, const uint64_t* omega,
                         uint64_t m, const double* y, uint64_t batch,
                         const fmpo_solve_config* cfg, int threads,
                         uint64_t* support, double* coeffs,
                         uint64_t* iterations, double* residual,
                         int* aborted);

/* CoSaMP with sparsity k (solvers.hpp:73-78, solvers.cpp:413-544); mode as
 * for OMP (0 conventional, 1 fast, 2 adaptive = adaptive_cosamp_uses_fast).
 * out->support / out->coeffs hold k entries (ascending atoms);
 * support_history (max_iterations x k, zero padded) may be NULL. */
int fmpo_cosamp_solve(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                      const double* y, uint64_t k, const fmpo_solve_config* cfg,
                      fmpo_solve_result* out, uint64_t* support_history);

/* which implementation this library is: "restatement" or "reference" */
const char* fmpo_impl(void);

#ifdef __cplusplus
}
#endif

#endif
