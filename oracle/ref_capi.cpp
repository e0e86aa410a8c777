// TEST INFRASTRUCTURE ONLY.  Thin extern "C" wrapper that exposes the
// unmodified reference library (/root/reference/proj/src, compiled by
// oracle/Makefile into oracle/_ref/libfmp_ref.so) through oracle_abi.h, so the
// tests and the bench's CPU arm can drive the reference with plain pointers.
// No reference source is copied here: this file only calls the public
// fastmp:: API declared in /root/reference/proj/include/fastmp/*.hpp.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <stdexcept>
#include <thread>
#include <vector>

#include "fastmp/kernel.hpp"
#include "fastmp/random.hpp"
#include "fastmp/sensing.hpp"
#include "fastmp/solvers.hpp"
#include "oracle_abi.h"

using namespace fastmp;

#include "../tests/cpp/counts_recipe.inc"

namespace {

TransformKind kind_of(int kind) {
  if (kind == 0) return TransformKind::Fourier;
  if (kind == 1) return TransformKind::Hadamard;
  throw std::invalid_argument("bad kind");
}

cvec load(const double* p, std::size_t n) {
  cvec v(n);
  for (std::size_t i = 0; i < n; ++i) v[i] = cplx(p[2 * i], p[2 * i + 1]);
  return v;
}

void store(const cvec& v, double* p) {
  for (std::size_t i = 0; i < v.size(); ++i) {
    p[2 * i] = v[i].real();
    p[2 * i + 1] = v[i].imag();
  }
}

SensingOperator make_op(int kind, uint64_t n, const uint64_t* omega,
                        uint64_t m) {
  std::vector<std::size_t> rows(omega, omega + m);
  return SensingOperator(StructuredUnitary(kind_of(kind), n),
                         make_row_selection(n, std::move(rows)));
}

template <class F>
int guard(F&& f, uint64_t* aux = nullptr) {
  try {
    f();
    return 0;
  } catch (const RankDeficientError& e) {
    if (aux) *aux = e.position();
    return 2;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (...) {
    return 9;
  }
}

CorrelationMode mode_of(int m) {
  return m == 0 ? CorrelationMode::Conventional
                : (m == 1 ? CorrelationMode::Fast : CorrelationMode::Adaptive);
}

SolveConfig config_of(const fmpo_solve_config* c) {
  SolveConfig cfg;
  cfg.max_iterations = c->max_iterations;
  cfg.residual_tolerance = c->residual_tolerance;
  cfg.correlation_mode = mode_of(c->mode);
  cfg.ls_method = c->ls_method == 1 ? LeastSquaresMethod::NormalEquations
                                    : LeastSquaresMethod::IncrementalQR;
  cfg.fourier_symmetry = c->fourier_symmetry != 0;
  cfg.record_correlations = c->record_correlations != 0;
  return cfg;
}

}  // namespace

extern "C" {

const char* fmpo_impl(void) { return "reference"; }

uint64_t fmpo_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t fmpo_derive_seed(uint64_t b, uint64_t i) { return derive_seed(b, i); }

void fmpo_rng_u64(uint64_t seed, uint64_t count, uint64_t* out) {
  Rng rng(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng.next_u64();
}

void fmpo_rng_complex_gaussian(uint64_t seed, uint64_t count, double* out) {
  Rng rng(seed);
  for (uint64_t i = 0; i < count; ++i) {
    const cplx z = rng.next_complex_gaussian();
    out[2 * i] = z.real();
    out[2 * i + 1] = z.imag();
  }
}

int fmpo_rng_sample(uint64_t seed, uint64_t n, uint64_t m, uint64_t* out) {
  return guard([&] {
    Rng rng(seed);
    const auto s = rng.sample_one_based(n, m);
    std::copy(s.begin(), s.end(), out);
  });
}

int fmpo_make_row_selection(uint64_t n, uint64_t m, uint64_t seed,
                            uint64_t* omega_out) {
  return guard([&] {
    const RowSelection sel = make_row_selection(n, m, seed);
    std::copy(sel.omega.begin(), sel.omega.end(), omega_out);
  });
}

int fmpo_make_instance(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                       uint64_t k, double noise_stddev, uint64_t seed,
                       double* x_out, double* y_out, double* noise_out) {
  return guard([&] {
    const SensingOperator op = make_op(kind, n, omega, m);
    const ProblemInstance inst = make_instance(op, k, noise_stddev, seed);
    store(inst.x_true, x_out);
    store(inst.y, y_out);
    if (noise_out) store(inst.noise, noise_out);
  });
}

int fmpo_make_real_instance(int kind, uint64_t n, const uint64_t* omega,
                            uint64_t m, uint64_t k, uint64_t seed,
                            double* x_out, double* y_out) {
  return guard([&] {
    const SensingOperator op = make_op(kind, n, omega, m);
    Rng rng(seed);
    cvec x(n, cplx(0.0));
    const auto support = rng.sample_one_based(n, k);
    for (std::size_t idx : support)
      x[idx - 1] = cplx(std::sqrt(2.0) * rng.next_complex_gaussian().real(), 0.0);
    store(x, x_out);
    store(op.apply(x), y_out);
  });
}

int fmpo_forward(int kind, uint64_t n, const double* v, double* out) {
  return guard([&] {
    store(StructuredUnitary(kind_of(kind), n).forward(load(v, n)), out);
  });
}

int fmpo_adjoint(int kind, uint64_t n, const double* v, double* out) {
  return guard([&] {
    store(StructuredUnitary(kind_of(kind), n).adjoint(load(v, n)), out);
  });
}

int fmpo_apply(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
               const double* x, double* y_out) {
  return guard([&] { store(make_op(kind, n, omega, m).apply(load(x, n)), y_out); });
}

int fmpo_apply_adjoint(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                       const double* r, double* h_out) {
  return guard([&] {
    store(make_op(kind, n, omega, m).apply_adjoint(load(r, m)), h_out);
  });
}

int fmpo_column(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                uint64_t j, double* out) {
  return guard([&] { store(make_op(kind, n, omega, m).column(j), out); });
}

int fmpo_entry(int kind, uint64_t n, uint64_t row, uint64_t col, double* out2) {
  return guard([&] {
    const cplx e = StructuredUnitary(kind_of(kind), n).entry(row, col);
    out2[0] = e.real();
    out2[1] = e.imag();
  });
}

int fmpo_compute_kernel(int kind, uint64_t n, const uint64_t* omega,
                        uint64_t m, double* c_out, double* values_out,
                        uint32_t* value_index_out, uint64_t* nvalues) {
  return guard([&] {
    const CorrelationKernel ker = compute_kernel(make_op(kind, n, omega, m));
    store(ker.c, c_out);
    *nvalues = ker.values.size();
    if (values_out)
      std::copy(ker.values.begin(), ker.values.end(), values_out);
    if (value_index_out)
      std::copy(ker.value_index.begin(), ker.value_index.end(),
                value_index_out);
  });
}

int fmpo_fast_update(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                     const double* h0, const uint64_t* support,
                     const double* coeffs, uint64_t t, int symmetry,
                     double* h_out) {
  return guard([&] {
    const CorrelationKernel ker = compute_kernel(make_op(kind, n, omega, m));
    std::vector<std::size_t> sup(support, support + t);
    FastUpdateOptions opts;
    opts.fourier_symmetry = symmetry != 0;
    store(fast_update(load(h0, n), ker, sup, load(coeffs, t), opts), h_out);
  });
}

uint64_t fmpo_crossover_iteration(int kind, uint64_t n) {
  return crossover_iteration(kind_of(kind), n);
}

uint64_t fmpo_argmax_magnitude(const double*, uint64_t) {
  return UINT64_MAX;  // not exported by the reference (anonymous namespace)
}

int fmpo_least_squares(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                       const uint64_t* support, uint64_t s, const double* y,
                       int ls_method, double* coeffs_out, uint64_t* aux) {
  return guard(
      [&] {
        std::vector<std::size_t> sup(support, support + s);
        const cvec b = least_squares(
            make_op(kind, n, omega, m), sup, load(y, m),
            ls_method == 1 ? LeastSquaresMethod::NormalEquations
                           : LeastSquaresMethod::IncrementalQR);
        store(b, coeffs_out);
      },
      aux);
}

int fmpo_omp_solve(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                   const double* y, const fmpo_solve_config* c,
                   fmpo_solve_result* out) {
  return guard([&] {
    const SensingOperator op = make_op(kind, n, omega, m);
    const RecoveryResult res = omp_solve(op, load(y, m), config_of(c));
    out->support_size = res.support.size();
    std::copy(res.support.begin(), res.support.end(), out->support);
    store(res.coeffs, out->coeffs);
    out->iterations_run = res.iterations_run;
    out->residual_norm = res.residual_norm;
    out->rank_deficient_abort = res.rank_deficient_abort ? 1 : 0;
    out->history_len = res.correlation_history.size();
    if (out->correlation_history)
      for (std::size_t i = 0; i < res.correlation_history.size(); ++i)
        store(res.correlation_history[i], out->correlation_history + 2 * n * i);
    if (out->mode_used)
      for (std::size_t i = 0; i < res.costs.iterations.size(); ++i)
        out->mode_used[i] =
            res.costs.iterations[i].mode_used == CorrelationMode::Fast ? 1 : 0;
  });
}

int fmpo_cosamp_solve(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                      const double* y, uint64_t k, const fmpo_solve_config* c,
                      fmpo_solve_result* out, uint64_t* support_history) {
  return guard([&] {
    const SensingOperator op = make_op(kind, n, omega, m);
    const RecoveryResult res = cosamp_solve(op, load(y, m), k, config_of(c));
    out->support_size = res.support.size();
    std::copy(res.support.begin(), res.support.end(), out->support);
    store(res.coeffs, out->coeffs);
    out->iterations_run = res.iterations_run;
    out->residual_norm = res.residual_norm;
    out->rank_deficient_abort = res.rank_deficient_abort ? 1 : 0;
    out->history_len = res.correlation_history.size();
    if (out->correlation_history)
      for (std::size_t i = 0; i < res.correlation_history.size(); ++i)
        store(res.correlation_history[i], out->correlation_history + 2 * n * i);
    if (out->mode_used)
      for (std::size_t i = 0; i < res.costs.iterations.size(); ++i)
        out->mode_used[i] =
            res.costs.iterations[i].mode_used == CorrelationMode::Fast ? 1 : 0;
    if (support_history)
      for (std::size_t i = 0; i < res.support_history.size(); ++i) {
        std::fill(support_history + k * i, support_history + k * (i + 1), 0);
        std::copy(res.support_history[i].begin(), res.support_history[i].end(),
                  support_history + k * i);
      }
  });
}

int fmpo_omp_solve_batch(int kind, uint64_t n, const uint64_t* omega,
                         uint64_t m, const double* y, uint64_t batch,
                         const fmpo_solve_config* c, int threads,
                         uint64_t* support, double* coeffs,
                         uint64_t* iterations, double* residual,
                         int* aborted) {
  return guard([&] {
    const SensingOperator op = make_op(kind, n, omega, m);
    const SolveConfig cfg = config_of(c);
    const uint64_t T = c->max_iterations;
    unsigned workers = threads > 0 ? unsigned(threads)
                                   : std::max(1u, std::thread::hardware_concurrency());
    workers = unsigned(std::min<uint64_t>(workers, std::max<uint64_t>(batch, 1)));
    std::atomic<uint64_t> next{0};
    std::atomic<bool> failed{false};
    auto work = [&] {
      for (;;) {
        const uint64_t b = next.fetch_add(1);
        if (b >= batch || failed.load()) return;
        try {
          const RecoveryResult res = omp_solve(op, load(y + 2 * m * b, m), cfg);
          std::fill(support + T * b, support + T * (b + 1), 0);
          std::fill(coeffs + 2 * T * b, coeffs + 2 * T * (b + 1), 0.0);
          std::copy(res.support.begin(), res.support.end(), support + T * b);
          store(res.coeffs, coeffs + 2 * T * b);
          iterations[b] = res.iterations_run;
          residual[b] = res.residual_norm;
          aborted[b] = res.rank_deficient_abort ? 1 : 0;
        } catch (...) {
          failed = true;
        }
      }
    };
    std::vector<std::thread> pool;
    for (unsigned w = 1; w < workers; ++w) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    if (failed) throw std::runtime_error("batch solve failed");
  });
}

}  // extern "C"

// ---- text formats (reference only: fixtures for the facade's I/O) --------
namespace {
int put_text(const std::string& t, char* buf, uint64_t cap, uint64_t* len) {
  if (len) *len = t.size();
  if (!buf || cap < t.size() + 1) return 3;
  std::memcpy(buf, t.data(), t.size() + 1);
  return 0;
}
}  // namespace

extern "C" {

/* save_instance (sensing.cpp:160-168) of make_instance(op, k, noise, seed)
 * with Omega = make_row_selection(n, m, derive_seed(seed, 1)) */
int fmpo_ref_instance_text(int kind, uint64_t n, uint64_t m, uint64_t k, double noise,
                           uint64_t seed, char* buf, uint64_t cap, uint64_t* len) {
  int st = 0;
  const int g = guard([&] {
    const SensingOperator op(StructuredUnitary(kind == 0 ? TransformKind::Fourier
                                                         : TransformKind::Hadamard, n),
                             make_row_selection(n, m, derive_seed(seed, 1)));
    std::ostringstream os;
    save_instance(make_instance(op, k, noise, seed), os);
    st = put_text(os.str(), buf, cap, len);
  });
  return g ? g : st;
}

/* load_instance -> omp_solve(default_config(k, |y|), mode) -> save_result
 * (solvers.cpp:546-562) and costs.write_csv (cost_model.cpp:98-113) */
int fmpo_ref_result_text(const char* instance, int mode, char* buf, uint64_t cap, uint64_t* len,
                         char* csv, uint64_t csvcap, uint64_t* csvlen) {
  int st = 0;
  const int g = guard([&] {
    std::istringstream is(instance);
    const ProblemInstance inst = load_instance(is);
    const SensingOperator op = make_operator(inst);
    SolveConfig cfg = default_config(inst.k, l2_norm(inst.y));
    cfg.correlation_mode = mode_of(mode);
    const RecoveryResult res = omp_solve(op, inst.y, cfg);
    std::ostringstream os, oc;
    save_result(res, os);
    res.costs.write_csv(oc);
    st = put_text(os.str(), buf, cap, len);
    if (!st) st = put_text(oc.str(), csv, csvcap, csvlen);
  });
  return g ? g : st;
}

/* the FlopCounter bookkeeping recipe (tests/cpp/counts_recipe.inc) on an
 * instance text */
int fmpo_ref_counts_text(const char* instance, char* buf, uint64_t cap, uint64_t* len) {
  int st = 0;
  const int g = guard([&] { st = put_text(flop_counts_text(instance), buf, cap, len); });
  return g ? g : st;
}

}  // extern "C"
