// C++ test of the drop-in facade (libfastmp_b200.so): the reference's own test
// recipes (proj/tests/test_kernel.cpp, test_solvers.cpp, test_sensing.cpp)
// written against the same fastmp:: API, plus agreement with the CPU oracle
// (oracle/_build/libfmp_oracle.so, loaded with dlopen as test infrastructure).
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <sstream>
#include <string>
#include <tuple>

#include "fastmp_b200/fastmp.hpp"

using namespace fastmp;

#include "counts_recipe.inc"

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                                 \
  do {                                                                              \
    if (cond) ++g_pass;                                                             \
    else { ++g_fail; std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); } \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                                 \
  do {                                                                              \
    bool thrown_ = false;                                                           \
    try { (void)(expr); } catch (const type&) { thrown_ = true; } catch (...) {}    \
    CHECK(thrown_);                                                                 \
  } while (0)

// oracle ABI subset (oracle/oracle_abi.h)
struct OSolveConfig { uint64_t max_iterations; double tol; int mode, ls, sym, record; };
struct OSolveResult {
  uint64_t* support; double* coeffs; uint64_t support_size, iterations_run; double residual_norm;
  int rank_deficient_abort; uint64_t history_len; double* hist; int* mode_used;
};
using omp_fn = int (*)(int, uint64_t, const uint64_t*, uint64_t, const double*, const OSolveConfig*,
                       OSolveResult*);
using ls_fn = int (*)(int, uint64_t, const uint64_t*, uint64_t, const uint64_t*, uint64_t, const double*,
                      int, double*, uint64_t*);

static cvec gaussian(std::size_t n, std::uint64_t seed) {
  // deterministic test data (not the reference RNG): Box-Muller on splitmix
  cvec v(n);
  std::uint64_t s = seed;
  for (auto& z : v) {
    s = splitmix64(s);
    const double u1 = ((s >> 11) + 1.0) * 0x1.0p-53;
    s = splitmix64(s);
    const double u2 = (s >> 11) * 0x1.0p-53;
    z = std::polar(std::sqrt(-std::log(u1)), 6.283185307179586 * u2);
  }
  return v;
}

int main(int argc, char** argv) {
  const char* oracle_path = argc > 1 ? argv[1] : "oracle/_build/libfmp_oracle.so";
  void* orc = dlopen(oracle_path, RTLD_NOW | RTLD_LOCAL);
  omp_fn oracle_omp = orc ? reinterpret_cast<omp_fn>(dlsym(orc, "fmpo_omp_solve")) : nullptr;
  if (!oracle_omp) std::fprintf(stderr, "oracle not loaded: %s\n", dlerror());
  ls_fn oracle_ls = orc ? reinterpret_cast<ls_fn>(dlsym(orc, "fmpo_least_squares")) : nullptr;

  // kernel invariants (test_kernel.cpp:65-107)
  {
    SensingOperator op(StructuredUnitary(TransformKind::Fourier, 64), make_row_selection(64, 16, 3));
    const CorrelationKernel k = compute_kernel(op);
    CHECK(k.c[0].imag() == 0.0 && k.c[32].imag() == 0.0);
    bool sym = true;
    for (std::size_t j = 1; j < 64; ++j) sym &= k.c[j] == std::conj(k.c[64 - j]);
    CHECK(sym);
    CHECK(std::abs(k.c[0] - cplx(16.0 / 64.0)) < 1e-12);
    SensingOperator oh(StructuredUnitary(TransformKind::Hadamard, 64), make_row_selection(64, 16, 3));
    const CorrelationKernel kh = compute_kernel(oh);
    CHECK(!kh.values.empty() && kh.values.size() <= 17);
    CHECK(std::is_sorted(kh.values.begin(), kh.values.end()));
    bool lat = true;
    for (std::size_t j = 0; j < 64; ++j)
      lat &= kh.c[j].real() == kh.values[kh.value_index[j]] && kh.c[j].imag() == 0.0;
    CHECK(lat);
  }
  // permutation closed forms (test_kernel.cpp:109-131)
  {
    CHECK((PermutationAction{TransformKind::Fourier, 8, 2}.map_index(1) == 8));
    CHECK((PermutationAction{TransformKind::Fourier, 8, 2}.map_index(2) == 1));
    CHECK((PermutationAction{TransformKind::Hadamard, 8, 3}.map_index(8) == 6));
    CHECK_THROWS_AS((PermutationAction{TransformKind::Fourier, 8, 9}.map_index(1)), std::invalid_argument);
    StructuredUnitary h8(TransformKind::Hadamard, 8), f8(TransformKind::Fourier, 8);
    CHECK(h8.product_index(4, 6) == 7 && f8.product_index(4, 6) == 1);
  }
  // fast update = conventional correlation of the residual (test_kernel.cpp:178-219)
  {
    int cases = 0;
    for (TransformKind kind : {TransformKind::Fourier, TransformKind::Hadamard})
      for (std::size_t n : {8, 32, 128, 1024})
        for (int trial = 0; trial < 8; ++trial) {
          const std::uint64_t seed = derive_seed(60, n * 1000 + trial + (kind == TransformKind::Hadamard ? 7 : 0));
          const std::size_t m = 2 + seed % (n - 2), k = 1 + (seed >> 20) % std::min<std::size_t>(8, m);
          SensingOperator op(StructuredUnitary(kind, n), make_row_selection(n, m, seed));
          const CorrelationKernel ker = compute_kernel(op);
          const cvec y = gaussian(m, seed + 1);
          std::vector<std::size_t> sup;
          for (std::size_t j = 0; sup.size() < k; ++j) {
            const std::size_t a = 1 + splitmix64(seed + 17 * j) % n;
            if (std::find(sup.begin(), sup.end(), a) == sup.end()) sup.push_back(a);
          }
          const cvec co = gaussian(k, seed + 2);
          cvec xs(n, cplx(0.0));
          for (std::size_t j = 0; j < k; ++j) xs[sup[j] - 1] = co[j];
          cvec r = y;
          const cvec ax = op.apply(xs);
          for (std::size_t i = 0; i < m; ++i) r[i] -= ax[i];
          const cvec want = op.apply_adjoint(r);
          const cvec got = fast_update(op.apply_adjoint(y), ker, sup, co);
          CHECK(l2_distance(got, want) <= 1e-10 * std::max(l2_norm(want), 1e-300));
          ++cases;
        }
    CHECK(cases == 64);
  }
  // validation (test_kernel.cpp:221-236, test_sensing.cpp:25-45)
  {
    SensingOperator op(StructuredUnitary(TransformKind::Hadamard, 16), make_row_selection(16, 4, 1));
    const CorrelationKernel ker = compute_kernel(op);
    const cvec h0(16, cplx(1.0));
    CHECK(fast_update(h0, ker, {}, {}) == h0);
    CHECK_THROWS_AS(fast_update(cvec(15), ker, {}, {}), std::invalid_argument);
    CHECK_THROWS_AS(fast_update(h0, ker, {1, 1}, cvec(2, cplx(1.0))), std::invalid_argument);
    CHECK_THROWS_AS(fast_update(h0, ker, {0}, cvec(1, cplx(1.0))), std::invalid_argument);
    CHECK_THROWS_AS(fast_update(h0, ker, {17}, cvec(1, cplx(1.0))), std::invalid_argument);
    CHECK_THROWS_AS(make_row_selection(16, {3, 3, 5}), std::invalid_argument);
    CHECK_THROWS_AS(make_row_selection(16, 17, 1), std::invalid_argument);
    CHECK_THROWS_AS(StructuredUnitary(TransformKind::Hadamard, 12), std::invalid_argument);
    CHECK(make_row_selection(16, {9, 2, 5}).omega == (std::vector<std::size_t>{2, 5, 9}));
  }
  // least squares and rank errors (test_solvers.cpp:39-86)
  {
    SensingOperator op(StructuredUnitary(TransformKind::Hadamard, 32), make_row_selection(32, 8, 5));
    const ProblemInstance inst = make_instance(op, 2, 0.0, 6);
    bool rank = false;
    try {
      least_squares(op, {7, 7}, inst.y);
    } catch (const RankDeficientError& e) {
      rank = e.position() == 1;
    }
    CHECK(rank);
    SensingOperator of(StructuredUnitary(TransformKind::Fourier, 64), make_row_selection(64, 16, 3));
    const ProblemInstance fi = make_instance(of, 5, 0.1, 4);
    const std::vector<std::size_t> sup{3, 17, 29, 40, 61};
    const cvec b = least_squares(of, sup, fi.y);
    cvec r = fi.y;
    for (std::size_t j = 0; j < sup.size(); ++j) {
      const cvec col = of.column(sup[j]);
      for (std::size_t i = 0; i < r.size(); ++i) r[i] -= b[j] * col[i];
    }
    bool orth = true;
    for (std::size_t a : sup) {
      const cvec col = of.column(a);
      cplx g = 0.0;
      for (std::size_t i = 0; i < r.size(); ++i) g += std::conj(col[i]) * r[i];
      orth &= std::abs(g) < 1e-10 * l2_norm(fi.y);
    }
    CHECK(orth);
  }
  // modes walk identical supports; agreement with the oracle (test_solvers.cpp:157-186)
  {
    for (TransformKind kind : {TransformKind::Fourier, TransformKind::Hadamard})
      for (int trial = 0; trial < 10; ++trial) {
        const std::uint64_t seed = derive_seed(70, trial);
        SensingOperator op(StructuredUnitary(kind, 128), make_row_selection(128, 32, derive_seed(seed, 1)));
        const ProblemInstance inst = make_instance(op, 5, 0.05, seed);
        SolveConfig cfg = default_config(inst.k, l2_norm(inst.y));
        cfg.record_correlations = true;
        cfg.correlation_mode = CorrelationMode::Conventional;
        const RecoveryResult conv = omp_solve(op, inst.y, cfg);
        cfg.correlation_mode = CorrelationMode::Fast;
        const RecoveryResult fast = omp_solve(op, inst.y, cfg);
        cfg.correlation_mode = CorrelationMode::Adaptive;
        const RecoveryResult adap = omp_solve(op, inst.y, cfg);
        CHECK(conv.support_history == fast.support_history);
        CHECK(conv.support_history == adap.support_history);
        CHECK(conv.correlation_history.size() == fast.correlation_history.size());
        for (std::size_t i = 0; i < conv.correlation_history.size(); ++i)
          CHECK(l2_distance(fast.correlation_history[i], conv.correlation_history[i]) <=
                1e-10 * std::max(l2_norm(conv.correlation_history[i]), 1e-300));
        if (oracle_omp) {
          std::vector<uint64_t> om(op.selection().omega.begin(), op.selection().omega.end());
          std::vector<uint64_t> osup(5);
          std::vector<double> oco(10);
          OSolveConfig oc{5, cfg.residual_tolerance, 1, 0, 0, 0};
          OSolveResult orr{osup.data(), oco.data(), 0, 0, 0.0, 0, 0, nullptr, nullptr};
          CHECK(oracle_omp(kind == TransformKind::Fourier ? 0 : 1, 128, om.data(), om.size(),
                           reinterpret_cast<const double*>(inst.y.data()), &oc, &orr) == 0);
          CHECK(std::equal(fast.support.begin(), fast.support.end(), osup.begin()) &&
                fast.support.size() == orr.support_size);
          double err = 0.0, nrm = 0.0;
          for (std::size_t j = 0; j < fast.coeffs.size(); ++j) {
            err += std::norm(fast.coeffs[j] - cplx(oco[2 * j], oco[2 * j + 1]));
            nrm += std::norm(cplx(oco[2 * j], oco[2 * j + 1]));
          }
          CHECK(std::sqrt(err) <= 1e-10 * std::sqrt(nrm));
        }
      }
  }
  // adaptive switch (test_solvers.cpp:210-234)
  {
    SensingOperator op(StructuredUnitary(TransformKind::Fourier, 64), make_row_selection(64, 32, 41));
    const ProblemInstance inst = make_instance(op, 10, 0.0, 42);
    SolveConfig cfg = default_config(inst.k, l2_norm(inst.y));
    cfg.correlation_mode = CorrelationMode::Adaptive;
    cfg.max_iterations = 10;
    cfg.residual_tolerance = 0.0;
    const RecoveryResult res = omp_solve(op, inst.y, cfg);
    CHECK(crossover_iteration(TransformKind::Fourier, 64) == 6);
    CHECK(res.costs.iterations.size() == 10);
    bool ok = true;
    for (const IterationCost& row : res.costs.iterations)
      ok &= (row.t <= 6) == (row.mode_used == CorrelationMode::Fast);
    CHECK(ok);
  }
  // noiseless recovery and edge cases (test_solvers.cpp:88-141)
  {
    for (TransformKind kind : {TransformKind::Fourier, TransformKind::Hadamard}) {
      SensingOperator op(StructuredUnitary(kind, 64), make_row_selection(64, 32, 11));
      const ProblemInstance inst = make_instance(op, 3, 0.0, 12);
      const RecoveryResult res = omp_solve(op, inst.y, default_config(inst.k, l2_norm(inst.y)));
      CHECK(res.iterations_run == 3);
      CHECK(l2_distance(res.x_hat, inst.x_true) < 1e-8 * l2_norm(inst.x_true));
      CHECK(res.residual_norm < 1e-9 * l2_norm(inst.y));
    }
    SensingOperator op(StructuredUnitary(TransformKind::Fourier, 32), make_row_selection(32, 8, 21));
    const RecoveryResult zero = omp_solve(op, cvec(8, cplx(0.0)), default_config(2, 0.0));
    CHECK(zero.iterations_run == 0 && zero.support.empty() && zero.residual_norm == 0.0);
    CHECK_THROWS_AS(omp_solve(op, cvec(7), default_config(1, 1.0)), std::invalid_argument);
  }
  // SolveConfig::check_invariants (test_solvers.cpp:88-107, :133-141, :236-250):
  // the checks run and pass on exact recoveries, past the sparsity with
  // tolerance 0 (monotone residual), in every mode, and for CoSaMP
  {
    for (TransformKind kind : {TransformKind::Fourier, TransformKind::Hadamard})
      for (CorrelationMode mode : {CorrelationMode::Fast, CorrelationMode::Conventional,
                                   CorrelationMode::Adaptive}) {
        SensingOperator op(StructuredUnitary(kind, 64), make_row_selection(64, 32, 11));
        const ProblemInstance inst = make_instance(op, 3, 0.0, 12);
        SolveConfig cfg = default_config(inst.k, l2_norm(inst.y));
        cfg.correlation_mode = mode;
        cfg.check_invariants = true;
        bool threw = false;
        RecoveryResult res;
        try { res = omp_solve(op, inst.y, cfg); } catch (const std::logic_error&) { threw = true; }
        CHECK(!threw && res.iterations_run == 3);
        // past the sparsity with tolerance 0 (test_solvers.cpp:133-141's instance)
        SensingOperator od(StructuredUnitary(kind, 32), make_row_selection(32, 8, 21));
        const ProblemInstance di = make_instance(od, 4, 0.0, 22);
        SolveConfig deep = default_config(di.k, l2_norm(di.y));
        deep.correlation_mode = mode;
        deep.max_iterations = 8;
        deep.residual_tolerance = 0.0;
        deep.check_invariants = true;
        threw = false;
        try { res = omp_solve(od, di.y, deep); } catch (const std::logic_error& e) {
          threw = true;
          std::fprintf(stderr, "deep (%s, mode %d): %s\n", to_string(kind), (int)mode, e.what());
        }
        CHECK(!threw && res.iterations_run >= 4);
        SensingOperator on(StructuredUnitary(kind, 256), make_row_selection(256, 64, 5));
        const ProblemInstance noisy = make_instance(on, 6, 0.05, 9);
        SolveConfig nc = default_config(noisy.k, l2_norm(noisy.y));
        nc.correlation_mode = mode;
        nc.max_iterations = 12;
        nc.residual_tolerance = 0.0;
        nc.check_invariants = true;
        threw = false;
        try { res = omp_solve(on, noisy.y, nc); } catch (const std::logic_error&) { threw = true; }
        CHECK(!threw && res.iterations_run == 12);
      }
    SensingOperator op(StructuredUnitary(TransformKind::Fourier, 64), make_row_selection(64, 32, 51));
    const ProblemInstance inst = make_instance(op, 4, 0.0, 52);
    SolveConfig cfg = default_config(inst.k, l2_norm(inst.y));
    cfg.max_iterations = 8;
    cfg.check_invariants = true;
    bool threw = false;
    try { (void)cosamp_solve(op, inst.y, inst.k, cfg); } catch (const std::logic_error&) { threw = true; }
    CHECK(!threw);
  }
  // least squares in both methods (test_solvers.cpp:39-86)
  {
    SensingOperator op(StructuredUnitary(TransformKind::Fourier, 64), make_row_selection(64, 16, 3));
    const ProblemInstance inst = make_instance(op, 5, 0.1, 4);
    const std::vector<std::size_t> support{3, 17, 29, 40, 61};
    const cvec a = least_squares(op, support, inst.y, LeastSquaresMethod::IncrementalQR);
    const cvec b = least_squares(op, support, inst.y, LeastSquaresMethod::NormalEquations);
    CHECK(a.size() == 5);
    bool close = a.size() == b.size();
    for (std::size_t i = 0; close && i < a.size(); ++i) close = std::abs(a[i] - b[i]) < 1e-8;
    CHECK(close);
    cvec r = inst.y;
    for (std::size_t j = 0; j < support.size(); ++j) {
      const cvec col = op.column(support[j]);
      for (std::size_t i = 0; i < r.size(); ++i) r[i] -= a[j] * col[i];
    }
    bool orth = true;
    for (std::size_t atom : support) {
      const cvec col = op.column(atom);
      cplx g = 0.0;
      for (std::size_t i = 0; i < r.size(); ++i) g += std::conj(col[i]) * r[i];
      orth &= std::abs(g) < 1e-10 * l2_norm(inst.y);
    }
    CHECK(orth);
    SensingOperator oh(StructuredUnitary(TransformKind::Hadamard, 32), make_row_selection(32, 8, 5));
    const ProblemInstance ih = make_instance(oh, 2, 0.0, 6);
    const std::vector<std::size_t> dup{7, 7};
    for (LeastSquaresMethod mth : {LeastSquaresMethod::IncrementalQR, LeastSquaresMethod::NormalEquations}) {
      std::size_t pos = 99;
      try {
        least_squares(oh, dup, ih.y, mth);
      } catch (const RankDeficientError& e) {
        pos = e.position();
      }
      CHECK(pos == 1);
    }
  }
  // IncrementalQR (test_solvers.cpp:65-86 recipe; agreement with the oracle's
  // two-pass MGS least squares, solvers.cpp:222-274)
  {
    SensingOperator op(StructuredUnitary(TransformKind::Hadamard, 32), make_row_selection(32, 8, 5));
    IncrementalQR qr(8);
    const cvec col = op.column(3);
    CHECK(qr.push_column(col));
    CHECK(!qr.push_column(col));
    CHECK(qr.cols() == 1);
    for (auto [kind, n, m, s] : {std::tuple{TransformKind::Fourier, std::size_t(256), std::size_t(64), 12},
                                 std::tuple{TransformKind::Hadamard, std::size_t(1024), std::size_t(256), 24},
                                 std::tuple{TransformKind::Fourier, std::size_t(65536), std::size_t(16384), 40}}) {
      SensingOperator o2(StructuredUnitary(kind, n), make_row_selection(n, m, 77 + s));
      const ProblemInstance in2 = make_instance(o2, 8, 0.05, 78 + s);
      IncrementalQR q2(m);
      std::vector<std::uint64_t> sup;
      for (int j = 0; j < s; ++j) {
        const std::size_t atom = 1 + (std::size_t(j) * 7919 + 13) % n;
        CHECK(q2.push_column(o2.column(atom)));
        sup.push_back(atom);
      }
      const cvec x = q2.solve(in2.y);
      CHECK(x.size() == sup.size());
      if (oracle_ls) {
        std::vector<uint64_t> om(o2.selection().omega.begin(), o2.selection().omega.end());
        std::vector<double> ox(2 * sup.size());
        uint64_t aux = 0;
        CHECK(oracle_ls(kind == TransformKind::Fourier ? 0 : 1, n, om.data(), m, sup.data(), sup.size(),
                        reinterpret_cast<const double*>(in2.y.data()), 0, ox.data(), &aux) == 0);
        double err = 0.0, nrm = 0.0;
        for (std::size_t j = 0; j < x.size(); ++j) {
          err += std::norm(x[j] - cplx(ox[2 * j], ox[2 * j + 1]));
          nrm += std::norm(cplx(ox[2 * j], ox[2 * j + 1]));
        }
        CHECK(std::sqrt(err) <= 1e-10 * std::sqrt(nrm));
      }
    }
  }
  // CoSaMP (test_solvers.cpp:236-305, test_cost_model.cpp:93-108)
  {
    CHECK(cosamp_fast_iteration_flops(TransformKind::Hadamard, 1024, 8, 2) == 2 * 1024 * 8);
    CHECK(cosamp_relative_cost(8192, 4) == 24.0 / 65.0);
    CHECK(adaptive_cosamp_uses_fast(TransformKind::Fourier, 8192, 4));
    CHECK(!adaptive_cosamp_uses_fast(TransformKind::Fourier, 8192, 16));
    for (TransformKind kind : {TransformKind::Fourier, TransformKind::Hadamard}) {
      SensingOperator op(StructuredUnitary(kind, 64), make_row_selection(64, 32, 51));
      const ProblemInstance inst = make_instance(op, 4, 0.0, 52);
      SolveConfig cfg = default_config(inst.k, l2_norm(inst.y));
      cfg.max_iterations = 8;
      const RecoveryResult res = cosamp_solve(op, inst.y, inst.k, cfg);
      std::vector<std::size_t> want;
      for (std::size_t j = 0; j < 64; ++j)
        if (inst.x_true[j] != cplx(0.0)) want.push_back(j + 1);
      CHECK(res.support == want);
      CHECK(res.residual_norm < 1e-9 * l2_norm(inst.y));
      CHECK(l2_distance(res.x_hat, inst.x_true) < 1e-8 * l2_norm(inst.x_true));
    }
    SensingOperator op(StructuredUnitary(TransformKind::Fourier, 64), make_row_selection(64, 8, 61));
    const ProblemInstance inst = make_instance(op, 4, 0.0, 62);
    const RecoveryResult empty = cosamp_solve(op, inst.y, 0, default_config(1, l2_norm(inst.y)));
    CHECK(empty.iterations_run == 0 && empty.support.empty());
    SolveConfig cfg = default_config(4, l2_norm(inst.y));
    cfg.max_iterations = 6;
    cfg.residual_tolerance = 0.0;
    cfg.correlation_mode = CorrelationMode::Conventional;
    const RecoveryResult conv = cosamp_solve(op, inst.y, 4, cfg);
    cfg.correlation_mode = CorrelationMode::Fast;
    const RecoveryResult fast = cosamp_solve(op, inst.y, 4, cfg);
    CHECK(conv.rank_deficient_abort && fast.rank_deficient_abort);
    CHECK(conv.support_history == fast.support_history);
    CHECK(conv.iterations_run == fast.iterations_run);
    for (TransformKind kind : {TransformKind::Fourier, TransformKind::Hadamard})
      for (int trial = 0; trial < 10; ++trial) {
        const std::uint64_t seed = derive_seed(80, trial);
        SensingOperator op2(StructuredUnitary(kind, 128), make_row_selection(128, 64, derive_seed(seed, 1)));
        const ProblemInstance in2 = make_instance(op2, 4, 0.05, seed);
        SolveConfig c2 = default_config(in2.k, l2_norm(in2.y));
        c2.record_correlations = true;
        c2.max_iterations = 6;
        c2.correlation_mode = CorrelationMode::Conventional;
        const RecoveryResult a = cosamp_solve(op2, in2.y, in2.k, c2);
        c2.correlation_mode = CorrelationMode::Fast;
        const RecoveryResult b = cosamp_solve(op2, in2.y, in2.k, c2);
        CHECK(a.support_history == b.support_history);
        CHECK(a.correlation_history.size() == b.correlation_history.size());
        for (std::size_t i = 0; i < a.correlation_history.size(); ++i)
          CHECK(l2_distance(b.correlation_history[i], a.correlation_history[i]) <=
                1e-10 * std::max(l2_norm(a.correlation_history[i]), 1e-300));
      }
  }
  // text formats against the reference's own files (tests/golden/*.txt, *.csv
  // written by save_instance / save_result / write_csv, make_golden.py)
  if (argc > 2) {
    const std::string dir = argv[2];
    auto slurp = [](const std::string& path) {
      std::ifstream f(path, std::ios::binary);
      std::ostringstream o;
      o << f.rdbuf();
      return o.str();
    };
    const char* stems[] = {"fourier_64_32_4_11", "hadamard_64_32_4_12", "fourier_256_64_8_13",
                           "hadamard_1024_256_16_14"};
    int files = 0;
    for (const char* stem : stems) {
      const std::string want = slurp(dir + "/instance_" + stem + ".txt");
      if (want.empty()) continue;
      ++files;
      std::istringstream is(want);
      const ProblemInstance inst = load_instance(is);
      std::ostringstream os;
      save_instance(inst, os);
      CHECK(os.str() == want);  // byte-for-byte round trip
      double nn = 0.0;
      for (const cplx& z : inst.noise) nn += std::norm(z);
      CHECK(std::sqrt(nn) < 0.2 * std::sqrt(double(inst.m)));  // noise recovered by apply()
      // FlopCounter bookkeeping: the reference's counts_*.txt line for line
      {
        const std::string got = flop_counts_text(want), ref = slurp(dir + "/counts_" + stem + ".txt");
        CHECK(!ref.empty() && got == ref);
        if (got != ref) std::fprintf(stderr, "counts %s:\n%s\nreference:\n%s\n", stem, got.c_str(), ref.c_str());
      }
      const SensingOperator op = make_operator(inst);
      for (const char* mode : {"conventional", "fast"}) {
        SolveConfig cfg = default_config(inst.k, l2_norm(inst.y));
        cfg.correlation_mode = parse_mode(mode);
        const RecoveryResult res = omp_solve(op, inst.y, cfg);
        std::ostringstream ro;
        save_result(res, ro);
        std::istringstream got(ro.str()), ref(slurp(dir + "/result_" + stem + "_" + mode + ".txt"));
        std::size_t gn, gs, gi, rn_, rs, ri;
        double gr, rr;
        int ga, ra;
        std::string gk, rk;
        got >> gn >> gs >> gi >> gr >> ga >> gk;
        ref >> rn_ >> rs >> ri >> rr >> ra >> rk;
        CHECK(gn == rn_ && gs == rs && gi == ri && ga == ra && gk == rk);
        CHECK(std::abs(gr - rr) <= 1e-10 * l2_norm(inst.y));
        bool same = true;
        for (std::size_t j = 0; j < rs; ++j) {
          std::size_t a = 0, b = 0;
          got >> a;
          ref >> b;
          same &= a == b;
        }
        CHECK(same);
        double err = 0.0, nrm = 0.0;
        for (std::size_t j = 0; j < 2 * rs; ++j) {
          double a = 0.0, b = 0.0;
          got >> a;
          ref >> b;
          err += (a - b) * (a - b);
          nrm += b * b;
        }
        CHECK(std::sqrt(err) <= 1e-10 * std::sqrt(nrm));
        // cost CSV: the reference's file line for line (t, mode, analytic and
        // counted flops, relative cost; counted totals)
        std::ostringstream co;
        res.costs.write_csv(co);
        std::istringstream gc(co.str()), rc(slurp(dir + "/costs_" + stem + "_" + mode + ".csv"));
        std::string gl, rl;
        bool rows_ok = true;
        while (std::getline(rc, rl)) {
          if (!std::getline(gc, gl)) { rows_ok = false; break; }
          if (rl.rfind("#", 0) == 0) {  // counted totals (kernel, least squares, identification)
            rows_ok &= gl == rl;
            continue;
          }
          auto cols = [](const std::string& l) {
            std::vector<std::string> v;
            std::stringstream ss(l);
            std::string c;
            while (std::getline(ss, c, ',')) v.push_back(c);
            return v;
          };
          const auto a = cols(gl), b = cols(rl);
          rows_ok &= a.size() == 5 && b.size() == 5 && a[0] == b[0] && a[1] == b[1] &&
                     a[2] == b[2] && a[3] == b[3] && a[4] == b[4];
        }
        CHECK(rows_ok);
      }
    }
    CHECK(files == 4);
  }
  std::printf("facade test: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
