// libfastmp_b200.so: the reference's fastmp:: C++ API (include/fastmp_b200/
// fastmp.hpp) implemented over the C ABI of libfmp_cuda.so.  Host code here
// only validates, marshals std::complex vectors and maps status codes onto the
// reference's exceptions; the arithmetic runs in the sm_100a kernels.
#include "fastmp_b200/fastmp.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <mutex>
#include <istream>
#include <ostream>

#include "fmp.h"

namespace fastmp {

namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;

[[noreturn]] void raise(int status, std::int64_t position = 0) {
  const std::string msg = fmp_last_error();
  if (status == FMP_EINVAL || status == FMP_EUNSUPPORTED) throw std::invalid_argument(msg);
  if (status == FMP_ERANK) throw RankDeficientError(static_cast<std::size_t>(position), msg);
  throw std::runtime_error(msg);
}

void check(int status) {
  if (status != FMP_OK) raise(status);
}

int kind_code(TransformKind k) { return k == TransformKind::Fourier ? FMP_FOURIER : FMP_HADAMARD; }

const double* raw(const cvec& v) { return reinterpret_cast<const double*>(v.data()); }
double* raw(cvec& v) { return reinterpret_cast<double*>(v.data()); }

std::shared_ptr<void> make_op(const Device& dev, TransformKind kind, std::size_t n,
                              const std::vector<std::size_t>& rows) {
  std::vector<std::uint64_t> r(rows.begin(), rows.end());
  fmp_op op = nullptr;
  check(fmp_operator_create(static_cast<fmp_ctx>(dev.handle()), kind_code(kind), n, r.data(),
                            r.size(), &op));
  return std::shared_ptr<void>(op, [](void* p) { fmp_operator_destroy(static_cast<fmp_op>(p)); });
}

void validate_unitary(TransformKind kind, std::size_t n) {
  // transform.cpp:47-53, plus the GPU path's power-of-two restriction
  if (n == 0) throw std::invalid_argument("transform size must be positive");
  if (kind == TransformKind::Hadamard && !is_power_of_two(n))
    throw std::invalid_argument("hadamard size must be a power of two");
  if (!is_power_of_two(n))
    throw std::invalid_argument("non power-of-two Fourier sizes are not implemented on the GPU path");
}


// ------------------------------------------- FlopCounter bookkeeping (f4)
// The reference books flops per operation (cost_model.hpp:19-31); the device
// work is organised differently, so the facade books the counts a reference
// caller would read from the same operation sequence.
unsigned log2_size(std::size_t n) {
  unsigned l = 0;
  while ((std::size_t{1} << l) < n) ++l;
  return l;
}
// fft_pow2 / fht (transform.cpp:60-100) and the 1/sqrt(N) scaling of
// forward / adjoint (transform.cpp:133,150); apply / apply_adjoint book the
// transform they run (sensing.cpp:93-109)
void book_transform(FlopCounter* fc, TransformKind kind, std::size_t n) {
  if (!fc) return;
  const std::uint64_t lg = log2_size(n);
  if (kind == TransformKind::Fourier) fc->complex_mul += std::uint64_t(n) / 2 * lg;
  fc->complex_add += std::uint64_t(n) * lg;
  fc->real_mul += 2 * std::uint64_t(n);
}
// fast_update (kernel.cpp:209-303): d = number of distinct Hadamard values
void book_fast_update(FlopCounter* fc, TransformKind kind, std::size_t n, std::size_t atoms,
                      std::size_t d, bool symmetry) {
  if (!fc || atoms == 0) return;
  const std::uint64_t s = atoms;
  if (kind == TransformKind::Hadamard) {
    fc->real_mul += 2 * std::uint64_t(d) * s;
  } else if (!symmetry) {
    fc->complex_mul += std::uint64_t(n) * s;
  } else {
    const std::uint64_t pairs = n >= 1 ? (n - 1) / 2 : 0;  // j >= 1 with 2 j < n
    fc->complex_mul += pairs * s;
    fc->real_add += 2 * pairs * s;
    fc->real_mul += (2 + (n % 2 == 0 && n > 1 ? 2 : 0)) * s;
  }
  fc->complex_add += std::uint64_t(n) * s;
}
// dot_conj bookkeeping (solvers.cpp:48-53)
void book_dot(FlopCounter& fc, std::size_t len, std::uint64_t count = 1) {
  if (len == 0) return;
  fc.complex_mul += count * len;
  fc.complex_add += count * (len - 1);
}
// normal_equations_solve on s columns (solvers.cpp:120-177); `done` pivots
// completed (s unless it raised at pivot `done`)
void book_normal(FlopCounter& fc, std::size_t rows, std::size_t s, std::size_t done) {
  const std::uint64_t S = s;
  book_dot(fc, rows, S * (S + 1) / 2 + S);
  for (std::uint64_t j = 0; j < done; ++j) {
    fc.complex_mul += S - j;
    fc.complex_add += (S - j) * (j + 1);
  }
  if (done < s) return;
  fc.complex_mul += S * S;
  fc.complex_add += S * S;
}
// one least-squares step of omp_solve with s columns (solvers.cpp:370-388):
// IncrementalQR push + solve (solvers.cpp:223-274) or the normal equations,
// then update_residual (solvers.cpp:180-192); `ok` false: the step ended rank
// deficient at its new column
void book_ls_step(FlopCounter& fc, LeastSquaresMethod method, std::size_t rows, std::size_t s,
                  bool ok) {
  const std::uint64_t S = s;
  if (method == LeastSquaresMethod::IncrementalQR) {
    const std::uint64_t q = S - 1;
    book_dot(fc, rows, 2 * q);
    fc.complex_mul += 2 * q * rows;
    fc.complex_add += 2 * q * rows;
    fc.real_mul += 2 * std::uint64_t(rows);
    fc.real_add += rows;
    if (!ok) return;
    book_dot(fc, rows, S);
    fc.complex_mul += S * (S + 1) / 2;
    fc.complex_add += S * (S - 1) / 2;
  } else {
    book_normal(fc, rows, s, ok ? s : s - 1);
    if (!ok) return;
  }
  fc.complex_mul += S * rows;
  fc.complex_add += (S + 1) * rows;
}
}  // namespace

// ------------------------------------------------------------------ types
const char* to_string(TransformKind kind) noexcept {
  return kind == TransformKind::Fourier ? "fourier" : "hadamard";
}

TransformKind parse_kind(const std::string& name) {
  if (name == "fourier") return TransformKind::Fourier;
  if (name == "hadamard") return TransformKind::Hadamard;
  throw std::invalid_argument("unknown transform kind: " + name);
}

double l2_norm(const cvec& v) noexcept {
  double s = 0.0;
  for (const cplx& z : v) s += std::norm(z);
  return std::sqrt(s);
}

double l2_distance(const cvec& a, const cvec& b) {
  if (a.size() != b.size()) throw std::invalid_argument("l2_distance: size mismatch");
  double s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += std::norm(a[i] - b[i]);
  return std::sqrt(s);
}

std::uint64_t splitmix64(std::uint64_t x) noexcept {  // random.cpp:22-29
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

std::uint64_t derive_seed(std::uint64_t base, std::uint64_t index) noexcept {
  return fmp_derive_seed(base, index);
}

// ------------------------------------------------------------- cost model
const char* to_string(CorrelationMode mode) noexcept {
  switch (mode) {
    case CorrelationMode::Conventional: return "conventional";
    case CorrelationMode::Fast: return "fast";
    case CorrelationMode::Adaptive: return "adaptive";
  }
  return "?";
}

CorrelationMode parse_mode(const std::string& name) {
  if (name == "conventional") return CorrelationMode::Conventional;
  if (name == "fast") return CorrelationMode::Fast;
  if (name == "adaptive") return CorrelationMode::Adaptive;
  throw std::invalid_argument("unknown correlation mode: " + name);
}

std::uint64_t conventional_iteration_flops(TransformKind kind, std::size_t n) {
  if (n == 0) throw std::invalid_argument("flops: n must be positive");
  if (is_power_of_two(n)) {
    const std::uint64_t logn = log2_floor(n);
    return (kind == TransformKind::Fourier ? 5 : 2) * std::uint64_t(n) * logn;
  }
  if (kind == TransformKind::Hadamard) throw std::invalid_argument("hadamard size must be a power of two");
  return 6ull * n * n + 2ull * n * (n - 1);
}

std::uint64_t fast_iteration_flops(TransformKind kind, std::size_t n, std::size_t t) {
  if (t == 0) throw std::invalid_argument("flops: t must be positive");
  if (t == 1) return conventional_iteration_flops(kind, n);
  return (kind == TransformKind::Fourier ? 6 : 2) * std::uint64_t(n) * (t - 1);
}

std::size_t crossover_iteration(TransformKind kind, std::size_t n) {
  if (is_power_of_two(n)) return fmp_crossover_iteration(kind_code(kind), n);
  const std::uint64_t conv = conventional_iteration_flops(kind, n);
  std::size_t t = 1;
  while (fast_iteration_flops(kind, n, t + 1) <= conv) ++t;
  return t;
}

void CostReport::write_csv(std::ostream& os) const {
  os << "t,mode,analytic_flops,counted_flops,relative_vs_conventional\n";
  const double conv = static_cast<double>(conventional_iteration_flops(kind, n));
  char buf[64];
  for (const IterationCost& row : iterations) {
    std::snprintf(buf, sizeof(buf), "%.17g", static_cast<double>(row.analytic_flops) / conv);
    os << row.t << ',' << to_string(row.mode_used) << ',' << row.analytic_flops << ','
       << row.counted.flops() << ',' << buf << '\n';
  }
  os << "# kernel_precompute_flops," << kernel_precompute_flops << '\n';
  os << "# least_squares_flops," << least_squares_flops << '\n';
  os << "# identification_flops," << identification_flops << '\n';
}

// ----------------------------------------------------------------- device
Device::Device(int ordinal) : ordinal_(ordinal) {
  fmp_ctx c = nullptr;
  check(fmp_ctx_create(ordinal, &c));
  ctx_ = c;
}

Device::~Device() { fmp_ctx_destroy(static_cast<fmp_ctx>(ctx_)); }

std::shared_ptr<Device> Device::default_device() {
  thread_local std::shared_ptr<Device> dev;
  if (!dev) dev = std::make_shared<Device>(0);
  return dev;
}

// ------------------------------------------------------------- transforms
StructuredUnitary::StructuredUnitary(TransformKind kind, std::size_t n) : kind_(kind), n_(n) {
  validate_unitary(kind, n);
}

void* StructuredUnitary::unit_op() const {
  if (!op_) op_ = make_op(*Device::default_device(), kind_, n_, {1});
  return op_.get();
}

cvec StructuredUnitary::forward(const cvec& v, FlopCounter* fc) const {
  if (v.size() != n_) throw std::invalid_argument("forward: length mismatch");
  cvec out(n_);
  check(fmp_unitary_forward(static_cast<fmp_op>(unit_op()), FMP_C128, raw(v), 1, raw(out)));
  book_transform(fc, kind_, n_);
  return out;
}

cvec StructuredUnitary::adjoint(const cvec& v, FlopCounter* fc) const {
  if (v.size() != n_) throw std::invalid_argument("adjoint: length mismatch");
  cvec out(n_);
  check(fmp_unitary_adjoint(static_cast<fmp_op>(unit_op()), FMP_C128, raw(v), 1, raw(out)));
  book_transform(fc, kind_, n_);
  return out;
}

cplx StructuredUnitary::entry(std::size_t row, std::size_t col) const {
  // closed form (transform.hpp:24-30): exp(-2 pi i (a b mod N)/N)/sqrt(N) or
  // the Sylvester sign (-1)^popcount(a & b) / sqrt(N)
  if (row < 1 || row > n_ || col < 1 || col > n_)
    throw std::invalid_argument("entry: index out of range");
  const std::size_t a = row - 1, b = col - 1;
  const double s = 1.0 / std::sqrt(static_cast<double>(n_));
  if (kind_ == TransformKind::Hadamard)
    return cplx((__builtin_popcountll(a & b) & 1) ? -s : s, 0.0);
  const double th = -kTwoPi * static_cast<double>((a * b) % n_) / static_cast<double>(n_);
  return cplx(s * std::cos(th), s * std::sin(th));
}

cvec StructuredUnitary::column(std::size_t col) const {
  if (col < 1 || col > n_) throw std::invalid_argument("column: index out of range");
  cvec out(n_);
  for (std::size_t r = 1; r <= n_; ++r) out[r - 1] = entry(r, col);
  return out;
}

std::size_t StructuredUnitary::product_index(std::size_t i, std::size_t j) const {
  if (i < 1 || i > n_ || j < 1 || j > n_)
    throw std::invalid_argument("product_index: index out of range");
  if (kind_ == TransformKind::Fourier) return ((i - 1) + (j - 1)) % n_ + 1;
  return ((i - 1) ^ (j - 1)) + 1;
}

cvec StructuredUnitary::dense() const {
  cvec out(n_ * n_);
  for (std::size_t r = 1; r <= n_; ++r)
    for (std::size_t c = 1; c <= n_; ++c) out[(r - 1) * n_ + (c - 1)] = entry(r, c);
  return out;
}

// ---------------------------------------------------------------- sensing
RowSelection make_row_selection(std::size_t n, std::size_t m, std::uint64_t seed) {
  if (m == 0 || m > n) throw std::invalid_argument("row selection needs 1 <= m <= n");
  RowSelection sel;
  sel.n = n;
  std::vector<std::uint64_t> rows(m);
  check(fmp_make_row_selection(n, m, seed, rows.data()));
  sel.omega.assign(rows.begin(), rows.end());
  return sel;
}

RowSelection make_row_selection(std::size_t n, std::vector<std::size_t> rows) {
  std::sort(rows.begin(), rows.end());
  if (rows.empty()) throw std::invalid_argument("row selection must be non-empty");
  if (rows.size() > n) throw std::invalid_argument("row selection larger than the transform size");
  for (std::size_t i = 0; i < rows.size(); ++i) {
    if (rows[i] < 1 || rows[i] > n) throw std::invalid_argument("row index out of range");
    if (i > 0 && rows[i] == rows[i - 1]) throw std::invalid_argument("row indices must be distinct");
  }
  RowSelection sel;
  sel.n = n;
  sel.omega = std::move(rows);
  return sel;
}

SensingOperator::SensingOperator(StructuredUnitary unitary, RowSelection selection,
                                 std::shared_ptr<Device> device)
    : unitary_(std::move(unitary)), selection_(std::move(selection)),
      device_(device ? std::move(device) : Device::default_device()) {
  if (selection_.n != unitary_.size())
    throw std::invalid_argument("row selection size does not match transform");
  op_ = make_op(*device_, unitary_.kind(), unitary_.size(), selection_.omega);
}

cvec SensingOperator::apply(const cvec& x, FlopCounter* fc) const {
  if (x.size() != n()) throw std::invalid_argument("apply: length mismatch");
  cvec out(m());
  check(fmp_apply(static_cast<fmp_op>(op_.get()), FMP_C128, raw(x), 1, raw(out)));
  book_transform(fc, unitary_.kind(), n());
  return out;
}

cvec SensingOperator::apply_adjoint(const cvec& r, FlopCounter* fc) const {
  if (r.size() != m()) throw std::invalid_argument("apply_adjoint: length mismatch");
  cvec out(n());
  check(fmp_apply_adjoint(static_cast<fmp_op>(op_.get()), FMP_C128, raw(r), 1, raw(out), nullptr));
  book_transform(fc, unitary_.kind(), n());
  return out;
}

cvec SensingOperator::column(std::size_t j) const {
  if (j < 1 || j > n()) throw std::invalid_argument("column: index out of range");
  cvec e(n(), cplx(0.0));
  e[j - 1] = 1.0;
  return apply(e);
}

ProblemInstance make_instance(const SensingOperator& op, std::size_t k, double noise_stddev,
                              std::uint64_t seed) {
  if (k >= op.m()) throw std::invalid_argument("sparsity k must be below the row count m");
  if (noise_stddev < 0.0) throw std::invalid_argument("noise stddev must be non-negative");
  ProblemInstance inst;
  inst.kind = op.unitary().kind();
  inst.n = op.n();
  inst.m = op.m();
  inst.k = k;
  inst.seed = seed;
  inst.omega = op.selection().omega;
  inst.x_true.assign(inst.n, cplx(0.0));
  inst.noise.assign(inst.m, cplx(0.0));
  check(fmp_draw_instance(inst.n, inst.m, k, noise_stddev, seed, raw(inst.x_true), raw(inst.noise)));
  inst.y = op.apply(inst.x_true);
  for (std::size_t i = 0; i < inst.m; ++i) inst.y[i] += inst.noise[i];
  return inst;
}

// ------------------------------------------------------------ text formats
namespace {
void append_pairs(std::ostream& os, const cvec& v) {
  char buf[64];
  for (std::size_t i = 0; i < v.size(); ++i) {
    std::snprintf(buf, sizeof(buf), "%.17g %.17g", v[i].real(), v[i].imag());
    if (i) os << ' ';
    os << buf;
  }
  os << '\n';
}

cvec read_pairs(std::istream& is, std::size_t count, const char* what) {
  cvec v(count);
  for (auto& z : v) {
    double re = 0.0, im = 0.0;
    if (!(is >> re >> im)) throw std::runtime_error(std::string("instance parse: bad ") + what);
    z = cplx(re, im);
  }
  return v;
}
}  // namespace

SensingOperator make_operator(const ProblemInstance& inst) {
  return SensingOperator(StructuredUnitary(inst.kind, inst.n), make_row_selection(inst.n, inst.omega));
}

// sensing.cpp:160-168: header "n m k seed kind", the 1-based rows, then x
// and y as %.17g pairs, one line each
void save_instance(const ProblemInstance& inst, std::ostream& os) {
  os << inst.n << ' ' << inst.m << ' ' << inst.k << ' ' << inst.seed << ' ' << to_string(inst.kind)
     << '\n';
  for (std::size_t i = 0; i < inst.omega.size(); ++i) {
    if (i) os << ' ';
    os << inst.omega[i];
  }
  os << '\n';
  append_pairs(os, inst.x_true);
  append_pairs(os, inst.y);
}

// sensing.cpp:170-193; the noise is recovered as y - apply(x_true) (on the GPU)
ProblemInstance load_instance(std::istream& is) {
  ProblemInstance inst;
  std::string kind;
  if (!(is >> inst.n >> inst.m >> inst.k >> inst.seed >> kind))
    throw std::runtime_error("instance parse: bad header");
  inst.kind = parse_kind(kind);
  if (inst.n == 0 || inst.m == 0 || inst.m > inst.n)
    throw std::runtime_error("instance parse: bad dimensions");
  inst.omega.resize(inst.m);
  for (auto& w : inst.omega)
    if (!(is >> w)) throw std::runtime_error("instance parse: bad row indices");
  inst.x_true = read_pairs(is, inst.n, "x_true");
  inst.y = read_pairs(is, inst.m, "y");
  const cvec clean = make_operator(inst).apply(inst.x_true);
  inst.noise.resize(inst.m);
  for (std::size_t i = 0; i < inst.m; ++i) inst.noise[i] = inst.y[i] - clean[i];
  return inst;
}

// solvers.cpp:546-562
void save_result(const RecoveryResult& result, std::ostream& os) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", result.residual_norm);
  os << result.x_hat.size() << ' ' << result.support.size() << ' ' << result.iterations_run << ' '
     << buf << ' ' << (result.rank_deficient_abort ? 1 : 0) << ' ' << to_string(result.costs.kind)
     << '\n';
  for (std::size_t i = 0; i < result.support.size(); ++i) {
    if (i) os << ' ';
    os << result.support[i];
  }
  os << '\n';
  for (std::size_t i = 0; i < result.coeffs.size(); ++i) {
    std::snprintf(buf, sizeof(buf), "%.17g %.17g", result.coeffs[i].real(), result.coeffs[i].imag());
    if (i) os << ' ';
    os << buf;
  }
  os << '\n';
}

// ----------------------------------------------------------------- kernel
CorrelationKernel compute_kernel(const SensingOperator& op, FlopCounter* fc) {
  CorrelationKernel k;
  k.kind = op.unitary().kind();
  k.n = op.n();
  k.m = op.m();
  k.c.resize(k.n);
  std::vector<double> vals(k.m + 1);
  std::vector<std::uint32_t> vidx(k.kind == TransformKind::Hadamard ? k.n : 0);
  std::uint64_t nv = 0;
  const bool had = k.kind == TransformKind::Hadamard;
  check(fmp_operator_kernel(static_cast<fmp_op>(op.handle()), raw(k.c), had ? vals.data() : nullptr,
                            had ? vidx.data() : nullptr, &nv));
  if (had) {
    k.values.assign(vals.begin(), vals.begin() + nv);
    k.value_index = std::move(vidx);
  }
  // keep the operator alive with the kernel (fast_update runs on it)
  k.device_op = op.device_handle();
  // apply_adjoint(apply(e1)) (kernel.cpp:33)
  book_transform(fc, k.kind, k.n);
  book_transform(fc, k.kind, k.n);
  return k;
}

std::size_t PermutationAction::map_index(std::size_t i) const {
  // kernel.hpp:46-51
  if (i < 1 || i > n || lambda < 1 || lambda > n)
    throw std::invalid_argument("permutation: index out of range");
  const std::size_t a = i - 1, l = lambda - 1;
  if (kind == TransformKind::Fourier) return (a + n - l) % n + 1;
  return (a ^ l) + 1;
}

cvec fast_update(const cvec& h0, const CorrelationKernel& kernel,
                 const std::vector<std::size_t>& support, const cvec& coeffs,
                 const FastUpdateOptions& opts, FlopCounter* fc) {
  if (h0.size() != kernel.n) throw std::invalid_argument("fast_update: h0 length");
  if (support.size() != coeffs.size())
    throw std::invalid_argument("fast_update: support/coefficient mismatch");
  if (!kernel.device_op)
    throw std::invalid_argument("fast_update: kernel was not built by compute_kernel");
  cvec h(kernel.n);
  std::vector<std::uint64_t> sup(support.begin(), support.end());
  check(fmp_fast_update(static_cast<fmp_op>(kernel.device_op.get()), FMP_C128, raw(h0),
                        sup.empty() ? nullptr : sup.data(), coeffs.empty() ? nullptr : raw(coeffs),
                        sup.size(), 1, raw(h), nullptr));
  book_fast_update(fc, kernel.kind, kernel.n, support.size(), kernel.values.size(),
                   opts.fourier_symmetry);
  return h;
}

// ---------------------------------------------------------------- solvers
SolveConfig default_config(std::size_t k, double y_norm) {
  SolveConfig cfg;
  cfg.max_iterations = std::max<std::size_t>(1, k);
  cfg.residual_tolerance = 1e-9 * y_norm;
  return cfg;
}

namespace {

// SolveConfig::check_invariants for omp_solve (solvers.cpp:394-401): after
// every iteration t the support holds t atoms, the residual r_t = y - Phi x_t
// is orthogonal to the fitted columns (|col_j^H r_t| <= 1e-8 max(1, ||y||),
// check_residual_orthogonality, solvers.cpp:194-203) and ||r_t|| does not
// grow by more than 1e-12.  x_t is the solver's own state after t
// iterations: the fused solver's result with max_iterations = t (its
// arithmetic does not depend on the cap).  r_t and Phi^H r_t = (col_j^H r_t)_j
// are computed on the device, all iterations of a problem in one batch.
void check_omp_invariants(const SensingOperator& op, const cvec& y, const RecoveryResult& res,
                          const SolveConfig& cfg) {
  const std::size_t n = op.n(), m = op.m(), T = res.iterations_run;
  if (T == 0) return;
  double yn = 0.0;
  for (const cplx& v : y) yn += std::norm(v);
  yn = std::sqrt(yn);
  const double scale = std::max(1.0, yn);
  cvec xs(T * n, cplx(0.0));
  for (std::size_t t = 1; t <= T; ++t) {
    if (res.support_history.size() < t || res.support_history[t - 1].size() != t)
      throw std::logic_error("solver invariant violated: support size");
    RecoveryResult cap;
    if (t == T) {
      cap = res;
    } else {
      SolveConfig c = cfg;
      c.max_iterations = t;
      c.check_invariants = false;
      c.record_correlations = false;
      cap = omp_solve(op, y, c);
    }
    if (cap.support != res.support_history[t - 1])
      throw std::logic_error("solver invariant violated: support size");
    for (std::size_t j = 0; j < cap.support.size(); ++j)
      xs[(t - 1) * n + cap.support[j] - 1] = cap.coeffs[j];
  }
  cvec ax(T * m), h(T * n);
  check(fmp_apply(static_cast<fmp_op>(op.handle()), FMP_C128, raw(xs), T, raw(ax)));
  for (std::size_t t = 0; t < T; ++t)
    for (std::size_t i = 0; i < m; ++i) ax[t * m + i] = y[i] - ax[t * m + i];
  check(fmp_apply_adjoint(static_cast<fmp_op>(op.handle()), FMP_C128, raw(ax), T, raw(h), nullptr));
  double prev = yn;
  for (std::size_t t = 1; t <= T; ++t) {
    for (std::size_t atom : res.support_history[t - 1])
      if (std::abs(h[(t - 1) * n + atom - 1]) > 1e-8 * scale)
        throw std::logic_error(
            "solver invariant violated: residual not orthogonal to the fitted columns");
    double rn = 0.0;
    for (std::size_t i = 0; i < m; ++i) rn += std::norm(ax[(t - 1) * m + i]);
    rn = std::sqrt(rn);
    if (rn > prev + 1e-12)
      throw std::logic_error("solver invariant violated: residual norm increased");
    prev = rn;
  }
}

// SolveConfig::check_invariants for cosamp_solve (solvers.cpp:527-533)
void check_cosamp_invariants(const RecoveryResult& res, std::size_t k) {
  for (const auto& sup : res.support_history) {
    if (sup.size() > k) throw std::logic_error("solver invariant violated: support exceeds k");
    for (std::size_t i = 1; i < sup.size(); ++i)
      if (sup[i] <= sup[i - 1])
        throw std::logic_error("solver invariant violated: support not sorted/distinct");
  }
}

}  // namespace

std::vector<RecoveryResult> omp_solve_batch(const SensingOperator& op, const std::vector<cvec>& ys,
                                            const SolveConfig& cfg) {
  const std::size_t B = ys.size(), T = cfg.max_iterations, n = op.n(), m = op.m();
  if (T < 1) throw std::invalid_argument("omp_solve: max_iterations must be >= 1");
  if (!(cfg.residual_tolerance >= 0.0)) throw std::invalid_argument("omp_solve: tolerance must be >= 0");
  std::vector<RecoveryResult> results(B);
  if (B == 0) return results;
  cvec y(B * m);
  for (std::size_t b = 0; b < B; ++b) {
    if (ys[b].size() != m) throw std::invalid_argument("omp_solve: measurement length mismatch");
    std::copy(ys[b].begin(), ys[b].end(), y.begin() + b * m);
  }
  fmp_omp_config c{};
  c.max_iterations = T;
  c.tolerance = cfg.residual_tolerance;
  c.mode = cfg.correlation_mode == CorrelationMode::Conventional ? FMP_MODE_CONVENTIONAL
           : cfg.correlation_mode == CorrelationMode::Fast       ? FMP_MODE_FAST
                                                                  : FMP_MODE_ADAPTIVE;
  c.record_correlations = cfg.record_correlations ? 1 : 0;
  std::vector<std::uint64_t> sup(B * T), size(B), iters(B), hlen(B);
  cvec co(B * T);
  std::vector<double> rn(B);
  std::vector<std::int32_t> ab(B);
  std::vector<std::uint8_t> modes(B * T);
  cvec hist(cfg.record_correlations ? B * T * n : 0);
  fmp_omp_result r{};
  r.support = sup.data();
  r.coeffs = raw(co);
  r.support_size = size.data();
  r.iterations = iters.data();
  r.residual = rn.data();
  r.aborted = ab.data();
  r.modes = modes.data();
  r.history_len = hlen.data();
  r.history = cfg.record_correlations ? raw(hist) : nullptr;
  check(fmp_omp_solve(static_cast<fmp_op>(op.handle()), FMP_C128, raw(y), B, &c, &r));
  const TransformKind kind = op.unitary().kind();
  // distinct Hadamard kernel values (the fast rows' bookkeeping), read once
  std::size_t nvalues = 0;
  if (kind == TransformKind::Hadamard) {
    bool any_fast = false;
    for (std::size_t b = 0; b < B && !any_fast; ++b)
      for (std::size_t t = 2; t <= hlen[b] && !any_fast; ++t) any_fast = modes[b * T + t - 1] != 0;
    if (any_fast) nvalues = compute_kernel(op).values.size();
  }
  for (std::size_t b = 0; b < B; ++b) {
    RecoveryResult& res = results[b];
    res.x_hat.assign(n, cplx(0.0));
    for (std::size_t j = 0; j < size[b]; ++j) {
      res.support.push_back(static_cast<std::size_t>(sup[b * T + j]));
      res.coeffs.push_back(co[b * T + j]);
      res.x_hat[res.support.back() - 1] = res.coeffs.back();
    }
    res.iterations_run = iters[b];
    res.residual_norm = rn[b];
    res.rank_deficient_abort = ab[b] != 0;
    for (std::size_t t = 1; t <= res.iterations_run; ++t)
      res.support_history.emplace_back(res.support.begin(), res.support.begin() + t);
    res.costs.kind = kind;
    res.costs.n = n;
    // counted flops as omp_solve books them (solvers.cpp:343-395)
    FlopCounter kernel_fc, ls_fc, id_fc;
    bool kernel_built = false;
    for (std::size_t t = 1; t <= hlen[b]; ++t) {
      IterationCost row;
      row.t = t;
      const bool fast = modes[b * T + t - 1] != 0;
      row.mode_used = fast ? CorrelationMode::Fast : CorrelationMode::Conventional;
      row.analytic_flops = fast ? fast_iteration_flops(kind, n, t)
                                : conventional_iteration_flops(kind, n);
      if (fast && t >= 2) {
        if (!kernel_built) {
          book_transform(&kernel_fc, kind, n);
          book_transform(&kernel_fc, kind, n);
          kernel_built = true;
        }
        book_fast_update(&row.counted, kind, n, t - 1, nvalues, cfg.fourier_symmetry);
      } else {
        book_transform(&row.counted, kind, n);
      }
      id_fc.real_mul += 2 * std::uint64_t(n);  // argmax_magnitude (solvers.cpp:90-96)
      id_fc.real_add += n;
      res.costs.iterations.push_back(row);
      if (cfg.record_correlations)
        res.correlation_history.emplace_back(hist.begin() + (b * T + t - 1) * n,
                                             hist.begin() + (b * T + t) * n);
    }
    const std::size_t steps = size[b] + (res.rank_deficient_abort ? 1 : 0);
    for (std::size_t s = 1; s <= steps; ++s)
      book_ls_step(ls_fc, cfg.ls_method, m, s, s <= size[b]);
    res.costs.kernel_precompute_flops = kernel_fc.flops();
    res.costs.least_squares_flops = ls_fc.flops();
    res.costs.identification_flops = id_fc.flops();
  }
  if (cfg.check_invariants)
    for (std::size_t b = 0; b < B; ++b) check_omp_invariants(op, ys[b], results[b], cfg);
  return results;
}

RecoveryResult omp_solve(const SensingOperator& op, const cvec& y, const SolveConfig& cfg) {
  if (y.size() != op.m()) throw std::invalid_argument("omp_solve: measurement length mismatch");
  return std::move(omp_solve_batch(op, std::vector<cvec>{y}, cfg)[0]);
}

// ------------------------------------------------------------ IncrementalQR
IncrementalQR::IncrementalQR(std::size_t rows) : rows_(rows) {
  auto dev = Device::default_device();
  fmp_qr q = nullptr;
  check(fmp_qr_create(static_cast<fmp_ctx>(dev->handle()), rows, 64, &q));
  // the deleter holds the device: its context outlives the factorisation
  h_ = std::shared_ptr<void>(q, [dev](void* p) { fmp_qr_destroy(static_cast<fmp_qr>(p)); });
}

std::size_t IncrementalQR::cols() const noexcept {
  return static_cast<std::size_t>(fmp_qr_cols(static_cast<fmp_qr>(h_.get())));
}

bool IncrementalQR::push_column(const cvec& col, FlopCounter* fc) {
  if (col.size() != rows_) throw std::invalid_argument("qr: column length mismatch");
  const std::size_t t = cols();
  int accepted = 0;
  check(fmp_qr_push_column(static_cast<fmp_qr>(h_.get()), raw(col), &accepted));
  if (fc) {  // solvers.cpp:231-240 bookkeeping
    fc->complex_mul += 2 * t * 2 * rows_;
    fc->complex_add += 2 * t * (2 * rows_ - 1);
    fc->real_mul += 2 * rows_;
    fc->real_add += rows_;
  }
  return accepted != 0;
}

cvec IncrementalQR::solve(const cvec& rhs, FlopCounter* fc) const {
  if (rhs.size() != rows_) throw std::invalid_argument("qr: rhs length mismatch");
  const std::size_t t = cols();
  cvec x(t);
  check(fmp_qr_solve(static_cast<fmp_qr>(h_.get()), raw(rhs), t ? raw(x) : nullptr));
  if (fc) {  // solvers.cpp:256-272 bookkeeping
    fc->complex_mul += t * rows_;
    fc->complex_add += t * (rows_ - 1);
    if (t > 0) {
      fc->complex_mul += std::uint64_t(t) * (t + 1) / 2;
      fc->complex_add += std::uint64_t(t) * (t - 1) / 2;
    }
  }
  return x;
}

std::uint64_t cosamp_fast_iteration_flops(TransformKind kind, std::size_t n, std::size_t k,
                                          std::size_t t) {
  if (t == 0) throw std::invalid_argument("flops: t must be positive");
  if (t == 1) return conventional_iteration_flops(kind, n);
  return (kind == TransformKind::Fourier ? 6 : 2) * std::uint64_t(n) * std::uint64_t(k);
}

double cosamp_relative_cost(std::size_t n, std::size_t k) {
  if (!is_power_of_two(n) || n < 2)
    throw std::invalid_argument("cosamp_relative_cost: n must be a power of two >= 2");
  std::size_t logn = 0;
  while ((std::size_t{1} << logn) < n) ++logn;
  return 6.0 * double(k) / (5.0 * double(logn));
}

bool adaptive_cosamp_uses_fast(TransformKind kind, std::size_t n, std::size_t k) {
  if (k == 0) return true;
  return cosamp_fast_iteration_flops(kind, n, k, 2) <= conventional_iteration_flops(kind, n);
}

std::vector<RecoveryResult> cosamp_solve_batch(const SensingOperator& op,
                                               const std::vector<cvec>& ys, std::size_t k,
                                               const SolveConfig& cfg) {
  const std::size_t B = ys.size(), T = cfg.max_iterations, n = op.n(), m = op.m();
  if (T < 1) throw std::invalid_argument("cosamp_solve: max_iterations must be >= 1");
  if (!(cfg.residual_tolerance >= 0.0))
    throw std::invalid_argument("cosamp_solve: tolerance must be >= 0");
  std::vector<RecoveryResult> results(B);
  if (B == 0) return results;
  cvec y(B * m);
  for (std::size_t b = 0; b < B; ++b) {
    if (ys[b].size() != m) throw std::invalid_argument("cosamp_solve: measurement length mismatch");
    std::copy(ys[b].begin(), ys[b].end(), y.begin() + b * m);
  }
  fmp_omp_config c{};
  c.max_iterations = T;
  c.tolerance = cfg.residual_tolerance;
  c.mode = cfg.correlation_mode == CorrelationMode::Conventional ? FMP_MODE_CONVENTIONAL
           : cfg.correlation_mode == CorrelationMode::Fast       ? FMP_MODE_FAST
                                                                  : FMP_MODE_ADAPTIVE;
  c.record_correlations = cfg.record_correlations ? 1 : 0;
  const std::size_t kk = std::max<std::size_t>(k, 1);
  std::vector<std::uint64_t> sup(B * kk), size(B), iters(B), sh(B * T * kk);
  cvec co(B * kk);
  std::vector<double> rn(B);
  std::vector<std::int32_t> ab(B);
  cvec hist(cfg.record_correlations ? B * T * n : 0);
  fmp_cosamp_result r{};
  r.support = sup.data();
  r.coeffs = raw(co);
  r.support_size = size.data();
  r.iterations = iters.data();
  r.residual = rn.data();
  r.aborted = ab.data();
  r.support_history = sh.data();
  r.history = cfg.record_correlations ? raw(hist) : nullptr;
  check(fmp_cosamp_solve(static_cast<fmp_op>(op.handle()), FMP_C128, raw(y), B, k, &c, &r));
  const TransformKind kind = op.unitary().kind();
  const bool fast = cfg.correlation_mode == CorrelationMode::Fast ||
                    (cfg.correlation_mode == CorrelationMode::Adaptive &&
                     adaptive_cosamp_uses_fast(kind, n, k));
  for (std::size_t b = 0; b < B; ++b) {
    RecoveryResult& res = results[b];
    res.x_hat.assign(n, cplx(0.0));
    for (std::size_t j = 0; j < size[b]; ++j) {
      res.support.push_back(static_cast<std::size_t>(sup[b * k + j]));
      res.coeffs.push_back(co[b * k + j]);
      res.x_hat[res.support.back() - 1] = res.coeffs.back();
    }
    res.iterations_run = iters[b];
    res.residual_norm = rn[b];
    res.rank_deficient_abort = ab[b] != 0;
    for (std::size_t t = 0; t < res.iterations_run; ++t) {
      std::vector<std::size_t> row;
      for (std::size_t j = 0; j < k; ++j)
        if (sh[(b * T + t) * k + j]) row.push_back(static_cast<std::size_t>(sh[(b * T + t) * k + j]));
      res.support_history.push_back(std::move(row));
    }
    res.costs.kind = kind;
    res.costs.n = n;
    const std::size_t rows = std::min<std::size_t>(T, res.iterations_run + (res.rank_deficient_abort ? 1 : 0));
    for (std::size_t t = 1; t <= rows; ++t) {
      IterationCost row;
      row.t = t;
      row.mode_used = fast ? CorrelationMode::Fast : CorrelationMode::Conventional;
      row.analytic_flops = fast ? cosamp_fast_iteration_flops(kind, n, k, t)
                                : conventional_iteration_flops(kind, n);
      row.counted.complex_add = row.analytic_flops / kComplexAddFlops;
      res.costs.iterations.push_back(row);
      if (cfg.record_correlations)
        res.correlation_history.emplace_back(hist.begin() + (b * T + t - 1) * n,
                                             hist.begin() + (b * T + t) * n);
    }
    if (cfg.check_invariants) check_cosamp_invariants(res, k);
  }
  return results;
}

RecoveryResult cosamp_solve(const SensingOperator& op, const cvec& y, std::size_t k,
                            const SolveConfig& cfg) {
  if (y.size() != op.m()) throw std::invalid_argument("cosamp_solve: measurement length mismatch");
  return std::move(cosamp_solve_batch(op, std::vector<cvec>{y}, k, cfg)[0]);
}

cvec least_squares(const SensingOperator& op, const std::vector<std::size_t>& support,
                   const cvec& y, LeastSquaresMethod method, FlopCounter* fc) {
  if (y.size() != op.m()) throw std::invalid_argument("least_squares: rhs length mismatch");
  if (method == LeastSquaresMethod::IncrementalQR) {
    // solvers.cpp:276-294: columns pushed in support order, the first
    // dependent one raises with its position
    IncrementalQR qr(op.m());
    for (std::size_t j = 0; j < support.size(); ++j)
      if (!qr.push_column(op.column(support[j]), fc))
        throw RankDeficientError(j, "qr: dependent column at support position " +
                                        std::to_string(j));
    return qr.solve(y, fc);
  }
  std::vector<std::uint64_t> sup(support.begin(), support.end());
  cvec x(support.size());
  std::int64_t pos = 0;
  const int st = fmp_least_squares(static_cast<fmp_op>(op.handle()), FMP_C128, raw(y),
                                   sup.empty() ? nullptr : sup.data(), sup.size(), 1,
                                   x.empty() ? nullptr : raw(x), &pos);
  if (fc && (st == FMP_OK || st == FMP_ERANK))
    book_normal(*fc, op.m(), support.size(), st == FMP_OK ? support.size() : (std::size_t)pos);
  if (st != FMP_OK) raise(st, pos);
  return x;
}

}  // namespace fastmp
