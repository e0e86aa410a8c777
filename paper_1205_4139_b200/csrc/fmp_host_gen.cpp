// Seeded synthetic problem generation for the bench / parity harness.
//
// Follows the reference's generators: Rng = std::mt19937_64 with hand-rolled
// distributions (random.hpp:32-54, random.cpp:34-67), make_row_selection
// (sensing.cpp:61-70), make_instance (sensing.cpp:119-153), and the harness
// rule for real N(0,1) nonzeros.  The measurement y = Phi x is
// synthesised directly from the K nonzeros with the closed-form entries of
// StructuredUnitary::entry (transform.cpp:154-163); it equals op.apply(x) up to
// rounding.  Signal b of a batch uses seed derive_seed(base, first + b), as the
// reference CLI's campaigns do (fastmp_cli.cpp:237-241).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdint>
#include <numeric>
#include <random>
#include <thread>
#include <vector>

#include "fmp.h"

namespace {

using cplx = std::complex<double>;
constexpr double kTwoPi = 6.283185307179586476925286766559;

uint64_t mix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

struct Rng {
  std::mt19937_64 e;
  explicit Rng(uint64_t s) : e(s) {}
  double unit() { return static_cast<double>(e() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t b) {
    const uint64_t limit = (UINT64_MAX / b) * b;
    uint64_t r;
    do r = e(); while (r >= limit);
    return r % b;
  }
  cplx cgauss() {
    const double u1 = (static_cast<double>(e() >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = unit();
    const double radius = std::sqrt(-std::log(u1));
    const double angle = 2.0 * M_PI * u2;
    return cplx(radius * std::cos(angle), radius * std::sin(angle));
  }
  std::vector<uint64_t> sample(uint64_t n, uint64_t m) {
    std::vector<uint64_t> pool(n);
    std::iota(pool.begin(), pool.end(), uint64_t{1});
    for (uint64_t i = 0; i < m; ++i) std::swap(pool[i], pool[i + below(n - i)]);
    pool.resize(m);
    std::sort(pool.begin(), pool.end());
    return pool;
  }
};

bool pow2(uint64_t n) { return n && !(n & (n - 1)); }

}  // namespace

extern "C" uint64_t fmp_derive_seed(uint64_t base, uint64_t index) {
  return mix(mix(base) ^ mix(index));
}

extern "C" int fmp_make_row_selection(uint64_t n, uint64_t m, uint64_t seed, uint64_t* rows) {
  if (m == 0 || m > n || !rows) return FMP_EINVAL;
  Rng rng(seed);
  const auto s = rng.sample(n, m);
  std::copy(s.begin(), s.end(), rows);
  return FMP_OK;
}

extern "C" int fmp_draw_instance(uint64_t n, uint64_t m, uint64_t k, double noise_stddev,
                                 uint64_t seed, double* x_out, double* noise_out) {
  if (k >= m || m > n || noise_stddev < 0.0 || !x_out || !noise_out) return FMP_EINVAL;
  Rng rng(seed);
  std::fill(x_out, x_out + 2 * n, 0.0);
  std::fill(noise_out, noise_out + 2 * m, 0.0);
  if (k > 0) {
    const auto sup = rng.sample(n, k);
    for (uint64_t idx : sup) {
      const cplx z = rng.cgauss();
      x_out[2 * (idx - 1)] = z.real();
      x_out[2 * (idx - 1) + 1] = z.imag();
    }
  }
  if (noise_stddev > 0.0) {
    const double sc = noise_stddev * std::sqrt(2.0);
    for (uint64_t i = 0; i < m; ++i) {
      const cplx z = rng.cgauss() * sc;
      noise_out[2 * i] = z.real();
      noise_out[2 * i + 1] = z.imag();
    }
  }
  return FMP_OK;
}

extern "C" int fmp_make_batch(int kind, uint64_t n, const uint64_t* rows, uint64_t m, uint64_t k,
                              double noise_stddev, int real, uint64_t base_seed, uint64_t first,
                              uint64_t batch, int threads, double* y_out, double* x_out,
                              double* noise_norm_out) {
  if ((kind != FMP_FOURIER && kind != FMP_HADAMARD) || !pow2(n) || m == 0 || m > n ||
      k >= m || noise_stddev < 0.0 || !rows || !y_out)
    return FMP_EINVAL;
  const double isn = 1.0 / std::sqrt(static_cast<double>(n));
  std::vector<cplx> tw;
  if (kind == FMP_FOURIER) {
    tw.resize(n);
    for (uint64_t e = 0; e < n; ++e) {
      const double th = -kTwoPi * static_cast<double>(e) / static_cast<double>(n);
      tw[e] = cplx(isn * std::cos(th), isn * std::sin(th));
    }
  }
  auto one = [&](uint64_t b) {
    Rng rng(fmp_derive_seed(base_seed, first + b));
    const auto sup = rng.sample(n, k);
    std::vector<cplx> xs(k);
    for (uint64_t i = 0; i < k; ++i) {
      const cplx z = rng.cgauss();
      xs[i] = real ? cplx(std::sqrt(2.0) * z.real(), 0.0) : z;
    }
    double* y = y_out + 2 * m * b;
    double nn = 0.0;
    std::vector<cplx> noise(m, cplx(0.0));
    if (!real && noise_stddev > 0.0) {
      const double sc = noise_stddev * std::sqrt(2.0);
      for (uint64_t i = 0; i < m; ++i) {
        noise[i] = rng.cgauss() * sc;
        nn += std::norm(noise[i]);
      }
    }
    for (uint64_t i = 0; i < m; ++i) {
      const uint64_t a = rows[i] - 1;
      cplx acc(0.0);
      for (uint64_t j = 0; j < k; ++j) {
        const uint64_t c = sup[j] - 1;
        if (kind == FMP_FOURIER)
          acc += xs[j] * tw[(a * c) % n];
        else
          acc += xs[j] * ((__builtin_popcountll(a & c) & 1) ? -isn : isn);
      }
      acc += noise[i];
      y[2 * i] = acc.real();
      y[2 * i + 1] = acc.imag();
    }
    if (x_out) {
      double* x = x_out + 2 * n * b;
      std::fill(x, x + 2 * n, 0.0);
      for (uint64_t j = 0; j < k; ++j) {
        x[2 * (sup[j] - 1)] = xs[j].real();
        x[2 * (sup[j] - 1) + 1] = xs[j].imag();
      }
    }
    if (noise_norm_out) noise_norm_out[b] = std::sqrt(nn);
  };
  unsigned w = threads > 0 ? unsigned(threads) : std::max(1u, std::thread::hardware_concurrency());
  w = unsigned(std::min<uint64_t>(w, std::max<uint64_t>(batch, 1)));
  std::atomic<uint64_t> next{0};
  auto work = [&] {
    for (uint64_t b; (b = next.fetch_add(1)) < batch;) one(b);
  };
  std::vector<std::thread> pool;
  for (unsigned i = 1; i < w; ++i) pool.emplace_back(work);
  work();
  for (auto& t : pool) t.join();
  return FMP_OK;
}
