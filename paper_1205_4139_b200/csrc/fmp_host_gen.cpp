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
  unsigned w = threads > 0 ? unsigned(threads) : std::max(1u, std::thread::hardware_concurrency());
  // run f(lo, hi) over [0, count) in w contiguous chunks
  auto par = [&](uint64_t count, unsigned nt, auto&& f) {
    nt = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(nt, count)));
    std::vector<std::thread> pool;
    const uint64_t chunk = (count + nt - 1) / nt;
    for (unsigned t = 1; t < nt; ++t)
      pool.emplace_back([&, t] { f(std::min(count, t * chunk), std::min(count, (t + 1) * chunk)); });
    f(0, std::min(count, chunk));
    for (auto& th : pool) th.join();
  };
  std::vector<cplx> tw;
  if (kind == FMP_FOURIER) {
    tw.resize(n);
    par(n, w, [&](uint64_t lo, uint64_t hi) {
      for (uint64_t e = lo; e < hi; ++e) {
        const double th = -kTwoPi * static_cast<double>(e) / static_cast<double>(n);
        tw[e] = cplx(isn * std::cos(th), isn * std::sin(th));
      }
    });
  }
  // the draws of one signal, in make_instance's order (sensing.cpp:132-147)
  struct Draw {
    std::vector<uint64_t> sup;
    std::vector<cplx> xs, noise;
    double nn = 0.0;
  };
  auto draw = [&](uint64_t b) {
    Draw d;
    Rng rng(fmp_derive_seed(base_seed, first + b));
    d.sup = rng.sample(n, k);
    d.xs.resize(k);
    for (uint64_t i = 0; i < k; ++i) {
      const cplx z = rng.cgauss();
      d.xs[i] = real ? cplx(std::sqrt(2.0) * z.real(), 0.0) : z;
    }
    d.noise.assign(m, cplx(0.0));
    if (!real && noise_stddev > 0.0) {
      const double sc = noise_stddev * std::sqrt(2.0);
      for (uint64_t i = 0; i < m; ++i) {
        d.noise[i] = rng.cgauss() * sc;
        d.nn += std::norm(d.noise[i]);
      }
    }
    return d;
  };
  // y rows [lo, hi) of signal b synthesised from its K nonzeros
  auto synth = [&](const Draw& d, uint64_t b, uint64_t lo, uint64_t hi) {
    double* y = y_out + 2 * m * b;
    for (uint64_t i = lo; i < hi; ++i) {
      const uint64_t a = rows[i] - 1;
      cplx acc(0.0);
      for (uint64_t j = 0; j < k; ++j) {
        const uint64_t c = d.sup[j] - 1;
        if (kind == FMP_FOURIER)
          acc += d.xs[j] * tw[(a * c) & (n - 1)];
        else
          acc += d.xs[j] * ((__builtin_popcountll(a & c) & 1) ? -isn : isn);
      }
      acc += d.noise[i];
      y[2 * i] = acc.real();
      y[2 * i + 1] = acc.imag();
    }
  };
  auto finish = [&](const Draw& d, uint64_t b) {
    if (x_out) {
      double* x = x_out + 2 * n * b;
      std::fill(x, x + 2 * n, 0.0);
      for (uint64_t j = 0; j < k; ++j) {
        x[2 * (d.sup[j] - 1)] = d.xs[j].real();
        x[2 * (d.sup[j] - 1) + 1] = d.xs[j].imag();
      }
    }
    if (noise_norm_out) noise_norm_out[b] = std::sqrt(d.nn);
  };
  if (batch >= w) {
    // many signals: one signal per thread at a time
    std::atomic<uint64_t> next{0};
    auto work = [&] {
      for (uint64_t b; (b = next.fetch_add(1)) < batch;) {
        const Draw d = draw(b);
        synth(d, b, 0, m);
        finish(d, b);
      }
    };
    std::vector<std::thread> pool;
    for (unsigned i = 1; i < w; ++i) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
  } else {
    // few (large) signals: the rows of each signal split over the threads
    for (uint64_t b = 0; b < batch; ++b) {
      const Draw d = draw(b);
      par(m, w, [&](uint64_t lo, uint64_t hi) { synth(d, b, lo, hi); });
      finish(d, b);
    }
  }
  return FMP_OK;
}
