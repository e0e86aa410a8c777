/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle (plain C restatement) of the
 * reference's OMP correlation path, /root/reference/proj (fastmp, C++20).
 *
 * It is the checker the GPU path is compared against; nothing in the product
 * package links or calls it.  Every function cites the reference file:line it
 * restates (paths relative to /root/reference/proj).  Arithmetic follows the
 * reference's operation order so that, compiled without FMA contraction
 * (-ffp-contract=off, as the reference's Release build is on x86-64 without
 * -march), its results agree bit for bit with oracle/_ref/libfmp_ref.so; the
 * tests in tests/test_oracle.py pin that agreement and also pin this file to
 * the golden vectors under tests/golden/ that the reference itself produced.
 *
 * Exports oracle/oracle_abi.h.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "oracle_abi.h"

typedef struct {
  double re, im;
} cx;

static inline cx cx_make(double re, double im) {
  cx z = {re, im};
  return z;
}
static inline cx cx_add(cx a, cx b) { return cx_make(a.re + b.re, a.im + b.im); }
static inline cx cx_sub(cx a, cx b) { return cx_make(a.re - b.re, a.im - b.im); }
/* (a.re + i a.im)(b.re + i b.im), GCC's inline order: ac - bd, ad + bc */
static inline cx cx_mul(cx a, cx b) {
  return cx_make(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re);
}
static inline cx cx_conj(cx a) { return cx_make(a.re, -a.im); }
static inline cx cx_scale(cx a, double s) { return cx_make(a.re * s, a.im * s); }
static inline cx cx_divr(cx a, double s) { return cx_make(a.re / s, a.im / s); }
static inline double cx_mag2(cx z) { return z.re * z.re + z.im * z.im; }

/* ---------------------------------------------------------------- random */

/* random.cpp:22-29 */
uint64_t fmpo_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

/* random.cpp:31-33 */
uint64_t fmpo_derive_seed(uint64_t base, uint64_t index) {
  return fmpo_splitmix64(fmpo_splitmix64(base) ^ fmpo_splitmix64(index));
}

/* std::mt19937_64 (random.hpp:32-54 wraps it); standard 64-bit Mersenne
 * Twister, seeded with the single-integer constructor. */
typedef struct {
  uint64_t mt[312];
  int idx;
} rng_t;

static void rng_seed(rng_t* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) +
               (uint64_t)i;
  r->idx = 312;
}

static uint64_t rng_next(rng_t* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (r->mt[i] & 0xFFFFFFFF80000000ULL) |
                         (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = v;
    }
    r->idx = 0;
  }
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* random.hpp:38-40 */
static double rng_unit(rng_t* r) {
  return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}

/* random.cpp:34-43: rejection sampling */
static uint64_t rng_below(rng_t* r, uint64_t b) {
  const uint64_t limit = (UINT64_MAX / b) * b;
  uint64_t v;
  do {
    v = rng_next(r);
  } while (v >= limit);
  return v % b;
}

/* random.cpp:45-53: radius^2 ~ Exp(1), uniform phase */
static cx rng_cgauss(rng_t* r) {
  const double u1 = ((double)(rng_next(r) >> 11) + 1.0) * 0x1.0p-53;
  const double u2 = rng_unit(r);
  const double radius = sqrt(-log(u1));
  const double angle = 2.0 * M_PI * u2;
  return cx_make(radius * cos(angle), radius * sin(angle));
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

/* random.cpp:55-67: partial Fisher-Yates, then sort */
static int rng_sample(rng_t* r, uint64_t n, uint64_t m, uint64_t* out) {
  if (m > n) return 1;
  uint64_t* pool = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  for (uint64_t i = 0; i < n; ++i) pool[i] = i + 1;
  for (uint64_t i = 0; i < m; ++i) {
    const uint64_t j = i + rng_below(r, n - i);
    const uint64_t t = pool[i];
    pool[i] = pool[j];
    pool[j] = t;
  }
  qsort(pool, m, sizeof(uint64_t), cmp_u64);
  memcpy(out, pool, sizeof(uint64_t) * m);
  free(pool);
  return 0;
}

void fmpo_rng_u64(uint64_t seed, uint64_t count, uint64_t* out) {
  rng_t r;
  rng_seed(&r, seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng_next(&r);
}

void fmpo_rng_complex_gaussian(uint64_t seed, uint64_t count, double* out) {
  rng_t r;
  rng_seed(&r, seed);
  for (uint64_t i = 0; i < count; ++i) {
    const cx z = rng_cgauss(&r);
    out[2 * i] = z.re;
    out[2 * i + 1] = z.im;
  }
}

int fmpo_rng_sample(uint64_t seed, uint64_t n, uint64_t m, uint64_t* out) {
  rng_t r;
  rng_seed(&r, seed);
  return rng_sample(&r, n, m, out);
}

/* ------------------------------------------------------------- transform */

static const double kTwoPi = 6.283185307179586476925286766559;

static int is_pow2(uint64_t n) { return n > 0 && (n & (n - 1)) == 0; }
static uint64_t log2_floor(uint64_t n) {
  uint64_t p = 0;
  while (n >>= 1) ++p;
  return p;
}

/* transform.cpp:28-36 */
static void bit_reverse_permute(cx* v, uint64_t n) {
  for (uint64_t i = 1, j = 0; i < n; ++i) {
    uint64_t bit = n >> 1;
    for (; j & bit; bit >>= 1) j ^= bit;
    j ^= bit;
    if (i < j) {
      const cx t = v[i];
      v[i] = v[j];
      v[j] = t;
    }
  }
}

/* transform.cpp:49-57: roots exp(-2 pi i k / N), N/2 of them (pow2) or N */
static cx* make_twiddles(uint64_t n) {
  const uint64_t count = is_pow2(n) ? (n > 1 ? n / 2 : 1) : n;
  cx* tw = (cx*)malloc(sizeof(cx) * count);
  for (uint64_t k = 0; k < count; ++k) {
    const double th = -kTwoPi * (double)k / (double)n;
    tw[k] = cx_make(cos(th), sin(th));
  }
  return tw;
}

/* transform.cpp:60-84: iterative radix-2 DIT */
static void fft_pow2(cx* v, uint64_t n, const cx* tw, int conjugate) {
  bit_reverse_permute(v, n);
  for (uint64_t len = 2; len <= n; len <<= 1) {
    const uint64_t half = len >> 1, step = n / len;
    for (uint64_t base = 0; base < n; base += len)
      for (uint64_t j = 0; j < half; ++j) {
        const cx w = conjugate ? cx_conj(tw[j * step]) : tw[j * step];
        const cx t = cx_mul(w, v[base + j + half]);
        const cx u = v[base + j];
        v[base + j] = cx_add(u, t);
        v[base + j + half] = cx_sub(u, t);
      }
  }
}

/* transform.cpp:86-100: in-place Walsh-Hadamard butterflies */
static void fht(cx* v, uint64_t n) {
  for (uint64_t half = 1; half < n; half <<= 1)
    for (uint64_t base = 0; base < n; base += half << 1)
      for (uint64_t j = base; j < base + half; ++j) {
        const cx a = v[j], b = v[j + half];
        v[j] = cx_add(a, b);
        v[j + half] = cx_sub(a, b);
      }
}

/* transform.cpp:102-118: O(N^2) fallback for non-power-of-two Fourier */
static void dense_fourier(const cx* v, cx* out, uint64_t n, const cx* tw,
                          int conjugate) {
  for (uint64_t a = 0; a < n; ++a) {
    cx acc = cx_make(0.0, 0.0);
    for (uint64_t b = 0; b < n; ++b) {
      const cx root = tw[(a * b) % n];
      acc = cx_add(acc, cx_mul(v[b], conjugate ? cx_conj(root) : root));
    }
    out[a] = acc;
  }
}

/* transform.cpp:120-152: forward / adjoint, then scale by 1/sqrt(N) */
static int transform(int kind, uint64_t n, const cx* v, cx* out, int adjoint) {
  if (n == 0 || (kind == 1 && !is_pow2(n)) || kind < 0 || kind > 1) return 1;
  const double inv_sqrt_n = 1.0 / sqrt((double)n);
  if (kind == 1) {
    memmove(out, v, sizeof(cx) * n);
    fht(out, n);
  } else {
    cx* tw = make_twiddles(n);
    if (is_pow2(n)) {
      memmove(out, v, sizeof(cx) * n);
      fft_pow2(out, n, tw, adjoint);
    } else {
      cx* tmp = (cx*)malloc(sizeof(cx) * n);
      dense_fourier(v, tmp, n, tw, adjoint);
      memcpy(out, tmp, sizeof(cx) * n);
      free(tmp);
    }
    free(tw);
  }
  for (uint64_t i = 0; i < n; ++i) out[i] = cx_scale(out[i], inv_sqrt_n);
  return 0;
}

int fmpo_forward(int kind, uint64_t n, const double* v, double* out) {
  return transform(kind, n, (const cx*)v, (cx*)out, 0);
}
int fmpo_adjoint(int kind, uint64_t n, const double* v, double* out) {
  return transform(kind, n, (const cx*)v, (cx*)out, 1);
}

/* transform.cpp:154-163 (sign_bit transform.cpp:38-40) */
static cx entry(int kind, uint64_t n, uint64_t row, uint64_t col) {
  const double inv_sqrt_n = 1.0 / sqrt((double)n);
  const uint64_t a = row - 1, b = col - 1;
  if (kind == 1) {
    const int sign = (__builtin_popcountll(a & b) & 1) ? -1 : 1;
    return cx_make((double)sign * inv_sqrt_n, 0.0);
  }
  const uint64_t e = (a * b) % n;
  const double th = -kTwoPi * (double)e / (double)n;
  return cx_make(inv_sqrt_n * cos(th), inv_sqrt_n * sin(th));
}

int fmpo_entry(int kind, uint64_t n, uint64_t row, uint64_t col, double* out2) {
  if (row < 1 || row > n || col < 1 || col > n) return 1;
  const cx e = entry(kind, n, row, col);
  out2[0] = e.re;
  out2[1] = e.im;
  return 0;
}

/* --------------------------------------------------------------- sensing */

/* sensing.cpp:27-38 */
static int validate_selection(uint64_t n, const uint64_t* rows, uint64_t m) {
  if (m == 0 || m > n) return 1;
  for (uint64_t i = 0; i < m; ++i) {
    if (rows[i] < 1 || rows[i] > n) return 1;
    if (i > 0 && rows[i] <= rows[i - 1]) return 1;
  }
  return 0;
}

int fmpo_make_row_selection(uint64_t n, uint64_t m, uint64_t seed,
                            uint64_t* omega_out) {
  /* sensing.cpp:61-70 */
  if (m == 0 || m > n) return 1;
  rng_t r;
  rng_seed(&r, seed);
  return rng_sample(&r, n, m, omega_out);
}

/* sensing.cpp:93-100: gather(U x) at Omega */
static int op_apply(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                    const cx* x, cx* y) {
  if (validate_selection(n, omega, m)) return 1;
  cx* full = (cx*)malloc(sizeof(cx) * n);
  const int st = transform(kind, n, x, full, 0);
  if (!st)
    for (uint64_t i = 0; i < m; ++i) y[i] = full[omega[i] - 1];
  free(full);
  return st;
}

/* sensing.cpp:102-109: U^H scatter(r) */
static int op_apply_adjoint(int kind, uint64_t n, const uint64_t* omega,
                            uint64_t m, const cx* r, cx* h) {
  if (validate_selection(n, omega, m)) return 1;
  cx* sc = (cx*)calloc(n, sizeof(cx));
  for (uint64_t i = 0; i < m; ++i) sc[omega[i] - 1] = r[i];
  const int st = transform(kind, n, sc, h, 1);
  free(sc);
  return st;
}

int fmpo_apply(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
               const double* x, double* y_out) {
  return op_apply(kind, n, omega, m, (const cx*)x, (cx*)y_out);
}

int fmpo_apply_adjoint(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                       const double* r, double* h_out) {
  return op_apply_adjoint(kind, n, omega, m, (const cx*)r, (cx*)h_out);
}

/* sensing.cpp:111-117 */
static void op_column(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                      uint64_t j, cx* out) {
  for (uint64_t i = 0; i < m; ++i) out[i] = entry(kind, n, omega[i], j);
}

int fmpo_column(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                uint64_t j, double* out) {
  if (validate_selection(n, omega, m) || j < 1 || j > n) return 1;
  op_column(kind, n, omega, m, j, (cx*)out);
  return 0;
}

/* sensing.cpp:119-153 */
int fmpo_make_instance(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                       uint64_t k, double noise_stddev, uint64_t seed,
                       double* x_out, double* y_out, double* noise_out) {
  if (k >= m || noise_stddev < 0.0 || validate_selection(n, omega, m)) return 1;
  rng_t r;
  rng_seed(&r, seed);
  cx* x = (cx*)x_out;
  cx* y = (cx*)y_out;
  for (uint64_t i = 0; i < n; ++i) x[i] = cx_make(0.0, 0.0);
  if (k > 0) {
    uint64_t* sup = (uint64_t*)malloc(sizeof(uint64_t) * k);
    rng_sample(&r, n, k, sup);
    for (uint64_t i = 0; i < k; ++i) x[sup[i] - 1] = rng_cgauss(&r);
    free(sup);
  }
  cx* noise = (cx*)calloc(m, sizeof(cx));
  if (noise_stddev > 0.0) {
    const double scale = noise_stddev * sqrt(2.0);
    for (uint64_t i = 0; i < m; ++i) noise[i] = cx_scale(rng_cgauss(&r), scale);
  }
  int st = op_apply(kind, n, omega, m, x, y);
  for (uint64_t i = 0; i < m; ++i) y[i] = cx_add(y[i], noise[i]);
  if (noise_out) memcpy(noise_out, noise, sizeof(cx) * m);
  free(noise);
  return st;
}

/* harness rule, SURVEY §8d (real N(0,1) nonzeros for the Hadamard configs) */
int fmpo_make_real_instance(int kind, uint64_t n, const uint64_t* omega,
                            uint64_t m, uint64_t k, uint64_t seed,
                            double* x_out, double* y_out) {
  if (k > n || validate_selection(n, omega, m)) return 1;
  rng_t r;
  rng_seed(&r, seed);
  cx* x = (cx*)x_out;
  for (uint64_t i = 0; i < n; ++i) x[i] = cx_make(0.0, 0.0);
  uint64_t* sup = (uint64_t*)malloc(sizeof(uint64_t) * (k ? k : 1));
  rng_sample(&r, n, k, sup);
  for (uint64_t i = 0; i < k; ++i)
    x[sup[i] - 1] = cx_make(sqrt(2.0) * rng_cgauss(&r).re, 0.0);
  free(sup);
  return op_apply(kind, n, omega, m, x, (cx*)y_out);
}

/* ---------------------------------------------------------------- kernel */

typedef struct {
  int kind;
  uint64_t n, m;
  cx* c;
  double* values;
  uint32_t* value_index;
  uint64_t nvalues;
} kernel_t;

static int cmp_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* kernel.cpp:24-72 */
static int compute_kernel(int kind, uint64_t n, const uint64_t* omega,
                          uint64_t m, kernel_t* k) {
  memset(k, 0, sizeof(*k));
  k->kind = kind;
  k->n = n;
  k->m = m;
  cx* e1 = (cx*)calloc(n, sizeof(cx));
  e1[0] = cx_make(1.0, 0.0);
  cx* ye = (cx*)malloc(sizeof(cx) * m);
  k->c = (cx*)malloc(sizeof(cx) * n);
  int st = op_apply(kind, n, omega, m, e1, ye);
  if (!st) st = op_apply_adjoint(kind, n, omega, m, ye, k->c);
  free(e1);
  free(ye);
  if (st) return st;
  cx* c = k->c;
  if (kind == 0) {
    /* kernel.cpp:35-45: exact conjugate symmetry */
    c[0] = cx_make(c[0].re, 0.0);
    if (n % 2 == 0 && n > 1) c[n / 2] = cx_make(c[n / 2].re, 0.0);
    for (uint64_t j = 1; 2 * j < n; ++j) {
      const cx avg = cx_scale(cx_add(c[j], cx_conj(c[n - j])), 0.5);
      c[j] = avg;
      c[n - j] = cx_conj(avg);
    }
  } else {
    /* kernel.cpp:46-70: snap onto the integer/N lattice, tabulate values */
    const double dn = (double)n;
    double* scaled = (double*)malloc(sizeof(double) * n);
    for (uint64_t j = 0; j < n; ++j) {
      scaled[j] = round(c[j].re * dn);
      c[j] = cx_make(scaled[j] / dn, 0.0);
    }
    double* distinct = (double*)malloc(sizeof(double) * n);
    memcpy(distinct, scaled, sizeof(double) * n);
    qsort(distinct, n, sizeof(double), cmp_double);
    uint64_t d = 0;
    for (uint64_t j = 0; j < n; ++j)
      if (d == 0 || distinct[j] != distinct[d - 1]) distinct[d++] = distinct[j];
    k->nvalues = d;
    k->values = (double*)malloc(sizeof(double) * d);
    for (uint64_t i = 0; i < d; ++i) k->values[i] = distinct[i] / dn;
    k->value_index = (uint32_t*)malloc(sizeof(uint32_t) * n);
    for (uint64_t j = 0; j < n; ++j) {
      uint64_t lo = 0, hi = d; /* lower_bound */
      while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (distinct[mid] < scaled[j]) lo = mid + 1; else hi = mid;
      }
      k->value_index[j] = (uint32_t)lo;
    }
    free(scaled);
    free(distinct);
  }
  return 0;
}

static void kernel_free(kernel_t* k) {
  free(k->c);
  free(k->values);
  free(k->value_index);
  memset(k, 0, sizeof(*k));
}

int fmpo_compute_kernel(int kind, uint64_t n, const uint64_t* omega,
                        uint64_t m, double* c_out, double* values_out,
                        uint32_t* value_index_out, uint64_t* nvalues) {
  kernel_t k;
  const int st = compute_kernel(kind, n, omega, m, &k);
  if (st) {
    kernel_free(&k);
    return st;
  }
  memcpy(c_out, k.c, sizeof(cx) * n);
  *nvalues = k.nvalues;
  if (values_out && k.nvalues) memcpy(values_out, k.values, sizeof(double) * k.nvalues);
  if (value_index_out && k.value_index)
    memcpy(value_index_out, k.value_index, sizeof(uint32_t) * n);
  kernel_free(&k);
  return 0;
}

/* kernel.cpp:209-303 */
static int fast_update(const kernel_t* k, const cx* h0, const uint64_t* support,
                       const cx* coeffs, uint64_t t, int symmetry, cx* h) {
  const uint64_t n = k->n;
  for (uint64_t i = 0; i < t; ++i) { /* kernel.cpp:216-222 */
    if (support[i] < 1 || support[i] > n) return 1;
    for (uint64_t j = i + 1; j < t; ++j)
      if (support[i] == support[j]) return 1;
  }
  memmove(h, h0, sizeof(cx) * n);
  if (t == 0) return 0;
  if (k->kind == 1) { /* kernel.cpp:227-244 */
    const uint64_t d = k->nvalues;
    cx* w = (cx*)malloc(sizeof(cx) * d);
    for (uint64_t tau = 0; tau < t; ++tau) {
      const uint64_t shift = support[tau] - 1;
      const cx x = coeffs[tau];
      for (uint64_t i = 0; i < d; ++i)
        w[i] = cx_make(x.re * k->values[i], x.im * k->values[i]);
      for (uint64_t a = 0; a < n; ++a)
        h[a] = cx_sub(h[a], w[k->value_index[a ^ shift]]);
    }
    free(w);
    return 0;
  }
  if (!symmetry) { /* kernel.cpp:246-261 */
    for (uint64_t tau = 0; tau < t; ++tau) {
      const uint64_t shift = support[tau] - 1;
      const cx x = coeffs[tau];
      for (uint64_t a = 0; a < n; ++a) {
        uint64_t src = a + n - shift;
        if (src >= n) src -= n;
        h[a] = cx_sub(h[a], cx_mul(x, k->c[src]));
      }
    }
    return 0;
  }
  /* kernel.cpp:263-302: paired products over conjugate entries */
  cx* p = (cx*)malloc(sizeof(cx) * n);
  for (uint64_t tau = 0; tau < t; ++tau) {
    const uint64_t shift = support[tau] - 1;
    const cx x = coeffs[tau];
    const double xr = x.re, xi = x.im;
    p[0] = cx_make(xr * k->c[0].re, xi * k->c[0].re);
    if (n % 2 == 0 && n > 1) {
      const double mid = k->c[n / 2].re;
      p[n / 2] = cx_make(xr * mid, xi * mid);
    }
    for (uint64_t j = 1; 2 * j < n; ++j) {
      const double cr = k->c[j].re, ci = k->c[j].im;
      const double rr = xr * cr, ii = xi * ci, ri = xr * ci, ir = xi * cr;
      p[j] = cx_make(rr - ii, ri + ir);
      p[n - j] = cx_make(rr + ii, ir - ri);
    }
    for (uint64_t a = 0; a < n; ++a) {
      uint64_t src = a + n - shift;
      if (src >= n) src -= n;
      h[a] = cx_sub(h[a], p[src]);
    }
  }
  free(p);
  return 0;
}

int fmpo_fast_update(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                     const double* h0, const uint64_t* support,
                     const double* coeffs, uint64_t t, int symmetry,
                     double* h_out) {
  kernel_t k;
  int st = compute_kernel(kind, n, omega, m, &k);
  if (!st)
    st = fast_update(&k, (const cx*)h0, support, (const cx*)coeffs, t, symmetry,
                     (cx*)h_out);
  kernel_free(&k);
  return st;
}

/* ------------------------------------------------------------ cost model */

/* cost_model.cpp:39-52 */
static uint64_t conventional_flops(int kind, uint64_t n) {
  if (is_pow2(n)) {
    const uint64_t logn = log2_floor(n);
    return kind == 0 ? 5 * n * logn : 2 * n * logn;
  }
  return 6 * n * n + 2 * n * (n - 1);
}

/* cost_model.cpp:54-60 */
static uint64_t fast_flops(int kind, uint64_t n, uint64_t t) {
  if (t == 1) return conventional_flops(kind, n);
  return (kind == 0 ? 6 : 2) * n * (t - 1);
}

/* cost_model.cpp:62-74 */
uint64_t fmpo_crossover_iteration(int kind, uint64_t n) {
  if (is_pow2(n)) {
    const uint64_t logn = log2_floor(n);
    return kind == 0 ? (5 * logn) / 6 + 1 : logn + 1;
  }
  const uint64_t conv = conventional_flops(kind, n);
  uint64_t t = 1;
  while (fast_flops(kind, n, t + 1) <= conv) ++t;
  return t;
}

/* --------------------------------------------------------------- solvers */

static const double kCholeskyPivotTol = 1e-12; /* solvers.cpp:32 */
static const double kTieBandRel = 1e-9;        /* solvers.cpp:40 */

/* solvers.cpp:42-46 */
static cx dot_conj(const cx* a, const cx* b, uint64_t len) {
  cx s = cx_make(0.0, 0.0);
  for (uint64_t i = 0; i < len; ++i) s = cx_add(s, cx_mul(cx_conj(a[i]), b[i]));
  return s;
}

/* types.cpp:32-36 */
static double l2_norm(const cx* v, uint64_t n) {
  double s = 0.0;
  for (uint64_t i = 0; i < n; ++i) s += v[i].re * v[i].re + v[i].im * v[i].im;
  return sqrt(s);
}

/* solvers.cpp:90-101: max magnitude, then first index within the tie band */
static uint64_t argmax_magnitude(const cx* h, uint64_t n) {
  double best = 0.0;
  for (uint64_t j = 0; j < n; ++j) {
    const double m2 = cx_mag2(h[j]);
    if (best < m2) best = m2;
  }
  const double cut = best * (1.0 - kTieBandRel);
  for (uint64_t j = 0; j < n; ++j)
    if (cx_mag2(h[j]) >= cut) return j;
  return 0;
}

uint64_t fmpo_argmax_magnitude(const double* h, uint64_t n) {
  return argmax_magnitude((const cx*)h, n);
}

/* solvers.cpp:223-274: two-pass modified Gram-Schmidt, one column at a time */
typedef struct {
  uint64_t rows, cols;
  cx* q;  /* cols x rows */
  cx* r;  /* cols x cols, r[j*cap + i] = R(i, j) */
  uint64_t cap;
} qr_t;

static void qr_init(qr_t* qr, uint64_t rows, uint64_t cap) {
  qr->rows = rows;
  qr->cols = 0;
  qr->cap = cap;
  qr->q = (cx*)malloc(sizeof(cx) * rows * cap);
  qr->r = (cx*)calloc(cap * cap, sizeof(cx));
}

static void qr_free(qr_t* qr) {
  free(qr->q);
  free(qr->r);
}

static int qr_push(qr_t* qr, const cx* col) {
  const uint64_t rows = qr->rows, c = qr->cols;
  const double orig = l2_norm(col, rows);
  cx* v = qr->q + c * rows;
  memcpy(v, col, sizeof(cx) * rows);
  cx* rcol = qr->r + c * qr->cap;
  for (uint64_t i = 0; i <= c; ++i) rcol[i] = cx_make(0.0, 0.0);
  for (int pass = 0; pass < 2; ++pass)
    for (uint64_t i = 0; i < c; ++i) {
      const cx* qi = qr->q + i * rows;
      const cx s = dot_conj(qi, v, rows);
      for (uint64_t row = 0; row < rows; ++row)
        v[row] = cx_sub(v[row], cx_mul(s, qi[row]));
      rcol[i] = cx_add(rcol[i], s);
    }
  const double rho = l2_norm(v, rows);
  if (rho <= 1e-10 * orig) return 0;
  rcol[c] = cx_make(rho, 0.0);
  for (uint64_t row = 0; row < rows; ++row) v[row] = cx_divr(v[row], rho);
  qr->cols = c + 1;
  return 1;
}

static void qr_solve(const qr_t* qr, const cx* rhs, cx* x) {
  const uint64_t t = qr->cols, rows = qr->rows;
  cx* z = (cx*)malloc(sizeof(cx) * (t ? t : 1));
  for (uint64_t i = 0; i < t; ++i) z[i] = dot_conj(qr->q + i * rows, rhs, rows);
  for (uint64_t jj = t; jj-- > 0;) {
    cx v = z[jj];
    for (uint64_t k = jj + 1; k < t; ++k)
      v = cx_sub(v, cx_mul(qr->r[k * qr->cap + jj], x[k]));
    /* complex / (rho + 0i): libgcc __divdc3 reduces to a componentwise divide */
    x[jj] = cx_divr(v, qr->r[jj * qr->cap + jj].re);
  }
  free(z);
}

/* solvers.cpp:120-177; returns 0 or (position + 1) of the dependent column */
static uint64_t normal_equations(const cx* cols, uint64_t s, uint64_t rows,
                                 const cx* y, cx* x) {
  cx* g = (cx*)malloc(sizeof(cx) * s * s);
  cx* b = (cx*)malloc(sizeof(cx) * s);
  for (uint64_t i = 0; i < s; ++i) {
    for (uint64_t j = i; j < s; ++j) {
      g[i * s + j] = dot_conj(cols + i * rows, cols + j * rows, rows);
      g[j * s + i] = cx_conj(g[i * s + j]);
    }
    b[i] = dot_conj(cols + i * rows, y, rows);
  }
  cx* l = (cx*)calloc(s * s, sizeof(cx));
  uint64_t bad = 0;
  for (uint64_t j = 0; j < s && !bad; ++j) {
    const double diag = g[j * s + j].re;
    double d = g[j * s + j].re;
    for (uint64_t k = 0; k < j; ++k) d -= cx_mag2(l[j * s + k]);
    if (!(d > kCholeskyPivotTol * diag)) {
      bad = j + 1;
      break;
    }
    const double ljj = sqrt(d);
    l[j * s + j] = cx_make(ljj, 0.0);
    for (uint64_t i = j + 1; i < s; ++i) {
      cx v = g[i * s + j];
      for (uint64_t k = 0; k < j; ++k)
        v = cx_sub(v, cx_mul(l[i * s + k], cx_conj(l[j * s + k])));
      l[i * s + j] = cx_divr(v, ljj);
    }
  }
  if (!bad) {
    cx* z = (cx*)malloc(sizeof(cx) * s);
    for (uint64_t i = 0; i < s; ++i) {
      cx v = b[i];
      for (uint64_t k = 0; k < i; ++k) v = cx_sub(v, cx_mul(l[i * s + k], z[k]));
      z[i] = cx_divr(v, l[i * s + i].re);
    }
    for (uint64_t ii = s; ii-- > 0;) {
      cx v = z[ii];
      for (uint64_t k = ii + 1; k < s; ++k)
        v = cx_sub(v, cx_mul(cx_conj(l[k * s + ii]), x[k]));
      x[ii] = cx_divr(v, l[ii * s + ii].re);
    }
    free(z);
  }
  free(g);
  free(b);
  free(l);
  return bad;
}

/* solvers.cpp:180-192 */
static void update_residual(const cx* cols, const cx* coeffs, uint64_t s,
                            uint64_t rows, const cx* y, cx* r) {
  cx* a = (cx*)calloc(rows, sizeof(cx));
  for (uint64_t j = 0; j < s; ++j)
    for (uint64_t i = 0; i < rows; ++i)
      a[i] = cx_add(a[i], cx_mul(coeffs[j], cols[j * rows + i]));
  for (uint64_t i = 0; i < rows; ++i) r[i] = cx_sub(y[i], a[i]);
  free(a);
}

/* solvers.cpp:276-294 */
int fmpo_least_squares(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                       const uint64_t* support, uint64_t s, const double* y,
                       int ls_method, double* coeffs_out, uint64_t* aux) {
  if (validate_selection(n, omega, m)) return 1;
  for (uint64_t i = 0; i < s; ++i)
    if (support[i] < 1 || support[i] > n) return 1;
  cx* cols = (cx*)malloc(sizeof(cx) * m * (s ? s : 1));
  for (uint64_t j = 0; j < s; ++j) op_column(kind, n, omega, m, support[j], cols + j * m);
  int st = 0;
  if (ls_method == 1) {
    const uint64_t bad = normal_equations(cols, s, m, (const cx*)y, (cx*)coeffs_out);
    if (bad) {
      if (aux) *aux = bad - 1;
      st = 2;
    }
  } else {
    qr_t qr;
    qr_init(&qr, m, s ? s : 1);
    for (uint64_t j = 0; j < s && !st; ++j)
      if (!qr_push(&qr, cols + j * m)) {
        if (aux) *aux = j;
        st = 2;
      }
    if (!st) qr_solve(&qr, (const cx*)y, (cx*)coeffs_out);
    qr_free(&qr);
  }
  free(cols);
  return st;
}

/* solvers.cpp:296-411 */
int fmpo_omp_solve(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                   const double* y_in, const fmpo_solve_config* cfg,
                   fmpo_solve_result* out) {
  if (validate_selection(n, omega, m)) return 1;
  if (cfg->max_iterations < 1 || !(cfg->residual_tolerance >= 0.0)) return 1;
  const cx* y = (const cx*)y_in;
  const uint64_t T = cfg->max_iterations;
  out->support_size = 0;
  out->iterations_run = 0;
  out->rank_deficient_abort = 0;
  out->history_len = 0;

  cx* r = (cx*)malloc(sizeof(cx) * m);
  memcpy(r, y, sizeof(cx) * m);
  double rn = l2_norm(r, m);
  out->residual_norm = rn;
  if (rn <= cfg->residual_tolerance) {
    free(r);
    return 0;
  }
  uint64_t fast_until = 0; /* solvers.cpp:316-323 */
  if (cfg->mode == 1) fast_until = UINT64_MAX;
  if (cfg->mode == 2) fast_until = fmpo_crossover_iteration(kind, n);

  kernel_t ker;
  int have_kernel = 0;
  qr_t qr;
  qr_init(&qr, m, T);
  cx* cols = (cx*)malloc(sizeof(cx) * m * T);
  cx* coeffs = (cx*)calloc(T, sizeof(cx));
  cx* h = (cx*)malloc(sizeof(cx) * n);
  cx* h0 = (cx*)malloc(sizeof(cx) * n);
  uint64_t* support = out->support;
  uint64_t s = 0;
  int st = 0;

  for (uint64_t t = 1; t <= T; ++t) {
    const int fast_row = t <= fast_until;
    if (out->mode_used) out->mode_used[t - 1] = fast_row;
    if (t == 1) {
      op_apply_adjoint(kind, n, omega, m, r, h);
      if (fast_until >= 2 && T >= 2) memcpy(h0, h, sizeof(cx) * n);
    } else if (fast_row) {
      if (!have_kernel) {
        st = compute_kernel(kind, n, omega, m, &ker);
        if (st) break;
        have_kernel = 1;
      }
      fast_update(&ker, h0, support, coeffs, s, cfg->fourier_symmetry, h);
    } else {
      op_apply_adjoint(kind, n, omega, m, r, h);
    }
    if (cfg->record_correlations && out->correlation_history) {
      memcpy(out->correlation_history + 2 * n * out->history_len, h, sizeof(cx) * n);
      out->history_len++;
    }
    const uint64_t pick = argmax_magnitude(h, n);
    if (cx_mag2(h[pick]) == 0.0) break;
    const uint64_t atom = pick + 1;
    int dup = 0;
    for (uint64_t i = 0; i < s; ++i) dup |= support[i] == atom;
    if (dup) break;

    support[s] = atom;
    op_column(kind, n, omega, m, atom, cols + s * m);
    ++s;
    if (cfg->ls_method == 0) {
      if (!qr_push(&qr, cols + (s - 1) * m)) {
        --s;
        out->rank_deficient_abort = 1;
        break;
      }
      qr_solve(&qr, y, coeffs);
    } else {
      if (normal_equations(cols, s, m, y, coeffs)) {
        --s;
        out->rank_deficient_abort = 1;
        break;
      }
    }
    update_residual(cols, coeffs, s, m, y, r);
    rn = l2_norm(r, m);
    out->iterations_run = t;
    out->residual_norm = rn;
    if (rn <= cfg->residual_tolerance) break;
  }
  out->support_size = s;
  memcpy(out->coeffs, coeffs, sizeof(cx) * s);
  if (have_kernel) kernel_free(&ker);
  qr_free(&qr);
  free(cols);
  free(coeffs);
  free(h);
  free(h0);
  free(r);
  return st;
}

/* solvers.cpp:62-86: the `count` largest values of m[0..n): positions above
 * the band around the rank-`count` boundary, then the smallest positions
 * inside the band; writes `count` positions (first the sure ones, then the
 * tied ones, each in index order) */
static int cmp_desc_double(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return (x < y) - (x > y);
}
static void select_largest(const double* m, uint64_t n, uint64_t count, uint64_t* out) {
  if (count >= n) {
    for (uint64_t j = 0; j < n; ++j) out[j] = j;
    return;
  }
  double* sorted = (double*)malloc(sizeof(double) * n);
  memcpy(sorted, m, sizeof(double) * n);
  qsort(sorted, n, sizeof(double), cmp_desc_double);
  const double boundary = sorted[count - 1];
  free(sorted);
  const double hi = boundary * (1.0 + kTieBandRel);
  const double lo = boundary * (1.0 - kTieBandRel);
  uint64_t o = 0;
  for (uint64_t j = 0; j < n; ++j)
    if (m[j] > hi) out[o++] = j;
  for (uint64_t j = 0; j < n && o < count; ++j)
    if (m[j] <= hi && m[j] >= lo) out[o++] = j;
}

static int cmp_u64_asc(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

/* cost_model.cpp:76-96 */
static int adaptive_cosamp_uses_fast(int kind, uint64_t n, uint64_t k) {
  if (k == 0) return 1;
  return (kind == 0 ? 6 : 2) * n * k <= conventional_flops(kind, n);
}

/* solvers.cpp:413-544.  out->support / coeffs need k entries; support_history
 * (max_iterations x k, zero padded) may be NULL. */
int fmpo_cosamp_solve(int kind, uint64_t n, const uint64_t* omega, uint64_t m,
                      const double* y_in, uint64_t k, const fmpo_solve_config* cfg,
                      fmpo_solve_result* out, uint64_t* support_history) {
  if (validate_selection(n, omega, m)) return 1;
  if (cfg->max_iterations < 1 || !(cfg->residual_tolerance >= 0.0)) return 1;
  const cx* y = (const cx*)y_in;
  const uint64_t T = cfg->max_iterations;
  out->support_size = 0;
  out->iterations_run = 0;
  out->rank_deficient_abort = 0;
  out->history_len = 0;
  cx* r = (cx*)malloc(sizeof(cx) * m);
  memcpy(r, y, sizeof(cx) * m);
  double rn = l2_norm(r, m);
  out->residual_norm = rn;
  if (k == 0 || rn <= cfg->residual_tolerance) {
    free(r);
    return 0;
  }
  const int fast = cfg->mode == 1 || (cfg->mode == 2 && adaptive_cosamp_uses_fast(kind, n, k));
  const uint64_t count = 2 * k < n ? 2 * k : n;
  kernel_t ker;
  int have_kernel = 0, st = 0;
  cx* h = (cx*)malloc(sizeof(cx) * n);
  cx* h0 = (cx*)malloc(sizeof(cx) * n);
  double* mg = (double*)malloc(sizeof(double) * (n > 3 * k ? n : 3 * k));
  uint64_t* pos = (uint64_t*)malloc(sizeof(uint64_t) * (n > 3 * k ? n : 3 * k));
  uint64_t* merged = (uint64_t*)malloc(sizeof(uint64_t) * 3 * k);
  cx* cols = (cx*)malloc(sizeof(cx) * m * 3 * k);
  cx* b = (cx*)malloc(sizeof(cx) * 3 * k);
  uint64_t* sup = out->support;
  cx* coeffs = (cx*)out->coeffs;
  uint64_t s = 0;

  for (uint64_t t = 1; t <= T; ++t) {
    if (out->mode_used) out->mode_used[t - 1] = fast;
    if (t == 1) {
      op_apply_adjoint(kind, n, omega, m, r, h);
      if (fast) memcpy(h0, h, sizeof(cx) * n);
    } else if (fast) {
      if (!have_kernel) {
        st = compute_kernel(kind, n, omega, m, &ker);
        if (st) break;
        have_kernel = 1;
      }
      fast_update(&ker, h0, sup, coeffs, s, cfg->fourier_symmetry, h);
    } else {
      op_apply_adjoint(kind, n, omega, m, r, h);
    }
    if (cfg->record_correlations && out->correlation_history) {
      memcpy(out->correlation_history + 2 * n * out->history_len, h, sizeof(cx) * n);
      out->history_len++;
    }
    /* top_atoms (solvers.cpp:105-118), then the sorted union with the support */
    for (uint64_t j = 0; j < n; ++j) mg[j] = cx_mag2(h[j]);
    select_largest(mg, n, count, pos);
    for (uint64_t j = 0; j < count; ++j) pos[j] += 1;
    qsort(pos, count, sizeof(uint64_t), cmp_u64_asc);
    uint64_t ns = 0, i = 0, j = 0;
    while (i < s || j < count) {
      if (j >= count || (i < s && sup[i] < pos[j])) merged[ns++] = sup[i++];
      else if (i >= s || pos[j] < sup[i]) merged[ns++] = pos[j++];
      else { merged[ns++] = sup[i++]; ++j; }
    }
    for (uint64_t q = 0; q < ns; ++q) op_column(kind, n, omega, m, merged[q], cols + q * m);
    if (normal_equations(cols, ns, m, y, b)) {
      out->rank_deficient_abort = 1;
      break;
    }
    /* prune to the k strongest (merged is ascending: band ties -> smallest atom) */
    for (uint64_t q = 0; q < ns; ++q) mg[q] = cx_mag2(b[q]);
    const uint64_t keep = k < ns ? k : ns;
    select_largest(mg, ns, keep, pos);
    qsort(pos, keep, sizeof(uint64_t), cmp_u64_asc); /* atom order == position order */
    s = keep;
    for (uint64_t q = 0; q < keep; ++q) {
      sup[q] = merged[pos[q]];
      coeffs[q] = b[pos[q]];
      op_column(kind, n, omega, m, sup[q], cols + q * m);
    }
    update_residual(cols, coeffs, s, m, y, r);
    rn = l2_norm(r, m);
    if (support_history)
      for (uint64_t q = 0; q < k; ++q) support_history[(t - 1) * k + q] = q < s ? sup[q] : 0;
    out->iterations_run = t;
    out->residual_norm = rn;
    if (rn <= cfg->residual_tolerance) break;
  }
  out->support_size = s;
  if (have_kernel) kernel_free(&ker);
  free(r);
  free(h);
  free(h0);
  free(mg);
  free(pos);
  free(merged);
  free(cols);
  free(b);
  return st;
}

/* batched driver: one solve per host thread, like fastmp_cli.cpp:273-303 */
typedef struct {
  int kind;
  uint64_t n, m, batch;
  const uint64_t* omega;
  const double* y;
  const fmpo_solve_config* cfg;
  uint64_t* support;
  double* coeffs;
  uint64_t* iterations;
  double* residual;
  int* aborted;
  uint64_t next;
  pthread_mutex_t lock;
  int failed;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* job = (batch_job*)arg;
  const uint64_t T = job->cfg->max_iterations;
  fmpo_solve_config cfg = *job->cfg;
  cfg.record_correlations = 0;
  for (;;) {
    pthread_mutex_lock(&job->lock);
    const uint64_t b = job->next++;
    pthread_mutex_unlock(&job->lock);
    if (b >= job->batch) return NULL;
    fmpo_solve_result res;
    memset(&res, 0, sizeof(res));
    res.support = job->support + T * b;
    res.coeffs = job->coeffs + 2 * T * b;
    memset(res.support, 0, sizeof(uint64_t) * T);
    memset(res.coeffs, 0, sizeof(double) * 2 * T);
    if (fmpo_omp_solve(job->kind, job->n, job->omega, job->m,
                       job->y + 2 * job->m * b, &cfg, &res))
      job->failed = 1;
    job->iterations[b] = res.iterations_run;
    job->residual[b] = res.residual_norm;
    job->aborted[b] = res.rank_deficient_abort;
  }
}

int fmpo_omp_solve_batch(int kind, uint64_t n, const uint64_t* omega,
                         uint64_t m, const double* y, uint64_t batch,
                         const fmpo_solve_config* cfg, int threads,
                         uint64_t* support, double* coeffs,
                         uint64_t* iterations, double* residual,
                         int* aborted) {
  batch_job job = {kind, n, m, batch, omega, y, cfg, support, coeffs,
                   iterations, residual, aborted, 0,
                   PTHREAD_MUTEX_INITIALIZER, 0};
  long w = threads > 0 ? threads : sysconf(_SC_NPROCESSORS_ONLN);
  if (w < 1) w = 1;
  if ((uint64_t)w > batch) w = (long)(batch ? batch : 1);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)w);
  for (long i = 1; i < w; ++i) pthread_create(&th[i], NULL, batch_worker, &job);
  batch_worker(&job);
  for (long i = 1; i < w; ++i) pthread_join(th[i], NULL);
  free(th);
  return job.failed ? 9 : 0;
}

const char* fmpo_impl(void) { return "restatement"; }
