// fmp_driver: the seeded multi-GPU driver of the batched OMP path (north
// star: "a seeded C++ driver that shards independent recovery problems
// across the GPUs of one box").  It replaces the reference's solve-per-worker
// pool (`fastmp equiv`, fastmp_cli.cpp:276-303) with one operator per GPU and
// fmp_omp_solve_multi, which splits the batch into contiguous blocks, one
// host thread per device, no collective.  Inputs follow SURVEY §8d's seed
// rule (the bench's): Omega = make_row_selection(N, M, derive_seed(S, 2^40)),
// signal b from derive_seed(S, b) through make_instance's draws.
//
//   fmp_driver [--config 1|2|4] [--gpus N] [--steps K] [--warmup W]
//              [--seed S] [--batch B] [--mode gpu|fast|adaptive|conventional]
//              [--dtype c128|c64|f64]
//
// Prints one JSON line: host-buffer (end-to-end) recoveries/s over all GPUs,
// the wall-clock time per batched call, and the fraction of true supports
// recovered.  Only the C ABI (include/fmp.h) is used.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "fmp.h"

namespace {

struct Config {
  int kind;
  uint64_t n, m, k, batch, iters, seed;
  double noise;
  std::string dtype;
  const char* name;
};

Config config_of(int c) {
  switch (c) {
    case 1:
      return {FMP_HADAMARD, 1024, 256, 16, 1, 16, 1, 0.0, "f64",
              "config1: partial Hadamard N=1024 M=256 K=16 f64 real, batch 1"};
    case 4:
      return {FMP_FOURIER, 16384, 4096, 128, 2048, 256, 4, std::sqrt(128.0 / (2.0 * 16384 * 1e3)), "c128",
              "config4: partial DFT N=16384 M=4096 K=128, 30 dB noise, halt at ||r|| <= ||noise|| or 2K"};
    default:
      return {FMP_FOURIER, 4096, 1024, 64, 4096, 64, 2, 0.0, "c128",
              "config2: partial DFT N=4096 M=1024 K=64 c128, noiseless, K iterations"};
  }
}

[[noreturn]] void die(const char* what, int st) {
  std::fprintf(stderr, "fmp_driver: %s failed (%d): %s\n", what, st, fmp_last_error());
  std::exit(1);
}
void ok(const char* what, int st) {
  if (st != FMP_OK) die(what, st);
}

}  // namespace

int main(int argc, char** argv) {
  int cfg_id = 2, gpus = 0, steps = 5, warmup = 2;
  uint64_t seed = 0, batch = 0;
  std::string mode = "gpu", dtype;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto next = [&]() -> const char* {
      if (i + 1 >= argc) { std::fprintf(stderr, "missing value for %s\n", a.c_str()); std::exit(2); }
      return argv[++i];
    };
    if (a == "--config") cfg_id = std::atoi(next());
    else if (a == "--gpus") gpus = std::atoi(next());
    else if (a == "--steps") steps = std::atoi(next());
    else if (a == "--warmup") warmup = std::atoi(next());
    else if (a == "--seed") seed = std::strtoull(next(), nullptr, 10);
    else if (a == "--batch") batch = std::strtoull(next(), nullptr, 10);
    else if (a == "--mode") mode = next();
    else if (a == "--dtype") dtype = next();
    else { std::fprintf(stderr, "unknown argument %s\n", a.c_str()); return 2; }
  }
  Config C = config_of(cfg_id);
  if (seed) C.seed = seed;
  if (batch) C.batch = batch;
  if (!dtype.empty()) C.dtype = dtype;
  int ndev = 0;
  ok("fmp_device_count", fmp_device_count(&ndev));
  if (ndev < 1) { std::fprintf(stderr, "fmp_driver: no CUDA device\n"); return 1; }
  if (gpus <= 0) gpus = ndev;
  if (gpus > ndev) { std::fprintf(stderr, "fmp_driver: %d GPUs asked, %d visible\n", gpus, ndev); return 1; }
  const int fmode = mode == "fast" ? FMP_MODE_FAST : mode == "adaptive" ? FMP_MODE_ADAPTIVE
                    : mode == "conventional" ? FMP_MODE_CONVENTIONAL : FMP_MODE_GPU;
  const int dt = C.dtype == "c64" ? FMP_C64 : C.dtype == "f64" ? FMP_F64 : FMP_C128;
  const bool real = dt == FMP_F64;

  // seeded inputs: rows, measurements, true supports, noise norms
  std::vector<uint64_t> rows(C.m);
  ok("fmp_make_row_selection", fmp_make_row_selection(C.n, C.m, fmp_derive_seed(C.seed, 1ull << 40), rows.data()));
  std::vector<double> y(2 * C.batch * C.m), x(2 * C.batch * C.n), nn(C.batch);
  ok("fmp_make_batch", fmp_make_batch(C.kind, C.n, rows.data(), C.m, C.k, C.noise, real ? 1 : 0, C.seed, 0,
                                      C.batch, 0, y.data(), x.data(), nn.data()));
  // the solve's element type
  std::vector<unsigned char> ybuf;
  if (dt == FMP_C128) {
    ybuf.resize(y.size() * 8);
    std::memcpy(ybuf.data(), y.data(), ybuf.size());
  } else if (dt == FMP_C64) {
    ybuf.resize(y.size() * 4);
    float* f = reinterpret_cast<float*>(ybuf.data());
    for (size_t i = 0; i < y.size(); ++i) f[i] = (float)y[i];
  } else {
    ybuf.resize(C.batch * C.m * 8);
    double* d = reinterpret_cast<double*>(ybuf.data());
    for (size_t i = 0; i < C.batch * C.m; ++i) d[i] = y[2 * i];
  }
  // tolerances: 1e-9 ||y|| (default_config, solvers.cpp:216-221), or the
  // noise norm for the noisy config 4
  std::vector<double> tol(C.batch);
  for (uint64_t b = 0; b < C.batch; ++b) {
    double s = 0.0;
    for (uint64_t i = 0; i < C.m; ++i) s += y[2 * (b * C.m + i)] * y[2 * (b * C.m + i)] + y[2 * (b * C.m + i) + 1] * y[2 * (b * C.m + i) + 1];
    tol[b] = C.noise > 0.0 ? nn[b] : 1e-9 * std::sqrt(s);
  }

  // one context and operator per GPU
  std::vector<fmp_ctx> ctx(gpus);
  std::vector<fmp_op> ops(gpus);
  for (int g = 0; g < gpus; ++g) {
    ok("fmp_ctx_create", fmp_ctx_create(g, &ctx[g]));
    ok("fmp_operator_create", fmp_operator_create(ctx[g], C.kind, C.n, rows.data(), C.m, &ops[g]));
  }
  fmp_omp_config cfg{};
  cfg.max_iterations = C.iters;
  cfg.tolerances = tol.data();
  cfg.mode = fmode;
  // page-locked measurement and result buffers: the solve streams its inputs
  // in and its results out while it runs
  auto pinned = [](size_t bytes) {
    void* p = nullptr;
    ok("fmp_host_alloc", fmp_host_alloc(bytes, &p));
    return p;
  };
  void* yp = pinned(ybuf.size());
  std::memcpy(yp, ybuf.data(), ybuf.size());
  auto* sup = static_cast<uint64_t*>(pinned(C.batch * C.iters * 8));
  auto* co = static_cast<double*>(pinned(C.batch * C.iters * 16));
  auto* size = static_cast<uint64_t*>(pinned(C.batch * 8));
  auto* iters = static_cast<uint64_t*>(pinned(C.batch * 8));
  auto* resid = static_cast<double*>(pinned(C.batch * 8));
  auto* ab = static_cast<int32_t*>(pinned(C.batch * 4));
  fmp_omp_result out{sup, co, size, iters, resid, ab, nullptr, nullptr, nullptr};
  for (int w = 0; w < warmup; ++w)
    ok("fmp_omp_solve_multi", fmp_omp_solve_multi(ops.data(), gpus, dt, yp, C.batch, &cfg, &out));
  std::vector<double> times;
  for (int s = 0; s < steps; ++s) {
    const auto t0 = std::chrono::steady_clock::now();
    ok("fmp_omp_solve_multi", fmp_omp_solve_multi(ops.data(), gpus, dt, yp, C.batch, &cfg, &out));
    times.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  std::sort(times.begin(), times.end());
  const double med = times[times.size() / 2];
  // true supports recovered (the K nonzeros of x among the selected atoms)
  uint64_t hit = 0;
  for (uint64_t b = 0; b < C.batch; ++b) {
    std::set<uint64_t> got(sup + b * C.iters, sup + b * C.iters + size[b]);
    bool all = true;
    for (uint64_t j = 0; j < C.n && all; ++j)
      if (x[2 * (b * C.n + j)] != 0.0 || x[2 * (b * C.n + j) + 1] != 0.0) all = got.count(j + 1) > 0;
    hit += all;
  }
  std::printf("{\"driver\": \"fmp_driver\", \"metric\": \"omp_recoveries_per_sec\", \"value\": %.6g, "
              "\"unit\": \"recoveries/s\", \"n_gpus\": %d, \"steps\": %d, \"warmup\": %d, "
              "\"ms_per_step\": %.6g, \"timing\": \"median wall clock of fmp_omp_solve_multi with host buffers\", "
              "\"dtype\": \"%s\", \"mode\": \"%s\", \"config\": {\"workload\": \"%s\", \"batch\": %llu, "
              "\"seed\": %llu, \"parallelism\": \"batch-sharded x%d (contiguous blocks, no collective)\"}, "
              "\"true_support_recovered\": %.6g}\n",
              C.batch / med, gpus, steps, warmup, med * 1e3, C.dtype.c_str(), mode.c_str(), C.name,
              (unsigned long long)C.batch, (unsigned long long)C.seed, gpus, (double)hit / (double)C.batch);
  for (void* p : {yp, (void*)sup, (void*)co, (void*)size, (void*)iters, (void*)resid, (void*)ab})
    fmp_host_free(p);
  for (int g = 0; g < gpus; ++g) {
    fmp_operator_destroy(ops[g]);
    fmp_ctx_destroy(ctx[g]);
  }
  return 0;
}
