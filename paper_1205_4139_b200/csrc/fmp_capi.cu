// C ABI (include/fmp.h) over the sm_100a kernels.  Validation mirrors the
// reference's std::invalid_argument checks so callers see the same error
// behaviour (kernel.cpp:212-222, sensing.cpp:27-38/94/104, solvers.cpp:299-304).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <limits>
#include <complex>
#include <cstring>
#include <mutex>
#include <thread>
#include <type_traits>
#include <string>
#include <vector>

#include "fmp.h"
#include "fmp_capi_internal.cuh"
#include "fmp_kernels.cuh"

using fmp::DevOp;
using namespace fmpi;

namespace fmpi {
thread_local std::string g_err;
int g_phase_prof = 0;
thread_local int g_launch_count = 0;
}  // namespace fmpi


extern "C" {

int fmp_version(void) { return 1; }

int fmp_host_alloc(size_t bytes, void** out) {
  if (!out) return fail(FMP_EINVAL, "null argument");
  *out = nullptr;
  cudaError_t e = cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(FMP_ENOMEM, "page-locked host allocation (%zu bytes): %s", bytes, cudaGetErrorString(e));
  }
  return FMP_OK;
}

int fmp_host_free(void* p) {
  if (p) CU(cudaFreeHost(p));
  return FMP_OK;
}

int fmp_device_count(int* out) {
  if (!out) return fail(FMP_EINVAL, "null argument");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *out = n;
  return FMP_OK;
}

int fmp_set_phase_profiling(int enabled) {
  g_phase_prof = enabled;
  return FMP_OK;
}

int fmp_phase_cycles(fmp_ctx ctx, double* out6) {
  if (!ctx || !out6) return fail(FMP_EINVAL, "null argument");
  CU(cudaSetDevice(ctx->device));
  cudaError_t e = cudaSuccess;
  void* ph = ctx->ws.get(S_PH, 64, &e);
  if (!ph) return fail(FMP_ENOMEM, "phase buffer");
  unsigned long long v[6];
  CU(cudaStreamSynchronize(ctx->cur));
  CU(cudaMemcpy(v, ph, sizeof(v), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 6; ++i) out6[i] = (double)v[i];
  return FMP_OK;
}

int fmp_refine_stats(fmp_ctx ctx, double* out3) {
  if (!ctx || !out3) return fail(FMP_EINVAL, "null argument");
  CU(cudaSetDevice(ctx->device));
  cudaError_t e = cudaSuccess;
  void* rs = ctx->ws.get(S_RST, 64, &e);
  if (!rs) return fail(FMP_ENOMEM, "refine statistics buffer");
  unsigned long long v[3];
  CU(cudaStreamSynchronize(ctx->cur));
  CU(cudaMemcpy(v, rs, sizeof(v), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 3; ++i) out3[i] = (double)v[i];
  return FMP_OK;
}

int fmp_fma_peak(fmp_ctx ctx, int is_double, double* out) {
  if (!ctx || !out) return fail(FMP_EINVAL, "null argument");
  CU(cudaSetDevice(ctx->device));
  std::lock_guard<std::mutex> lk(ctx->mu);
  CU(fmp::fma_peak(is_double, out));
  return FMP_OK;
}
const char* fmp_last_error(void) { return g_err.c_str(); }
int fmp_last_launch_count(void) { return g_launch_count; }

uint64_t fmp_crossover_iteration(int kind, uint64_t n) {
  // cost_model.cpp:62-74 (power-of-two sizes)
  if (!pow2(n)) return 0;
  const uint64_t logn = (uint64_t)ilog2(n);
  return kind == FMP_FOURIER ? (5 * logn) / 6 + 1 : logn + 1;
}

uint64_t fmp_gpu_crossover(int kind, uint64_t n) {
  // measured on B200 (bench.py --mode custom:T sweeps): the
  // fused kernel's transform iteration costs about as much as 8 log2(N) / 3
  // fast-update atoms for Fourier; the Hadamard FWHT needs no twiddles
  if (!pow2(n)) return 0;
  const uint64_t logn = (uint64_t)ilog2(n);
  return kind == FMP_FOURIER ? (8 * logn) / 3 : 2 * logn;
}

uint64_t fmp_gpu_crossover_for(fmp_op op, int dtype, uint64_t batch, uint64_t max_iterations) {
  if (!op || dtype < 0 || dtype > 3) return 0;
  cudaSetDevice(op->ctx->device);
  return (uint64_t)fmp::omp_gpu_fast_until(op->d, dtype, (int64_t)batch, (int64_t)max_iterations);
}

int fmp_omp_plan_info(fmp_op op, int dtype, uint64_t batch, uint64_t max_iterations, int* out4) {
  if (!op || !out4) return fail(FMP_EINVAL, "null argument");
  if (int s = check_dtype(op->d, dtype)) return s;
  CU(cudaSetDevice(op->ctx->device));
  fmp::omp_info(op->d, dtype, (int64_t)batch, (int64_t)max_iterations, out4);
  return FMP_OK;
}

int fmp_ctx_create(int device, fmp_ctx* out) {
  if (!out) return fail(FMP_EINVAL, "null output handle");
  int count = 0;
  CU(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) return fail(FMP_EINVAL, "device %d of %d", device, count);
  CU(cudaSetDevice(device));
  fmp_ctx_s* c = new fmp_ctx_s;
  c->device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return fail(FMP_ECUDA, "stream: %s", cudaGetErrorString(e));
  }
  c->cur = c->own;
  *out = c;
  return FMP_OK;
}

int fmp_ctx_destroy(fmp_ctx ctx) {
  if (!ctx) return FMP_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->cur);
  for (cudaStream_t x : {ctx->copy, ctx->alt})
    if (x) {
      cudaStreamSynchronize(x);
      cudaStreamDestroy(x);
    }
  for (cudaEvent_t e : ctx->events) cudaEventDestroy(e);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->own) cudaStreamDestroy(ctx->own);
  delete ctx;
  return FMP_OK;
}

int fmp_ctx_set_stream(fmp_ctx ctx, void* stream) {
  if (!ctx) return fail(FMP_EINVAL, "null context");
  ctx->cur = stream ? (cudaStream_t)stream : ctx->own;
  return FMP_OK;
}

void* fmp_ctx_stream(fmp_ctx ctx) { return ctx ? (void*)ctx->cur : nullptr; }

int fmp_ctx_synchronize(fmp_ctx ctx) {
  if (!ctx) return fail(FMP_EINVAL, "null context");
  CU(cudaSetDevice(ctx->device));
  CU(cudaStreamSynchronize(ctx->cur));
  return FMP_OK;
}

int fmp_operator_create(fmp_ctx ctx, int kind, uint64_t n, const uint64_t* rows, uint64_t m,
                        fmp_op* out) {
  if (!ctx || !out) return fail(FMP_EINVAL, "null handle");
  if (kind != FMP_FOURIER && kind != FMP_HADAMARD) return fail(FMP_EINVAL, "unknown kind %d", kind);
  if (n == 0) return fail(FMP_EINVAL, "transform size must be positive");
  if (!pow2(n)) {
    if (kind == FMP_HADAMARD) return fail(FMP_EINVAL, "hadamard size must be a power of two");
    return fail(FMP_EUNSUPPORTED, "non power-of-two Fourier sizes (the reference's dense "
                                  "fallback) are not implemented on the GPU path");
  }
  if (n > (1ull << 28)) return fail(FMP_EUNSUPPORTED, "n = %llu exceeds 2^28", (unsigned long long)n);
  if (!rows || m == 0) return fail(FMP_EINVAL, "row selection must be non-empty");
  if (m > n) return fail(FMP_EINVAL, "row selection larger than the transform size");
  std::vector<uint64_t> r(rows, rows + m);
  std::sort(r.begin(), r.end());
  for (uint64_t i = 0; i < m; ++i) {
    if (r[i] < 1 || r[i] > n) return fail(FMP_EINVAL, "row index out of range");
    if (i && r[i] == r[i - 1]) return fail(FMP_EINVAL, "row indices must be distinct");
  }
  CU(cudaSetDevice(ctx->device));
  CtxLock lk(ctx);
  lk.use(ctx->cur);
  fmp_op_s* op = new fmp_op_s;
  op->ctx = ctx;
  op->rows = r;
  DevOp& d = op->d;
  d.kind = kind;
  d.n = (int64_t)n;
  d.m = (int64_t)m;
  d.log2n = ilog2(n);
  auto cleanup = [&](int code) {
    fmp_operator_destroy(op);
    return code;
  };
  std::vector<uint32_t> om(m);
  for (uint64_t i = 0; i < m; ++i) om[i] = (uint32_t)(r[i] - 1);
  // transform slot of each row (bit-reversed for the Fourier DIT), sorted
  std::vector<std::pair<uint32_t, uint32_t>> slots(m);
  for (uint64_t i = 0; i < m; ++i) {
    uint32_t p = om[i];
    if (kind == FMP_FOURIER) {
      uint32_t q = 0;
      for (int b = 0; b < d.log2n; ++b) q |= ((p >> b) & 1u) << (d.log2n - 1 - b);
      p = q;
    }
    slots[i] = {p, (uint32_t)i};
  }
  std::sort(slots.begin(), slots.end());
  std::vector<uint32_t> spos(m), srow(m);
  for (uint64_t i = 0; i < m; ++i) {
    spos[i] = slots[i].first;
    srow[i] = slots[i].second;
  }
  // scatter offsets per 256 slots (large-n transform blocks start on them)
  const uint64_t noff = n / 256 + 1;
  std::vector<uint32_t> soff(noff, 0);
  for (uint64_t i = 0, k = 0; i < noff; ++i) {
    while (k < m && spos[k] < i * 256) ++k;
    soff[i] = (uint32_t)k;
  }
  // two-pass transform lists (n = N1 N2): Omega by column for the scatter,
  // by output row for the gather (fmp_transform_4s.cu)
  d.fs_l1 = fmp::fs_split(d.log2n);
  std::vector<uint32_t> fa_off, fa_pos, fa_row, fb_off, fb_pos, fb_row;
  if (d.fs_l1) {
    const int L1 = d.fs_l1, L2 = d.log2n - L1;
    const uint32_t N1 = 1u << L1, N2 = 1u << L2;
    auto build = [&](auto key, uint32_t groups, std::vector<uint32_t>& off,
                     std::vector<uint32_t>& pos, std::vector<uint32_t>& row) {
      off.assign(groups + 1, 0);
      for (uint64_t i = 0; i < m; ++i) off[key(om[i]) + 1]++;
      for (uint32_t g = 0; g < groups; ++g) off[g + 1] += off[g];
      std::vector<uint32_t> fill(off.begin(), off.end() - 1);
      pos.resize(m);
      row.resize(m);
      for (uint64_t i = 0; i < m; ++i) {
        const uint32_t q = fill[key(om[i])]++;
        pos[q] = om[i];
        row[q] = (uint32_t)i;
      }
    };
    build([&](uint32_t p) { return p & (N2 - 1); }, N2, fa_off, fa_pos, fa_row);
    if (kind == FMP_FOURIER) build([&](uint32_t p) { return p & (N1 - 1); }, N1, fb_off, fb_pos, fb_row);
    else build([&](uint32_t p) { return p >> L2; }, N1, fb_off, fb_pos, fb_row);
  }
  cudaError_t e = cudaSuccess;
#define OPALLOC(p, bytes) \
  if ((e = cudaMalloc(&p, (bytes))) != cudaSuccess) return cleanup(fail(FMP_ENOMEM, "operator alloc: %s", cudaGetErrorString(e)))
  OPALLOC(d.omega, m * 4);
  OPALLOC(d.scat_pos, m * 4);
  OPALLOC(d.scat_row, m * 4);
  OPALLOC(d.scat_off, noff * 4);
  std::vector<uint32_t> f16_omt;
  std::vector<uint16_t> f16_yidx;
  if (kind == FMP_FOURIER && n == 4096) {
    std::vector<uint32_t> mask(256, 0), off(257, 0);
    for (uint64_t i = 0; i < m; ++i) mask[om[i] & 255] |= 1u << (om[i] >> 8);
    for (int u = 0; u < 256; ++u) off[u + 1] = off[u] + (uint32_t)__builtin_popcount(mask[u]);
    f16_omt.resize(256);
    for (int u = 0; u < 256; ++u) f16_omt[u] = (off[u] << 16) | mask[u];
    f16_yidx.resize(m);
    for (uint64_t i = 0; i < m; ++i) {
      const uint32_t u = om[i] & 255, j = om[i] >> 8;
      f16_yidx[i] = (uint16_t)(off[u] + (uint32_t)__builtin_popcount(mask[u] & ((1u << j) - 1)));
    }
    OPALLOC(d.f16_omt, 256 * 4);
    OPALLOC(d.f16_yidx, m * 2);
  }
  OPALLOC(d.g64, n * 16);
  if (kind == FMP_FOURIER) {
    OPALLOC(d.tw64, n * 16);
    OPALLOC(d.tw32, n * 8);
    OPALLOC(d.g32, n * 8);
  } else {
    OPALLOC(d.gr64, n * 8);
    if (m <= 32767) OPALLOC(d.glat, n * 2);
  }
  if (d.fs_l1) {
    OPALLOC(d.fs_aoff, fa_off.size() * 4);
    OPALLOC(d.fs_apos, m * 4);
    OPALLOC(d.fs_arow, m * 4);
    OPALLOC(d.fs_boff, fb_off.size() * 4);
    OPALLOC(d.fs_bpos, m * 4);
    OPALLOC(d.fs_brow, m * 4);
  }
  // one-pass large Hadamard adjoint: per block size, rows ordered by (row of
  // 32, position, input block) (fmp_transform_fold.cu)
  std::vector<uint32_t> fold_tab[4], fold_off[4];
  if (kind == FMP_HADAMARD && m < (1u << 20)) {
    for (int q = 2; q < 4; ++q) {  // block sizes in use: 2^14 (f32, f64, c64), 2^13 (c128)
      const int lb = 11 + q, s = d.log2n - lb;
      if (s < 1 || s > 6) continue;
      const uint32_t rows_per_block = 1u << (lb - 5);
      std::vector<std::pair<uint64_t, uint32_t>> key(m);
      for (uint64_t i = 0; i < m; ++i) {
        const uint32_t p = om[i], ih = p >> lb, lo = p & ((1u << lb) - 1);
        key[i] = {((uint64_t)(lo >> 5) << 16) | ((lo & 31u) << 8) | ih, (uint32_t)i};
      }
      std::sort(key.begin(), key.end());
      fold_tab[q].resize(m);
      fold_off[q].assign(rows_per_block + 1, 0);
      for (uint64_t i = 0; i < m; ++i) {
        const uint32_t mi = key[i].second, p = om[mi], lo = p & ((1u << lb) - 1);
        fold_tab[q][i] = mi | ((p >> lb) << 20) | ((lo & 31u) << 26);
        fold_off[q][(lo >> 5) + 1]++;
      }
      for (uint32_t g = 0; g < rows_per_block; ++g) fold_off[q][g + 1] += fold_off[q][g];
      OPALLOC(d.fold_tab[q], m * 4);
      OPALLOC(d.fold_off[q], (rows_per_block + 1) * 4);
    }
  }
  std::vector<uint2> om_wr;
  if (kind == FMP_HADAMARD && n >= 4096) {
    om_wr.assign(n / 32, make_uint2(0u, 0u));
    for (uint64_t i = 0; i < m; ++i) om_wr[om[i] >> 5].x |= 1u << (om[i] & 31u);
    uint32_t run = 0;
    for (uint64_t w = 0; w < n / 32; ++w) {
      om_wr[w].y = run;
      run += (uint32_t)__builtin_popcount(om_wr[w].x);
    }
    OPALLOC(d.om_wr, (n / 32) * 8);
  }
#undef OPALLOC
  cudaStream_t st = ctx->cur;
  if (d.om_wr && (e = cudaMemcpyAsync(d.om_wr, om_wr.data(), om_wr.size() * 8, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return cleanup(fail(FMP_ECUDA, "Omega bitmap: %s", cudaGetErrorString(e)));
  for (int q = 0; q < 4; ++q)
    if (d.fold_tab[q] &&
        ((e = cudaMemcpyAsync(d.fold_tab[q], fold_tab[q].data(), m * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
         (e = cudaMemcpyAsync(d.fold_off[q], fold_off[q].data(), fold_off[q].size() * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess))
      return cleanup(fail(FMP_ECUDA, "fold tables: %s", cudaGetErrorString(e)));
  if (d.fs_l1 &&
      ((e = cudaMemcpyAsync(d.fs_aoff, fa_off.data(), fa_off.size() * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
       (e = cudaMemcpyAsync(d.fs_apos, fa_pos.data(), m * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
       (e = cudaMemcpyAsync(d.fs_arow, fa_row.data(), m * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
       (e = cudaMemcpyAsync(d.fs_boff, fb_off.data(), fb_off.size() * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
       (e = cudaMemcpyAsync(d.fs_bpos, fb_pos.data(), m * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
       (e = cudaMemcpyAsync(d.fs_brow, fb_row.data(), m * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess))
    return cleanup(fail(FMP_ECUDA, "two-pass lists: %s", cudaGetErrorString(e)));
  int launches = 0;
  if ((e = cudaMemcpyAsync(d.omega, om.data(), m * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(d.scat_pos, spos.data(), m * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(d.scat_row, srow.data(), m * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(d.scat_off, soff.data(), noff * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
      (d.f16_omt && (e = cudaMemcpyAsync(d.f16_omt, f16_omt.data(), 256 * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess) ||
      (d.f16_yidx && (e = cudaMemcpyAsync(d.f16_yidx, f16_yidx.data(), m * 2, cudaMemcpyHostToDevice, st)) != cudaSuccess))
    return cleanup(fail(FMP_ECUDA, "omega copy: %s", cudaGetErrorString(e)));
  if (kind == FMP_FOURIER) {
    if ((e = fmp::launch_twiddles(d, st)) != cudaSuccess)
      return cleanup(fail(FMP_ECUDA, "twiddles: %s", cudaGetErrorString(e)));
    ++launches;
  }
  // c = apply_adjoint(apply(e1)) with apply(e1) = 1/sqrt(N) on every row
  // (kernel.cpp:33); the transform runs in fp64
  std::vector<double> ones(2 * m, 0.0);
  const double isn = 1.0 / std::sqrt((double)n);
  for (uint64_t i = 0; i < m; ++i) ones[2 * i] = isn;
  void* din = nullptr;
  int st2 = copy_in(ctx, S_AUX, ones.data(), ones.size() * 8, &din, st);
  if (st2) return cleanup(st2);
  st2 = run_transform(op, FMP_C128, 1, 1, 0, din, d.g64, 1, nullptr, st);
  if (st2) return cleanup(st2);
  launches += g_launch_count;
  if ((e = fmp::launch_kernel_finish(d, st)) != cudaSuccess)
    return cleanup(fail(FMP_ECUDA, "kernel finish: %s", cudaGetErrorString(e)));
  launches += 2;
  // max_{k != 0} |c_k| for the fp32 paths' rounding bounds
  unsigned long long* goff = nullptr;
  {
    cudaError_t ea = cudaSuccess;
    goff = (unsigned long long*)ctx->ws.get(S_GOFF, 8, &ea);
    if (!goff) return cleanup(fail(FMP_ENOMEM, "operator build scratch: %s", cudaGetErrorString(ea)));
  }
  if ((e = fmp::launch_gmax_off(d, goff, st)) != cudaSuccess)
    return cleanup(fail(FMP_ECUDA, "kernel bound: %s", cudaGetErrorString(e)));
  ++launches;
  unsigned long long gbits = 0;
  if ((e = cudaMemcpyAsync(&gbits, goff, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess ||
      (e = cudaStreamSynchronize(st)) != cudaSuccess)
    return cleanup(fail(FMP_ECUDA, "operator build: %s", cudaGetErrorString(e)));
  std::memcpy(&d.goff, &gbits, 8);
  g_launch_count = launches;
  *out = op;
  return FMP_OK;
}

int fmp_operator_destroy(fmp_op op) {
  if (!op) return FMP_OK;
  cudaSetDevice(op->ctx->device);
  cudaStreamSynchronize(op->ctx->cur);
  DevOp& d = op->d;
  for (void* p : {(void*)d.omega, (void*)d.scat_pos, (void*)d.scat_row, (void*)d.scat_off, (void*)d.f16_omt, (void*)d.f16_yidx, (void*)d.tw64, (void*)d.tw32, (void*)d.g64, (void*)d.g32,
                  (void*)d.gr64, (void*)d.glat, (void*)d.fs_aoff, (void*)d.fs_apos, (void*)d.fs_arow,
                  (void*)d.fs_boff, (void*)d.fs_bpos, (void*)d.fs_brow, (void*)d.om_wr})
    if (p) cudaFree(p);
  for (int q = 0; q < 4; ++q) {
    if (d.fold_tab[q]) cudaFree(d.fold_tab[q]);
    if (d.fold_off[q]) cudaFree(d.fold_off[q]);
  }
  delete op;
  return FMP_OK;
}

int fmp_operator_info(fmp_op op, int* kind, uint64_t* n, uint64_t* m) {
  if (!op) return fail(FMP_EINVAL, "null operator");
  if (kind) *kind = op->d.kind;
  if (n) *n = (uint64_t)op->d.n;
  if (m) *m = (uint64_t)op->d.m;
  return FMP_OK;
}

int fmp_operator_kernel(fmp_op op, double* c_out, double* values_out, uint32_t* value_index_out,
                        uint64_t* nvalues) {
  if (!op || !c_out) return fail(FMP_EINVAL, "null argument");
  CU(cudaSetDevice(op->ctx->device));
  const uint64_t n = (uint64_t)op->d.n;
  CU(cudaMemcpyAsync(c_out, op->d.g64, n * 16, cudaMemcpyDeviceToHost, op->ctx->cur));
  CU(cudaStreamSynchronize(op->ctx->cur));
  if (op->d.kind == fmp::FOURIER) {
    if (nvalues) *nvalues = 0;
    return FMP_OK;
  }
  // value table of the snapped lattice (kernel.cpp:56-69), from the exact c
  std::vector<double> scaled(n);
  for (uint64_t j = 0; j < n; ++j) scaled[j] = std::round(c_out[2 * j] * (double)n);
  std::vector<double> distinct = scaled;
  std::sort(distinct.begin(), distinct.end());
  distinct.erase(std::unique(distinct.begin(), distinct.end()), distinct.end());
  if (nvalues) *nvalues = distinct.size();
  if (values_out)
    for (size_t i = 0; i < distinct.size(); ++i) values_out[i] = distinct[i] / (double)n;
  if (value_index_out)
    for (uint64_t j = 0; j < n; ++j)
      value_index_out[j] = (uint32_t)(std::lower_bound(distinct.begin(), distinct.end(), scaled[j]) -
                                      distinct.begin());
  return FMP_OK;
}

// ------------------------------------------------------------- transforms
static int transform_host(fmp_op op, int dtype, int inverse, int in_omega, int out_omega,
                          const void* in, uint64_t batch, void* out, uint64_t* amax) {
  if (!op) return fail(FMP_EINVAL, "null operator");
  if (int s = check_dtype(op->d, dtype)) return s;
  if (!in || (!out && !amax)) return fail(FMP_EINVAL, "null buffer");
  fmp_ctx_s* ctx = op->ctx;
  CU(cudaSetDevice(ctx->device));
  CtxLock lk(ctx);
  const size_t eb = fmp::elem_bytes(dtype);
  const size_t inb = batch * (in_omega ? op->d.m : op->d.n) * eb;
  const size_t outb = batch * (out_omega ? op->d.m : op->d.n) * eb;
  cudaStream_t st = ctx->cur;
  lk.use(st);
  void *din = nullptr, *dout = nullptr;
  uint64_t* damax = nullptr;
  if (int s = copy_in(ctx, S_IN, in, inb, &din, st)) return s;
  if (out) ALLOC(dout, S_OUT, outb);
  if (amax) ALLOC(damax, S_IDX, batch * 8);
  if (int s = run_transform(op, dtype, inverse, in_omega, out_omega, din, dout, batch, damax, st))
    return s;
  if (out) CU(cudaMemcpyAsync(out, dout, outb, cudaMemcpyDeviceToHost, st));
  if (amax) CU(cudaMemcpyAsync(amax, damax, batch * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return FMP_OK;
}

int fmp_apply(fmp_op op, int dtype, const void* x, uint64_t batch, void* y_out) {
  if (!y_out) return fail(FMP_EINVAL, "null output");
  return transform_host(op, dtype, 0, 0, 1, x, batch, y_out, nullptr);
}

int fmp_apply_adjoint(fmp_op op, int dtype, const void* r, uint64_t batch, void* h_out,
                      uint64_t* argmax_out) {
  return transform_host(op, dtype, 1, 1, 0, r, batch, h_out, argmax_out);
}

int fmp_unitary_forward(fmp_op op, int dtype, const void* v, uint64_t batch, void* out) {
  if (!out) return fail(FMP_EINVAL, "null output");
  return transform_host(op, dtype, 0, 0, 0, v, batch, out, nullptr);
}

int fmp_unitary_adjoint(fmp_op op, int dtype, const void* v, uint64_t batch, void* out) {
  if (!out) return fail(FMP_EINVAL, "null output");
  return transform_host(op, dtype, 1, 0, 0, v, batch, out, nullptr);
}

int fmp_apply_dev(fmp_op op, int dtype, const void* x, uint64_t batch, void* y_out, void* stream) {
  if (!op || !x || !y_out) return fail(FMP_EINVAL, "null argument");
  if (int s = check_dtype(op->d, dtype)) return s;
  CU(cudaSetDevice(op->ctx->device));
  CtxLock lk(op->ctx);
  cudaStream_t st = pick_stream(op->ctx, stream);
  lk.use(st);
  return run_transform(op, dtype, 0, 0, 1, x, y_out, batch, nullptr, st);
}

int fmp_apply_adjoint_dev(fmp_op op, int dtype, const void* r, uint64_t batch, void* h_out,
                          uint64_t* argmax_out, void* stream) {
  if (!op || !r || (!h_out && !argmax_out)) return fail(FMP_EINVAL, "null argument");
  if (int s = check_dtype(op->d, dtype)) return s;
  CU(cudaSetDevice(op->ctx->device));
  CtxLock lk(op->ctx);
  cudaStream_t st = pick_stream(op->ctx, stream);
  lk.use(st);
  return run_transform(op, dtype, 1, 1, 0, r, h_out, batch, argmax_out, st);
}

// ------------------------------------------------------------ fast update
static int fast_update_dev_locked(fmp_op op, int dtype, const void* h0, const uint32_t* sup0,
                                  const void* coeffs, uint64_t t, uint64_t batch, void* h_out,
                                  uint64_t* amax, cudaStream_t st) {
  fmp_ctx_s* ctx = op->ctx;
  if (op->d.kind == fmp::HADAMARD && !op->d.glat)
    return fail(FMP_EUNSUPPORTED, "hadamard fast update needs m <= 32767 (int16 lattice)");
  fmp::FastUpdateArgs a{};
  a.op = &op->d;
  a.dtype = dtype;
  a.h0 = h0;
  a.support = sup0;
  a.coeffs = coeffs;
  a.t = (int64_t)t;
  a.batch = (int64_t)batch;
  a.h_out = h_out;
  a.argmax_out = amax;
  a.grid = fmp::fast_update_grid(op->d, dtype, (int64_t)batch);
  if (!h_out && t > 1024) {
    void* hb;
    ALLOC(hb, S_AUX, batch * op->d.n * fmp::elem_bytes(dtype));
    a.h_out = hb;
  }
  double* mag;
  ALLOC(mag, S_MAG, (size_t)a.grid * op->d.n * 8);
  a.mag_ws = mag;
  CU(fmp::launch_fast_update(a, st));
  g_launch_count = fmp::last_launch_count();
  return FMP_OK;
}

int fmp_fast_update(fmp_op op, int dtype, const void* h0, const uint64_t* support,
                    const void* coeffs, uint64_t t, uint64_t batch, void* h_out,
                    uint64_t* argmax_out) {
  if (!op) return fail(FMP_EINVAL, "null operator");
  if (int s = check_dtype(op->d, dtype)) return s;
  if (!h0 || (t && (!support || !coeffs)) || (!h_out && !argmax_out))
    return fail(FMP_EINVAL, "null buffer");
  const uint64_t n = (uint64_t)op->d.n;
  // kernel.cpp:213-222: support within 1..n and distinct, per problem
  std::vector<uint32_t> s0(batch * t);
  std::vector<uint64_t> tmp(t);
  for (uint64_t b = 0; b < batch; ++b) {
    for (uint64_t i = 0; i < t; ++i) {
      const uint64_t v = support[b * t + i];
      if (v < 1 || v > n) return fail(FMP_EINVAL, "fast_update: support index out of range");
      s0[b * t + i] = (uint32_t)(v - 1);
      tmp[i] = v;
    }
    std::sort(tmp.begin(), tmp.end());
    for (uint64_t i = 1; i < t; ++i)
      if (tmp[i] == tmp[i - 1]) return fail(FMP_EINVAL, "fast_update: duplicate support index");
  }
  fmp_ctx_s* ctx = op->ctx;
  CU(cudaSetDevice(ctx->device));
  CtxLock lk(ctx);
  cudaStream_t st = ctx->cur;
  lk.use(st);
  const size_t eb = fmp::elem_bytes(dtype);
  void *dh0, *dsup = nullptr, *dco = nullptr, *dout = nullptr;
  uint64_t* damax = nullptr;
  if (int s = copy_in(ctx, S_IN, h0, batch * n * eb, &dh0, st)) return s;
  if (t) {
    if (int s = copy_in(ctx, S_SUP, s0.data(), s0.size() * 4, &dsup, st)) return s;
    if (int s = copy_in(ctx, S_CO, coeffs, batch * t * eb, &dco, st)) return s;
  }
  if (h_out) ALLOC(dout, S_OUT, batch * n * eb);
  if (argmax_out) ALLOC(damax, S_IDX, batch * 8);
  if (int s = fast_update_dev_locked(op, dtype, dh0, (const uint32_t*)dsup, dco, t, batch, dout,
                                     damax, st))
    return s;
  if (h_out) CU(cudaMemcpyAsync(h_out, dout, batch * n * eb, cudaMemcpyDeviceToHost, st));
  if (argmax_out) CU(cudaMemcpyAsync(argmax_out, damax, batch * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return FMP_OK;
}

int fmp_fast_update_dev(fmp_op op, int dtype, const void* h0, const uint32_t* support0,
                        const void* coeffs, uint64_t t, uint64_t batch, void* h_out,
                        uint64_t* argmax_out, void* stream) {
  if (!op) return fail(FMP_EINVAL, "null operator");
  if (int s = check_dtype(op->d, dtype)) return s;
  if (!h0 || (t && (!support0 || !coeffs)) || (!h_out && !argmax_out))
    return fail(FMP_EINVAL, "null buffer");
  CU(cudaSetDevice(op->ctx->device));
  CtxLock lk(op->ctx);
  cudaStream_t st = pick_stream(op->ctx, stream);
  lk.use(st);
  return fast_update_dev_locked(op, dtype, h0, support0, coeffs, t, batch, h_out, argmax_out, st);
}

int fmp_argmax_band(fmp_ctx ctx, int dtype, const void* h, uint64_t n, uint64_t batch,
                    uint64_t* idx_out) {
  if (!ctx || !h || !idx_out) return fail(FMP_EINVAL, "null argument");
  if (dtype < 0 || dtype > 3) return fail(FMP_EINVAL, "unknown dtype");
  if (n == 0) return fail(FMP_EINVAL, "empty vector");
  CU(cudaSetDevice(ctx->device));
  CtxLock lk(ctx);
  cudaStream_t st = ctx->cur;
  lk.use(st);
  void* dh;
  uint64_t* di;
  if (int s = copy_in(ctx, S_IN, h, batch * n * fmp::elem_bytes(dtype), &dh, st)) return s;
  ALLOC(di, S_IDX, batch * 8);
  fmp::ArgmaxArgs a{dtype, dh, (int64_t)n, (int64_t)batch, di};
  CU(fmp::launch_argmax(a, st));
  g_launch_count = 1;
  CU(cudaMemcpyAsync(idx_out, di, batch * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return FMP_OK;
}

// ------------------------------------------------------------ least squares
int fmp_least_squares(fmp_op op, int dtype, const void* y, const uint64_t* support, uint64_t s,
                      uint64_t batch, double* coeffs_out, int64_t* position) {
  if (!op || !y || (s && (!support || !coeffs_out))) return fail(FMP_EINVAL, "null argument");
  if (int st = check_dtype(op->d, dtype)) return st;
  if (s > 4096) return fail(FMP_EUNSUPPORTED, "support larger than 4096");
  const uint64_t n = (uint64_t)op->d.n, m = (uint64_t)op->d.m;
  std::vector<uint32_t> s0(batch * s);
  for (uint64_t i = 0; i < batch * s; ++i) {
    if (support[i] < 1 || support[i] > n) return fail(FMP_EINVAL, "least_squares: support index out of range");
    s0[i] = (uint32_t)(support[i] - 1);
  }
  if (s == 0) return FMP_OK;
  fmp_ctx_s* ctx = op->ctx;
  CU(cudaSetDevice(ctx->device));
  CtxLock lk(ctx);
  cudaStream_t st = ctx->cur;
  lk.use(st);
  void *dy, *dsup;
  if (int e = copy_in(ctx, S_IN, y, batch * m * fmp::elem_bytes(dtype), &dy, st)) return e;
  if (int e = copy_in(ctx, S_SUP, s0.data(), s0.size() * 4, &dsup, st)) return e;
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(batch, 1024));
  double2 *dx, *dL;
  int64_t* dbad;
  ALLOC(dx, S_OCO, batch * s * 16);
  ALLOC(dbad, S_IDX, batch * 8);
  ALLOC(dL, S_W, (size_t)grid * s * s * 16);
  CU(fmp::launch_least_squares(op->d, dtype, dy, (const uint32_t*)dsup, (int)s, (int64_t)batch, dx,
                               dbad, dL, grid, st));
  g_launch_count = 1;
  std::vector<int64_t> bad(batch);
  CU(cudaMemcpyAsync(coeffs_out, dx, batch * s * 16, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(bad.data(), dbad, batch * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  for (uint64_t b = 0; b < batch; ++b)
    if (bad[b] >= 0) {
      if (position) *position = bad[b];
      return fail(FMP_ERANK, "least_squares: dependent column at support position %lld (problem %llu)",
                  (long long)bad[b], (unsigned long long)b);
    }
  return FMP_OK;
}

// -------------------------------------------------------------------- OMP
static int omp_validate(fmp_op op, int dtype, const fmp_omp_config* cfg) {
  if (!op || !cfg) return fail(FMP_EINVAL, "null argument");
  if (int s = check_dtype(op->d, dtype)) return s;
  if (cfg->max_iterations < 1) return fail(FMP_EINVAL, "omp_solve: max_iterations must be >= 1");
  if (!cfg->tolerances && !(cfg->tolerance >= 0.0))
    return fail(FMP_EINVAL, "omp_solve: tolerance must be >= 0");
  if (cfg->mode < 0 || cfg->mode > 4) return fail(FMP_EINVAL, "unknown correlation mode");
  if (cfg->max_iterations > 4096) return fail(FMP_EUNSUPPORTED, "max_iterations > 4096");
  if (op->d.kind == fmp::HADAMARD && !op->d.glat)
    return fail(FMP_EUNSUPPORTED, "hadamard solve needs m <= 32767 (int16 lattice)");
  return FMP_OK;
}

static int64_t fast_until_of(fmp_op op, const fmp_omp_config* cfg, int dtype, uint64_t batch) {
  switch (cfg->mode) {
    case FMP_MODE_CONVENTIONAL: return 0;
    case FMP_MODE_FAST: return std::numeric_limits<int64_t>::max();
    case FMP_MODE_ADAPTIVE: return (int64_t)fmp_crossover_iteration(op->d.kind, (uint64_t)op->d.n);
    case FMP_MODE_GPU:
      return fmp::omp_gpu_fast_until(op->d, dtype, (int64_t)batch, (int64_t)cfg->max_iterations);
    default: return (int64_t)std::min<uint64_t>(cfg->fast_until, (uint64_t)INT64_MAX);
  }
}

// wsset: which set of per-CTA workspaces (two launches may run concurrently
// on different streams, each with its own set)
static int omp_dev_locked(fmp_op op, int dtype, const void* y, uint64_t batch,
                          const fmp_omp_config* cfg, const double* dtol, fmp_omp_result* out,
                          cudaStream_t st, int wsset = 0, const int* ready = nullptr,
                          int64_t ready_chunk = 0, int* queue_zeroed = nullptr) {
  const int wo = wsset ? S_ALT : 0;  // slot offset of the alternate set
  fmp_ctx_s* ctx = op->ctx;
  const int64_t T = (int64_t)cfg->max_iterations;
  const int64_t n = op->d.n, m = op->d.m;
  const size_t eb = fmp::elem_bytes(dtype);
  fmp::OmpArgs a{};
  a.op = &op->d;
  a.dtype = dtype;
  a.y = y;
  a.tol = dtol;
  a.batch = (int64_t)batch;
  a.max_iter = T;
  a.fast_until = fast_until_of(op, cfg, dtype, batch);
  a.support = out->support;
  a.coeffs = (double2*)out->coeffs;
  a.size = out->support_size;
  a.iters = out->iterations;
  a.resid = out->residual;
  a.aborted = out->aborted;
  a.modes = out->modes;
  a.hlen = out->history_len;
  a.hist = cfg->record_correlations ? out->history : nullptr;
  a.grid = fmp::omp_grid(op->d, dtype, (int64_t)batch, T);
  a.ready = ready;
  a.ready_chunk = ready_chunk;
  a.abort_word = ctx->abort_dev;
  if (!fmp::is_double(dtype)) {
    // fp32 data: the fp64 h0 = Phi^H y of every problem (the widened fp32
    // measurements through the fp64 transform), from which the solver
    // re-evaluates its identification candidates and takes the least-squares
    // right-hand side.  Needs the whole input: not on the streamed path.
    if (ready) return fail(FMP_EINVAL, "internal: streamed input with fp32 data");
    const int wdt = fmp::is_complex(dtype) ? FMP_C128 : FMP_F64;
    const size_t web = (size_t)fmp::elem_bytes(wdt);
    double* y64;
    ALLOC(y64, wo + S_Y64, batch * m * web);
    CU(fmp::launch_widen((const float*)y, y64, (int64_t)(batch * m * (web / 8)), st));
    void* h0x;
    ALLOC(h0x, wo + S_H0X, batch * n * web);
    if (int s = run_transform(op, wdt, 1, 1, 0, y64, h0x, batch, nullptr, st, wo)) return s;
    a.h0x = h0x;
    if (g_phase_prof) {
      unsigned long long* rs;
      ALLOC(rs, S_RST, 64);
      CU(cudaMemsetAsync(rs, 0, 64, st));
      a.rstats = rs;
    }
  }
  double2* w;
  ALLOC(w, wo + S_W, (size_t)a.grid * (T * (T + 1) / 2) * 16);
  a.w_ws = w;
  void* h0;
  ALLOC(h0, wo + S_H0, (size_t)a.grid * n * eb);
  a.h0_ws = h0;
  double* mag;
  ALLOC(mag, wo + S_MAG, (size_t)a.grid * n * 8);
  a.mag_ws = mag;
  void* r;
  ALLOC(r, wo + S_R, (size_t)a.grid * m * eb);
  a.r_ws = r;
  void* ysw;
  ALLOC(ysw, wo + S_YS, (size_t)a.grid * m * eb);
  a.ys_ws = ysw;
  if (n > fmp::transform_max_n(dtype) / 2) {
    void* bw;
    ALLOC(bw, wo + S_BUF, (size_t)a.grid * (n + n / 8) * eb);
    a.buf_ws = bw;
  }
  int* q = queue_zeroed;  // (a caller's copy already cleared it)
  if (!q) {
    ALLOC(q, wo + S_Q, 64);
    CU(cudaMemsetAsync(q, 0, 4, st));
  }
  a.queue = q;
  if (g_phase_prof) {
    unsigned long long* ph;
    ALLOC(ph, S_PH, 64);
    CU(cudaMemsetAsync(ph, 0, 64, st));
    a.phase_ws = ph;
  }
  cudaError_t e = fmp::launch_omp(a, st);
  g_launch_count = fmp::last_launch_count();
  if (e == cudaErrorInvalidConfiguration)
    return fail(FMP_EUNSUPPORTED, "n = %lld, max_iterations = %lld exceed the fused solver's "
                "shared-memory plan", (long long)n, (long long)T);
  CU(e);
  return FMP_OK;
}

int fmp_omp_solve_dev(fmp_op op, int dtype, const void* y, uint64_t batch,
                      const fmp_omp_config* cfg, fmp_omp_result* out, void* stream) {
  if (int s = omp_validate(op, dtype, cfg)) return s;
  if (!y || !out || !out->support || !out->coeffs || !out->support_size || !out->iterations ||
      !out->residual || !out->aborted)
    return fail(FMP_EINVAL, "null buffer");
  fmp_ctx_s* ctx = op->ctx;
  CU(cudaSetDevice(ctx->device));
  CtxLock lk(ctx);
  cudaStream_t st = pick_stream(ctx, stream);
  lk.use(st);
  const double* dtol = cfg->tolerances;
  if (!dtol) {
    std::vector<double> tv(batch, cfg->tolerance);
    void* p;
    if (int s = copy_in(ctx, S_TOL, tv.data(), batch * 8, &p, st)) return s;
    CU(cudaStreamSynchronize(st));  // the host vector dies here
    dtol = (const double*)p;
  }
  return omp_dev_locked(op, dtype, y, batch, cfg, dtol, out, st);
}

static bool host_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

static int pinned_reserve(fmp_ctx_s* ctx, size_t bytes) {
  if (ctx->pinned_bytes >= bytes) return FMP_OK;
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  ctx->pinned = nullptr;
  ctx->pinned_bytes = 0;
  cudaError_t e = cudaHostAlloc(&ctx->pinned, bytes, cudaHostAllocDefault);
  if (e != cudaSuccess) return fail(FMP_ENOMEM, "page-locked staging (%zu bytes): %s", bytes, cudaGetErrorString(e));
  ctx->pinned_bytes = bytes;
  return FMP_OK;
}

// Host buffers, one launch: the solver starts at once and each CTA waits
// (acquire spin) for the chunk holding its next problem; the copy stream moves
// the measurements in chunks of one problem per CTA, each followed by a 4-byte
// copy that raises the chunk's flag.  Results go straight into the caller's
// page-locked buffers (stores over the host link as problems finish), so
// nothing is exposed but the first chunk's copy and the wave tail.  Used when
// every result buffer is page-locked (else omp_host_chunked).
// stream_in_setup: device buffers for y and the tolerances, the cleared
// flags, the tolerances copied; the copy stream ordered after the clear.
static int stream_in_setup(fmp_ctx_s* ctx, const void* y, uint64_t batch, size_t row_bytes,
                           const fmp_omp_config* cfg, uint64_t nchunk, void** dy, void** dtol,
                           int** flags, cudaStream_t st) {
  if (!ctx->copy) CU(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
  if (!ctx->abort_host) {
    int* h = nullptr;
    CU(cudaHostAlloc((void**)&h, 64, cudaHostAllocMapped));
    void* dv = nullptr;
    cudaError_t e = cudaHostGetDevicePointer(&dv, h, 0);
    if (e != cudaSuccess) {
      cudaFreeHost(h);
      return fail(FMP_ECUDA, "abort word: %s", cudaGetErrorString(e));
    }
    ctx->abort_host = h;
    ctx->abort_dev = (const volatile int*)dv;
  }
  *(volatile int*)ctx->abort_host = 0;
  // page-locked: the staged measurements (pageable callers), then the flag
  // source (one int = 1)
  const size_t in_bytes = !host_pinned(y) ? ((batch * row_bytes + 255) & ~size_t(255)) : 0;
  if (int e = pinned_reserve(ctx, in_bytes + 256 + batch * 8)) return e;
  *(int*)((char*)ctx->pinned + in_bytes) = 1;
  double* ptol = (double*)((char*)ctx->pinned + in_bytes + 256);  // tolerances, page-locked
  if (ctx->events.empty()) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->events.push_back(e);
  }
  ALLOC(*dy, S_IN, batch * row_bytes);
  ALLOC(*dtol, S_TOL, batch * 8);
  ALLOC(*flags, S_SYNC, nchunk * 4);
  CU(cudaMemsetAsync(*flags, 0, nchunk * 4, st));
  if (cfg->tolerances) std::memcpy(ptol, cfg->tolerances, batch * 8);
  else std::fill(ptol, ptol + batch, cfg->tolerance);
  CU(cudaMemcpyAsync(*dtol, ptol, batch * 8, cudaMemcpyHostToDevice, st));
  CU(cudaEventRecord(ctx->events[0], st));
  CU(cudaStreamWaitEvent(ctx->copy, ctx->events[0], 0));
  return FMP_OK;
}

// after the launch: the chunks and their flags on the copy stream, then wait.
// Any failure raises the abort word first, so the kernel spinning on the
// remaining flags returns (its problems marked kInputLost) instead of hanging
static int stream_in_chunks(fmp_ctx_s* ctx, const void* y, uint64_t batch, size_t row_bytes,
                            uint64_t per, void* dy, int* flags, cudaStream_t st);
static int stream_in_finish(fmp_ctx_s* ctx, const void* y, uint64_t batch, size_t row_bytes,
                            uint64_t per, void* dy, int* flags, cudaStream_t st,
                            const int32_t* aborted_host = nullptr) {
  const int rc = stream_in_chunks(ctx, y, batch, row_bytes, per, dy, flags, st);
  if (rc != FMP_OK) {
    *(volatile int*)ctx->abort_host = 1;
    cudaStreamSynchronize(st);
    cudaStreamSynchronize(ctx->copy);
    return rc;
  }
  if (aborted_host)
    for (uint64_t b = 0; b < batch; ++b)
      if (aborted_host[b] == 2)
        return fail(FMP_ECUDA, "streamed input: problem %llu never arrived (copy stream stalled)",
                    (unsigned long long)b);
  return FMP_OK;
}
static int stream_in_chunks(fmp_ctx_s* ctx, const void* y, uint64_t batch, size_t row_bytes,
                            uint64_t per, void* dy, int* flags, cudaStream_t st) {
  cudaStream_t cp = ctx->copy;
  const bool stage_in = !host_pinned(y);
  const size_t in_bytes = stage_in ? ((batch * row_bytes + 255) & ~size_t(255)) : 0;
  char* pin_in = (char*)ctx->pinned;
  const int* one = (const int*)((char*)ctx->pinned + in_bytes);
  const uint64_t nchunk = (batch + per - 1) / per;
  // test hook: the host side fails after the first chunk (error-path test)
  const char* stall = getenv("FMP_TEST_STALL_INPUT");
  for (uint64_t c = 0; c < nchunk; ++c) {
    if (c == 1 && stall && *stall == '1') return fail(FMP_ECUDA, "input stream failed (test hook)");
    const uint64_t b0 = c * per, nb = std::min(per, batch - b0);
    const char* src = (const char*)y + b0 * row_bytes;
    if (stage_in) {  // overlaps the solve and the previous chunk's transfer
      std::memcpy(pin_in + b0 * row_bytes, src, nb * row_bytes);
      src = pin_in + b0 * row_bytes;
    }
    CU(cudaMemcpyAsync((char*)dy + b0 * row_bytes, src, nb * row_bytes, cudaMemcpyHostToDevice, cp));
    CU(cudaMemcpyAsync(flags + c, one, 4, cudaMemcpyHostToDevice, cp));
  }
  CU(cudaStreamSynchronize(st));
  CU(cudaStreamSynchronize(cp));
  return FMP_OK;
}

static int omp_host_streamed(fmp_op op, int dtype, const void* y, uint64_t batch,
                             const fmp_omp_config* cfg, fmp_omp_result* out, uint64_t per) {
  fmp_ctx_s* ctx = op->ctx;
  cudaStream_t st = ctx->cur;
  const size_t row_bytes = (size_t)op->d.m * fmp::elem_bytes(dtype);
  const uint64_t nchunk = (batch + per - 1) / per;
  void *dy, *dtol;
  int* flags;
  if (int e = stream_in_setup(ctx, y, batch, row_bytes, cfg, nchunk, &dy, &dtol, &flags, st)) return e;
  if (int e = omp_dev_locked(op, dtype, dy, batch, cfg, (const double*)dtol, out, st, 0, flags,
                             (int64_t)per)) {
    *(volatile int*)ctx->abort_host = 1;  // nothing was launched, or it must not wait
    cudaStreamSynchronize(st);
    return e;
  }
  return stream_in_finish(ctx, y, batch, row_bytes, per, dy, flags, st, out->aborted);
}

// host-buffer solve in chunks: the copy stream moves chunk c + 1 in (and
// chunk c - 1's results out) while the context stream solves chunk c
static int omp_host_chunked(fmp_op op, int dtype, const void* y, uint64_t batch,
                            const fmp_omp_config* cfg, fmp_omp_result* out, uint64_t nchunk) {
  fmp_ctx_s* ctx = op->ctx;
  cudaStream_t st = ctx->cur;
  if (!ctx->copy) CU(cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking));
  if (!ctx->alt) CU(cudaStreamCreateWithFlags(&ctx->alt, cudaStreamNonBlocking));
  cudaStream_t cp = ctx->copy;
  // pageable host buffers go through a page-locked staging area (a host
  // memcpy per chunk that overlaps the device work of the other chunks)
  // instead of the driver's synchronous staged copies
  const uint64_t T_ = cfg->max_iterations, m_ = (uint64_t)op->d.m;
  const size_t eb_ = fmp::elem_bytes(dtype);
  const bool stage_in = !host_pinned(y), stage_out = !host_pinned(out->support);
  const size_t in_bytes = stage_in ? batch * m_ * eb_ : 0;
  const size_t out_row = T_ * 8 + T_ * 16 + 8 + 8 + 8 + 4;  // support, coeffs, size, iters, resid, aborted
  const size_t out_bytes = stage_out ? batch * out_row : 0;
  if (stage_in || stage_out)
    if (int e = pinned_reserve(ctx, in_bytes + out_bytes)) return e;
  char* pin_in = (char*)ctx->pinned;
  char* pin_out = (char*)ctx->pinned + in_bytes;
  while (ctx->events.size() < 3 * nchunk + 2) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ctx->events.push_back(e);
  }
  cudaEvent_t* ev_in = ctx->events.data();
  cudaEvent_t* ev_out = ev_in + nchunk;
  cudaEvent_t ev_ready = ev_in[2 * nchunk], ev_alt = ev_in[2 * nchunk + 1];
  cudaEvent_t* ev_d2h = ev_in + 2 * nchunk + 2;
  // chunks alternate between the context stream and a second one, each with
  // its own workspaces, so a chunk's CTAs backfill SMs while the previous
  // chunk's last problems finish
  cudaStream_t cs[2] = {st, ctx->alt};
  const uint64_t T = cfg->max_iterations, m = (uint64_t)op->d.m;
  const size_t eb = fmp::elem_bytes(dtype);
  // device buffers for the whole batch (results stay addressable per chunk)
  void *dy, *dtol;
  ALLOC(dy, S_IN, batch * m * eb);
  ALLOC(dtol, S_TOL, batch * 8);
  fmp_omp_result d{};
  ALLOC(d.support, S_OSUP, batch * T * 8);
  ALLOC(d.coeffs, S_OCO, batch * T * 16);
  ALLOC(d.support_size, S_OSZ, batch * 8);
  ALLOC(d.iterations, S_OIT, batch * 8);
  ALLOC(d.residual, S_ORES, batch * 8);
  ALLOC(d.aborted, S_OAB, batch * 4);
  if (out->modes) ALLOC(d.modes, S_OMOD, batch * T);
  if (out->history_len) ALLOC(d.history_len, S_OHL, batch * 8);
  std::vector<double> tv;
  if (!cfg->tolerances) tv.assign(batch, cfg->tolerance);
  // the copy stream starts after everything already queued on the context stream
  CU(cudaEventRecord(ev_ready, st));
  CU(cudaStreamWaitEvent(cp, ev_ready, 0));
  CU(cudaStreamWaitEvent(ctx->alt, ev_ready, 0));
  CU(cudaMemcpyAsync(dtol, cfg->tolerances ? cfg->tolerances : tv.data(), batch * 8,
                     cudaMemcpyHostToDevice, cp));
  const uint64_t per = (batch + nchunk - 1) / nchunk;
  for (uint64_t c = 0; c < nchunk; ++c) {
    const uint64_t b0 = c * per, nb = std::min(per, batch - b0);
    const char* src = (const char*)y + b0 * m * eb;
    if (stage_in) {  // (the host copy of chunk c overlaps the transfer of chunk c - 1)
      std::memcpy(pin_in + b0 * m * eb, src, nb * m * eb);
      src = pin_in + b0 * m * eb;
    }
    CU(cudaMemcpyAsync((char*)dy + b0 * m * eb, src, nb * m * eb, cudaMemcpyHostToDevice, cp));
    CU(cudaEventRecord(ev_in[c], cp));
  }
  for (uint64_t c = 0; c < nchunk; ++c) {
    const uint64_t b0 = c * per, nb = std::min(per, batch - b0);
    cudaStream_t sc = cs[c & 1];
    CU(cudaStreamWaitEvent(sc, ev_in[c], 0));
    fmp_omp_result dc{};
    dc.support = d.support + b0 * T;
    dc.coeffs = d.coeffs + 2 * b0 * T;
    dc.support_size = d.support_size + b0;
    dc.iterations = d.iterations + b0;
    dc.residual = d.residual + b0;
    dc.aborted = d.aborted + b0;
    dc.modes = d.modes ? d.modes + b0 * T : nullptr;
    dc.history_len = d.history_len ? d.history_len + b0 : nullptr;
    if (int e = omp_dev_locked(op, dtype, (const char*)dy + b0 * m * eb, nb, cfg,
                               (const double*)dtol + b0, &dc, sc, (int)(c & 1)))
      return e;
    CU(cudaEventRecord(ev_out[c], sc));
    CU(cudaStreamWaitEvent(cp, ev_out[c], 0));
    // results of chunk c: straight into page-locked user buffers, or into
    // the staging area (copied out below, chunk by chunk)
    uint64_t* o_sup = out->support + b0 * T;
    double* o_co = out->coeffs + 2 * b0 * T;
    uint64_t* o_sz = out->support_size + b0;
    uint64_t* o_it = out->iterations + b0;
    double* o_rn = out->residual + b0;
    int32_t* o_ab = out->aborted + b0;
    if (stage_out) {
      char* base = pin_out + b0 * out_row;
      o_sup = (uint64_t*)base;
      o_co = (double*)(base + nb * T * 8);
      o_sz = (uint64_t*)(base + nb * (T * 24));
      o_it = o_sz + nb;
      o_rn = (double*)(o_it + nb);
      o_ab = (int32_t*)(o_rn + nb);
    }
    CU(cudaMemcpyAsync(o_sup, dc.support, nb * T * 8, cudaMemcpyDeviceToHost, cp));
    CU(cudaMemcpyAsync(o_co, dc.coeffs, nb * T * 16, cudaMemcpyDeviceToHost, cp));
    CU(cudaMemcpyAsync(o_sz, dc.support_size, nb * 8, cudaMemcpyDeviceToHost, cp));
    CU(cudaMemcpyAsync(o_it, dc.iterations, nb * 8, cudaMemcpyDeviceToHost, cp));
    CU(cudaMemcpyAsync(o_rn, dc.residual, nb * 8, cudaMemcpyDeviceToHost, cp));
    CU(cudaMemcpyAsync(o_ab, dc.aborted, nb * 4, cudaMemcpyDeviceToHost, cp));
    CU(cudaEventRecord(ev_d2h[c], cp));
    if (out->modes) CU(cudaMemcpyAsync(out->modes + b0 * T, dc.modes, nb * T, cudaMemcpyDeviceToHost, cp));
    if (out->history_len)
      CU(cudaMemcpyAsync(out->history_len + b0, dc.history_len, nb * 8, cudaMemcpyDeviceToHost, cp));
  }
  if (stage_out)
    for (uint64_t c = 0; c < nchunk; ++c) {  // overlaps the device work of later chunks
      const uint64_t b0 = c * per, nb = std::min(per, batch - b0);
      CU(cudaEventSynchronize(ev_d2h[c]));
      const char* base = pin_out + b0 * out_row;
      std::memcpy(out->support + b0 * T, base, nb * T * 8);
      std::memcpy(out->coeffs + 2 * b0 * T, base + nb * T * 8, nb * T * 16);
      const char* tail = base + nb * T * 24;
      std::memcpy(out->support_size + b0, tail, nb * 8);
      std::memcpy(out->iterations + b0, tail + nb * 8, nb * 8);
      std::memcpy(out->residual + b0, tail + nb * 16, nb * 8);
      std::memcpy(out->aborted + b0, tail + nb * 24, nb * 4);
    }
  // the context stream owns the end of the call (later work queued on it
  // sees every chunk)
  CU(cudaEventRecord(ev_alt, ctx->alt));
  CU(cudaStreamWaitEvent(st, ev_alt, 0));
  CU(cudaStreamSynchronize(cp));
  CU(cudaStreamSynchronize(st));
  return FMP_OK;
}

// Host buffers, small batches (latency regime, e.g. config 1): the inputs
// (measurements, tolerances, a zeroed work counter) staged in the context's
// page-locked block and moved by ONE copy, one launch, every result written
// to one device block and returned by ONE copy, one synchronisation; the
// per-call API work is four calls instead of a dozen
static int omp_host_small(fmp_op op, int dtype, const void* y, uint64_t batch,
                          const fmp_omp_config* cfg, fmp_omp_result* out, cudaStream_t st) {
  fmp_ctx_s* ctx = op->ctx;
  const uint64_t T = cfg->max_iterations, m = (uint64_t)op->d.m;
  const size_t eb = fmp::elem_bytes(dtype);
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  // input block: y | tolerances | work counter
  const size_t o_tol = al(batch * m * eb), o_q = o_tol + al(batch * 8), in_bytes = o_q + 256;
  // result block, each array 256-aligned
  const size_t o_sup = 0, o_co = o_sup + al(batch * T * 8), o_sz = o_co + al(batch * T * 16),
               o_it = o_sz + al(batch * 8), o_rn = o_it + al(batch * 8), o_ab = o_rn + al(batch * 8),
               o_md = o_ab + al(batch * 4), o_hl = o_md + al(batch * T),
               out_bytes = o_hl + al(batch * 8);
  if (int e = pinned_reserve(ctx, in_bytes + out_bytes)) return e;
  char* hin = (char*)ctx->pinned;
  char* hout = hin + in_bytes;
  std::memcpy(hin, y, batch * m * eb);
  double* htol = (double*)(hin + o_tol);
  if (cfg->tolerances) std::memcpy(htol, cfg->tolerances, batch * 8);
  else std::fill(htol, htol + batch, cfg->tolerance);
  std::memset(hin + o_q, 0, 4);
  char* din;
  ALLOC(din, S_IN, in_bytes + out_bytes);
  char* dout = din + in_bytes;
  CU(cudaMemcpyAsync(din, hin, in_bytes, cudaMemcpyHostToDevice, st));
  fmp_omp_result d{};
  d.support = (uint64_t*)(dout + o_sup);
  d.coeffs = (double*)(dout + o_co);
  d.support_size = (uint64_t*)(dout + o_sz);
  d.iterations = (uint64_t*)(dout + o_it);
  d.residual = (double*)(dout + o_rn);
  d.aborted = (int32_t*)(dout + o_ab);
  d.modes = out->modes ? (uint8_t*)(dout + o_md) : nullptr;
  d.history_len = out->history_len ? (uint64_t*)(dout + o_hl) : nullptr;
  if (int s = omp_dev_locked(op, dtype, din, batch, cfg, (const double*)(din + o_tol), &d, st, 0,
                             nullptr, 0, (int*)(din + o_q)))
    return s;
  CU(cudaMemcpyAsync(hout, dout, out_bytes, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  std::memcpy(out->support, hout + o_sup, batch * T * 8);
  std::memcpy(out->coeffs, hout + o_co, batch * T * 16);
  std::memcpy(out->support_size, hout + o_sz, batch * 8);
  std::memcpy(out->iterations, hout + o_it, batch * 8);
  std::memcpy(out->residual, hout + o_rn, batch * 8);
  std::memcpy(out->aborted, hout + o_ab, batch * 4);
  if (out->modes) std::memcpy(out->modes, hout + o_md, batch * T);
  if (out->history_len) std::memcpy(out->history_len, hout + o_hl, batch * 8);
  return FMP_OK;
}

int fmp_omp_solve(fmp_op op, int dtype, const void* y, uint64_t batch, const fmp_omp_config* cfg,
                  fmp_omp_result* out) {
  if (int s = omp_validate(op, dtype, cfg)) return s;
  if (!y || !out || !out->support || !out->coeffs || !out->support_size || !out->iterations ||
      !out->residual || !out->aborted)
    return fail(FMP_EINVAL, "null buffer");
  if (cfg->record_correlations && !out->history)
    return fail(FMP_EINVAL, "record_correlations needs a history buffer");
  if (cfg->tolerances)
    for (uint64_t b = 0; b < batch; ++b)
      if (!(cfg->tolerances[b] >= 0.0)) return fail(FMP_EINVAL, "omp_solve: tolerance must be >= 0");
  fmp_ctx_s* ctx = op->ctx;
  CU(cudaSetDevice(ctx->device));
  CtxLock lk(ctx);
  cudaStream_t st = ctx->cur;
  lk.use(st);
  const uint64_t T = cfg->max_iterations, n = (uint64_t)op->d.n, m = (uint64_t)op->d.m;
  const size_t eb = fmp::elem_bytes(dtype);
  // large batches: copies overlapped with the solve, chunk by chunk (each
  // chunk still fills the GPU several times over)
  const uint64_t grid = (uint64_t)fmp::omp_grid(op->d, dtype, (int64_t)batch, (int64_t)T);
  if (!cfg->record_correlations && !g_phase_prof && batch >= 8 * grid) {
    const char* e = getenv("FMP_HOST_PATH");  // "chunked": the multi-launch path (timing tools)
    const bool pinned_out = host_pinned(out->support) && host_pinned(out->coeffs) &&
                            host_pinned(out->support_size) && host_pinned(out->iterations) &&
                            host_pinned(out->residual) && host_pinned(out->aborted) &&
                            (!out->modes || host_pinned(out->modes)) &&
                            (!out->history_len || host_pinned(out->history_len));
    // (fp32 data needs the whole batch for its fp64 h0 before the solve)
    if (pinned_out && !(e && !strcmp(e, "chunked")) && fmp::is_double(dtype))
      return omp_host_streamed(op, dtype, y, batch, cfg, out, grid);
    return omp_host_chunked(op, dtype, y, batch, cfg, out, std::min<uint64_t>(8, batch / (2 * grid)));
  }
  if (!cfg->record_correlations && batch <= grid) return omp_host_small(op, dtype, y, batch, cfg, out, st);
  void* dy;
  if (int s = copy_in(ctx, S_IN, y, batch * m * eb, &dy, st)) return s;
  std::vector<double> tv;
  if (!cfg->tolerances) tv.assign(batch, cfg->tolerance);
  void* dtol;
  if (int s = copy_in(ctx, S_TOL, cfg->tolerances ? cfg->tolerances : tv.data(), batch * 8, &dtol, st))
    return s;
  fmp_omp_result d{};
  ALLOC(d.support, S_OSUP, batch * T * 8);
  ALLOC(d.coeffs, S_OCO, batch * T * 16);
  ALLOC(d.support_size, S_OSZ, batch * 8);
  ALLOC(d.iterations, S_OIT, batch * 8);
  ALLOC(d.residual, S_ORES, batch * 8);
  ALLOC(d.aborted, S_OAB, batch * 4);
  if (out->modes) ALLOC(d.modes, S_OMOD, batch * T);
  if (out->history_len || cfg->record_correlations) ALLOC(d.history_len, S_OHL, batch * 8);
  if (cfg->record_correlations) ALLOC(d.history, S_OHIST, batch * T * n * eb);
  if (int s = omp_dev_locked(op, dtype, dy, batch, cfg, (const double*)dtol, &d, st)) return s;
  CU(cudaMemcpyAsync(out->support, d.support, batch * T * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(out->coeffs, d.coeffs, batch * T * 16, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(out->support_size, d.support_size, batch * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(out->iterations, d.iterations, batch * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(out->residual, d.residual, batch * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(out->aborted, d.aborted, batch * 4, cudaMemcpyDeviceToHost, st));
  if (out->modes) CU(cudaMemcpyAsync(out->modes, d.modes, batch * T, cudaMemcpyDeviceToHost, st));
  if (out->history_len)
    CU(cudaMemcpyAsync(out->history_len, d.history_len, batch * 8, cudaMemcpyDeviceToHost, st));
  if (cfg->record_correlations)
    CU(cudaMemcpyAsync(out->history, d.history, batch * T * n * eb, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return FMP_OK;
}

// one host thread per device, contiguous blocks of the batch
int fmp_omp_solve_multi(const fmp_op* ops, int nops, int dtype, const void* y, uint64_t batch,
                        const fmp_omp_config* cfg, fmp_omp_result* out) {
  if (!ops || nops < 1 || !cfg || !out) return fail(FMP_EINVAL, "null argument");
  for (int i = 0; i < nops; ++i) {
    if (!ops[i]) return fail(FMP_EINVAL, "null operator %d", i);
    if (ops[i]->d.kind != ops[0]->d.kind || ops[i]->d.n != ops[0]->d.n || ops[i]->rows != ops[0]->rows)
      return fail(FMP_EINVAL, "fmp_omp_solve_multi: operator %d differs from operator 0", i);
  }
  if (nops == 1) return fmp_omp_solve(ops[0], dtype, y, batch, cfg, out);
  if (int s = omp_validate(ops[0], dtype, cfg)) return s;
  const uint64_t T = cfg->max_iterations, m = (uint64_t)ops[0]->d.m, n = (uint64_t)ops[0]->d.n;
  const size_t eb = fmp::elem_bytes(dtype);
  std::vector<int> status(nops, FMP_OK);
  std::vector<std::string> msg(nops);
  std::vector<std::thread> th;
  const uint64_t q = batch / nops, r = batch % nops;
  for (int i = 0; i < nops; ++i) {
    const uint64_t b0 = i * q + std::min<uint64_t>(i, r), nb = q + (i < (int)r ? 1 : 0);
    if (!nb) continue;
    th.emplace_back([=, &status, &msg]() {
      fmp_omp_config c = *cfg;
      if (cfg->tolerances) c.tolerances = cfg->tolerances + b0;
      fmp_omp_result o = *out;
      o.support = out->support + b0 * T;
      o.coeffs = out->coeffs + 2 * b0 * T;
      o.support_size = out->support_size + b0;
      o.iterations = out->iterations + b0;
      o.residual = out->residual + b0;
      o.aborted = out->aborted + b0;
      if (out->modes) o.modes = out->modes + b0 * T;
      if (out->history_len) o.history_len = out->history_len + b0;
      if (out->history) o.history = (char*)out->history + b0 * T * n * eb;
      status[i] = fmp_omp_solve(ops[i], dtype, (const char*)y + b0 * m * eb, nb, &c, &o);
      if (status[i] != FMP_OK) msg[i] = g_err;
    });
  }
  for (auto& t : th) t.join();
  for (int i = 0; i < nops; ++i)
    if (status[i] != FMP_OK) return fail(status[i], "device block %d: %s", i, msg[i].c_str());
  return FMP_OK;
}

// ------------------------------------------------------------------ CoSaMP
static int cosamp_validate(fmp_op op, int dtype, uint64_t k, const fmp_omp_config* cfg) {
  if (!op || !cfg) return fail(FMP_EINVAL, "null argument");
  if (int s = check_dtype(op->d, dtype)) return s;
  if (cfg->max_iterations < 1) return fail(FMP_EINVAL, "cosamp_solve: max_iterations must be >= 1");
  if (!cfg->tolerances && !(cfg->tolerance >= 0.0))
    return fail(FMP_EINVAL, "cosamp_solve: tolerance must be >= 0");
  if (cfg->mode < 0 || cfg->mode > 4) return fail(FMP_EINVAL, "unknown correlation mode");
  if (k > 1024) return fail(FMP_EUNSUPPORTED, "cosamp_solve: k > 1024");
  if (op->d.kind == fmp::HADAMARD && !op->d.glat)
    return fail(FMP_EUNSUPPORTED, "hadamard solve needs m <= 32767 (int16 lattice)");
  return FMP_OK;
}

static int cosamp_dev_locked(fmp_op op, int dtype, const void* y, uint64_t batch, uint64_t k,
                             const fmp_omp_config* cfg, const double* dtol, fmp_cosamp_result* out,
                             cudaStream_t st, const int* ready = nullptr, int64_t ready_chunk = 0) {
  fmp_ctx_s* ctx = op->ctx;
  const int64_t T = (int64_t)cfg->max_iterations, n = op->d.n, m = op->d.m;
  const size_t eb = fmp::elem_bytes(dtype);
  fmp::CosArgs a{};
  a.op = &op->d;
  a.dtype = dtype;
  a.y = y;
  a.tol = dtol;
  a.batch = (int64_t)batch;
  a.max_iter = T;
  a.k = (int64_t)k;
  bool fast = true;  // FAST, GPU, CUSTOM
  if (cfg->mode == FMP_MODE_CONVENTIONAL) fast = false;
  if (cfg->mode == FMP_MODE_ADAPTIVE)  // cost_model.cpp:76-96
    fast = k == 0 || (op->d.kind == fmp::FOURIER ? 6u : 2u) * (uint64_t)n * k <=
                         (op->d.kind == fmp::FOURIER ? 5u : 2u) * (uint64_t)n * (uint64_t)op->d.log2n;
  a.fast = fast ? 1 : 0;
  a.support = out->support;
  a.coeffs = (double2*)out->coeffs;
  a.size = out->support_size;
  a.iters = out->iterations;
  a.resid = out->residual;
  a.aborted = out->aborted;
  a.hist_sup = out->support_history;
  a.hist = cfg->record_correlations ? out->history : nullptr;
  a.grid = fmp::omp_grid(op->d, dtype, (int64_t)batch, T);
  a.ready = ready;
  a.ready_chunk = ready_chunk;
  a.abort_word = ctx->abort_dev;
  const size_t c3 = 3 * (size_t)std::max<uint64_t>(k, 1);
  double2* L;
  ALLOC(L, S_W, (size_t)std::max(a.grid, 1) * c3 * (c3 + 1) / 2 * 16);
  a.L_ws = L;
  void* h0;
  ALLOC(h0, S_H0, (size_t)std::max(a.grid, 1) * n * eb);
  a.h0_ws = h0;
  double* mag;
  ALLOC(mag, S_MAG, (size_t)std::max(a.grid, 1) * n * 8);
  a.mag_ws = mag;
  void* r;
  ALLOC(r, S_R, (size_t)std::max(a.grid, 1) * m * eb);
  a.r_ws = r;
  int* q;
  ALLOC(q, S_Q, 64);
  a.queue = q;
  CU(cudaMemsetAsync(q, 0, 4, st));
  if (out->support_history)
    CU(cudaMemsetAsync(out->support_history, 0, (size_t)batch * T * k * 8, st));
  if (g_phase_prof) {
    unsigned long long* ph;
    ALLOC(ph, S_PH, 64);
    CU(cudaMemsetAsync(ph, 0, 64, st));
    a.phase_ws = ph;
  }
  if (batch == 0) return FMP_OK;
  cudaError_t e = fmp::launch_cosamp(a, st);
  g_launch_count = fmp::last_launch_count();
  if (e == cudaErrorInvalidConfiguration)
    return fail(FMP_EUNSUPPORTED, "n = %lld, k = %llu exceed the CoSaMP kernel's shared-memory plan",
                (long long)n, (unsigned long long)k);
  CU(e);
  return FMP_OK;
}

int fmp_cosamp_solve_dev(fmp_op op, int dtype, const void* y, uint64_t batch, uint64_t k,
                         const fmp_omp_config* cfg, fmp_cosamp_result* out, void* stream) {
  if (int s = cosamp_validate(op, dtype, k, cfg)) return s;
  if (!y || !out || !out->support || !out->coeffs || !out->support_size || !out->iterations ||
      !out->residual || !out->aborted)
    return fail(FMP_EINVAL, "null buffer");
  fmp_ctx_s* ctx = op->ctx;
  CU(cudaSetDevice(ctx->device));
  CtxLock lk(ctx);
  cudaStream_t st = pick_stream(ctx, stream);
  lk.use(st);
  const double* dtol = cfg->tolerances;
  if (!dtol) {
    std::vector<double> tv(batch, cfg->tolerance);
    void* p;
    if (int s = copy_in(ctx, S_TOL, tv.data(), batch * 8, &p, st)) return s;
    CU(cudaStreamSynchronize(st));
    dtol = (const double*)p;
  }
  return cosamp_dev_locked(op, dtype, y, batch, k, cfg, dtol, out, st);
}

int fmp_cosamp_solve(fmp_op op, int dtype, const void* y, uint64_t batch, uint64_t k,
                     const fmp_omp_config* cfg, fmp_cosamp_result* out) {
  if (int s = cosamp_validate(op, dtype, k, cfg)) return s;
  if (!y || !out || !out->support || !out->coeffs || !out->support_size || !out->iterations ||
      !out->residual || !out->aborted)
    return fail(FMP_EINVAL, "null buffer");
  if (cfg->record_correlations && !out->history)
    return fail(FMP_EINVAL, "record_correlations needs a history buffer");
  if (cfg->tolerances)
    for (uint64_t b = 0; b < batch; ++b)
      if (!(cfg->tolerances[b] >= 0.0)) return fail(FMP_EINVAL, "cosamp_solve: tolerance must be >= 0");
  fmp_ctx_s* ctx = op->ctx;
  CU(cudaSetDevice(ctx->device));
  CtxLock lk(ctx);
  cudaStream_t st = ctx->cur;
  lk.use(st);
  const uint64_t T = cfg->max_iterations, n = (uint64_t)op->d.n, m = (uint64_t)op->d.m;
  const uint64_t kk = std::max<uint64_t>(k, 1);
  const size_t eb = fmp::elem_bytes(dtype);
  // large batches with page-locked results: one launch fed by per-chunk
  // ready flags, results stored straight into the caller's buffers (as
  // omp_host_streamed)
  const uint64_t grid = (uint64_t)fmp::omp_grid(op->d, dtype, (int64_t)batch, (int64_t)T);
  if (k && !cfg->record_correlations && !g_phase_prof && batch >= 8 * grid &&
      host_pinned(out->support) && host_pinned(out->coeffs) && host_pinned(out->support_size) &&
      host_pinned(out->iterations) && host_pinned(out->residual) && host_pinned(out->aborted) &&
      (!out->support_history || host_pinned(out->support_history))) {
    void *dy, *dtol;
    int* flags;
    const uint64_t per = grid, nchunk = (batch + per - 1) / per;
    if (int e = stream_in_setup(ctx, y, batch, m * eb, cfg, nchunk, &dy, &dtol, &flags, st)) return e;
    if (int e = cosamp_dev_locked(op, dtype, dy, batch, k, cfg, (const double*)dtol, out, st, flags,
                                  (int64_t)per)) {
      *(volatile int*)ctx->abort_host = 1;
      cudaStreamSynchronize(st);
      return e;
    }
    return stream_in_finish(ctx, y, batch, m * eb, per, dy, flags, st, out->aborted);
  }
  void* dy;
  if (int s = copy_in(ctx, S_IN, y, batch * m * eb, &dy, st)) return s;
  std::vector<double> tv;
  if (!cfg->tolerances) tv.assign(batch, cfg->tolerance);
  void* dtol;
  if (int s = copy_in(ctx, S_TOL, cfg->tolerances ? cfg->tolerances : tv.data(), batch * 8, &dtol, st))
    return s;
  fmp_cosamp_result d{};
  ALLOC(d.support, S_OSUP, batch * kk * 8);
  ALLOC(d.coeffs, S_OCO, batch * kk * 16);
  ALLOC(d.support_size, S_OSZ, batch * 8);
  ALLOC(d.iterations, S_OIT, batch * 8);
  ALLOC(d.residual, S_ORES, batch * 8);
  ALLOC(d.aborted, S_OAB, batch * 4);
  if (out->support_history) ALLOC(d.support_history, S_OHSUP, batch * T * kk * 8);
  if (cfg->record_correlations) ALLOC(d.history, S_OHIST, batch * T * n * eb);
  if (int s = cosamp_dev_locked(op, dtype, dy, batch, k, cfg, (const double*)dtol, &d, st)) return s;
  if (k) {
    CU(cudaMemcpyAsync(out->support, d.support, batch * k * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(out->coeffs, d.coeffs, batch * k * 16, cudaMemcpyDeviceToHost, st));
    if (out->support_history)
      CU(cudaMemcpyAsync(out->support_history, d.support_history, batch * T * k * 8,
                         cudaMemcpyDeviceToHost, st));
  }
  CU(cudaMemcpyAsync(out->support_size, d.support_size, batch * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(out->iterations, d.iterations, batch * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(out->residual, d.residual, batch * 8, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(out->aborted, d.aborted, batch * 4, cudaMemcpyDeviceToHost, st));
  if (cfg->record_correlations)
    CU(cudaMemcpyAsync(out->history, d.history, batch * T * n * eb, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  return FMP_OK;
}

}  // extern "C"

// ============================================================ IncrementalQR
struct fmp_qr_s {
  fmp_ctx_s* ctx = nullptr;
  int64_t rows = 0;
  int t = 0, cap = 0;
  double2 *Q = nullptr, *v = nullptr, *part = nullptr, *s = nullptr, *acc = nullptr;
  double *npart = nullptr, *dval = nullptr;
  std::vector<std::vector<std::complex<double>>> R;  // column j: R(0..j, j)
};

namespace {
void qr_free(fmp_qr_s* q) {
  for (void* p : {(void*)q->Q, (void*)q->v, (void*)q->part, (void*)q->s, (void*)q->acc,
                  (void*)q->npart, (void*)q->dval})
    if (p) cudaFree(p);
}

int qr_reserve(fmp_qr_s* q, int cap) {
  if (cap <= q->cap) return FMP_OK;
  const int nc = std::max(cap, 2 * q->cap);
  const int nb = fmp::qr_dot_blocks(q->rows);
  double2 *Q2 = nullptr, *p2 = nullptr, *s2 = nullptr, *a2 = nullptr;
  cudaError_t e;
  if ((e = cudaMalloc(&Q2, (size_t)nc * q->rows * 16)) != cudaSuccess ||
      (e = cudaMalloc(&p2, (size_t)nc * nb * 16)) != cudaSuccess ||
      (e = cudaMalloc(&s2, (size_t)nc * 16)) != cudaSuccess ||
      (e = cudaMalloc(&a2, (size_t)nc * 16)) != cudaSuccess) {
    for (void* p : {(void*)Q2, (void*)p2, (void*)s2, (void*)a2}) if (p) cudaFree(p);
    return fail(FMP_ENOMEM, "qr capacity %d: %s", nc, cudaGetErrorString(e));
  }
  if (q->t) CU(cudaMemcpyAsync(Q2, q->Q, (size_t)q->t * q->rows * 16, cudaMemcpyDeviceToDevice, q->ctx->cur));
  CU(cudaStreamSynchronize(q->ctx->cur));
  for (void* p : {(void*)q->Q, (void*)q->part, (void*)q->s, (void*)q->acc}) if (p) cudaFree(p);
  q->Q = Q2;
  q->part = p2;
  q->s = s2;
  q->acc = a2;
  q->cap = nc;
  return FMP_OK;
}
}  // namespace

extern "C" {

int fmp_qr_create(fmp_ctx ctx, uint64_t rows, uint64_t capacity, fmp_qr* out) {
  if (!ctx || !out) return fail(FMP_EINVAL, "null argument");
  if (rows == 0) return fail(FMP_EINVAL, "qr: rows must be positive");
  CU(cudaSetDevice(ctx->device));
  fmp_qr_s* q = new fmp_qr_s;
  q->ctx = ctx;
  q->rows = (int64_t)rows;
  cudaError_t e;
  if ((e = cudaMalloc(&q->v, rows * 16)) != cudaSuccess ||
      (e = cudaMalloc(&q->npart, 4096 * 8)) != cudaSuccess ||  // >= the norm kernel grid
      (e = cudaMalloc(&q->dval, 64)) != cudaSuccess) {
    qr_free(q);
    delete q;
    return fail(FMP_ENOMEM, "qr: %s", cudaGetErrorString(e));
  }
  if (int st = qr_reserve(q, (int)std::max<uint64_t>(capacity, 8))) {
    qr_free(q);
    delete q;
    return st;
  }
  *out = q;
  return FMP_OK;
}

int fmp_qr_destroy(fmp_qr q) {
  if (!q) return FMP_OK;
  cudaSetDevice(q->ctx->device);
  cudaStreamSynchronize(q->ctx->cur);
  qr_free(q);
  delete q;
  return FMP_OK;
}

uint64_t fmp_qr_cols(fmp_qr q) { return q ? (uint64_t)q->t : 0; }

// solvers.cpp:222-251
int fmp_qr_push_column(fmp_qr q, const double* col, int* accepted) {
  if (!q || !col || !accepted) return fail(FMP_EINVAL, "null argument");
  CU(cudaSetDevice(q->ctx->device));
  CtxLock lk(q->ctx);
  cudaStream_t st = q->ctx->cur;
  lk.use(st);
  double o2 = 0.0;  // l2_norm(col) in the reference's order (types.cpp:32-36)
  for (int64_t i = 0; i < 2 * q->rows; ++i) o2 += col[i] * col[i];
  const double orig = std::sqrt(o2);
  if (int e = qr_reserve(q, q->t + 1)) return e;
  CU(cudaMemcpyAsync(q->v, col, (size_t)q->rows * 16, cudaMemcpyHostToDevice, st));
  CU(cudaMemsetAsync(q->acc, 0, (size_t)std::max(q->t, 1) * 16, st));
  for (int pass = 0; pass < 2; ++pass)  // the second mops up the first's rounding
    CU(fmp::launch_qr_project(q->Q, q->rows, q->t, q->v, q->part, q->s, q->acc, st));
  CU(fmp::launch_qr_norm(q->v, q->rows, q->npart, q->dval, st));
  std::vector<std::complex<double>> rcol((size_t)q->t + 1);
  double r2 = 0.0;
  if (q->t) CU(cudaMemcpyAsync(rcol.data(), q->acc, (size_t)q->t * 16, cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(&r2, q->dval, 8, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  const double rho = std::sqrt(r2);
  if (rho <= 1e-10 * orig) {  // nothing left outside the span
    *accepted = 0;
    return FMP_OK;
  }
  rcol[(size_t)q->t] = rho;
  CU(fmp::launch_qr_store(q->Q + (size_t)q->t * q->rows, q->v, q->rows, 1.0 / rho, st));
  q->R.push_back(std::move(rcol));
  q->t += 1;
  *accepted = 1;
  return FMP_OK;
}

// solvers.cpp:253-274: z = Q^H rhs on the device, back substitution on the host
int fmp_qr_solve(fmp_qr q, const double* rhs, double* x_out) {
  if (!q || !rhs || (!x_out && q->t)) return fail(FMP_EINVAL, "null argument");
  CU(cudaSetDevice(q->ctx->device));
  CtxLock lk(q->ctx);
  cudaStream_t st = q->ctx->cur;
  lk.use(st);
  const int t = q->t;
  if (t == 0) return FMP_OK;
  CU(cudaMemcpyAsync(q->v, rhs, (size_t)q->rows * 16, cudaMemcpyHostToDevice, st));
  CU(fmp::launch_qr_dots(q->Q, q->rows, t, q->v, q->part, q->s, q->acc, st));
  std::vector<std::complex<double>> z((size_t)t), x((size_t)t);
  CU(cudaMemcpyAsync(z.data(), q->s, (size_t)t * 16, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  for (int jj = t; jj-- > 0;) {
    std::complex<double> v = z[(size_t)jj];
    for (int k = jj + 1; k < t; ++k) v -= q->R[(size_t)k][(size_t)jj] * x[(size_t)k];
    x[(size_t)jj] = v / q->R[(size_t)jj][(size_t)jj];
  }
  std::memcpy(x_out, x.data(), (size_t)t * 16);
  return FMP_OK;
}

}  // extern "C"

int fmp_make_batch_dev(fmp_op op, uint64_t k, double noise_stddev, int real, uint64_t base_seed,
                       uint64_t first, uint64_t batch, double* y_out, double* x_out,
                       double* noise_norm_out, uint64_t* fixups_out, void* stream) {
  if (!op || !y_out) return fail(FMP_EINVAL, "null argument");
  // make_instance's checks (sensing.cpp:121-124)
  if (k >= (uint64_t)op->d.m) return fail(FMP_EINVAL, "sparsity k must be below the row count m");
  if (!(noise_stddev >= 0.0)) return fail(FMP_EINVAL, "noise stddev must be non-negative");
  if (real && op->d.kind != FMP_HADAMARD) return fail(FMP_EINVAL, "real nonzeros need a Hadamard operator");
  if (batch == 0) return FMP_OK;
  CU(cudaSetDevice(op->ctx->device));
  std::lock_guard<std::mutex> lk(op->ctx->mu);
  CU(fmp::gen_batch(op->d, (int64_t)k, noise_stddev, real, base_seed, first, (int64_t)batch, y_out,
                    x_out, noise_norm_out, fixups_out, pick_stream(op->ctx, stream)));
  return FMP_OK;
}

int fmp_dd_eval(int fn, const double* x, uint64_t count, double* out, double* frac) {
  if (fn < 0 || fn > 2) return fail(FMP_EINVAL, "unknown function %d", fn);
  if (count && (!x || !out)) return fail(FMP_EINVAL, "null argument");
  fmp::dd_eval_host(fn, x, (int64_t)count, out, frac);
  return FMP_OK;
}

int fmp_dd_eval_dev(int fn, const double* x, uint64_t count, double* out, double* frac, void* stream) {
  if (fn < 0 || fn > 2) return fail(FMP_EINVAL, "unknown function %d", fn);
  if (count && (!x || !out || !frac)) return fail(FMP_EINVAL, "null argument");
  CU(fmp::dd_eval_dev(fn, x, (int64_t)count, out, frac, (cudaStream_t)stream));
  return FMP_OK;
}
