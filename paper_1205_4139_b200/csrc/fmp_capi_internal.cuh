// Internal declarations shared by the C-ABI translation units (fmp_capi.cu,
// fmp_large_host.cu): error reporting, per-context workspaces and locking,
// the operator handle, and the batched-transform helper.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "fmp.h"
#include "fmp_kernels.cuh"

using fmp::DevOp;

namespace fmpi {

extern thread_local std::string g_err;
extern int g_phase_prof;
extern thread_local int g_launch_count;

inline int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(expr)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (expr);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(e_ == cudaErrorMemoryAllocation ? FMP_ENOMEM : FMP_ECUDA,        \
                  "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

inline bool pow2(uint64_t n) { return n && !(n & (n - 1)); }
inline int ilog2(uint64_t n) {
  int p = 0;
  while (n >>= 1) ++p;
  return p;
}

// grow-only device scratch, one buffer per slot
struct Workspace {
  std::vector<std::pair<void*, size_t>> slot;
  void* get(int i, size_t bytes, cudaError_t* err) {
    if ((int)slot.size() <= i) slot.resize(i + 1, {nullptr, 0});
    bytes = std::max<size_t>(bytes, 256);
    if (slot[i].second < bytes) {
      if (slot[i].first) cudaFree(slot[i].first);
      slot[i] = {nullptr, 0};
      void* p = nullptr;
      *err = cudaMalloc(&p, bytes);
      if (*err != cudaSuccess) return nullptr;
      slot[i] = {p, bytes};
    }
    return slot[i].first;
  }
  ~Workspace() {
    for (auto& s : slot)
      if (s.first) cudaFree(s.first);
  }
};

enum Slot { S_IN, S_OUT, S_AUX, S_SUP, S_CO, S_WORK, S_MAG, S_W, S_H0, S_R, S_Q, S_TOL,
            S_OSUP, S_OCO, S_OSZ, S_OIT, S_ORES, S_OAB, S_OMOD, S_OHL, S_OHIST, S_IDX, S_BUF, S_PH, S_SYNC,
            S_OHSUP, S_Y64, S_H0X, S_GOFF, S_RST, S_YS,
            S_ALT = 64 };  // S_ALT + slot: the alternate per-CTA workspace set

}  // namespace fmpi

struct fmp_ctx_s {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t cur = nullptr;
  cudaStream_t copy = nullptr;        // host<->device copies overlapped with solves (lazy)
  cudaStream_t alt = nullptr;         // second compute stream (lazy)
  void* pinned = nullptr;             // page-locked staging for pageable host buffers (lazy)
  size_t pinned_bytes = 0;
  std::vector<cudaEvent_t> events;    // chunk hand-offs between the two streams (lazy)
  // abort word of the streamed-input paths: page-locked, mapped into the
  // device address space; the host raises it on an error path so a kernel
  // spinning on ready flags returns without any further CUDA call (lazy)
  int* abort_host = nullptr;
  const volatile int* abort_dev = nullptr;
  // the workspaces are one set per context: a call on another stream waits
  // for the last call that used them (ws_done, recorded on ws_stream)
  cudaEvent_t ws_done = nullptr;
  cudaStream_t ws_stream = nullptr;
  bool ws_pending = false;
  fmpi::Workspace ws;
  std::mutex mu;
};

// The context mutex plus workspace ordering: the grow-only workspaces are
// one set per context, so a call that enqueues work on stream st first waits
// for the previous call's work if that went to another stream (use), and
// marks the end of its own on destruction.  Calls on one stream are ordered
// by the stream itself.
struct CtxLock {
  fmp_ctx_s* c;
  std::lock_guard<std::mutex> lk;
  cudaStream_t st = nullptr;
  bool used = false;
  explicit CtxLock(fmp_ctx_s* ctx) : c(ctx), lk(ctx->mu) {}
  void use(cudaStream_t s) {
    if (c->ws_pending && c->ws_stream != s) cudaStreamWaitEvent(s, c->ws_done, 0);
    st = s;
    used = true;
  }
  ~CtxLock() {
    if (!used) return;
    if (!c->ws_done && cudaEventCreateWithFlags(&c->ws_done, cudaEventDisableTiming) != cudaSuccess) return;
    if (cudaEventRecord(c->ws_done, st) == cudaSuccess) {
      c->ws_stream = st;
      c->ws_pending = true;
    }
  }
};

struct fmp_op_s {
  fmp_ctx_s* ctx = nullptr;
  DevOp d;
  std::vector<uint64_t> rows;  // sorted, 1-based
};

namespace fmpi {

#define ALLOC(var, slot, bytes)                                       \
  do {                                                                \
    cudaError_t e_ = cudaSuccess;                                     \
    var = (std::remove_reference_t<decltype(var)>)ctx->ws.get(slot, (bytes), &e_);             \
    if (!var) return fail(FMP_ENOMEM, "device workspace (%zu bytes): %s", \
                          (size_t)(bytes), cudaGetErrorString(e_));   \
  } while (0)

inline int check_dtype(const DevOp& d, int dtype) {
  if (dtype < 0 || dtype > 3) return fail(FMP_EINVAL, "unknown dtype %d", dtype);
  if (d.kind == fmp::FOURIER && !fmp::is_complex(dtype))
    return fail(FMP_EINVAL, "real dtypes need a Hadamard operator");
  return FMP_OK;
}

inline cudaStream_t pick_stream(fmp_ctx_s* ctx, void* s) {
  return s ? (cudaStream_t)s : ctx->cur;
}

// batched transform on device pointers
inline int run_transform(fmp_op_s* op, int dtype, int inverse, int in_omega, int out_omega,
                         const void* in, void* out, uint64_t batch, uint64_t* amax, cudaStream_t st,
                         int slot_off = 0) {
  fmp_ctx_s* ctx = op->ctx;
  fmp::TransformArgs a{};
  a.op = &op->d;
  a.dtype = dtype;
  a.inverse = inverse;
  a.in_omega = in_omega;
  a.out_omega = out_omega;
  a.in = in;
  a.out = out;
  a.batch = (int64_t)batch;
  a.argmax_out = amax;
  if (op->d.n > fmp::transform_max_n(dtype)) {
    void* w;
    ALLOC(w, slot_off + S_WORK, (size_t)batch * op->d.n * fmp::elem_bytes(dtype));
    a.work = w;
    int* sy;
    ALLOC(sy, slot_off + S_SYNC, (32 + batch) * sizeof(int));
    a.sync = sy;
  }
  CU(fmp::launch_transform(a, st));
  g_launch_count = fmp::last_launch_count();
  return FMP_OK;
}

inline int copy_in(fmp_ctx_s* ctx, int slot, const void* host, size_t bytes, void** dev, cudaStream_t st) {
  ALLOC(*dev, slot, bytes);
  CU(cudaMemcpyAsync(*dev, host, bytes, cudaMemcpyHostToDevice, st));
  return FMP_OK;
}

}  // namespace fmpi
