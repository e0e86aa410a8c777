// C ABI of the sharded single-signal solver (include/fmp.h, fmp_large_*;
// kernels in fmp_large.cu): one signal, N up to 2^28, shard p of P owning
// the correlation entries k = p + P k'.  The host drives the local shards in
// lockstep — omp_solve's loop (solvers.cpp:296-411) with the correlation of
// iteration t + 1 enqueued before the host waits for iteration t's
// decisions — and the shards exchange on the device: NCCL collectives
// (libnccl.so.2, loaded at first use) or, for shards of one process on one
// GPU, copies and fixed-order reductions.
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <limits>
#include <memory>

#include "fmp_capi_internal.cuh"

using namespace fmpi;

namespace {

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi* nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the process's NCCL if one is loaded already (torch's), else the system one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = dlerror();
      return;
    }
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      return f != nullptr;
    };
    api.ok = sym(api.GetUniqueId, "ncclGetUniqueId") && sym(api.CommInitRank, "ncclCommInitRank") &&
             sym(api.CommInitAll, "ncclCommInitAll") && sym(api.CommDestroy, "ncclCommDestroy") &&
             sym(api.AllGather, "ncclAllGather") && sym(api.AllReduce, "ncclAllReduce") &&
             sym(api.GroupStart, "ncclGroupStart") && sym(api.GroupEnd, "ncclGroupEnd") &&
             sym(api.GetErrorString, "ncclGetErrorString");
    if (!api.ok) api.why = "libnccl.so.2 lacks a symbol";
  });
  return &api;
}

#define NC(expr)                                                                        \
  do {                                                                                  \
    ncclResult_t r_ = (expr);                                                           \
    if (r_ != ncclSuccess)                                                              \
      return fail(FMP_ENCCL, "%s: %s (%s:%d)", #expr, nccl()->GetErrorString(r_), __FILE__, \
                  __LINE__);                                                            \
  } while (0)

}  // namespace

struct fmp_comm_s {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0, device = 0;
};

struct fmp_large_s {
  fmp_op_s* op = nullptr;
  fmp_op_s* opn = nullptr;  // np-point transform operator (P > 1)
  fmp_comm_s* comm = nullptr;
  int dtype = FMP_C64;
  int P = 1, p = 0;
  int64_t n = 0, m = 0, np = 0;
  int T = 1;
  int64_t fast_until = 0;
  double ecoef = 0.0;
  fmp::LgShard S{};
  std::vector<void*> allocs;
  void* X = nullptr;       // np (dtype): forward transform of this shard's atoms (P > 1)
  void* X64 = nullptr;     // np (c128)
  void* xd = nullptr;      // dense scatter of the atoms when the transform takes no sparse input
  void* ax64 = nullptr;    // m (c128): Phi x at Omega, or this shard's part of it
  void* axsum64 = nullptr; // m (c128): the sum over shards
  void* y64own = nullptr;  // m (c128): widened fp32 measurements
  void** dptrs = nullptr;  // emulated exchange: the shards' partial pointers (device)
  double* stage = nullptr; // emulated exchange: P scalars
  struct Dec {
    fmp::LgPick pick;
    double scal[11];
    uint32_t count;
  }* dec = nullptr;        // page-locked mirror of the decisions
  cudaEvent_t ev = nullptr;
  // host state (omp_solve's loop variables, solvers.cpp:306-403)
  int t = 0, s = 0, iters = 0, aborted = 0;
  double yy = 0, tol = 0, rn = 0;
  std::vector<uint64_t> support;
};

namespace {

cudaStream_t st_of(fmp_large_s* lg) { return lg->op->ctx->cur; }

int lg_alloc(fmp_large_s* lg, void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, std::max<size_t>(bytes, 256));
  if (e != cudaSuccess)
    return fail(FMP_ENOMEM, "large solver alloc (%zu bytes): %s", bytes, cudaGetErrorString(e));
  lg->allocs.push_back(*p);
  return FMP_OK;
}

void lg_free(fmp_large_s* lg) {
  cudaSetDevice(lg->op->ctx->device);
  cudaStreamSynchronize(st_of(lg));
  for (void* p : lg->allocs) cudaFree(p);
  lg->allocs.clear();
  if (lg->dec) cudaFreeHost(lg->dec);
  if (lg->ev) cudaEventDestroy(lg->ev);
  if (lg->opn) fmp_operator_destroy(lg->opn);
  delete lg;
}

// ------------------------------------------------------------- exchanges
using Group = std::vector<fmp_large_s*>;  // local shards, indexed by shard p when emulated

bool use_nccl(const Group& g) { return g[0]->comm != nullptr; }

int ex_gather(const Group& g) {
  if (g[0]->P == 1) return FMP_OK;  // rec_all aliases rec_send
  if (use_nccl(g)) {
    NC(nccl()->GroupStart());
    for (auto* lg : g)
      NC(nccl()->AllGather(lg->S.rec_send, lg->S.rec_all, sizeof(fmp::LgRec), ncclUint8, lg->comm->comm,
                           st_of(lg)));
    NC(nccl()->GroupEnd());
    return FMP_OK;
  }
  cudaStream_t st = st_of(g[0]);
  for (auto* dst : g)
    for (auto* src : g)
      CU(cudaMemcpyAsync(dst->S.rec_all + src->p, src->S.rec_send, sizeof(fmp::LgRec),
                         cudaMemcpyDeviceToDevice, st));
  return FMP_OK;
}

// sum over shards of an m-vector (dtype rdt): src -> dst on every shard
int ex_sum(const Group& g, int rdt, void* (*src)(fmp_large_s*), void* (*dst)(fmp_large_s*)) {
  const int64_t m = g[0]->m;
  if (use_nccl(g)) {
    NC(nccl()->GroupStart());
    for (auto* lg : g)
      NC(nccl()->AllReduce(src(lg), dst(lg), (size_t)(2 * m), rdt == FMP_C128 ? ncclFloat64 : ncclFloat32,
                           ncclSum, lg->comm->comm, st_of(lg)));
    NC(nccl()->GroupEnd());
    return FMP_OK;
  }
  cudaStream_t st = st_of(g[0]);
  std::vector<void*> ptrs(g.size());
  for (auto* lg : g) ptrs[lg->p] = src(lg);
  fmp_large_s* h = g[0];
  CU(cudaMemcpyAsync(h->dptrs, ptrs.data(), ptrs.size() * sizeof(void*), cudaMemcpyHostToDevice, st));
  CU(fmp::lg_sum_partials(rdt, (const void* const*)h->dptrs, (int)g.size(), dst(h), m, st));
  for (auto* lg : g)
    if (lg != h) CU(cudaMemcpyAsync(dst(lg), dst(h), (size_t)m * fmp::elem_bytes(rdt), cudaMemcpyDeviceToDevice, st));
  CU(cudaStreamSynchronize(st));  // (the host pointer array is stack memory)
  return FMP_OK;
}

// fallback scalars: max of fb[0] -> fb[1]; min of u64 fb[2] -> fb[3]
int ex_fb(const Group& g, bool first) {
  if (use_nccl(g)) {
    NC(nccl()->GroupStart());
    for (auto* lg : g) {
      if (!first)
        NC(nccl()->AllReduce(lg->S.fb, lg->S.fb + 1, 1, ncclFloat64, ncclMax, lg->comm->comm, st_of(lg)));
      else
        NC(nccl()->AllReduce(lg->S.fb + 2, lg->S.fb + 3, 1, ncclUint64, ncclMin, lg->comm->comm, st_of(lg)));
    }
    NC(nccl()->GroupEnd());
    return FMP_OK;
  }
  cudaStream_t st = st_of(g[0]);
  fmp_large_s* h = g[0];
  const int k = first ? 2 : 0;
  for (auto* lg : g) CU(cudaMemcpyAsync(h->stage + lg->p, lg->S.fb + k, 8, cudaMemcpyDeviceToDevice, st));
  if (first) CU(fmp::lg_reduce_u64_min((const unsigned long long*)h->stage, (int)g.size(),
                                       (unsigned long long*)(h->S.fb + 3), st));
  else CU(fmp::lg_reduce_f64(h->stage, (int)g.size(), 1, h->S.fb + 1, st));
  for (auto* lg : g)
    if (lg != h) CU(cudaMemcpyAsync(lg->S.fb + k + 1, h->S.fb + k + 1, 8, cudaMemcpyDeviceToDevice, st));
  return FMP_OK;
}

// ----------------------------------------------------------- solver steps
// Phi x at Omega for the first cnt atoms, summed over shards, then r = y -
// Phi x and ||r||^2 into scal[9]; rdt C128 for fp32 data gives the fp64 norm
// (r itself stays in the working precision)
int residual(const Group& g, int rdt, int cnt) {
  const bool wide = rdt != g[0]->dtype;
  for (auto* lg : g) {
    cudaStream_t st = st_of(lg);
    fmp_ctx_s* ctx = lg->op->ctx;
    const size_t eb = (size_t)fmp::elem_bytes(rdt);
    void* out = wide ? lg->ax64 : lg->S.ax;
    CU(fmp::lg_class_positions(lg->S, cnt, st));
    fmp_op_s* top = lg->P == 1 ? lg->op : lg->opn;
    void* X = lg->P == 1 ? out : (wide ? lg->X64 : lg->X);
    if (top->d.fs_l1) {
      void* w;
      ALLOC(w, S_WORK, (size_t)top->d.n * eb);
      fmp::FsTransform t{};
      t.op = &top->d;
      t.dtype = rdt;
      t.inverse = 0;
      t.in_mode = 2;
      t.lam = lg->S.lamc;
      t.xs = lg->S.x;
      t.cnt = cnt;
      t.mid = w;
      t.out_mode = lg->P == 1 ? 1 : 0;
      t.out = X;
      t.batch = 1;
      CU(fmp::launch_transform_fs(t, st));
    } else {
      CU(fmp::lg_scatter_dense(lg->S, rdt, lg->xd, top->d.n, cnt, st));
      if (int e = run_transform(top, rdt, 0, 0, lg->P == 1 ? 1 : 0, lg->xd, X, 1, nullptr, st)) return e;
    }
    if (lg->P > 1) CU(fmp::lg_partial(lg->S, rdt, X, out, st));
  }
  if (g[0]->P > 1) {
    if (wide) {
      if (int e = ex_sum(g, rdt, [](fmp_large_s* l) { return l->ax64; }, [](fmp_large_s* l) { return l->axsum64; }))
        return e;
    } else {
      if (int e = ex_sum(g, rdt, [](fmp_large_s* l) { return l->S.ax; }, [](fmp_large_s* l) { return l->S.axsum; }))
        return e;
    }
  }
  for (auto* lg : g) {
    const void* ax = lg->P == 1 ? (wide ? lg->ax64 : lg->S.ax) : (wide ? lg->axsum64 : lg->S.axsum);
    CU(fmp::lg_resid(lg->S, rdt, ax, st_of(lg)));
  }
  return FMP_OK;
}

// correlation row t (s atoms in the estimate) and its identification record
int correlate(const Group& g, int t, int s, int prev) {
  for (auto* lg : g) {
    cudaStream_t st = st_of(lg);
    const void* h = lg->S.hs;
    if (t == 1) {
      h = lg->S.h0s;
      CU(fmp::lg_max(lg->S, h, st));
    } else if ((int64_t)t <= lg->fast_until) {
      CU(fmp::lg_fast(lg->S, s, st));
    } else {
      // conventional row: the adjoint transform of the residual (sensing.cpp:102-109)
      if (lg->P == 1) {
        if (int e = run_transform(lg->op, lg->dtype, 1, 1, 0, lg->S.r, lg->S.hs, 1, nullptr, st)) return e;
      } else {
        CU(fmp::lg_fold(lg->S, st));
        if (int e = run_transform(lg->opn, lg->dtype, 1, 0, 0, lg->S.fold, lg->S.hs, 1, nullptr, st)) return e;
      }
      CU(fmp::lg_max(lg->S, h, st));
    }
    CU(fmp::lg_identify(lg->S, h, s, lg->ecoef, prev, st));
  }
  return ex_gather(g);
}

int merge(const Group& g, int cur, int prev) {
  for (auto* lg : g) CU(fmp::lg_merge(lg->S, cur, prev, st_of(lg)));
  return FMP_OK;
}

// exact pick after an overflowing record (every candidate of every shard)
int fallback(const Group& g, int cur) {
  for (auto* lg : g) CU(fmp::lg_fb_local_best(lg->S, st_of(lg)));
  if (int e = ex_fb(g, false)) return e;
  for (auto* lg : g) CU(fmp::lg_fb_local_first(lg->S, st_of(lg)));
  if (int e = ex_fb(g, true)) return e;
  for (auto* lg : g) CU(fmp::lg_fb_pick(lg->S, cur, st_of(lg)));
  return FMP_OK;
}

int decisions(const Group& g, int cur) {
  for (auto* lg : g) {
    cudaStream_t st = st_of(lg);
    CU(cudaMemcpyAsync(&lg->dec->pick, lg->S.pick + cur, sizeof(fmp::LgPick), cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(lg->dec->scal, lg->S.scal, 11 * 8, cudaMemcpyDeviceToHost, st));
    CU(cudaMemcpyAsync(&lg->dec->count, lg->S.ccount, 4, cudaMemcpyDeviceToHost, st));
    CU(cudaEventRecord(lg->ev, st));
  }
  return FMP_OK;
}

int wait_decisions(const Group& g) {
  for (auto* lg : g) CU(cudaEventSynchronize(lg->ev));
  return FMP_OK;
}

int final_residual(const Group& g) {
  if (int e = residual(g, FMP_C128, g[0]->s)) return e;
  for (auto* lg : g) CU(cudaMemcpyAsync(lg->dec->scal + 9, lg->S.scal + 9, 8, cudaMemcpyDeviceToHost, st_of(lg)));
  for (auto* lg : g) CU(cudaStreamSynchronize(st_of(lg)));
  for (auto* lg : g) lg->rn = std::sqrt(lg->dec->scal[9]);
  return FMP_OK;
}

int setup(fmp_large_s* lg, const void* y, double tol) {
  cudaStream_t st = st_of(lg);
  fmp::LgShard& S = lg->S;
  const size_t eb = (size_t)fmp::elem_bytes(lg->dtype);
  CU(cudaMemcpyAsync((void*)S.y, y, (size_t)lg->m * eb, cudaMemcpyHostToDevice, st));
  if (lg->dtype == FMP_C64) CU(fmp::launch_widen((const float*)S.y, (double*)lg->y64own, 2 * lg->m, st));
  CU(cudaMemsetAsync(S.scal, 0, 16 * 8, st));
  CU(cudaMemsetAsync(S.selbits, 0, (size_t)(lg->n + 31) / 32 * 4, st));
  // fp64 h0 = Phi^H y over all n (replicated), this shard's class narrowed
  if (int e = run_transform(lg->op, FMP_C128, 1, 1, 0, S.y64, (void*)S.h0x, 1, nullptr, st)) return e;
  CU(fmp::lg_take_narrow(S, st));
  // ||y||^2 in fp64, in the order one thread sums (types.cpp:32-36)
  double yy = 0.0;
  if (lg->dtype == FMP_C128) {
    const double* v = (const double*)y;
    for (int64_t i = 0; i < 2 * lg->m; ++i) yy += v[i] * v[i];
  } else {
    const float* v = (const float*)y;
    for (int64_t i = 0; i < 2 * lg->m; ++i) yy += (double)v[i] * v[i];
  }
  double sc[11] = {};
  sc[0] = (double)lg->m / (double)lg->n;  // gamma = c(1) = M / N
  sc[1] = yy;
  sc[10] = std::sqrt((double)lg->m / (double)lg->n * yy);  // |h0_j| <= sqrt(M/N) ||y||
  CU(cudaMemcpyAsync(S.scal, sc, sizeof(sc), cudaMemcpyHostToDevice, st));
  CU(cudaStreamSynchronize(st));  // (sc is stack memory)
  lg->yy = yy;
  lg->tol = tol;
  lg->rn = std::sqrt(yy);
  lg->t = lg->s = lg->iters = lg->aborted = 0;
  lg->support.clear();
  return FMP_OK;
}

int group_solve(Group g, const void* y, double tol) {
  const int P = g[0]->P;
  // (emulated shards: all P, in shard order, on one context)
  if (!use_nccl(g)) {
    if ((int)g.size() != P) return fail(FMP_EINVAL, "without communicators every shard must be passed");
    std::sort(g.begin(), g.end(), [](fmp_large_s* a, fmp_large_s* b) { return a->p < b->p; });
    for (int i = 0; i < P; ++i) {
      if (g[i]->p != i) return fail(FMP_EINVAL, "duplicate shard %d", g[i]->p);
      if (g[i]->op->ctx != g[0]->op->ctx)
        return fail(FMP_EINVAL, "emulated shards must share one context");
    }
  }
  for (auto* lg : g) {
    if (lg->P != P || lg->T != g[0]->T || lg->dtype != g[0]->dtype || (lg->comm == nullptr) != !use_nccl(g))
      return fail(FMP_EINVAL, "shards of different solves in one group");
    CU(cudaSetDevice(lg->op->ctx->device));
    if (int e = setup(lg, y, tol)) return e;
  }
  fmp_large_s* h = g[0];
  const int T = h->T;
  auto all = [&](auto f) { for (auto* lg : g) f(lg); };
  if (h->rn <= tol) return FMP_OK;  // solvers.cpp:327-331
  // iteration 1 identification (pick[1])
  if (int e = correlate(g, 1, 0, -1)) return e;
  if (int e = merge(g, 1, -1)) return e;
  int t = 1, s = 0;
  bool explicit_rn = false;
  for (;;) {
    const int cur = t & 1;
    for (auto* lg : g) CU(fmp::lg_ls(lg->S, s, cur, st_of(lg)));
    const bool next_conv = t < T && !((int64_t)(t + 1) <= h->fast_until);
    if (next_conv)
      if (int e = residual(g, h->dtype, s + 1)) return e;
    if (int e = decisions(g, cur)) return e;
    // the next correlation and its pick, before waiting on this iteration
    if (t < T) {
      if (int e = correlate(g, t + 1, s + 1, cur)) return e;
      if (int e = merge(g, cur ^ 1, cur)) return e;
    }
    if (int e = wait_decisions(g)) return e;
    const auto& d = *h->dec;
    const int flags = d.pick.flags;
    if (flags & fmp::LG_TOOMANY)
      return fail(FMP_EUNSUPPORTED, "more than %d correlations within the rounding bound of the maximum",
                  fmp::LG_LCAP);
    if (flags & fmp::LG_OVERFLOW) {
      // exact pick from every candidate of iteration t (kept: the speculative
      // identification skipped itself on the flag), then redo iteration t
      if (int e = fallback(g, cur)) return e;
      continue;
    }
    if (flags & (fmp::LG_ZERO | fmp::LG_STAGNANT)) break;  // solvers.cpp:363-367
    if (d.scal[6] != 0.0) {                                 // rank deficient (solvers.cpp:380-385)
      all([](fmp_large_s* lg) { lg->aborted = 1; });
      break;
    }
    ++s;
    all([&](fmp_large_s* lg) {
      lg->s = s;
      lg->support.push_back(d.pick.j);
      lg->iters = t;
    });
    // residual and halting (solvers.cpp:388-402): the fp64 identity
    // ||y||^2 - ||z||^2 (b is fp64 h0, LS in fp64) unless it is within
    // 1e-10 ||y||^2 of tol^2, then the explicit fp64 residual
    const double r2id = h->yy - d.scal[2];
    bool halt;
    explicit_rn = false;
    if (std::fabs(r2id - tol * tol) <= 1e-10 * h->yy) {
      if (int e = final_residual(g)) return e;
      explicit_rn = true;
      halt = h->rn <= tol;
    } else {
      halt = r2id <= tol * tol;
    }
    if (halt || t >= T) break;
    ++t;
  }
  if (!explicit_rn)
    if (int e = final_residual(g)) return e;
  return FMP_OK;
}

}  // namespace

extern "C" {

int fmp_comm_unique_id(void* id128) {
  if (!id128) return fail(FMP_EINVAL, "null argument");
  NcclApi* api = nccl();
  if (!api->ok) return fail(FMP_ENCCL, "NCCL unavailable: %s", api->why.c_str());
  ncclUniqueId id;
  NC(api->GetUniqueId(&id));
  std::memcpy(id128, &id, sizeof(id));
  return FMP_OK;
}

int fmp_comm_init_rank(int device, int nranks, int rank, const void* id128, fmp_comm* out) {
  if (!id128 || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(FMP_EINVAL, "bad argument");
  NcclApi* api = nccl();
  if (!api->ok) return fail(FMP_ENCCL, "NCCL unavailable: %s", api->why.c_str());
  CU(cudaSetDevice(device));
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  auto* c = new fmp_comm_s;
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  ncclResult_t r = api->CommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(FMP_ENCCL, "ncclCommInitRank: %s", api->GetErrorString(r));
  }
  *out = c;
  return FMP_OK;
}

int fmp_comm_init_all(const int* devices, int n, fmp_comm* out) {
  if (!devices || !out || n < 1) return fail(FMP_EINVAL, "bad argument");
  NcclApi* api = nccl();
  if (!api->ok) return fail(FMP_ENCCL, "NCCL unavailable: %s", api->why.c_str());
  std::vector<ncclComm_t> comms(n);
  NC(api->CommInitAll(comms.data(), n, devices));
  for (int i = 0; i < n; ++i) {
    out[i] = new fmp_comm_s;
    out[i]->comm = comms[i];
    out[i]->nranks = n;
    out[i]->rank = i;
    out[i]->device = devices[i];
  }
  return FMP_OK;
}

int fmp_comm_destroy(fmp_comm c) {
  if (!c) return FMP_OK;
  if (c->comm && nccl()->ok) nccl()->CommDestroy(c->comm);
  delete c;
  return FMP_OK;
}

int fmp_large_create(fmp_op op, int dtype, uint64_t shard, uint64_t nshards, const fmp_omp_config* cfg,
                     fmp_comm comm, fmp_large* out) {
  if (!op || !cfg || !out) return fail(FMP_EINVAL, "null argument");
  if (op->d.kind != fmp::FOURIER)
    return fail(FMP_EUNSUPPORTED, "the sharded solver is implemented for Fourier operators");
  if (dtype != FMP_C64 && dtype != FMP_C128) return fail(FMP_EINVAL, "complex dtypes only");
  if (nshards < 1 || shard >= nshards || (nshards & (nshards - 1)) || (uint64_t)op->d.n % nshards ||
      (uint64_t)op->d.n / nshards < 64)
    return fail(FMP_EINVAL, "bad shard %llu of %llu (a power of two, n / nshards >= 64)",
                (unsigned long long)shard, (unsigned long long)nshards);
  if (cfg->max_iterations < 1) return fail(FMP_EINVAL, "omp_solve: max_iterations must be >= 1");
  if (cfg->max_iterations > 65536) return fail(FMP_EUNSUPPORTED, "max_iterations > 65536");
  if (comm && (comm->nranks != (int)nshards || comm->rank != (int)shard || comm->device != op->ctx->device))
    return fail(FMP_EINVAL, "communicator rank / size / device differ from the shard");
  fmp_ctx_s* ctx = op->ctx;
  CU(cudaSetDevice(ctx->device));
  auto* lg = new fmp_large_s;
  lg->op = op;
  lg->comm = comm;
  lg->dtype = dtype;
  lg->P = (int)nshards;
  lg->p = (int)shard;
  lg->n = op->d.n;
  lg->m = op->d.m;
  lg->np = lg->n / lg->P;
  lg->T = (int)cfg->max_iterations;
  switch (cfg->mode) {
    case FMP_MODE_CONVENTIONAL: lg->fast_until = 0; break;
    case FMP_MODE_FAST: lg->fast_until = std::numeric_limits<int64_t>::max(); break;
    case FMP_MODE_ADAPTIVE: lg->fast_until = (int64_t)fmp_crossover_iteration(FMP_FOURIER, (uint64_t)lg->n); break;
    case FMP_MODE_GPU: lg->fast_until = (int64_t)fmp_gpu_crossover(FMP_FOURIER, (uint64_t)lg->n); break;
    default: lg->fast_until = (int64_t)std::min<uint64_t>(cfg->fast_until, INT64_MAX);
  }
  // rounding bound of the working precision per transform level (cf. the
  // fused solver's REFINE path, fmp_omp_impl.cuh)
  lg->ecoef = 8.0 * (dtype == FMP_C64 ? 0x1p-24 : 0x1p-53) * (double)(op->d.log2n + 2);
  const size_t eb = (size_t)fmp::elem_bytes(dtype);
  const int grid = fmp::lg_grid();
  const int64_t n = lg->n, m = lg->m, np = lg->np, T = lg->T;
  int st = FMP_OK;
  auto A = [&](auto** p, size_t b) {
    void* v = nullptr;
    if (!st) st = lg_alloc(lg, &v, b);
    *p = reinterpret_cast<std::remove_reference_t<decltype(*p)>>(v);
  };
  fmp::LgShard& S = lg->S;
  S.op = op->d;
  S.dtype = dtype;
  S.P = lg->P;
  S.p = lg->p;
  S.log2P = ilog2((uint64_t)lg->P);
  S.T = lg->T;
  S.n = n;
  S.m = m;
  S.np = np;
  void *h0s, *hs, *h0x, *y, *r, *ax, *xn, *fold = nullptr, *axsum = nullptr;
  A(&h0s, np * eb);
  A(&hs, np * eb);
  A(&h0x, n * 16);
  A(&S.blkmax, ((size_t)grid + (size_t)(np + 127) / 128) * 8);
  A(&S.cand, (size_t)fmp::LG_LCAP * 4);
  A(&S.cval, (size_t)fmp::LG_LCAP * 8);
  A(&S.ccount, 64);
  A(&S.rec_send, sizeof(fmp::LgRec));
  A(&S.pick, 2 * sizeof(fmp::LgPick));
  A(&S.fb, 64);
  A(&S.W, (size_t)T * (T + 1) / 2 * 16);
  A(&S.x, (size_t)T * 16);
  A(&S.z, (size_t)T * 16);
  A(&S.l, (size_t)T * 16);
  A(&S.lam, (size_t)T * 4);
  A(&S.lamc, (size_t)T * 4);
  A(&xn, (size_t)T * eb);
  A(&S.part, (size_t)std::max<int64_t>(grid, (T + 7) / 8) * 3 * 8);
  A(&S.scal, 16 * 8);
  A(&S.selbits, (size_t)(n + 31) / 32 * 4);
  A(&y, m * eb);
  A(&r, m * eb);
  A(&ax, m * eb);
  A(&lg->ax64, m * 16);
  if (dtype == FMP_C64) A(&lg->y64own, m * 16);
  if (lg->P > 1) {
    A(&S.rec_all, (size_t)lg->P * sizeof(fmp::LgRec));
    A(&fold, np * eb);
    A(&axsum, m * eb);
    A(&lg->axsum64, m * 16);
    A(&lg->X, np * eb);
    A(&lg->X64, np * 16);
    A(&lg->dptrs, 64 * sizeof(void*));
    A(&lg->stage, 64 * 8);
  }
  if (st) {
    lg_free(lg);
    return st;
  }
  S.h0s = h0s;
  S.hs = hs;
  S.h0x = (const double2*)h0x;
  S.y = y;
  S.y64 = dtype == FMP_C64 ? (const double2*)lg->y64own : (const double2*)y;
  S.r = r;
  S.ax = ax;
  S.xn = xn;
  S.fold = fold;
  S.axsum = axsum;
  if (lg->P == 1) S.rec_all = S.rec_send;
  if (cudaHostAlloc((void**)&lg->dec, sizeof(fmp_large_s::Dec), cudaHostAllocDefault) != cudaSuccess ||
      cudaEventCreateWithFlags(&lg->ev, cudaEventDisableTiming) != cudaSuccess) {
    lg_free(lg);
    return fail(FMP_ENOMEM, "large solver: page-locked decision buffer / event");
  }
  cudaStream_t cs = ctx->cur;
  const void* g = dtype == FMP_C128 ? (const void*)op->d.g64 : (const void*)op->d.g32;
  if (lg->P > 1) {
    // the np-point transform operator (one row: only its transform plan is used)
    const uint64_t one = 1;
    fmp_op opn = nullptr;
    if (int e = fmp_operator_create(ctx, FMP_FOURIER, (uint64_t)np, &one, 1, &opn)) {
      lg_free(lg);
      return e;
    }
    lg->opn = opn;
    void* gcm = nullptr;
    if (!(st = lg_alloc(lg, &gcm, n * eb))) {
      cudaError_t e = fmp::lg_classmajor(dtype, g, gcm, n, lg->P, cs);
      if (e != cudaSuccess) st = fail(FMP_ECUDA, "class-major kernel: %s", cudaGetErrorString(e));
    }
    S.gcm = gcm;
    // rows by bin omega mod np (the fold of the residual), ascending row order per bin
    std::vector<uint32_t> off((size_t)np + 1, 0), rows_by_bin((size_t)m);
    for (int64_t i = 0; i < m; ++i) off[(op->rows[i] - 1) % np + 1]++;
    for (int64_t j = 0; j < np; ++j) off[j + 1] += off[j];
    std::vector<uint32_t> fill(off.begin(), off.end() - 1);
    for (int64_t i = 0; i < m; ++i) rows_by_bin[fill[(op->rows[i] - 1) % np]++] = (uint32_t)i;
    void *doff = nullptr, *drow = nullptr;
    if (!st) st = lg_alloc(lg, &doff, off.size() * 4);
    if (!st) st = lg_alloc(lg, &drow, (size_t)m * 4);
    if (!st && (cudaMemcpy(doff, off.data(), off.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
                cudaMemcpy(drow, rows_by_bin.data(), (size_t)m * 4, cudaMemcpyHostToDevice) != cudaSuccess))
      st = fail(FMP_ECUDA, "large solver: fold lists");
    S.bin_off = (const uint32_t*)doff;
    S.bin_row = (const uint32_t*)drow;
  } else {
    S.gcm = g;
  }
  fmp_op_s* top = lg->P == 1 ? op : lg->opn;
  if (!st && top && !top->d.fs_l1) st = lg_alloc(lg, &lg->xd, (size_t)top->d.n * 16);
  if (st) {
    lg_free(lg);
    return st;
  }
  *out = lg;
  return FMP_OK;
}

int fmp_large_destroy(fmp_large lg) {
  if (lg) lg_free(lg);
  return FMP_OK;
}

int fmp_large_group_solve(fmp_large* shards, int count, const void* y, double tol) {
  if (!shards || count < 1 || !y) return fail(FMP_EINVAL, "null argument");
  if (!(tol >= 0.0)) return fail(FMP_EINVAL, "omp_solve: tolerance must be >= 0");
  Group g(shards, shards + count);
  for (auto* lg : g)
    if (!lg) return fail(FMP_EINVAL, "null shard");
  // every local context locked for the solve (workspaces ordered on its stream)
  std::vector<std::unique_ptr<CtxLock>> locks;
  for (auto* lg : g) {
    bool seen = false;
    for (auto& l : locks) seen |= l->c == lg->op->ctx;
    if (seen) continue;
    CU(cudaSetDevice(lg->op->ctx->device));
    locks.emplace_back(new CtxLock(lg->op->ctx));
    locks.back()->use(lg->op->ctx->cur);
  }
  return group_solve(g, y, tol);
}

int fmp_large_result(fmp_large lg, uint64_t* support, double* coeffs, uint64_t* support_size,
                     uint64_t* iterations, double* residual, int32_t* aborted) {
  if (!lg) return fail(FMP_EINVAL, "null argument");
  CU(cudaSetDevice(lg->op->ctx->device));
  if (support)
    for (size_t j = 0; j < lg->support.size(); ++j) support[j] = lg->support[j] + 1;
  if (coeffs && lg->s) {
    CU(cudaStreamSynchronize(st_of(lg)));
    CU(cudaMemcpy(coeffs, lg->S.x, (size_t)lg->s * 16, cudaMemcpyDeviceToHost));
  }
  if (support_size) *support_size = (uint64_t)lg->s;
  if (iterations) *iterations = (uint64_t)lg->iters;
  if (residual) *residual = lg->rn;
  if (aborted) *aborted = lg->aborted;
  return FMP_OK;
}

int fmp_large_solve(fmp_op op, int dtype, const void* y, const fmp_omp_config* cfg, fmp_omp_result* out) {
  if (!op || !y || !cfg || !out) return fail(FMP_EINVAL, "null argument");
  fmp_large lg = nullptr;
  if (int e = fmp_large_create(op, dtype, 0, 1, cfg, nullptr, &lg)) return e;
  int st = fmp_large_group_solve(&lg, 1, y, cfg->tolerances ? cfg->tolerances[0] : cfg->tolerance);
  if (!st)
    st = fmp_large_result(lg, out->support, out->coeffs, out->support_size, out->iterations, out->residual,
                          out->aborted);
  fmp_large_destroy(lg);
  return st;
}

int fmp_large_record_size(void) { return (int)sizeof(fmp::LgRec); }

int fmp_large_merge_records(const void* recs, int nshards, const uint32_t* selbits, double* out4) {
  if (!recs || nshards < 1 || !out4) return fail(FMP_EINVAL, "null argument");
  fmp::LgPick pk;
  fmp::lg_merge_host((const fmp::LgRec*)recs, nshards, selbits, &pk);
  out4[0] = pk.flags ? -1.0 : (double)pk.j;
  out4[1] = pk.best64;
  out4[2] = (double)pk.flags;
  out4[3] = 0.0;
  return FMP_OK;
}

}  // extern "C"
