// Batched structured transforms: conventional correlation Phi^H r,
// Phi x, U v (transform.cpp:120-152, sensing.cpp:93-109), the band argmax
// (solvers.cpp:90-101) and the correlation-kernel build (kernel.cpp:24-72).
#include "fmp_kcommon.cuh"

namespace fmp {
namespace {
// ------------------------------------------------------------- transform
template <class V, bool INV, bool HAD>
__global__ void __launch_bounds__(512) k_transform(DevOp op, const V* __restrict__ in,
                                                   V* __restrict__ out, int64_t batch,
                                                   int in_omega, int out_omega,
                                                   uint64_t* __restrict__ amax) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[32];
  __shared__ unsigned redu[32];
  V* buf = reinterpret_cast<V*>(smem_raw);
  const int n = (int)op.n, m = (int)op.m, log2n = op.log2n;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int nbuf = n + (n >> LOGP);
  const V* tw = twiddles<V>(op);
  const double sc = inv_sqrt_n(n);
  const V z = zero_of(V{});
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    if (in_omega) {
      for (int i = tid; i < nbuf; i += nth) buf[i] = z;
      __syncthreads();
      const V* r = in + b * m;
      for (int j = tid; j < m; j += nth) buf[in_slot<HAD>(op.omega[j], log2n)] = r[j];
    } else {
      const V* v = in + b * n;
      for (int k = tid; k < n; k += nth) buf[in_slot<HAD>((unsigned)k, log2n)] = v[k];
    }
    __syncthreads();
    block_transform<RMAX, INV, HAD>(buf, log2n, TwTable<V>{tw}, tid, nth);
    if (out_omega) {
      V* o = out + b * m;
      for (int j = tid; j < m; j += nth) o[j] = scale(buf[padx<LOGP>((int)op.omega[j])], sc);
    } else {
      V* o = out ? out + b * n : nullptr;
      double best = 0.0;
      for (int k = tid; k < n; k += nth) {
        const V v = scale(buf[padx<LOGP>(k)], sc);
        if (o) o[k] = v;
        best = fmax(best, mag2(v));
      }
      if (amax) {
        best = block_max(best, red);
        const double cut = best * (1.0 - kTieBandRel);
        unsigned first = 0xffffffffu;
        for (int k = tid; k < n; k += nth)
          if (mag2(scale(buf[padx<LOGP>(k)], sc)) >= cut) { first = (unsigned)k; break; }
        first = block_min_u(first, redu);
        if (tid == 0) amax[b] = (first == 0xffffffffu ? 0u : first) + 1;  // 1-based
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------ large-n transform path
// n beyond one CTA's shared memory: the same radix passes, one launch per
// pass, each thread one radix-R sub-problem of one vector in global memory.
template <class V, bool HAD>
__global__ void k_scatter_in(const V* __restrict__ in, V* __restrict__ work, int64_t batch,
                             int in_omega, const uint32_t* __restrict__ omega, int64_t m,
                             int log2n) {
  const int64_t n = 1ll << log2n;
  const int64_t len = in_omega ? m : n;
  const int64_t total = batch * len;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = u / len, j = u - b * len;
    const unsigned p = in_omega ? omega[j] : (unsigned)j;
    const unsigned slot = HAD ? p : brev_n(p, log2n);
    work[b * n + slot] = in[u];
  }
}

template <class V, int R, bool INV, bool HAD>
__global__ void k_gpass(V* data, int64_t batch, int log2n, int logS, const V* __restrict__ tw) {
  constexpr int LOGR = log2_of<R>::v;
  const int64_t nsub = 1ll << (log2n - LOGR);
  const int64_t total = batch * nsub;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = u >> (log2n - LOGR);
    pass_one<R, 31, INV, HAD>(data + (b << log2n), log2n, logS, log2n, TwTable<V>{tw},
                              (int)(u & (nsub - 1)));
  }
}

template <class V>
__global__ void k_out(V* work, V* __restrict__ out, int64_t batch, int out_omega,
                      const uint32_t* __restrict__ omega, int64_t m, int log2n, int scaled) {
  const int64_t n = 1ll << log2n;
  const int64_t len = out_omega ? m : n;
  const int64_t total = batch * len;
  const double sc = scaled ? 1.0 : 1.0 / sqrt((double)n);
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = u / len, j = u - b * len;
    const V v = scale(work[b * n + (out_omega ? omega[j] : j)], sc);
    if (out) out[u] = v;
    else work[u] = v;  // dense, in place
  }
}

// --------------------------------------------------------- kernel finish
// c arrives in g64 from the adjoint transform of the Omega indicator scaled
// by 1/sqrt(N) (= apply_adjoint(apply(e1)), kernel.cpp:33).
__global__ void k_kernel_finish(DevOp op) {
  const int64_t n = op.n;
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (op.kind == FOURIER) {
    // exact conjugate symmetry (kernel.cpp:35-45)
    if (i == 0) {
      op.g64[0].y = 0.0;
      if (n % 2 == 0 && n > 1) op.g64[n / 2].y = 0.0;
    } else if (2 * i < n) {
      const double2 a = op.g64[i], b = op.g64[n - i];
      const double2 avg = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
      op.g64[i] = avg;
      op.g64[n - i] = make_double2(avg.x, -avg.y);
    }
  } else if (i < n) {
    // snap onto the integer lattice N*c (kernel.cpp:46-55)
    const double k = round(op.g64[i].x * (double)n);
    op.g64[i] = make_double2(k / (double)n, 0.0);
    op.gr64[i] = k / (double)n;
    if (op.glat) op.glat[i] = (uint16_t)((int)k + 32768);
  }
}

__global__ void k_kernel_f32(DevOp op) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < op.n) op.g32[i] = make_float2((float)op.g64[i].x, (float)op.g64[i].y);
}

__global__ void k_twiddles(DevOp op) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < op.n) {
    double s, c;
    sincospi(-2.0 * (double)k / (double)op.n, &s, &c);
    op.tw64[k] = make_double2(c, s);
    op.tw32[k] = make_float2((float)c, (float)s);
  }
}

template <class V, bool INV, bool HAD>
cudaError_t launch_tr_t(const TransformArgs& a, cudaStream_t st) {
  const DevOp& op = *a.op;
  const int64_t n = op.n;
  const size_t smem = (size_t)(n + (n >> LOGP)) * sizeof(V);
  int threads = (int)std::min<int64_t>(512, std::max<int64_t>(32, n / RMAX));
  threads = ((threads + 31) / 32) * 32;
  auto k = k_transform<V, INV, HAD>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, smem);
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(a.batch, (int64_t)num_sms() * std::max(occ, 1)));
  k<<<(int)grid, threads, smem, st>>>(op, (const V*)a.in, (V*)a.out, a.batch, a.in_omega,
                                       a.out_omega, a.argmax_out);
  ++g_launches;
  return cudaGetLastError();
}

// ------------------------------------------------ cluster transform path
// n beyond one CTA: a thread-block cluster of K CTAs owns one vector.
// Phase A: CTA c runs the first log2(n/K) stages on its contiguous block in
// shared memory (these stages never leave the block).  A cluster barrier
// (release/acquire) makes every block visible through distributed shared
// memory.  Phase B: the last log2(K) stages are a radix-K pass of span n/K;
// CTA c owns 1/K of the offsets, reads the K operands from the cluster's
// shared memory and writes the final values.  HBM traffic is the input plus
// one output write.
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// generic pointer to the same shared-memory location in cluster CTA `rank`
template <class T>
__device__ __forceinline__ T* dsmem(T* p, unsigned rank) {
  T* out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"(p), "r"(rank));
  return out;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <class V, bool INV, bool HAD, int K>
__global__ void __launch_bounds__(256) k_transform_cluster(DevOp op, const V* __restrict__ in,
                                                           V* dst, int64_t batch, int in_omega) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* buf = reinterpret_cast<V*>(smem_raw);
  constexpr int LOGK = log2_of<K>::v;
  const int log2n = op.log2n, n = (int)op.n, m = (int)op.m;
  const int log2b = log2n - LOGK, B = 1 << log2b;
  const int tid = threadIdx.x, nth = blockDim.x;
  const unsigned c = cluster_rank();
  const int64_t cid = blockIdx.x / K, ncl = gridDim.x / K;
  const V* tw = twiddles<V>(op);
  const double sc = 1.0 / sqrt((double)n);
  const V z = zero_of(V{});
  const int lo_slot = (int)c * B;
  // this block's Omega rows: bisection in the slot-sorted scatter
  int k0 = 0, k1 = 0;
  if (in_omega) {  // B is a multiple of 256
    k0 = (int)op.scat_off[lo_slot >> 8];
    k1 = (int)op.scat_off[(lo_slot + B) >> 8];
  }
  for (int64_t b = cid; b < batch; b += ncl) {
    V* vec = dst + b * n;
    // ---- phase A
    if (in_omega) {
      for (int i = tid; i < B + (B >> LOGP); i += nth) buf[i] = z;
      __syncthreads();
      const V* r = in + b * m;
      for (int k = k0 + tid; k < k1; k += nth)
        buf[padx<LOGP>((int)op.scat_pos[k] - lo_slot)] = r[op.scat_row[k]];
    } else {
      const V* v = in + b * n;
      for (int i = tid; i < B; i += nth) {
        const unsigned p = (unsigned)(lo_slot + i);
        buf[padx<LOGP>(i)] = v[HAD ? p : brev_n(p, log2n)];
      }
    }
    __syncthreads();
    block_transform<RMAX, INV, HAD>(buf, log2b, TwTable<V>{tw}, tid, nth, log2n);
    cluster_sync_all();  // every block's phase A is in its shared memory
    // ---- phase B: offsets o in [c B/K, (c+1) B/K), elements o + j B, read
    // straight from the cluster's shared memory (no HBM round trip)
    const int o0 = (int)c * (B / K);
    for (int o = o0 + tid; o < o0 + B / K; o += nth) {
      V v[K];
#pragma unroll
      for (int j = 0; j < K; ++j) v[j] = dsmem(buf, (unsigned)j)[padx<LOGP>(o)];
      if constexpr (HAD) {
        wht_reg<K>(v);
      } else {
#pragma unroll
        for (int j = 1; j < K; ++j) {
          V w = tw[brev_small<K>(j) * o];
          if (INV) w.y = -w.y;
          v[j] = cmul(v[j], w);
        }
        dft_reg<K, INV>(v);
      }
#pragma unroll
      for (int j = 0; j < K; ++j) vec[o + j * B] = scale(v[j], sc);
    }
    cluster_sync_all();  // no block refills its buffer while others still read it
  }
}

// ------------------------------------------- job-queue large-n transform
// Same two-phase factorisation as the cluster path, but scheduled as a queue
// of jobs over a persistent grid: job A(b, c) transforms block c of vector b in
// smem and publishes it (release); job B(b, c) waits for vector b's K A-jobs
// (acquire) and finishes offsets [c B/K, (c+1) B/K) in registers.  Jobs are
// issued in vector order with B(b, .) lagging A(b, .) by D vectors, so a
// B-job's inputs are normally complete (and L2-resident) when it starts and no
// CTA ever idles at a barrier.  A-jobs never wait, and every job is claimed by
// a running CTA, so the waits cannot deadlock.
template <class V, bool INV, bool HAD, int K>
__global__ void __launch_bounds__(256, 3) k_transform_queue(DevOp op, const V* __restrict__ in,
                                                         V* dst, int64_t batch, int in_omega,
                                                         int* __restrict__ counter,
                                                         int* __restrict__ done, int lag) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_job;
  V* buf = reinterpret_cast<V*>(smem_raw);
  constexpr int LOGK = log2_of<K>::v;
  const int log2n = op.log2n, n = (int)op.n, m = (int)op.m;
  const int log2b = log2n - LOGK, B = 1 << log2b;
  const int tid = threadIdx.x, nth = blockDim.x;
  const V* tw = twiddles<V>(op);
  const double sc = 1.0 / sqrt((double)n);
  const V z = zero_of(V{});
  // job j -> step i = j / (2K); within a step: K A-jobs of vector i, then K
  // B-jobs of vector i - lag
  const int64_t steps = batch + lag;
  const int64_t njobs = steps * 2 * K;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_job = atomicAdd(counter, 1);
    __syncthreads();
    const int64_t j = s_job;
    if (j >= njobs) break;
    const int64_t step = j / (2 * K);
    const int r = (int)(j - step * 2 * K);
    const bool isA = r < K;
    const int c = isA ? r : r - K;
    const int64_t b = isA ? step : step - lag;
    if (b < 0 || b >= batch) continue;
    V* vec = dst + b * (int64_t)n;
    if (isA) {
      const int lo_slot = c * B;
      if (in_omega) {
        for (int i = tid; i < B + (B >> LOGP); i += nth) buf[i] = z;
        // this block's rows in the slot-sorted scatter (B is a multiple of 256)
        const int k0 = (int)op.scat_off[lo_slot >> 8], k1 = (int)op.scat_off[(lo_slot + B) >> 8];
        __syncthreads();
        const V* rr = in + b * m;
        // unrolled: the slot / row loads and the gathers of several rows are
        // in flight together (L2 latency, not bandwidth, bounds this loop)
#pragma unroll 4
        for (int k = k0 + tid; k < k1; k += nth)
          buf[padx<LOGP>((int)op.scat_pos[k] - lo_slot)] = rr[op.scat_row[k]];
      } else {
        const V* v = in + b * n;
        for (int i = tid; i < B; i += nth) {
          const unsigned p = (unsigned)(lo_slot + i);
          buf[padx<LOGP>(i)] = v[HAD ? p : brev_n(p, log2n)];
        }
      }
      __syncthreads();
      block_transform<RMAX, INV, HAD>(buf, log2b, TwTable<V>{tw}, tid, nth, log2n);
      for (int i = tid; i < B; i += nth) __stcg(vec + lo_slot + i, buf[padx<LOGP>(i)]);
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicAdd(done + b, 1);
      }
    } else {
      if (tid == 0) {
        while (atomicAdd(done + b, 0) < K) __nanosleep(64);
        __threadfence();
      }
      __syncthreads();
      const int o0 = c * (B / K);
      // two offsets in flight per thread where the registers allow it
      constexpr int UB = sizeof(V) * K <= 64 ? 2 : 1;
#pragma unroll UB
      for (int o = o0 + tid; o < o0 + B / K; o += nth) {
        V v[K];
#pragma unroll
        for (int q = 0; q < K; ++q) v[q] = __ldcg(vec + o + q * B);
        if constexpr (HAD) {
          wht_reg<K>(v);
        } else {
#pragma unroll
          for (int q = 1; q < K; ++q) {
            V w = tw[brev_small<K>(q) * o];
            if (INV) w.y = -w.y;
            v[q] = cmul(v[q], w);
          }
          dft_reg<K, INV>(v);
        }
#pragma unroll
        for (int q = 0; q < K; ++q) __stcg(vec + o + q * B, scale(v[q], sc));
      }
    }
  }
}

template <class V, bool INV, bool HAD, int K>
cudaError_t launch_tr_queue_k(const TransformArgs& a, cudaStream_t st) {
  const DevOp& op = *a.op;
  const int64_t B = op.n / K;
  const size_t smem = (size_t)(B + (B >> LOGP)) * sizeof(V);
  auto kern = k_transform_queue<V, INV, HAD, K>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  V* dst = a.out_omega ? (V*)a.work : (V*)a.out;
  if (!dst) dst = (V*)a.work;
  if (!dst || !a.sync) return cudaErrorInvalidValue;
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
  const int grid = std::max(1, occ) * num_sms();
  // lag in vectors: enough jobs in flight that a vector's A-jobs are done
  // when its B-jobs are claimed
  const int lag = std::max(1, (2 * grid) / (2 * K) + 1);
  int* counter = a.sync;
  int* done = a.sync + 32;
  cudaError_t e = cudaMemsetAsync(a.sync, 0, (size_t)(32 + a.batch) * sizeof(int), st);
  if (e != cudaSuccess) return e;
  kern<<<grid, 256, smem, st>>>(op, (const V*)a.in, dst, a.batch, a.in_omega, counter, done, lag);
  ++g_launches;
  const int g2 = num_sms() * 8;
  if (a.out_omega) {
    k_out<V><<<g2, 256, 0, st>>>(dst, (V*)a.out, a.batch, 1, op.omega, op.m, op.log2n, 1);
    ++g_launches;
  }
  if (a.argmax_out && !a.out_omega) {
    const int g3 = (int)std::max<int64_t>(1, std::min<int64_t>(a.batch, 4 * num_sms()));
    k_argmax<V><<<g3, 512, 0, st>>>(dst, op.n, a.batch, a.argmax_out);
    ++g_launches;
  }
  return cudaGetLastError();
}

template <class V, bool INV, bool HAD>
cudaError_t launch_tr_queue(const TransformArgs& a, cudaStream_t st, int k) {
  switch (k) {
    case 2: return launch_tr_queue_k<V, INV, HAD, 2>(a, st);
    case 4: return launch_tr_queue_k<V, INV, HAD, 4>(a, st);
    case 8: return launch_tr_queue_k<V, INV, HAD, 8>(a, st);
    case 16: return launch_tr_queue_k<V, INV, HAD, 16>(a, st);
  }
  return cudaErrorInvalidValue;
}

template <class V, bool INV, bool HAD, int K>
cudaError_t launch_tr_cluster_k(const TransformArgs& a, cudaStream_t st) {
  const DevOp& op = *a.op;
  const int64_t B = op.n / K;
  const size_t smem = (size_t)(B + (B >> LOGP)) * sizeof(V);
  auto kern = k_transform_cluster<V, INV, HAD, K>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (K > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  V* dst = a.out_omega ? (V*)a.work : (V*)a.out;
  if (!dst) dst = (V*)a.work;
  if (!dst) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = K;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  cfg.gridDim = dim3(K);
  cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
  if (ncl <= 0) ncl = std::max(1, num_sms() / K);
  ncl = (int)std::min<int64_t>(ncl, a.batch);
  cfg.gridDim = dim3(ncl * K);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, op, (const V*)a.in, dst, a.batch, a.in_omega);
  if (e != cudaSuccess) return e;
  ++g_launches;
  const int grid = num_sms() * 8;
  if (a.out_omega) {
    k_out<V><<<grid, 256, 0, st>>>(dst, (V*)a.out, a.batch, 1, op.omega, op.m, op.log2n, 1);
    ++g_launches;
  }
  if (a.argmax_out && !a.out_omega) {
    const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>(a.batch, 4 * num_sms()));
    k_argmax<V><<<g2, 512, 0, st>>>(dst, op.n, a.batch, a.argmax_out);
    ++g_launches;
  }
  return cudaGetLastError();
}

// cluster size for a vector of n elements: blocks of at most 32 KB, so that
// several clusters are resident per SM group and hide each other's barriers
template <class V>
int cluster_k(int64_t n, int dtype) {
  int64_t k = 2;
  while (k <= 16 && (n / k) * (int64_t)sizeof(V) > 64 * 1024) k *= 2;
  if (k > 16 || n / k > transform_max_n(dtype)) return 0;
  return (int)k;
}

// block size for the job-queue path (three CTAs per SM): 64 KB blocks, 32 KB
// for 4-byte elements (measured on config 3)
template <class V>
int queue_k(int64_t n, int dtype) {
  int64_t target = sizeof(V) <= 4 ? 32 * 1024 : 64 * 1024;
  if (const char* e = getenv("FMP_QUEUE_KB")) target = (int64_t)atoi(e) * 1024;  // tuning
  int64_t k = 2;
  while (k <= 16 && (n / k) * (int64_t)sizeof(V) > target) k *= 2;
  if (k > 16 || n / k > transform_max_n(dtype)) return 0;
  return (int)k;
}

template <class V, bool INV, bool HAD>
cudaError_t launch_tr_cluster(const TransformArgs& a, cudaStream_t st, int k) {
  switch (k) {
    case 2: return launch_tr_cluster_k<V, INV, HAD, 2>(a, st);
    case 4: return launch_tr_cluster_k<V, INV, HAD, 4>(a, st);
    case 8: return launch_tr_cluster_k<V, INV, HAD, 8>(a, st);
    case 16: return launch_tr_cluster_k<V, INV, HAD, 16>(a, st);
  }
  return cudaErrorInvalidValue;
}

template <class V, bool INV, bool HAD>
cudaError_t launch_tr_global(const TransformArgs& a, cudaStream_t st) {
  const DevOp& op = *a.op;
  if (!a.work) return cudaErrorInvalidValue;
  V* work = (V*)a.work;
  const int log2n = op.log2n;
  const int64_t n = op.n;
  const int grid = num_sms() * 8;
  cudaError_t e;
  if (a.in_omega) {
    e = cudaMemsetAsync(work, 0, (size_t)a.batch * n * sizeof(V), st);
    if (e != cudaSuccess) return e;
  }
  k_scatter_in<V, HAD><<<grid, 256, 0, st>>>((const V*)a.in, work, a.batch, a.in_omega,
                                             op.omega, op.m, log2n);
  ++g_launches;
  const V* tw = nullptr;
  if constexpr (!HAD) tw = (const V*)(sizeof(V) == 16 ? (const void*)op.tw64 : (const void*)op.tw32);
  int s = 0;
  for (; log2n - s >= LOGP; s += LOGP) {
    k_gpass<V, 16, INV, HAD><<<grid, 256, 0, st>>>(work, a.batch, log2n, s, tw);
    ++g_launches;
  }
  switch (log2n - s) {
    case 1: k_gpass<V, 2, INV, HAD><<<grid, 256, 0, st>>>(work, a.batch, log2n, s, tw); ++g_launches; break;
    case 2: k_gpass<V, 4, INV, HAD><<<grid, 256, 0, st>>>(work, a.batch, log2n, s, tw); ++g_launches; break;
    case 3: k_gpass<V, 8, INV, HAD><<<grid, 256, 0, st>>>(work, a.batch, log2n, s, tw); ++g_launches; break;
    default: break;
  }
  V* out = (V*)a.out;
  k_out<V><<<grid, 256, 0, st>>>(work, (a.out_omega || out) ? out : nullptr, a.batch,
                                 a.out_omega, op.omega, op.m, log2n, 0);
  ++g_launches;
  if (a.argmax_out && !a.out_omega) {
    const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>(a.batch, 4 * num_sms()));
    k_argmax<V><<<g2, 512, 0, st>>>(out ? out : work, n, a.batch, a.argmax_out);
    ++g_launches;
  }
  return cudaGetLastError();
}

template <class V, bool HAD>
cudaError_t launch_tr_v(const TransformArgs& a, cudaStream_t st) {
  if (a.op->n > transform_max_n(a.dtype) && a.op->fs_l1 && a.work && a.out) {
    // two passes over HBM (n >= 2^18; fmp_transform_4s.cu)
    FsTransform t{};
    t.op = a.op;
    t.dtype = a.dtype;
    t.inverse = a.inverse;
    t.in_mode = a.in_omega ? 1 : 0;
    t.in = a.in;
    t.mid = a.work;
    t.out_mode = a.out_omega ? 1 : 0;
    t.out = a.out;
    t.batch = a.batch;
    cudaError_t e = launch_transform_fs(t, st);
    if (e != cudaSuccess) return e;
    if (a.argmax_out && !a.out_omega) {
      const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>(a.batch, 4 * num_sms()));
      k_argmax<V><<<g2, 512, 0, st>>>((const V*)a.out, a.op->n, a.batch, a.argmax_out);
      ++g_launches;
    }
    return cudaGetLastError();
  }
  if (a.op->n > transform_max_n(a.dtype)) {
    if constexpr (HAD) {
      // one pass over HBM: sparse input folded at load time (fmp_transform_fold.cu)
      cudaError_t e = launch_wht_fold(a, st);
      if (e == cudaSuccess) {
        if (a.argmax_out) {
          const int g2 = (int)std::max<int64_t>(1, std::min<int64_t>(a.batch, 4 * num_sms()));
          k_argmax<V><<<g2, 512, 0, st>>>((const V*)a.out, a.op->n, a.batch, a.argmax_out);
          ++g_launches;
        }
        return cudaGetLastError();
      }
      if (e != cudaErrorNotSupported) return e;
    }
    const int k = a.op->scat_pos ? cluster_k<V>(a.op->n, a.dtype) : 0;
    const int kq = a.op->scat_pos ? queue_k<V>(a.op->n, a.dtype) : 0;
    // distributed-shared-memory cluster for 4-byte elements (config 3 f32:
    // 0.20 ms against 0.26 ms for the job queue); for 8- and 16-byte
    // elements the job queue measured faster (f64: 0.34 ms against 0.46)
    if (k && k <= 8 && sizeof(V) <= 4)
      return a.inverse ? launch_tr_cluster<V, true, HAD>(a, st, k)
                       : launch_tr_cluster<V, false, HAD>(a, st, k);
    if (kq && a.sync)
      return a.inverse ? launch_tr_queue<V, true, HAD>(a, st, kq)
                       : launch_tr_queue<V, false, HAD>(a, st, kq);
    if (k && a.sync)
      return a.inverse ? launch_tr_queue<V, true, HAD>(a, st, k)
                       : launch_tr_queue<V, false, HAD>(a, st, k);
    if (k)
      return a.inverse ? launch_tr_cluster<V, true, HAD>(a, st, k)
                       : launch_tr_cluster<V, false, HAD>(a, st, k);
    return a.inverse ? launch_tr_global<V, true, HAD>(a, st) : launch_tr_global<V, false, HAD>(a, st);
  }
  return a.inverse ? launch_tr_t<V, true, HAD>(a, st) : launch_tr_t<V, false, HAD>(a, st);
}

}  // namespace

thread_local int g_launches = 0;

int last_launch_count() { return g_launches; }

int64_t transform_max_n(int dtype) {
  const int64_t cap = (int64_t)smem_optin() - 2048;
  int64_t n = 1;
  while ((2 * n + ((2 * n) >> LOGP)) * elem_bytes(dtype) <= cap) n *= 2;
  return n;
}

cudaError_t launch_transform(const TransformArgs& a, cudaStream_t st) {
  g_launches = 0;
  const bool had = a.op->kind == HADAMARD;
  switch (a.dtype) {
    case C128: return had ? launch_tr_v<double2, true>(a, st) : launch_tr_v<double2, false>(a, st);
    case C64: return had ? launch_tr_v<float2, true>(a, st) : launch_tr_v<float2, false>(a, st);
    case F64: return had ? launch_tr_v<double, true>(a, st) : cudaErrorInvalidValue;
    case F32: return had ? launch_tr_v<float, true>(a, st) : cudaErrorInvalidValue;
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_argmax(const ArgmaxArgs& a, cudaStream_t st) {
  g_launches = 1;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(a.batch, 4 * num_sms()));
  switch (a.dtype) {
    case C128: k_argmax<double2><<<grid, 512, 0, st>>>((const double2*)a.h, a.n, a.batch, a.out); break;
    case C64: k_argmax<float2><<<grid, 512, 0, st>>>((const float2*)a.h, a.n, a.batch, a.out); break;
    case F64: k_argmax<double><<<grid, 512, 0, st>>>((const double*)a.h, a.n, a.batch, a.out); break;
    case F32: k_argmax<float><<<grid, 512, 0, st>>>((const float*)a.h, a.n, a.batch, a.out); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_kernel_finish(const DevOp& op, cudaStream_t st) {
  const int64_t blocks = (op.n + 255) / 256;
  k_kernel_finish<<<(unsigned)blocks, 256, 0, st>>>(op);
  g_launches += 1;
  if (op.g32) {
    k_kernel_f32<<<(unsigned)blocks, 256, 0, st>>>(op);
    g_launches += 1;
  }
  return cudaGetLastError();
}

// max_{k != 0} |c_k|: non-negative doubles order like their bit patterns
__global__ void k_gmax_off(DevOp op, unsigned long long* out) {
  double v = 0.0;
  for (int64_t k = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < op.n;
       k += (int64_t)gridDim.x * blockDim.x) {
    const double2 g = op.g64[k];
    v = fmax(v, sqrt(g.x * g.x + g.y * g.y));
  }
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(v));
}

__global__ void k_widen(const float* __restrict__ in, double* __restrict__ out, int64_t count) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)in[i];
}

cudaError_t launch_gmax_off(const DevOp& op, unsigned long long* out, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(out, 0, 8, st);
  if (e != cudaSuccess) return e;
  const int64_t blocks = std::min<int64_t>((op.n + 255) / 256, 8 * num_sms());
  k_gmax_off<<<(unsigned)std::max<int64_t>(1, blocks), 256, 0, st>>>(op, out);
  g_launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_widen(const float* in, double* out, int64_t count, cudaStream_t st) {
  const int64_t blocks = std::min<int64_t>((count + 255) / 256, 16 * num_sms());
  k_widen<<<(unsigned)std::max<int64_t>(1, blocks), 256, 0, st>>>(in, out, count);
  g_launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_twiddles(const DevOp& op, cudaStream_t st) {
  const int64_t blocks = (op.n + 255) / 256;
  k_twiddles<<<(unsigned)blocks, 256, 0, st>>>(op);
  g_launches += 1;
  return cudaGetLastError();
}

}  // namespace fmp

// ------------------------------------------------ FMA-pipe calibration
// Independent FMA chains (8 per thread) over a full-occupancy grid: the
// roofline denominator for the accumulate path (measured on the box, since
// MEASURED_PEAKS.json carries HBM and tensor peaks only).
namespace {
template <class T>
__global__ void __launch_bounds__(256) k_fma_peak(T* out, int iters, T a, T b) {
  T v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = (T)(threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = v[j] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += v[j];
  if (s == (T)-1.2345) out[threadIdx.x] = s;  // keep the chains live
}
}  // namespace

namespace fmp {
cudaError_t fma_peak(int is_double, double* fma_per_s) {
  const int sms = num_sms();
  const int blocks = sms * 8, threads = 256, iters = 4096;
  void* out = nullptr;
  cudaError_t e = cudaMalloc(&out, 4096 * 8);
  if (e != cudaSuccess) return e;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    if (is_double)
      k_fma_peak<double><<<blocks, threads>>>((double*)out, iters, 0.999999, 1e-7);
    else
      k_fma_peak<float><<<blocks, threads>>>((float*)out, iters, 0.9999f, 1e-4f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (rep > 0) best = std::min(best, ms);
  }
  e = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(out);
  *fma_per_s = (double)blocks * threads * iters * 8 / (best * 1e-3);
  return e;
}
}  // namespace fmp

// ------------------------------------------------------ least squares
// least_squares (solvers.cpp:276-294, normal-equations form solvers.cpp:120-177)
// for a given support: Gram entries are kernel lookups, the right-hand side
// b_j = phi_j^H y is a direct sum over the rows with closed-form entries
// (transform.cpp:154-163), then a Cholesky factorisation with the reference's
// pivot floor 1e-12 * diag and two triangular solves.  One CTA per problem;
// the s x s factor lives in global scratch.
namespace fmp {
namespace {
template <class V>
__global__ void __launch_bounds__(256) k_least_squares(DevOp op, const V* __restrict__ y,
                                                       const uint32_t* __restrict__ sup, int s,
                                                       int64_t batch, double2* __restrict__ x,
                                                       int64_t* __restrict__ bad,
                                                       double2* __restrict__ L) {
  __shared__ double red[64];
  const int tid = threadIdx.x, nth = blockDim.x;
  const int n = (int)op.n, m = (int)op.m;
  const double isn = 1.0 / sqrt((double)n);
  for (int64_t b = blockIdx.x; b < batch; b += gridDim.x) {
    const V* yb = y + b * m;
    const uint32_t* sb = sup + b * s;
    double2* Lb = L + (size_t)blockIdx.x * s * s;
    double2* xb = x + b * s;
    // rhs z_j = phi_j^H y
    for (int j = 0; j < s; ++j) {
      double ar = 0.0, ai = 0.0;
      for (int i = tid; i < m; i += nth) {
        const double2 yv = to_c128(yb[i]);
        double er, ei;
        if (op.kind == FOURIER) {
          const double2 e = op.tw64[((uint64_t)op.omega[i] * sb[j]) & (uint64_t)(n - 1)];
          er = e.x * isn;
          ei = -e.y * isn;  // conj(U[omega, j])
        } else {
          er = (__popc(op.omega[i] & sb[j]) & 1) ? -isn : isn;
          ei = 0.0;
        }
        ar += er * yv.x - ei * yv.y;
        ai += er * yv.y + ei * yv.x;
      }
      ar = warp_sum(ar);
      ai = warp_sum(ai);
      __syncthreads();
      if ((tid & 31) == 0) { red[tid >> 5] = ar; red[32 + (tid >> 5)] = ai; }
      __syncthreads();
      if (tid == 0) {
        double sr = 0.0, si = 0.0;
        for (int w = 0; w < (nth + 31) / 32; ++w) { sr += red[w]; si += red[32 + w]; }
        xb[j] = make_double2(sr, si);
      }
    }
    __syncthreads();
    // Cholesky of G(i, j) = c[(lambda_i - lambda_j) mod N] / c[lambda_i ^ lambda_j]
    if (tid == 0) {
      int64_t badpos = -1;
      auto G = [&](int i, int j) -> double2 {
        const unsigned a = sb[i], c = sb[j];
        if (op.kind == FOURIER) return op.g64[(a - c) & (unsigned)(n - 1)];
        return make_double2(op.gr64[a ^ c], 0.0);
      };
      for (int j = 0; j < s && badpos < 0; ++j) {
        const double diag = G(j, j).x;
        double d = diag;
        for (int k = 0; k < j; ++k) d -= mag2(Lb[j * s + k]);
        if (!(d > 1e-12 * diag)) { badpos = j; break; }
        const double ljj = sqrt(d);
        Lb[j * s + j] = make_double2(ljj, 0.0);
        for (int i = j + 1; i < s; ++i) {
          double2 v = G(i, j);
          for (int k = 0; k < j; ++k) {
            const double2 p = Lb[i * s + k], q = Lb[j * s + k];
            v.x -= p.x * q.x + p.y * q.y;  // L(i,k) conj(L(j,k))
            v.y -= p.y * q.x - p.x * q.y;
          }
          Lb[i * s + j] = make_double2(v.x / ljj, v.y / ljj);
        }
      }
      if (badpos < 0) {
        for (int i = 0; i < s; ++i) {  // forward: L z = b
          double2 v = xb[i];
          for (int k = 0; k < i; ++k) {
            const double2 p = Lb[i * s + k], q = xb[k];
            v.x -= p.x * q.x - p.y * q.y;
            v.y -= p.x * q.y + p.y * q.x;
          }
          const double l = Lb[i * s + i].x;
          xb[i] = make_double2(v.x / l, v.y / l);
        }
        for (int i = s - 1; i >= 0; --i) {  // backward: L^H x = z
          double2 v = xb[i];
          for (int k = i + 1; k < s; ++k) {
            const double2 p = Lb[k * s + i], q = xb[k];
            v.x -= p.x * q.x + p.y * q.y;  // conj(L(k,i)) x_k
            v.y -= p.x * q.y - p.y * q.x;
          }
          const double l = Lb[i * s + i].x;
          xb[i] = make_double2(v.x / l, v.y / l);
        }
      }
      bad[b] = badpos;
    }
    __syncthreads();
  }
}
}  // namespace

cudaError_t launch_least_squares(const DevOp& op, int dtype, const void* y, const uint32_t* sup,
                                 int s, int64_t batch, double2* x, int64_t* bad, double2* L,
                                 int grid, cudaStream_t st) {
  switch (dtype) {
    case C128: k_least_squares<double2><<<grid, 256, 0, st>>>(op, (const double2*)y, sup, s, batch, x, bad, L); break;
    case C64: k_least_squares<float2><<<grid, 256, 0, st>>>(op, (const float2*)y, sup, s, batch, x, bad, L); break;
    case F64: k_least_squares<double><<<grid, 256, 0, st>>>(op, (const double*)y, sup, s, batch, x, bad, L); break;
    case F32: k_least_squares<float><<<grid, 256, 0, st>>>(op, (const float*)y, sup, s, batch, x, bad, L); break;
    default: return cudaErrorInvalidValue;
  }
  g_launches = 1;
  return cudaGetLastError();
}
}  // namespace fmp
