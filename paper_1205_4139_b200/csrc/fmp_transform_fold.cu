// Conventional Hadamard correlation Phi^H r for vectors larger than one CTA's
// shared memory (config 3: N = 65536, M = 8192), in ONE pass over HBM with no
// intermediate vector.
//
// Reference: SensingOperator::apply_adjoint (sensing.cpp:102-109) = scatter r
// at Omega into zeros, StructuredUnitary::fht (transform.cpp:86-100), scale by
// 1/sqrt(N) (transform.cpp:132).
//
// Factorisation.  Write i = i_hi B + i_lo, k = k_hi B + k_lo (B = N / S).
// H_N = H_S (x) H_B, so
//     h[k_hi B + k_lo] = sum_{i_lo} H_B[k_lo, i_lo] z_{k_hi}[i_lo],
//     z_{k_hi}[i_lo]   = sum_{i_hi} (-1)^{popc(k_hi & i_hi)} x[i_hi B + i_lo].
// Output block k_hi therefore needs only a fold of the sparse input into a
// B-point buffer z (the S-point high-bit stages, done at load time: x is only
// M nonzeros, the rows of Omega), a B-point transform of z in shared memory
// and a contiguous store.  Each persistent CTA stages a vector's r in shared
// memory once (one bulk copy) and produces its S output blocks in turn, so
// HBM traffic is exactly the algorithmic (M + N) * sizeof(V) per vector and
// nothing intermediate leaves the SM.
//
// Register-tile passes: pass p transforms index bits [lo_p, lo_p + R_p) of z;
// each thread holds 2^R_p elements of one group.  z is stored with one pad
// element per row of 32 (the first pass's rows), which makes every pass
// conflict-free: in pass 1 the lanes' rows are 33 elements apart, in later
// passes consecutive lanes own consecutive low indices.
#include "fmp_kcommon.cuh"

namespace fmp {
namespace {

template <int R, class V>
__device__ __forceinline__ void wht_regs(V* v) {
#pragma unroll
  for (int s = 0; s < R; ++s) {
#pragma unroll
    for (int j = 0; j < (1 << R); ++j) {
      if (j & (1 << s)) continue;
      const V a = v[j], b = v[j + (1 << s)];
      v[j] = add(a, b);
      v[j + (1 << s)] = sub(a, b);
    }
  }
}

// packed fp32 pairs (Blackwell FADD2: two IEEE adds per instruction)
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(reinterpret_cast<unsigned long long&>(a)), "l"(reinterpret_cast<unsigned long long&>(b)));
  return reinterpret_cast<float2&>(r);
}
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(reinterpret_cast<unsigned long long&>(a)), "l"(reinterpret_cast<unsigned long long&>(b)));
  return reinterpret_cast<float2&>(r);
}

// N elements of one register tile.  The generic tile is a plain array; the
// f32 tile keeps elements 2k, 2k + 1 as one packed pair, so every butterfly
// stage above the first is one FADD2 per two outputs, and the c64 tile adds
// its (re, im) pairs the same way.  get / set take compile-time indices
// (callers unroll), so everything stays in registers.
template <class V, int N>
struct Tile {
  V v[N];
  __device__ __forceinline__ V get(int j) const { return v[j]; }
  __device__ __forceinline__ void set(int j, V x) { v[j] = x; }
  template <int R>
  __device__ __forceinline__ void wht() { wht_regs<R>(v); }
};
template <int N>
struct Tile<float2, N> {
  float2 v[N];
  __device__ __forceinline__ float2 get(int j) const { return v[j]; }
  __device__ __forceinline__ void set(int j, float2 x) { v[j] = x; }
  template <int R>
  __device__ __forceinline__ void wht() {
#pragma unroll
    for (int s = 0; s < R; ++s) {
#pragma unroll
      for (int j = 0; j < (1 << R); ++j) {
        if (j & (1 << s)) continue;
        const float2 a = v[j], b = v[j + (1 << s)];
        v[j] = add2(a, b);
        v[j + (1 << s)] = sub2(a, b);
      }
    }
  }
};
template <int N>
struct Tile<float, N> {
  float2 p[N / 2];
  __device__ __forceinline__ float get(int j) const { return (j & 1) ? p[j >> 1].y : p[j >> 1].x; }
  __device__ __forceinline__ void set(int j, float x) {
    if (j & 1) p[j >> 1].y = x;
    else p[j >> 1].x = x;
  }
  template <int R>
  __device__ __forceinline__ void wht() {
#pragma unroll
    for (int k = 0; k < (1 << R) / 2; ++k) {
      const float a = p[k].x, b = p[k].y;
      p[k].x = a + b;
      p[k].y = a - b;
    }
#pragma unroll
    for (int s = 1; s < R; ++s) {
#pragma unroll
      for (int k = 0; k < (1 << R) / 2; ++k) {
        if (k & (1 << (s - 1))) continue;
        const float2 a = p[k], b = p[k + (1 << (s - 1))];
        p[k] = add2(a, b);
        p[k + (1 << (s - 1))] = sub2(a, b);
      }
    }
  }
};

__device__ __forceinline__ void st_stream(double* p, double v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(float* p, float v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(float2* p, float2 v) { __stcs(p, v); }

// one register-tile pass over bits [LO, LO + R) of the padded buffer z; the
// last pass scales and streams its block to global memory instead
template <class V, int LOGB, int R1, int LO, int R, int NTH, bool LAST>
__device__ __forceinline__ void fold_pass(V* z, V* __restrict__ out, double sc, int tid) {
  constexpr int G = 1 << (LOGB - R);
#pragma unroll 1
  for (int g = tid; g < G; g += NTH) {
    const int gl = g & ((1 << LO) - 1), gh = g >> LO;
    const int base = (gh << (LO + R)) + gl;
    // LO >= R1: element j sits (j << LO) + (j << (LO - R1)) padded slots
    // after the group's first (compile-time offsets)
    static_assert(LO >= R1, "pass bits start above the row bits");
    V* zp = z + base + (base >> R1);
    Tile<V, 1 << R> v;
#pragma unroll
    for (int j = 0; j < (1 << R); ++j) v.set(j, zp[(j << LO) + (j << (LO - R1))]);
    v.template wht<R>();
#pragma unroll
    for (int j = 0; j < (1 << R); ++j) {
      if constexpr (LAST) st_stream(out + base + (j << LO), scale(v.get(j), sc));
      else zp[(j << LO) + (j << (LO - R1))] = v.get(j);
    }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* mb, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(mb)), "r"(parity)
        : "memory");
  } while (!ok);
}
// one bulk (TMA) copy global -> shared, completion counted on `mb`
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* mb) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(mb))
      : "memory");
}

// Persistent: CTA c takes vectors c, c + grid, ...  Per vector, r is staged
// in shared memory once (bulk copy; the next vector's copy is issued while
// the last output block's passes 2-3 still run) and the S output blocks are
// produced one after the other.  Thread g owns row g (32 consecutive i_lo)
// during the fold: its rows of Omega come from the operator's fold table in
// (position, input block) order, so every position's sum is formed in a
// register in ascending i_hi order (deterministic) and the first register
// pass (bits 0-4) follows without touching shared memory.
template <class V, int LOGB, int R2, int R3, int NTH, int NZ>
__global__ void __launch_bounds__(NTH, 1) k_wht_fold(const uint32_t* __restrict__ tab,
                                                     const uint32_t* __restrict__ roff, int m,
                                                     int log2n, const V* __restrict__ in,
                                                     V* __restrict__ out, int64_t batch, double sc,
                                                     int use_bulk) {
  constexpr int R1 = 5;
  static_assert(R1 + R2 + R3 == LOGB && NTH == (1 << (LOGB - R1)), "pass widths");
  constexpr int B = 1 << LOGB;
  constexpr int ZN = B + (B >> R1);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t mbar;
  V* z = reinterpret_cast<V*>(smem_raw);                            // NZ blocks
  // use_bulk: 1 = r staged by a bulk copy, 0 = by plain loads, 2 = r read
  // in place through L1 (8-byte elements: no room beside the block buffer)
  const bool rglob = use_bulk == 2;
  // use_bulk >= 4: as use_bulk - 4, with the fold table read in place
  // (through L1) instead of staged, which leaves room to stage r
  const bool tglob = use_bulk >= 4;
  if (tglob) use_bulk -= 4;
  V* rb = z + NZ * ZN;                                              // m values
  const uint32_t* tb = tglob ? tab : reinterpret_cast<uint32_t*>(rb + (rglob ? 0 : ((m + 3) & ~3)));
  const int tid = threadIdx.x;
  const int S = 1 << (log2n - LOGB);
  const uint32_t rbytes = (uint32_t)m * (uint32_t)sizeof(V);
  int64_t b = blockIdx.x;
  if (b >= batch) return;
  if (rglob) use_bulk = 0;
  if (tid == 0 && use_bulk) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (!tglob) {
    uint32_t* ts = reinterpret_cast<uint32_t*>(rb + (rglob ? 0 : ((m + 3) & ~3)));  // m entries
    for (int k = tid; k < m; k += NTH) ts[k] = tab[k];
  }
  const uint32_t e0 = roff[tid], e1 = roff[tid + 1];
  __syncthreads();
  if (use_bulk) {
    if (tid == 0) bulk_load(rb, in + b * m, rbytes, &mbar);
  } else if (!rglob) {
    for (int k = tid; k < m; k += NTH) rb[k] = in[b * m + k];
    __syncthreads();
  }
  const V zero = zero_of(V{});
  for (uint32_t it = 0; b < batch; b += gridDim.x, ++it) {
    if (use_bulk) mbar_wait(&mbar, it & 1);
    V* ob = out + b * ((int64_t)S << LOGB);
    const V* rv = rglob ? in + b * m : rb;
    // NZ output blocks per walk of the fold table: block khi0 + q takes the
    // sign (-1)^popc((khi0 + q) & i_hi), i.e. that of khi0 flipped by the
    // parity of i_hi & q (khi0 is a multiple of NZ)
    for (int khi0 = 0; khi0 < S; khi0 += NZ) {
      // entries of row tid in (position, input block) order: one running sum
      // per position and block, stored when the position changes; positions
      // without rows read as zero through `seen` (no zero fill)
      uint32_t seen = 0, jc = 32;
      V acc[NZ];
#pragma unroll
      for (int q = 0; q < NZ; ++q) acc[q] = zero;
      const uint32_t neg_mask = (uint32_t)khi0;
      for (uint32_t e = e0; e < e1; e += 4) {
        uint32_t u[4];
        V x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = e + q < e1 ? tb[e + q] : 0xffffffffu;
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = u[q] != 0xffffffffu ? rv[u[q] & 0xfffffu] : zero;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (u[q] == 0xffffffffu) break;
          const uint32_t j = u[q] >> 26;
          if (j != jc) {
            if (jc < 32) {
#pragma unroll
              for (int w = 0; w < NZ; ++w) z[w * ZN + tid * 33 + jc] = acc[w];
            }
#pragma unroll
            for (int w = 0; w < NZ; ++w) acc[w] = zero;
            jc = j;
            seen |= 1u << j;
          }
          const uint32_t ih = (u[q] >> 20) & 63u;
          const uint32_t par = __popc(ih & neg_mask) & 1;
#pragma unroll
          for (int w = 0; w < NZ; ++w)
            acc[w] = ((par ^ (__popc(ih & (uint32_t)w) & 1)) != 0) ? sub(acc[w], x[q]) : add(acc[w], x[q]);
        }
      }
      if (jc < 32) {
#pragma unroll
        for (int w = 0; w < NZ; ++w) z[w * ZN + tid * 33 + jc] = acc[w];
      }
#pragma unroll
      for (int w = 0; w < NZ; ++w) {
        V* row = z + w * ZN + tid * 33;
        V v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = (seen >> j) & 1 ? row[j] : zero;
        wht_regs<R1>(v);
#pragma unroll
        for (int j = 0; j < 32; ++j) row[j] = v[j];
      }
      __syncthreads();
      if (khi0 + NZ >= S) {
        // every read of this vector's r is done: stage the next one
        const int64_t nb = b + gridDim.x;
        if (nb < batch) {
          if (use_bulk) {
            if (tid == 0) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              bulk_load(rb, in + nb * m, rbytes, &mbar);
            }
          }
        }
      }
#pragma unroll
      for (int w = 0; w < NZ; ++w) {
        V* zw = z + w * ZN;
        V* o = ob + ((int64_t)(khi0 + w) << LOGB);
        if constexpr (R3 == 0) {
          fold_pass<V, LOGB, R1, R1, R2, NTH, true>(zw, o, sc, tid);
        } else {
          fold_pass<V, LOGB, R1, R1, R2, NTH, false>(zw, o, sc, tid);
          __syncthreads();
          fold_pass<V, LOGB, R1, R1 + R2, R3, NTH, true>(zw, o, sc, tid);
        }
      }
      __syncthreads();
    }
    if (!use_bulk && !rglob) {
      const int64_t nb = b + gridDim.x;
      if (nb < batch) {
        for (int k = tid; k < m; k += NTH) rb[k] = in[nb * m + k];
        __syncthreads();
      }
    }
  }
}

// Register fold (f32, S = 2^LS <= 8 input blocks).  Thread
// g still owns row g of every block, but walks no table: Omega is ascending,
// so the inputs of row g in input block ih are the contiguous run
// r[rank, rank + popc(mask)) of DevOp::om_wr[ih B/32 + g], whose two words
// per block the thread keeps in registers for the whole launch.  One walk
// visits the S x 32 (block, position) slots with predicated loads and adds
// (no data-dependent control flow, signs known at compile time), forming the
// rows of NZ output blocks in registers, where the first register pass
// follows at once; sums run in ascending input block order like k_wht_fold,
// so the two kernels agree bitwise.
template <class V, int LOGB, int R2, int R3, int NTH, int NZ, int LS>
__global__ void __launch_bounds__(NTH, 1) k_wht_fold_reg(const uint2* __restrict__ om_wr, int m,
                                                         const V* __restrict__ in, V* __restrict__ out,
                                                         int64_t batch, double sc, int use_bulk) {
  constexpr int R1 = 5, S = 1 << LS;
  static_assert(R1 + R2 + R3 == LOGB && NTH == (1 << (LOGB - R1)) && S % NZ == 0, "pass widths");
  constexpr int B = 1 << LOGB;
  constexpr int ZN = B + (B >> R1);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t mbar;
  V* z = reinterpret_cast<V*>(smem_raw);  // NZ blocks
  V* rb = z + NZ * ZN;                    // m values (+ one pad element)
  const int tid = threadIdx.x;
  const uint32_t rbytes = (uint32_t)m * (uint32_t)sizeof(V);
  int64_t b = blockIdx.x;
  if (b >= batch) return;
  if (tid == 0 && use_bulk) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t wd[S], rk[S];
#pragma unroll
  for (int ih = 0; ih < S; ++ih) {
    const uint2 e = om_wr[ih * NTH + tid];
    wd[ih] = e.x;
    rk[ih] = e.y;
  }
  __syncthreads();
  if (use_bulk) {
    if (tid == 0) bulk_load(rb, in + b * m, rbytes, &mbar);
  } else {
    for (int k = tid; k < m; k += NTH) rb[k] = in[b * m + k];
    __syncthreads();
  }
  const V zero = zero_of(V{});
  for (uint32_t it = 0; b < batch; b += gridDim.x, ++it) {
    if (use_bulk) mbar_wait(&mbar, it & 1);
    V* ob = out + b * ((int64_t)S << LOGB);
#pragma unroll
    for (int khi0 = 0; khi0 < S; khi0 += NZ) {
      Tile<V, 32> acc[NZ];
#pragma unroll
      for (int w = 0; w < NZ; ++w)
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[w].set(j, zero);
#pragma unroll
      for (int ih = 0; ih < S; ++ih) {
        const V* rp = rb + rk[ih];
        const uint32_t wdi = wd[ih];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (wdi & (1u << j)) {
            const V x = *rp++;
#pragma unroll
            for (int w = 0; w < NZ; ++w)
              acc[w].set(j, (__builtin_popcount((unsigned)((khi0 + w) & ih)) & 1) ? sub(acc[w].get(j), x)
                                                                                 : add(acc[w].get(j), x));
          }
        }
      }
#pragma unroll
      for (int w = 0; w < NZ; ++w) {
        acc[w].template wht<R1>();
        V* row = z + w * ZN + tid * 33;
#pragma unroll
        for (int j = 0; j < 32; ++j) row[j] = acc[w].get(j);
      }
      __syncthreads();
      if (khi0 + NZ >= S) {
        // every read of this vector's r is done: stage the next one
        const int64_t nb = b + gridDim.x;
        if (nb < batch && use_bulk && tid == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          bulk_load(rb, in + nb * m, rbytes, &mbar);
        }
      }
#pragma unroll
      for (int w = 0; w < NZ; ++w) {
        V* zw = z + w * ZN;
        V* o = ob + ((int64_t)(khi0 + w) << LOGB);
        if constexpr (R3 == 0) {
          fold_pass<V, LOGB, R1, R1, R2, NTH, true>(zw, o, sc, tid);
        } else {
          fold_pass<V, LOGB, R1, R1, R2, NTH, false>(zw, o, sc, tid);
          __syncthreads();
          fold_pass<V, LOGB, R1, R1 + R2, R3, NTH, true>(zw, o, sc, tid);
        }
      }
      __syncthreads();
    }
    if (!use_bulk) {
      const int64_t nb = b + gridDim.x;
      if (nb < batch) {
        for (int k = tid; k < m; k += NTH) rb[k] = in[nb * m + k];
        __syncthreads();
      }
    }
  }
}

template <class V, int LOGB, int R2, int R3, int NZ, int LS>
cudaError_t launch_fold_reg(const TransformArgs& a, cudaStream_t st) {
  const DevOp& op = *a.op;
  constexpr int B = 1 << LOGB, NTH = B >> 5;
  if (!op.om_wr || op.log2n - LOGB != LS || a.batch < 64) return cudaErrorNotSupported;
  const int64_t m = op.m;
  const size_t smem = (size_t)NZ * (B + (B >> 5)) * sizeof(V) + (size_t)((m + 4) & ~3) * sizeof(V);
  if (smem + 1024 > (size_t)smem_optin()) return cudaErrorNotSupported;
  auto kern = k_wht_fold_reg<V, LOGB, R2, R3, NTH, NZ, LS>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = std::min<int64_t>(a.batch, (int64_t)num_sms());
  const bool bulk = ((uintptr_t)a.in % 16 == 0) && ((m * (int64_t)sizeof(V)) % 16 == 0);
  kern<<<(unsigned)grid, NTH, smem, st>>>(op.om_wr, (int)m, (const V*)a.in, (V*)a.out, a.batch,
                                          1.0 / sqrt((double)op.n), bulk ? 1 : 0);
  ++g_launches;
  return cudaGetLastError();
}

// the register fold for the block counts it is built for, else the table walk
template <class V, int LOGB, int R2, int R3, int NZ>
cudaError_t launch_fold_reg_any(const TransformArgs& a, cudaStream_t st) {
  const int ls = a.op->log2n - LOGB;
  const char* fe = getenv("FMP_FOLD");  // FMP_FOLD=4: the table walk (timing tools)
  if (fe && atoi(fe) == 4) return cudaErrorNotSupported;
  if (ls == 1) return launch_fold_reg<V, LOGB, R2, R3, (NZ > 2 ? 2 : NZ), 1>(a, st);
  if (ls == 2) return launch_fold_reg<V, LOGB, R2, R3, NZ, 2>(a, st);
  if (ls == 3) return launch_fold_reg<V, LOGB, R2, R3, NZ, 3>(a, st);
  return cudaErrorNotSupported;
}

template <class V, int LOGB, int R2, int R3, int NZ>
cudaError_t launch_fold_k(const TransformArgs& a, cudaStream_t st) {
  const DevOp& op = *a.op;
  constexpr int B = 1 << LOGB, NTH = B >> 5;
  const int q = LOGB - 11;
  if (q < 0 || q > 3 || !op.fold_tab[q]) return cudaErrorNotSupported;
  // one persistent CTA per vector in flight: small batches keep the job queue
  if (a.batch < 64) return cudaErrorNotSupported;
  const int64_t m = op.m;
  if ((1 << (op.log2n - LOGB)) % NZ) return cudaErrorNotSupported;
  const char* fe = getenv("FMP_FOLD");
  // 8-byte elements: r staged with the table read in place through L1
  // (f64 0.279 -> 0.264 ms, c64 0.289 -> 0.279 ms at config 3), or with
  // FMP_FOLD=2 r read in place and the table staged; c128: r in place
  const bool tglob = sizeof(V) == 8 && !(fe && atoi(fe) == 2);
  const bool rglob = sizeof(V) >= 8 && !tglob;  // r through L1 (see the kernel)
  const size_t smem = (size_t)NZ * (B + (B >> 5)) * sizeof(V) +
                      (rglob ? 0 : (size_t)((m + 3) & ~3) * sizeof(V)) + (tglob ? 0 : (size_t)m * 4);
  if (smem + 1024 > (size_t)smem_optin()) return cudaErrorNotSupported;
  auto kern = k_wht_fold<V, LOGB, R2, R3, NTH, NZ>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NTH, smem);
  const int64_t grid = std::min<int64_t>(a.batch, (int64_t)std::max(1, occ) * num_sms());
  const bool bulk = ((uintptr_t)a.in % 16 == 0) && ((m * (int64_t)sizeof(V)) % 16 == 0);
  kern<<<(unsigned)grid, NTH, smem, st>>>(op.fold_tab[q], op.fold_off[q], (int)m, op.log2n,
                                          (const V*)a.in, (V*)a.out, a.batch,
                                          1.0 / sqrt((double)op.n),
                                          (rglob ? 2 : (bulk ? 1 : 0)) + (tglob ? 4 : 0));
  ++g_launches;
  return cudaGetLastError();
}

// f32: 2^14-point blocks, two per walk of the fold table (smem: 2 x 66 KB +
// r + the table), passes 5 + 5 + 4.  8-byte elements (f64, c64): 2^14-point
// blocks one per walk, r staged and the table read through L1 (no room for
// both; r read through L1 instead measured slower); c128: 2^13-point blocks,
// r through L1.  Config 3 (1024 vectors): f32 0.162 (one block per
// walk) -> 0.126 ms; f64 0.318 (job queue) -> 0.277 ms; c64 0.328 -> 0.287 ms;
// c128 0.826 -> 0.691 ms.  Measured slower: f64 / c64 at 2^13 with two
// blocks per walk (0.327 / 0.341 ms), f32 at 2^13 with one (0.242 ms).
}  // namespace

cudaError_t launch_wht_fold(const TransformArgs& a, cudaStream_t st) {
  const DevOp& op = *a.op;
  if (op.kind != HADAMARD || !a.in_omega || a.out_omega || !a.out) return cudaErrorNotSupported;
  const char* e = getenv("FMP_FOLD");  // FMP_FOLD=-1: job queue instead (timing tools)
  if (e && atoi(e) < 0) return cudaErrorNotSupported;
  const int plan = e ? atoi(e) : 0;
  if (a.dtype == F32) {
    // register fold (no table walk), when built for this block count.  f32
    // only: with 8-byte elements one walk feeds a single output block and
    // the 32-element accumulator tile spills (config 3: f64 0.39 vs 0.26 ms,
    // c64 0.40 vs 0.27 ms for the table walk)
    const cudaError_t r = launch_fold_reg_any<float, 14, 5, 4, 2>(a, st);
    if (r != cudaErrorNotSupported) return r;
  }
  if (a.dtype == F32) {
    if (plan != 1) {  // FMP_FOLD=1: one block per walk (timing tools)
      const cudaError_t r = launch_fold_k<float, 14, 5, 4, 2>(a, st);
      if (r != cudaErrorNotSupported) return r;
    }
    return launch_fold_k<float, 14, 5, 4, 1>(a, st);
  }
  if (a.dtype == F64) return launch_fold_k<double, 14, 5, 4, 1>(a, st);
  if (a.dtype == C64) return launch_fold_k<float2, 14, 5, 4, 1>(a, st);
  if (a.dtype == C128) return launch_fold_k<double2, 13, 4, 4, 1>(a, st);
  return cudaErrorNotSupported;
}

}  // namespace fmp
