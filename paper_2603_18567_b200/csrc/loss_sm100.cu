// loss_sm100.cu — masked soft-label log-softmax loss and its in-place backward
// (Alg. 3; §4.2.1 "Memory-Efficient Gradient Computation",
// PAPER.md:338-340). C-ABI in include/ttt_loss.h; readings R17-R20 in DESIGN.md.
//
// HBM-bound row kernels. Every thread of a 512-thread CTA holds its NV 16-byte
// vectors of one row's z and p in registers; the row statistics (max, sum of
// exp, sum p, sum p z) are reduced warp -> CTA (-> cluster through DSMEM when a
// row needs several CTAs), in a fixed order so every CTA holds bit-identical
// statistics, and the gradient of Alg. 3 is written straight from the registers
// over z. Rows of <= 64 KB per tensor take the persistent ttt_loss_ring_kernel
// (the next row bulk-copied into smem under the current row's math); larger rows
// one row per CTA / cluster (ttt_loss_kernel). Bytes per row: read z, read p,
// write grad (fused mode) — the minimum for an in-place backward; nothing of size
// [N][V] is allocated.
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "../../include/ttt_loss.h"
#include "ptx_sm100.cuh"
#include "ttt_params.cuh"

namespace cg = cooperative_groups;

namespace tttk {
namespace {

#ifndef TTT_LOSS_THREADS
#define TTT_LOSS_THREADS 512
#endif
constexpr int kLossThreads = TTT_LOSS_THREADS;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

enum : int { kModeLoss = 1, kModeGrad = 2 };

struct LossParams {
  const void* z;
  const void* p;
  void* grad;             // == z for in place
  const uint8_t* mask;    // NULL = all rows
  const float* g_rows;    // NULL = 1
  float* lse;             // NULL = not written
  float* row_loss;        // workspace [rows] (loss mode)
  const int* count;       // workspace: masked-row count (MEAN)
  int64_t rows;
  int vocab;
  int cs;                 // CTAs per row (cluster size)
  float g_scale;
  int mode;
  int mean;
};

// ---- element access: a "vector" is E elements of T held in registers ----
template <typename T, int E>
struct VecT;
template <>
struct VecT<__nv_bfloat16, 8> {
  using type = uint4;
};
template <>
struct VecT<float, 4> {
  using type = uint4;
};
template <>
struct VecT<__nv_bfloat16, 1> {
  using type = __nv_bfloat16;
};
template <>
struct VecT<float, 1> {
  using type = float;
};

__device__ __forceinline__ float elem(const __nv_bfloat16& v, int, __nv_bfloat16*) { return __bfloat162float(v); }
__device__ __forceinline__ float elem(const float& v, int, float*) { return v; }

// k-th pair of elements of a 16-byte vector as fp32 (bf16 -> fp32 is exact: a shift / mask)
__device__ __forceinline__ void pair(const uint4& v, int k, __nv_bfloat16*, float& lo, float& hi) {
  const uint32_t w = (&v.x)[k];
  lo = __uint_as_float(w << 16);
  hi = __uint_as_float(w & 0xffff0000u);
}
__device__ __forceinline__ void pair(const uint4& v, int k, float*, float& lo, float& hi) {
  lo = __uint_as_float((&v.x)[2 * k]);
  hi = __uint_as_float((&v.x)[2 * k + 1]);
}
__device__ __forceinline__ float vec_max(const uint4& v, float m, __nv_bfloat16*) {
  uint32_t a, b;  // bf16x2 maxima (exact), then one fp32 max3 over the four candidates' pairs
  asm("max.bf16x2 %0, %1, %2;" : "=r"(a) : "r"(v.x), "r"(v.y));
  asm("max.bf16x2 %0, %1, %2;" : "=r"(b) : "r"(v.z), "r"(v.w));
  asm("max.bf16x2 %0, %0, %1;" : "+r"(a) : "r"(b));
  return fmax3(m, __uint_as_float(a << 16), __uint_as_float(a & 0xffff0000u));
}
__device__ __forceinline__ float vec_max(const uint4& v, float m, float*) {
  return fmax3(fmax3(m, __uint_as_float(v.x), __uint_as_float(v.y)), __uint_as_float(v.z), __uint_as_float(v.w));
}

__device__ __forceinline__ uint4 ld_stream(const uint4* a) { return __ldcs(a); }
__device__ __forceinline__ float ld_stream(const float* a) { return __ldcs(a); }
__device__ __forceinline__ __nv_bfloat16 ld_stream(const __nv_bfloat16* a) {
  unsigned short u;
  asm volatile("ld.global.cs.u16 %0, [%1];" : "=h"(u) : "l"(a));
  return __ushort_as_bfloat16(u);
}

// pack E gradient values into the storage vector (RNE for bf16)
template <typename T, int E>
struct Pack;
template <>
struct Pack<__nv_bfloat16, 8> {
  __device__ __forceinline__ static void store(void* dst, const float* g) {
    uint4 o;
    uint32_t* w = &o.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(g[2 * i], g[2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    __stcs(reinterpret_cast<uint4*>(dst), o);
  }
};
template <>
struct Pack<float, 4> {
  __device__ __forceinline__ static void store(void* dst, const float* g) {
    __stcs(reinterpret_cast<float4*>(dst), make_float4(g[0], g[1], g[2], g[3]));
  }
};
template <>
struct Pack<__nv_bfloat16, 1> {
  __device__ __forceinline__ static void store(void* dst, const float* g) {
    __nv_bfloat16 h = __float2bfloat16_rn(g[0]);
    asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(dst), "h"(__bfloat16_as_ushort(h)) : "memory");
  }
};
template <>
struct Pack<float, 1> {
  __device__ __forceinline__ static void store(void* dst, const float* g) { __stcs(reinterpret_cast<float*>(dst), g[0]); }
};

// Row statistics in the log2 domain: m = max_v z_v log2e, l = sum_v 2^(z_v log2e - m),
// sp = sum_v p_v, spz = sum_v p_v z_v.
struct Stats {
  float m, l, sp, spz;
};
__device__ __forceinline__ Stats combine(Stats a, Stats b) {
  const float M = fmaxf(a.m, b.m);
  Stats r;
  r.m = M;
  r.l = (M == -INFINITY) ? 0.f : a.l * ex2(a.m - M) + b.l * ex2(b.m - M);
  r.sp = a.sp + b.sp;
  r.spz = a.spz + b.spz;
  return r;
}
__device__ __forceinline__ Stats shfl_xor(Stats s, int o) {
  Stats r;
  r.m = __shfl_xor_sync(0xffffffffu, s.m, o);
  r.l = __shfl_xor_sync(0xffffffffu, s.l, o);
  r.sp = __shfl_xor_sync(0xffffffffu, s.sp, o);
  r.spz = __shfl_xor_sync(0xffffffffu, s.spz, o);
  return r;
}

template <typename T, int E, int NV>
__device__ __forceinline__ void load_row(const LossParams& P, int64_t row, int base, int nvec,
                                         typename VecT<T, E>::type (&zv)[NV], typename VecT<T, E>::type (&pv)[NV]) {
  using V = typename VecT<T, E>::type;
  const size_t row_off = (size_t)row * (size_t)P.vocab;
  const V* zrow = reinterpret_cast<const V*>(static_cast<const T*>(P.z) + row_off);
  const V* prow = reinterpret_cast<const V*>(static_cast<const T*>(P.p) + row_off);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int idx = base + i * kLossThreads;
    if (idx < nvec) {
      zv[i] = ld_stream(zrow + idx);
      pv[i] = ld_stream(prow + idx);
    }
  }
}

// One row: thread-local statistics -> warp -> cluster (every warp of every CTA combines all
// warp partials of the cluster in the same fixed order, so all hold bit-identical row
// statistics) -> loss / Alg. 3 gradient from the registers.
template <typename T, int E, int NV>
__device__ __forceinline__ void process_row(const LossParams& P, int64_t row, int base, int nvec, int rank,
                                            const typename VecT<T, E>::type (&zv)[NV],
                                            const typename VecT<T, E>::type (&pv)[NV], Stats* parts) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int cs = P.cs;
  (void)cs;
  // 1. thread-local statistics (packed fp32x2 math, MUFU ex2)
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < NV; ++i)
    if (base + i * kLossThreads < nvec) {
      if constexpr (E > 1) {
        m = vec_max(zv[i], m, (T*)nullptr);
      } else {
        m = fmaxf(m, elem(zv[i], 0, (T*)nullptr));
      }
    }
  const float m2 = m * kLog2e;
  Stats st{m2, 0.f, 0.f, 0.f};
  if constexpr (E > 1) {
    const uint64_t l2e = f2pack(kLog2e, kLog2e), nm2 = f2pack(-m2, -m2);
    uint64_t l = 0, sp = 0, spz = 0;
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (base + i * kLossThreads < nvec) {
#pragma unroll
        for (int k = 0; k < E / 2; ++k) {
          float z0, z1, p0, p1, t0, t1;
          pair(zv[i], k, (T*)nullptr, z0, z1);
          pair(pv[i], k, (T*)nullptr, p0, p1);
          const uint64_t zz = f2pack(z0, z1), pp = f2pack(p0, p1);
          f2unpack(ffma2(zz, l2e, nm2), t0, t1);
          l = fadd2(l, f2pack(ex2(t0), ex2(t1)));
          sp = fadd2(sp, pp);
          spz = ffma2(pp, zz, spz);
        }
      }
    float a, b;
    f2unpack(l, a, b);
    st.l = a + b;
    f2unpack(sp, a, b);
    st.sp = a + b;
    f2unpack(spz, a, b);
    st.spz = a + b;
  } else {
#pragma unroll
    for (int i = 0; i < NV; ++i)
      if (base + i * kLossThreads < nvec) {
        const float zz = elem(zv[i], 0, (T*)nullptr);
        const float pp = elem(pv[i], 0, (T*)nullptr);
        st.l += ex2(fmaf(zz, kLog2e, -m2));
        st.sp += pp;
        st.spz = fmaf(pp, zz, st.spz);
      }
  }

  // 2. warp partials -> smem -> (cluster barrier) -> every warp combines all partials
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) st = combine(st, shfl_xor(st, o));
  constexpr int kWarps = kLossThreads / 32;
  if (lane == 0) parts[tid >> 5] = st;
  Stats rs{-INFINITY, 0.f, 0.f, 0.f};
  if (cs > 1) {
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    for (int k = lane; k < cs * kWarps; k += 32) rs = combine(rs, *cl.map_shared_rank(parts + (k % kWarps), k / kWarps));
  } else {
    __syncthreads();
    if (lane < kWarps) rs = parts[lane];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) rs = combine(rs, shfl_xor(rs, o));
  const float lse2 = rs.m + log2f(rs.l);  // log2 of sum_v exp(z_v)
  const bool on = P.mask == nullptr || P.mask[row] != 0;

  if ((P.mode & kModeLoss) && rank == 0 && tid == 0) {
    const float lse = lse2 * kLn2;
    // row loss = -sum_v p_v (z_v - lse) = lse * sum p - sum p z
    P.row_loss[row] = on ? fmaf(lse, rs.sp, -rs.spz) : 0.f;
    if (P.lse) P.lse[row] = lse;
  }

  if (P.mode & kModeGrad) {
    // upstream gradient of this row (reading R19) and Alg. 3's s = sum_v p_v g
    float g = 0.f;
    if (on) {
      g = P.g_scale * (P.g_rows ? P.g_rows[row] : 1.f);
      if (P.mean) {
        const int n = *P.count;
        g = n > 0 ? g / (float)n : 0.f;
      }
    }
    const float s = rs.sp * g;
    T* grow = static_cast<T*>(P.grad) + (size_t)row * (size_t)P.vocab;
    // Alg. 3: pi <- softmax(z) = 2^(z log2e - lse2); z <- -(p g - pi s) = fl(pi s + p (-g))
    // (RNE is sign-symmetric, so this is bit-identical to negating fl(p g - pi s))
    if constexpr (E > 1) {
      const uint64_t l2e = f2pack(kLog2e, kLog2e), nl = f2pack(-lse2, -lse2);
      const uint64_t s2 = f2pack(s, s), ng2 = f2pack(-g, -g);
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int idx = base + i * kLossThreads;
        if (idx < nvec) {
          float out[E];
#pragma unroll
          for (int k = 0; k < E / 2; ++k) {
            float z0, z1, p0, p1, t0, t1;
            pair(zv[i], k, (T*)nullptr, z0, z1);
            pair(pv[i], k, (T*)nullptr, p0, p1);
            f2unpack(ffma2(f2pack(z0, z1), l2e, nl), t0, t1);
            const uint64_t npg = fmul2(f2pack(p0, p1), ng2);
            f2unpack(ffma2(f2pack(ex2(t0), ex2(t1)), s2, npg), out[2 * k], out[2 * k + 1]);
          }
          Pack<T, E>::store(grow + (size_t)idx * E, out);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int idx = base + i * kLossThreads;
        if (idx < nvec) {
          const float zz = elem(zv[i], 0, (T*)nullptr);
          const float pp = elem(pv[i], 0, (T*)nullptr);
          const float pi = ex2(fmaf(zz, kLog2e, -lse2));
          float out[1] = {fmaf(pi, s, pp * -g)};
          Pack<T, E>::store(grow + (size_t)idx, out);
        }
      }
    }
  }
}

// One row per CTA or cluster of CS CTAs (grid = rows x CS), for rows the ring kernel does not
// take (odd vocab, or > 64 KB per tensor). A persistent variant that kept the next row in a
// second register set measured slower (894 vs 690 us at the bench shape: 2 CTAs / SM at 128
// registers); the smem-staged ring kernel below is the persistent form that paid off.
template <typename T, int E, int NV>
__global__ void __launch_bounds__(kLossThreads, (NV <= 4 ? 65536 / (kLossThreads * 64) : 1)) ttt_loss_kernel(const LossParams P) {
  using V = typename VecT<T, E>::type;
  __shared__ Stats parts[kLossThreads / 32];
  const int cs = P.cs;
  const int rank = cs > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const int nvec = P.vocab / E;
  const int base = rank * NV * kLossThreads + threadIdx.x;
  const int64_t row = blockIdx.x / cs;
  V zv[NV], pv[NV];
  load_row<T, E, NV>(P, row, base, nvec, zv, pv);
  process_row<T, E, NV>(P, row, base, nvec, rank, zv, pv, parts);
  if (cs > 1) cg::this_cluster().sync();  // no CTA leaves while its partials may still be read
}

// Persistent variant for rows that fit one CTA (z and p rows <= 64 KB each): the next row is
// bulk-copied (cp.async.bulk, mbarrier completion) into shared memory while the current row is
// reduced and written from registers, then moved smem -> registers in one conflict-free pass
// and the row after it is requested. HBM reads stay in flight across row boundaries (the
// one-row-per-CTA kernel leaves an SM's memory pipe idle from its last load to the next CTA's
// first). 128 KB of smem + 128 registers: one 512-thread CTA per SM.
template <typename T, int E, int NV>
__global__ void __launch_bounds__(kLossThreads, 1) ttt_loss_ring_kernel(const LossParams P) {
  using V = typename VecT<T, E>::type;
  static_assert(E > 1, "vector path only");
  __shared__ Stats parts[kLossThreads / 32];
  __shared__ __align__(8) uint64_t landed;
  extern __shared__ __align__(128) uint8_t ring[];  // [z row | p row], each padded to 16 B
  const int nvec = P.vocab / E;
  const uint32_t row_bytes = (uint32_t)P.vocab * (uint32_t)sizeof(T);
  V* sz = reinterpret_cast<V*>(ring);
  V* sp = reinterpret_cast<V*>(ring + row_bytes);
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&landed, 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto request = [&](int64_t row) {  // one thread
    mbar_expect_tx(&landed, 2 * row_bytes);
    bulk_load(sz, static_cast<const T*>(P.z) + (size_t)row * P.vocab, row_bytes, &landed);
    bulk_load(sp, static_cast<const T*>(P.p) + (size_t)row * P.vocab, row_bytes, &landed);
  };
  int64_t row = blockIdx.x;
  if (row >= P.rows) return;
  if (tid == 0) request(row);
  V zv[NV], pv[NV];
  uint32_t phase = 0;
  while (row < P.rows) {
    mbar_wait(&landed, phase);
    phase ^= 1u;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int idx = tid + i * kLossThreads;
      if (idx < nvec) {
        zv[i] = sz[idx];
        pv[i] = sp[idx];
      }
    }
    __syncthreads();  // the ring is free: every thread holds its share of this row
    const int64_t next = row + gridDim.x;
    if (tid == 0 && next < P.rows) request(next);
    process_row<T, E, NV>(P, row, tid, nvec, 0, zv, pv, parts);
    row = next;
  }
}

// Masked-row count for TTT_LOSS_MEAN (one CTA; fixed order).
__global__ void __launch_bounds__(1024) ttt_loss_count_kernel(const uint8_t* mask, int64_t rows, int* count) {
  __shared__ int part[32];
  int c = 0;
  for (int64_t r = threadIdx.x; r < rows; r += blockDim.x) c += (mask == nullptr || mask[r] != 0) ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
    *count = t;
  }
}

// stats = {sum of masked row losses / n, n}: fp64, per-thread strided sums then a fixed tree.
__global__ void __launch_bounds__(1024) ttt_loss_finalize_kernel(const float* row_loss, const uint8_t* mask,
                                                                 int64_t rows, double* stats) {
  __shared__ double sh_sum[1024];
  __shared__ int sh_n[1024];
  double s = 0.0;
  int n = 0;
  for (int64_t r = threadIdx.x; r < rows; r += 1024) {
    s += (double)row_loss[r];
    n += (mask == nullptr || mask[r] != 0) ? 1 : 0;
  }
  sh_sum[threadIdx.x] = s;
  sh_n[threadIdx.x] = n;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) {
      sh_sum[threadIdx.x] += sh_sum[threadIdx.x + w];
      sh_n[threadIdx.x] += sh_n[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int nn = sh_n[0];
    stats[0] = nn > 0 ? sh_sum[0] / (double)nn : __longlong_as_double(0x7ff8000000000000ll);
    stats[1] = (double)nn;
  }
}

struct LossWs {
  size_t row_loss, count, total;
};
LossWs loss_ws_layout(int64_t rows) {
  LossWs w{};
  w.row_loss = 0;
  w.count = ((size_t)rows * 4 + 255) / 256 * 256;
  w.total = w.count + 256;
  return w;
}

int validate_loss(const ttt_loss_desc* d) {
  if (!d) return TTT_ERR_INVALID_ARG;
  if (d->rows < 1 || d->vocab < 2) return TTT_ERR_INVALID_ARG;
  if (d->dtype != TTT_BF16 && d->dtype != TTT_FP32_CHECK) return TTT_ERR_INVALID_ARG;
  if ((double)d->rows * (double)d->vocab >= 1099511627776.0) return TTT_ERR_UNSUPPORTED;
  if (d->rows * 8 > (int64_t)INT32_MAX) return TTT_ERR_UNSUPPORTED;  // grid.x = rows * cs
  return TTT_OK;
}

// Launch shape: elements per vector E, vectors per thread NV, CTAs per row CS.
struct LossShape {
  int e, nv, cs;
};
bool loss_shape(const ttt_loss_desc* d, bool vec_ok, LossShape* s) {
  // Fewest CTAs per row wins (measured at 16384 x 32000 bf16, bench_tools/time_loss.py:
  // 256 thr x 4 vec x 4-CTA cluster 709 us, 512 x 4 x 2-CTA 667 us, 512 x 8 x 1 CTA 597 us):
  // the cluster barrier per row costs more than the occupancy it buys. So: the smallest
  // NV in {1, 4, 8} that fits one CTA, else clusters of 2..8 CTAs at NV = 8.
  const int esz = d->dtype == TTT_BF16 ? 2 : 4;
  s->e = vec_ok ? 16 / esz : 1;
  const int nvec = d->vocab / s->e;
  const int nvs[3] = {1, 4, 8};
  for (int k = 0; k < 3; ++k)
    if (nvec <= nvs[k] * kLossThreads) {
      s->nv = nvs[k];
      s->cs = 1;
      return true;
    }
  int cs = 2;
  while (cs * 8 * kLossThreads < nvec && cs < 8) cs *= 2;
  if (cs * 8 * kLossThreads < nvec) return false;
  s->nv = 8;
  s->cs = cs;
  return true;
}

bool aligned16(const void* a) { return (reinterpret_cast<uintptr_t>(a) & 15u) == 0; }

template <typename T, int E, int NV>
cudaError_t launch_loss_t(LossParams P, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(P.rows * P.cs), 1, 1);
  cfg.blockDim = dim3(kLossThreads, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = P.cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, ttt_loss_kernel<T, E, NV>, P);
}

template <typename T, int E, int NV>
cudaError_t launch_loss_ring_t(const LossParams& P, cudaStream_t st) {
  const int smem = 2 * ((P.vocab * (int)sizeof(T) + 15) & ~15);
  static std::atomic<unsigned long long> attr_done{0};  // per device
  {
    cudaError_t e = set_smem_attr(ttt_loss_ring_kernel<T, E, NV>, 2 * 65536, attr_done);
    if (e != cudaSuccess) return e;
  }
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = P.rows < (int64_t)sms ? P.rows : (int64_t)sms;
  ttt_loss_ring_kernel<T, E, NV><<<(unsigned)grid, kLossThreads, smem, st>>>(P);
  return cudaGetLastError();
}

template <typename T, int E>
cudaError_t launch_loss_e(const LossParams& P, int nv, cudaStream_t st) {
#ifndef TTT_LOSS_NO_RING
  if constexpr (E > 1) {
    if (P.cs == 1 && nv == 8 && P.vocab * (int)sizeof(T) <= 65536) return launch_loss_ring_t<T, E, 8>(P, st);
  }
#endif
  switch (nv) {
    case 1: return launch_loss_t<T, E, 1>(P, st);
    case 4: return launch_loss_t<T, E, 4>(P, st);
    default: return launch_loss_t<T, E, 8>(P, st);
  }
}

int run_loss(const ttt_loss_desc* d, const void* z, const void* p, const uint8_t* mask, const float* g_rows,
             float g_scale, unsigned flags, void* grad, float* lse, double* stats, void* ws, size_t ws_bytes,
             void* stream, int mode) {
  int rc = validate_loss(d);
  if (rc != TTT_OK) return rc;
  if (!z || !p || !ws) return TTT_ERR_INVALID_ARG;
  if ((mode & kModeLoss) && !stats) return TTT_ERR_INVALID_ARG;
  if (flags & ~TTT_LOSS_MEAN) return TTT_ERR_INVALID_ARG;
  const LossWs lw = loss_ws_layout(d->rows);
  if (ws_bytes < lw.total) return TTT_ERR_WORKSPACE;
  if (!aligned16(ws)) return TTT_ERR_ALIGNMENT;
  if (grad == nullptr) grad = const_cast<void*>(z);
  const int esz = d->dtype == TTT_BF16 ? 2 : 4;
  const bool vec_ok = ((size_t)d->vocab * esz) % 16 == 0 && aligned16(z) && aligned16(p) && aligned16(grad);
  if (!vec_ok && ((reinterpret_cast<uintptr_t>(z) | reinterpret_cast<uintptr_t>(p) |
                   reinterpret_cast<uintptr_t>(grad)) & (uintptr_t)(esz - 1)))
    return TTT_ERR_ALIGNMENT;
  LossShape sh;
  if (!loss_shape(d, vec_ok, &sh)) return TTT_ERR_UNSUPPORTED;

  char* wsb = static_cast<char*>(ws);
  LossParams P{};
  P.z = z;
  P.p = p;
  P.grad = grad;
  P.mask = mask;
  P.g_rows = g_rows;
  P.lse = lse;
  P.row_loss = reinterpret_cast<float*>(wsb + lw.row_loss);
  P.count = reinterpret_cast<const int*>(wsb + lw.count);
  P.rows = d->rows;
  P.vocab = d->vocab;
  P.cs = sh.cs;
  P.g_scale = g_scale;
  P.mode = mode;
  P.mean = (mode & kModeGrad) && (flags & TTT_LOSS_MEAN) ? 1 : 0;

  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaGetLastError();
  if (P.mean) {
    prof_mark(kKindLossAux, true, st);
    ttt_loss_count_kernel<<<1, 1024, 0, st>>>(mask, d->rows, reinterpret_cast<int*>(wsb + lw.count));
    prof_mark(kKindLossAux, false, st);
  }
  prof_mark(kKindLoss, true, st);
  cudaError_t e;
  if (d->dtype == TTT_BF16)
    e = vec_ok ? launch_loss_e<__nv_bfloat16, 8>(P, sh.nv, st) : launch_loss_e<__nv_bfloat16, 1>(P, sh.nv, st);
  else
    e = vec_ok ? launch_loss_e<float, 4>(P, sh.nv, st) : launch_loss_e<float, 1>(P, sh.nv, st);
  prof_mark(kKindLoss, false, st);
  if (e != cudaSuccess) return TTT_ERR_CUDA;
  if (mode & kModeLoss) {
    prof_mark(kKindLossAux, true, st);
    ttt_loss_finalize_kernel<<<1, 1024, 0, st>>>(P.row_loss, mask, d->rows, stats);
    prof_mark(kKindLossAux, false, st);
  }
  return cudaGetLastError() == cudaSuccess ? TTT_OK : TTT_ERR_CUDA;
}

}  // namespace
}  // namespace tttk

extern "C" {

size_t ttt_loss_workspace_size(const ttt_loss_desc* d) {
  if (tttk::validate_loss(d) != TTT_OK) return 0;
  return tttk::loss_ws_layout(d->rows).total;
}

int ttt_loss_fwd(const ttt_loss_desc* d, const void* z, const void* p, const uint8_t* mask, float* lse,
                 double* stats, void* ws, size_t ws_bytes, void* stream) {
  return tttk::run_loss(d, z, p, mask, nullptr, 1.f, 0u, const_cast<void*>(z), lse, stats, ws, ws_bytes, stream,
                        tttk::kModeLoss);
}

int ttt_loss_bwd_inplace(const ttt_loss_desc* d, void* z, const void* p, const uint8_t* mask, const float* g_rows,
                         float g_scale, unsigned flags, void* grad, void* ws, size_t ws_bytes, void* stream) {
  return tttk::run_loss(d, z, p, mask, g_rows, g_scale, flags, grad, nullptr, nullptr, ws, ws_bytes, stream,
                        tttk::kModeGrad);
}

int ttt_loss_fwd_bwd_inplace(const ttt_loss_desc* d, void* z, const void* p, const uint8_t* mask,
                             const float* g_rows, float g_scale, unsigned flags, void* grad, float* lse,
                             double* stats, void* ws, size_t ws_bytes, void* stream) {
  return tttk::run_loss(d, z, p, mask, g_rows, g_scale, flags, grad, lse, stats, ws, ws_bytes, stream,
                        tttk::kModeLoss | tttk::kModeGrad);
}

}  // extern "C"
