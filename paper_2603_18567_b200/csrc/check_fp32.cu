// check_fp32.cu — TTT_FP32_CHECK mode: the same semantics as the tensor-core
// path on CUDA cores in fp32, used to check mask / GQA / diagonal-fold / lse /
// accumulate semantics at 1e-5 against the fp64 oracle.
// tcgen05 .kind::tf32 has a 10-bit mantissa and cannot meet 1e-5, hence SIMT.
//
// One warp per query row (b, h, r); lanes split head_dim. Streaming (online)
// softmax over the allowed set of Alg. 2 enumerated
// directly: base keys k <= r with k < T_b, then — for r < T_b — the j
// diagonal keys K_i[r] (Alg. 1 "concat s_i").
#include <cuda_runtime.h>

#include "ttt_params.cuh"

namespace tttk {

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <int D>
__global__ void __launch_bounds__(256) fwd_check_kernel(const Params p) {
  constexpr int E = D / 32;
  const int lane = threadIdx.x & 31;
  const long warp = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long rows = (long)p.nrows * p.Hq;
  if (warp >= rows) return;
  // warp -> (head h, row of the [rows][H][D] view) -> (sequence b, position r); padded or packed
  const int grow = (int)(warp % p.nrows);
  const int h = (int)(warp / p.nrows);
  const int b = seq_of_row(p, p.packed, grow);
  const int r = grow - p.row0[b];
  const int g = h / p.G;
  const int T = p.seq_lens[b];
  const float* qrow = (const float*)p.q + ((size_t)grow * p.Hq + h) * D;
  float qv[E], acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    qv[e] = qrow[lane + 32 * e];
    acc[e] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  auto visit = [&](const float* krow, const float* vrow) {
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) s = fmaf(qv[e], krow[lane + 32 * e], s);
    s = warp_sum(s) * p.scale;
    const float mn = fmaxf(m, s);
    const float a = expf(m - mn), w = expf(s - mn);
    l = l * a + w;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = fmaf(w, vrow[lane + 32 * e], acc[e] * a);
    m = mn;
  };
  const size_t kv_stride = (size_t)p.Hkv * D;
  const float* K0 = (const float*)p.k + ((size_t)p.row0[b] * p.Hkv + g) * D;
  const float* V0 = (const float*)p.v + ((size_t)p.row0[b] * p.Hkv + g) * D;
  const int nbase = r < T ? r + 1 : T;
  for (int k = 0; k < nbase; ++k) visit(K0 + k * kv_stride, V0 + k * kv_stride);
  if (r < T) {
    for (int i = 0; i < p.step; ++i) {
      const size_t off = ((size_t)grow * p.Hkv + g) * D;
      visit((const float*)p.ks[i] + off, (const float*)p.vs[i] + off);
    }
  }
  float* orow = (float*)p.out + ((size_t)grow * p.Hq + h) * D;
  const float inv = 1.f / l;
#pragma unroll
  for (int e = 0; e < E; ++e) orow[lane + 32 * e] = acc[e] * inv;
  if (lane == 0) p.lse[lse_at(p, p.packed, b, h, r)] = m + logf(l);
}

template <int D>
__global__ void __launch_bounds__(256) bwd_check_kernel(const Params p) {
  constexpr int E = D / 32;
  const int lane = threadIdx.x & 31;
  const long warp = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long rows = (long)p.nrows * p.Hq;
  if (warp >= rows) return;
  // warp -> (head h, row of the [rows][H][D] view) -> (sequence b, position r); padded or packed
  const int grow = (int)(warp % p.nrows);
  const int h = (int)(warp / p.nrows);
  const int b = seq_of_row(p, p.packed, grow);
  const int r = grow - p.row0[b];
  const int g = h / p.G;
  const int T = p.seq_lens[b];
  const size_t qoff = ((size_t)grow * p.Hq + h) * D;
  const float* qrow = (const float*)p.q + qoff;
  const float* orow = (const float*)p.o + qoff;
  const float* dorow = (const float*)p.dout + qoff;
  float qv[E], dov[E], dq[E];
  float delta = 0.f;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    qv[e] = qrow[lane + 32 * e];
    dov[e] = dorow[lane + 32 * e];
    delta = fmaf(dov[e], orow[lane + 32 * e], delta);
    dq[e] = 0.f;
  }
  delta = warp_sum(delta);  // Delta_r = dO_r . O_r
  const float lse = p.lse_in[lse_at(p, p.packed, b, h, r)];
  // dK / dV contributions of every row meet in fp64 accumulators (workspace): an fp32 sum of up to
  // (rows x heads) terms in arbitrary order would drift past 1e-5 where the terms cancel
  auto visit = [&](const float* krow, const float* vrow, double* dkrow, double* dvrow) {
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      s = fmaf(qv[e], krow[lane + 32 * e], s);
      dp = fmaf(dov[e], vrow[lane + 32 * e], dp);
    }
    s = warp_sum(s) * p.scale;
    dp = warp_sum(dp);
    const float pr = expf(s - lse);         // P = exp(S - lse)
    const float ds = pr * (dp - delta);     // dS = P o (dP - Delta)
#pragma unroll
    for (int e = 0; e < E; ++e) {
      dq[e] = fmaf(p.scale * ds, krow[lane + 32 * e], dq[e]);   // dQ += c dS K
      atomicAdd(dkrow + lane + 32 * e, (double)(p.scale * ds) * (double)qv[e]);  // dK += c dS^T Q
      atomicAdd(dvrow + lane + 32 * e, (double)pr * (double)dov[e]);             // dV += P^T dO
    }
  };
  const size_t kv_stride = (size_t)p.Hkv * D;
  const size_t base = ((size_t)p.row0[b] * p.Hkv + g) * D;
  const float* K0 = (const float*)p.k + base;
  const float* V0 = (const float*)p.v + base;
  const size_t kv_elems = (size_t)p.nrows * p.Hkv * D;
  double* dk0 = p.dacc;
  double* dv0 = p.dacc + kv_elems;
  const int nbase = r < T ? r + 1 : T;
  for (int k = 0; k < nbase; ++k)
    visit(K0 + k * kv_stride, V0 + k * kv_stride, dk0 + base + k * kv_stride, dv0 + base + k * kv_stride);
  if (r < T) {
    const size_t off = ((size_t)grow * p.Hkv + g) * D;
    for (int i = 0; i < p.step; ++i)
      visit((const float*)p.ks[i] + off, (const float*)p.vs[i] + off, p.dacc + (2 + i) * kv_elems + off,
            p.dacc + (2 + p.step + i) * kv_elems + off);
  }
  float* dqrow = (float*)p.dq + qoff;
#pragma unroll
  for (int e = 0; e < E; ++e) dqrow[lane + 32 * e] = dq[e];
}

// dK / dV outputs (+)= fp32(the fp64 accumulators): array a of [dK_0, dV_0, dK_1.., dV_1..]
__global__ void check_dkv_finalize_kernel(const Params p, size_t kv_elems) {
  const size_t n = (size_t)(2 + 2 * p.step) * kv_elems;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int a = (int)(i / kv_elems);
    const size_t e = i - (size_t)a * kv_elems;
    float* dst = a == 0 ? p.dk : a == 1 ? p.dv : a < 2 + p.step ? p.dks[a - 2] : p.dvs[a - 2 - p.step];
    const float v = (float)p.dacc[i];
    dst[e] = p.accumulate ? dst[e] + v : v;
  }
}

size_t check_bwd_ws_bytes(const Params& p) { return (size_t)(2 + 2 * p.step) * p.nrows * p.Hkv * p.D * 8; }

__global__ void zero_f32_kernel(float* __restrict__ x, size_t n) {
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) x[i] = 0.f;
}

cudaError_t launch_zero_f32(float* x, size_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  prof_mark(kKindZero, true, st);
  zero_f32_kernel<<<blocks, 256, 0, st>>>(x, n);
  prof_mark(kKindZero, false, st);
  return cudaGetLastError();
}

cudaError_t launch_fwd_check(const Params& p, cudaStream_t st) {
  const long rows = (long)p.nrows * p.Hq;
  const int blocks = (int)((rows + 7) / 8);
  prof_mark(kKindCheckFwd, true, st);
  if (p.D == 64) fwd_check_kernel<64><<<blocks, 256, 0, st>>>(p);
  else fwd_check_kernel<128><<<blocks, 256, 0, st>>>(p);
  prof_mark(kKindCheckFwd, false, st);
  return cudaGetLastError();
}

// Tree-attention verification, fp32 check path: one warp per (b, node t, head h) row; keys =
// the P_b context rows, then the tree rows of t's ancestors and t itself (walking the parents).
template <int D>
__global__ void __launch_bounds__(256) tree_check_kernel(const Params p) {
  constexpr int E = D / 32;
  const int lane = threadIdx.x & 31;
  const long warp = (long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int n = p.tree_n;
  if (warp >= (long)p.B * n * p.Hq) return;
  const int h = (int)(warp % p.Hq);
  const int t = (int)((warp / p.Hq) % n);
  const int b = (int)(warp / ((long)p.Hq * n));
  const int g = h / p.G;
  const int P = p.seq_lens[b];
  const float* qrow = (const float*)p.q + (((size_t)b * n + t) * p.Hq + h) * D;
  float qv[E], acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    qv[e] = qrow[lane + 32 * e];
    acc[e] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  const size_t kv_stride = (size_t)p.Hkv * D;
  const float* K = (const float*)p.k + ((size_t)b * p.tree_kv_len * p.Hkv + g) * D;
  const float* V = (const float*)p.v + ((size_t)b * p.tree_kv_len * p.Hkv + g) * D;
  auto visit = [&](int k) {
    const float* krow = K + k * kv_stride;
    const float* vrow = V + k * kv_stride;
    float s = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) s = fmaf(qv[e], krow[lane + 32 * e], s);
    s = warp_sum(s) * p.scale;
    const float mn = fmaxf(m, s);
    const float a = expf(m - mn), w = expf(s - mn);
    l = l * a + w;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = fmaf(w, vrow[lane + 32 * e], acc[e] * a);
    m = mn;
  };
  for (int k = 0; k < P; ++k) visit(k);
  const int32_t* par = p.tree_parents + (size_t)b * n;
  int u = t, prev = t + 1;
  while (u >= 0 && u < prev) {  // t, parent(t), ... (a parent index >= the child ends the walk)
    visit(P + u);
    prev = u;
    u = par[u];
  }
  float* orow = (float*)p.out + (((size_t)b * n + t) * p.Hq + h) * D;
  const float inv = 1.f / l;
#pragma unroll
  for (int e = 0; e < E; ++e) orow[lane + 32 * e] = acc[e] * inv;
  if (lane == 0) p.lse[((size_t)b * p.Hq + h) * n + t] = m + logf(l);
}

cudaError_t launch_tree_check(const Params& p, cudaStream_t st) {
  const long rows = (long)p.B * p.Hq * p.tree_n;
  const int blocks = (int)((rows + 7) / 8);
  prof_mark(kKindCheckFwd, true, st);
  if (p.D == 64) tree_check_kernel<64><<<blocks, 256, 0, st>>>(p);
  else tree_check_kernel<128><<<blocks, 256, 0, st>>>(p);
  prof_mark(kKindCheckFwd, false, st);
  return cudaGetLastError();
}

cudaError_t launch_bwd_check(const Params& p, cudaStream_t st) {
  const long rows = (long)p.nrows * p.Hq;
  const int blocks = (int)((rows + 7) / 8);
  cudaError_t e = cudaMemsetAsync(p.dacc, 0, check_bwd_ws_bytes(p), st);
  if (e != cudaSuccess) return e;
  prof_mark(kKindCheckBwd, true, st);
  if (p.D == 64) bwd_check_kernel<64><<<blocks, 256, 0, st>>>(p);
  else bwd_check_kernel<128><<<blocks, 256, 0, st>>>(p);
  prof_mark(kKindCheckBwd, false, st);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const size_t kv_elems = (size_t)p.nrows * p.Hkv * p.D;
  check_dkv_finalize_kernel<<<148 * 8, 256, 0, st>>>(p, kv_elems);
  return cudaGetLastError();
}

}  // namespace tttk
