// rope_sm100.cu — the TTT step's fresh projections into the attention's inputs, one HBM pass:
// qkv [B][L][Hq + 2 Hkv][D] (fused q/k/v projection output) -> q [B][L][Hq][D] and the step's
// K / V slots [B][L][Hkv][D], q and k rotated by rotate-half RoPE at positions 0..L-1 (or given
// ones) — "a TTT step reuses position ids 0..T_pad-1" (
// DESIGN.md R23-R25). C-ABI ttt_qkv_rope_split in include/ttt_attn.h.
//
// HBM-bound: read 2 B and write 2 B per element. The angles are shared by every head of a row,
// so cos / sin come from a table built once per call: theta = pos * base^(-2i/D) in fp64 (it
// reaches 10^4 rad at L = 16K, where an fp32 product would already be off by ~1e-3 rad), reduced
// to [-pi, pi] in fp64, then an fp32 sincosf of the small angle.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/ttt_attn.h"
#include "ttt_params.cuh"

namespace tttk {
namespace {

__global__ void ttt_rope_table_kernel(const int32_t* positions, int rows, int L, int half, double base, float2* table) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * half) return;
  const int r = i / half, f = i - r * half;
  const double pos = positions ? (double)positions[r] : (double)(r % L);
  const double theta = pos * exp2(-2.0 * f / (2.0 * half) * log2(base));
  // reduce to [-pi, pi] in fp64 (theta reaches ~1e4 rad), then an fp32 sincos of the small angle
  const double kTwoPi = 6.283185307179586476925286766559;
  const float red = (float)(theta - kTwoPi * rint(theta / kTwoPi));
  float s, c;
  sincosf(red, &s, &c);
  table[i] = make_float2(c, s);
}

// one CTA per (b, l) row; a thread item = 8 consecutive pair indices i of one head: 16 B of each
// half (32-bit index math only; the row's table entry is shared by all its heads)
__global__ void __launch_bounds__(256) ttt_qkv_rope_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                           const float2* __restrict__ table, int per_seq_table,
                                                           int L, int Hq, int Hkv, int D,
                                                           __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ k,
                                                           __nv_bfloat16* __restrict__ v) {
  const int half = D / 2, cpp = half / 8;  // 8-element chunks per half
  const int H = Hq + 2 * Hkv;
  const size_t bl = blockIdx.x;  // b * L + l
  const float2* trow = table + (per_seq_table ? bl : bl % (size_t)L) * half;
  const __nv_bfloat16* srow = qkv + bl * (size_t)H * D;
  for (int i = threadIdx.x; i < H * cpp; i += blockDim.x) {
    const int h = i / cpp, c = i - h * cpp;
    const __nv_bfloat16* src = srow + h * D + c * 8;
    const uint4 a = *reinterpret_cast<const uint4*>(src);
    const uint4 bb = *reinterpret_cast<const uint4*>(src + half);
    __nv_bfloat16* dst;
    if (h < Hq) dst = q + (bl * Hq + h) * D;
    else if (h < Hq + Hkv) dst = k + (bl * Hkv + (h - Hq)) * D;
    else dst = v + (bl * Hkv + (h - Hq - Hkv)) * D;
    if (h >= Hq + Hkv) {  // V: copied into its slot
      *reinterpret_cast<uint4*>(dst + c * 8) = a;
      *reinterpret_cast<uint4*>(dst + half + c * 8) = bb;
      continue;
    }
    const float2* tb = trow + c * 8;
    const __nv_bfloat162* x1 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* x2 = reinterpret_cast<const __nv_bfloat162*>(&bb);
    uint4 o1, o2;
    __nv_bfloat162* y1 = reinterpret_cast<__nv_bfloat162*>(&o1);
    __nv_bfloat162* y2 = reinterpret_cast<__nv_bfloat162*>(&o2);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 u = __bfloat1622float2(x1[e]), w = __bfloat1622float2(x2[e]);
      const float2 cs0 = tb[2 * e], cs1 = tb[2 * e + 1];
      // x'_i = x_i cos - x_{i+D/2} sin ;  x'_{i+D/2} = x_{i+D/2} cos + x_i sin
      y1[e] = __floats2bfloat162_rn(u.x * cs0.x - w.x * cs0.y, u.y * cs1.x - w.y * cs1.y);
      y2[e] = __floats2bfloat162_rn(w.x * cs0.x + u.x * cs0.y, w.y * cs1.x + u.y * cs1.y);
    }
    *reinterpret_cast<uint4*>(dst + c * 8) = o1;
    *reinterpret_cast<uint4*>(dst + half + c * 8) = o2;
  }
}

// backward of the split: dqkv = [R(-theta) dq | R(-theta) dk | dv] in the fused layout (the
// rotation is orthogonal, so its adjoint is the rotation by -theta); same row-per-CTA layout
__global__ void __launch_bounds__(256) ttt_qkv_rope_join_kernel(const __nv_bfloat16* __restrict__ dq,
                                                                const __nv_bfloat16* __restrict__ dk,
                                                                const __nv_bfloat16* __restrict__ dv,
                                                                const float2* __restrict__ table, int per_seq_table,
                                                                int L, int Hq, int Hkv, int D,
                                                                __nv_bfloat16* __restrict__ dqkv) {
  const int half = D / 2, cpp = half / 8;
  const int H = Hq + 2 * Hkv;
  const size_t bl = blockIdx.x;
  const float2* trow = table + (per_seq_table ? bl : bl % (size_t)L) * half;
  __nv_bfloat16* drow = dqkv + bl * (size_t)H * D;
  for (int i = threadIdx.x; i < H * cpp; i += blockDim.x) {
    const int h = i / cpp, c = i - h * cpp;
    const __nv_bfloat16* src;
    if (h < Hq) src = dq + (bl * Hq + h) * D;
    else if (h < Hq + Hkv) src = dk + (bl * Hkv + (h - Hq)) * D;
    else src = dv + (bl * Hkv + (h - Hq - Hkv)) * D;
    const uint4 a = *reinterpret_cast<const uint4*>(src + c * 8);
    const uint4 bb = *reinterpret_cast<const uint4*>(src + half + c * 8);
    __nv_bfloat16* dst = drow + h * D + c * 8;
    if (h >= Hq + Hkv) {
      *reinterpret_cast<uint4*>(dst) = a;
      *reinterpret_cast<uint4*>(dst + half) = bb;
      continue;
    }
    const float2* tb = trow + c * 8;
    const __nv_bfloat162* g1 = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&bb);
    uint4 o1, o2;
    __nv_bfloat162* y1 = reinterpret_cast<__nv_bfloat162*>(&o1);
    __nv_bfloat162* y2 = reinterpret_cast<__nv_bfloat162*>(&o2);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 u = __bfloat1622float2(g1[e]), w = __bfloat1622float2(g2[e]);
      const float2 cs0 = tb[2 * e], cs1 = tb[2 * e + 1];
      // [dx_i, dx_{i+D/2}] = R(-theta) [dy_i, dy_{i+D/2}]
      y1[e] = __floats2bfloat162_rn(u.x * cs0.x + w.x * cs0.y, u.y * cs1.x + w.y * cs1.y);
      y2[e] = __floats2bfloat162_rn(w.x * cs0.x - u.x * cs0.y, w.y * cs1.x - u.y * cs1.y);
    }
    *reinterpret_cast<uint4*>(dst) = o1;
    *reinterpret_cast<uint4*>(dst + half) = o2;
  }
}

bool a16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace
}  // namespace tttk

extern "C" {

size_t ttt_rope_workspace_size(const ttt_rope_desc* d, int per_sequence_positions) {
  if (!d || d->batch < 1 || d->seq_len < 1 || d->head_dim < 16 || d->head_dim % 16) return 0;
  const size_t rows = per_sequence_positions ? (size_t)d->batch * d->seq_len : (size_t)d->seq_len;
  return (rows * (d->head_dim / 2) * sizeof(float2) + 255) & ~(size_t)255;
}

int ttt_qkv_rope_split(const ttt_rope_desc* d, const void* qkv, const int32_t* positions, void* q, void* k_slot,
                       void* v_slot, void* workspace, size_t workspace_bytes, void* stream) {
  using namespace tttk;
  if (!d || !qkv || !q || !k_slot || !v_slot) return TTT_ERR_INVALID_ARG;
  if (d->batch < 1 || d->seq_len < 1 || d->num_q_heads < 1 || d->num_kv_heads < 1 || !(d->rope_base > 1.f))
    return TTT_ERR_INVALID_ARG;
  if (d->head_dim < 16 || d->head_dim % 16) return TTT_ERR_UNSUPPORTED;
  if ((long long)d->batch * d->seq_len >= (1ll << 31)) return TTT_ERR_UNSUPPORTED;  // one CTA per row
  if (!a16(qkv) || !a16(q) || !a16(k_slot) || !a16(v_slot) || !a16(workspace)) return TTT_ERR_ALIGNMENT;
  const size_t need = ttt_rope_workspace_size(d, positions != nullptr);
  if (!workspace || workspace_bytes < need) return TTT_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int half = d->head_dim / 2;
  const int rows = positions ? d->batch * d->seq_len : d->seq_len;
  float2* table = static_cast<float2*>(workspace);
  cudaGetLastError();
  ttt_rope_table_kernel<<<(rows * half + 255) / 256, 256, 0, st>>>(positions, rows, d->seq_len, half,
                                                                   (double)d->rope_base, table);
  const unsigned rows_bl = (unsigned)(d->batch * d->seq_len);
  ttt_qkv_rope_kernel<<<rows_bl, 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(qkv), table, positions != nullptr, d->seq_len, d->num_q_heads,
      d->num_kv_heads, d->head_dim, static_cast<__nv_bfloat16*>(q), static_cast<__nv_bfloat16*>(k_slot),
      static_cast<__nv_bfloat16*>(v_slot));
  return cudaGetLastError() == cudaSuccess ? TTT_OK : TTT_ERR_CUDA;
}

int ttt_qkv_rope_join_bwd(const ttt_rope_desc* d, const void* dq, const void* dk_slot, const void* dv_slot,
                          const int32_t* positions, void* dqkv, void* workspace, size_t workspace_bytes, void* stream) {
  using namespace tttk;
  if (!d || !dq || !dk_slot || !dv_slot || !dqkv) return TTT_ERR_INVALID_ARG;
  if (d->batch < 1 || d->seq_len < 1 || d->num_q_heads < 1 || d->num_kv_heads < 1 || !(d->rope_base > 1.f))
    return TTT_ERR_INVALID_ARG;
  if (d->head_dim < 16 || d->head_dim % 16) return TTT_ERR_UNSUPPORTED;
  if (!a16(dq) || !a16(dk_slot) || !a16(dv_slot) || !a16(dqkv) || !a16(workspace)) return TTT_ERR_ALIGNMENT;
  const size_t need = ttt_rope_workspace_size(d, positions != nullptr);
  if (!workspace || workspace_bytes < need) return TTT_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int half = d->head_dim / 2;
  const int rows = positions ? d->batch * d->seq_len : d->seq_len;
  float2* table = static_cast<float2*>(workspace);
  cudaGetLastError();
  ttt_rope_table_kernel<<<(rows * half + 255) / 256, 256, 0, st>>>(positions, rows, d->seq_len, half,
                                                                   (double)d->rope_base, table);
  const unsigned rows_bl = (unsigned)(d->batch * d->seq_len);
  ttt_qkv_rope_join_kernel<<<rows_bl, 256, 0, st>>>(
      static_cast<const __nv_bfloat16*>(dq), static_cast<const __nv_bfloat16*>(dk_slot),
      static_cast<const __nv_bfloat16*>(dv_slot), table, positions != nullptr, d->seq_len, d->num_q_heads,
      d->num_kv_heads, d->head_dim, static_cast<__nv_bfloat16*>(dqkv));
  return cudaGetLastError() == cudaSuccess ? TTT_OK : TTT_ERR_CUDA;
}

}  // extern "C"
