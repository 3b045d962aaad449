// ttt_params.cuh — kernel parameter block shared by the launchers (api.cu) and
// the kernels. Passed BY VALUE (kernel params live in constant bank), so a call
// keeps no state in the library.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/ttt_attn.h"

namespace tttk {

constexpr int kTile = 128;  // q-tile rows = kv-tile rows (UMMA M = N = 128)


struct Params {
  int B, L, Hq, Hkv, D, G;  // G = Hq / Hkv (GQA group size, kv head = h / G)
  int step;                 // j: number of step-list entries (diagonal keys) used
  int accumulate;           // bwd: += into dk/dv
  int nqt;                  // L / 128 (tensor-core path)
  int head_split;           // bwd: CTAs per (b, kv head, kv tile) sharing the G q-heads
  int order_batch;          // CTA order: (b, kv head[, head subset]) groups per longest-first batch
  float scale;              // c
  float scale_log2;         // c * log2(e)
  // forward / shared inputs
  const void* q;
  const void* k;  // K_0
  const void* v;  // V_0
  const void* ks[TTT_MAX_STEPS];
  const void* vs[TTT_MAX_STEPS];
  void* out;
  void* out_lo;  // optional bf16 residual O - bf16(O)
  float* lse;
  // backward
  const void* o;
  const void* o_lo;  // optional residual of o
  const void* dout;
  const float* lse_in;
  void* dq;
  float* dk;
  float* dv;
  float* dks[TTT_MAX_STEPS];
  float* dvs[TTT_MAX_STEPS];
  float* delta;   // workspace [B][Hq][L]: -Delta = -rowsum(dO o O)  (stored negated)
  float* lse2;    // workspace [B][Hq][L]: -lse * log2(e)           (stored negated)
  float* dq_acc;  // workspace fp32, tile-contiguous [B][Hq][L/128][D/32][128][32]
  // fp32 check path backward: fp64 accumulators [dK_0 | dV_0 | dK_1..dK_j | dV_1..dV_j] (workspace)
  double* dacc;
  int seq_lens[TTT_MAX_BATCH];
  // Row layout. Padded: [B][L][H][D], row0[b] = b L, tile0[b] = b nqt. Packed (desc.cu_seqlens):
  // one [nrows][H][D] view, sequence b = rows [row0[b], row0[b] + T_b) with no padding, its
  // 128-row tiles numbered from tile0[b]; the tensor maps then have batch extent 1; lse is
  // [Hq][nrows]. The delta / lse2 workspaces are [Hq][ntiles][128] in both layouts (padded: the
  // same as [B][Hq][L]), so the main kernel's 128-row bulk loads start 512-B aligned; packed, the
  // rows >= T_b of a sequence's last tile are zeroed before the pre-pass.
  int packed;
  int nrows;   // rows of the [rows][H][D] view (B L or sum T_b)
  int ntiles;  // 128-row tiles over all sequences (B nqt or sum ceil(T_b / 128))
  int row0[TTT_MAX_BATCH + 1];
  int tile0[TTT_MAX_BATCH + 1];
  // tree-attention verification (ttt_tree_attn_fwd): seq_lens = prefix lengths, L = tree size
  int tree_n;                              // n tree tokens (queries), <= 64
  const unsigned long long* tree_mask;     // [B][n] ancestor-or-self bit masks (bit u = tree key u)
  int tree_splits;                         // context splits per (b, kv head); > 1: partial out / lse
  int tree_kv_len;                         // rows of the K / V cache (check path)
  const int32_t* tree_parents;             // [B][n] parent indices (check path)
};

#ifdef __CUDACC__
// ---- row-layout helpers (padded / packed; see Params). `pk` is the layout: the tensor-core kernels
// pass their PACKED template flag (the padded instantiations compile exactly as before), the
// CUDA-core check kernels pass p.packed ----
// index of lse[b][h][r] (padded [B][Hq][L], packed [Hq][nrows])
__device__ __forceinline__ size_t lse_at(const Params& p, bool pk, int b, int h, int r) {
  return pk ? (size_t)h * p.nrows + p.row0[b] + r : ((size_t)b * p.Hq + h) * p.L + r;
}
// 128-row tile (b, h, tile t of the sequence) of the dq accumulator and the delta / lse2 workspaces
__device__ __forceinline__ size_t dq_tile(const Params& p, bool pk, int b, int h, int t) {
  return pk ? (size_t)h * p.ntiles + p.tile0[b] + t : ((size_t)b * p.Hq + h) * p.nqt + t;
}
__device__ __forceinline__ size_t ws_at(const Params& p, bool pk, int b, int h, int r) {
  return dq_tile(p, pk, b, h, r >> 7) * 128 + (r & 127);
}
// sequence of a global row / tile: b with start[b] <= x < start[b + 1] (binary search when packed)
__device__ __forceinline__ int seq_search(const int* start, int B, int x) {
  int lo = 0, hi = B - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}
__device__ __forceinline__ int seq_of_row(const Params& p, bool pk, int row) {
  return pk ? seq_search(p.row0, p.B, row) : row / p.L;
}
__device__ __forceinline__ int seq_of_tile(const Params& p, bool pk, int t) {
  return pk ? seq_search(p.tile0, p.B, t) : t / p.nqt;
}
#endif

// Tensor maps for the tcgen05 paths (4-D: D, H, L, B; box 64 x 1 x 128 x 1, SW128)
// TTT_FWD_TC_DIAG = 1 (dev, off): the forward treats step j's diagonal keys as j extra kv tiles (K_i / V_i
// rows of the q tile, 128-row SW128 boxes in FwdMaps::kd / vd) on the tensor cores with a diagonal-only
// mask and a second P_lo pass, instead of the CUDA-core diagonal warps (0). Measured (r04g-r04j): without
// the P_lo pass the forward was 7% faster but the bf16-rounded diagonal weights broke the plain bound on
// accumulated dK_i at the Llama shape (6 of 16.7M elements, 4.9e-2); with it every test passes but the
// forward is 1.6-3% slower (three 1024-clk MMAs per diagonal step for the two heads). Shared by api.cu (map
// boxes) and fwd_sm100.cu.
#ifndef TTT_FWD_TC_DIAG
#define TTT_FWD_TC_DIAG 0
#endif
struct FwdMaps {
  CUtensorMap q, k, v, out, out_lo;
  // step lists K_i / V_i (i < step) as 4-D BSHD maps with 16-row boxes: the forward's diagonal ring
  CUtensorMap kd[TTT_MAX_STEPS], vd[TTT_MAX_STEPS];
};
// forward diagonal pre-pass: q and out viewed as [B*L*Hq rows][D], box 64 x (NR*G) rows, SW128;
// backward pre-pass (bwd_sm100.cu): 2-D [rows][D] bf16 views, SW128, 64-column boxes
struct PreMaps {
  CUtensorMap dout, o, olo, q;                      // [B L Hq rows][D] bf16, box 64 x NR*G
  CUtensorMap k[TTT_MAX_STEPS], v[TTT_MAX_STEPS];  // [B L Hkv rows][D] bf16, box 64 x NR
};
// Unroll-level backward pre-pass (ttt_attn_bwd_unroll): per-step inputs / workspaces of the S
// reverse-order calls, so one persistent pass covers every step's diagonal terms.
constexpr int kMaxUnroll = TTT_MAX_UNROLL;
struct UnrollPre {
  int S;  // steps of the unroll: items j = S-1 .. 0 of every row group
  int M;  // row groups per j-sweep (>= the stage count; see ttt_bwd_pre_kernel)
  const float* lse_in[kMaxUnroll];
  float* delta[kMaxUnroll];
  float* lse2[kMaxUnroll];
  float* dq_acc[kMaxUnroll];
  CUtensorMap dout[kMaxUnroll], o[kMaxUnroll], olo[kMaxUnroll], q[kMaxUnroll];
};
struct DiagMaps {
  CUtensorMap q, out;
  CUtensorMap k[TTT_MAX_STEPS], v[TTT_MAX_STEPS];  // K_i, V_i as [B*L*Hkv rows][D], box 64 x NR
};
struct BwdMaps {
  CUtensorMap q, k, v, dout;
  CUtensorMap dout64;  // dO with 64-row boxes (the 64-query sub-item halves)
  CUtensorMap dqacc;  // 2-D fp32 view of the tiled dq_acc: {32 cols, rows}, box 32 x 32, SW128
};

// Instrumentation hook (api.cu): brackets one kernel launch with events when
// ttt_attn_profile_begin() armed the calling thread; no-op otherwise.
enum KernelKind {
  kKindFwdDiag = 0, kKindFwdMain = 1, kKindBwdPre = 2, kKindBwdMain = 3,
  kKindBwdConvert = 4, kKindCheckFwd = 5, kKindCheckBwd = 6, kKindZero = 7,
  kKindLoss = 8, kKindLossAux = 9
};
void prof_mark(int kind, bool start, cudaStream_t st);

// Host: CTA-order batch size for a non-persistent grid of `ngroups` groups x `nlen` CTAs whose
// length is (len_unit(i) + overhead) for the i-th CTA of a group in longest-first order. Picks the
// batch (groups interleaved longest-first inside a batch) with the smallest simulated makespan
// over 148 greedy SMs, among batches whose L2 working set stays under ~80 MB.
// `copies` CTAs share each (group, rank); len_of_rank[i] in units of one work item.
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per (function, device context): set it once
// per device ordinal (bit d of `done`), thread-safely; devices >= 64 set it on every launch.
template <typename F>
inline cudaError_t set_smem_attr(F* fn, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = dev < 64 ? (1ull << dev) : 0ull;
  if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && bit) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

int pick_order_batch(int ngroups, int nranks, int copies, const double* len_of_rank, double overhead,
                     double bytes_per_group);
// dev-only schedule overrides (A/B experiments): integer environment variable, read once; `def` when unset
int dev_env_int(const char* name, int def);

}  // namespace tttk
