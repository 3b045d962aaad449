// api.cu — the C-ABI of libtttattn.so (include/ttt_attn.h): validation, TMA
// tensor-map encoding, kernel launches. No allocation, no per-call state.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <functional>
#include <cstdlib>
#include <mutex>
#include <queue>
#include <vector>

#include "../../include/ttt_attn.h"
#include "ttt_params.cuh"

namespace tttk {
cudaError_t launch_zero_f32(float* x, size_t n, cudaStream_t st);
cudaError_t launch_fwd_check(const Params& p, cudaStream_t st);
cudaError_t launch_bwd_check(const Params& p, cudaStream_t st);
size_t check_bwd_ws_bytes(const Params& p);
cudaError_t launch_fwd_sm100(const Params& p, const FwdMaps& maps, const DiagMaps& dmaps, cudaStream_t st);
int fwd_diag_rows_per_group(const Params& p);
bool fwd_uses_diag_kernel();
cudaError_t launch_bwd_sm100(const Params& p, const BwdMaps& maps, const PreMaps& pmaps, cudaStream_t st);
int bwd_pre_rows_per_group(const Params& p);
cudaError_t launch_tree_sm100(const Params& p, const FwdMaps& maps, const int32_t* parents, cudaStream_t st);
cudaError_t launch_tree_check(const Params& p, cudaStream_t st);
cudaError_t launch_tree_combine(const void* part, const float* lse_part, int nsplit, int B, int n, int Hq, int D,
                                void* out, float* lse, cudaStream_t st);
cudaError_t launch_bwd_unroll_sm100(const Params* ps, const BwdMaps* maps, const PreMaps& pmaps,
                                    const UnrollPre& up, cudaStream_t st);
}  // namespace tttk

using namespace tttk;

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// BSHD bf16 tensor [B][L][H][D] -> 4-D map (D, H, L, B), box (64, 1, 128, 1), 128B swizzle.
bool encode_bshd(CUtensorMap* m, const void* ptr, int B, int L, int H, int D, int box_rows = 128) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)L, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)D * 2, (cuuint64_t)H * D * 2, (cuuint64_t)L * H * D * 2};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// tiled fp32 dq accumulator as a 2-D tensor {32, rows}: box {32, 32} (4 KB), 128B swizzle.
// [rows][D] bf16 view of a BSHD tensor (rows = B*L*H), box 64 columns x box_rows rows, SW128
bool encode_rows2d(CUtensorMap* m, const void* ptr, long long rows, int D, int box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// BSHD bf16 tensor -> 4-D map with box (D, 1, box_rows, 1), no swizzle: whole rows of one head
bool encode_bshd_rows(CUtensorMap* m, const void* ptr, int B, int L, int H, int D, int box_rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)H, (cuuint64_t)L, (cuuint64_t)B};
  cuuint64_t strides[3] = {(cuuint64_t)D * 2, (cuuint64_t)H * D * 2, (cuuint64_t)L * H * D * 2};
  cuuint32_t box[4] = {(cuuint32_t)D, 1, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_dqacc(CUtensorMap* m, void* ptr, size_t rows) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {32, (cuuint64_t)rows};
  cuuint64_t strides[1] = {32 * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int validate_desc(const ttt_attn_desc* d, int step) {
  if (!d) return TTT_ERR_INVALID_ARG;
  if (d->batch < 1 || d->batch > TTT_MAX_BATCH || d->seq_len < 1 || d->num_q_heads < 1 || d->num_kv_heads < 1)
    return TTT_ERR_INVALID_ARG;
  if (d->num_q_heads % d->num_kv_heads) return TTT_ERR_INVALID_ARG;
  if (d->dtype != TTT_BF16 && d->dtype != TTT_FP32_CHECK) return TTT_ERR_INVALID_ARG;
  if (d->head_dim != 64 && d->head_dim != 128) return TTT_ERR_UNSUPPORTED;
  if (d->num_q_heads / d->num_kv_heads > 32) return TTT_ERR_UNSUPPORTED;  // GQA group <= 32 heads
  if (!(d->softmax_scale >= 0.f) || std::isinf(d->softmax_scale)) return TTT_ERR_INVALID_ARG;
  if (step < 0 || step >= TTT_MAX_STEPS) return TTT_ERR_STEP_RANGE;
  if (d->cu_seqlens) {  // packed layout
    if (d->seq_lens) return TTT_ERR_INVALID_ARG;
    if (d->cu_seqlens[0] != 0) return TTT_ERR_INVALID_ARG;
    for (int b = 0; b < d->batch; ++b)
      if ((long long)d->cu_seqlens[b + 1] - d->cu_seqlens[b] < 1) return TTT_ERR_DEGENERATE;
    if ((long long)d->cu_seqlens[d->batch] * d->num_q_heads >= (1ll << 31)) return TTT_ERR_UNSUPPORTED;
    return TTT_OK;
  }
  if (d->dtype == TTT_BF16 && (d->seq_len % kTile)) return TTT_ERR_UNSUPPORTED;
  // row indices (b L + r) Hq + h are decoded in 32-bit arithmetic on the device
  if ((long long)d->batch * d->seq_len * d->num_q_heads >= (1ll << 31)) return TTT_ERR_UNSUPPORTED;
  if (d->seq_lens) {
    for (int b = 0; b < d->batch; ++b)
      if (d->seq_lens[b] < 1 || d->seq_lens[b] > d->seq_len) return TTT_ERR_DEGENERATE;
  }
  return TTT_OK;
}

void fill_common(Params& p, const ttt_attn_desc* d, int step) {
  std::memset(&p, 0, sizeof(p));
  p.B = d->batch;
  p.L = d->seq_len;
  p.Hq = d->num_q_heads;
  p.Hkv = d->num_kv_heads;
  p.D = d->head_dim;
  p.G = p.Hq / p.Hkv;
  p.step = step;
  p.nqt = p.L / kTile;
  p.scale = d->softmax_scale > 0.f ? d->softmax_scale : 1.0f / std::sqrt((float)p.D);
  p.scale_log2 = p.scale * 1.4426950408889634f;
  if (d->cu_seqlens) {  // packed: one [nrows][H][D] view, each sequence's tiles numbered in turn
    p.packed = 1;
    int maxT = 1, tiles = 0;
    for (int b = 0; b < p.B; ++b) {
      const int T = d->cu_seqlens[b + 1] - d->cu_seqlens[b];
      p.seq_lens[b] = T;
      p.row0[b] = d->cu_seqlens[b];
      p.tile0[b] = tiles;
      tiles += (T + kTile - 1) / kTile;
      maxT = std::max(maxT, T);
    }
    p.nrows = p.row0[p.B] = d->cu_seqlens[p.B];
    p.ntiles = p.tile0[p.B] = tiles;
    p.L = (maxT + kTile - 1) / kTile * kTile;  // bounds only (host heuristics); no tensor is [B][L]
    p.nqt = p.L / kTile;
    return;
  }
  for (int b = 0; b < p.B; ++b) p.seq_lens[b] = d->seq_lens ? d->seq_lens[b] : p.L;
  for (int b = 0; b <= p.B; ++b) {
    p.row0[b] = b * p.L;
    p.tile0[b] = b * p.nqt;
  }
  p.nrows = p.B * p.L;
  p.ntiles = p.B * p.nqt;
}

// tensor-map extents of a [B][L][H][D] tensor: (B, L) padded, (1, nrows) packed
int map_b(const Params& p) { return p.packed ? 1 : p.B; }
int map_l(const Params& p) { return p.packed ? p.nrows : p.L; }

}  // namespace

namespace tttk {
int dev_env_int(const char* name, int def) {
  const char* v = std::getenv(name);
  return (v && *v) ? std::atoi(v) : def;
}

int pick_order_batch(int ngroups, int nranks, int copies, const double* len_of_rank, double overhead,
                     double bytes_per_group) {
  struct Key {
    int ng, nr, cp;
    double l0, l1, ov, bpg;
    int best;
  };
  static std::mutex mu;
  static Key cache[8];
  static int ncache = 0;
  const double l0 = len_of_rank[0], l1 = len_of_rank[nranks - 1];
  {
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < ncache; ++i) {
      const Key& k = cache[i];
      if (k.ng == ngroups && k.nr == nranks && k.cp == copies && k.l0 == l0 && k.l1 == l1 && k.ov == overhead &&
          k.bpg == bytes_per_group)
        return k.best;
    }
  }
  constexpr int kSMs = 148;
  int best = 1;
  double best_ms = 0.0;
  for (int bsz = 1; bsz <= std::min(ngroups, 32); ++bsz) {
    if (bsz > 1 && bsz * bytes_per_group > 80e6) break;
    std::priority_queue<double, std::vector<double>, std::greater<double>> sm;
    for (int i = 0; i < kSMs; ++i) sm.push(0.0);
    double ms = 0.0;
    for (int g0 = 0; g0 < ngroups; g0 += bsz)
      for (int r = 0; r < nranks; ++r)
        for (int g = g0; g < std::min(ngroups, g0 + bsz); ++g)
          for (int c = 0; c < copies; ++c) {
            const double t = sm.top() + len_of_rank[r] + overhead;
            sm.pop();
            sm.push(t);
            ms = std::max(ms, t);
          }
    if (bsz == 1 || ms < best_ms * 0.995) {  // a larger batch must win clearly (it costs L2 reuse)
      best = bsz;
      best_ms = ms;
    }
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[ncache < 8 ? ncache++ : 7] = Key{ngroups, nranks, copies, l0, l1, overhead, bytes_per_group, best};
  return best;
}
}  // namespace tttk

namespace {

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct BwdWs {
  size_t delta, lse2, dq_acc, total;
};
BwdWs bwd_ws_layout(const ttt_attn_desc* d) {
  BwdWs w{};
  // delta / lse2 [Hq][ntiles][128], dq_acc [Hq][ntiles][128][D] (padded: ntiles = B L / 128)
  size_t tiles = (size_t)d->batch * ((d->seq_len + kTile - 1) / kTile);
  if (d->cu_seqlens) {
    tiles = 0;
    for (int b = 0; b < d->batch; ++b) tiles += (size_t)(d->cu_seqlens[b + 1] - d->cu_seqlens[b] + kTile - 1) / kTile;
  }
  const size_t rows = tiles * kTile * d->num_q_heads;
  w.delta = 0;
  w.lse2 = align256(rows * 4);
  w.dq_acc = w.lse2 + align256(rows * 4);
  w.total = w.dq_acc + align256(rows * (size_t)d->head_dim * 4);
  return w;
}

int cuda_status(cudaError_t e) { return e == cudaSuccess ? TTT_OK : TTT_ERR_CUDA; }

// ---- instrumentation: library-owned event pool, armed per host thread ----
constexpr int kProfPairs = 4096;
struct ProfRec {
  int kind;
  int slot;
};
struct ProfState {
  bool armed = false;
  int used = 0;
  int pending_kind = -1;
  cudaEvent_t ev[2 * kProfPairs];
  bool created = false;
  ProfRec rec[kProfPairs];
};
thread_local ProfState g_prof;

}  // namespace

namespace tttk {
void prof_mark(int kind, bool start, cudaStream_t st) {
  ProfState& P = g_prof;
  if (!P.armed) return;
  if (start) {
    if (P.used >= kProfPairs) return;
    P.pending_kind = kind;
    cudaEventRecord(P.ev[2 * P.used], st);
  } else if (P.pending_kind == kind && P.used < kProfPairs) {
    cudaEventRecord(P.ev[2 * P.used + 1], st);
    P.rec[P.used] = {kind, P.used};
    ++P.used;
    P.pending_kind = -1;
  }
}
}  // namespace tttk

extern "C" {

const char* ttt_attn_strerror(int code) {
  switch (code) {
    case TTT_OK: return "ok";
    case TTT_ERR_INVALID_ARG: return "invalid argument";
    case TTT_ERR_UNSUPPORTED: return "unsupported configuration (head_dim must be 64/128; bf16 needs seq_len % 128 == 0)";
    case TTT_ERR_STEP_RANGE: return "step out of range [0, TTT_MAX_STEPS)";
    case TTT_ERR_ALIGNMENT: return "device pointer not 16-byte aligned";
    case TTT_ERR_DEGENERATE: return "degenerate sequence length (need 1 <= seq_lens[b] <= seq_len)";
    case TTT_ERR_WORKSPACE: return "workspace too small";
    case TTT_ERR_CUDA: return "CUDA error";
    default: return "unknown error";
  }
}

int ttt_attn_profile_begin(void) {
  ProfState& P = g_prof;
  if (!P.created) {
    for (int i = 0; i < 2 * kProfPairs; ++i)
      if (cudaEventCreate(&P.ev[i]) != cudaSuccess) return -TTT_ERR_CUDA;
    P.created = true;
  }
  P.used = 0;
  P.pending_kind = -1;
  P.armed = true;
  return 0;
}

int ttt_attn_profile_end(double* ms_by_kind, int* launches_by_kind, int n_kinds) {
  ProfState& P = g_prof;
  if (!P.armed) return -TTT_ERR_INVALID_ARG;
  P.armed = false;
  const int nk = n_kinds < TTT_KERNEL_KINDS ? n_kinds : TTT_KERNEL_KINDS;
  for (int k = 0; k < nk; ++k) {
    if (ms_by_kind) ms_by_kind[k] = 0.0;
    if (launches_by_kind) launches_by_kind[k] = 0;
  }
  for (int i = 0; i < P.used; ++i) {
    if (cudaEventSynchronize(P.ev[2 * i + 1]) != cudaSuccess) return -TTT_ERR_CUDA;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, P.ev[2 * i], P.ev[2 * i + 1]) != cudaSuccess) return -TTT_ERR_CUDA;
    const int k = P.rec[i].kind;
    if (k < nk) {
      if (ms_by_kind) ms_by_kind[k] += ms;
      if (launches_by_kind) launches_by_kind[k] += 1;
    }
  }
  return nk;
}

const char* ttt_attn_kernel_name(int kind) {
  static const char* names[TTT_KERNEL_KINDS] = {
      "ttt_fwd_diag_kernel", "ttt_fwd_sm100_kernel", "ttt_bwd_pre_kernel", "ttt_bwd_sm100_kernel",
      "ttt_bwd_dq_convert_kernel", "fwd_check_kernel", "bwd_check_kernel", "zero_f32_kernel",
      "ttt_loss_kernel", "ttt_loss_aux_kernel"};
  return (kind >= 0 && kind < TTT_KERNEL_KINDS) ? names[kind] : "unknown";
}

const char* ttt_attn_version(void) { return "libtttattn 0.1 sm_100a (tcgen05/TMEM/TMA + fp32 check path)"; }

size_t ttt_attn_workspace_size(const ttt_attn_desc* d, int step, int is_bwd) {
  if (validate_desc(d, step) != TTT_OK) return 0;
  if (!is_bwd) return 0;
  if (d->dtype == TTT_FP32_CHECK) {  // fp64 dK / dV accumulators of the check path
    Params p;
    fill_common(p, d, step);
    return check_bwd_ws_bytes(p);
  }
  return bwd_ws_layout(d).total;
}

int ttt_attn_fwd(const ttt_attn_desc* d, int step, const void* q, const void* k_base, const void* v_base,
                 const void* const* k_steps, const void* const* v_steps, void* out, void* out_lo, float* lse,
                 void* workspace, size_t workspace_bytes, void* stream) {
  (void)workspace;
  (void)workspace_bytes;
  int st = validate_desc(d, step);
  if (st) return st;
  if (!q || !k_base || !v_base || !out || !lse) return TTT_ERR_INVALID_ARG;
  if (step > 0 && (!k_steps || !v_steps)) return TTT_ERR_INVALID_ARG;
  for (int i = 0; i < step; ++i)
    if (!k_steps[i] || !v_steps[i]) return TTT_ERR_INVALID_ARG;
  if (!aligned16(q) || !aligned16(k_base) || !aligned16(v_base) || !aligned16(out) || !aligned16(lse) ||
      !aligned16(out_lo))
    return TTT_ERR_ALIGNMENT;
  for (int i = 0; i < step; ++i)
    if (!aligned16(k_steps[i]) || !aligned16(v_steps[i])) return TTT_ERR_ALIGNMENT;
  Params p;
  fill_common(p, d, step);
  p.q = q;
  p.k = k_base;
  p.v = v_base;
  for (int i = 0; i < step; ++i) {
    p.ks[i] = k_steps[i];
    p.vs[i] = v_steps[i];
  }
  p.out = out;
  p.out_lo = d->dtype == TTT_BF16 ? out_lo : nullptr;
  p.lse = lse;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (d->dtype == TTT_FP32_CHECK) return cuda_status(launch_fwd_check(p, s));
  FwdMaps maps;
  if (!encode_bshd(&maps.q, q, map_b(p), map_l(p), p.Hq, p.D) || !encode_bshd(&maps.k, k_base, map_b(p), map_l(p), p.Hkv, p.D) ||
      !encode_bshd(&maps.v, v_base, map_b(p), map_l(p), p.Hkv, p.D) || !encode_bshd(&maps.out, out, map_b(p), map_l(p), p.Hq, p.D) ||
      (p.out_lo && !encode_bshd(&maps.out_lo, p.out_lo, map_b(p), map_l(p), p.Hq, p.D)))
    return TTT_ERR_CUDA;
  for (int i = 0; i < p.step; ++i)  // the forward's in-kernel diagonal ring: 16-row boxes of K_i / V_i
    if (TTT_FWD_TC_DIAG ? (!encode_bshd(&maps.kd[i], p.ks[i], map_b(p), map_l(p), p.Hkv, p.D) ||  // 128-row tiles
                           !encode_bshd(&maps.vd[i], p.vs[i], map_b(p), map_l(p), p.Hkv, p.D))
                        : (!encode_bshd_rows(&maps.kd[i], p.ks[i], map_b(p), map_l(p), p.Hkv, p.D, 16) ||
                           !encode_bshd_rows(&maps.vd[i], p.vs[i], map_b(p), map_l(p), p.Hkv, p.D, 16)))
      return TTT_ERR_CUDA;
  DiagMaps dmaps;
  if (p.step > 0 && fwd_uses_diag_kernel()) {
    const int nr = fwd_diag_rows_per_group(p);
    const long long rows = (long long)p.nrows * p.Hq;
    if (nr <= 0) return TTT_ERR_UNSUPPORTED;
    if (!encode_rows2d(&dmaps.q, q, rows, p.D, nr * p.G) || !encode_rows2d(&dmaps.out, out, rows, p.D, nr * p.G))
      return TTT_ERR_CUDA;
    const long long kv_rows = (long long)p.nrows * p.Hkv;
    for (int i = 0; i < p.step; ++i)
      if (!encode_rows2d(&dmaps.k[i], p.ks[i], kv_rows, p.D, nr) || !encode_rows2d(&dmaps.v[i], p.vs[i], kv_rows, p.D, nr))
        return TTT_ERR_CUDA;
  }
  return cuda_status(launch_fwd_sm100(p, maps, dmaps, s));
}

int ttt_attn_bwd(const ttt_attn_desc* d, int step, const void* q, const void* k_base, const void* v_base,
                 const void* const* k_steps, const void* const* v_steps, const void* out, const void* out_lo,
                 const float* lse, const void* dout, void* dq, float* dk_base, float* dv_base, float* const* dk_steps,
                 float* const* dv_steps, unsigned flags, void* workspace, size_t workspace_bytes, void* stream) {
  int st = validate_desc(d, step);
  if (st) return st;
  if (flags & ~TTT_ACCUMULATE_DKV) return TTT_ERR_INVALID_ARG;
  if (!q || !k_base || !v_base || !out || !lse || !dout || !dq || !dk_base || !dv_base)
    return TTT_ERR_INVALID_ARG;
  if (step > 0 && (!k_steps || !v_steps || !dk_steps || !dv_steps)) return TTT_ERR_INVALID_ARG;
  for (int i = 0; i < step; ++i)
    if (!k_steps[i] || !v_steps[i] || !dk_steps[i] || !dv_steps[i]) return TTT_ERR_INVALID_ARG;
  const void* ptrs[] = {q, k_base, v_base, out, lse, dout, dq, dk_base, dv_base, out_lo};
  for (const void* ptr : ptrs)
    if (!aligned16(ptr)) return TTT_ERR_ALIGNMENT;
  for (int i = 0; i < step; ++i)
    if (!aligned16(k_steps[i]) || !aligned16(v_steps[i]) || !aligned16(dk_steps[i]) || !aligned16(dv_steps[i]))
      return TTT_ERR_ALIGNMENT;
  Params p;
  fill_common(p, d, step);
  p.accumulate = (flags & TTT_ACCUMULATE_DKV) ? 1 : 0;
  p.q = q;
  p.k = k_base;
  p.v = v_base;
  p.o = out;
  p.o_lo = d->dtype == TTT_BF16 ? out_lo : nullptr;
  p.lse_in = lse;
  p.dout = dout;
  p.dq = dq;
  p.dk = dk_base;
  p.dv = dv_base;
  for (int i = 0; i < step; ++i) {
    p.ks[i] = k_steps[i];
    p.vs[i] = v_steps[i];
    p.dks[i] = dk_steps[i];
    p.dvs[i] = dv_steps[i];
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t kv_elems = (size_t)p.nrows * p.Hkv * p.D;
  (void)kv_elems;
  if (d->dtype == TTT_FP32_CHECK) {
    if (!workspace || workspace_bytes < check_bwd_ws_bytes(p)) return TTT_ERR_WORKSPACE;
    if (!aligned16(workspace)) return TTT_ERR_ALIGNMENT;
    p.dacc = static_cast<double*>(workspace);
    return cuda_status(launch_bwd_check(p, s));
  }
  const BwdWs w = bwd_ws_layout(d);
  if (!workspace || workspace_bytes < w.total) return TTT_ERR_WORKSPACE;
  if (!aligned16(workspace)) return TTT_ERR_ALIGNMENT;
  char* ws = static_cast<char*>(workspace);
  p.delta = reinterpret_cast<float*>(ws + w.delta);
  p.lse2 = reinterpret_cast<float*>(ws + w.lse2);
  p.dq_acc = reinterpret_cast<float*>(ws + w.dq_acc);
  BwdMaps maps;
  if (!encode_bshd(&maps.q, q, map_b(p), map_l(p), p.Hq, p.D) || !encode_bshd(&maps.k, k_base, map_b(p), map_l(p), p.Hkv, p.D) ||
      !encode_bshd(&maps.v, v_base, map_b(p), map_l(p), p.Hkv, p.D) || !encode_bshd(&maps.dout, dout, map_b(p), map_l(p), p.Hq, p.D) ||
      !encode_bshd(&maps.dout64, dout, map_b(p), map_l(p), p.Hq, p.D, 64) ||
      !encode_dqacc(&maps.dqacc, p.dq_acc, (size_t)p.ntiles * kTile * p.Hq * p.D / 32))
    return TTT_ERR_CUDA;
  PreMaps pmaps;
  {
    const int nr = bwd_pre_rows_per_group(p);
    if (nr <= 0) return TTT_ERR_UNSUPPORTED;
    const long long rows = (long long)p.nrows * p.Hq, kv_rows = (long long)p.nrows * p.Hkv;
    const int br = nr * p.G;
    if (!encode_rows2d(&pmaps.dout, dout, rows, p.D, br) || !encode_rows2d(&pmaps.o, out, rows, p.D, br) ||
        (p.o_lo && !encode_rows2d(&pmaps.olo, p.o_lo, rows, p.D, br)) ||
        (p.step > 0 && !encode_rows2d(&pmaps.q, q, rows, p.D, br)))
      return TTT_ERR_CUDA;
    for (int i = 0; i < p.step; ++i)
      if (!encode_rows2d(&pmaps.k[i], p.ks[i], kv_rows, p.D, nr) || !encode_rows2d(&pmaps.v[i], p.vs[i], kv_rows, p.D, nr))
        return TTT_ERR_CUDA;
  }
  return cuda_status(launch_bwd_sm100(p, maps, pmaps, s));
}

// Context splits per (sequence, kv head, head pair), only when those CTAs would leave more than
// half of the 148 SMs idle: enough splits for about one CTA per SM, at most one per kv tile of the
// shortest sequence (splits are never empty), at most 16. (Measured: splitting 128 CTAs into
// 3 x 128 was slower, 98 vs 75 us, each CTA's fixed cost repeating per split.)
int tree_splits(const ttt_tree_desc* d) {
  const int base = d->batch * d->num_kv_heads * ((d->num_q_heads / d->num_kv_heads + 3) / 4);
  if (2 * base > 148) return 1;
  int min_tiles = 1 << 30;
  for (int b = 0; b < d->batch; ++b) min_tiles = std::min(min_tiles, (d->prefix_lens[b] + d->num_tree + 127) / 128);
  const int s = 148 / base;
  return std::max(1, std::min(std::min(s, 16), min_tiles));
}
struct TreeWs {
  size_t mask, part, lse, total;
  int splits;
};
TreeWs tree_ws_layout(const ttt_tree_desc* d) {
  TreeWs w{};
  w.splits = tree_splits(d);
  w.mask = 0;
  w.part = align256((size_t)d->batch * d->num_tree * 8);
  w.lse = w.part;
  if (w.splits > 1) w.lse += align256((size_t)w.splits * d->batch * d->num_tree * d->num_q_heads * d->head_dim * 2);
  w.total = w.lse + (w.splits > 1 ? align256((size_t)w.splits * d->batch * d->num_q_heads * d->num_tree * 4) : 0);
  return w;
}

size_t ttt_tree_attn_workspace_size(const ttt_tree_desc* d) {
  if (!d || !d->prefix_lens || d->batch < 1 || d->batch > TTT_MAX_BATCH || d->num_tree < 1 ||
      d->num_tree > TTT_MAX_TREE || d->num_kv_heads < 1 || d->num_q_heads < d->num_kv_heads)
    return 0;
  return tree_ws_layout(d).total;
}

int ttt_tree_attn_fwd(const ttt_tree_desc* d, const void* q, const void* k_cache, const void* v_cache,
                      const int32_t* parents, void* out, float* lse, void* workspace, size_t workspace_bytes,
                      void* stream) {
  if (!d || !q || !k_cache || !v_cache || !parents || !out || !lse || !d->prefix_lens) return TTT_ERR_INVALID_ARG;
  if (d->batch < 1 || d->batch > TTT_MAX_BATCH || d->num_tree < 1 || d->kv_len < 1 || d->num_q_heads < 1 ||
      d->num_kv_heads < 1 || d->num_q_heads % d->num_kv_heads)
    return TTT_ERR_INVALID_ARG;
  if (d->num_tree > TTT_MAX_TREE) return TTT_ERR_UNSUPPORTED;
  if (d->head_dim != 64 && d->head_dim != 128) return TTT_ERR_UNSUPPORTED;
  if (d->num_q_heads / d->num_kv_heads > 32) return TTT_ERR_UNSUPPORTED;
  if (!(d->softmax_scale >= 0.f) || std::isinf(d->softmax_scale)) return TTT_ERR_INVALID_ARG;
  if ((long long)d->batch * d->kv_len * d->num_kv_heads >= (1ll << 31)) return TTT_ERR_UNSUPPORTED;
  for (int b = 0; b < d->batch; ++b)
    if (d->prefix_lens[b] < 0 || d->prefix_lens[b] + d->num_tree > d->kv_len) return TTT_ERR_DEGENERATE;
  if (d->dtype != TTT_BF16 && d->dtype != TTT_FP32_CHECK) return TTT_ERR_INVALID_ARG;
  const void* ptrs[] = {q, k_cache, v_cache, out, lse};
  for (const void* ptr : ptrs)
    if (!aligned16(ptr)) return TTT_ERR_ALIGNMENT;
  if (d->dtype == TTT_FP32_CHECK) {  // fp32 CUDA-core check path, no workspace
    Params p;
    std::memset(&p, 0, sizeof(p));
    p.B = d->batch;
    p.Hq = d->num_q_heads;
    p.Hkv = d->num_kv_heads;
    p.D = d->head_dim;
    p.G = p.Hq / p.Hkv;
    p.scale = d->softmax_scale > 0.f ? d->softmax_scale : 1.0f / std::sqrt((float)p.D);
    for (int b = 0; b < p.B; ++b) p.seq_lens[b] = d->prefix_lens[b];
    p.tree_n = d->num_tree;
    p.tree_kv_len = d->kv_len;
    p.tree_parents = parents;
    p.q = q;
    p.k = k_cache;
    p.v = v_cache;
    p.out = out;
    p.lse = lse;
    return cuda_status(launch_tree_check(p, static_cast<cudaStream_t>(stream)));
  }
  const TreeWs tw = tree_ws_layout(d);
  if (!workspace || workspace_bytes < tw.total) return TTT_ERR_WORKSPACE;
  if (!aligned16(workspace)) return TTT_ERR_ALIGNMENT;
  Params p;
  std::memset(&p, 0, sizeof(p));
  p.B = d->batch;
  p.L = d->num_tree;
  p.Hq = d->num_q_heads;
  p.Hkv = d->num_kv_heads;
  p.D = d->head_dim;
  p.G = p.Hq / p.Hkv;
  p.step = 0;
  p.nqt = 1;
  p.scale = d->softmax_scale > 0.f ? d->softmax_scale : 1.0f / std::sqrt((float)p.D);
  p.scale_log2 = p.scale * 1.4426950408889634f;
  for (int b = 0; b < p.B; ++b) p.seq_lens[b] = d->prefix_lens[b];
  p.tree_n = d->num_tree;
  char* wsb = static_cast<char*>(workspace);
  p.tree_mask = reinterpret_cast<const unsigned long long*>(wsb + tw.mask);
  p.tree_splits = tw.splits;
  void* part = tw.splits > 1 ? static_cast<void*>(wsb + tw.part) : out;      // per-split partial outputs
  float* lse_part = tw.splits > 1 ? reinterpret_cast<float*>(wsb + tw.lse) : lse;
  p.q = q;
  p.k = k_cache;
  p.v = v_cache;
  p.out = part;
  p.out_lo = nullptr;
  p.lse = lse_part;
  FwdMaps maps;
  if (!encode_bshd(&maps.q, q, p.B, d->num_tree, p.Hq, p.D, 64) ||
      !encode_bshd(&maps.k, k_cache, p.B, d->kv_len, p.Hkv, p.D) ||
      !encode_bshd(&maps.v, v_cache, p.B, d->kv_len, p.Hkv, p.D) ||
      !encode_bshd(&maps.out, part, p.B * tw.splits, d->num_tree, p.Hq, p.D, 64))
    return TTT_ERR_CUDA;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = launch_tree_sm100(p, maps, parents, s);
  if (e == cudaSuccess && tw.splits > 1)
    e = launch_tree_combine(part, lse_part, tw.splits, p.B, d->num_tree, p.Hq, p.D, out, lse, s);
  return cuda_status(e);
}

size_t ttt_attn_bwd_unroll_workspace_size(const ttt_attn_desc* d, int num_steps) {
  if (num_steps < 1 || num_steps > TTT_MAX_UNROLL || validate_desc(d, num_steps - 1) != TTT_OK) return 0;
  if (d->dtype == TTT_FP32_CHECK) return ttt_attn_workspace_size(d, num_steps - 1, 1);  // calls run in order
  return (size_t)num_steps * bwd_ws_layout(d).total;
}

int ttt_attn_bwd_unroll(const ttt_attn_desc* d, int num_steps, const void* const* q, const void* k_base,
                        const void* v_base, const void* const* k_steps, const void* const* v_steps,
                        const void* const* out, const void* const* out_lo, const float* const* lse,
                        const void* const* dout, void* const* dq, float* dk_base, float* dv_base,
                        float* const* dk_steps, float* const* dv_steps, unsigned flags, void* workspace,
                        size_t workspace_bytes, void* stream) {
  const int S = num_steps;
  if (S < 1 || S > TTT_MAX_UNROLL) return TTT_ERR_STEP_RANGE;
  int st = validate_desc(d, S - 1);
  if (st) return st;
  if (flags & ~TTT_ACCUMULATE_DKV) return TTT_ERR_INVALID_ARG;
  if (!q || !out || !lse || !dout || !dq) return TTT_ERR_INVALID_ARG;
  if (d->dtype == TTT_FP32_CHECK) {  // check mode: the S calls of the contract, in order
    for (int j = S - 1; j >= 0; --j) {
      const int rc = ttt_attn_bwd(d, j, q[j], k_base, v_base, k_steps, v_steps, out[j], nullptr, lse[j], dout[j],
                                  dq[j], dk_base, dv_base, dk_steps, dv_steps,
                                  j == S - 1 ? flags : (flags | TTT_ACCUMULATE_DKV), workspace, workspace_bytes,
                                  stream);
      if (rc) return rc;
    }
    return TTT_OK;
  }
  // the same validation as S ttt_attn_bwd calls, all before the first launch
  if (!k_base || !v_base || !dk_base || !dv_base) return TTT_ERR_INVALID_ARG;
  if (S > 1 && (!k_steps || !v_steps || !dk_steps || !dv_steps)) return TTT_ERR_INVALID_ARG;
  for (int i = 0; i < S - 1; ++i) {
    if (!k_steps[i] || !v_steps[i] || !dk_steps[i] || !dv_steps[i]) return TTT_ERR_INVALID_ARG;
    if (!aligned16(k_steps[i]) || !aligned16(v_steps[i]) || !aligned16(dk_steps[i]) || !aligned16(dv_steps[i]))
      return TTT_ERR_ALIGNMENT;
  }
  if (!aligned16(k_base) || !aligned16(v_base) || !aligned16(dk_base) || !aligned16(dv_base))
    return TTT_ERR_ALIGNMENT;
  for (int j = 0; j < S; ++j) {
    if (!q[j] || !out[j] || !lse[j] || !dout[j] || !dq[j]) return TTT_ERR_INVALID_ARG;
    const void* ptrs[] = {q[j], out[j], lse[j], dout[j], dq[j], out_lo ? out_lo[j] : nullptr};
    for (const void* ptr : ptrs)
      if (!aligned16(ptr)) return TTT_ERR_ALIGNMENT;
  }
  const BwdWs w = bwd_ws_layout(d);
  if (!workspace || workspace_bytes < (size_t)S * w.total) return TTT_ERR_WORKSPACE;
  if (!aligned16(workspace)) return TTT_ERR_ALIGNMENT;
  static thread_local Params ps[TTT_MAX_UNROLL];
  static thread_local BwdMaps maps[TTT_MAX_UNROLL];
  static thread_local UnrollPre up;
  static thread_local PreMaps pmaps;
  up = UnrollPre{};
  up.S = S;
  for (int j = 0; j < S; ++j) {
    Params& p = ps[j];
    fill_common(p, d, j);
    p.accumulate = (j == S - 1) ? ((flags & TTT_ACCUMULATE_DKV) ? 1 : 0) : 1;
    p.q = q[j];
    p.k = k_base;
    p.v = v_base;
    p.o = out[j];
    p.o_lo = out_lo ? out_lo[j] : nullptr;
    p.lse_in = lse[j];
    p.dout = dout[j];
    p.dq = dq[j];
    p.dk = dk_base;
    p.dv = dv_base;
    for (int i = 0; i < S - 1; ++i) {  // every step list: the unroll pass of step S-1 reads all of them
      p.ks[i] = k_steps[i];
      p.vs[i] = v_steps[i];
      p.dks[i] = dk_steps[i];
      p.dvs[i] = dv_steps[i];
    }
    char* ws = static_cast<char*>(workspace) + (size_t)j * w.total;
    p.delta = reinterpret_cast<float*>(ws + w.delta);
    p.lse2 = reinterpret_cast<float*>(ws + w.lse2);
    p.dq_acc = reinterpret_cast<float*>(ws + w.dq_acc);
    up.lse_in[j] = p.lse_in;
    up.delta[j] = p.delta;
    up.lse2[j] = p.lse2;
    up.dq_acc[j] = p.dq_acc;
    if (!encode_bshd(&maps[j].q, q[j], map_b(p), map_l(p), p.Hq, p.D) || !encode_bshd(&maps[j].k, k_base, map_b(p), map_l(p), p.Hkv, p.D) ||
        !encode_bshd(&maps[j].v, v_base, map_b(p), map_l(p), p.Hkv, p.D) ||
        !encode_bshd(&maps[j].dout, dout[j], map_b(p), map_l(p), p.Hq, p.D) ||
        !encode_bshd(&maps[j].dout64, dout[j], map_b(p), map_l(p), p.Hq, p.D, 64) ||
        !encode_dqacc(&maps[j].dqacc, p.dq_acc, (size_t)p.ntiles * kTile * p.Hq * p.D / 32))
      return TTT_ERR_CUDA;
  }
  // pre-pass maps: layout of the largest step (S - 1); per-step q / dO / O / O_lo views
  const Params& last = ps[S - 1];
  if (out_lo)
    for (int j = 0; j < S; ++j)
      if (!out_lo[j]) return TTT_ERR_INVALID_ARG;  // all or none
  const int nr = bwd_pre_rows_per_group(last);
  if (nr <= 0) return TTT_ERR_UNSUPPORTED;
  const long long rows = (long long)last.nrows * last.Hq, kv_rows = (long long)last.nrows * last.Hkv;
  const int br = nr * last.G;
  for (int j = 0; j < S; ++j) {
    if (!encode_rows2d(&up.dout[j], dout[j], rows, last.D, br) || !encode_rows2d(&up.o[j], out[j], rows, last.D, br) ||
        (out_lo && !encode_rows2d(&up.olo[j], out_lo[j], rows, last.D, br)) ||
        !encode_rows2d(&up.q[j], q[j], rows, last.D, br))
      return TTT_ERR_CUDA;
  }
  for (int i = 0; i < S - 1; ++i)
    if (!encode_rows2d(&pmaps.k[i], k_steps[i], kv_rows, last.D, nr) ||
        !encode_rows2d(&pmaps.v[i], v_steps[i], kv_rows, last.D, nr))
      return TTT_ERR_CUDA;
  return cuda_status(launch_bwd_unroll_sm100(ps, maps, pmaps, up, static_cast<cudaStream_t>(stream)));
}

}  // extern "C"
