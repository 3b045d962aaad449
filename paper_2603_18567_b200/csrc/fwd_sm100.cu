// fwd_sm100.cu — TTT attention forward on sm_100a tensor cores.
//
// What it computes: SURVEY.md §8(a) rows 1-6 — for each query row r the
// softmax over the allowed set of Alg. 2: base keys
// k <= r with k < T_b, streamed in 128-key tiles with online softmax
// ("FlashAttention-style streaming"; BlockMask skipping,
// PAPER.md:331), then — in the epilogue — the j per-step diagonal keys
// K_i[r] (Alg. 1 "concat s_i ... o_t += alpha_i v_i") folded
// into the same running max / sum, so the L x (j+1)L mask is never built.
//
// CTA work item: one 128-row q tile of TWO query heads of the same GQA group
// (same K/V stream, identical causal length), so every K/V tile TMA'd into
// shared memory feeds two S = Q K^T MMAs. Warp roles (512 threads):
//   warps 0-3   softmax + epilogue, head slot 0 (TMEM lanes 0-127)
//   warps 4-7   softmax + epilogue, head slot 1
//   warp  8     TMA producer (Q once, then K/V tiles through a 2-stage ring)
//   warp  9     TMEM allocator + single-thread tcgen05.mma issuer
//   warps 10-13 diagonal fold, concurrent with the main loop:
//               for the tile's rows r < T_b and both heads, t_i = c log2e q_r . K_i[r]
//               (i = 1..j), A_d = log2 sum_i 2^t_i, O_d = sum_i 2^(t_i - A_d) V_i[r]
//               (Alg. 1 "concat s_i ... o_t += alpha_i v_i") on CUDA
//               cores, 8 lanes per row; K_i / V_i rows arrive through their own 4-stage
//               TMA ring of 16-row blocks; O_d leaves as bf16 through L2 (the out rows, read
//               back by TMA into the freed Q tile), A_d through shared memory
//   warp  14    TMA producer of the diagonal ring; warp 15 idle
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512);
// P (bf16, packed 2/column) is written over S and consumed by the PV MMA
// straight from TMEM (A operand in TMEM, "ts" form).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "ptx_sm100.cuh"
#include "ttt_params.cuh"

// Pairs (c mod 8) of a full tile whose exp2 runs as an FMA-pipe polynomial instead of MUFU.
#ifndef TTT_FWD_EMU_MASK
#define TTT_FWD_EMU_MASK 0x88
#endif
// 1: the softmax warps read each S row once (128 registers, setmaxnreg-rebalanced roles); 0: round-2
// form, S read in 64-column halves with keys [0,64) read twice (1.5x the TMEM reads per tile)
#ifndef TTT_FWD_ONEREAD
#define TTT_FWD_ONEREAD 1
#endif

namespace tttk {
#ifdef TTT_TRACE
__device__ unsigned long long g_ttt_ftrace[4][kTraceCap];
__device__ unsigned int g_ttt_ftrace_cta;
#define g_ttt_trace g_ttt_ftrace
#define g_ttt_trace_cta g_ttt_ftrace_cta
extern "C" int ttt_debug_ftrace_read(void* host, unsigned int cta) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(host, g_ttt_ftrace, sizeof(g_ttt_ftrace)) != cudaSuccess) return 1;
  unsigned long long z[4 * 1024] = {};
  for (int r = 0; r < 4; ++r) cudaMemcpyToSymbol(g_ttt_ftrace, z, sizeof(z), (size_t)r * kTraceCap * 8);
  return cudaMemcpyToSymbol(g_ttt_ftrace_cta, &cta, sizeof(cta)) != cudaSuccess;
}
#endif
namespace {

constexpr int kFwdThreads = 512;
// ONEREAD register split per SMSP: 2 softmax + 1 diagonal + 1 role warp <= 512 per lane
#ifndef TTT_FWD_REG_SOFTMAX
#define TTT_FWD_REG_SOFTMAX 176
#endif
#ifndef TTT_FWD_REG_DIAG
#define TTT_FWD_REG_DIAG (TTT_FWD_TC_DIAG ? 24 : 128)  // TC_DIAG: the diagonal warps idle, the role warps get the rest
#endif
constexpr uint32_t kFwdRegSoftmax = TTT_FWD_REG_SOFTMAX, kFwdRegDiag = TTT_FWD_REG_DIAG,
                   kFwdRegRole = 512 - 2 * TTT_FWD_REG_SOFTMAX - TTT_FWD_REG_DIAG;
static_assert(2 * kFwdRegSoftmax + kFwdRegDiag + kFwdRegRole <= 512, "register file per SMSP");
// setmaxnreg from the launch allocation (128 per thread at 512 threads) to N: inc or dec by direction
template <uint32_t N>
__device__ __forceinline__ void regs_to() {
  if constexpr (N > 128) regs_inc<N>();
  else if constexpr (N < 128) regs_dec<N>();
}
#ifndef TTT_FWD_DIAG_MODE
#define TTT_FWD_DIAG_MODE 0  // dev timing probes only: 1 = diagonal warps skip the math, 2 = skip the loads
#endif
#ifndef TTT_FWD_FUSED_DIAG
#define TTT_FWD_FUSED_DIAG 1  // 0: dev A/B build with round 1's separate ttt_fwd_diag_kernel
#endif
constexpr int kDgRows = 16;    // rows per diagonal-ring stage (one TMA box per 64 columns per tensor)
constexpr int kDgStages = 4;   // diagonal-ring depth
// Short CTAs (nkv <= TTT_FWD_SHD_NKV kv tiles) finish their main loop long before the diagonal (r03g: a
// 1-tile CTA at j = 6 ran 53k clk vs 16k at j = 0): there the softmax warps take the last 2/3 of the
// diagonal's 16-row blocks after their main loop, loading K_i / V_i rows straight from global memory.
#ifndef TTT_FWD_SHD_NKV
#define TTT_FWD_SHD_NKV 4
#endif
// Q (2 tiles) | K (2 stages) | V (2 stages) | diagonal ring | 1 KB alignment slack
constexpr int fwd_smem_bytes(int D) { return 6 * kTile * D * 2 + kDgStages * 2 * (D / 64) * kDgRows * 128 + 1024; }
constexpr float kRescaleThreshold = 8.0f;  // log2 domain: rescale O only when the max grows by > 2^8

struct FwdBars {
  uint64_t q;
  uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[2], p_lo[2], p_hi[2], o_full[2];  // P published in two 64-column halves
  uint64_t s_done, od;  // all S MMAs complete (Q / K smem free); diagonal partial tile landed
  uint64_t dg_full[kDgStages], dg_empty[kDgStages];  // diagonal K_i / V_i ring
  uint64_t diag_done;                                // diagonal partial (O_d rows, A_d) complete
  uint32_t tmem_base;
  float a_d[2][kTile];  // A_d = log2 sum_i 2^t_i per (head slot, row), from the diagonal warps
};

// ---- the diagonal fold's per-row math, shared by the diagonal warps and, in
// short CTAs, the softmax warps. Thread layout: 8 lanes per row (lane k8 owns columns 8 k8 .. 8 k8 + 7 of
// every 64-column box, E = 8 NBOX elements), both head slots of the CTA per row.
// q row (bf16 in the SW128 Q tiles) -> fp32 scaled by c log2 e; acc, l = 0; m = -inf
template <int NBOX>
__device__ __forceinline__ void diag_row_init(const uint8_t* sQ, int TB, int row, int k8, float sl2, float (&qf)[2][8 * NBOX],
                                              float (&acc)[2][8 * NBOX], float (&m)[2], float (&l)[2]) {
#pragma unroll
  for (int hs = 0; hs < 2; ++hs) {
    m[hs] = -INFINITY;
    l[hs] = 0.f;
#pragma unroll
    for (int bx = 0; bx < NBOX; ++bx) {
      const uint4 u = lds128(smem_u32(sQ + hs * TB + bx * 16384) + sw128_off(row, k8));
      const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w4[e]));
        qf[hs][bx * 8 + 2 * e] = f.x * sl2;
        qf[hs][bx * 8 + 2 * e + 1] = f.y * sl2;
        acc[hs][bx * 8 + 2 * e] = 0.f;
        acc[hs][bx * 8 + 2 * e + 1] = 0.f;
      }
    }
  }
}
// One pass over ns (1 or 2) stages (i, i + 1) of this lane's K_i / V_i words (bf16 pairs): the two
// stages' dot products, shuffles and exps are independent, and the running max only moves (a
// warp-uniform rescale) when a score exceeds it by 2^8 — the j-long chain of an exact online softmax
// was the fused pass's critical path. t = c log2e q . K_i[r]; p = 2^(t - m); acc += p V_i[r].
template <int E>
__device__ __forceinline__ void diag_pair_update(const float (&qf)[2][E], float (&acc)[2][E], float (&m)[2], float (&l)[2],
                                                 const uint32_t (&kw)[2][E / 2], const uint32_t (&vw)[2][E / 2], int ns) {
  float t[2][2];  // 8-lane partial dots (two FFMA2 chains each)
#pragma unroll
  for (int hs = 0; hs < 2; ++hs)
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      uint64_t d0 = 0, d1 = 0;
#pragma unroll
      for (int e = 0; e < E / 2; e += 2) {
        d0 = ffma2(f2pack(qf[hs][2 * e], qf[hs][2 * e + 1]), bf2_to_f2(kw[u][e]), d0);
        d1 = ffma2(f2pack(qf[hs][2 * e + 2], qf[hs][2 * e + 3]), bf2_to_f2(kw[u][e + 1]), d1);
      }
      float a0, a1, b0, b1;
      f2unpack(d0, a0, a1);
      f2unpack(d1, b0, b1);
      t[hs][u] = (a0 + a1) + (b0 + b1);
    }
#pragma unroll
  for (int sh = 1; sh < 8; sh <<= 1)
#pragma unroll
    for (int hs = 0; hs < 2; ++hs)
#pragma unroll
      for (int u = 0; u < 2; ++u) t[hs][u] += __shfl_xor_sync(0xffffffffu, t[hs][u], sh);
#pragma unroll
  for (int hs = 0; hs < 2; ++hs) {
    const float tmax = ns > 1 ? fmaxf(t[hs][0], t[hs][1]) : t[hs][0];
    if (__any_sync(0xffffffffu, tmax > m[hs] + 8.f)) {  // rare: the max moved (always at i = 0)
      const float m_new = fmaxf(m[hs], tmax);
      const float alpha = ex2(m[hs] - m_new);  // 0 when m was -inf
      l[hs] *= alpha;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[hs][e] *= alpha;
      m[hs] = m_new;
    }
    const float p0 = ex2(t[hs][0] - m[hs]), p1 = ns > 1 ? ex2(t[hs][1] - m[hs]) : 0.f;
    l[hs] += p0 + p1;
    const uint64_t p02 = f2pack(p0, p0), p12 = f2pack(p1, p1);
#pragma unroll
    for (int e = 0; e < E / 2; ++e) {
      uint64_t o = ffma2(bf2_to_f2(vw[0][e]), p02, f2pack(acc[hs][2 * e], acc[hs][2 * e + 1]));
      o = ffma2(bf2_to_f2(vw[1][e]), p12, o);
      f2unpack(o, acc[hs][2 * e], acc[hs][2 * e + 1]);
    }
  }
}
// O_d (normalised, bf16) -> the out rows (staging; read back by TMA), A_d = m + log2 l -> shared memory
template <int NBOX>
__device__ __forceinline__ void diag_row_store(__nv_bfloat16* orow0, int Dh, int k8, bool has1, const float (&acc)[2][8 * NBOX],
                                               const float (&m)[2], const float (&l)[2], float* a_d0, float* a_d1) {
#pragma unroll
  for (int hs = 0; hs < 2; ++hs) {
    if (hs == 0 || has1) {
      const float inv = 1.f / l[hs];
      __nv_bfloat16* orow = orow0 + hs * Dh;
#pragma unroll
      for (int bx = 0; bx < NBOX; ++bx) {
        uint4 w;
        w.x = pack_bf16(acc[hs][bx * 8 + 0] * inv, acc[hs][bx * 8 + 1] * inv);
        w.y = pack_bf16(acc[hs][bx * 8 + 2] * inv, acc[hs][bx * 8 + 3] * inv);
        w.z = pack_bf16(acc[hs][bx * 8 + 4] * inv, acc[hs][bx * 8 + 5] * inv);
        w.w = pack_bf16(acc[hs][bx * 8 + 6] * inv, acc[hs][bx * 8 + 7] * inv);
        *reinterpret_cast<uint4*>(orow + bx * 64 + k8 * 8) = w;
      }
      if (k8 == 0) *(hs == 0 ? a_d0 : a_d1) = m[hs] + log2f(l[hs]);
    }
  }
}

// TREE = true: tree-attention verification (ttt_tree_attn_fwd) on the
// same pipeline: one q tile of the n <= 64 tree tokens per (b, head pair); keys = the prefix
// (all allowed) followed by the tree tokens' own keys, allowed per query row by its
// ancestor-or-self bit mask; no diagonal step keys.
template <int D, bool TREE, bool PACKED>
__global__ void __launch_bounds__(kFwdThreads, 1)
    ttt_fwd_sm100_kernel(const __grid_constant__ Params p, const __grid_constant__ FwdMaps maps) {
  constexpr int TB = kTile * D * 2;  // bytes of one 128 x D bf16 tile
  constexpr int NBOX = D / 64;       // 64-column (128 B) swizzle boxes per tile
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment for SW128 tiles, keeping the pointer in the shared window (LDS/STS, not generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;           // 2 tiles (head slots)
  uint8_t* sK = smem + 2 * TB;  // 2 stages
  uint8_t* sV = smem + 4 * TB;  // 2 stages
  constexpr int DGB = kDgRows * 128;       // 16 rows x 64 columns of bf16 (a tensor's block is NBOX x DGB)
  constexpr int DGS = 2 * NBOX * DGB;      // one stage: K_i and V_i rows of a 16-row block
  uint8_t* sDg = smem + 6 * TB;            // diagonal ring, kDgStages stages
  __shared__ FwdBars bars;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef TTT_TRACE
  if (blockIdx.x == g_ttt_trace_cta && threadIdx.x == 0)
    g_ttt_trace[1][kTraceCap - 2] = (clock64() << 20) | (9ull << 12);  // CTA start
#endif

  // ---- work decode: (b, g)-major so one kv head's K/V stay hot in L2; within
  // it the longest (highest) q tiles first; head pairs of a tile adjacent ----
  // TTT: two heads per CTA (one per slot). TREE: four heads (n <= 64 tree rows each; slot s holds
  // heads 4 hp + 2 s in rows [0, 64) and 4 hp + 2 s + 1 in rows [64, 128)), so no row is padding.
  const int npairs = TREE ? (p.G + 3) >> 2 : (p.G + 1) >> 1;
  const int hp = (int)blockIdx.x % npairs;
  const int t_ = (int)blockIdx.x / npairs;
  int qt, g, b, split = 0;
  if constexpr (TREE) {  // (split of the context, b, g); the q tile is the tree
    const int gi = t_ % (p.B * p.Hkv);
    split = t_ / (p.B * p.Hkv);
    qt = 0;
    g = gi % p.Hkv;
    b = gi / p.Hkv;
  } else if (PACKED) {
    // packed: (tile, kv head) with the kv head fastest; each sequence's q tiles longest first
    g = t_ % p.Hkv;
    const int tt = t_ / p.Hkv;
    b = seq_of_tile(p, true, tt);
    qt = p.tile0[b + 1] - 1 - tt;  // local tile: nqt_b - 1 - (tt - tile0[b])
  } else {
#ifdef TTT_ORDER_GROUP
    qt = p.nqt - 1 - t_ % p.nqt;
    g = (t_ / p.nqt) % p.Hkv;
    b = t_ / (p.nqt * p.Hkv);
#else
    // batched longest-first: (b, g) groups in batches of p.order_batch, q tile slowest inside a batch
    const int ngrp = p.B * p.Hkv, bsz = p.order_batch * p.nqt;
    const int bat = t_ / bsz, gbase = bat * p.order_batch;
    const int gb = min(p.order_batch, ngrp - gbase), rr = t_ - bat * bsz;
    qt = p.nqt - 1 - rr / gb;
    const int gi = gbase + rr % gb;
    g = gi % p.Hkv;
    b = gi / p.Hkv;
#endif
  }
  const int h0 = g * p.G + (TREE ? 4 : 2) * hp;
  const int nheads = TREE ? min(4, p.G - 4 * hp) : min(2, p.G - 2 * hp);  // heads of this CTA
  const bool has1 = TREE ? nheads > 2 : nheads > 1;
  const int T = p.seq_lens[b];  // TREE: prefix length P_b
  // TREE: kv tiles [kvt0, kvt0 + nkv) of this context split (balanced, never empty: host keeps
  // splits <= tiles); the tree result of a split goes to partial buffers merged by a combine pass
  int kvt0 = 0, nkv;
  if constexpr (TREE) {
    const int tiles = (T + p.tree_n + kTile - 1) / kTile;
    kvt0 = split * tiles / p.tree_splits;
    nkv = (split + 1) * tiles / p.tree_splits - kvt0;
  } else {
    nkv = min(qt + 1, (T + kTile - 1) / kTile);  // BlockMask: skip k0 > q0+127 and k0 >= T
  }
  const int bst = TREE ? split * p.B + b : b;  // batch index of this CTA's out / lse rows
  // diagonal row blocks: nrb of this q tile hold rows r < T_b; the diagonal warps take [0, nrb_d), the
  // softmax warps (SHD, short CTAs) the rest
  const int nrb = (!TREE && T > qt * kTile) ? min(kTile / kDgRows, (T - qt * kTile + kDgRows - 1) / kDgRows) : 0;
  const bool shd = !TREE && !TTT_FWD_TC_DIAG && TTT_FWD_FUSED_DIAG && p.step > 0 && nkv <= TTT_FWD_SHD_NKV;
  // TC_DIAG: the j diagonal steps run as kv tiles nkv .. ntot-1 (none when the whole q tile is padding)
  const int ntot = nkv + ((TTT_FWD_TC_DIAG && !TREE && T > qt * kTile) ? p.step : 0);
  const int nrb_d = shd ? (nrb + 2) / 3 : nrb;
  // TMA (row, batch) origin of this sequence: (0, b) padded, (row0[b], 0) packed (TREE: never packed)
  const int ry = PACKED ? p.row0[b] : 0, by = PACKED ? 0 : b;

  // The TMA producer thread (warp 8, lane 0) initialises the barriers and issues the Q and first K / V
  // loads before the CTA-wide barrier, so their latency overlaps the TMEM allocation and the sync.
  auto load_q = [&]() {
    tma_prefetch_desc(&maps.q);
    tma_prefetch_desc(&maps.k);
    tma_prefetch_desc(&maps.v);
    if constexpr (TREE) {  // 64-row boxes: head h0 + k -> slot k / 2, rows 64 (k % 2) ..
      mbar_expect_tx(&bars.q, nheads * (TB / 2));
#pragma unroll
      for (int bx = 0; bx < NBOX; ++bx)
        for (int k = 0; k < nheads; ++k)
          tma_load_4d(sQ + (k >> 1) * TB + bx * 16384 + (k & 1) * 8192, &maps.q, &bars.q, bx * 64, h0 + k, 0, b);
    } else {
      mbar_expect_tx(&bars.q, (has1 ? 2 : 1) * TB);
#pragma unroll
      for (int bx = 0; bx < NBOX; ++bx) {
        tma_load_4d(sQ + bx * 16384, &maps.q, &bars.q, bx * 64, h0, ry + qt * kTile, by);
        if (has1) tma_load_4d(sQ + TB + bx * 16384, &maps.q, &bars.q, bx * 64, h0 + 1, ry + qt * kTile, by);
      }
    }
  };
  auto load_kv = [&](int n) {
    const int st = n & 1, ph = (n >> 1) & 1;
    // TC_DIAG: tiles n >= nkv are step i = n - nkv's K_i / V_i rows of this q tile
    const bool dg = TTT_FWD_TC_DIAG && n >= nkv;
    const CUtensorMap* mk = dg ? &maps.kd[n - nkv] : &maps.k;
    const CUtensorMap* mv = dg ? &maps.vd[n - nkv] : &maps.v;
    const int row = ry + (dg ? qt : kvt0 + n) * kTile;
    mbar_wait(&bars.k_empty[st], ph ^ 1);
    mbar_expect_tx(&bars.k_full[st], TB);
#pragma unroll
    for (int bx = 0; bx < NBOX; ++bx)
      tma_load_4d(sK + st * TB + bx * 16384, mk, &bars.k_full[st], bx * 64, g, row, by);
    mbar_wait(&bars.v_empty[st], ph ^ 1);
    mbar_expect_tx(&bars.v_full[st], TB);
#pragma unroll
    for (int bx = 0; bx < NBOX; ++bx)
      tma_load_4d(sV + st * TB + bx * 16384, mv, &bars.v_full[st], bx * 64, g, row, by);
  };
  if (threadIdx.x == 256) {
    mbar_init(&bars.q, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars.k_full[i], 1);
      mbar_init(&bars.k_empty[i], 1);
      mbar_init(&bars.v_full[i], 1);
      mbar_init(&bars.v_empty[i], 1);
      mbar_init(&bars.s_full[i], 1);
      mbar_init(&bars.p_lo[i], 128);
      mbar_init(&bars.p_hi[i], 128);
      mbar_init(&bars.o_full[i], 1);
    }
    mbar_init(&bars.s_done, 1);
    mbar_init(&bars.od, 1);
    for (int i = 0; i < kDgStages; ++i) {
      mbar_init(&bars.dg_full[i], 1);
      mbar_init(&bars.dg_empty[i], 4);  // the four diagonal compute warps
    }
    // every thread of the diagonal warps (and, SHD, of the active softmax warps) arrives after its own reads / writes
    mbar_init(&bars.diag_done, 128 + (shd ? (has1 ? 256 : 128) : 0));
    fence_mbar_init();
    load_q();
    load_kv(0);  // nkv >= 1 (T_b >= 1; tree splits are never empty)
  }
  if (warp == 9) {
    tmem_alloc(&bars.tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = bars.tmem_base;

  // Per SMSP (warps s, s+4, 8+s, 12+s): two softmax warps, one diagonal warp and one of
  // {TMA producer, MMA issuer, diagonal producer, idle}. ONEREAD: softmax 168 + 168, diagonal 128
  // (launch value), the fourth 48 = 512 registers per lane.
  if (warp == 8) {
    // ================= TMA producer =================
    if (TTT_FWD_ONEREAD) regs_to<kFwdRegRole>();
    if (lane == 0) {
      for (int n = 1; n < ntot; ++n) load_kv(n);  // Q and tile 0 were issued with the barrier setup
      if (!TREE && !TTT_FWD_TC_DIAG && p.step > 0) {  // diagonal partial of the two heads into the Q tiles once no S MMA
                                  // reads them and the diagonal warps have written it
        mbar_wait(&bars.s_done, 0);
        if (TTT_FWD_FUSED_DIAG) mbar_wait(&bars.diag_done, 0);
        mbar_expect_tx(&bars.od, (has1 ? 2 : 1) * TB);
#pragma unroll
        for (int bx = 0; bx < NBOX; ++bx) {
          tma_load_4d(sQ + bx * 16384, &maps.out, &bars.od, bx * 64, h0, ry + qt * kTile, by);
          if (has1) tma_load_4d(sQ + TB + bx * 16384, &maps.out, &bars.od, bx * 64, h0 + 1, ry + qt * kTile, by);
        }
      }
    }
  } else if (warp == 9) {
    // ================= MMA issuer (whole warp, converged; elect.sync inside each issue) =================
    if (TTT_FWD_ONEREAD) regs_to<kFwdRegRole>();
    {
      constexpr uint32_t idS = idesc_bf16_f32(128, 128, false, false);  // S = Q K^T, both K-major
      constexpr uint32_t idO = idesc_bf16_f32(128, D, false, true);     // O += P V, V MN-major
      const uint64_t dQ0 = sdesc_sw128(smem_u32(sQ), 16, 1024), dK0 = sdesc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t dV0 = sdesc_sw128(smem_u32(sV), 16384, 1024);
      TTT_TRACE_DECL(0);
      auto issue_S = [&](int slot, int kst) {
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          umma_ss_e(tbase + slot * 128, sdesc_add(dQ0, slot * TB + off), sdesc_add(dK0, kst * TB + off), idS, ks > 0);
        }
      };
      // O += P V in two halves of the key dimension: keys [64,128) as soon as the softmax warps
      // have published them (p_hi; P at TMEM columns [96,128) of the slot's S buffer), then keys
      // [0,64) after p_lo (columns [0,32))
      auto issue_PV = [&](int slot, int vst, bool acc, int n) {
        mbar_wait(&bars.p_hi[slot], n & 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 4; ks < 8; ++ks)
          umma_ts_e(tbase + 256 + slot * 128, tbase + slot * 128 + 96 + (ks - 4) * 8,
                    sdesc_add(dV0, vst * TB + ks * 2048), idO, (acc || ks > 4) ? 1u : 0u);
        mbar_wait(&bars.p_lo[slot], n & 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          umma_ts_e(tbase + 256 + slot * 128, tbase + slot * 128 + ks * 8, sdesc_add(dV0, vst * TB + ks * 2048), idO, 1u);
        if (TTT_FWD_TC_DIAG && n >= nkv) {
          // diagonal tile: P = P_hi + P_lo (the bf16 residual at columns [64, 96) for keys 64..127 and
          // [32, 64) for keys 0..63), so the diagonal weight enters O with ~16-bit precision as the
          // CUDA-core diagonal did
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            umma_ts_e(tbase + 256 + slot * 128, tbase + slot * 128 + (ks < 4 ? 32 + ks * 8 : 64 + (ks - 4) * 8),
                      sdesc_add(dV0, vst * TB + ks * 2048), idO, 1u);
        }
      };
      mbar_wait(&bars.q, 0);
      mbar_wait(&bars.k_full[0], 0);
      TTT_TRACE_EV(0, 8, 0);
      tc_fence_after();
      issue_S(0, 0);
      umma_commit_e(&bars.s_full[0]);
      if (has1) {
        issue_S(1, 0);
        umma_commit_e(&bars.s_full[1]);
      }
      umma_commit_e(&bars.k_empty[0]);
      for (int n = 0; n < ntot; ++n) {
        const int vst = n & 1, vph = (n >> 1) & 1;
        const bool more = n + 1 < ntot;
        const int kst = (n + 1) & 1, kph = ((n + 1) >> 1) & 1;
        if (!more) umma_commit_e(&bars.s_done);
        mbar_wait(&bars.v_full[vst], vph);
        TTT_TRACE_EV(0, 1, n);
        issue_PV(0, vst, n > 0, n);
        TTT_TRACE_EV(0, 2, n);
        if (more) {
          mbar_wait(&bars.k_full[kst], kph);
          tc_fence_after();
          issue_S(0, kst);
          umma_commit_e(&bars.s_full[0]);  // also covers PV0_n (commit tracks all prior MMAs)
        } else {
          umma_commit_e(&bars.o_full[0]);
        }
        if (has1) {
          issue_PV(1, vst, n > 0, n);
          TTT_TRACE_EV(0, 3, n);
          umma_commit_e(&bars.v_empty[vst]);
          if (more) {
            issue_S(1, kst);
            umma_commit_e(&bars.s_full[1]);
            umma_commit_e(&bars.k_empty[kst]);
          } else {
            umma_commit_e(&bars.o_full[1]);
          }
        } else {
          umma_commit_e(&bars.v_empty[vst]);
          if (more) umma_commit_e(&bars.k_empty[kst]);
        }
      }
    }
  } else if (warp >= 14) {
    // ================= TMA producer of the diagonal ring (warp 14); warp 15 idle =================
    if (TTT_FWD_ONEREAD) regs_to<kFwdRegRole>();
    if (TTT_FWD_FUSED_DIAG && !TTT_FWD_TC_DIAG && !TREE && p.step > 0 && warp == 14 && lane == 0) {
      const int j = p.step;
      int n = 0;
      for (int rb = 0; rb < nrb_d; ++rb)
        for (int i = 0; i < j; ++i, ++n) {
          const int st = n % kDgStages, use = n / kDgStages;
          mbar_wait(&bars.dg_empty[st], (use & 1) ^ 1);
          if (TTT_FWD_DIAG_MODE == 2) {  // dev probe: no loads
            mbar_arrive(&bars.dg_full[st]);
            continue;
          }
          mbar_expect_tx(&bars.dg_full[st], DGS);
          uint8_t* base = sDg + st * DGS;
          const int r0 = qt * kTile + rb * kDgRows;
          // one box per tensor: 16 rows x D columns, no swizzle (rows of D x 2 bytes)
          tma_load_4d(base, &maps.kd[i], &bars.dg_full[st], 0, g, ry + r0, by);
          tma_load_4d(base + NBOX * DGB, &maps.vd[i], &bars.dg_full[st], 0, g, ry + r0, by);
        }
    }
  } else if (warp >= 10) {
    // ================= diagonal fold (warps 10-13) =================
    if (TTT_FWD_ONEREAD) regs_to<kFwdRegDiag>();

    if (TTT_FWD_FUSED_DIAG && !TTT_FWD_TC_DIAG && !TREE && p.step > 0) {
      const int j = p.step;
      {
        // thread layout: 8 lanes per row (lane k = lane & 7 owns columns 8k..8k+7 of every 64-column
        // box), 4 rows per warp, 16 rows per stage; both head slots per row
        constexpr int E = 8 * NBOX;  // elements per lane
        const int dw = warp - 10, k8 = lane & 7;
        const int srow = dw * 4 + (lane >> 3);  // row within a 16-row block
        const float sl2 = p.scale_log2;
        mbar_wait(&bars.q, 0);  // q rows are read from the Q tiles (shared with the S MMAs, read-only)
        TTT_TRACE_DECL(3);
        if (threadIdx.x == 320) TTT_TRACE_EV(3, 4, 0);
        int n = 0;
        for (int rb = 0; rb < nrb_d; ++rb) {
          const int row = rb * kDgRows + srow;
          const int r = qt * kTile + row;
          float qf[2][E], acc[2][E], m[2], l[2];
          diag_row_init<NBOX>(sQ, TB, row, k8, sl2, qf, acc, m, l);
          for (int i = 0; i < j; i += 2) {
            const int ns = min(2, j - i);
            uint32_t kw[2][E / 2], vw[2][E / 2];  // packed bf16 pairs of K_i, V_i (this lane's columns)
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              if (u < ns) {
                const int st = (n + u) % kDgStages, use = (n + u) / kDgStages;
                mbar_wait(&bars.dg_full[st], use & 1);
                if (threadIdx.x == 320) TTT_TRACE_EV(3, 1, n + u);
                const uint32_t base = smem_u32(sDg + st * DGS);
#pragma unroll
                for (int bx = 0; bx < NBOX; ++bx) {
                  const uint32_t off = (uint32_t)srow * (D * 2) + bx * 128 + k8 * 16;  // row-major rows
                  const uint4 uk = lds128(base + off);
                  const uint4 uv = lds128(base + NBOX * DGB + off);
                  kw[u][bx * 4 + 0] = uk.x; kw[u][bx * 4 + 1] = uk.y; kw[u][bx * 4 + 2] = uk.z; kw[u][bx * 4 + 3] = uk.w;
                  vw[u][bx * 4 + 0] = uv.x; vw[u][bx * 4 + 1] = uv.y; vw[u][bx * 4 + 2] = uv.z; vw[u][bx * 4 + 3] = uv.w;
                }
              } else {
#pragma unroll
                for (int e = 0; e < E / 2; ++e) kw[u][e] = vw[u][e] = 0u;
              }
            }
            __syncwarp();
            if (lane == 0)
              for (int u = 0; u < ns; ++u) mbar_arrive(&bars.dg_empty[(n + u) % kDgStages]);  // values in registers
            n += ns;
            if (TTT_FWD_DIAG_MODE == 1) continue;  // dev probe: no math
            diag_pair_update<E>(qf, acc, m, l, kw, vw, ns);
          }
          if (r < T)
            diag_row_store<NBOX>(reinterpret_cast<__nv_bfloat16*>(p.out) + (((size_t)(PACKED ? p.row0[b] : b * p.L) + r) * p.Hq + h0) * D,
                                 D, k8, has1, acc, m, l, &bars.a_d[0][row], &bars.a_d[1][row]);
        }
        if (threadIdx.x == 320) TTT_TRACE_EV(3, 2, n);
        fence_async_global();  // the out rows are read back by the producer's TMA (async proxy)
        __threadfence_block();
        mbar_arrive(&bars.diag_done);
      }
    }
  } else {
    // ================= softmax + epilogue (warps 0-7) =================
    if (TTT_FWD_ONEREAD) regs_to<kFwdRegSoftmax>();
    const int slot = warp >> 2;
    const int wq = warp & 3;
    if (slot == 0 || has1) {
      const int row = wq * 32 + lane;
      // TREE: row = 64 (head within the slot) + tree node
      const int r = TREE ? (row & 63) : qt * kTile + row;
      const int h = TREE ? h0 + 2 * slot + (row >> 6) : h0 + slot;
      const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
      const uint32_t tS = tbase + lane_off + slot * 128;
      const uint32_t tO = tbase + lane_off + 256 + slot * 128;
      const float sl2 = p.scale_log2;
      float m_run = -INFINITY, l_run = 0.f;
      // TREE: this row's ancestor-or-self mask (rows >= n are tile padding)
      const bool tree_row = TREE && r < p.tree_n && (2 * slot + (row >> 6)) < nheads;
      const unsigned long long tree_am = tree_row ? p.tree_mask[(size_t)b * p.tree_n + r] : 0ull;
      TTT_TRACE_DECL(1);
      TTT_TRACE_DECL(2);
      for (int n = 0; n < ntot; ++n) {
        mbar_wait(&bars.s_full[slot], n & 1);
        if (threadIdx.x == 0) TTT_TRACE_EV(1, 1, n);
        if (threadIdx.x == 128) TTT_TRACE_EV(2, 1, n);
        tc_fence_after();
        if (TTT_FWD_TC_DIAG && n >= nkv) {
          // ---- diagonal tile (step i = n - nkv + 1): only column c = row is allowed (Alg. 2 M_suffix,
          // PAPER.md:305-309), and only for rows r < T. The warp's rows are TMEM lanes 32 wq + lane, so
          // their diagonal entries are columns 32 wq .. 32 wq + 31: one 32-column load, lane picks its own.
          uint32_t d32[32];
          tmem_ld32(tS + wq * 32, d32);
          float sd = __uint_as_float(d32[0]);
#pragma unroll
          for (int c = 1; c < 32; ++c) sd = (lane == c) ? __uint_as_float(d32[c]) : sd;
          const float xd = (r < T) ? sd * sl2 : -INFINITY;
          const float m_new = fmaxf(m_run, xd);
          if (__any_sync(0xffffffffu, m_new > m_run + kRescaleThreshold)) {  // rare: rescale O (PV_{n-1} done)
            const float alpha = ex2(m_run - m_new);
            const uint64_t a2 = f2pack(alpha, alpha);
#pragma unroll 1
            for (int c0 = 0; c0 < D; c0 += 32) {
              uint32_t o[32];
              tmem_ld32(tO + c0, o);
#pragma unroll
              for (int i2 = 0; i2 < 32; i2 += 2) {
                float lo, hi;
                f2unpack(fmul2(f2pack(__uint_as_float(o[i2]), __uint_as_float(o[i2 + 1])), a2), lo, hi);
                o[i2] = __float_as_uint(lo);
                o[i2 + 1] = __float_as_uint(hi);
              }
              tmem_st32(tO + c0, o);
            }
            l_run *= alpha;
            m_run = m_new;
          }
          const float pd = ex2(xd - m_run);  // 0 for masked rows
          l_run += pd;
          // P row: zero except key `row` (bf16 pairs, 2 keys per 32-bit column): keys 64..127 -> columns
          // [96, 128) (p_hi, published first), keys 0..63 -> columns [0, 32) (p_lo)
          const float pd_hi = __bfloat162float(__float2bfloat16_rn(pd)), pd_lo = pd - pd_hi;
          const uint32_t pw = (row & 1) ? pack_bf16(0.f, pd_hi) : pack_bf16(pd_hi, 0.f);
          const uint32_t pwl = (row & 1) ? pack_bf16(0.f, pd_lo) : pack_bf16(pd_lo, 0.f);
          const int wsel = (row & 63) >> 1;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int hf = 1 - hh;
            uint32_t pk[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) pk[c] = ((row >> 6) == hf && c == wsel) ? pw : 0u;
            tmem_st32(tS + (hf ? 96 : 0), pk);
#pragma unroll
            for (int c = 0; c < 32; ++c) pk[c] = ((row >> 6) == hf && c == wsel) ? pwl : 0u;
            tmem_st32(tS + (hf ? 64 : 32), pk);  // P_lo (second PV pass of the diagonal tile)
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(hf == 0 ? &bars.p_lo[slot] : &bars.p_hi[slot]);
          }
          continue;
        }
        // ONEREAD: the whole S row is read once (raw0 = keys [0,64), raw = keys [64,128)); P(keys
        // 64..127) is written over the already-read S columns [96,128) and published first (p_hi),
        // then P(keys 0..63) over columns [0,32) (p_lo). Otherwise S is read in two 64-column halves
        // (64 registers each): keys [0,64) for their max only, then re-read for P.
        uint32_t raw[64];
#if TTT_FWD_ONEREAD
        uint32_t raw0[64];
#endif
        const int kv0 = (kvt0 + n) * kTile;
        const bool partial = TREE ? (kv0 + kTile > T) : ((n == qt) || (kv0 + kTile > T));
        // TTT: allowed columns c < lim (k <= r and k < T); TREE: per 32-column word bit masks
        const int lim = min(r + 1, T) - kv0;
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        if constexpr (TREE) {
          // column c = key kv0 + c: prefix key (< P) or tree key u = kv0 + c - P of this row's
          // ancestor-or-self mask; rows past the tree (padding of the tile) keep key 0 only
          const unsigned long long am = tree_am;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int c0 = q4 * 32, lo = T - kv0 - c0;  // columns c0 + i < lo are prefix keys
            uint32_t pre = lo >= 32 ? 0xffffffffu : (lo <= 0 ? 0u : ((1u << lo) - 1u));
            // tree bits: column c0 + i holds u = c0 + i - (T - kv0) = i - lo
            uint32_t tb = 0u;
            if (lo < 32 && lo > -64) {
              const int sh = lo;  // bit i of tb = bit (i - sh) of am
              tb = sh >= 0 ? (uint32_t)(am << sh) : (uint32_t)(am >> (-sh));
            }
            w[q4] = pre | tb;
          }
          if (!tree_row) w[0] = w[1] = w[2] = w[3] = 0u, w[0] = (kv0 == 0) ? 1u : 0u;
        }
        // masked columns of half hf (columns 64 hf + c) -> -inf
        auto mask_half = [&](int hf, uint32_t(&rr)[64]) {
#pragma unroll
          for (int c = 0; c < 64; ++c) {
            const int cc = 64 * hf + c;
            const bool ok = TREE ? (((w[cc >> 5] >> (cc & 31)) & 1u) != 0u) : (cc < lim);
            rr[c] = ok ? rr[c] : __float_as_uint(-INFINITY);
          }
        };
        // row max of the raw scores (scale > 0 commutes with max): 8 independent chains of
        // 3-input max (FMNMX3), two new columns per instruction
        float mx8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
        auto max_half = [&](const uint32_t(&rr)[64]) {
#pragma unroll
          for (int c = 0; c < 64; c += 16)
#pragma unroll
            for (int u = 0; u < 8; ++u)
              mx8[u] = fmax3(mx8[u], __uint_as_float(rr[c + u]), __uint_as_float(rr[c + 8 + u]));
        };
#if TTT_FWD_ONEREAD
        tmem_ld128w(tS, raw0, raw);
        if (partial) {
          mask_half(0, raw0);
          mask_half(1, raw);
        }
        max_half(raw0);
        max_half(raw);
#else
        tmem_ld64w(tS, raw);
        if (partial) mask_half(0, raw);
        max_half(raw);
        tmem_ld64w(tS + 64, raw);
        if (partial) mask_half(1, raw);
        max_half(raw);
#endif
        const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * sl2;
        const float m_new = fmaxf(m_run, mx);
        const bool need = m_new > m_run + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          // (TREE: a lane whose row has no allowed key yet has m_run = m_new = -inf; its alpha is 0,
          // not 2^NaN — the branch is warp-uniform)
          const float alpha = (TREE && m_run == -INFINITY) ? 0.f : ex2(m_run - m_new);
          if (n > 0) {  // PV_{n-1} is complete: s_full's commit covers it (rare path: 32-col chunks)
            const uint64_t a2 = f2pack(alpha, alpha);
#pragma unroll 1
            for (int c0 = 0; c0 < D; c0 += 32) {
              uint32_t o[32];
              tmem_ld32(tO + c0, o);
#pragma unroll
              for (int i = 0; i < 32; i += 2) {
                float lo, hi;
                f2unpack(fmul2(f2pack(__uint_as_float(o[i]), __uint_as_float(o[i + 1])), a2), lo, hi);
                o[i] = __float_as_uint(lo);
                o[i + 1] = __float_as_uint(hi);
              }
              tmem_st32(tO + c0, o);
            }
          }
          l_run *= alpha;
          m_run = m_new;
        }
        // P = 2^(s c log2e - m): one FFMA2 per pair, 4 independent pair-sum chains (FADD2),
        // written to TMEM and published per 64-key half (the PV MMA starts on the first)
        // TREE: a row may have no allowed key in this context split yet (m = -inf): exponents
        // against 0 give exact zeros instead of NaN
        const float m_use = (TREE && m_run == -INFINITY) ? 0.f : m_run;
        const uint64_t sl2x2 = f2pack(sl2, sl2), negm = f2pack(-m_use, -m_use);
        uint64_t rs2[4] = {0, 0, 0, 0};
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int hf = 1 - hh;  // keys [64,128) (in registers) first, then [0,64)
#if TTT_FWD_ONEREAD
          if (hf == 0) {
#pragma unroll
            for (int c = 0; c < 64; ++c) raw[c] = raw0[c];  // register renaming only
          }
#else
          if (hf == 0) {
            tmem_ld64w(tS, raw);
            if (partial) mask_half(0, raw);
          }
#endif
          uint32_t pk[32];
          if (partial) {  // masked columns are -inf: hardware ex2 gives exact zeros
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) {
              float x0, x1;
              f2unpack(ffma2(f2pack(__uint_as_float(raw[2 * cc]), __uint_as_float(raw[2 * cc + 1])), sl2x2, negm), x0, x1);
              const float e0 = ex2(x0), e1 = ex2(x1);
              rs2[cc & 3] = fadd2(rs2[cc & 3], f2pack(e0, e1));
              pk[cc] = pack_bf16(e0, e1);
            }
          } else {  // full tile: the pairs TTT_FWD_EMU_MASK selects (of every 8) on the FMA pipe
                    // (MUFU ex2 is the co-bottleneck)
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) {
              float x0, x1, e0, e1;
              f2unpack(ffma2(f2pack(__uint_as_float(raw[2 * cc]), __uint_as_float(raw[2 * cc + 1])), sl2x2, negm), x0, x1);
              if ((TTT_FWD_EMU_MASK >> (cc & 7)) & 1) {
                ex2_emu2(x0, x1, e0, e1);
              } else {
                e0 = ex2(x0);
                e1 = ex2(x1);
              }
              rs2[cc & 3] = fadd2(rs2[cc & 3], f2pack(e0, e1));
              pk[cc] = pack_bf16(e0, e1);
            }
          }
          tmem_st32(tS + (hf ? 96 : 0), pk);
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(hf == 0 ? &bars.p_lo[slot] : &bars.p_hi[slot]);
        }
        {
          float a0, a1, b0, b1, c0, c1, d0, d1;
          f2unpack(rs2[0], a0, a1);
          f2unpack(rs2[1], b0, b1);
          f2unpack(rs2[2], c0, c1);
          f2unpack(rs2[3], d0, d1);
          l_run += ((a0 + a1) + (b0 + b1)) + ((c0 + c1) + (d0 + d1));
        }
        if (threadIdx.x == 0) TTT_TRACE_EV(1, 2, n);
        if (threadIdx.x == 128) TTT_TRACE_EV(2, 2, n);
      }
      if (shd) {
        // ---- SHD: diagonal rows [nrb_d 16, nrb 16) on the softmax warps (same math as warps 10-13) ----
        // 8 lanes per row (lane k owns columns 8k..8k+7 of every 64-column box), 4 rows per warp, both head
        // slots per row; K_i / V_i rows from global memory, the next stage pair's loads issued before the
        // current pair's math.
        constexpr int E = 8 * NBOX;
        const int hw = warp, k8 = lane & 7;            // helper warp 0..7 (0..3 without slot 1)
        const int hrows = (has1 ? 8 : 4) * 4;           // rows per pass
        const int j = p.step;
        const float hsl2 = p.scale_log2;
        const size_t kvrow0 = (size_t)(PACKED ? p.row0[b] : b * p.L);
        for (int hrow = nrb_d * kDgRows + hw * 4 + (lane >> 3); hrow < nrb * kDgRows; hrow += hrows) {
          const int hr = qt * kTile + hrow;
          const bool valid = hr < T;
          float qf[2][E], acc[2][E], m[2], l[2];
          diag_row_init<NBOX>(sQ, TB, hrow, k8, hsl2, qf, acc, m, l);
          const size_t eoff = ((kvrow0 + hr) * p.Hkv + g) * D + k8 * 8;  // this lane's first element
          auto load_step = [&](int i, uint32_t (&kw)[E / 2], uint32_t (&vw)[E / 2]) {
            if (valid && i < j) {
              const __nv_bfloat16* kp = reinterpret_cast<const __nv_bfloat16*>(p.ks[i]) + eoff;
              const __nv_bfloat16* vp = reinterpret_cast<const __nv_bfloat16*>(p.vs[i]) + eoff;
#pragma unroll
              for (int bx = 0; bx < NBOX; ++bx) {
                const uint4 uk = __ldg(reinterpret_cast<const uint4*>(kp + bx * 64));
                const uint4 uv = __ldg(reinterpret_cast<const uint4*>(vp + bx * 64));
                kw[bx * 4 + 0] = uk.x; kw[bx * 4 + 1] = uk.y; kw[bx * 4 + 2] = uk.z; kw[bx * 4 + 3] = uk.w;
                vw[bx * 4 + 0] = uv.x; vw[bx * 4 + 1] = uv.y; vw[bx * 4 + 2] = uv.z; vw[bx * 4 + 3] = uv.w;
              }
            } else {
#pragma unroll
              for (int e = 0; e < E / 2; ++e) kw[e] = vw[e] = 0u;
            }
          };
          uint32_t kc[2][E / 2], vc[2][E / 2];  // current pair
          load_step(0, kc[0], vc[0]);
          load_step(1, kc[1], vc[1]);
          for (int i = 0; i < j; i += 2) {
            const int ns = min(2, j - i);
            uint32_t kn[2][E / 2], vn[2][E / 2];  // next pair, in flight during this pair's math
            load_step(i + 2, kn[0], vn[0]);
            load_step(i + 3, kn[1], vn[1]);
            diag_pair_update<E>(qf, acc, m, l, kc, vc, ns);
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
              for (int e = 0; e < E / 2; ++e) {
                kc[u][e] = kn[u][e];
                vc[u][e] = vn[u][e];
              }
          }
          if (valid)
            diag_row_store<NBOX>(reinterpret_cast<__nv_bfloat16*>(p.out) + ((kvrow0 + hr) * p.Hq + h0) * D, D, k8, has1, acc,
                                 m, l, &bars.a_d[0][hrow], &bars.a_d[1][hrow]);
        }
        fence_async_global();  // the out rows are read back by the producer's TMA (async proxy)
        __threadfence_block();
        mbar_arrive(&bars.diag_done);
      }
      // ---- epilogue: merge the diagonal partial, normalise, store ----
      // The j diagonal keys of row r (Alg. 1 "concat s_i") were reduced
      // by the diagonal warps into (A_d = log2 sum_i 2^{t_i}, O_d = normalised sum); the
      // merge is the same online-softmax update as one more "tile".
      const size_t lse_idx = TREE ? ((size_t)bst * p.Hq + h) * p.L + r : lse_at(p, PACKED, b, h, r);
      const bool has_diag = !TREE && !TTT_FWD_TC_DIAG && (r < T) && (p.step > 0);
      if (threadIdx.x == 0) TTT_TRACE_EV(1, 3, 0);
      mbar_wait(&bars.o_full[slot], 0);
      if (threadIdx.x == 0) TTT_TRACE_EV(1, 4, 0);
      tc_fence_after();
      if (!TREE && !TTT_FWD_TC_DIAG && p.step > 0) {
        if (TTT_FWD_FUSED_DIAG) mbar_wait(&bars.diag_done, 0);  // A_d in shared memory
        mbar_wait(&bars.od, 0);                                 // O_d tile in the Q buffer
      }
      const float A_d = !has_diag ? -INFINITY : TTT_FWD_FUSED_DIAG ? bars.a_d[slot][row] : p.lse[lse_idx];
      // The diagonal partial O_d sits in this slot's Q tile (SW128 boxes); each thread reads its
      // row there and overwrites it in place with the output, which the TMA store then drains.
      // out_lo is staged in the K stage of the same index. Both are free: o_full[slot] and
      // s_done follow every S MMA of the CTA.
      uint8_t* st_hi = sQ + slot * TB;
      uint8_t* st_lo = sK + slot * TB;
      const uint32_t sw = (uint32_t)(row & 7);
      const float m_f = fmaxf(m_run, A_d);
      const float alpha = (TREE && m_f == -INFINITY) ? 0.f : ex2(m_run - m_f);
      const float beta = has_diag ? ex2(A_d - m_f) : 0.f;
      const float l_f = l_run * alpha + beta;
      // TREE: a row with no allowed key in this split leaves O = 0 and lse = -inf (weight 0 in
      // the combine pass)
      const float inv_l = (TREE && l_f == 0.f) ? 0.f : 1.f / l_f;
      const float a_n = alpha * inv_l, b_n = beta * inv_l;
      // packed layout, the sequence's last (partial) tile: rows >= T belong to the next sequence, so
      // each thread stores its own row (r < T) straight to global instead of the 128-row TMA boxes
      const bool direct = !TREE && PACKED && (qt * kTile + kTile > T);
      __nv_bfloat16* const orow = direct ? reinterpret_cast<__nv_bfloat16*>(p.out) + ((size_t)(ry + r) * p.Hq + h) * D : nullptr;
      __nv_bfloat16* const lrow = direct && p.out_lo ? reinterpret_cast<__nv_bfloat16*>(p.out_lo) + ((size_t)(ry + r) * p.Hq + h) * D : nullptr;
      // per 64-column box: one 64-column TMEM load (a single wait), the box written to the staging tile,
      // then its TMA store issued right away so it drains under the next box's math (measured: the
      // epilogue, o_full -> CTA end, took ~8k clk with four 32-column load waits and one store at the end)
#pragma unroll
      for (int bx = 0; bx < NBOX; ++bx) {
        uint32_t o[64];
        tmem_ld64w(tO + bx * 64, o);
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(o[q4 * 8 + e]) * a_n;
          const uint32_t soff = (uint32_t)bx * 16384u + (uint32_t)row * 128u + ((((uint32_t)q4) ^ sw) << 4);
          if (has_diag) {
            const uint4 odv = *reinterpret_cast<const uint4*>(st_hi + soff);
            const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&odv);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 df = __bfloat1622float2(d2[e]);
              v[2 * e] = fmaf(b_n, df.x, v[2 * e]);
              v[2 * e + 1] = fmaf(b_n, df.y, v[2 * e + 1]);
            }
          }
          uint4 w;
          w.x = pack_bf16(v[0], v[1]);
          w.y = pack_bf16(v[2], v[3]);
          w.z = pack_bf16(v[4], v[5]);
          w.w = pack_bf16(v[6], v[7]);
          if (direct) {
            if (r < T) *reinterpret_cast<uint4*>(orow + bx * 64 + q4 * 8) = w;
          } else {
            *reinterpret_cast<uint4*>(st_hi + soff) = w;
          }
          if (p.out_lo) {  // residual O - bf16(O), so the backward's Delta sees ~16-bit O
            const uint32_t hi[4] = {w.x, w.y, w.z, w.w};
            uint32_t lo[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hi[e]));
              lo[e] = pack_bf16(v[2 * e] - hf.x, v[2 * e + 1] - hf.y);
            }
            if (direct) {
              if (r < T) *reinterpret_cast<uint4*>(lrow + bx * 64 + q4 * 8) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            } else {
              *reinterpret_cast<uint4*>(st_lo + soff) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            }
          }
        }
        if (direct) continue;
        fence_async_smem();
        named_bar_sync(1 + slot, 128);
        if (row == 0) {
          if constexpr (TREE) {  // the slot's two heads, 64-row boxes
            for (int k = 2 * slot; k < min(2 * slot + 2, nheads); ++k)
              tma_store_4d(&maps.out, st_hi + bx * 16384 + (k & 1) * 8192, bx * 64, h0 + k, 0, bst);
          } else {
            tma_store_4d(&maps.out, st_hi + bx * 16384, bx * 64, h, ry + qt * kTile, by);
            if (p.out_lo) tma_store_4d(&maps.out_lo, st_lo + bx * 16384, bx * 64, h, ry + qt * kTile, by);
          }
          bulk_commit();
        }
      }
      if (threadIdx.x == 0) TTT_TRACE_EV(1, 6, 0);
      if ((!TREE || tree_row) && !(PACKED && r >= T)) p.lse[lse_idx] = (m_f + log2f(l_f)) * 0.69314718055994531f;
      if (row == 0) {
        if (threadIdx.x == 0) TTT_TRACE_EV(1, 8, 0);
        bulk_wait_read0();  // smem must stay valid until the bulk engine has read it
      }
      if (threadIdx.x == 0) TTT_TRACE_EV(1, 5, 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc(tbase, 512);
#ifdef TTT_TRACE
  if (blockIdx.x == g_ttt_trace_cta && threadIdx.x == 0)
    g_ttt_trace[1][kTraceCap - 3] = (clock64() << 20) | (10ull << 12);  // CTA end
#endif
}

// Diagonal pre-pass (TTT-specific): for every row r < T_b
// and query head h, t_i = c log2(e) q_r . K_i[r] (i = 1..j) reduced by a softmax over i
// (Alg. 1 "concat s_i"):
//   A_d = log2 sum_i 2^{t_i},  O_d = sum_i 2^{t_i - A_d} V_i[r]
// written into lse (log2 units) and out (bf16); the main kernel merges them.
// Per kv row w = (b, r, g) this is two tiny products, S_w = Q_w K_w^T (G x j) and
// O_w = P_w V_w (G x D). A warp does R rows at once with mma.sync: M = R*G query rows
// (w', h), N / K = j*R columns (i, w') i-major, and a block-diagonal mask (w' = w') —
// the padding costs tensor-core slots, which are free here, instead of per-row
// instructions, which bound the kernel (ncu: a CUDA-core version issued ~1300 and a one-row
// mma version ~675 instructions per row, at 26-33% of DRAM bandwidth).
// Pipeline: a producer warp TMA-loads groups of NR consecutive rows (64-column SW128 boxes: q
// as NR*G rows, K_i and V_i as NR rows) into an NS-deep ring; 7 compute warps take items
// round-robin and release a stage through its `empty` mbarrier (no block barriers); O_d and
// A_d leave straight from the mma fragments.
#ifndef TTT_DIAG_STAGE_KB
#define TTT_DIAG_STAGE_KB 0  // dev override of the stage target (KB); 0 = by j (measured: 72 KB for j <= 2, else 100 KB)
#endif
struct DiagLayout {
  int NR, NS, R;
  uint32_t qbytes, kbytes;  // bytes one TMA box delivers (NR G or NR rows x 128 B)
  uint32_t qbox, kbox, off_k, off_v, stage_bytes, total;
  void init(int nr, int g, int d, int j, int ns, int rr) {
    NR = nr;
    NS = ns;
    R = rr;
    const uint32_t nb = (uint32_t)(d / 64);
    qbytes = (uint32_t)nr * g * 128;
    kbytes = (uint32_t)nr * 128;
    qbox = (qbytes + 1023) & ~1023u;  // box allocations 1 KB-aligned (SW128)
    kbox = (kbytes + 1023) & ~1023u;
    off_k = qbox * nb;
    off_v = off_k + (uint32_t)j * nb * kbox;
    stage_bytes = (off_v + (uint32_t)j * nb * kbox + 1023) & ~1023u;
    total = 1024 + (uint32_t)ns * stage_bytes + 1024;  // barriers | stages | alignment slack
  }
};

constexpr int kDiagCompute = 7;  // compute warps (+ 1 producer warp): 256 threads, so up to 255 registers

template <int D>
__global__ void __launch_bounds__(32 * (kDiagCompute + 1), 1)
    ttt_fwd_diag_kernel(const __grid_constant__ Params p, const __grid_constant__ DiagMaps maps, DiagLayout lay) {
  constexpr int NB = D / 64;
  extern __shared__ uint8_t dsm_raw[];
  uint8_t* dsm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm);
  uint64_t* empty = full + 8;
  uint8_t* stages = dsm + 1024;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = p.G, j = p.step, NR = lay.NR, NS = lay.NS, R = lay.R;
  const int nrows = p.B * p.L * p.Hkv;  // < 2^31 (host check)
  const int ngroups = (nrows + NR - 1) / NR;
  const int MT = (G + 15) / 16;  // m-tiles per item (R == 1 when G > 16)
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kDiagCompute);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    // ================= producer: q (NR G rows), K_i, V_i (NR rows) boxes per group =================
    if (lane == 0) {
      tma_prefetch_desc(&maps.q);
      int n = 0;
      for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++n) {
        const int st = n % NS;
        if (n >= NS) mbar_wait(&empty[st], ((n / NS) - 1) & 1);
        uint8_t* base = stages + st * lay.stage_bytes;
        mbar_expect_tx(&full[st], NB * (lay.qbytes + 2u * j * lay.kbytes));  // OOB rows zero-filled, counted
#pragma unroll
        for (int bx = 0; bx < NB; ++bx) {
          tma_load_2d(base + bx * lay.qbox, &maps.q, &full[st], bx * 64, grp * NR * G);
          for (int i = 0; i < j; ++i) {
            tma_load_2d(base + lay.off_k + (i * NB + bx) * lay.kbox, &maps.k[i], &full[st], bx * 64, grp * NR);
            tma_load_2d(base + lay.off_v + (i * NB + bx) * lay.kbox, &maps.v[i], &full[st], bx * 64, grp * NR);
          }
        }
      }
    }
    return;
  }
  // ================= compute warps: R stacked rows per item, round-robin =================
  const int cw = warp - 1;
  const int g8 = lane >> 2, c4 = lane & 3;
  const float sl2 = p.scale_log2;
  const int ncols = j * R;
  const int ipg = (NR + R - 1) / R;
  // per-thread column bookkeeping (independent of the group): column n = i R + w'
  int colw[4][2];  // w' of the thread's C-fragment columns, -1 when n >= j R
#pragma unroll
  for (int nt = 0; nt < 4; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int n = nt * 8 + 2 * c4 + e;
      colw[nt][e] = n < ncols ? n % R : -1;
    }
  int brow_i[4], brow_w[4];  // ldmatrix row (lanes 0-7 of each 8x8) of B n-tile nt: step i, row w'
#pragma unroll
  for (int nt = 0; nt < 4; ++nt) {
    const int n = min(nt * 8 + (lane & 7), ncols - 1);
    brow_i[nt] = n / R;
    brow_w[nt] = n % R;
  }
  int n = 0;
  for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x, ++n) {
    const int st = n % NS;
    mbar_wait(&full[st], (n / NS) & 1);
    const uint32_t sb = smem_u32(stages + st * lay.stage_bytes);
    const int w0 = grp * NR, nv = min(NR, nrows - w0);
    const int nitems = (nv + R - 1) / R;
    for (int k = (cw - (n * ipg) % kDiagCompute + kDiagCompute) % kDiagCompute; k < nitems; k += kDiagCompute) {
      const int lr0 = k * R;
      // rows w' = 0..R-1 of this item: active iff in range and r < T_b (their lse / O are used)
      uint32_t act = 0;
      for (int wq = 0; wq < R && lr0 + wq < nv; ++wq) {
        const uint32_t w = (uint32_t)(w0 + lr0 + wq);
        const uint32_t bl = w / (uint32_t)p.Hkv;
        const int b = (int)(bl / (uint32_t)p.L);
        const int r = (int)(bl - (uint32_t)b * (uint32_t)p.L);
        if (r < p.seq_lens[b]) act |= 1u << wq;
      }
      if (!act) continue;  // warp-uniform; the main kernel ignores such rows
      for (int mt = 0; mt < MT; ++mt) {
        // query row m of the tile: (w', h) = (m / G, m % G) when R > 1, head mt*16 + m when R == 1
        const int mrows = R > 1 ? R * G : min(16, G - mt * 16);
        // ---- S = Q K^T ----
        float s[4][4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
        const uint32_t arow = (uint32_t)(lr0 * G + mt * 16 + min((lane & 7) + ((lane >> 3) & 1) * 8, mrows - 1));
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          uint32_t a[4];
          const uint32_t chunk = (uint32_t)ks * 2 + (lane >> 4);
          ldsm_x4(sb + (chunk >> 3) * lay.qbox + sw128_off(arow, chunk), a);
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) {
            if (nt * 8 < ncols) {
              const uint32_t bch = (uint32_t)ks * 2 + ((lane >> 3) & 1);
              const uint32_t brow = (uint32_t)(lr0 + brow_w[nt]);
              uint32_t bb[2];
              ldsm_x2(sb + lay.off_k + (uint32_t)(brow_i[nt] * NB + (bch >> 3)) * lay.kbox + sw128_off(brow, bch), bb);
              mma_16816(s[nt], a, bb[0], bb[1]);
            }
          }
        }
        // ---- block-diagonal softmax: row m keeps the columns of its own w' ----
        const int m0r = g8, m1r = g8 + 8;
        const int wr0 = R > 1 ? m0r / G : 0, wr1 = R > 1 ? m1r / G : 0;
        const bool ok0 = m0r < mrows && ((act >> wr0) & 1), ok1 = m1r < mrows && ((act >> wr1) & 1);
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            s[nt][e] = (ok0 && colw[nt][e] == wr0) ? s[nt][e] * sl2 : -INFINITY;
            s[nt][2 + e] = (ok1 && colw[nt][e] == wr1) ? s[nt][2 + e] * sl2 : -INFINITY;
            mx0 = fmaxf(mx0, s[nt][e]);
            mx1 = fmaxf(mx1, s[nt][2 + e]);
          }
        }
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float b0 = ok0 ? mx0 : 0.f, b1 = ok1 ? mx1 : 0.f;  // rows without columns: p = 0, no NaN
        float l0 = 0.f, l1 = 0.f;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            s[nt][e] = ex2(s[nt][e] - b0);
            s[nt][2 + e] = ex2(s[nt][2 + e] - b1);
            l0 += s[nt][e];
            l1 += s[nt][2 + e];
          }
        }
        l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
        l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
        const float i0 = ok0 ? 1.f / l0 : 0.f, i1 = ok1 ? 1.f / l1 : 0.f;
        // ---- O = P V (m16n8k8 per 8-column k-tile) ----
        float o[D / 8][4];
#pragma unroll
        for (int dt = 0; dt < D / 8; ++dt) o[dt][0] = o[dt][1] = o[dt][2] = o[dt][3] = 0.f;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          if (nt * 8 < ncols) {
            const uint32_t pa0 = pack_bf16(s[nt][0] * i0, s[nt][1] * i0);
            const uint32_t pa1 = pack_bf16(s[nt][2] * i1, s[nt][3] * i1);
            const uint32_t vrow = (uint32_t)(lr0 + brow_w[nt]);
            const uint32_t vbase = sb + lay.off_v + (uint32_t)(brow_i[nt] * NB) * lay.kbox;
#pragma unroll
            for (int d4 = 0; d4 < D / 32; ++d4) {
              const uint32_t ch = (uint32_t)(d4 * 4 + (lane >> 3));
              uint32_t vb[4];
              ldsm_x4_t(vbase + (ch >> 3) * lay.kbox + sw128_off(vrow, ch), vb);
#pragma unroll
              for (int q = 0; q < 4; ++q) mma_1688(o[d4 * 4 + q], pa0, pa1, vb[q]);
            }
          }
        }
        // ---- O_d -> out (bf16 pairs straight from the fragments), A_d -> lse ----
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int m = g8 + hf * 8;
          if (hf ? ok1 : ok0) {
            const uint32_t w = (uint32_t)(w0 + lr0) + (R > 1 ? (uint32_t)(m / G) : 0u);
            const int h_in = R > 1 ? m % G : mt * 16 + m;
            __nv_bfloat16* orow = reinterpret_cast<__nv_bfloat16*>(p.out) + ((size_t)w * G + h_in) * D + 2 * c4;
#pragma unroll
            for (int dt = 0; dt < D / 8; ++dt)
              *reinterpret_cast<uint32_t*>(orow + dt * 8) = pack_bf16(o[dt][2 * hf], o[dt][2 * hf + 1]);
            if (c4 == 0) {
              const uint32_t bl = w / (uint32_t)p.Hkv;
              const int g = (int)(w - bl * (uint32_t)p.Hkv);
              const int b = (int)(bl / (uint32_t)p.L);
              const int r = (int)(bl - (uint32_t)b * (uint32_t)p.L);
              p.lse[((size_t)b * p.Hq + g * G + h_in) * p.L + r] = hf ? mx1 + log2f(l1) : mx0 + log2f(l0);
            }
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
}

// R rows per warp item: M = R*G <= 16 query rows, j*R <= 32 columns (4 n-tiles); a power of 2.
// NR rows per group: a multiple of R with NR*G <= 256 (TMA box rows), stage ~72-100 KB;
// 4 down to 1 stages.
bool diag_layout(const Params& p, int D, DiagLayout* lay) {
  int R = 1;
  while (R * 2 * p.G <= 16 && R * 2 * p.step <= 32) R *= 2;
  const int row_bytes = (p.G + 2 * p.step) * D * 2;
  const int stage_kb = TTT_DIAG_STAGE_KB > 0 ? TTT_DIAG_STAGE_KB : (p.step <= 2 ? 72 : 100);
  for (int nr = std::max(R, (stage_kb * 1024 / row_bytes) / R * R); nr >= R; nr -= R) {
    if (nr * p.G > 256) continue;
    for (int ns = 4; ns >= 1; --ns) {
      lay->init(nr, p.G, D, p.step, ns, R);
      if (lay->total <= 220 * 1024 && (ns >= 2 || nr == R)) return true;
    }
  }
  return false;
}

template <int D>
cudaError_t launch_fwd_d(const Params& p_in, const FwdMaps& maps, const DiagMaps& dmaps, cudaStream_t st) {
  Params p = p_in;
  if (!p.packed) {  // CTA order: the CTA of q tile qt runs qt + 1 kv tiles (~3.3k clk each) plus ~7k clk of fixed
     // cost (measured traces); a (b, g) group's K / V: 4 B per kv element
    std::vector<double> len(p.nqt);
    for (int r = 0; r < p.nqt; ++r) len[r] = (double)(p.nqt - r) * 3.3;
    p.order_batch = pick_order_batch(p.B * p.Hkv, p.nqt, (p.G + 1) / 2, len.data(), 7.0, (double)p.L * D * 4);
    // at most 4 (b, g) groups per batch: the model (tail balance only) picks 32 at the Llama shape, but fewer
    // groups in flight measured faster (r03s / r03y: 4 groups -1.2% at Llama, -2% at L = 16K; 1-2 slower)
    p.order_batch = std::min(p.order_batch, 4);
    static const int env_ob = dev_env_int("TTT_DEV_FWD_ORDER_BATCH", 0);
    if (env_ob > 0) p.order_batch = env_ob;
  }
  const int smem = fwd_smem_bytes(D);
  static std::atomic<unsigned long long> attr_done{0}, attr_done_pk{0};
  {
    cudaError_t e = set_smem_attr(ttt_fwd_sm100_kernel<D, false, false>, smem, attr_done);
    if (e == cudaSuccess) e = set_smem_attr(ttt_fwd_sm100_kernel<D, false, true>, smem, attr_done_pk);
    if (e != cudaSuccess) return e;
  }
#if !TTT_FWD_FUSED_DIAG
  if (p.packed) return cudaErrorNotSupported;  // the dev-only separate pass knows the padded layout only
  if (p.step > 0) {  // dev A/B: the separate diagonal pre-pass of round 1
    DiagLayout lay;
    if (!diag_layout(p, D, &lay)) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(ttt_fwd_diag_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)lay.total);
    if (e != cudaSuccess) return e;
    const int rows = p.B * p.L * p.Hkv;
    const int groups = (rows + lay.NR - 1) / lay.NR;
    prof_mark(kKindFwdDiag, true, st);
    ttt_fwd_diag_kernel<D><<<std::min(groups, 148), 32 * (kDiagCompute + 1), lay.total, st>>>(p, dmaps, lay);
    prof_mark(kKindFwdDiag, false, st);
  }
#else
  (void)dmaps;
#endif
  const int npairs = (p.G + 1) / 2;
  const int grid = p.ntiles * p.Hkv * npairs;  // padded: ntiles = B nqt
  prof_mark(kKindFwdMain, true, st);
  if (p.packed) ttt_fwd_sm100_kernel<D, false, true><<<grid, kFwdThreads, smem, st>>>(p, maps);
  else ttt_fwd_sm100_kernel<D, false, false><<<grid, kFwdThreads, smem, st>>>(p, maps);
  prof_mark(kKindFwdMain, false, st);
  return cudaGetLastError();
}

}  // namespace

bool fwd_uses_diag_kernel() { return !TTT_FWD_FUSED_DIAG; }

int fwd_diag_rows_per_group(const Params& p) {
  DiagLayout lay;
  return diag_layout(p, p.D, &lay) ? lay.NR : 0;
}

cudaError_t launch_fwd_sm100(const Params& p, const FwdMaps& maps, const DiagMaps& dmaps, cudaStream_t st) {
  return p.D == 64 ? launch_fwd_d<64>(p, maps, dmaps, st) : launch_fwd_d<128>(p, maps, dmaps, st);
}

// ancestor-or-self masks of the draft trees (parents precede children); a parent
// index that is not an earlier node ends the walk (the node then hangs off the context tip)
__global__ void ttt_tree_mask_kernel(const int32_t* parents, int B, int n, unsigned long long* mask) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * n) return;
  const int b = i / n, t = i - b * n;
  const int32_t* par = parents + (size_t)b * n;
  unsigned long long m = 1ull << t;
  int u = par[t], prev = t;
  while (u >= 0 && u < prev) {
    m |= 1ull << u;
    prev = u;
    u = par[u];
  }
  mask[i] = m;
}

// merge the context splits of the tree pass: out = sum_s 2^(lse_s - lse) out_s, lse = logsumexp_s lse_s
// (natural log; one warp per (b, node, head) row, lanes over D)
__global__ void ttt_tree_combine_kernel(const __nv_bfloat16* part, const float* lse_part, int nsplit, int B, int n,
                                        int Hq, int D, __nv_bfloat16* out, float* lse) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= B * n * Hq) return;
  const int h = row % Hq, t = (row / Hq) % n, b = row / (Hq * n);
  float m = -INFINITY;
  for (int s = 0; s < nsplit; ++s) m = fmaxf(m, lse_part[(((size_t)s * B + b) * Hq + h) * n + t]);
  float wsum = 0.f, acc[4] = {0.f, 0.f, 0.f, 0.f};
  const int per = D / 32;  // 2 or 4 consecutive elements per lane
  for (int s = 0; s < nsplit; ++s) {
    const float w = __expf(lse_part[(((size_t)s * B + b) * Hq + h) * n + t] - m);
    wsum += w;
    const __nv_bfloat16* src = part + ((((size_t)s * B + b) * n + t) * Hq + h) * D + lane * per;
    for (int e = 0; e < per; ++e) acc[e] = fmaf(w, __bfloat162float(src[e]), acc[e]);
  }
  const float inv = 1.f / wsum;
  __nv_bfloat16* dst = out + (((size_t)b * n + t) * Hq + h) * D + lane * per;
  for (int e = 0; e < per; ++e) dst[e] = __float2bfloat16_rn(acc[e] * inv);
  if (lane == 0) lse[((size_t)b * Hq + h) * n + t] = m + __logf(wsum);
}

template <int D>
cudaError_t launch_tree_d(const Params& p_in, const FwdMaps& maps, const int32_t* parents, cudaStream_t st) {
  Params p = p_in;
  p.nqt = 1;
  p.order_batch = p.B * p.Hkv;
  const int smem = fwd_smem_bytes(D);
  static std::atomic<unsigned long long> attr_done{0};
  {
    cudaError_t e = set_smem_attr(ttt_fwd_sm100_kernel<D, true, false>, smem, attr_done);
    if (e != cudaSuccess) return e;
  }
  const int nm = p.B * p.tree_n;
  ttt_tree_mask_kernel<<<(nm + 127) / 128, 128, 0, st>>>(parents, p.B, p.tree_n,
                                                        const_cast<unsigned long long*>(p.tree_mask));
  const int grid = p.B * p.Hkv * ((p.G + 3) / 4) * p.tree_splits;
  prof_mark(kKindFwdMain, true, st);
  ttt_fwd_sm100_kernel<D, true, false><<<grid, kFwdThreads, smem, st>>>(p, maps);
  prof_mark(kKindFwdMain, false, st);
  return cudaGetLastError();
}

cudaError_t launch_tree_combine(const void* part, const float* lse_part, int nsplit, int B, int n, int Hq, int D,
                                void* out, float* lse, cudaStream_t st) {
  const int rows = B * n * Hq;
  ttt_tree_combine_kernel<<<(rows + 7) / 8, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(part), lse_part, nsplit,
                                                          B, n, Hq, D, static_cast<__nv_bfloat16*>(out), lse);
  return cudaGetLastError();
}

cudaError_t launch_tree_sm100(const Params& p, const FwdMaps& maps, const int32_t* parents, cudaStream_t st) {
  return p.D == 64 ? launch_tree_d<64>(p, maps, parents, st) : launch_tree_d<128>(p, maps, parents, st);
}

}  // namespace tttk
