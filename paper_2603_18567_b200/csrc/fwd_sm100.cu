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
// shared memory feeds two S = Q K^T MMAs. Warp roles (320 threads):
//   warps 0-3  softmax + epilogue, head slot 0 (TMEM lanes 0-127)
//   warps 4-7  softmax + epilogue, head slot 1
//   warp  8    TMA producer (Q once, then K/V tiles through a 2-stage ring)
//   warp  9    TMEM allocator + single-thread tcgen05.mma issuer
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512);
// P (bf16, packed 2/column) is written over S and consumed by the PV MMA
// straight from TMEM (A operand in TMEM, "ts" form).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "ptx_sm100.cuh"
#include "ttt_params.cuh"

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

constexpr int kFwdThreads = 320;
constexpr float kRescaleThreshold = 8.0f;  // log2 domain: rescale O only when the max grows by > 2^8

struct FwdBars {
  uint64_t q;
  uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[2], p_lo[2], p_hi[2], o_full[2];  // P published in two 64-column halves
  uint32_t tmem_base;
};

template <int D>
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
  __shared__ FwdBars bars;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- work decode: (b, g)-major so one kv head's K/V stay hot in L2; within
  // it the longest (highest) q tiles first; head pairs of a tile adjacent ----
  const int npairs = (p.G + 1) >> 1;
  const int hp = (int)blockIdx.x % npairs;
  const int t_ = (int)blockIdx.x / npairs;
  const int qt = p.nqt - 1 - t_ % p.nqt;
  const int g = (t_ / p.nqt) % p.Hkv;
  const int b = t_ / (p.nqt * p.Hkv);
  const int h0 = g * p.G + 2 * hp;
  const bool has1 = (2 * hp + 1) < p.G;
  const int T = p.seq_lens[b];
  const int nkv = min(qt + 1, (T + kTile - 1) / kTile);  // BlockMask: skip k0 > q0+127 and k0 >= T

  if (threadIdx.x == 0) {
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
    fence_mbar_init();
  }
  if (warp == 9) {
    tmem_alloc(&bars.tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = bars.tmem_base;

  if (warp == 8) {
    // ================= TMA producer =================
    if (lane == 0) {
      tma_prefetch_desc(&maps.q);
      tma_prefetch_desc(&maps.k);
      tma_prefetch_desc(&maps.v);
      mbar_expect_tx(&bars.q, (has1 ? 2 : 1) * TB);
#pragma unroll
      for (int bx = 0; bx < NBOX; ++bx) {
        tma_load_4d(sQ + bx * 16384, &maps.q, &bars.q, bx * 64, h0, qt * kTile, b);
        if (has1) tma_load_4d(sQ + TB + bx * 16384, &maps.q, &bars.q, bx * 64, h0 + 1, qt * kTile, b);
      }
      for (int n = 0; n < nkv; ++n) {
        const int st = n & 1, ph = (n >> 1) & 1;
        mbar_wait(&bars.k_empty[st], ph ^ 1);
        mbar_expect_tx(&bars.k_full[st], TB);
#pragma unroll
        for (int bx = 0; bx < NBOX; ++bx)
          tma_load_4d(sK + st * TB + bx * 16384, &maps.k, &bars.k_full[st], bx * 64, g, n * kTile, b);
        mbar_wait(&bars.v_empty[st], ph ^ 1);
        mbar_expect_tx(&bars.v_full[st], TB);
#pragma unroll
        for (int bx = 0; bx < NBOX; ++bx)
          tma_load_4d(sV + st * TB + bx * 16384, &maps.v, &bars.v_full[st], bx * 64, g, n * kTile, b);
      }
    }
  } else if (warp == 9) {
    // ================= MMA issuer (whole warp, converged; elect.sync inside each issue) =================
    {
      constexpr uint32_t idS = idesc_bf16_f32(128, 128, false, false);  // S = Q K^T, both K-major
      constexpr uint32_t idO = idesc_bf16_f32(128, D, false, true);     // O += P V, V MN-major
      const uint64_t dQ0 = sdesc_sw128(smem_u32(sQ), 16, 1024), dK0 = sdesc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t dV0 = sdesc_sw128(smem_u32(sV), 16384, 1024);
      auto issue_S = [&](int slot, int kst) {
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks) {
          const uint32_t off = (ks >> 2) * 16384 + (ks & 3) * 32;
          umma_ss_e(tbase + slot * 128, sdesc_add(dQ0, slot * TB + off), sdesc_add(dK0, kst * TB + off), idS, ks > 0);
        }
      };
      // O += P V in two halves of the key dimension: keys [0,64) as soon as the softmax warps have
      // published P's first half (p_lo), keys [64,128) after p_hi
      auto issue_PV = [&](int slot, int vst, bool acc, int n) {
        mbar_wait(&bars.p_lo[slot], n & 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          umma_ts_e(tbase + 256 + slot * 128, tbase + slot * 128 + ks * 8, sdesc_add(dV0, vst * TB + ks * 2048), idO,
                    (acc || ks > 0) ? 1u : 0u);
        mbar_wait(&bars.p_hi[slot], n & 1);
        tc_fence_after();
#pragma unroll
        for (int ks = 4; ks < 8; ++ks)
          umma_ts_e(tbase + 256 + slot * 128, tbase + slot * 128 + ks * 8, sdesc_add(dV0, vst * TB + ks * 2048), idO, 1u);
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
      for (int n = 0; n < nkv; ++n) {
        const int vst = n & 1, vph = (n >> 1) & 1;
        const bool more = n + 1 < nkv;
        const int kst = (n + 1) & 1, kph = ((n + 1) >> 1) & 1;
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
  } else {
    // ================= softmax + epilogue (warps 0-7) =================
    const int slot = warp >> 2;
    const int wq = warp & 3;
    if (slot == 0 || has1) {
      const int row = wq * 32 + lane;
      const int r = qt * kTile + row;
      const int h = h0 + slot;
      const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
      const uint32_t tS = tbase + lane_off + slot * 128;
      const uint32_t tO = tbase + lane_off + 256 + slot * 128;
      const float sl2 = p.scale_log2;
      float m_run = -INFINITY, l_run = 0.f;
      TTT_TRACE_DECL(1);
      TTT_TRACE_DECL(2);
      for (int n = 0; n < nkv; ++n) {
        mbar_wait(&bars.s_full[slot], n & 1);
        if (threadIdx.x == 0) TTT_TRACE_EV(1, 1, n);
        if (threadIdx.x == 128) TTT_TRACE_EV(2, 1, n);
        tc_fence_after();
        uint32_t raw[128];
        tmem_ld128(tS, raw);
        const int kv0 = n * kTile;
        const bool partial = (n == qt) || (kv0 + kTile > T);
        // row max of the raw scores (scale > 0 commutes with max): 8 independent chains
        float mx8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
        if (partial) {
          const int lim = min(r + 1, T) - kv0;  // allowed columns c < lim  (k <= r and k < T)
#pragma unroll
          for (int c = 0; c < 128; ++c) {
            const float x = c < lim ? __uint_as_float(raw[c]) : -INFINITY;
            raw[c] = __float_as_uint(x);
            mx8[c & 7] = fmaxf(mx8[c & 7], x);
          }
        } else {
#pragma unroll
          for (int c = 0; c < 128; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], __uint_as_float(raw[c]));
        }
        const float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7]))) * sl2;
        const float m_new = fmaxf(m_run, mx);
        const bool need = m_new > m_run + kRescaleThreshold;
        if (__any_sync(0xffffffffu, need)) {
          const float alpha = ex2(m_run - m_new);
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
        // written to TMEM and published in two 64-column halves (the PV MMA starts on the first)
        const uint64_t sl2x2 = f2pack(sl2, sl2), negm = f2pack(-m_run, -m_run);
        uint64_t rs2[4] = {0, 0, 0, 0};
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          uint32_t pk[32];
          if (partial) {  // masked columns are -inf: hardware ex2 gives exact zeros
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) {
              const int c = hf * 32 + cc;
              float x0, x1;
              f2unpack(ffma2(f2pack(__uint_as_float(raw[2 * c]), __uint_as_float(raw[2 * c + 1])), sl2x2, negm), x0, x1);
              const float e0 = ex2(x0), e1 = ex2(x1);
              rs2[c & 3] = fadd2(rs2[c & 3], f2pack(e0, e1));
              pk[cc] = pack_bf16(e0, e1);
            }
          } else {  // full tile: every 4th pair on the FMA pipe (MUFU ex2 is the co-bottleneck)
#pragma unroll
            for (int cc = 0; cc < 32; ++cc) {
              const int c = hf * 32 + cc;
              float x0, x1, e0, e1;
              f2unpack(ffma2(f2pack(__uint_as_float(raw[2 * c]), __uint_as_float(raw[2 * c + 1])), sl2x2, negm), x0, x1);
              if ((c & 3) == 3) {
                ex2_emu2(x0, x1, e0, e1);
              } else {
                e0 = ex2(x0);
                e1 = ex2(x1);
              }
              rs2[c & 3] = fadd2(rs2[c & 3], f2pack(e0, e1));
              pk[cc] = pack_bf16(e0, e1);
            }
          }
          tmem_st32(tS + 32 * hf, pk);
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
      // ---- epilogue: merge the diagonal partial (fwd_diag_kernel), normalise, store ----
      // The j diagonal keys of row r (Alg. 1 "concat s_i") were reduced
      // by ttt_fwd_diag_kernel into (A_d = log2 sum_i 2^{t_i}, O_d = normalised sum); the
      // merge is the same online-softmax update as one more "tile".
      const size_t q_off = (((size_t)b * p.L + r) * p.Hq + h) * D;
      const size_t lse_idx = ((size_t)b * p.Hq + h) * p.L + r;
      const __nv_bfloat16* orow = reinterpret_cast<const __nv_bfloat16*>(p.out) + q_off;
      const bool has_diag = (r < T) && (p.step > 0);
      uint4 od[D / 8];
      float A_d = -INFINITY;
      if (has_diag) {
        A_d = p.lse[lse_idx];
#pragma unroll
        for (int c = 0; c < D / 8; ++c) od[c] = *reinterpret_cast<const uint4*>(orow + c * 8);
      }
      if (threadIdx.x == 0) TTT_TRACE_EV(1, 3, 0);
      mbar_wait(&bars.o_full[slot], 0);
      if (threadIdx.x == 0) TTT_TRACE_EV(1, 4, 0);
      tc_fence_after();
      // Staging tiles for the TMA stores (SW128 boxes of 64 columns, same layout the loads use).
      // o_full[slot] follows every S MMA of the CTA in issue order, so the K stages (slot 0) and
      // the Q tiles (slot 1) are no longer read by the tensor core.
      uint8_t* st_hi = slot == 0 ? sK : sQ;
      uint8_t* st_lo = st_hi + TB;
      const uint32_t sw = (uint32_t)(row & 7);
      const float m_f = fmaxf(m_run, A_d);
      const float alpha = ex2(m_run - m_f);
      const float beta = has_diag ? ex2(A_d - m_f) : 0.f;
      const float l_f = l_run * alpha + beta;
      const float inv_l = 1.f / l_f;
      const float a_n = alpha * inv_l, b_n = beta * inv_l;
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t o[32];
        tmem_ld32(tO + c0, o);
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(o[q4 * 8 + e]) * a_n;
          if (has_diag) {
            const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&od[c0 / 8 + q4]);
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
          const int col = c0 + q4 * 8;
          const uint32_t soff = (uint32_t)(col >> 6) * 16384u + (uint32_t)row * 128u + ((((uint32_t)(col & 63) >> 3) ^ sw) << 4);
          *reinterpret_cast<uint4*>(st_hi + soff) = w;
          if (p.out_lo) {  // residual O - bf16(O), so the backward's Delta sees ~16-bit O
            const uint32_t hi[4] = {w.x, w.y, w.z, w.w};
            uint32_t lo[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 hf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&hi[e]));
              lo[e] = pack_bf16(v[2 * e] - hf.x, v[2 * e + 1] - hf.y);
            }
            *reinterpret_cast<uint4*>(st_lo + soff) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
          }
        }
      }
      p.lse[lse_idx] = (m_f + log2f(l_f)) * 0.69314718055994531f;
      fence_async_smem();
      named_bar_sync(1 + slot, 128);
      if (row == 0) {
#pragma unroll
        for (int bx = 0; bx < D / 64; ++bx) {
          tma_store_4d(&maps.out, st_hi + bx * 16384, bx * 64, h, qt * kTile, b);
          if (p.out_lo) tma_store_4d(&maps.out_lo, st_lo + bx * 16384, bx * 64, h, qt * kTile, b);
        }
        bulk_commit();
        bulk_wait_read0();  // smem must stay valid until the bulk engine has read it
      }
      if (threadIdx.x == 0) TTT_TRACE_EV(1, 5, 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc(tbase, 512);
}

// Diagonal pre-pass (TTT-specific): for every row r < T_b
// and query head h, t_i = c log2(e) q_r . K_i[r] (i = 1..j) reduced with an online
// softmax over i (Alg. 1 "concat s_i"):
//   A_d = log2 sum_i 2^{t_i},  O_d = sum_i 2^{t_i - A_d} V_i[r]
// written into lse (log2 units) and out (bf16); the main kernel merges them.
// HBM-streaming, TMA-staged: a persistent block walks groups of NR consecutive
// (b, r, g) rows; q (NR*G*D), K_i and V_i (NR*D each) of a group are single
// contiguous blocks moved by 1-D cp.async.bulk into a double-buffered stage.
struct DiagLayout {
  int NR;
  uint32_t off_q, off_k, off_v, stage_bytes, total;
  __host__ __device__ void init(int nr, int g, int d, int j) {
    NR = nr;
    off_q = 0;
    off_k = (uint32_t)nr * g * d * 2;
    off_v = off_k + (uint32_t)j * nr * d * 2;
    stage_bytes = (off_v + (uint32_t)j * nr * d * 2 + 127) & ~127u;
    total = 2 * stage_bytes + 64;
  }
};

template <int D>
__global__ void __launch_bounds__(512) ttt_fwd_diag_kernel(const __grid_constant__ Params p, DiagLayout lay) {
  constexpr int E = D / 16, H = D / 32;
  extern __shared__ __align__(128) uint8_t dsm[];
  const int tid = threadIdx.x, hl = tid & 15, pair = tid >> 4;
  const int NR = lay.NR, G = p.G, j = p.step;
  const long nrows = (long)p.B * p.L * p.Hkv;
  const long ngroups = (nrows + NR - 1) / NR;
  uint64_t* full = reinterpret_cast<uint64_t*>(dsm + lay.total - 64);
  // one half-warp per (row, query head); lane hl owns elements [hl*H, +H) and [D/2 + hl*H, +H)
  const bool ghost = pair >= NR * G;
  const int pc = ghost ? 0 : pair;
  const int lr = pc / G, hh = pc % G;
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](long grp, int st) {  // thread 0 only
    const long w0 = grp * NR;
    const int nv = (int)min((long)NR, nrows - w0);
    uint8_t* base = dsm + st * lay.stage_bytes;
    const uint32_t qb = (uint32_t)nv * G * D * 2, kb = (uint32_t)nv * D * 2;
    mbar_expect_tx(&full[st], qb + 2 * j * kb);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(base + lay.off_q)),
                 "l"(reinterpret_cast<const __nv_bfloat16*>(p.q) + (size_t)w0 * G * D), "r"(qb),
                 "r"(smem_u32(&full[st]))
                 : "memory");
    for (int i = 0; i < j; ++i) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(base + lay.off_k + i * NR * D * 2)),
                   "l"(reinterpret_cast<const __nv_bfloat16*>(p.ks[i]) + (size_t)w0 * D), "r"(kb),
                   "r"(smem_u32(&full[st]))
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(base + lay.off_v + i * NR * D * 2)),
                   "l"(reinterpret_cast<const __nv_bfloat16*>(p.vs[i]) + (size_t)w0 * D), "r"(kb),
                   "r"(smem_u32(&full[st]))
                   : "memory");
    }
  };
  auto lds = [&](const uint8_t* row, float (&x)[E]) {
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      const uint8_t* src = row + (part * (D / 2) + hl * H) * 2;
      if constexpr (H == 4) {  // bf16 -> fp32: one shift / mask per element
        const uint2 u = *reinterpret_cast<const uint2*>(src);
        x[part * 4 + 0] = __uint_as_float(u.x << 16);
        x[part * 4 + 1] = __uint_as_float(u.x & 0xFFFF0000u);
        x[part * 4 + 2] = __uint_as_float(u.y << 16);
        x[part * 4 + 3] = __uint_as_float(u.y & 0xFFFF0000u);
      } else {
        const uint32_t u = *reinterpret_cast<const uint32_t*>(src);
        x[part * 2 + 0] = __uint_as_float(u << 16);
        x[part * 2 + 1] = __uint_as_float(u & 0xFFFF0000u);
      }
    }
  };
  long grp = blockIdx.x;
  if (tid == 0 && grp < ngroups) issue(grp, 0);
  for (int n = 0; grp < ngroups; ++n, grp += gridDim.x) {
    const int st = n & 1;
    const long nxt = grp + gridDim.x;
    if (tid == 0 && nxt < ngroups) issue(nxt, st ^ 1);  // stage st^1 was released by the last __syncthreads
    mbar_wait(&full[st], (n >> 1) & 1);
    const uint8_t* base = dsm + st * lay.stage_bytes;
    const long w = grp * NR + lr;
    const bool valid = !ghost && w < nrows;
    const long wc = w < nrows ? w : grp * NR;
    const int g = (int)(wc % p.Hkv);
    const int r = (int)((wc / p.Hkv) % p.L);
    const int b = (int)(wc / ((long)p.Hkv * p.L));
    const bool act = valid && r < p.seq_lens[b];
    float qf[E], o[E];
    lds(base + lay.off_q + (uint32_t)(lr * G + hh) * D * 2, qf);
#pragma unroll
    for (int e = 0; e < E; ++e) o[e] = 0.f;
    float m = -INFINITY, l = 0.f;
    for (int i = 0; i < j; ++i) {
      float kk[E], vv[E];
      lds(base + lay.off_k + (uint32_t)(i * NR + lr) * D * 2, kk);
      lds(base + lay.off_v + (uint32_t)(i * NR + lr) * D * 2, vv);
      float acc = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) acc = fmaf(qf[e], kk[e], acc);
      const float t = half_allsum(acc) * p.scale_log2;  // s_i = c q_r . k_i (log2 units)
      const float mn = fmaxf(m, t);
      const float a = ex2(m - mn), wgt = ex2(t - mn);
      l = l * a + wgt;
#pragma unroll
      for (int e = 0; e < E; ++e) o[e] = fmaf(wgt, vv[e], o[e] * a);
      m = mn;
    }
    if (act) {
      const int h = g * G + hh;
      const size_t q_off = (((size_t)b * p.L + r) * p.Hq + h) * D;
      const float inv = 1.f / l;
      __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(p.out) + q_off;
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        __nv_bfloat16* dst = op + part * (D / 2) + hl * H;
        if constexpr (H == 4)
          *reinterpret_cast<uint2*>(dst) = make_uint2(pack_bf16(o[part * 4] * inv, o[part * 4 + 1] * inv),
                                                      pack_bf16(o[part * 4 + 2] * inv, o[part * 4 + 3] * inv));
        else
          *reinterpret_cast<uint32_t*>(dst) = pack_bf16(o[part * 2] * inv, o[part * 2 + 1] * inv);
      }
      if (hl == 0) p.lse[((size_t)b * p.Hq + h) * p.L + r] = m + log2f(l);
    }
    __syncthreads();  // stage st fully consumed before it is refilled
  }
}

template <int D>
cudaError_t launch_fwd_d(const Params& p, const FwdMaps& maps, cudaStream_t st) {
  const int smem = 6 * kTile * D * 2 + 1024;
  static bool attr_set = false;  // benign race: idempotent attribute set
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(ttt_fwd_sm100_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  if (p.step > 0) {
    DiagLayout lay;
    int nr = std::max(1, 32 / p.G);  // 32 half-warps (512 threads) of (row, head) pairs
    for (; nr > 1; nr >>= 1) {
      lay.init(nr, p.G, D, p.step);
      if (lay.total <= 200 * 1024) break;
    }
    lay.init(nr, p.G, D, p.step);
    if (lay.total > 227 * 1024) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaFuncSetAttribute(ttt_fwd_diag_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)lay.total);
    if (e != cudaSuccess) return e;
    const long rows = (long)p.B * p.L * p.Hkv;
    const long groups = (rows + nr - 1) / nr;
    const int per_sm = lay.total <= 110 * 1024 ? 2 : 1;
    const int blocks = (int)std::min<long>(groups, 148L * per_sm);
    prof_mark(kKindFwdDiag, true, st);
    const int threads = std::min(512, std::max(32, ((nr * p.G * 16 + 31) / 32) * 32));
    ttt_fwd_diag_kernel<D><<<blocks, threads, lay.total, st>>>(p, lay);
    prof_mark(kKindFwdDiag, false, st);
  }
  const int npairs = (p.G + 1) / 2;
  const int grid = p.nqt * p.B * p.Hkv * npairs;
  prof_mark(kKindFwdMain, true, st);
  ttt_fwd_sm100_kernel<D><<<grid, kFwdThreads, smem, st>>>(p, maps);
  prof_mark(kKindFwdMain, false, st);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fwd_sm100(const Params& p, const FwdMaps& maps, cudaStream_t st) {
  return p.D == 64 ? launch_fwd_d<64>(p, maps, st) : launch_fwd_d<128>(p, maps, st);
}

}  // namespace tttk
