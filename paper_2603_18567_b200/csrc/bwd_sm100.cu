// bwd_sm100.cu — TTT attention backward on sm_100a.
//
// Recompute-based (no saved probabilities): P = exp(S - lse) is
// rebuilt from the forward's lse. Three kernels per call, all on `stream`:
//
//  1. ttt_bwd_pre_kernel (HBM-streaming, CUDA cores), one warp per (b, r, kv head g):
//       Delta_{h,r} = dO_{h,r} . O_{h,r};  lse2 = lse * log2(e)
//       TTT diagonal keys (the j step entries of row r < T_b, Alg. 2 M_suffix,
//       PAPER.md:305-309): p_i = exp(c q.K_i[r] - lse), dp_i = dO.V_i[r],
//       ds_i = p_i (dp_i - Delta), dq_acc[r] = c sum_i ds_i K_i[r] (initialises the
//       fp32 dq accumulator), dK_i[r] (+)= c sum_h ds_i q_h, dV_i[r] (+)= sum_h p_i dO_h.
//       Zeroes dK_0/dV_0 rows when not accumulating (the main kernel adds into them).
//  2. ttt_bwd_sm100_kernel (tcgen05), KV-outer: one CTA per (b, g, 128-key tile kt,
//     head subset); loops over its query heads x causal q tiles qt >= kt:
//       S^T = K Q^T, dP^T = V dO^T                         (SS MMAs, TMEM)
//       P^T = exp2(S^T c log2e - lse2), dS^T = P^T o (dP^T - Delta)   (compute warps)
//       dV += P^T dO, dK += dS^T Q                         (A operand from TMEM)
//       dQ  = dS K  -> TMA reduce-add into dq_acc           (A = dS from smem)
//  3. ttt_bwd_dq_convert_kernel: dq = bf16(dq_acc).
// dq_acc is a tile-contiguous fp32 workspace (see dqacc_index) reduced into by TMA.
//
// Warp roles of the main kernel (512 threads, setmaxnreg-rebalanced; see ttt_bwd_sm100_kernel):
//   warps 0-3 dQ drain (thread = query row), warps 4-7 / 8-11 compute for the 64-query sub-items
//   a / b (thread = key row, TMEM lanes 0-127), warp 12 TMEM owner + MMA issuer, warp 13 TMA
//   producer, warps 14-15 idle.
// TMEM columns: S^T[a,b] [0,128) dP^T[a,b] / dS^T, aliased by dQ [128,256) dV [256,256+D) dK [384,384+D).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "ptx_sm100.cuh"
#include "ttt_params.cuh"

namespace tttk {
#ifdef TTT_TRACE
__device__ unsigned long long g_ttt_trace[4][kTraceCap];
__device__ unsigned int g_ttt_trace_cta;
#endif
namespace {

constexpr float kLog2e = 1.4426950408889634f;
#ifndef TTT_BWD_DK_SS
#define TTT_BWD_DK_SS 0  // dev: 1 = dK as an SS MMA from the shared-memory dS^T with dQ between dK(a) and dK(b) (r02t: 4.73 vs 4.61 ms, slower)
#endif
#ifndef TTT_BWD_DQ_RED
#define TTT_BWD_DQ_RED 0  // dev: dQ drain by red.global.add.v4 instead of staged TMA reduce-adds
#endif
#ifndef TTT_BWD_ORDER
#define TTT_BWD_ORDER 0  // dev: MMA issue order of an item's dP / dV halves (see the MMA warp)
#endif
#ifndef TTT_BWD_DQ_HALVES
#define TTT_BWD_DQ_HALVES 1  // 1: the dQ drain frees dP^T[a] after its first 64 columns, so dP(t+1,a) need
                             // not wait for the whole 128-column read-out
#endif
#ifndef TTT_BWD_DQT
#define TTT_BWD_DQT 0  // dev, 1 (D = 128): dQ^T = K^T dS^T per 64-query sub-item (M = D, N = 64) so the two sub-items'
                       // dP -> dS -> dK -> dQ -> drain chains run independently; 0: one dQ = dS K per tile.
                       // Measured (r03b / r03e): 5.11 vs 4.66 ms per unroll (5.06 with the reduce-adds probed out):
                       // the two N = 64 SS MMAs (48 clk per K step) and the serial per-sub-item drain cost more
                       // than the decoupled chains gain
#endif
#if TTT_BWD_DQT && (TTT_BWD_DK_SS || TTT_BWD_DQ_RED || TTT_BWD_ORDER)
#error "the per-sub-item dQ^T path has no DK_SS / DQ_RED / ORDER variants; build them with TTT_BWD_DQT=0"
#endif
#ifndef TTT_BWD_LSU_LOADS
#define TTT_BWD_LSU_LOADS 0  // dev, 1: Q / lse2 / Delta (warp 14) and dO halves (warp 15) by cp.async on the LSU path, so
                             // they do not queue in the SM's TMA engine behind the dQ reduce-adds; 0: TMA loads.
                             // Measured (r03d): 6.64 vs 4.63 ms per unroll (cp.async tiles arrive later than TMA's)
#endif
#if TTT_BWD_DQ_HALVES && TTT_BWD_ORDER == 1
#error "TTT_BWD_ORDER == 1 waits on the whole-tile dq_empty; build it with TTT_BWD_DQ_HALVES=0"
#endif
#ifndef TTT_BWD_PSPLIT
#define TTT_BWD_PSPLIT 1  // P phase: a mask-free copy of the exp loop for full tiles
#endif
#ifndef TTT_BWD_EMU_MASK
#define TTT_BWD_EMU_MASK 0  // quads (c4 mod 8) of the P phase whose 2^x runs as an FMA-pipe polynomial (r03f: none 4.57, 1 in 8 4.58, 1 in 4 4.58, 1 in 2 4.61 ms)
#endif
#ifndef TTT_BWD_PROBE
#define TTT_BWD_PROBE 0  // dev timing probes (wrong results): 1 = no dQ reduce-adds, 2 = Q / dO loaded for the first two
                         // items only (later items reuse the stale tiles). r03e: 4.63 -> 3.99 (1), 4.31 (2) ms per
                         // unroll: the dQ egress and the load latency are each only part of the per-item period
#endif
#ifndef TTT_BWD_PREFETCH
#define TTT_BWD_PREFETCH 0  // dev: items of L2-prefetch lookahead for Q / dO in the main kernel (2 measured
                            // 5.03 vs 4.76 ms per unroll, r02f: off)
#endif

__device__ __forceinline__ float warp_allsum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <int E>
__device__ __forceinline__ void load_bf16(const void* base, size_t off, float (&x)[E]) {
  const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(base) + off;
  if constexpr (E == 4) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
    const float2 c = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
    x[0] = a.x; x[1] = a.y; x[2] = c.x; x[3] = c.y;
  } else {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u));
    x[0] = a.x; x[1] = a.y;
  }
}

// dq_acc workspace layout (tile-contiguous so a warp's 32 rows x 32 columns of a
// dQ tile are one 4 KB block the TMA reduce-add writes in full 128 B lines):
//   [B][Hq][L/128][D/32][128 rows][32 cols] fp32
__device__ __forceinline__ size_t dqacc_index(const Params& p, int b, int h, int r, int d) {
  const int nc = p.D / 32;
  return ((dq_tile(p, p.packed, b, h, r >> 7) * nc + (d >> 5)) * 128 + (r & 127)) * 32 + (d & 31);
}

// ------------------------------------------------------------------ kernel 1
// Diagonal / preprocess pass, an HBM stream. Per kv row w = (b, r, g) with G query heads
// and the j diagonal keys K_i[r], V_i[r] (Alg. 2 M_suffix):
//   Delta_h = dO_h . (O_h + O_lo_h),  lse2_h = lse_h log2 e          (all rows)
//   S = Q K^T, dP = dO V^T          (G x j),  P = 2^(S c log2e - lse2) on the allowed set
//   dS = P o (dP - Delta);  dq_acc = c dS K  (initialises the fp32 dq accumulator)
//   dK_i[r] (+)= c dS^T Q,  dV_i[r] (+)= P^T dO     (GQA sums fall out of the products)
// Tiny matrices per row, so a compute warp takes R rows at once with mma.sync: M = R G query
// rows (w', h), N = j R columns (i, w') i-major, block-diagonal mask (as in the forward
// diagonal pass). Delta is the diagonal of dO (O + O_lo)^T on the same tensor pipe.
// Pipeline: one producer warp TMA-loads groups of NR rows (SW128 boxes: dO, O, O_lo, q as
// NR G rows, K_i and V_i as NR rows) into an NS-deep ring; compute warps take items
// round-robin and release a stage through its `empty` mbarrier — no block barriers. Outputs
// leave straight from the mma fragments: dq_acc (tiled fp32) and -Delta / -lse2 by plain
// stores, dK_i / dV_i by st.global.v2 (overwrite) or red.global.add.v2 (accumulate; L2 does
// the read-modify-write), so no stage space is spent on fp32 outputs.
#ifndef TTT_PRE_WARPS
#define TTT_PRE_WARPS 8
#endif
constexpr int kPreCompute = TTT_PRE_WARPS;  // compute warps (+ 1 producer warp)
// n / d for 0 <= n < 2^31 by multiply-high (Granlund-Montgomery): the pre-pass decodes a kv row
// w = (b L + r) Hkv + g per query row and item, and runtime divisions were ~20 instructions each
struct FastDiv {
  uint32_t d, mul, shift;
  void init(uint32_t div) {
    d = div;
    shift = 0;
    while ((1u << shift) < div) ++shift;
    mul = (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << shift) - div)) / div + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, mul) + n) >> shift; }
};
struct PreLayout {
  int NR, NS, R, lgR, has_lo;
  FastDiv div_hkv, div_L;
  uint32_t qbytes, kbytes;  // bytes one TMA box delivers (NR G or NR rows x 128 B)
  uint32_t qbox, kbox, off_do, off_o, off_olo, off_q, off_k, off_v, stage_bytes, off_scr, total;
  void init(int nr, int g, int d, int j, int ns, int rr, int lo) {
    NR = nr;
    NS = ns;
    R = rr;
    lgR = 0;
    while ((1 << lgR) < rr) ++lgR;
    has_lo = lo;
    const uint32_t nb = (uint32_t)(d / 64);
    qbytes = (uint32_t)nr * g * 128;
    kbytes = (uint32_t)nr * 128;
    qbox = (qbytes + 1023) & ~1023u;  // box allocations 1 KB-aligned (SW128)
    kbox = (kbytes + 1023) & ~1023u;
    off_do = 0;
    off_o = off_do + nb * qbox;
    off_olo = off_o + nb * qbox;
    off_q = off_olo + (lo ? nb * qbox : 0u);
    off_k = off_q + (j > 0 ? nb * qbox : 0u);
    off_v = off_k + (uint32_t)j * nb * kbox;
    stage_bytes = (off_v + (uint32_t)j * nb * kbox + 1023) & ~1023u;
    off_scr = 1024 + (uint32_t)ns * stage_bytes;             // per compute warp: P, dS bf16 [16][40]
    total = off_scr + kPreCompute * 2 * 1280 + 1024;         // + alignment slack
  }
};

// U = true: the unroll-level pass of ttt_attn_bwd_unroll. Each row group is visited once per
// step j = S-1 .. 0 (items (group, j), per-step q / dO / O / O_lo maps and lse / Delta / lse2 /
// dq_acc pointers from `up`), in sweeps over M groups: for M groups, every step, so a group's
// dK_i / dV_i rows (first written at j = S-1, then reduce-added by j < S-1) and its K_i / V_i rows
// (re-read by every j >= i) stay in L2 between visits — HBM sees one write of dK_i / dV_i and one
// read of K_i / V_i per unroll instead of one per call. Ordering of a row's store before its
// reduce-adds: the item -> warp mapping depends on the group only and an element's (lane, register)
// slot depends on (i, row, column) only, so both come from the same thread in program order
// (a per-stage __threadfence here measured 20% of the pass's stall samples, r02a ncu).
template <int D, bool U, bool PACKED>
__global__ void __launch_bounds__(32 * (kPreCompute + 1), 1)
    ttt_bwd_pre_kernel(const __grid_constant__ Params p, const __grid_constant__ PreMaps maps,
                       const __grid_constant__ UnrollPre up, PreLayout lay) {
  constexpr int NB = D / 64;
  extern __shared__ uint8_t psm_raw[];
  uint8_t* psm = psm_raw + ((1024u - (smem_u32(psm_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(psm);
  uint64_t* empty = full + 8;
  uint8_t* stages = psm + 1024;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = p.G, NR = lay.NR, NS = lay.NS, R = lay.R;
  const int nrows = p.nrows * p.Hkv;  // kv rows (B L or sum T_b) x Hkv < 2^31 (host check)
  const int ngroups = (nrows + NR - 1) / NR;
  const int ng = (ngroups - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;  // this CTA's groups
  const int S = U ? up.S : 1;
  // groups per j-sweep starting at group index g0 of this CTA (the tail joins the last sweep)
  auto sweep = [&](int g0) { return U ? ((ng - g0 >= 2 * up.M) ? up.M : ng - g0) : 1; };
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kPreCompute);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ================= producer =================
    if (lane == 0) {
      int n = 0;
      for (int g0 = 0; g0 < ng;) {
        const int msg = sweep(g0);
        for (int jj = 0; jj < S; ++jj) {
          const int j = U ? S - 1 - jj : p.step;
          const CUtensorMap* mdo = U ? &up.dout[j] : &maps.dout;
          const CUtensorMap* mo = U ? &up.o[j] : &maps.o;
          const CUtensorMap* molo = U ? &up.olo[j] : &maps.olo;
          const CUtensorMap* mq = U ? &up.q[j] : &maps.q;
          const uint32_t bytes =
              NB * ((2u + (lay.has_lo ? 1u : 0u) + (j > 0 ? 1u : 0u)) * lay.qbytes + 2u * j * lay.kbytes);
          for (int gi = 0; gi < msg; ++gi, ++n) {
            const int grp = (int)blockIdx.x + (g0 + gi) * (int)gridDim.x;
            const int st = n % NS;
            if (n >= NS) mbar_wait(&empty[st], ((n / NS) - 1) & 1);
            if (U && jj > 0 && msg < NS) {  // the same group's previous step released (see above)
              const int m = n - msg;
              mbar_wait(&empty[m % NS], (m / NS) & 1);
            }
            uint8_t* base = stages + st * lay.stage_bytes;
            mbar_expect_tx(&full[st], bytes);  // full boxes (OOB rows are zero-filled and counted)
            const int rq = grp * NR * G, rk = grp * NR;
#pragma unroll
            for (int bx = 0; bx < NB; ++bx) {
              tma_load_2d(base + lay.off_do + bx * lay.qbox, mdo, &full[st], bx * 64, rq);
              tma_load_2d(base + lay.off_o + bx * lay.qbox, mo, &full[st], bx * 64, rq);
              if (lay.has_lo) tma_load_2d(base + lay.off_olo + bx * lay.qbox, molo, &full[st], bx * 64, rq);
              if (j > 0) tma_load_2d(base + lay.off_q + bx * lay.qbox, mq, &full[st], bx * 64, rq);
              for (int i = 0; i < j; ++i) {
                tma_load_2d(base + lay.off_k + (i * NB + bx) * lay.kbox, &maps.k[i], &full[st], bx * 64, rk);
                tma_load_2d(base + lay.off_v + (i * NB + bx) * lay.kbox, &maps.v[i], &full[st], bx * 64, rk);
              }
            }
          }
        }
        g0 += msg;
      }
    }
    return;
  }

  // ================= compute warps =================
  const int cw = warp - 1;
  const int g8 = lane >> 2, c4 = lane & 3;
  const float sl2 = p.scale_log2, cs = p.scale;
  const int MT = (G + 15) / 16;     // 16-row tiles of query rows (R == 1 when G > 16)
  const int ipg = (NR + R - 1) >> lay.lgR;
  // the thread's two fragment rows m = g8, g8 + 8 of a 16-row tile: (row w' of the item, head) when
  // R > 1 (R G <= 16 rows); for R == 1 the head is mt 16 + m (computed per tile)
  int wr_m[2], hh_m[2];
#pragma unroll
  for (int hf = 0; hf < 2; ++hf) {
    const int m = g8 + hf * 8;
    wr_m[hf] = R > 1 ? m / G : 0;
    hh_m[hf] = R > 1 ? m % G : m;
  }
  auto decode = [&](uint32_t w, int& b_, int& r_, int& g_) {  // w = (b L + r) Hkv + g
    const uint32_t bl = lay.div_hkv.div(w);
    g_ = (int)(w - bl * (uint32_t)p.Hkv);
    b_ = PACKED ? seq_of_row(p, true, (int)bl) : (int)lay.div_L.div(bl);
    r_ = (int)bl - (PACKED ? p.row0[b_] : b_ * p.L);
  };
  uint8_t* scrP = psm + lay.off_scr + cw * 2560;  // [16 rows m][40] bf16 (80-B rows: conflict-free)
  uint8_t* scrS = scrP + 1280;
  const uint32_t sP = smem_u32(scrP), sS = smem_u32(scrS);
  int n = 0;
  for (int g0 = 0; g0 < ng;) {
    const int msg = sweep(g0);
    for (int jj = 0; jj < S; ++jj) {
      const int j = U ? S - 1 - jj : p.step;
      const float* lse_in = U ? up.lse_in[j] : p.lse_in;
      float* delta_p = U ? up.delta[j] : p.delta;
      float* lse2_p = U ? up.lse2[j] : p.lse2;
      float* dq_acc_p = U ? up.dq_acc[j] : p.dq_acc;
      // dK_i / dV_i: stored by the first contribution (overwrite mode, j = S-1), else reduce-added
      const bool radd = U ? (p.accumulate != 0 || j != S - 1) : (p.accumulate != 0);
      const int ncols = j * R;
      const int NT = (ncols + 7) / 8;   // 8-column tiles of S / dP (<= 4)
      const int MT2 = (ncols + 15) / 16;  // 16-row tiles of dK / dV (<= 2)
      int colw[4][2];  // w' of the thread's C-fragment columns, -1 past j R
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = nt * 8 + 2 * c4 + e;
          colw[nt][e] = c < ncols ? (c & (R - 1)) : -1;
        }
      int brow_i[4], brow_w[4];  // ldmatrix row (lane & 7) of column tile nt: step i, row w'
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = ncols > 0 ? min(nt * 8 + (lane & 7), ncols - 1) : 0;
        brow_i[nt] = c >> lay.lgR;
        brow_w[nt] = c & (R - 1);
      }
      for (int gi = 0; gi < msg; ++gi, ++n) {
        const int grp = (int)blockIdx.x + (g0 + gi) * (int)gridDim.x;
        const int st = n % NS;
        const int w0 = grp * NR, nv = min(NR, nrows - w0);
        const int nitems = (nv + R - 1) >> lay.lgR;
        // items of this group owned by this warp: item id gidx*ipg + k, round-robin over warps. The
        // mapping depends on the group's position only (not on j), so in the unroll pass the SAME
        // thread writes a given dK_i / dV_i element at every step: its j = S-1 store and the later
        // steps' reduce-adds are ordered by program order (no fence, no cross-warp hand-off)
        const int gidx = g0 + gi;
        const int k_first = (cw - (gidx * ipg) % kPreCompute + kPreCompute) % kPreCompute;
        // the first item's lse rows are a global load: issue it before waiting for the stage's TMA
        // data so its latency overlaps that wait (it sat on the item's critical path)
        float lse_pf[2] = {0.f, 0.f};
        if (k_first < nitems) {
#pragma unroll
          for (int hf = 0; hf < 2; ++hf) {
            const int m = g8 + hf * 8;
            const int mrows0 = R > 1 ? R * G : min(16, G);
            const int wr0 = wr_m[hf], hh0 = hh_m[hf];
            if (m < mrows0 && k_first * R + wr0 < nv) {
              int b_, r_, g_;
              decode((uint32_t)(w0 + k_first * R + wr0), b_, r_, g_);
              lse_pf[hf] = lse_in[lse_at(p, PACKED, b_, g_ * G + hh0, r_)];
            }
          }
        }
        mbar_wait(&full[st], (n / NS) & 1);
        const uint32_t sb = smem_u32(stages + st * lay.stage_bytes);
        for (int k = k_first; k < nitems; k += kPreCompute) {
          const int lr0 = k * R;
          for (int mt = 0; mt < MT; ++mt) {
            const int mrows = R > 1 ? R * G : min(16, G - mt * 16);
            // ---- the thread's two query rows (g8, g8 + 8): (w', head), validity, lse2 ----
            int wr[2], hh[2], bb[2], rr[2], gg[2];
            bool okr[2], act[2];
            float l2[2];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              const int m = g8 + hf * 8;
              wr[hf] = wr_m[hf];
              hh[hf] = R > 1 ? hh_m[hf] : mt * 16 + m;
              okr[hf] = m < mrows && lr0 + wr[hf] < nv;
              decode((uint32_t)(w0 + min(lr0 + wr[hf], nv - 1)), bb[hf], rr[hf], gg[hf]);
              act[hf] = okr[hf] && rr[hf] < p.seq_lens[bb[hf]];
              l2[hf] = okr[hf] ? ((k == k_first && mt == 0) ? lse_pf[hf]
                                                          : lse_in[lse_at(p, PACKED, bb[hf], gg[hf] * G + hh[hf], rr[hf])]) *
                                     kLog2e
                               : 0.f;
            }
            // ---- S = Q K^T, dP = dO V^T, Delta = diag(dO (O + O_lo)^T) ----
            float s[4][4], dp[4][4], cd[2][4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
#pragma unroll
              for (int e = 0; e < 4; ++e) s[t][e] = dp[t][e] = 0.f;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) cd[0][e] = cd[1][e] = 0.f;
            const uint32_t qrow0 = (uint32_t)(lr0 * G + mt * 16);
            const uint32_t arow = qrow0 + (uint32_t)min((lane & 7) + ((lane >> 3) & 1) * 8, mrows - 1);
            const uint32_t orow = qrow0 + (uint32_t)min((lane & 7) + ((lane >> 4) & 1) * 8, mrows - 1);  // B: rows m'
#pragma unroll 2
            for (int ks = 0; ks < D / 16; ++ks) {
              const uint32_t ach = (uint32_t)ks * 2 + (lane >> 4);
              uint32_t ado[4];
              ldsm_x4(sb + lay.off_do + (ach >> 3) * lay.qbox + sw128_off(arow, ach), ado);
              {  // Delta: B = O rows m' (n-tiles m' 0-7, 8-15), k = 16 columns of D
                const uint32_t och = (uint32_t)ks * 2 + ((lane >> 3) & 1);
                uint32_t bo[4];
                ldsm_x4(sb + lay.off_o + (och >> 3) * lay.qbox + sw128_off(orow, och), bo);
                mma_16816(cd[0], ado, bo[0], bo[1]);
                mma_16816(cd[1], ado, bo[2], bo[3]);
                if (lay.has_lo) {
                  ldsm_x4(sb + lay.off_olo + (och >> 3) * lay.qbox + sw128_off(orow, och), bo);
                  mma_16816(cd[0], ado, bo[0], bo[1]);
                  mma_16816(cd[1], ado, bo[2], bo[3]);
                }
              }
              if (ncols > 0) {
                uint32_t aq[4];
                ldsm_x4(sb + lay.off_q + (ach >> 3) * lay.qbox + sw128_off(arow, ach), aq);
                const uint32_t bch = (uint32_t)ks * 2 + ((lane >> 3) & 1);
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                  if (nt < NT) {
                    const uint32_t brow = (uint32_t)(lr0 + brow_w[nt]);
                    const uint32_t boff = (uint32_t)(brow_i[nt] * NB + (bch >> 3)) * lay.kbox + sw128_off(brow, bch);
                    uint32_t bk[2], bv[2];
                    ldsm_x2(sb + lay.off_k + boff, bk);
                    ldsm_x2(sb + lay.off_v + boff, bv);
                    mma_16816(s[nt], aq, bk[0], bk[1]);
                    mma_16816(dp[nt], ado, bv[0], bv[1]);
                  }
                }
              }
            }
            // Delta of row m sits at column m: thread (g8, c4 = g8 / 2), element g8 & 1 (rows g8, g8 + 8)
            float del[2];
            {
              const int src = g8 * 4 + (g8 >> 1);
              const float d0 = (g8 & 1) ? cd[0][1] : cd[0][0];
              const float d1 = (g8 & 1) ? cd[1][3] : cd[1][2];
              del[0] = __shfl_sync(0xffffffffu, d0, src);
              del[1] = __shfl_sync(0xffffffffu, d1, src);
            }
            // ---- P and c dS on the allowed (block-diagonal) entries; bf16 copies to the scratch ----
            uint32_t pa[4][2], da[4][2];  // A fragments (m16n8k8) of P and c dS per column tile
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              if (nt < NT) {
                float pv[4], dv[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int hf = e >> 1;
                  const bool ok = act[hf] && colw[nt][e & 1] == wr[hf];
                  const float pr = ok ? ex2(s[nt][e] * sl2 - l2[hf]) : 0.f;  // p_i = exp(c q.k_i - lse)
                  pv[e] = pr;
                  dv[e] = cs * pr * (dp[nt][e] - del[hf]);  // c ds_i, ds_i = p_i (dp_i - Delta)
                }
                pa[nt][0] = pack_bf16(pv[0], pv[1]);
                pa[nt][1] = pack_bf16(pv[2], pv[3]);
                da[nt][0] = pack_bf16(dv[0], dv[1]);
                da[nt][1] = pack_bf16(dv[2], dv[3]);
                const uint32_t o0 = (uint32_t)g8 * 80 + (uint32_t)(nt * 8 + 2 * c4) * 2;
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(sP + o0), "r"(pa[nt][0]));
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(sP + o0 + 640), "r"(pa[nt][1]));
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(sS + o0), "r"(da[nt][0]));
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(sS + o0 + 640), "r"(da[nt][1]));
              }
            }
            __syncwarp();
            // ---- dq_acc = c dS K (zeros at j = 0), -Delta, -lse2 ----
            size_t qbase[2];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
              const int h = gg[hf] * G + hh[hf];
              qbase[hf] = ((dq_tile(p, PACKED, bb[hf], h, rr[hf] >> 7) * (D / 32)) * 128 + (rr[hf] & 127)) * 32;
              if (okr[hf] && c4 == 0) {
                const size_t li = ws_at(p, PACKED, bb[hf], h, rr[hf]);
                delta_p[li] = -del[hf];  // stored negated: the main kernel's FFMA2 / FADD2 consume -lse2, -Delta
                lse2_p[li] = -l2[hf];
              }
            }
#pragma unroll
            for (int d4 = 0; d4 < D / 32; ++d4) {
              float acc[4][4];
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = acc[q][2] = acc[q][3] = 0.f;
#pragma unroll
              for (int nt = 0; nt < 4; ++nt) {
                if (nt < NT) {
                  const uint32_t ch = (uint32_t)(d4 * 4 + (lane >> 3));
                  const uint32_t brow = (uint32_t)(lr0 + brow_w[nt]);
                  uint32_t kb[4];
                  ldsm_x4_t(sb + lay.off_k + (uint32_t)(brow_i[nt] * NB + (ch >> 3)) * lay.kbox + sw128_off(brow, ch), kb);
#pragma unroll
                  for (int q = 0; q < 4; ++q) mma_1688(acc[q], da[nt][0], da[nt][1], kb[q]);
                }
              }
#pragma unroll
              for (int hf = 0; hf < 2; ++hf) {
                if (okr[hf]) {
#pragma unroll
                  for (int q = 0; q < 4; ++q) {
                    const int d = (d4 * 4 + q) * 8 + 2 * c4;
                    *reinterpret_cast<float2*>(dq_acc_p + qbase[hf] + (size_t)(d >> 5) * 4096 + (d & 31)) =
                        make_float2(acc[q][2 * hf], acc[q][2 * hf + 1]);
                  }
                }
              }
            }
            // ---- dK_i = (c dS)^T Q, dV_i = P^T dO: rows n = (i, w'), K = the 16 query rows ----
            for (int t2 = 0; t2 < MT2; ++t2) {
              // A' = (c dS)^T / P^T: ldmatrix.trans of the [m][n] scratch, matrices (m 0-7 | 8-15) x (n 0-7 | 8-15)
              const int mi = lane >> 3;
              const uint32_t aoff = (uint32_t)(((mi >> 1) * 8 + (lane & 7)) * 80 + (t2 * 16 + (mi & 1) * 8) * 2);
              uint32_t ads[4], ap[4];
              ldsm_x4_t(sS + aoff, ads);
              ldsm_x4_t(sP + aoff, ap);
              // output rows of this tile: n = t2*16 + g8 (+8) -> (i, w')
              int oi[2], ow[2];
              bool ook[2];
#pragma unroll
              for (int hf = 0; hf < 2; ++hf) {
                const int nn = t2 * 16 + g8 + hf * 8;
                oi[hf] = nn >> lay.lgR;
                ow[hf] = nn & (R - 1);
                ook[hf] = nn < ncols && lr0 + ow[hf] < nv;
              }
              const uint32_t brow = qrow0 + (uint32_t)min((mi & 1) * 8 + (lane & 7), mrows - 1);  // B' rows m
#pragma unroll 2
              for (int dc = 0; dc < D / 8; dc += 2) {
                const uint32_t ch = (uint32_t)(dc + (mi >> 1));
                uint32_t bq[4], bo[4];
                ldsm_x4_t(sb + lay.off_q + (ch >> 3) * lay.qbox + sw128_off(brow, ch), bq);
                ldsm_x4_t(sb + lay.off_do + (ch >> 3) * lay.qbox + sw128_off(brow, ch), bo);
                float k0[4] = {0.f, 0.f, 0.f, 0.f}, k1[4] = {0.f, 0.f, 0.f, 0.f};
                float v0[4] = {0.f, 0.f, 0.f, 0.f}, v1[4] = {0.f, 0.f, 0.f, 0.f};
                mma_16816(k0, ads, bq[0], bq[1]);
                mma_16816(k1, ads, bq[2], bq[3]);
                mma_16816(v0, ap, bo[0], bo[1]);
                mma_16816(v1, ap, bo[2], bo[3]);
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                  if (ook[hf]) {
                    const size_t ro = (size_t)(w0 + lr0 + ow[hf]) * D;
                    float* dk = p.dks[oi[hf]] + ro;
                    float* dv = p.dvs[oi[hf]] + ro;
                    const int d0 = dc * 8 + 2 * c4, d1 = d0 + 8;
                    if (radd) {
                      asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(dk + d0), "f"(k0[2 * hf]), "f"(k0[2 * hf + 1]) : "memory");
                      asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(dk + d1), "f"(k1[2 * hf]), "f"(k1[2 * hf + 1]) : "memory");
                      asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(dv + d0), "f"(v0[2 * hf]), "f"(v0[2 * hf + 1]) : "memory");
                      asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(dv + d1), "f"(v1[2 * hf]), "f"(v1[2 * hf + 1]) : "memory");
                    } else if (mt == 0) {
                      *reinterpret_cast<float2*>(dk + d0) = make_float2(k0[2 * hf], k0[2 * hf + 1]);
                      *reinterpret_cast<float2*>(dk + d1) = make_float2(k1[2 * hf], k1[2 * hf + 1]);
                      *reinterpret_cast<float2*>(dv + d0) = make_float2(v0[2 * hf], v0[2 * hf + 1]);
                      *reinterpret_cast<float2*>(dv + d1) = make_float2(v1[2 * hf], v1[2 * hf + 1]);
                    } else {  // G > 16: later head tiles add to the first tile's values (same thread wrote them)
                      float2* a = reinterpret_cast<float2*>(dk + d0);
                      float2* c = reinterpret_cast<float2*>(dk + d1);
                      float2* e2 = reinterpret_cast<float2*>(dv + d0);
                      float2* f2 = reinterpret_cast<float2*>(dv + d1);
                      float2 x = *a; *a = make_float2(x.x + k0[2 * hf], x.y + k0[2 * hf + 1]);
                      x = *c; *c = make_float2(x.x + k1[2 * hf], x.y + k1[2 * hf + 1]);
                      x = *e2; *e2 = make_float2(x.x + v0[2 * hf], x.y + v0[2 * hf + 1]);
                      x = *f2; *f2 = make_float2(x.x + v1[2 * hf], x.y + v1[2 * hf + 1]);
                    }
                  }
                }
              }
            }
            __syncwarp();  // scratch reused by the next item / head tile
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
    }
    g0 += msg;
  }
}

// ------------------------------------------------------------------ kernel 2
struct BwdBars {
  uint64_t kv_full;
  uint64_t q_full[2], q_empty[2];
  uint64_t do_full, do_empty;
  uint64_t s_full, dp_full, p_full, ds_full, ds_empty, dq_full, dq_empty, acc_full;
  uint32_t tmem_base;
};

__device__ __forceinline__ void bulk_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
template <uint32_t N>
__device__ __forceinline__ void reg_alloc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <uint32_t N>
__device__ __forceinline__ void reg_dealloc() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}
// two back-to-back 32-column TMEM loads, one wait (64 regs)
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%64];\n"
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%65];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr), "r"(taddr + 32)
      : "memory");
}

// Work item = one 128-query tile (head h, tile qt) split into two 64-query
// sub-items x = a, b, each with its own S^T / dP^T buffers in TMEM and its own
// compute warpgroup. dQ (M = 128 queries, N = D) aliases the two dP^T buffers,
// so the next dP waits for the dQ drain only; the issue order (MMA warp) keeps
// the tensor pipe busy with dV while dQ is drained.
// Warp roles (16 warps; setmaxnreg rebalances the register file):
//   warps 0-3   dQ drain            (thread = query row of TMEM lane quadrant w)
//   warps 4-7   compute sub-item a  (thread = key row, 64 query columns)
//   warps 8-11  compute sub-item b
//   warp  12    TMEM owner + MMA issuer, warp 13 TMA producer, warps 14-15 idle
// Per SMSP: {dQ 152, compute 136, compute 136, role 88 / idle 24} <= 512 registers.
// TMEM: S^T[a] [0,64) S^T[b] [64,128) dP^T[a] [128,192) dP^T[b] [192,256) dV [256,+D) dK [384,+D);
// P^T / dS^T (bf16, 2 per column) over the first 32 columns of their own S / dP buffer.
// Shared memory (D = 128): K, V 64 KB | Q 2 x 32 KB | dO 3 x 16 KB ring of 64-row halves |
// dS 32 KB ([kv][q], two 64-query SW128 boxes) | lse2, Delta 2 KB | dQ staging 4 x 4 KB.
constexpr int kBwdThreads = 512;
// setmaxnreg split per SMSP (warps s, 4+s, 8+s, 12+s): dQ drain + 2 compute + role (MMA / TMA / idle) <= 512
#ifndef TTT_BWD_DS_ONEWAIT
#define TTT_BWD_DS_ONEWAIT 0  // dev, 1: dS phase loads dP^T with one 64-column TMEM load (152-register split); r04b: equal (4.55-4.56 ms)
#endif
#ifndef TTT_BWD_REG_CMP
#define TTT_BWD_REG_CMP (TTT_BWD_DS_ONEWAIT ? 152 : 136)
#endif
#ifndef TTT_BWD_REG_DRAIN
#define TTT_BWD_REG_DRAIN 152
#endif
constexpr uint32_t kBwdRegDrain = TTT_BWD_REG_DRAIN, kBwdRegCmp = TTT_BWD_REG_CMP, kBwdRegRole = 512 - kBwdRegDrain - 2 * kBwdRegCmp;
static_assert(kBwdRegRole >= 24, "register file per SMSP");

template <int D>
struct BwdSmem {
  static constexpr int TB = kTile * D * 2;  // 128 x D bf16 tile
  static constexpr int HB = TB / 2;         // 64 x D half tile
  static constexpr int oK = 0, oV = TB, oQ = 2 * TB, oDO = 4 * TB, oDS = 4 * TB + 3 * HB;
  static constexpr int oL = oDS + 32768, oDel = oL + 1024, oDQ = oDel + 1024, oBar = oDQ + 16384;
  static constexpr int bytes = oBar + 256;
};

struct BwdBars3 {
  uint64_t kv_full;
  uint64_t q_full[2], q_empty[2];
  uint64_t do_full[3], do_empty[3];
  uint64_t s_full[2], dp_full[2], p_full[2], ds_full[2];
  uint64_t ds_empty, dq_full, dq_empty, acc_full;
  uint64_t dq_empty_h[2];  // DQ_HALVES: dQ columns [64x, 64x + 64) (over dP^T[x]) read out
  uint64_t dq_full_x[2], ds_empty_x[2];  // DQT: dQ^T(t, x) in TMEM; dS(t, x) smem box read by dQ^T(t, x)
  uint32_t tmem_base;
};

template <int D, bool PACKED>
__global__ void __launch_bounds__(kBwdThreads, 1)
    ttt_bwd_sm100_kernel(const __grid_constant__ Params p, const __grid_constant__ BwdMaps maps) {
  using SM = BwdSmem<D>;
  constexpr int TB = SM::TB, HB = SM::HB;
  constexpr bool DQT = TTT_BWD_DQT && D == 128;  // D = 64 keeps the per-tile dQ = dS K (M = 64 would run at half rate)
  constexpr int NBOX = D / 64;
  // dynamic smem only (no static __shared__): the window base is 1024-B aligned, checked below
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sK = smem + SM::oK;
  uint8_t* sV = smem + SM::oV;
  uint8_t* sQ = smem + SM::oQ;    // 2 stages of 128 x D
  uint8_t* sDO = smem + SM::oDO;  // 3-slot ring of 64 x D halves (boxes of 64 rows x 64 cols)
  uint8_t* sDS = smem + SM::oDS;  // 128 x 128 bf16, [kv][q], box x = sub-item x
  float* sL = reinterpret_cast<float*>(smem + SM::oL);     // [2][128] -lse2
  float* sDel = reinterpret_cast<float*>(smem + SM::oDel);  // [2][128] -Delta
  uint8_t* sDQ = smem + SM::oDQ;                            // 4 warps x 4 KB dQ staging (SW128)
  BwdBars3& bars = *reinterpret_cast<BwdBars3*>(smem + SM::oBar);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hsplit = p.head_split;
  const int nh = p.G / hsplit;
  // (b, g, head subset)-major, kv tile fastest (ascending = longest first): the CTAs of one
  // kv head run together, so its Q / dO tiles and dq_acc rows stay hot in L2. (A global
  // longest-first order — kv tile slowest — measured slower: 5.3 vs 5.26 ms bwd, 2.73-2.85 vs
  // 2.63-2.66 ms fwd per unroll in an interleaved A/B, bench_tools/ab.sh.)
  int kt, grp;
  if (PACKED) {
    // packed: (tile, kv head, head subset), head subsets fastest; each sequence's kv tiles in
    // ascending order (the longest CTAs of the sequence first)
    const int per = p.Hkv * p.head_split;
    const int tt = (int)blockIdx.x / per;
    const int bq = seq_of_tile(p, true, tt);
    kt = tt - p.tile0[bq];
    grp = bq * per + (int)blockIdx.x % per;
  } else {
#ifdef TTT_ORDER_GROUP
  kt = (int)blockIdx.x % p.nqt;
  grp = (int)blockIdx.x / p.nqt;
#else
  // Batched longest-first: kv heads in batches of p.order_batch; inside a batch kv tile slowest (the
  // longest CTAs, kt = 0, first), then the batch's heads. The last batch ends with short CTAs (a
  // small tail), while one batch's Q / dO / dq_acc (~8 x 8 MB at the Llama shape) stay in L2.
  const int ngrp = p.B * p.Hkv * p.head_split;
  const int bsz = p.order_batch * p.nqt;
  const int bat = (int)blockIdx.x / bsz, gbase = bat * p.order_batch;
  const int gb = min(p.order_batch, ngrp - gbase), rr = (int)blockIdx.x - bat * bsz;
  kt = rr / gb;
  grp = gbase + rr % gb;
#endif
  }
  const int hs = grp % hsplit;
  const int g = (grp / hsplit) % p.Hkv;
  const int b = grp / (hsplit * p.Hkv);
  const int T = p.seq_lens[b];
  if (kt * kTile >= T) return;  // every key of the tile is padding: no gradient flows
  const int nqt_b = PACKED ? p.tile0[b + 1] - p.tile0[b] : p.nqt;  // q tiles of this sequence
  // TMA (row, batch) origin of this sequence: (0, b) padded, (row0[b], 0) packed
  const int ry = PACKED ? p.row0[b] : 0, by = PACKED ? 0 : b;
  const int nq = nqt_b - kt;
  const int n_items = nh * nq;  // 128-query tiles
  const int h_first = g * p.G + hs * nh;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0) __trap();  // SW128 tiles need 1 KB alignment

  // producer: the loads of item t (Q tile + lse2 / Delta, then the two dO halves), each after its slot is free
  auto issue_item = [&](int t) {
#ifdef TTT_TRACE
    int trace_n_2 = 32768 + 4 * t;
#endif
    const int h = h_first + t / nq, qt = kt + t % nq;
    const int qs = t & 1, qph = (t >> 1) & 1;
    if (TTT_BWD_PREFETCH && t + TTT_BWD_PREFETCH < n_items) {
      // L2 prefetch of a later item's Q and dO tiles: the 2-slot Q / 3-half dO rings give ~1 item
      // of lookahead, less than a TMA load's latency when the tile is not in L2 (r02e trace: the
      // MMA pipe idled ~0.8k clk per item waiting for dO halves)
      const int tp = t + TTT_BWD_PREFETCH;
      const int hp = h_first + tp / nq, qtp = kt + tp % nq;
#pragma unroll
      for (int bx = 0; bx < NBOX; ++bx) {
        tma_prefetch_4d(&maps.q, bx * 64, hp, ry + qtp * kTile, by);
        tma_prefetch_4d(&maps.dout, bx * 64, hp, ry + qtp * kTile, by);
      }
    }
    mbar_wait(&bars.q_empty[qs], qph ^ 1);
    if (TTT_BWD_PROBE == 2 && t >= 2) {  // dev probe: no loads after the first two items
      mbar_arrive(&bars.q_full[qs]);
      for (int x = 0; x < 2; ++x) {
        const int u = 2 * t + x, slot = u % 3, use = u / 3;
        mbar_wait(&bars.do_empty[slot], (use & 1) ^ 1);
        mbar_arrive(&bars.do_full[slot]);
      }
      return;
    }
    mbar_expect_tx(&bars.q_full[qs], TB + 1024);
#pragma unroll
    for (int bx = 0; bx < NBOX; ++bx)
      tma_load_4d(sQ + qs * TB + bx * 16384, &maps.q, &bars.q_full[qs], bx * 64, h, ry + qt * kTile, by);
    const size_t li = ws_at(p, PACKED, b, h, qt * kTile);
    bulk_load_1d(sL + qs * 128, p.lse2 + li, 512, &bars.q_full[qs]);
    bulk_load_1d(sDel + qs * 128, p.delta + li, 512, &bars.q_full[qs]);
    TTT_TRACE_EV(2, 11, t);
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const int u = 2 * t + x, slot = u % 3, use = u / 3;
      mbar_wait(&bars.do_empty[slot], (use & 1) ^ 1);
      mbar_expect_tx(&bars.do_full[slot], HB);
#pragma unroll
      for (int bx = 0; bx < NBOX; ++bx)
        tma_load_4d(sDO + slot * HB + bx * (HB / NBOX), &maps.dout64, &bars.do_full[slot], bx * 64, h,
                    ry + qt * kTile + 64 * x, by);
      TTT_TRACE_EV(2, 12 + x, t);
    }
  };
  // The TMA producer thread (warp 13, lane 0) initialises the barriers and issues K / V and item 0's loads
  // before the CTA-wide barrier, so their latency overlaps the TMEM allocation and the sync.
  if (threadIdx.x == 416) {
    mbar_init(&bars.kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars.q_full[i], TTT_BWD_LSU_LOADS ? 32 : 1);  // LSU: one noinc arrive per loader lane
      mbar_init(&bars.q_empty[i], 1);
      mbar_init(&bars.s_full[i], 1);
      mbar_init(&bars.dp_full[i], 1);
      mbar_init(&bars.p_full[i], 128);
      mbar_init(&bars.ds_full[i], 128);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&bars.do_full[i], TTT_BWD_LSU_LOADS ? 32 : 1);
      mbar_init(&bars.do_empty[i], 1);
    }
    mbar_init(&bars.ds_empty, 1);
    mbar_init(&bars.dq_full, 1);
    mbar_init(&bars.dq_empty, 128);
    mbar_init(&bars.dq_empty_h[0], 128);
    mbar_init(&bars.dq_empty_h[1], 128);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars.dq_full_x[i], 1);
      mbar_init(&bars.ds_empty_x[i], 1);
    }
    mbar_init(&bars.acc_full, 1);
    fence_mbar_init();
    tma_prefetch_desc(&maps.q);
    tma_prefetch_desc(&maps.k);
    tma_prefetch_desc(&maps.v);
    tma_prefetch_desc(&maps.dout);
    mbar_expect_tx(&bars.kv_full, 2 * TB);
#pragma unroll
    for (int bx = 0; bx < NBOX; ++bx) {
      tma_load_4d(sK + bx * 16384, &maps.k, &bars.kv_full, bx * 64, g, ry + kt * kTile, by);
      tma_load_4d(sV + bx * 16384, &maps.v, &bars.kv_full, bx * 64, g, ry + kt * kTile, by);
    }
    if (!TTT_BWD_LSU_LOADS) issue_item(0);  // n_items >= 1
  }
  if (warp == 12) {
    tmem_alloc(&bars.tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = bars.tmem_base;

  if (warp == 13) {
    // ================= TMA producer =================
    reg_dealloc<kBwdRegRole>();
    if (lane == 0)
      for (int t = 1; t < (TTT_BWD_LSU_LOADS ? 0 : n_items); ++t) issue_item(t);
  } else if (warp == 12) {
    // ================= MMA issuer (whole warp, converged; elect.sync inside each issue) =================
    reg_dealloc<kBwdRegRole>();
    {
      TTT_TRACE_DECL(0);
      constexpr uint32_t idS = idesc_bf16_f32(128, 128, false, false);  // S^T = K Q^T
      constexpr uint32_t idSP = idesc_bf16_f32(128, 64, false, false);  // dP^T = V dO_x^T
      constexpr uint32_t idKV = idesc_bf16_f32(128, D, false, true);    // dV += P^T dO_x, dK += dS^T Q_x
      constexpr uint32_t idDQ = idesc_bf16_f32(128, D, true, true);     // dQ = dS K
      // descriptor bases (built once; per k-step only a constant is added to the start field)
      const uint64_t dK_kmaj = sdesc_sw128(smem_u32(sK), 16, 1024), dV_kmaj = sdesc_sw128(smem_u32(sV), 16, 1024);
      const uint64_t dQ_kmaj = sdesc_sw128(smem_u32(sQ), 16, 1024), dDO_kmaj = sdesc_sw128(smem_u32(sDO), 16, 1024);
      const uint64_t dDO_mn = sdesc_sw128(smem_u32(sDO), HB / NBOX, 1024), dQ_mn = sdesc_sw128(smem_u32(sQ), 16384, 1024);
      const uint64_t dDS_mn = sdesc_sw128(smem_u32(sDS), 16384, 1024), dK_mn = sdesc_sw128(smem_u32(sK), 16384, 1024);
      const uint64_t dDS_k = sdesc_sw128(smem_u32(sDS), 16, 1024);  // dS^T boxes as a K-major A operand
      auto kofs = [](int ks, uint32_t box_bytes) { return (uint32_t)((ks >> 2) * box_bytes + (ks & 3) * 32); };
      // S^T = K Q^T for the whole 128-query tile in one N = 128 MMA chain: columns [0,64) are
      // sub-item a, [64,128) sub-item b. (An N = 64 SS MMA is SMEM-read bound at 48 clk per
      // K = 16 step vs 32 of tensor floor — bench_tools/mma_rate.cu — N = 128 runs at the floor.)
      auto issue_S = [&](int qs) {
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          umma_ss_e(tbase, sdesc_add(dK_kmaj, kofs(ks, 16384)), sdesc_add(dQ_kmaj, qs * TB + kofs(ks, 16384)), idS,
                    ks > 0);
        umma_commit_e(&bars.s_full[0]);
        umma_commit_e(&bars.s_full[1]);
      };
      auto issue_dP = [&](int slot, int x) {  // dP^T[x] = V dO_x^T
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          umma_ss_e(tbase + 128 + 64 * x, sdesc_add(dV_kmaj, kofs(ks, 16384)),
                    sdesc_add(dDO_kmaj, slot * HB + kofs(ks, HB / NBOX)), idSP, ks > 0);
      };
      auto issue_dV = [&](int slot, int x, bool first) {  // dV += P^T[x] dO_x  (K = 64 queries)
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          umma_ts_e(tbase + 256, tbase + 64 * x + 8 * ks, sdesc_add(dDO_mn, slot * HB + ks * 2048), idKV,
                    (!first || ks > 0) ? 1u : 0u);
      };
      auto issue_dK = [&](int qs, int x, bool first) {  // dK += dS^T[x] Q_x
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
#if TTT_BWD_DK_SS
          // A = dS^T[x] from shared memory ([kv][q] box x is K-major for M = keys, K = queries), so the
          // dQ MMA may overwrite the dP^T / dS^T TMEM columns before dK(t, b) runs
          umma_ss_e(tbase + 384, sdesc_add(dDS_k, x * 16384 + ks * 32), sdesc_add(dQ_mn, qs * TB + (64 * x + 16 * ks) * 128),
                    idKV, (!first || ks > 0) ? 1u : 0u);
#else
          umma_ts_e(tbase + 384, tbase + 128 + 64 * x + 8 * ks, sdesc_add(dQ_mn, qs * TB + (64 * x + 16 * ks) * 128),
                    idKV, (!first || ks > 0) ? 1u : 0u);
#endif
        }
      };
      // Issue order (program order of this warp = tensor-pipe order):
      //   prologue: S(0) dP(0,a) dP(0,b) dV(0,a) dV(0,b) S(1)
      //   tile t:   dK(t,a) dK(t,b) dQ(t) | [dQ drained] dP(t+1,a) dP(t+1,b) | dV(t+1,a) dV(t+1,b)
      //             | S(t+2)
      // dP(t+1) goes ahead of dV(t+1) so the compute warps find it done when they finish P(t+1)
      // (their dS phase then follows P without a wait); dV(t+1) runs under that dS phase.
      // A dO half is released after its second reader (dV).
      auto slot_of = [](int t, int x) { return (2 * t + x) % 3; };
      auto use_of = [](int t, int x) { return ((2 * t + x) / 3) & 1; };
      auto issue_dP_pair = [&](int t) {
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          // DQ_HALVES: dP^T[x] columns held dQ(t-1) columns [64x, 64x+64) (aliased only when 64x < D)
          // DQT: dP^T[x] held dQ^T(t-1, x)
          if ((DQT || TTT_BWD_DQ_HALVES) && t > 0 && (DQT || 64 * x < D)) mbar_wait(&bars.dq_empty_h[x], (t - 1) & 1);
          tc_fence_after();
          mbar_wait(&bars.do_full[slot_of(t, x)], use_of(t, x));
          TTT_TRACE_EV(0, 12 + x, t);
          tc_fence_after();
          issue_dP(slot_of(t, x), x);
          umma_commit_e(&bars.dp_full[x]);
        }
      };
      auto issue_dV_pair = [&](int t) {
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          mbar_wait(&bars.p_full[x], t & 1);
          TTT_TRACE_EV(0, 1 + x, t);
          tc_fence_after();
          issue_dV(slot_of(t, x), x, t == 0 && x == 0);
          umma_commit_e(&bars.do_empty[slot_of(t, x)]);  // dP(t,x) was issued before: both readers done
        }
      };
      mbar_wait(&bars.kv_full, 0);
      mbar_wait(&bars.q_full[0], 0);
      tc_fence_after();
      issue_S(0);
      issue_dP_pair(0);
      issue_dV_pair(0);
      if (n_items > 1) {
        mbar_wait(&bars.q_full[1], 0);
        tc_fence_after();
        issue_S(1);
      }
      if constexpr (DQT) {
        // Per sub-item x: dK(t,x) (TS, A = dS^T[x] in TMEM) then dQ^T(t,x) = K^T dS^T[x] (SS: A = K^T, the K
        // tile as an MN-major operand; B = the smem dS box x, MN-major) into the dP^T[x] columns, which
        // dK(t,x) has just read (in-order pipe). Order per tile t:
        //   dK(t,a) dQ^T(t,a) | dK(t,b) dQ^T(t,b) | [drain a] dP(t+1,a) [drain b] dP(t+1,b) | dV(t+1,a)
        //   dV(t+1,b) | S(t+2)
        // The drain of dQ^T(t,a) runs under dK / dQ^T(t,b); sub-item a's dS(t+1) compute runs under
        // dP(t+1,b) / dV(t+1) / S(t+2): no whole-tile dQ drain on the critical path.
        constexpr uint32_t idDQT = idesc_bf16_f32(128, 64, true, true);
        for (int t = 0; t < n_items; ++t) {
          const int qs = t & 1;
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            mbar_wait(&bars.ds_full[x], t & 1);
            TTT_TRACE_EV(0, 3 + x, t);
            tc_fence_after();
            issue_dK(qs, x, t == 0 && x == 0);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
              umma_ss_e(tbase + 128 + 64 * x, sdesc_add(dK_mn, ks * 2048), sdesc_add(dDS_mn, x * 16384 + ks * 2048),
                        idDQT, ks > 0);
            umma_commit_e(&bars.dq_full_x[x]);
            umma_commit_e(&bars.ds_empty_x[x]);
            TTT_TRACE_EV(0, 7 + x, t);
          }
          umma_commit_e(&bars.q_empty[qs]);
          if (t + 1 < n_items) {
            issue_dP_pair(t + 1);  // waits dq_empty_h[x] (dQ^T(t,x) drained) before dP(t+1,x)
            TTT_TRACE_EV(0, 6, t);
            issue_dV_pair(t + 1);
            if (t + 2 < n_items) {
              mbar_wait(&bars.q_full[(t + 2) & 1], ((t + 2) >> 1) & 1);
              TTT_TRACE_EV(0, 11, t + 2);
              tc_fence_after();
              issue_S((t + 2) & 1);
              TTT_TRACE_EV(0, 10, t);
            }
          }
        }
      } else
      for (int t = 0; t < n_items; ++t) {
        const int qs = t & 1;
#if TTT_BWD_DK_SS
        // dK(t,a) on dS(a); then dQ(t) as soon as dS(b) is in, then dK(t,b): the dQ drain overlaps dK(t,b)
        // instead of idling the pipe before dP(t+1) (r02g trace: ~0.4k clk per item)
        mbar_wait(&bars.ds_full[0], t & 1);
        TTT_TRACE_EV(0, 3, t);
        tc_fence_after();
        issue_dK(qs, 0, t == 0);
        TTT_TRACE_EV(0, 7, t);
        mbar_wait(&bars.ds_full[1], t & 1);
        TTT_TRACE_EV(0, 4, t);
        tc_fence_after();
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          umma_ss_e(tbase + 128, sdesc_add(dDS_mn, ks * 2048), sdesc_add(dK_mn, ks * 2048), idDQ, ks > 0);
        umma_commit_e(&bars.dq_full);
        issue_dK(qs, 1, false);
        TTT_TRACE_EV(0, 8, t);
        umma_commit_e(&bars.q_empty[qs]);
        umma_commit_e(&bars.ds_empty);
#else
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          mbar_wait(&bars.ds_full[x], t & 1);
          TTT_TRACE_EV(0, 3 + x, t);
          tc_fence_after();
          issue_dK(qs, x, t == 0 && x == 0);
          TTT_TRACE_EV(0, 7 + x, t);
        }
        umma_commit_e(&bars.q_empty[qs]);
        // dQ = dS K for the whole 128-query tile -> TMEM [128, 128+D)  (A = dS from smem, MN-major)
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          umma_ss_e(tbase + 128, sdesc_add(dDS_mn, ks * 2048), sdesc_add(dK_mn, ks * 2048), idDQ, ks > 0);
        umma_commit_e(&bars.dq_full);
        umma_commit_e(&bars.ds_empty);
#endif
        TTT_TRACE_EV(0, 9, t);
        if (t + 1 < n_items) {
          if (!TTT_BWD_DQ_HALVES) mbar_wait(&bars.dq_empty, t & 1);  // dQ(t) drained: the dP^T buffers are free
          TTT_TRACE_EV(0, 5, t);
          tc_fence_after();
#if TTT_BWD_ORDER == 1
          // dP(t+1,a) dV(t+1,a) dP(t+1,b) dV(t+1,b): dO half (t+1,a) is released (dV done) earlier, so
          // the producer's load of dO(t+2,b) into that slot starts sooner (r02g trace: that load's
          // ~3.5k clk latency stalled dP(t+2,b))
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            const int u = t + 1;
            mbar_wait(&bars.do_full[slot_of(u, x)], use_of(u, x));
            tc_fence_after();
            issue_dP(slot_of(u, x), x);
            umma_commit_e(&bars.dp_full[x]);
            mbar_wait(&bars.p_full[x], u & 1);
            tc_fence_after();
            issue_dV(slot_of(u, x), x, false);
            umma_commit_e(&bars.do_empty[slot_of(u, x)]);
          }
          TTT_TRACE_EV(0, 6, t);
#else
          issue_dP_pair(t + 1);
          TTT_TRACE_EV(0, 6, t);
          issue_dV_pair(t + 1);
#endif
          if (t + 2 < n_items) {  // S(t+2) over P^T(t+1), consumed by dV(t+1) above
            mbar_wait(&bars.q_full[(t + 2) & 1], ((t + 2) >> 1) & 1);
            TTT_TRACE_EV(0, 11, t + 2);
            tc_fence_after();
            issue_S((t + 2) & 1);
            TTT_TRACE_EV(0, 10, t);
          }
        }
      }
      umma_commit_e(&bars.acc_full);
    }
  } else if (warp >= 4 && warp < 12) {
    // ================= compute: P^T, dS^T of sub-item x (thread = key row, 64 query columns) ====
    reg_alloc<kBwdRegCmp>();
    const int quad = warp & 3, x = (warp - 4) >> 2;
    const int row = quad * 32 + lane;
    const int k = kt * kTile + row;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t tS = tbase + lane_off + 64 * x, tdP = tbase + lane_off + 128 + 64 * x;
    const float sl2 = p.scale_log2;
    const uint64_t sl2x2 = f2pack(sl2, sl2);
    TTT_TRACE_DECL(1);
    for (int t = 0; t < n_items; ++t) {
      const int qs = t & 1;
      const int qt = kt + t % nq;
      mbar_wait(&bars.q_full[qs], (t >> 1) & 1);
      mbar_wait(&bars.s_full[x], t & 1);
      if (threadIdx.x == 128) TTT_TRACE_EV(1, 1, t);
      tc_fence_after();
      const float4* Lq = reinterpret_cast<const float4*>(sL + qs * 128 + 64 * x);    // -lse2
      const float4* Dq = reinterpret_cast<const float4*>(sDel + qs * 128 + 64 * x);  // -Delta
      float pr[64];
      {
        uint32_t raw[64];
        tmem_ld64w(tS, raw);
        // allowed (k, q): k <= q and k < T; full tiles (qt > kt, whole key tile < T) skip the test
        // packed: query rows >= T are the next sequence's (local columns >= cmax are masked too)
        const bool full = (qt > kt) && (kt * kTile + kTile <= T) && (!PACKED || qt * kTile + kTile <= T);
        const int cmin = (k < T) ? k - qt * kTile - 64 * x : kTile;  // local columns [cmin, 64) allowed
        const unsigned span = (unsigned)max((PACKED ? T - qt * kTile - 64 * x : kTile) - cmin, 0);  // [cmin, cmin + span)
        // P = exp(S c - lse); full tiles take a mask-free copy of the loop (TTT_BWD_PSPLIT)
        auto p_phase = [&](auto masked_t) {
          constexpr bool masked = decltype(masked_t)::value;
#pragma unroll
          for (int c4 = 0; c4 < 16; ++c4) {
            const float4 l4 = Lq[c4];
            float x0, x1, x2, x3;
            f2unpack(ffma2(f2pack(__uint_as_float(raw[4 * c4]), __uint_as_float(raw[4 * c4 + 1])), sl2x2,
                           f2pack(l4.x, l4.y)), x0, x1);
            f2unpack(ffma2(f2pack(__uint_as_float(raw[4 * c4 + 2]), __uint_as_float(raw[4 * c4 + 3])), sl2x2,
                           f2pack(l4.z, l4.w)), x2, x3);
            float ys[4];
            if ((TTT_BWD_EMU_MASK >> (c4 & 7)) & 1) {  // 2^x on the FMA pipe for the selected quads
              ex2_emu2(x0, x1, ys[0], ys[1]);
              ex2_emu2(x2, x3, ys[2], ys[3]);
            } else {
              ys[0] = ex2(x0);
              ys[1] = ex2(x1);
              ys[2] = ex2(x2);
              ys[3] = ex2(x3);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c = 4 * c4 + e;
              pr[c] = (!masked || full || (unsigned)(c - cmin) < span) ? ys[e] : 0.f;
            }
          }
        };
        if (TTT_BWD_PSPLIT && full) p_phase(std::false_type{});
        else p_phase(std::true_type{});
      }
      {
        uint32_t pk[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) pk[c] = pack_bf16(pr[2 * c], pr[2 * c + 1]);
        tmem_st32(tS, pk);  // P^T over this sub-item's own (already read) S^T columns
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars.p_full[x]);
      if (threadIdx.x == 128) TTT_TRACE_EV(1, 2, t);
#ifdef TTT_TRACE
      if (lane == 0 && blockIdx.x == g_ttt_trace_cta && t < 2000)
        g_ttt_trace[3][t * 16 + warp] = (clock64() << 20) | ((unsigned long long)warp << 12) | (unsigned long long)(t & 0xFFF);
#endif
      mbar_wait(&bars.dp_full[x], t & 1);
      if constexpr (DQT) mbar_wait(&bars.ds_empty_x[x], (t & 1) ^ 1);  // dQ^T(t-1, x) has read dS box x
      else mbar_wait(&bars.ds_empty, (t & 1) ^ 1);  // dQ of the previous tile has read the dS buffer
      if (threadIdx.x == 128) TTT_TRACE_EV(1, 3, t);
      tc_fence_after();
#pragma unroll
#if TTT_BWD_DS_ONEWAIT
      uint32_t rawdp[64];
      tmem_ld64w(tdP, rawdp);  // both 32-column halves of dP^T with one wait (needs the 152-register split)
#endif
      for (int cc = 0; cc < 2; ++cc) {
#if TTT_BWD_DS_ONEWAIT
        const uint32_t* raw = rawdp + cc * 32;
#else
        uint32_t raw[32];
        tmem_ld32(tdP + cc * 32, raw);
#endif
        uint32_t pk[16];
#pragma unroll
        for (int e4 = 0; e4 < 8; ++e4) {
          const float4 d4 = Dq[cc * 8 + e4];
          const int c = cc * 32 + 4 * e4;
          float a0, a1, b0, b1;
          f2unpack(fmul2(f2pack(pr[c], pr[c + 1]),
                         fadd2(f2pack(__uint_as_float(raw[4 * e4]), __uint_as_float(raw[4 * e4 + 1])),
                               f2pack(d4.x, d4.y))), a0, a1);  // dS = P (dP - Delta)
          f2unpack(fmul2(f2pack(pr[c + 2], pr[c + 3]),
                         fadd2(f2pack(__uint_as_float(raw[4 * e4 + 2]), __uint_as_float(raw[4 * e4 + 3])),
                               f2pack(d4.z, d4.w))), b0, b1);
          pk[2 * e4] = pack_bf16(a0, a1);
          pk[2 * e4 + 1] = pack_bf16(b0, b1);
        }
        if (!TTT_BWD_DK_SS) tmem_st16(tdP + cc * 16, pk);  // dS^T (bf16) over this sub-item's read dP^T columns
        // smem dS: row = key row, q columns [64 x + 32 cc, +32): box x, 8-column chunks 4 cc + e8
        uint8_t* boxp = sDS + x * 16384 + row * 128;
#pragma unroll
        for (int e8 = 0; e8 < 4; ++e8) {
          const int chunk = cc * 4 + e8;
          *reinterpret_cast<uint4*>(boxp + ((chunk ^ (row & 7)) << 4)) =
              make_uint4(pk[e8 * 4 + 0], pk[e8 * 4 + 1], pk[e8 * 4 + 2], pk[e8 * 4 + 3]);
        }
      }
      fence_async_smem();
      if (!TTT_BWD_DK_SS) tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars.ds_full[x]);
      if (threadIdx.x == 128) TTT_TRACE_EV(1, 4, t);
#ifdef TTT_TRACE
      if (lane == 0 && blockIdx.x == g_ttt_trace_cta && t < 2000)
        g_ttt_trace[3][32768 + t * 16 + warp] =
            (clock64() << 20) | ((unsigned long long)(16 + warp) << 12) | (unsigned long long)(t & 0xFFF);
#endif
    }
    // ---- dK, dV accumulators -> global (fp32 adds in L2, so head splits and accumulated steps
    // add up). TMEM rows (thread = key row) are staged in the operand smem (K / V / Q, free once
    // acc_full follows the last MMA) and read back transposed, so each red.global.add.v4 covers
    // two 256-B half-rows (4 lines) instead of 32 rows 4 KB apart (that scattered form took ~9.5k
    // clk per CTA; a TMA bulk reduce-add of the staged tile ~6.5k, being bound near 20 B/clk).
    // Each warp reads back only the rows it staged (__syncwarp). Rows k >= T are skipped.
    mbar_wait(&bars.acc_full, 0);
    if (threadIdx.x == 128) TTT_TRACE_EV(1, 8, 0);
    tc_fence_after();
    constexpr int NCH = D / 64;  // 32-column chunks per half
    uint8_t* stg = smem + x * 65536 + quad * 4096;  // box i of this half: stg + i * 16384, rows of this warp
#pragma unroll 1
    for (int i = 0; i < 2 * NCH; ++i) {  // boxes: dV chunks | dK chunks of this half's D / 2 columns
      const int c0 = x * (D / 2) + (i % NCH) * 32;
      uint32_t raw[32];
      tmem_ld32(tbase + lane_off + (i < NCH ? 256 : 384) + c0, raw);
      const float sc = i < NCH ? 1.f : p.scale;
      uint8_t* rowp = stg + i * 16384 + lane * 128;
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4)
        *reinterpret_cast<float4*>(rowp + ((k4 ^ (lane & 7)) << 4)) =
            make_float4(sc * __uint_as_float(raw[4 * k4]), sc * __uint_as_float(raw[4 * k4 + 1]),
                        sc * __uint_as_float(raw[4 * k4 + 2]), sc * __uint_as_float(raw[4 * k4 + 3]));
    }
    __syncwarp();
    {
      constexpr int LPR = D / 8;        // lanes per half-row (16 B each): 16 at D = 128, 8 at D = 64
      constexpr int RPI = 32 / LPR;     // half-rows per instruction
      const int sub = lane / LPR, c = lane % LPR;  // 16-B chunk c of the half-row
#pragma unroll 1
      for (int tsr = 0; tsr < 2; ++tsr) {  // 0: dV, 1: dK
        float* dst = tsr == 0 ? p.dv : p.dk;
#pragma unroll 4
        for (int r0 = 0; r0 < 32; r0 += RPI) {
          const int lr = r0 + sub, kk = kt * kTile + quad * 32 + lr;
          const float4 val = *reinterpret_cast<const float4*>(stg + (tsr * NCH + c / 8) * 16384 + lr * 128 +
                                                              (((c & 7) ^ (lr & 7)) << 4));
          if (kk < T)
            red_add_v4(dst + (((size_t)(PACKED ? p.row0[b] : b * p.L) + kk) * p.Hkv + g) * D + x * (D / 2) + c * 4, val.x, val.y, val.z,
                       val.w);
        }
      }
    }
    if (threadIdx.x == 128) TTT_TRACE_EV(1, 9, 0);
  } else if (warp < 4) {
    // ================= dQ drain (warps 0-3, thread = query row) =================
    // TMEM -> registers (scaled by c) -> warp-private SW128 staging -> TMA reduce-add into
    // the tile-contiguous fp32 dq_acc (one 32 x 32 box per 32-column chunk).
    reg_alloc<kBwdRegDrain>();
    const int wq = warp;
    const uint32_t tQ = tbase + ((uint32_t)(wq * 32) << 16) + 128;
    uint8_t* stage = sDQ + wq * 4096;
    if (lane == 0) tma_prefetch_desc(&maps.dqacc);
    TTT_TRACE_DECL(2);
    if constexpr (DQT) {
      // dQ^T(t, x): TMEM lane = d (this warp: d in [32 wq, 32 wq + 32), i.e. column chunk wq of the dq_acc
      // tile), column = query 64 x + c. Each 32-query half is staged as a 32 x 32 box (row = query,
      // SW128 16-B chunks XOR (row & 7); a lane writes column d % 32 of every row: conflict-free) and
      // TMA reduce-added into rows 64 x + 32 hh of chunk wq.
      const uint32_t tQT = tbase + ((uint32_t)(wq * 32) << 16) + 128;
      const float c = p.scale;
      const uint32_t sbase = smem_u32(stage);
      for (int t = 0; t < n_items; ++t) {
        const int h = h_first + t / nq, qt = kt + t % nq;
        const int row_base = (int)(dq_tile(p, PACKED, b, h, qt) * (D / 32)) * 128 + wq * 128;
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          mbar_wait(&bars.dq_full_x[x], t & 1);
          if (threadIdx.x == 0) TTT_TRACE_EV(2, 1, t);
          tc_fence_after();
          uint32_t v[64];
          tmem_ld64w(tQT + 64 * x, v);
          tc_fence_before();
          mbar_arrive(&bars.dq_empty_h[x]);
          if (threadIdx.x == 0) TTT_TRACE_EV(2, 2, t);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            if (lane == 0) bulk_wait_read0();  // the previous reduce has read the staging buffer
            __syncwarp();
#pragma unroll
            for (int qi = 0; qi < 32; ++qi)
              asm volatile("st.shared.f32 [%0], %1;" ::"r"(sbase + qi * 128 + ((((uint32_t)(lane >> 2)) ^ (qi & 7)) << 4) +
                                                           (lane & 3) * 4),
                           "f"(c * __uint_as_float(v[32 * hh + qi]))
                           : "memory");
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_reduce_add_2d(&maps.dqacc, stage, 0, row_base + 64 * x + 32 * hh);
              bulk_commit();
            }
          }
        }
      }
    } else
    for (int t = 0; t < n_items; ++t) {
      const int h = h_first + t / nq, qt = kt + t % nq;
      mbar_wait(&bars.dq_full, t & 1);
      if (threadIdx.x == 0) TTT_TRACE_EV(2, 1, t);
      tc_fence_after();
      uint32_t v[D];
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 64) {
        tmem_ld64w(tQ + c0, *reinterpret_cast<uint32_t(*)[64]>(&v[c0]));
        if (TTT_BWD_DQ_HALVES) {
          tc_fence_before();
          mbar_arrive(&bars.dq_empty_h[c0 / 64]);
        }
      }
      tc_fence_before();
      if (!TTT_BWD_DQ_HALVES) mbar_arrive(&bars.dq_empty);
      if (threadIdx.x == 0) TTT_TRACE_EV(2, 2, t);
      const int row_base = (int)(dq_tile(p, PACKED, b, h, qt) * (D / 32)) * 128 + wq * 32;
#if TTT_BWD_DQ_RED
      {  // dev variant: reduce-add straight from registers (LSU path; the TMA unit then only loads)
        float* dst = p.dq_acc + (size_t)(row_base + lane) * 32;
        const float c = p.scale;
#pragma unroll
        for (int cc = 0; cc < D / 32; ++cc)
#pragma unroll
          for (int k4 = 0; k4 < 8; ++k4)
            red_add_v4(dst + (size_t)cc * 4096 + 4 * k4, c * __uint_as_float(v[cc * 32 + 4 * k4]),
                       c * __uint_as_float(v[cc * 32 + 4 * k4 + 1]), c * __uint_as_float(v[cc * 32 + 4 * k4 + 2]),
                       c * __uint_as_float(v[cc * 32 + 4 * k4 + 3]));
      }
      if (false)
#endif
#pragma unroll
      for (int cc = 0; cc < D / 32; ++cc) {
        if (lane == 0) bulk_wait_read0();  // the previous reduce has read the staging buffer
        __syncwarp();
        const float c = p.scale;
#pragma unroll
        for (int k4 = 0; k4 < 8; ++k4) {
          const float4 val =
              make_float4(c * __uint_as_float(v[cc * 32 + 4 * k4]), c * __uint_as_float(v[cc * 32 + 4 * k4 + 1]),
                          c * __uint_as_float(v[cc * 32 + 4 * k4 + 2]), c * __uint_as_float(v[cc * 32 + 4 * k4 + 3]));
          *reinterpret_cast<float4*>(stage + lane * 128 + ((k4 ^ (lane & 7)) << 4)) = val;
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0 && TTT_BWD_PROBE != 1) {
          tma_reduce_add_2d(&maps.dqacc, stage, 0, row_base + cc * 128);
          bulk_commit();
        }
      }
    }
    if (lane == 0) bulk_wait_read0();
  } else if (TTT_BWD_LSU_LOADS) {
    // ================= LSU loaders: warp 14 Q tiles + lse2 / Delta, warp 15 dO halves =================
    // 16-byte cp.async per lane into the SW128 layout the TMA would produce (box bx = 64 columns, row r,
    // chunk c at bx 16 KB (or bx 8 KB for a 64-row half) + r 128 + ((c ^ (r & 7)) << 4)); rows past the
    // sequence view zero-fill. Completion: one cp.async.mbarrier.arrive.noinc per lane (count 32); the
    // MMA warp fences the async proxy after its wait.
    reg_dealloc<88>();
    const bool isq = warp == 14;
    const size_t rstride = (size_t)p.Hq * D;  // elements between consecutive rows of one head
    const int lim = PACKED ? p.nrows : p.L;   // bound on (PACKED ? global : local) rows
    const int c = lane & 7, r4 = lane >> 3;   // chunk c of rows r4, r4 + 4, ...
    for (int t = 0; t < n_items; ++t) {
      const int h = h_first + t / nq, qt = kt + t % nq;
      const int loc0 = qt * kTile;  // first local row of the tile
      if (isq) {
        const int qs = t & 1, qph = (t >> 1) & 1;
        mbar_wait(&bars.q_empty[qs], qph ^ 1);
        const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(p.q) + ((size_t)p.row0[b] + loc0) * rstride + (size_t)h * D;
        const uint32_t dst = smem_u32(sQ + qs * TB);
#pragma unroll 4
        for (int i = 0; i < kTile * NBOX / 4; ++i) {  // (row, box) pairs: 4 rows per instruction
          const int r = (i % (kTile / 4)) * 4 + r4, bx = i / (kTile / 4);
          const int lr = loc0 + r;
          const bool ok = (PACKED ? p.row0[b] + lr : lr) < lim;
          cp_async16(dst + bx * 16384 + r * 128 + ((c ^ (r & 7)) << 4), src + (ok ? (size_t)r * rstride + bx * 64 + c * 8 : 0),
                     ok ? 16u : 0u);
        }
        const size_t li = ws_at(p, PACKED, b, h, loc0);
        cp_async16(smem_u32(sL + qs * 128) + lane * 16, p.lse2 + li + lane * 4, 16u);
        cp_async16(smem_u32(sDel + qs * 128) + lane * 16, p.delta + li + lane * 4, 16u);
        cp_async_arrive_noinc(&bars.q_full[qs]);
      } else {
#pragma unroll 1
        for (int x = 0; x < 2; ++x) {
          const int u = 2 * t + x, slot = u % 3, use = u / 3;
          mbar_wait(&bars.do_empty[slot], (use & 1) ^ 1);
          const int lb = loc0 + 64 * x;
          const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(p.dout) + ((size_t)p.row0[b] + lb) * rstride + (size_t)h * D;
          const uint32_t dst = smem_u32(sDO + slot * HB);
#pragma unroll 4
          for (int i = 0; i < 64 * NBOX / 4; ++i) {
            const int r = (i % 16) * 4 + r4, bx = i / 16;
            const int lr = lb + r;
            const bool ok = (PACKED ? p.row0[b] + lr : lr) < lim;
            cp_async16(dst + bx * (HB / NBOX) + r * 128 + ((c ^ (r & 7)) << 4),
                       src + (ok ? (size_t)r * rstride + bx * 64 + c * 8 : 0), ok ? 16u : 0u);
          }
          cp_async_arrive_noinc(&bars.do_full[slot]);
        }
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else {
    reg_dealloc<24>();  // warps 14-15: idle (a dq conversion of the previous unroll step here measured
                        // 5.78 vs 4.47 ms of main passes per unroll, r02c: reverted)
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 12) tmem_dealloc(tbase, 512);
}

// ------------------------------------------------------------------ kernel 3
// dq[b][r][h][:] = bf16(dq_acc tiled). One thread per 8 consecutive d of one row.
__global__ void __launch_bounds__(256) ttt_bwd_dq_convert_kernel(const __grid_constant__ Params p) {
  // thread -> (row, 8-column chunk); rows (b L + r) Hq + h in 32-bit (B L Hq < 2^31)
  const uint32_t d8 = (uint32_t)p.D / 8, rows_per_block = blockDim.x / d8;
  const uint32_t nrows = (uint32_t)p.nrows * p.Hq;
  const int d = (int)(threadIdx.x % d8) * 8;
  for (uint32_t row = blockIdx.x * rows_per_block + threadIdx.x / d8; row < nrows; row += gridDim.x * rows_per_block) {
    const uint32_t bl = row / (uint32_t)p.Hq;
    const int h = (int)(row - bl * (uint32_t)p.Hq);
    const int b = seq_of_row(p, p.packed, (int)bl);
    const int r = (int)bl - p.row0[b];
    const float4* src = reinterpret_cast<const float4*>(p.dq_acc + dqacc_index(p, b, h, r, d));
    const float4 a = src[0], c = src[1];
    uint4 o;
    o.x = pack_bf16(a.x, a.y);
    o.y = pack_bf16(a.z, a.w);
    o.z = pack_bf16(c.x, c.y);
    o.w = pack_bf16(c.z, c.w);
    reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.dq) + (size_t)row * p.D + d)[0] = o;
  }
}

int pick_head_split(const Params& p) {
  const int base = p.ntiles * p.Hkv;
  int hs = 1;
  while (hs < p.G && base * hs < 2 * 148) {
    int nx = hs + 1;
    while (nx < p.G && p.G % nx) ++nx;
    hs = nx;
  }
  return hs;
}

// R rows per warp item (R G <= 16 query rows, j R <= 32 columns, power of 2); NR rows per
// group: a multiple of R, NR G <= 256 (TMA box rows), stage ~64 KB; 4 down to 1 stages.
bool pre_layout(const Params& p, int D, PreLayout* lay) {
#ifndef TTT_PRE_RMAX
#define TTT_PRE_RMAX 16
#endif
  int R = 1;
  while (R * 2 * p.G <= 16 && R * 2 * p.step <= 32 && R * 2 <= TTT_PRE_RMAX) R *= 2;
  const int lo = p.o_lo != nullptr;
  const int row_bytes = ((2 + lo + (p.step > 0)) * p.G + 2 * p.step) * D * 2;
#ifndef TTT_PRE_STAGE_KB
#define TTT_PRE_STAGE_KB 64
#endif
  for (int nr = std::max(R, (TTT_PRE_STAGE_KB * 1024 / row_bytes) / R * R); nr >= R; nr -= R) {
    if (nr * p.G > 256) continue;
    for (int ns = 4; ns >= 1; --ns) {
      lay->init(nr, p.G, D, p.step, ns, R, lo);
      if (lay->total <= 225 * 1024 && (ns >= 2 || nr == R)) {
        lay->div_hkv.init((uint32_t)p.Hkv);
        lay->div_L.init((uint32_t)p.L);
        return true;
      }
    }
  }
  return false;
}

// dK_0 / dV_0 are accumulated by the main kernel; overwrite mode starts them at zero
cudaError_t zero_dkv0(const Params& p, int D, cudaStream_t st) {
  const size_t kvb = (size_t)p.nrows * p.Hkv * D * sizeof(float);
  cudaError_t e = cudaMemsetAsync(p.dk, 0, kvb, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p.dv, 0, kvb, st);
  return e;
}

// packed layout: the delta / lse2 rows >= T_b of each sequence's last tile are never written by the
// pre-pass, but the main kernel bulk-loads whole 128-row tiles of them (masked columns: P = 0, and
// dS = P (dP - Delta) needs a finite Delta) -> zero both workspaces first
cudaError_t zero_packed_ws(const Params& p, cudaStream_t st) {
  if (!p.packed) return cudaSuccess;
  const size_t bytes = (size_t)p.Hq * p.ntiles * kTile * sizeof(float);
  cudaError_t e = cudaMemsetAsync(p.delta, 0, bytes, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(p.lse2, 0, bytes, st);
  return e;
}

// 1. pre-pass (TMA-staged, persistent, warp-specialised); U: all steps of an unroll at once
template <int D, bool U>
cudaError_t launch_pre(const Params& p, const PreMaps& pmaps, const UnrollPre& up, cudaStream_t st) {
  PreLayout lay;
  if (!pre_layout(p, D, &lay)) return cudaErrorInvalidConfiguration;
  auto* kern = p.packed ? ttt_bwd_pre_kernel<D, U, true> : ttt_bwd_pre_kernel<D, U, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.total);
  if (e != cudaSuccess) return e;
  const int rows = p.nrows * p.Hkv;
  const int groups = (rows + lay.NR - 1) / lay.NR;
  UnrollPre u = up;
  if (U) u.M = std::max(lay.NS, 4);  // >= NS: the ring's own wait orders a group's steps
  prof_mark(kKindBwdPre, true, st);
  kern<<<std::min(groups, 148), 32 * (kPreCompute + 1), lay.total, st>>>(p, pmaps, u, lay);
  prof_mark(kKindBwdPre, false, st);
  return cudaGetLastError();
}

// 2. main tensor-core kernel, 3. dq = bf16(dq_acc)
template <int D>
cudaError_t launch_main_convert(const Params& p_in, const BwdMaps& maps, cudaStream_t st, bool convert = true) {
  Params p = p_in;
  static const int env_hs = dev_env_int("TTT_DEV_BWD_HSPLIT", 0), env_ob = dev_env_int("TTT_DEV_BWD_ORDER_BATCH", 0);
  p.head_split = env_hs > 0 && p.G % env_hs == 0 ? env_hs : pick_head_split(p);
  if (!p.packed) {  // CTA order: CTA kt of a group runs (nqt - kt) items of G / head_split heads; ~4.5k clk per
     // item and ~12k of fixed cost (measured traces); a group's Q, dO, dq_acc: 8 B per q element
    std::vector<double> len(p.nqt);
    const int nh = p.G / p.head_split;
    for (int r = 0; r < p.nqt; ++r) len[r] = (double)nh * (p.nqt - r) * 4.5;
    p.order_batch = pick_order_batch(p.B * p.Hkv * p.head_split, p.nqt, 1, len.data(), 12.0,
                                     (double)nh * p.L * D * 8);
    if (env_ob > 0) p.order_batch = env_ob;
  }
  {
    const int smem = BwdSmem<D>::bytes;
    static std::atomic<unsigned long long> attr_done{0}, attr_done_pk{0};
    cudaError_t ea = p.packed ? set_smem_attr(ttt_bwd_sm100_kernel<D, true>, smem, attr_done_pk)
                              : set_smem_attr(ttt_bwd_sm100_kernel<D, false>, smem, attr_done);
    if (ea != cudaSuccess) return ea;
    const int grid = p.ntiles * p.Hkv * p.head_split;  // padded: ntiles = B nqt
    prof_mark(kKindBwdMain, true, st);
    if (p.packed) ttt_bwd_sm100_kernel<D, true><<<grid, kBwdThreads, smem, st>>>(p, maps);
    else ttt_bwd_sm100_kernel<D, false><<<grid, kBwdThreads, smem, st>>>(p, maps);
    prof_mark(kKindBwdMain, false, st);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (convert) {
    const size_t n8 = (size_t)p.nrows * p.Hq * D / 8;
    unsigned blocks = (unsigned)((n8 + 255) / 256);
    if (blocks > 148u * 8u) blocks = 148u * 8u;
    prof_mark(kKindBwdConvert, true, st);
    ttt_bwd_dq_convert_kernel<<<blocks, 256, 0, st>>>(p);
    prof_mark(kKindBwdConvert, false, st);
    return cudaGetLastError();
  }
  return cudaSuccess;
}

template <int D>
cudaError_t launch_bwd_d(const Params& p, const BwdMaps& maps, const PreMaps& pmaps, cudaStream_t st) {
  cudaError_t e = p.accumulate ? cudaSuccess : zero_dkv0(p, D, st);
  static const UnrollPre kNoUnroll{};
  if (e == cudaSuccess) e = zero_packed_ws(p, st);
  if (e == cudaSuccess) e = launch_pre<D, false>(p, pmaps, kNoUnroll, st);
  if (e == cudaSuccess) e = launch_main_convert<D>(p, maps, st);
  return e;
}

// Whole-unroll backward: ps[j] are the per-call parameter blocks of steps j = 0..S-1 (their own
// delta / lse2 / dq_acc workspaces); ps[S-1] carries the unroll's accumulate flag and every step
// list. Same results as the S calls j = S-1..0 (the first with that flag, the rest accumulating).
template <int D>
cudaError_t launch_bwd_unroll_d(const Params* ps, const BwdMaps* maps, const PreMaps& pmaps, const UnrollPre& up,
                                cudaStream_t st) {
  const int S = up.S;
  const Params& last = ps[S - 1];
  cudaError_t e = last.accumulate ? cudaSuccess : zero_dkv0(last, D, st);
  for (int j = 0; j < S && e == cudaSuccess; ++j) e = zero_packed_ws(ps[j], st);
  if (e == cudaSuccess) e = launch_pre<D, true>(last, pmaps, up, st);
  for (int j = S - 1; j >= 0 && e == cudaSuccess; --j) e = launch_main_convert<D>(ps[j], maps[j], st);
  return e;
}

}  // namespace

#ifdef TTT_TRACE
extern "C" int ttt_debug_trace_read(void* host, unsigned int cta) {
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(host, g_ttt_trace, sizeof(g_ttt_trace)) != cudaSuccess) return 1;
  unsigned long long z[4 * 1024] = {};
  for (int r = 0; r < 4; ++r) cudaMemcpyToSymbol(g_ttt_trace, z, sizeof(z), (size_t)r * kTraceCap * 8);
  return cudaMemcpyToSymbol(g_ttt_trace_cta, &cta, sizeof(cta)) != cudaSuccess;
}
#endif

int bwd_pre_rows_per_group(const Params& p) {
  PreLayout lay;
  return pre_layout(p, p.D, &lay) ? lay.NR : 0;
}

cudaError_t launch_bwd_sm100(const Params& p, const BwdMaps& maps, const PreMaps& pmaps, cudaStream_t st) {
  return p.D == 64 ? launch_bwd_d<64>(p, maps, pmaps, st) : launch_bwd_d<128>(p, maps, pmaps, st);
}

cudaError_t launch_bwd_unroll_sm100(const Params* ps, const BwdMaps* maps, const PreMaps& pmaps,
                                    const UnrollPre& up, cudaStream_t st) {
  return ps[0].D == 64 ? launch_bwd_unroll_d<64>(ps, maps, pmaps, up, st)
                       : launch_bwd_unroll_d<128>(ps, maps, pmaps, up, st);
}

}  // namespace tttk
