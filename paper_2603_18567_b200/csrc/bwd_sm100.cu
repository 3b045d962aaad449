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
// Warp roles of the main kernel (320 threads):
//   warps 0-3 compute (thread = key row, TMEM lanes 0-127), warps 4-7 dQ drain
//   (thread = query row), warp 8 TMA producer, warp 9 TMEM owner + MMA issuer.
// TMEM columns: S^T/P^T [0,128) dP^T/dS^T/dQ [128,256) dV [256,256+D) dK [384,384+D).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "ptx_sm100.cuh"
#include "ttt_params.cuh"

namespace tttk {
#ifdef TTT_TRACE
__device__ unsigned long long g_ttt_trace[4][kTraceCap];
__device__ unsigned int g_ttt_trace_cta;
#endif
namespace {

constexpr float kLog2e = 1.4426950408889634f;

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
  return ((((size_t)(b * p.Hq + h) * p.nqt + (r >> 7)) * nc + (d >> 5)) * 128 + (r & 127)) * 32 + (d & 31);
}

// ------------------------------------------------------------------ kernel 1
// HBM-streaming, TMA-staged: a persistent block walks groups of NR consecutive
// (b, r, g) rows. For such a group every operand is ONE contiguous block in HBM
// (q / dO / O / O_lo: NR*G*D bf16; K_i, V_i: NR*D bf16; dK_i, dV_i: NR*D fp32), so
// thread 0 moves each with a single 1-D cp.async.bulk into a double-buffered
// stage. One HALF-warp per (row, query head): Delta, the diagonal p_i / ds_i and
// dq stay in registers; dK_i / dV_i (sums over the G heads) are accumulated with
// shared-memory atomics in the stage and written back with bulk stores. Lane hl
// owns elements [hl*E/2, +E/2) and [D/2 + hl*E/2, +E/2): every half-warp smem
// access is contiguous (bank-conflict free).
struct PreLayout {
  int NR, G, D, step, acc, has_lo;
  uint32_t off_q, off_do, off_o, off_olo, off_k, off_v, off_dk, off_dv, stage_bytes, off_sc, total;
  __host__ __device__ void init(int nr, int g, int d, int j, int accumulate, int lo) {
    NR = nr; G = g; D = d; step = j; acc = accumulate; has_lo = lo;
    const uint32_t qb = (uint32_t)nr * g * d * 2, kb = (uint32_t)nr * d * 2, fb = (uint32_t)nr * d * 4;
    off_q = 0; off_do = qb; off_o = 2 * qb; off_olo = 3 * qb;
    off_k = 4 * qb; off_v = off_k + j * kb; off_dk = off_v + j * kb; off_dv = off_dk + j * fb;
    stage_bytes = (off_dv + j * fb + 127) & ~127u;
    off_sc = 2 * stage_bytes;                            // fp32 [NR][j][G][2]: (p_i, c ds_i) per head
    total = off_sc + ((uint32_t)nr * (j > 0 ? j : 1) * g * 8 + 127) / 128 * 128 + 64;  // + 2 mbarriers
  }
};

__device__ __forceinline__ void bulk_store_1d(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_load_1d_(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// split-lane bf16 row chunk: E/2 elements at hl*E/2 and at D/2 + hl*E/2 -> fp32
// (bf16 -> fp32 is a 16-bit shift: one SHL / LOP per element)
__device__ __forceinline__ void bf2_to_f(uint32_t w, float& lo, float& hi) {
  lo = __uint_as_float(w << 16);
  hi = __uint_as_float(w & 0xFFFF0000u);
}
template <int D>
__device__ __forceinline__ void lds_split(const uint8_t* row, int hl, float (&x)[D / 16]) {
  constexpr int H = D / 32;  // elements per half (4 for D=128, 2 for D=64)
#pragma unroll
  for (int part = 0; part < 2; ++part) {
    const uint8_t* src = row + (part * (D / 2) + hl * H) * 2;
    if constexpr (H == 4) {
      const uint2 u = *reinterpret_cast<const uint2*>(src);
      bf2_to_f(u.x, x[part * 4 + 0], x[part * 4 + 1]);
      bf2_to_f(u.y, x[part * 4 + 2], x[part * 4 + 3]);
    } else {
      const uint32_t u = *reinterpret_cast<const uint32_t*>(src);
      bf2_to_f(u, x[part * 2 + 0], x[part * 2 + 1]);
    }
  }
}
template <int D>
__device__ __forceinline__ int split_col(int hl, int e) {  // D index of lane element e
  constexpr int H = D / 32;
  return (e < H) ? hl * H + e : D / 2 + hl * H + (e - H);
}

template <int D, int GT>  // GT: GQA group size (compile time; 0 = runtime p.G)
__global__ void __launch_bounds__(512) ttt_bwd_pre_kernel(const __grid_constant__ Params p, PreLayout lay) {
  constexpr int E = D / 16;
  extern __shared__ __align__(128) uint8_t psm[];
  const int tid = threadIdx.x, hl = tid & 15, pair = tid >> 4;
  const int G = GT > 0 ? GT : p.G;
  const int NR = lay.NR, j = p.step;
  const long nrows = (long)p.B * p.L * p.Hkv;
  const long ngroups = (nrows + NR - 1) / NR;
  uint64_t* full = reinterpret_cast<uint64_t*>(psm + lay.total - 64);
  // half-warp `pair` -> (row lr, head hh); ghosts (pair >= NR*G) mirror pair 0 without storing
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
    uint8_t* base = psm + st * lay.stage_bytes;
    const uint32_t qb = (uint32_t)nv * G * D * 2, kb = (uint32_t)nv * D * 2, fb = (uint32_t)nv * D * 4;
    const uint32_t bytes = 3 * qb + j * 2 * kb + (lay.has_lo ? qb : 0) + (lay.acc ? j * 2 * fb : 0);
    mbar_expect_tx(&full[st], bytes);
    const size_t qo = (size_t)w0 * G * D, ko = (size_t)w0 * D;
    bulk_load_1d_(base + lay.off_q, reinterpret_cast<const __nv_bfloat16*>(p.q) + qo, qb, &full[st]);
    bulk_load_1d_(base + lay.off_do, reinterpret_cast<const __nv_bfloat16*>(p.dout) + qo, qb, &full[st]);
    bulk_load_1d_(base + lay.off_o, reinterpret_cast<const __nv_bfloat16*>(p.o) + qo, qb, &full[st]);
    if (lay.has_lo)
      bulk_load_1d_(base + lay.off_olo, reinterpret_cast<const __nv_bfloat16*>(p.o_lo) + qo, qb, &full[st]);
    for (int i = 0; i < j; ++i) {
      bulk_load_1d_(base + lay.off_k + i * (NR * D * 2), reinterpret_cast<const __nv_bfloat16*>(p.ks[i]) + ko, kb,
                    &full[st]);
      bulk_load_1d_(base + lay.off_v + i * (NR * D * 2), reinterpret_cast<const __nv_bfloat16*>(p.vs[i]) + ko, kb,
                    &full[st]);
      if (lay.acc) {
        bulk_load_1d_(base + lay.off_dk + i * (NR * D * 4), p.dks[i] + ko, fb, &full[st]);
        bulk_load_1d_(base + lay.off_dv + i * (NR * D * 4), p.dvs[i] + ko, fb, &full[st]);
      }
    }
  };
  long grp = blockIdx.x;
  if (tid == 0 && grp < ngroups) issue(grp, 0);
  for (int n = 0; grp < ngroups; ++n, grp += gridDim.x) {
    const int st = n & 1;
    const long nxt = grp + gridDim.x;
    if (tid == 0 && nxt < ngroups) {
      bulk_wait_read0();  // bulk stores of group n-1 (same stage as n+1) have read their smem
      issue(nxt, st ^ 1);
    }
    uint8_t* base = psm + st * lay.stage_bytes;
    const long w = grp * NR + lr;
    const bool valid = !ghost && w < nrows;
    const long wc = w < nrows ? w : grp * NR;
    // 32-bit decode of wc = (b L + r) Hkv + g (host guarantees B L Hq < 2^31)
    const uint32_t bl = (uint32_t)wc / (uint32_t)p.Hkv;
    const int g = (int)((uint32_t)wc - bl * (uint32_t)p.Hkv);
    const int b = (int)(bl / (uint32_t)p.L);
    const int r = (int)(bl - (uint32_t)b * (uint32_t)p.L);
    const int h = g * G + hh;
    const bool act = valid && r < p.seq_lens[b];  // diagonal keys exist only for rows r < T_b
    if (!lay.acc && valid && hh == 0) {  // dK_0 / dV_0 rows in HBM: the main kernel adds into them
#pragma unroll
      for (int e = 0; e < E; ++e) {
        p.dk[(size_t)w * D + split_col<D>(hl, e)] = 0.f;
        p.dv[(size_t)w * D + split_col<D>(hl, e)] = 0.f;
      }
    }
    mbar_wait(&full[st], (n >> 1) & 1);
    const uint32_t ro = (uint32_t)(lr * G + hh) * D * 2;
    float o[E], dd[E], qq[E], dq[E];
    lds_split<D>(base + lay.off_o + ro, hl, o);
    lds_split<D>(base + lay.off_do + ro, hl, dd);
    if (lay.has_lo) {
      float lo[E];
      lds_split<D>(base + lay.off_olo + ro, hl, lo);
#pragma unroll
      for (int e = 0; e < E; ++e) o[e] += lo[e];
    }
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) acc = fmaf(o[e], dd[e], acc);
    const float del = half_allsum(acc);  // Delta_r = dO_r . O_r
    const size_t li = ((size_t)b * p.Hq + h) * p.L + r;
    const float l2 = p.lse_in[li] * kLog2e;
    if (valid && hl == 0) {  // stored negated: the main kernel's FFMA2 / FADD2 consume -lse2 and -Delta
      p.delta[li] = -del;
      p.lse2[li] = -l2;
    }
    lds_split<D>(base + lay.off_q + ro, hl, qq);
#pragma unroll
    for (int e = 0; e < E; ++e) dq[e] = 0.f;
    // ---- phase A: per (row, head) the diagonal scalars (Alg. 2 M_suffix) and dq ----
    float* scal = reinterpret_cast<float*>(psm + lay.off_sc);  // [NR][j][G][2]
    {
      const uint8_t* kp = base + lay.off_k + lr * D * 2;
      const uint8_t* vp = base + lay.off_v + lr * D * 2;
      float* sp = scal + ((lr * j) * G + hh) * 2;
      const bool wr = !ghost && hl == 0;
      const float sl2 = p.scale_log2, cs = p.scale;
      for (int i = 0; i < j; ++i, kp += NR * D * 2, vp += NR * D * 2, sp += 2 * G) {
        float kk[E], vv[E];
        lds_split<D>(kp, hl, kk);
        lds_split<D>(vp, hl, vv);
        float sdot = 0.f, dp = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          sdot = fmaf(qq[e], kk[e], sdot);
          dp = fmaf(dd[e], vv[e], dp);
        }
#pragma unroll
        for (int o2 = 8; o2 > 0; o2 >>= 1) {
          sdot += __shfl_xor_sync(0xffffffffu, sdot, o2);
          dp += __shfl_xor_sync(0xffffffffu, dp, o2);
        }
        const float pr = act ? ex2(sdot * sl2 - l2) : 0.f;  // p_i = exp(c q.k_i - lse)
        const float cds = cs * pr * (dp - del);             // c ds_i, ds_i = p_i (dp_i - Delta)
#pragma unroll
        for (int e = 0; e < E; ++e) dq[e] = fmaf(cds, kk[e], dq[e]);
        if (wr) {
          sp[0] = pr;
          sp[1] = cds;
        }
      }
    }
    if (valid) {
#pragma unroll
      for (int part = 0; part < 2; ++part) {
        const int d0 = part * (D / 2) + hl * (E / 2);
        float* q4 = p.dq_acc + dqacc_index(p, b, h, r, d0);
        if constexpr (E / 2 == 4)
          *reinterpret_cast<float4*>(q4) = make_float4(dq[part * 4], dq[part * 4 + 1], dq[part * 4 + 2], dq[part * 4 + 3]);
        else
          *reinterpret_cast<float2*>(q4) = make_float2(dq[part * 2], dq[part * 2 + 1]);
      }
    }
    __syncthreads();  // all (p_i, c ds_i) of the group visible
    // ---- phase B: per (row, step, D-slice): dK_i = sum_h c ds_h q_h, dV_i = sum_h p_h dO_h ----
    // (exclusive ownership of each stage row: no atomics; overwrite or accumulate)
    {
      const int nitems = NR * j;
      for (int it = pair; it < nitems; it += blockDim.x / 16) {
        const int brow = it % NR, i = it / NR;
        const long wb = grp * NR + brow;
        if (wb >= nrows) continue;
        float dk[E], dv[E];
#pragma unroll
        for (int e = 0; e < E; ++e) dk[e] = dv[e] = 0.f;
        const float* sp = scal + ((brow * j + i) * G) * 2;
        const uint8_t* qp = base + lay.off_q + brow * G * D * 2;
        const uint8_t* op = base + lay.off_do + brow * G * D * 2;
#pragma unroll(GT > 0 ? GT : 1)
        for (int h2 = 0; h2 < G; ++h2, qp += D * 2, op += D * 2) {
          const float pr = sp[2 * h2], cds = sp[2 * h2 + 1];
          float q2[E], d2[E];
          lds_split<D>(qp, hl, q2);
          lds_split<D>(op, hl, d2);
#pragma unroll
          for (int e = 0; e < E; ++e) {
            dk[e] = fmaf(cds, q2[e], dk[e]);
            dv[e] = fmaf(pr, d2[e], dv[e]);
          }
        }
        float* dkr = reinterpret_cast<float*>(base + lay.off_dk + i * (NR * D * 4)) + brow * D;
        float* dvr = reinterpret_cast<float*>(base + lay.off_dv + i * (NR * D * 4)) + brow * D;
#pragma unroll
        for (int part = 0; part < 2; ++part) {
          const int d0 = part * (D / 2) + hl * (E / 2);
          if constexpr (E / 2 == 4) {
            float4 a = make_float4(dk[part * 4], dk[part * 4 + 1], dk[part * 4 + 2], dk[part * 4 + 3]);
            float4 c = make_float4(dv[part * 4], dv[part * 4 + 1], dv[part * 4 + 2], dv[part * 4 + 3]);
            if (lay.acc) {
              const float4 a0 = *reinterpret_cast<const float4*>(dkr + d0), c0 = *reinterpret_cast<const float4*>(dvr + d0);
              a.x += a0.x; a.y += a0.y; a.z += a0.z; a.w += a0.w;
              c.x += c0.x; c.y += c0.y; c.z += c0.z; c.w += c0.w;
            }
            *reinterpret_cast<float4*>(dkr + d0) = a;
            *reinterpret_cast<float4*>(dvr + d0) = c;
          } else {
#pragma unroll
            for (int e = 0; e < E / 2; ++e) {
              const int k2 = part * (E / 2) + e;
              dkr[d0 + e] = lay.acc ? dkr[d0 + e] + dk[k2] : dk[k2];
              dvr[d0 + e] = lay.acc ? dvr[d0 + e] + dv[k2] : dv[k2];
            }
          }
        }
      }
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      const long w0 = grp * NR;
      const int nv = (int)min((long)NR, nrows - w0);
      for (int i = 0; i < j; ++i) {
        bulk_store_1d(p.dks[i] + (size_t)w0 * D, base + lay.off_dk + i * (NR * D * 4), (uint32_t)nv * D * 4);
        bulk_store_1d(p.dvs[i] + (size_t)w0 * D, base + lay.off_dv + i * (NR * D * 4), (uint32_t)nv * D * 4);
      }
      bulk_commit();
    }
  }
  if (tid == 0) bulk_wait0();
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
  uint32_t tmem_base;
};

template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    ttt_bwd_sm100_kernel(const __grid_constant__ Params p, const __grid_constant__ BwdMaps maps) {
  using SM = BwdSmem<D>;
  constexpr int TB = SM::TB, HB = SM::HB;
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
  // kv head run together, so its Q / dO tiles and dq_acc rows stay hot in L2.
  const int kt = (int)blockIdx.x % p.nqt;
  const int grp = (int)blockIdx.x / p.nqt;
  const int hs = grp % hsplit;
  const int g = (grp / hsplit) % p.Hkv;
  const int b = grp / (hsplit * p.Hkv);
  const int T = p.seq_lens[b];
  if (kt * kTile >= T) return;  // every key of the tile is padding: no gradient flows
  const int nq = p.nqt - kt;
  const int n_items = nh * nq;  // 128-query tiles
  const int h_first = g * p.G + hs * nh;
  if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0) __trap();  // SW128 tiles need 1 KB alignment

  if (threadIdx.x == 0) {
    mbar_init(&bars.kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars.q_full[i], 1);
      mbar_init(&bars.q_empty[i], 1);
      mbar_init(&bars.s_full[i], 1);
      mbar_init(&bars.dp_full[i], 1);
      mbar_init(&bars.p_full[i], 128);
      mbar_init(&bars.ds_full[i], 128);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&bars.do_full[i], 1);
      mbar_init(&bars.do_empty[i], 1);
    }
    mbar_init(&bars.ds_empty, 1);
    mbar_init(&bars.dq_full, 1);
    mbar_init(&bars.dq_empty, 128);
    mbar_init(&bars.acc_full, 1);
    fence_mbar_init();
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
    reg_dealloc<88>();
    if (lane == 0) {
      tma_prefetch_desc(&maps.q);
      tma_prefetch_desc(&maps.k);
      tma_prefetch_desc(&maps.v);
      tma_prefetch_desc(&maps.dout);
      mbar_expect_tx(&bars.kv_full, 2 * TB);
#pragma unroll
      for (int bx = 0; bx < NBOX; ++bx) {
        tma_load_4d(sK + bx * 16384, &maps.k, &bars.kv_full, bx * 64, g, kt * kTile, b);
        tma_load_4d(sV + bx * 16384, &maps.v, &bars.kv_full, bx * 64, g, kt * kTile, b);
      }
      for (int t = 0; t < n_items; ++t) {
        const int h = h_first + t / nq, qt = kt + t % nq;
        const int qs = t & 1, qph = (t >> 1) & 1;
        mbar_wait(&bars.q_empty[qs], qph ^ 1);
        mbar_expect_tx(&bars.q_full[qs], TB + 1024);
#pragma unroll
        for (int bx = 0; bx < NBOX; ++bx)
          tma_load_4d(sQ + qs * TB + bx * 16384, &maps.q, &bars.q_full[qs], bx * 64, h, qt * kTile, b);
        const size_t li = ((size_t)b * p.Hq + h) * p.L + (size_t)qt * kTile;
        bulk_load_1d(sL + qs * 128, p.lse2 + li, 512, &bars.q_full[qs]);
        bulk_load_1d(sDel + qs * 128, p.delta + li, 512, &bars.q_full[qs]);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          const int u = 2 * t + x, slot = u % 3, use = u / 3;
          mbar_wait(&bars.do_empty[slot], (use & 1) ^ 1);
          mbar_expect_tx(&bars.do_full[slot], HB);
#pragma unroll
          for (int bx = 0; bx < NBOX; ++bx)
            tma_load_4d(sDO + slot * HB + bx * (HB / NBOX), &maps.dout64, &bars.do_full[slot], bx * 64, h,
                        qt * kTile + 64 * x, b);
        }
      }
    }
  } else if (warp == 12) {
    // ================= MMA issuer (whole warp, converged; elect.sync inside each issue) =================
    reg_dealloc<88>();
    {
      TTT_TRACE_DECL(0);
      constexpr uint32_t idSP = idesc_bf16_f32(128, 64, false, false);  // S^T = K Q_x^T, dP^T = V dO_x^T
      constexpr uint32_t idKV = idesc_bf16_f32(128, D, false, true);    // dV += P^T dO_x, dK += dS^T Q_x
      constexpr uint32_t idDQ = idesc_bf16_f32(128, D, true, true);     // dQ = dS K
      // descriptor bases (built once; per k-step only a constant is added to the start field)
      const uint64_t dK_kmaj = sdesc_sw128(smem_u32(sK), 16, 1024), dV_kmaj = sdesc_sw128(smem_u32(sV), 16, 1024);
      const uint64_t dQ_kmaj = sdesc_sw128(smem_u32(sQ), 16, 1024), dDO_kmaj = sdesc_sw128(smem_u32(sDO), 16, 1024);
      const uint64_t dDO_mn = sdesc_sw128(smem_u32(sDO), HB / NBOX, 1024), dQ_mn = sdesc_sw128(smem_u32(sQ), 16384, 1024);
      const uint64_t dDS_mn = sdesc_sw128(smem_u32(sDS), 16384, 1024), dK_mn = sdesc_sw128(smem_u32(sK), 16384, 1024);
      auto kofs = [](int ks, uint32_t box_bytes) { return (uint32_t)((ks >> 2) * box_bytes + (ks & 3) * 32); };
      auto issue_S = [&](int qs, int x) {  // S^T[x] = K Q_x^T  (Q_x = rows 64x.. of the Q stage)
#pragma unroll
        for (int ks = 0; ks < D / 16; ++ks)
          umma_ss_e(tbase + 64 * x, sdesc_add(dK_kmaj, kofs(ks, 16384)),
                    sdesc_add(dQ_kmaj, qs * TB + 64 * x * 128 + kofs(ks, 16384)), idSP, ks > 0);
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
        for (int ks = 0; ks < 4; ++ks)
          umma_ts_e(tbase + 384, tbase + 128 + 64 * x + 8 * ks, sdesc_add(dQ_mn, qs * TB + (64 * x + 16 * ks) * 128),
                    idKV, (!first || ks > 0) ? 1u : 0u);
      };
      // Issue order (program order of this warp = tensor-pipe order):
      //   prologue: S(0,a) S(0,b) dP(0,a) dP(0,b) dV(0,a) dV(0,b) S(1,a) S(1,b)
      //   tile t:   dK(t,a) dK(t,b) dQ(t) | dV(t+1,a) dV(t+1,b) | [dQ drained] dP(t+1,a) dP(t+1,b)
      //             | S(t+2,a) S(t+2,b)
      // dV(t+1) fills the pipe while dQ(t) is drained; the compute warps' P(t+1) runs under
      // dK(t) / dQ(t). A dO half is released only after both of its readers (dV, dP).
      auto slot_of = [](int t, int x) { return (2 * t + x) % 3; };
      auto use_of = [](int t, int x) { return ((2 * t + x) / 3) & 1; };
      mbar_wait(&bars.kv_full, 0);
      mbar_wait(&bars.q_full[0], 0);
      tc_fence_after();
      issue_S(0, 0);
      umma_commit_e(&bars.s_full[0]);
      issue_S(0, 1);
      umma_commit_e(&bars.s_full[1]);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        mbar_wait(&bars.do_full[slot_of(0, x)], use_of(0, x));
        tc_fence_after();
        issue_dP(slot_of(0, x), x);
        umma_commit_e(&bars.dp_full[x]);
      }
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        mbar_wait(&bars.p_full[x], 0);
        tc_fence_after();
        issue_dV(slot_of(0, x), x, x == 0);
        umma_commit_e(&bars.do_empty[slot_of(0, x)]);  // dP(0,x) was issued before: both readers done
      }
      if (n_items > 1) {
        mbar_wait(&bars.q_full[1], 0);
        tc_fence_after();
        issue_S(1, 0);
        umma_commit_e(&bars.s_full[0]);
        issue_S(1, 1);
        umma_commit_e(&bars.s_full[1]);
      }
      for (int t = 0; t < n_items; ++t) {
        const int qs = t & 1;
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
        TTT_TRACE_EV(0, 9, t);
        if (t + 1 < n_items) {
          const int t1 = t + 1;
#pragma unroll
          for (int x = 0; x < 2; ++x) {  // dV(t+1, x): P^T(t+1, x) and the dO half are ready
            mbar_wait(&bars.p_full[x], t1 & 1);
            TTT_TRACE_EV(0, 1 + x, t1);
            mbar_wait(&bars.do_full[slot_of(t1, x)], use_of(t1, x));
            tc_fence_after();
            issue_dV(slot_of(t1, x), x, false);
          }
          mbar_wait(&bars.dq_empty, t & 1);  // dQ(t) drained: the dP^T buffers are free
          TTT_TRACE_EV(0, 5, t);
          tc_fence_after();
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            issue_dP(slot_of(t1, x), x);
            umma_commit_e(&bars.dp_full[x]);
            umma_commit_e(&bars.do_empty[slot_of(t1, x)]);
          }
          TTT_TRACE_EV(0, 6, t);
          if (t + 2 < n_items) {  // S(t+2, x) over P^T(t+1, x), consumed by dV(t+1, x) above
            mbar_wait(&bars.q_full[(t + 2) & 1], ((t + 2) >> 1) & 1);
            tc_fence_after();
            issue_S((t + 2) & 1, 0);
            umma_commit_e(&bars.s_full[0]);
            issue_S((t + 2) & 1, 1);
            umma_commit_e(&bars.s_full[1]);
            TTT_TRACE_EV(0, 10, t);
          }
        }
      }
      umma_commit_e(&bars.acc_full);
    }
  } else if (warp >= 4 && warp < 12) {
    // ================= compute: P^T, dS^T of sub-item x (thread = key row, 64 query columns) ====
    reg_alloc<136>();
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
        const bool full = (qt > kt) && (kt * kTile + kTile <= T);
        const int cmin = (k < T) ? k - qt * kTile - 64 * x : kTile;  // local columns [cmin, 64) allowed
#pragma unroll
        for (int c4 = 0; c4 < 16; ++c4) {
          const float4 l4 = Lq[c4];
          float x0, x1, x2, x3;
          f2unpack(ffma2(f2pack(__uint_as_float(raw[4 * c4]), __uint_as_float(raw[4 * c4 + 1])), sl2x2,
                         f2pack(l4.x, l4.y)), x0, x1);
          f2unpack(ffma2(f2pack(__uint_as_float(raw[4 * c4 + 2]), __uint_as_float(raw[4 * c4 + 3])), sl2x2,
                         f2pack(l4.z, l4.w)), x2, x3);
          const float xs[4] = {x0, x1, x2, x3};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int c = 4 * c4 + e;
            const float v = ex2(xs[e]);  // P = exp(S c - lse)
            pr[c] = (full || c >= cmin) ? v : 0.f;
          }
        }
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
      mbar_wait(&bars.ds_empty, (t & 1) ^ 1);  // dQ of the previous tile has read the dS buffer
      if (threadIdx.x == 128) TTT_TRACE_EV(1, 3, t);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        uint32_t raw[32];
        tmem_ld32(tdP + cc * 32, raw);
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
        tmem_st16(tdP + cc * 16, pk);  // dS^T (bf16) over this sub-item's already-read dP^T columns
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
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&bars.ds_full[x]);
      if (threadIdx.x == 128) TTT_TRACE_EV(1, 4, t);
#ifdef TTT_TRACE
      if (lane == 0 && blockIdx.x == g_ttt_trace_cta && t < 2000)
        g_ttt_trace[3][32768 + t * 16 + warp] =
            (clock64() << 20) | ((unsigned long long)(16 + warp) << 12) | (unsigned long long)(t & 0xFFF);
#endif
    }
    // ---- dK, dV accumulators -> global (fp32 atomics: head splits and steps add up) ----
    mbar_wait(&bars.acc_full, 0);
    tc_fence_after();
    // tcgen05.ld is warp-collective (.sync.aligned): every lane loads, only rows k < T store
    const bool store = k < T;
    const size_t off = (((size_t)b * p.L + (store ? k : 0)) * p.Hkv + g) * D;
    const int cbeg = x * (D / 2);
#pragma unroll 1
    for (int c0 = cbeg; c0 < cbeg + D / 2; c0 += 32) {
      uint32_t raw[32];
      tmem_ld32(tbase + lane_off + 256 + c0, raw);
      if (store) {
#pragma unroll
        for (int e = 0; e < 32; e += 4)
          red_add_v4(p.dv + off + c0 + e, __uint_as_float(raw[e]), __uint_as_float(raw[e + 1]),
                     __uint_as_float(raw[e + 2]), __uint_as_float(raw[e + 3]));
      }
      tmem_ld32(tbase + lane_off + 384 + c0, raw);
      if (store) {
        const float c = p.scale;
#pragma unroll
        for (int e = 0; e < 32; e += 4)
          red_add_v4(p.dk + off + c0 + e, c * __uint_as_float(raw[e]), c * __uint_as_float(raw[e + 1]),
                     c * __uint_as_float(raw[e + 2]), c * __uint_as_float(raw[e + 3]));
      }
    }
  } else if (warp < 4) {
    // ================= dQ drain (warps 0-3, thread = query row) =================
    // TMEM -> registers (scaled by c) -> warp-private SW128 staging -> TMA reduce-add into
    // the tile-contiguous fp32 dq_acc (one 32 x 32 box per 32-column chunk).
    reg_alloc<152>();
    const int wq = warp;
    const uint32_t tQ = tbase + ((uint32_t)(wq * 32) << 16) + 128;
    uint8_t* stage = sDQ + wq * 4096;
    if (lane == 0) tma_prefetch_desc(&maps.dqacc);
    TTT_TRACE_DECL(2);
    for (int t = 0; t < n_items; ++t) {
      const int h = h_first + t / nq, qt = kt + t % nq;
      mbar_wait(&bars.dq_full, t & 1);
      if (threadIdx.x == 0) TTT_TRACE_EV(2, 1, t);
      tc_fence_after();
      uint32_t v[D];
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += 64) tmem_ld64w(tQ + c0, *reinterpret_cast<uint32_t(*)[64]>(&v[c0]));
      tc_fence_before();
      mbar_arrive(&bars.dq_empty);
      if (threadIdx.x == 0) TTT_TRACE_EV(2, 2, t);
      const int row_base = (((b * p.Hq + h) * p.nqt + qt) * (D / 32)) * 128 + wq * 32;
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
        if (lane == 0) {
          tma_reduce_add_2d(&maps.dqacc, stage, 0, row_base + cc * 128);
          bulk_commit();
        }
      }
    }
    if (lane == 0) bulk_wait0();
  } else {
    reg_dealloc<24>();  // warps 14-15: idle
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
  const uint32_t nrows = (uint32_t)p.B * p.L * p.Hq;
  const int d = (int)(threadIdx.x % d8) * 8;
  for (uint32_t row = blockIdx.x * rows_per_block + threadIdx.x / d8; row < nrows; row += gridDim.x * rows_per_block) {
    const uint32_t bl = row / (uint32_t)p.Hq;
    const int h = (int)(row - bl * (uint32_t)p.Hq);
    const int b = (int)(bl / (uint32_t)p.L);
    const int r = (int)(bl - (uint32_t)b * (uint32_t)p.L);
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
  const int base = p.nqt * p.B * p.Hkv;
  int hs = 1;
  while (hs < p.G && base * hs < 2 * 148) {
    int nx = hs + 1;
    while (nx < p.G && p.G % nx) ++nx;
    hs = nx;
  }
  return hs;
}

template <int D>
cudaError_t launch_bwd_d(const Params& p_in, const BwdMaps& maps, cudaStream_t st) {
  Params p = p_in;
  p.head_split = pick_head_split(p);
  // 1. pre-pass (TMA-staged, persistent)
  {
    PreLayout lay;
    int nr = std::max(1, 32 / p.G);  // 32 half-warps (512 threads) of (row, head) pairs
    for (; nr > 1; nr >>= 1) {
      lay.init(nr, p.G, D, p.step, p.accumulate, p.o_lo != nullptr);
      if (lay.total <= 220 * 1024) break;
    }
    lay.init(nr, p.G, D, p.step, p.accumulate, p.o_lo != nullptr);
    if (lay.total > 227 * 1024) return cudaErrorInvalidConfiguration;
    const long rows = (long)p.B * p.L * p.Hkv;
    const long groups = (rows + nr - 1) / nr;
    const int blocks = (int)std::min<long>(groups, 148);
    const int threads = std::min(512, std::max(32, ((nr * p.G * 16 + 31) / 32) * 32));
    auto run = [&](auto kern) -> cudaError_t {
      cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lay.total);
      if (e2 != cudaSuccess) return e2;
      prof_mark(kKindBwdPre, true, st);
      kern<<<blocks, threads, lay.total, st>>>(p, lay);
      return cudaSuccess;
    };
    cudaError_t e;
    switch (p.G) {  // compile-time group size for the common GQA ratios
      case 1: e = run(ttt_bwd_pre_kernel<D, 1>); break;
      case 2: e = run(ttt_bwd_pre_kernel<D, 2>); break;
      case 4: e = run(ttt_bwd_pre_kernel<D, 4>); break;
      case 8: e = run(ttt_bwd_pre_kernel<D, 8>); break;
      case 16: e = run(ttt_bwd_pre_kernel<D, 16>); break;
      default: e = run(ttt_bwd_pre_kernel<D, 0>); break;
    }
    if (e != cudaSuccess) return e;
    prof_mark(kKindBwdPre, false, st);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  // 2. main tensor-core kernel
  {
    const int smem = BwdSmem<D>::bytes;
    static bool attr_set = false;
    if (!attr_set) {
      cudaError_t e =
          cudaFuncSetAttribute(ttt_bwd_sm100_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return e;
      attr_set = true;
    }
    const int grid = p.nqt * p.B * p.Hkv * p.head_split;
    prof_mark(kKindBwdMain, true, st);
    ttt_bwd_sm100_kernel<D><<<grid, kBwdThreads, smem, st>>>(p, maps);
    prof_mark(kKindBwdMain, false, st);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  // 3. dq = bf16(dq_acc)
  {
    const size_t n8 = (size_t)p.B * p.L * p.Hq * D / 8;
    unsigned blocks = (unsigned)((n8 + 255) / 256);
    if (blocks > 148u * 8u) blocks = 148u * 8u;
    prof_mark(kKindBwdConvert, true, st);
    ttt_bwd_dq_convert_kernel<<<blocks, 256, 0, st>>>(p);
    prof_mark(kKindBwdConvert, false, st);
    return cudaGetLastError();
  }
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

cudaError_t launch_bwd_sm100(const Params& p, const BwdMaps& maps, cudaStream_t st) {
  return p.D == 64 ? launch_bwd_d<64>(p, maps, st) : launch_bwd_d<128>(p, maps, st);
}

}  // namespace tttk
