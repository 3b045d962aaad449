/*
 * ttt_oracle.c — TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, obviously-correct fp64 CPU oracle for the TTT attention of
 * EAGLE-3 draft training in SpecForge (arXiv 2603.18567). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library. It shares no code, header or constant with the CUDA
 * path (paper_2603_18567_b200/csrc); neither includes the other.
 *
 * It is the plain definition, written out:
 *   1. KVcat = [K_0; K_1; ...; K_j]  (K^train / K^pred)
 *   2. the explicit mask M of Alg. 2 over (r, k),
 *      k in [0, (j+1)L)
 *   3. dense logits s_k = c * q_r . KVcat[k] for ALL k (the "naive" method,
 *      PAPER.md:325), softmax over the allowed k only, o_r = sum_k P_rk V_k
 *      (§2.4 equation), lse_r = m + ln l
 *   4. analytic backward of softmax attention:
 *      Delta_r = dO_r . O_r,  dP = dO V^T,  dS = P o (dP - Delta),
 *      dQ = c dS KVcat, dKVcat = c dS^T Q, dVcat = P^T dO (summed over the
 *      query heads of a GQA group), then split into K_0 / K_i blocks.
 *
 * Inputs are fp32 arrays (the bf16 / fp32 values the GPU sees, exactly);
 * every arithmetic step is fp64. Sums run in natural index order.
 * Work is split over (b, kv-group) tasks on plain pthreads; each task owns
 * its output rows, so results do not depend on the thread count.
 *
 * Layouts match include/ttt_attn.h by design, but nothing is shared:
 *   q, out, dq, dout [B][L][Hq][D]; K_i, V_i, dK_i, dV_i [B][L][Hkv][D];
 *   lse [B][Hq][L].
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Alg. 2 predicate, verbatim:
 *   m_causal = (q_i >= kv_i); m_pad = (kv_i < T); M_causal = m_causal && m_pad
 *   m_suffix = (kv_i >= Q_LEN); m_pad = (kv_i mod Q_LEN < T);
 *   m_diag = ((kv_i - q_i) mod Q_LEN == 0); M_suffix = all three
 *   M = M_causal || M_suffix
 * Q_LEN = L, T = T_b. kv_i >= Q_LEN is tested first so kv_i - q_i > 0 and
 * the modulo is never taken of a negative number (reading R12). */
int ttt_oracle_mask(int L, int T, int q_i, int kv_i) {
  int m_causal = (q_i >= kv_i) && (kv_i < T);
  int m_suffix = 0;
  if (kv_i >= L) {
    m_suffix = ((kv_i % L) < T) && (((kv_i - q_i) % L) == 0);
  }
  return m_causal || m_suffix;
}

/* Fill dense mask[L][(j+1)L] (unsigned char) for one sequence. */
void ttt_oracle_mask_dense(int L, int T, int j, unsigned char* mask) {
  int n = (j + 1) * L;
  for (int r = 0; r < L; ++r)
    for (int k = 0; k < n; ++k) mask[(size_t)r * n + k] = (unsigned char)ttt_oracle_mask(L, T, r, k);
}

typedef struct {
  int B, L, Hq, Hkv, D, j;
  const int* seq_lens; /* [B] or NULL */
  double scale;
  const float* q;
  const float* k_base;
  const float* v_base;
  const float* const* k_steps;
  const float* const* v_steps;
  const unsigned char* row_sel; /* [B][Hq][L] or NULL: rows to compute (others untouched) */
  /* forward outputs */
  double* out;
  double* lse;
  /* backward */
  const float* dout;
  double* dq;
  double* dk_base;
  double* dv_base;
  double* const* dk_steps;
  double* const* dv_steps;
  int is_bwd;
  int status; /* set to 1 if a row had no allowed key */
  /* tasks */
  int next_task;
  pthread_mutex_t lock;
} job_t;

/* KVcat[k] row for sequence b, kv head g: K_0 for k < L else K_{k/L}[k mod L]
 * (PAPER.md:174 "K^train", :175 "K^pred"). */
static const float* kv_row(const job_t* J, int is_v, int b, int g, int k) {
  int blk = k / J->L, t = k % J->L;
  const float* base = blk == 0 ? (is_v ? J->v_base : J->k_base)
                               : (is_v ? J->v_steps[blk - 1] : J->k_steps[blk - 1]);
  return base + (((size_t)b * J->L + t) * J->Hkv + g) * J->D;
}

static double* dkv_row(const job_t* J, int is_v, int b, int g, int k) {
  int blk = k / J->L, t = k % J->L;
  double* base = blk == 0 ? (is_v ? J->dv_base : J->dk_base)
                          : (is_v ? J->dv_steps[blk - 1] : J->dk_steps[blk - 1]);
  return base + (((size_t)b * J->L + t) * J->Hkv + g) * J->D;
}

/* One (b, kv group g) task: all query heads h of the group, all rows. */
static void run_task(job_t* J, int b, int g, double* s, double* p, double* dp, double* o) {
  const int L = J->L, D = J->D, Hq = J->Hq, G = J->Hq / J->Hkv;
  const int n = (J->j + 1) * L;
  const int T = J->seq_lens ? J->seq_lens[b] : L;
  for (int h = g * G; h < (g + 1) * G; ++h) {
    for (int r = 0; r < L; ++r) {
      if (J->row_sel && !J->row_sel[((size_t)b * Hq + h) * L + r]) continue;
      const float* qr = J->q + (((size_t)b * L + r) * Hq + h) * D;
      /* step 3.1: dense logits against every key */
      for (int k = 0; k < n; ++k) {
        const float* kk = kv_row(J, 0, b, g, k);
        double acc = 0.0;
        for (int d = 0; d < D; ++d) acc += (double)qr[d] * (double)kk[d];
        s[k] = J->scale * acc;
      }
      /* step 3.2: softmax over the allowed set only */
      double m = -INFINITY;
      int any = 0;
      for (int k = 0; k < n; ++k)
        if (ttt_oracle_mask(L, T, r, k)) { any = 1; if (s[k] > m) m = s[k]; }
      if (!any) { J->status = 1; continue; }
      double l = 0.0;
      for (int k = 0; k < n; ++k) l += ttt_oracle_mask(L, T, r, k) ? exp(s[k] - m) : 0.0;
      for (int k = 0; k < n; ++k) p[k] = ttt_oracle_mask(L, T, r, k) ? exp(s[k] - m) / l : 0.0;
      /* step 3.3: o_r = sum_k P_rk V_k ; lse_r = m + ln l */
      for (int d = 0; d < D; ++d) o[d] = 0.0;
      for (int k = 0; k < n; ++k) {
        if (p[k] == 0.0) continue;
        const float* vv = kv_row(J, 1, b, g, k);
        for (int d = 0; d < D; ++d) o[d] += p[k] * (double)vv[d];
      }
      if (!J->is_bwd) {
        double* orow = J->out + (((size_t)b * L + r) * Hq + h) * D;
        for (int d = 0; d < D; ++d) orow[d] = o[d];
        J->lse[((size_t)b * Hq + h) * L + r] = m + log(l);
        continue;
      }
      /* step 4: analytic backward of row r */
      const float* dor = J->dout + (((size_t)b * L + r) * Hq + h) * D;
      double delta = 0.0;
      for (int d = 0; d < D; ++d) delta += (double)dor[d] * o[d];
      for (int k = 0; k < n; ++k) {
        const float* vv = kv_row(J, 1, b, g, k);
        double acc = 0.0;
        for (int d = 0; d < D; ++d) acc += (double)dor[d] * (double)vv[d];
        dp[k] = acc;
      }
      double* dqr = J->dq + (((size_t)b * L + r) * Hq + h) * D;
      for (int d = 0; d < D; ++d) dqr[d] = 0.0;
      for (int k = 0; k < n; ++k) {
        double ds = p[k] * (dp[k] - delta); /* dS = P o (dP - Delta) */
        const float* kk = kv_row(J, 0, b, g, k);
        double* dkk = dkv_row(J, 0, b, g, k);
        double* dvv = dkv_row(J, 1, b, g, k);
        for (int d = 0; d < D; ++d) {
          dqr[d] += J->scale * ds * (double)kk[d];  /* dQ = c dS K */
          dkk[d] += J->scale * ds * (double)qr[d];  /* dK = c dS^T Q */
          dvv[d] += p[k] * (double)dor[d];          /* dV = P^T dO */
        }
      }
    }
  }
}

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  const int n = (J->j + 1) * J->L;
  double* s = (double*)malloc(sizeof(double) * n);
  double* p = (double*)malloc(sizeof(double) * n);
  double* dp = (double*)malloc(sizeof(double) * n);
  double* o = (double*)malloc(sizeof(double) * J->D);
  const int ntask = J->B * J->Hkv;
  for (;;) {
    pthread_mutex_lock(&J->lock);
    int t = J->next_task++;
    pthread_mutex_unlock(&J->lock);
    if (t >= ntask) break;
    run_task(J, t / J->Hkv, t % J->Hkv, s, p, dp, o);
  }
  free(s); free(p); free(dp); free(o);
  return NULL;
}

static int run_job(job_t* J, int nthreads) {
  if (J->B < 1 || J->L < 1 || J->Hq < 1 || J->Hkv < 1 || J->D < 1 || J->j < 0) return 2;
  if (J->Hq % J->Hkv) return 2;
  if (nthreads < 1) nthreads = 1;
  J->next_task = 0;
  J->status = 0;
  pthread_mutex_init(&J->lock, NULL);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, worker, J);
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
  pthread_mutex_destroy(&J->lock);
  return J->status;
}

/* Forward: out [B][L][Hq][D] (double), lse [B][Hq][L] (double).
 * Returns 0, 1 if some computed row had no allowed key, 2 on bad sizes. */
int ttt_oracle_fwd(int B, int L, int Hq, int Hkv, int D, int j, const int* seq_lens, double scale,
                   const float* q, const float* k_base, const float* v_base,
                   const float* const* k_steps, const float* const* v_steps,
                   const unsigned char* row_sel, double* out, double* lse, int nthreads) {
  job_t J;
  memset(&J, 0, sizeof(J));
  J.B = B; J.L = L; J.Hq = Hq; J.Hkv = Hkv; J.D = D; J.j = j;
  J.seq_lens = seq_lens; J.scale = scale > 0 ? scale : 1.0 / sqrt((double)D);
  J.q = q; J.k_base = k_base; J.v_base = v_base; J.k_steps = k_steps; J.v_steps = v_steps;
  J.row_sel = row_sel; J.out = out; J.lse = lse; J.is_bwd = 0;
  return run_job(&J, nthreads);
}

/* Backward contribution of ONE step call: dq overwritten for computed rows;
 * dk_base/dv_base/dk_steps/dv_steps ADDED INTO (caller zeroes them for an
 * overwrite). Rows not selected by row_sel contribute nothing, which equals
 * the full gradient when dout is zero on those rows. */
int ttt_oracle_bwd(int B, int L, int Hq, int Hkv, int D, int j, const int* seq_lens, double scale,
                   const float* q, const float* k_base, const float* v_base,
                   const float* const* k_steps, const float* const* v_steps,
                   const float* dout, const unsigned char* row_sel,
                   double* dq, double* dk_base, double* dv_base,
                   double* const* dk_steps, double* const* dv_steps, int nthreads) {
  job_t J;
  memset(&J, 0, sizeof(J));
  J.B = B; J.L = L; J.Hq = Hq; J.Hkv = Hkv; J.D = D; J.j = j;
  J.seq_lens = seq_lens; J.scale = scale > 0 ? scale : 1.0 / sqrt((double)D);
  J.q = q; J.k_base = k_base; J.v_base = v_base; J.k_steps = k_steps; J.v_steps = v_steps;
  J.row_sel = row_sel; J.dout = dout; J.dq = dq; J.dk_base = dk_base; J.dv_base = dv_base;
  J.dk_steps = dk_steps; J.dv_steps = dv_steps; J.is_bwd = 1;
  return run_job(&J, nthreads);
}
