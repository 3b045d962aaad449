/*
 * ttt_attn.h — C-ABI of libtttattn.so, the B200 (sm_100a) Training-Time-Test
 * (TTT) attention library for EAGLE-3 draft training (SpecForge,
 * arXiv 2603.18567).
 *
 * What it computes (the operation the paper defines):
 *
 *   TTT step j (0 <= j < TTT_MAX_STEPS) of the unrolled draft layer attends,
 *   for every query row r of every sequence b and query head h, over the
 *   concatenated keys/values  K = [K_0; K_1; ...; K_j]  (each L rows):
 *
 *     o_r = softmax( q_r K^T * c ) V          restricted to the allowed set
 *
 *   - Alg. 1 "TTT Attention"            PAPER.md:139-162 (§2.4)
 *   - §2.4 equations, c = 1/sqrt(d_k)
 *   - Alg. 2 "BlockMask Construction"   PAPER.md:289-317 (§4.2.1):
 *       M_causal = (r >= k) && (k < T_b)                       (k < L)
 *       M_suffix = (k >= L) && (k mod L < T_b) && ((k - r) mod L == 0)
 *     i.e. row r sees base keys k <= r with k < T_b, plus — only if r < T_b —
 *     exactly one "diagonal" key from each step list: K_i[r], i = 1..j.
 *   - streaming (never materialising the L x (j+1)L logits) and block
 *     skipping are PAPER.md:323-331 (§4.2.1 "Sparse Tree Attention").
 *
 *   Rows r >= T_b (padding) follow Alg. 2 verbatim: they attend to all base
 *   keys k < T_b and to no step key (reading R4).
 *
 * Layouts (all row-major, "BSHD"):
 *   q, out, dq           [batch][seq_len][num_q_heads][head_dim]
 *   k_base, v_base,
 *   k_steps[i], v_steps[i],
 *   dk_*, dv_*           [batch][seq_len][num_kv_heads][head_dim]
 *   lse                  [batch][num_q_heads][seq_len]  fp32, natural log,
 *                        over the full allowed set (diagonal terms included)
 *   GQA: query head h reads kv head  h / (num_q_heads / num_kv_heads).
 *
 * Element types:
 *   TTT_BF16       q,k,v,out,dq: bf16; lse: fp32; dk/dv outputs: fp32
 *                  (they are accumulators across the S reverse-order calls).
 *                  Tensor-core path (tcgen05 + TMEM + TMA).
 *   TTT_FP32_CHECK every tensor fp32; CUDA-core fp32 path used to check
 *                  semantics at 1e-5 (SURVEY.md §8b "check mode").
 *
 * Ownership / lifetime: every data pointer is caller-owned DEVICE memory;
 * the pointer arrays k_steps/v_steps/dk_steps/dv_steps and the desc (with
 * its seq_lens) are HOST memory read during the call only. The library
 * allocates nothing and keeps no per-call state; all work is enqueued on
 * `stream` (cudaStream_t passed as void*; NULL = legacy default stream).
 * Inputs must stay alive until the stream reaches the kernels.
 *
 * Errors: return codes only, nothing is thrown or aborted across the ABI.
 * All argument validation runs before the first launch, so a non-zero
 * return other than TTT_ERR_CUDA means nothing was enqueued or written.
 * Asynchronous device faults surface at the caller's next synchronisation.
 */
#ifndef TTT_ATTN_H_
#define TTT_ATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TTT_MAX_STEPS 32    /* step j in [0, TTT_MAX_STEPS); paper max TTT length 17 */
#define TTT_MAX_BATCH 512   /* seq_lens are passed to the kernels by value */

typedef enum { TTT_BF16 = 0, TTT_FP32_CHECK = 1 } ttt_dtype;

typedef enum {
  TTT_OK = 0,
  TTT_ERR_INVALID_ARG = 1,  /* null pointer, non-positive size, Hq % Hkv != 0, bad flags */
  TTT_ERR_UNSUPPORTED = 2,  /* head_dim not in {64,128}; Hq/Hkv > 32; BF16 mode needs seq_len % 128 == 0;
                               batch * seq_len * num_q_heads >= 2^31 */
  TTT_ERR_STEP_RANGE = 3,   /* step < 0 or step >= TTT_MAX_STEPS */
  TTT_ERR_ALIGNMENT = 4,    /* a device pointer not 16-byte aligned */
  TTT_ERR_DEGENERATE = 5,   /* some seq_lens[b] < 1 (a row with no allowed key) or > seq_len */
  TTT_ERR_WORKSPACE = 6,    /* workspace too small (see ttt_attn_workspace_size) */
  TTT_ERR_CUDA = 7          /* a CUDA launch / driver call failed */
} ttt_status;

typedef struct {
  int32_t batch;          /* B >= 1, <= TTT_MAX_BATCH */
  int32_t seq_len;        /* L = padded per-step length (Alg. 2 Q_LEN) */
  int32_t num_q_heads;    /* Hq */
  int32_t num_kv_heads;   /* Hkv, Hq % Hkv == 0 */
  int32_t head_dim;       /* D in {64, 128} */
  int32_t dtype;          /* ttt_dtype */
  float softmax_scale;    /* c; 0 => 1/sqrt(head_dim) */
  const int32_t* seq_lens;/* HOST int32[batch]: T_b, 1 <= T_b <= L (Alg. 2 T); NULL => all T_b = L */
  const int32_t* cu_seqlens;/* HOST int32[batch + 1] or NULL (padded layout). Non-NULL: PACKED layout
                             (SURVEY.md §8(f) NEXT #3): sequence b is rows [cu_seqlens[b], cu_seqlens[b+1])
                             — T_b = the difference >= 1, cu_seqlens[0] = 0 — of q / out / out_lo / dq /
                             dout [N][Hq][D] and k_base / v_base / k_steps[i] / v_steps[i] / dk_* / dv_*
                             [N][Hkv][D], N = cu_seqlens[batch], with no padding rows; lse is [Hq][N].
                             Semantics: each sequence alone is Alg. 2 with Q_LEN = T_b (PAPER.md:294, 300,
                             307: m_pad vacuous), i.e. the padded result's rows r < T_b. seq_lens must be
                             NULL; seq_len is ignored (>= 1); BF16 mode has no multiple-of-128 requirement.
                             N x num_q_heads < 2^31. Zero-initialise the struct for the padded layout. */
} ttt_attn_desc;

/* flags for ttt_attn_bwd */
#define TTT_ACCUMULATE_DKV 1u /* += into dk_base/dv_base/dk_steps/dv_steps instead of overwrite.
                                 Step j's backward adds its contribution; the S calls of one
                                 unroll run in reverse order j = S-1..0. */

/* Bytes of device workspace ttt_attn_fwd (is_bwd=0) / ttt_attn_bwd (is_bwd=1)
 * need for this desc and step. 0 for fwd. Returns 0 on invalid desc. */
size_t ttt_attn_workspace_size(const ttt_attn_desc* desc, int step, int is_bwd);

/* Forward of TTT step `step` (= j, the number of step-list entries used).
 *   q        [B][L][Hq][D]                 in
 *   k_base   [B][L][Hkv][D], v_base        in   (K_0, V_0: "K^train")
 *   k_steps  HOST array of `step` device ptrs, each [B][L][Hkv][D]  (K_1..K_j, "K^pred")
 *   v_steps  likewise
 *   out      [B][L][Hq][D]                 out
 *   out_lo   [B][L][Hq][D] bf16 or NULL    out  (BF16 mode only: the rounding residual O - bf16(O)
 *            of the fp32 output; lets ttt_attn_bwd form Delta = dO.O from ~16-bit-accurate O.
 *            Ignored in FP32_CHECK mode.)
 *   lse      [B][Hq][L] fp32               out  (natural-log logsumexp of c*q.k over the allowed set)
 * step == 0 is ordinary causal attention with key padding (Alg. 2, suffix term vacuous). */
int ttt_attn_fwd(const ttt_attn_desc* desc, int step,
                 const void* q, const void* k_base, const void* v_base,
                 const void* const* k_steps, const void* const* v_steps,
                 void* out, void* out_lo, float* lse,
                 void* workspace, size_t workspace_bytes, void* stream);

/* Backward of TTT step `step`, recompute-based (no saved probabilities).
 *   out, out_lo, lse  from ttt_attn_fwd of the same step (out_lo may be NULL: Delta then
 *             uses the bf16 out); dout = dL/d out (layout of out).
 *   dq        [B][L][Hq][D]   (bf16 / fp32)  overwritten with this step's dq
 *   dk_base, dv_base          fp32 [B][L][Hkv][D]  dL/dK_0, dL/dV_0
 *   dk_steps, dv_steps        HOST arrays of `step` device ptrs, fp32 [B][L][Hkv][D]
 *   flags     TTT_ACCUMULATE_DKV or 0
 *   workspace >= ttt_attn_workspace_size(desc, step, 1) bytes of device memory (BF16: Delta, lse2 and
 *             the fp32 dq accumulator; FP32_CHECK: fp64 dK / dV accumulators, (2 + 2 step) x
 *             B L Hkv D x 8 bytes, so the check path's sums over all rows stay within 1e-5). */
int ttt_attn_bwd(const ttt_attn_desc* desc, int step,
                 const void* q, const void* k_base, const void* v_base,
                 const void* const* k_steps, const void* const* v_steps,
                 const void* out, const void* out_lo, const float* lse, const void* dout,
                 void* dq, float* dk_base, float* dv_base,
                 float* const* dk_steps, float* const* dv_steps,
                 unsigned flags, void* workspace, size_t workspace_bytes, void* stream);

/* Whole-unroll backward: the S = num_steps backward calls of one TTT unroll in one call,
 *   identical in semantics to
 *     for j = S-1 .. 0:  ttt_attn_bwd(desc, j, q[j], k_base, v_base, k_steps, v_steps, out[j],
 *                                     out_lo ? out_lo[j] : NULL, lse[j], dout[j], dq[j], dk_base,
 *                                     dv_base, dk_steps, dv_steps,
 *                                     j == S-1 ? flags : flags | TTT_ACCUMULATE_DKV, ...)
 *   (dq[j] identical bit for bit; the dK / dV accumulators equal up to fp32 summation order).
 *   q, out, out_lo, lse, dout, dq: HOST arrays of S device pointers (step j's tensors, layouts as
 *   in ttt_attn_bwd; out_lo all or NULL); k_steps / v_steps / dk_steps / dv_steps: HOST arrays of
 *   S-1 device pointers. 1 <= num_steps <= TTT_MAX_UNROLL.
 *   Why: the diagonal terms of all steps run as ONE pass (bwd_sm100.cu, ttt_bwd_pre_kernel<U>) that
 *   visits each row group for j = S-1 .. 0 back to back, so dK_i / dV_i are written to HBM once and
 *   K_i / V_i read once per unroll instead of once per call (the step-j call reads and writes
 *   every dK_i, i <= j).
 *   workspace >= ttt_attn_bwd_unroll_workspace_size(desc, num_steps) bytes (S per-call
 *   workspaces: each step keeps its Delta / lse2 / dq accumulator until its main pass). */
#define TTT_MAX_UNROLL 8
size_t ttt_attn_bwd_unroll_workspace_size(const ttt_attn_desc* desc, int num_steps);
int ttt_attn_bwd_unroll(const ttt_attn_desc* desc, int num_steps,
                        const void* const* q, const void* k_base, const void* v_base,
                        const void* const* k_steps, const void* const* v_steps,
                        const void* const* out, const void* const* out_lo, const float* const* lse,
                        const void* const* dout, void* const* dq,
                        float* dk_base, float* dv_base, float* const* dk_steps, float* const* dv_steps,
                        unsigned flags, void* workspace, size_t workspace_bytes, void* stream);

/* ---- Tree-attention verification (inference side) ----------------
 * The target's forward over a draft token tree: query t (tree node t, t < num_tree) attends every
 * context key of its sequence (rows [0, P_b) of the cache) and the cache rows P_b + u of its
 * ancestors u and itself — "each candidate token attends only to its ancestors" (
 * SPEC.md:507-509, 528; readings R21-R22). Same tcgen05 pipeline as ttt_attn_fwd.
 *   q        bf16 [batch][num_tree][Hq][D]             in   (the tree tokens' queries)
 *   k_cache, v_cache bf16 [batch][kv_len][Hkv][D]      in   (prefix rows then the tree's own rows)
 *   parents  DEVICE int32 [batch][num_tree]            in   parent node index, -1 = child of the
 *            context tip; nodes in topological order (a parent index >= t is treated as -1)
 *   out      bf16 [batch][num_tree][Hq][D]             out
 *   lse      fp32 [batch][Hq][num_tree]                out  natural-log logsumexp over the allowed keys
 *   workspace >= ttt_tree_attn_workspace_size(desc) bytes (the per-node ancestor bit masks).
 * Errors: 1 <= num_tree <= TTT_MAX_TREE, 0 <= prefix_lens[b], prefix_lens[b] + num_tree <= kv_len
 * (else TTT_ERR_DEGENERATE), head_dim 64 / 128. dtype TTT_FP32_CHECK: every tensor fp32, a
 * CUDA-core kernel that checks the semantics at 1e-5 (no workspace needed). */
#define TTT_MAX_TREE 64
typedef struct {
  int32_t batch, num_tree, kv_len, num_q_heads, num_kv_heads, head_dim;
  float softmax_scale;         /* 0 => 1/sqrt(head_dim) */
  int32_t dtype;               /* TTT_BF16 (tensor-core path) or TTT_FP32_CHECK (fp32 CUDA-core check path) */
  const int32_t* prefix_lens;  /* HOST int32[batch]: P_b, the verified context length */
} ttt_tree_desc;
size_t ttt_tree_attn_workspace_size(const ttt_tree_desc* desc);
int ttt_tree_attn_fwd(const ttt_tree_desc* desc, const void* q, const void* k_cache, const void* v_cache,
                      const int32_t* parents, void* out, float* lse, void* workspace, size_t workspace_bytes,
                      void* stream);

/* ---- The TTT step's fresh projections into attention inputs (SURVEY.md §8(f) NEXT #2 part) ----
 * qkv (bf16 [batch][seq_len][Hq + 2 Hkv][D]: a fused q/k/v projection's output, q heads first)
 * -> q [batch][seq_len][Hq][D], k_slot / v_slot [batch][seq_len][Hkv][D] (e.g. k_steps[j-1] /
 * v_steps[j-1] of ttt_attn_fwd, written in place), q and k rotated by rotate-half RoPE:
 *   theta_i = pos * rope_base^(-2i/D),  x'_i = x_i cos - x_{i+D/2} sin,  x'_{i+D/2} = x_{i+D/2} cos + x_i sin
 * at pos = row index 0..seq_len-1 ("a TTT step reuses position ids 0..T_pad-1"), or
 * positions (DEVICE int32 [batch][seq_len]) when not NULL. One HBM pass; angles from an fp64-built
 * cos / sin table in the workspace (>= ttt_rope_workspace_size(desc, positions != NULL) bytes).
 * head_dim a multiple of 16; all pointers 16-byte aligned. */
typedef struct {
  int32_t batch, seq_len, num_q_heads, num_kv_heads, head_dim;
  float rope_base;  /* e.g. 500000 (Llama-3.1) */
} ttt_rope_desc;
size_t ttt_rope_workspace_size(const ttt_rope_desc* desc, int per_sequence_positions);
int ttt_qkv_rope_split(const ttt_rope_desc* desc, const void* qkv, const int32_t* positions, void* q,
                       void* k_slot, void* v_slot, void* workspace, size_t workspace_bytes, void* stream);
/* Its backward (the adjoint): dqkv [batch][seq_len][Hq + 2 Hkv][D] = [R(-theta) dq | R(-theta) dk | dv]. */
int ttt_qkv_rope_join_bwd(const ttt_rope_desc* desc, const void* dq, const void* dk_slot, const void* dv_slot,
                          const int32_t* positions, void* dqkv, void* workspace, size_t workspace_bytes,
                          void* stream);

/* ---- Optional instrumentation (off by default; used by bench.py) ----------
 * ttt_attn_profile_begin() arms per-kernel timing for the CALLING HOST THREAD:
 * each kernel the library launches afterwards is bracketed by cudaEventRecord
 * on its launch stream (events come from a library-owned pool of up to 4096
 * pairs). ttt_attn_profile_end() synchronises on those events, writes the
 * summed device milliseconds and launch counts per kernel kind into the
 * caller's arrays (n_kinds entries, kinds listed by ttt_attn_kernel_name),
 * and disarms. Returns the number of kinds filled, or < 0 on error.
 * This is the only library state; computations never depend on it. */
#define TTT_KERNEL_KINDS 10
int ttt_attn_profile_begin(void);
int ttt_attn_profile_end(double* ms_by_kind, int* launches_by_kind, int n_kinds);
const char* ttt_attn_kernel_name(int kind);

/* Static string for a ttt_status code. */
const char* ttt_attn_strerror(int code);

/* Library version / build info string (arch it was compiled for). */
const char* ttt_attn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TTT_ATTN_H_ */
