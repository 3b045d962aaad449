/*
 * ttt_loss.h — C-ABI (in libtttattn.so) of the masked soft-label log-softmax
 * loss of EAGLE-3 draft training and its in-place backward (SpecForge,
 * arXiv 2603.18567). SURVEY.md §8(f) NEXT #1.
 *
 * What it computes (the operations the paper defines):
 *
 *   Loss (§4.2.1 "Memory-Efficient Gradient Computation",
 *   "the masked softmax loss"; reading R17 = SPEC.md:255):
 *       L = -(1/n) sum_{r : mask_r} sum_v p_rv * log_softmax(z_r)_v ,
 *       n = number of rows with mask_r true.
 *
 *   In-place backward, Alg. 3 "In-place Backward for Log-Softmax Loss"
 *   (PAPER.md:342-354), per row r (reading R18: s is a per-row sum):
 *       s  <- sum_v (p_rv * g_r)
 *       pi <- softmax(z_r)
 *       z_r <- -(p_r * g_r - pi * s)
 *   i.e. the logits buffer is overwritten with dL/dz ("the kernel overwrites
 *   the logits tensor with the gradient"). The upstream
 *   gradient of row r (reading R19) is
 *       g_r = mask_r ? g_scale * (g_rows ? g_rows[r] : 1) / (MEAN ? n : 1) : 0,
 *   so masked-out rows receive exactly zero gradient. pi is recomputed from z
 *   inside the same row pass (reading R20), so no [N][V] buffer exists
 *   besides z and p.
 *
 * Layouts: z, p, grad  [rows][vocab] row-major, contiguous.
 *          mask        uint8 [rows] (non-zero = row contributes), NULL = all rows.
 *          g_rows      fp32 [rows] or NULL; lse fp32 [rows] (natural log) or NULL.
 *          stats       fp64 [2] device: {L (the masked mean loss), n}.
 * Element types: TTT_BF16 (ttt_attn.h): z, p, grad bf16, arithmetic fp32,
 *                cross-row loss sum fp64 in a fixed order (deterministic);
 *                TTT_FP32_CHECK: z, p, grad fp32.
 * Limits: rows >= 1, rows * vocab < 2^40, 2 <= vocab <= 262144 (bf16) / 131072 (fp32) when
 *         vocab * element size is a multiple of 16 bytes and z, p, grad are 16-byte aligned
 *         (vectorised path), else vocab <= 32768 (element path). Larger: TTT_ERR_UNSUPPORTED.
 *         (EAGLE-3 draft vocabularies are 32000.)
 *
 * Ownership: all data pointers are caller-owned DEVICE memory; the desc is
 * HOST memory read during the call. The library allocates nothing; work is
 * enqueued on `stream` (cudaStream_t as void*; NULL = legacy default stream).
 *
 * Errors: return codes (ttt_status, ttt_attn.h) only; validation runs before
 * any launch. n == 0 (no masked row; SPEC.md:257's empty batch) is device
 * data, so it cannot be rejected without a host sync: it is reported as
 * stats = {NaN, 0} and, under TTT_LOSS_MEAN, an all-zero gradient; callers
 * check stats[1].
 */
#ifndef TTT_LOSS_H_
#define TTT_LOSS_H_
#include <stddef.h>
#include <stdint.h>

#include "ttt_attn.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t rows;   /* N = number of (sequence, position) rows, e.g. batch * seq_len */
  int32_t vocab;  /* V = draft vocabulary size */
  int32_t dtype;  /* ttt_dtype */
} ttt_loss_desc;

#define TTT_LOSS_MEAN 1u /* divide g by n (the masked-row count, counted on the device) */

/* Bytes of device workspace the three calls need (per-row losses + counters). 0 on a bad desc. */
size_t ttt_loss_workspace_size(const ttt_loss_desc* desc);

/* Forward: stats = {L, n}; lse (optional) = ln sum_v exp(z_rv) per row. One read of z and p. */
int ttt_loss_fwd(const ttt_loss_desc* desc, const void* z, const void* p, const uint8_t* mask,
                 float* lse, double* stats, void* workspace, size_t workspace_bytes, void* stream);

/* Alg. 3 backward. grad == NULL or grad == z: in place (z is overwritten with dL/dz);
 * otherwise the gradient goes to grad (out of place, bit-identical to the in-place result)
 * and z is only read. One read of z and p, one write. */
int ttt_loss_bwd_inplace(const ttt_loss_desc* desc, void* z, const void* p, const uint8_t* mask,
                         const float* g_rows, float g_scale, unsigned flags, void* grad,
                         void* workspace, size_t workspace_bytes, void* stream);

/* Forward and Alg. 3 backward in ONE pass over the rows (z, p read once, the gradient written
 * once): stats/lse as ttt_loss_fwd, gradient as ttt_loss_bwd_inplace. */
int ttt_loss_fwd_bwd_inplace(const ttt_loss_desc* desc, void* z, const void* p, const uint8_t* mask,
                             const float* g_rows, float g_scale, unsigned flags, void* grad,
                             float* lse, double* stats, void* workspace, size_t workspace_bytes,
                             void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TTT_LOSS_H_ */
