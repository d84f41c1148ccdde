/*
 * attn_softmax_debug.h -- test / tuning surface of libattnsm.so.
 *
 * Not needed by users of the stage.  The parity tests use it to compare the
 * stashed intermediates of a finished attn_softmax_fwd_bwd call (which live in
 * the caller's workspace) with the oracle stage by stage, to exercise the
 * tcgen05 GEMM core on its own, and to set tuning knobs.
 */
#ifndef ATTN_SOFTMAX_DEBUG_H
#define ATTN_SOFTMAX_DEBUG_H

#include "attn_softmax.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Byte offsets, inside the workspace, of the intermediates that stay valid
 * after attn_softmax_fwd_bwd returns and its stream work completes.  T = B*N.
 *   alpha  fp32 [B*N, alpha_ld] (columns < M) attention weights (Eq. 1), exact 0
 *          where masked; alpha_ld = M (fp32 path) or M rounded up to 64 (bf16)
 *   ctx    dtype [T,d]   context vectors C (Eq. 3)
 *   hc     dtype [T,d]   attentional states H_c (Eq. 4)
 *   lse    fp32 [T]      log-sum-exp of the Eq. 5 logits per row
 *   nll    fp32 [T]      per-row token NLL (0 on padded rows)
 *   vocab_chunk          V-chunk width the backward uses (columns)          */
typedef struct {
  size_t alpha, ctx, hc, lse, nll;
  int64_t vocab_chunk;
  int64_t alpha_ld;
} attn_ws_views_t;

attn_status_t attn_softmax_workspace_views(const attn_shape_t* s,
                                           attn_ws_views_t* out);

/* C[M,N] (fp32, row-major, ldc = N) = A * B^T on the tcgen05 GEMM core.
 *   A: a_mn == 0 -> K-major bf16 [M,K] (row stride K)
 *      a_mn == 1 -> MN-major bf16 [K,M] (row stride M)
 *   B: b_mn == 0 -> K-major bf16 [N,K];  b_mn == 1 -> MN-major bf16 [K,N]
 * K % 8 == 0 and M % 8 == 0 / N % 8 == 0 for the MN-major operands (16-byte
 * TMA row strides). */
attn_status_t attn_debug_gemm_bf16(int M, int N, int K,
                                   const void* A, int a_mn,
                                   const void* B, int b_mn,
                                   float* C, void* stream);

/* Per-step timing of the last attn_softmax_fwd_bwd call on this process,
 * recorded with CUDA events on the caller's stream when the "stage_events"
 * option is 1.  Steps, in order: attn_fwd, proj_tanh, vocab_fwd, lse_reduce,
 * vocab_bwd, proj_bwd, attn_bwd.  attn_softmax_stage_time synchronizes on the
 * step's closing event. */
int attn_softmax_stage_count(void);
attn_status_t attn_softmax_stage_time(int i, const char** name, float* ms);

/* Number of kernels the last attn_softmax_fwd_bwd call launched. */
long long attn_softmax_last_launches(void);

/* Tuning knobs (process-wide; a call reads them once, at its start, under a
 * lock, so a concurrent set_option never changes a call in flight.  Options
 * that change the workspace layout -- vocab_chunk, dl_budget_mb, dl_buffers,
 * store_logits -- must be set before attn_softmax_workspace_size; a call whose
 * workspace is too small for the current options fails with
 * ATTN_ERR_WORKSPACE).  Keys:
 *   "vocab_chunk"   V-chunk width of the vocab backward (multiple of 256,
 *                   0 = automatic: the dL chunk buffers fit dl_budget_mb)
 *   "dl_budget_mb"  budget of the bf16 dL chunk scratch, all buffers
 *                   (default 200; C1: Vc = 5376)
 *   "dl_buffers"    dL chunk buffers of the persistent backward (1-4, default 3)
 *   "vb_pair"       1 (default) = the persistent vocabulary launch on CTA
 *                   pairs (tcgen05 cta_group::2, 256 x 256 tiles); 0 = single
 *                   CTAs (128 x 256)
 *   "vb_fwd_fused"  1 = F4 + F5 (logit tiles, lse, loss) inside the persistent
 *                   launch; 0 (default) = the single-CTA forward GEMM and the
 *                   lse_reduce kernel before it
 *   "vb_order"      dispatch blocks of the persistent backward: 1 (default) =
 *                   [G1(c+1), G3(c), G2(c)], 0 = [G3(c), G2(c), G1(c+1)],
 *                   2 = row-interleaved (G3 of row block rb after G1 of
 *                   rb + vb_lag, dW_out tiles split over T in two row halves
 *                   when vb_g2split; works with dl_buffers = 1)
 *   "vb_lag", "vb_g2split"  order 2 parameters (defaults 2, 1)
 *   "vb_claim"      when a CTA pair claims its next tile: 0 = right after
 *                   the current tile's first load, 1 (default) = two
 *                   k-blocks before the end of its loads, k >= 2 = k
 *                   k-blocks before the end; -1 = late for order 2 only
 *   "vb_wide"       1 (default, d % 512 == 0): 512-column dW_out / dHc tiles
 *                   on both accumulators
 *   "vb_g1wide"     1 = 512-column dL tiles too (measured slower; default 0)
 *   "gemm_claim"    bitmask of GEMM groups (the "wide_tiles" bits) of the
 *                   generic engine whose tiles are claimed late (default 4:
 *                   the projection backward)
 *   "comm_reserve_1rank" tests: a 1-rank communicator reserves NCCL's SMs as
 *                   with several ranks
 *   "vb_last_g2_first" 1 (default): the last block dispatches dW_out tiles first
 *   "vb_l2hints"    bit 0: H_c loads evict-last; bit 1: dHc updates evict-last
 *                   (default 3)
 *   "vb_trace"      device address of an int64 buffer (32 per tile) that the
 *                   next persistent launch fills with per-tile stamps (debug)
 *   "vb_debug"      timing experiments only (WRONG results): bit 0 skip the
 *                   dL stores, bit 1 skip the exponentials, bit 2 skip the
 *                   dW_out / dHc stores, bit 3 publish without waiting for
 *                   the stores, bits 4 / 5 skip the B / A loads, bit 7 G1
 *                   epilogue without TMEM loads, bits 13 / 14 skip the G2 /
 *                   G3 loads (bits 6, 8-12: MMA-issue probes compiled only
 *                   with -DVB_DEBUG_MMA=1)
 *   "gemm_ctas"     persistent GEMM grid size (0 = number of SMs)
 *   "comm_max_ctas" CTA cap given to NCCL by attn_comm_init calls made after
 *                   it (default 8, 0 = NCCL's default); while gradients are
 *                   being allreduced the stage's persistent GEMMs leave that
 *                   many SMs free for NCCL's kernels
 *   "stage_events"  1 = record per-step CUDA events (see above); 2 = only the
 *                   marks around the vocab GEMMs (vocab_fwd, lse_reduce,
 *                   vocab_bwd: fewer events between the step's kernels)
 *   "store_logits"  ABLATION (violates "logits never round-tripped through
 *                   HBM"; kept to quantify the trade): 1 = the forward vocab
 *                   GEMM also stores the logits as fp16 [T, V] (workspace
 *                   grows by 2 T V bytes) and the backward makes each
 *                   V-chunk's dlogits from them with an elementwise kernel
 *                   beside the previous chunk's launch; 2 = the same,
 *                   serialised; 0 (default) = the persistent recompute launch
 *   "wide_tiles"    bitmask of GEMM groups on wide single-CTA 256 x 256 tiles
 *                   (1 = forward vocab / projection, 2 = stored-logits
 *                   vocab-backward launches, 4 = projection backward, 8 = the
 *                   debug GEMM entry).  Default 2.
 *   "debug_skip_dlogits" stored-logits ablation, timing only: 1 = skip the
 *                   elementwise dlogits of chunks >= 1 (gradients WRONG)
 *   "db_gemm"       stored-logits ablation: how db_out (F_c bias) is summed:
 *                   0 = column-sum kernels after each launch; 2 = by the
 *                   dlogits kernels; -1 (default) = 2
 *   "gemm_trace"    device address of an int64 buffer (16 per tile) that the
 *                   next tcgen05 launches fill with per-tile clock64 stamps
 *                   (0 = off; debug only)
 *   "gemm_trace_launch" trace only the launch with this index inside an
 *                   attn_softmax_fwd_bwd call (-1 = every launch)
 *   "mn_3d_tma"     1 (default) = load MN-major operand tiles with one 3D TMA
 *                   box per stage; 0 = one 2D box per 64-wide atom
 *   "debug_epilogue" attn_debug_gemm_bf16 epilogue: 0 = fp32 TMA store,
 *                   1 = read the accumulator only (mainloop timing)         */
attn_status_t attn_softmax_set_option(const char* key, int64_t value);

#ifdef __cplusplus
}
#endif
#endif /* ATTN_SOFTMAX_DEBUG_H */
