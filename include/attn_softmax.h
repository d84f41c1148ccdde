/*
 * attn_softmax.h -- C ABI of libattnsm.so, the B200 (sm_100a) attention-softmax
 * stage of arXiv 1909.00562 (the data-parallel half of the hybrid scheme,
 * Fig. 3), forward and backward.
 *
 * The operation (section 3.2, Eqs. 1-6; readings R1-R11 in DESIGN.md):
 *   per sentence b and target row i (all rows computed, only valid rows count)
 *     e_ij   = H_dec[b,i] . H_enc[b,j]                    Eq. 2,
 *                                                          dot form, W_alpha = I (R1);
 *                                                          with W_alpha: (H_dec W_alpha) . H_enc
 *     alpha  = softmax_j(e_i) over j < src_len[b]; 0 else  Eq. 1
 *     C_i    = sum_j alpha_ij H_enc[b,j]                   Eq. 3
 *     Hc_i   = tanh(W_c[:, :d] H_i + W_c[:, d:] C_i)       Eq. 4
 *     l_iv   = W_out[v] . Hc_i                             Eq. 5
 *     loss   = loss_scale * sum_{valid (b,i)} (logsumexp_v l_iv - l_{i,y_i})
 *                                                          Eq. 6
 *   and the gradients of loss w.r.t. H_dec, H_enc, W_c, W_out.  With a
 *   communicator, dW_c, dW_out and loss are summed over ranks (the rootless
 *   equivalent of "GPU 0 as the root for accumulating and synchronizing",
 *   PAPER.md:121).
 *
 * Layouts: all matrices are dense row-major with no padding between rows.
 *   H_dec [B,N,d]  decoder top-layer states (the paper's H, transposed)
 *   H_enc [B,M,d]  encoder top-layer states (the paper's S, transposed)
 *   W_c   [d,2d]   columns [0,d) multiply H, [d,2d) multiply C (paper order
 *                  [H;C], R5; north_star's "W_c[c;h]" is the same matrix with
 *                  its column halves swapped)
 *   W_out [V,d]    F_c of Eq. 5, no bias (R6)
 *   tgt_ids [B,N] int32, read only where i < tgt_len[b]
 * dtype ATTN_BF16: H_dec, H_enc, W_c, W_out, dH_dec, dH_enc are bf16; all
 *   accumulation, softmax statistics, loss and dW_c / dW_out are fp32.
 * dtype ATTN_F32: everything fp32 (CUDA-core path, for the parity config).
 *
 * Ownership: the caller allocates and frees every buffer, including the
 *   workspace (size from attn_softmax_workspace_size).  The library never
 *   allocates device memory inside attn_softmax_fwd_bwd.  attn_comm_t is owned
 *   by the library between attn_comm_init and attn_comm_destroy.
 * Semantics: calls are asynchronous on `stream` (a cudaStream_t); every output
 *   is final when the stream reaches the end of the enqueued work (including
 *   the allreduce).  Gradients are OVERWRITTEN.  Inputs are read-only.  Padded
 *   slots (j >= src_len, i >= tgt_len) may hold any finite values and do not
 *   affect any output; padded rows of dH_dec / dH_enc are written as exact 0.
 * Errors: every entry point returns attn_status_t; attn_last_error() gives a
 *   thread-local message naming the offending argument (and both shapes for a
 *   shape mismatch).  No partial work is enqueued on a validation
 *   error.
 */
#ifndef ATTN_SOFTMAX_H
#define ATTN_SOFTMAX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ATTN_OK = 0,
  ATTN_ERR_INVALID_ARG = 1,  /* null pointer, bad enum, negative size        */
  ATTN_ERR_SHAPE = 2,        /* src_len > M, tgt_len > N, or d, V, B <= 0    */
  ATTN_ERR_EMPTY_SOURCE = 3, /* some src_len[b] < 1       */
  ATTN_ERR_NO_TARGETS = 4,   /* sum_b tgt_len[b] == 0          */
  ATTN_ERR_TOKEN_RANGE = 5,  /* a valid target id outside [0, V);
                                checked only by attn_softmax_check_ids      */
  ATTN_ERR_WORKSPACE = 6,    /* workspace_bytes < attn_softmax_workspace_size */
  ATTN_ERR_UNSUPPORTED = 7,  /* dtype/shape/alignment the kernels do not take:
                                bf16 needs d % 64 == 0 and 16-byte aligned
                                pointers                                     */
  ATTN_ERR_CUDA = 8,         /* a CUDA runtime/driver call failed            */
  ATTN_ERR_NCCL = 9          /* NCCL missing or a NCCL call failed           */
} attn_status_t;

typedef enum { ATTN_F32 = 0, ATTN_BF16 = 1 } attn_dtype_t;

/* Local (per-GPU) shard shape: B sentences, N padded target steps, M padded
 * source positions, d hidden size, V vocabulary size. */
typedef struct {
  int32_t batch;    /* B */
  int32_t tgt_len;  /* N */
  int32_t src_len;  /* M */
  int32_t hidden;   /* d */
  int32_t vocab;    /* V */
  attn_dtype_t dtype;
} attn_shape_t;

typedef struct attn_comm attn_comm_t; /* opaque: NCCL communicator + comm stream */

/* Bytes of device workspace attn_softmax_fwd_bwd needs for shape *s (0 on an
 * invalid shape; see attn_last_error). */
size_t attn_softmax_workspace_size(const attn_shape_t* s);

/* The whole stage, forward + backward, on `stream`.
 *   src_lens_host, tgt_lens_host: [B] HOST arrays, validated and copied.
 *   tgt_ids: [B,N] device int32.
 *   W_alpha / dW_alpha: both NULL = the dot score of the hot path (R1:
 *     e_ij = H_dec[b,i] . H_enc[b,j]); both set = the Eq. 2 "general" score
 *     alpha_hat = H^T W_alpha S, row form
 *     e_ij = (H_dec[b,i] W_alpha) . H_enc[b,j].  W_alpha [d,d] row-major in
 *     s->dtype (read-only); dW_alpha [d,d] fp32, overwritten (allreduced with
 *     the other weight gradients when comm != NULL).  Exactly one of the two
 *     NULL is ATTN_ERR_INVALID_ARG.  The host-buffer variants below use the
 *     dot score.
 *   loss_scale: multiplies the summed token NLL (the harness passes
 *     1 / global valid target tokens, R9).
 *   loss: [1] device fp32 = loss_scale * sum of this shard's token NLL
 *     (summed over ranks when comm != NULL).
 *   dH_dec [B,N,d], dH_enc [B,M,d]: dtype s->dtype, overwritten.
 *   dW_c [d,2d], dW_out [V,d]: fp32, overwritten (allreduced when comm).
 *   comm: NULL for local gradients.  The first call of a path (shape,
 *     operands, options) with a communicator on a device first runs the stage
 *     once locally (same outputs, overwritten): it loads every kernel of the
 *     path before the comm stream's spinning per-chunk wait kernels start
 *     (under lazy module loading a first launch could otherwise wait for
 *     them: a deadlock). */
attn_status_t attn_softmax_fwd_bwd(
    const attn_shape_t* s,
    const void* H_dec, const void* H_enc,
    const int32_t* src_lens_host, const int32_t* tgt_lens_host,
    const int32_t* tgt_ids,
    const void* W_c, const void* W_out, const void* W_alpha,
    float loss_scale,
    float* loss,
    void* dH_dec, void* dH_enc,
    float* dW_c, float* dW_out, float* dW_alpha,
    void* workspace, size_t workspace_bytes,
    attn_comm_t* comm,
    void* stream);

/* attn_softmax_fwd_bwd plus the optional F_c bias of Eq. 5 (NEXT-1):
 *   b_out [V] (s->dtype, read-only) makes the logits l_iv = W_out[v] . Hc_i +
 *   b_out[v] (SPEC.md:171's "Hdim x V plus bias" reading of the paper's
 *   linear F_c); db_out [V] fp32 receives
 *   sum_{valid rows} loss_scale (softmax(l_i) - onehot(y_i)), overwritten
 *   (allreduced when comm != NULL).  b_out and db_out are both NULL (no bias:
 *   identical to attn_softmax_fwd_bwd) or both set, else
 *   ATTN_ERR_INVALID_ARG.  Everything else as attn_softmax_fwd_bwd. */
attn_status_t attn_softmax_fwd_bwd_ex(
    const attn_shape_t* s,
    const void* H_dec, const void* H_enc,
    const int32_t* src_lens_host, const int32_t* tgt_lens_host,
    const int32_t* tgt_ids,
    const void* W_c, const void* W_out, const void* W_alpha, const void* b_out,
    float loss_scale,
    float* loss,
    void* dH_dec, void* dH_enc,
    float* dW_c, float* dW_out, float* dW_alpha, float* db_out,
    void* workspace, size_t workspace_bytes,
    attn_comm_t* comm,
    void* stream);

/* End-to-end variant for callers whose per-step activations live in HOST
 * memory (pinned for overlap): H_dec_host, H_enc_host and tgt_ids_host are
 * copied host->device into `staging` (size attn_softmax_host_staging_size),
 * the stage runs as attn_softmax_fwd_bwd, and the loss is copied back into
 * loss_host.  Weights and gradients stay on the device.  loss_host is valid
 * once `stream` has reached the end of the enqueued work. */
size_t attn_softmax_host_staging_size(const attn_shape_t* s);
attn_status_t attn_softmax_fwd_bwd_host(
    const attn_shape_t* s,
    const void* H_dec_host, const void* H_enc_host,
    const int32_t* src_lens_host, const int32_t* tgt_lens_host,
    const int32_t* tgt_ids_host,
    const void* W_c, const void* W_out,
    float loss_scale,
    float* loss_host,
    void* dH_dec, void* dH_enc,
    float* dW_c, float* dW_out,
    void* staging, size_t staging_bytes,
    void* workspace, size_t workspace_bytes,
    attn_comm_t* comm,
    void* stream);

/* Pipelined host-buffer variant (double-buffered staging).
 * attn_softmax_prefetch_host enqueues the host->device copy of one step's
 * activations (H_dec, H_enc, tgt_ids from HOST, pinned for overlap) into
 * `staging` on the library's own copy stream, ordered after all work already
 * enqueued on `stream` (so a staging buffer the previous step still reads is
 * not overwritten).  attn_softmax_fwd_bwd_staged then runs the stage on a
 * prefetched staging buffer (waiting only for that buffer's copy) and copies
 * the loss into loss_host.  A training loop prefetches step i+1 into the
 * other buffer before running step i, so the copies overlap the compute.
 * staging_bytes >= attn_softmax_host_staging_size(s). */
attn_status_t attn_softmax_prefetch_host(
    const attn_shape_t* s,
    const void* H_dec_host, const void* H_enc_host, const int32_t* tgt_ids_host,
    void* staging, size_t staging_bytes,
    void* stream);
attn_status_t attn_softmax_fwd_bwd_staged(
    const attn_shape_t* s,
    const void* staging, size_t staging_bytes,
    const int32_t* src_lens_host, const int32_t* tgt_lens_host,
    const void* W_c, const void* W_out,
    float loss_scale,
    float* loss_host,
    void* dH_dec, void* dH_enc,
    float* dW_c, float* dW_out,
    void* workspace, size_t workspace_bytes,
    attn_comm_t* comm,
    void* stream);

/* Debug-build style check of the valid target ids: synchronous, returns
 * ATTN_ERR_TOKEN_RANGE if any tgt_ids[b,i] (i < tgt_len[b]) is outside [0,V). */
attn_status_t attn_softmax_check_ids(const attn_shape_t* s,
                                     const int32_t* tgt_lens_host,
                                     const int32_t* tgt_ids, void* stream);

/* In-place sum allreduce of `count` fp32 values over the communicator's ranks,
 * enqueued on `stream`. */
attn_status_t attn_grad_allreduce(attn_comm_t* c, float* buf, size_t count,
                                  void* stream);

/* Communicator bootstrap: rank 0 creates a 128-byte id, the harness
 * broadcasts it, every rank calls attn_comm_init on its own device. */
attn_status_t attn_comm_get_unique_id(uint8_t id[128]);
attn_status_t attn_comm_init(const uint8_t id[128], int nranks, int rank,
                             int device, attn_comm_t** out);
attn_status_t attn_comm_destroy(attn_comm_t* c);

/* Failure detection: wait until every collective this
 * communicator has enqueued (by attn_softmax_fwd_bwd or attn_grad_allreduce)
 * has completed, polling ncclCommGetAsyncError every millisecond.  Returns
 * ATTN_OK when the work is done; ATTN_ERR_NCCL (after ncclCommAbort, which
 * leaves the communicator unusable: destroy it) when NCCL reports an
 * asynchronous error -- a peer died, a link failed -- or when `timeout_ms`
 * (> 0) elapses first (a hang: some rank never joined the collective).  The
 * caller keeps running either way instead of blocking forever in a
 * synchronize.  Host-blocking; call it from the training loop between steps. */
attn_status_t attn_comm_poll(attn_comm_t* c, int64_t timeout_ms);
/* Ranks in the communicator (1 for a NULL communicator). */
int attn_comm_nranks(const attn_comm_t* c);

/* ---- NEXT-4: forward-only decoding step -----------------------------------
 * One step of beam-search decoding (section 4.4) on the stage:
 * shape s holds B sentences with N = live hypotheses per sentence (tgt_len),
 * M source positions; H_dec [B,N,d] are the hypotheses' decoder top-layer
 * states, H_enc [B,M,d] the sentences' encoder states (shared by their
 * hypotheses); Eqs. 1-5 (W_alpha: general score, b_out: F_c bias, both
 * nullable) give log P(v) = l_v - logsumexp(l) per row.  Outputs, per row
 * t = b*N + i: topk_ids [T,k] int32 and topk_logp [T,k] fp32, the k best
 * tokens by log-probability descending (ties: lower id first),
 * and lse [T] fp32 (nullable).  1 <= k <= 8.  The logits are never stored:
 * the vocab GEMM epilogue keeps per-tile (max, sumexp) and top-8 lists.
 * bf16 only (ATTN_ERR_UNSUPPORTED for fp32).  Workspace from
 * attn_softmax_decode_workspace_size (0 for an invalid / fp32 shape). */
size_t attn_softmax_decode_workspace_size(const attn_shape_t* s);
attn_status_t attn_softmax_decode_step(
    const attn_shape_t* s,
    const void* H_dec, const void* H_enc,
    const int32_t* src_lens_host,
    const void* W_c, const void* W_out, const void* W_alpha, const void* b_out,
    int k, int32_t* topk_ids, float* topk_logp, float* lse,
    void* workspace, size_t workspace_bytes,
    void* stream);

/* ---- NEXT-2: the optimizer step after the gradient exchange --------------
 * Adam (Kingma & Ba 2015, Algorithm 1), the optimizer of the paper
 * (PAPER.md:195 Table 2, :207: beta1 0.9, beta2 0.999, eps 1e-8, lr 1e-3):
 *   m = b1 m + (1-b1) g;  v = b2 v + (1-b2) g^2;
 *   w -= lr (m / (1 - b1^step)) / (sqrt(v / (1 - b2^step)) + eps)
 * in fp32 on device buffers, asynchronously on `stream`. */
typedef struct {
  double lr, beta1, beta2, eps; /* double so 1 - beta2 = 1e-3 is exact enough */
  int32_t step; /* t >= 1 of Algorithm 1 (bias corrections 1 - beta^t) */
} attn_adam_t;

/* Replicated update of n parameters: w, m, v [n] fp32 (in/out, 16-byte
 * aligned), g [n] fp32 (the summed gradient, read-only); w_bf16 [n] bf16 (out,
 * 8-byte aligned) receives bf16(w) for the next step's GEMMs, or NULL. */
attn_status_t attn_adam_step(const attn_adam_t* h, size_t n, float* w, float* m,
                             float* v, const float* g, void* w_bf16, void* stream);

/* Per-rank shard length S of an n-parameter vector on communicator c: the
 * smallest multiple of 4 with nranks * S >= n (1 rank when c is NULL). */
size_t attn_adam_shard_len(const attn_comm_t* c, size_t n);

/* Sharded update (data-parallel ZeRO-1 style): g [nranks*S] fp32 holds this
 * rank's LOCAL gradient of n parameters (the tail [n, nranks*S) is zeroed by
 * the call); it is reduce-scattered in place (sum over ranks, NCCL), rank r
 * updates its shard [r S, (r+1) S) with w_shard, m_shard, v_shard [S] fp32
 * (its fp32 master weights and moments), writes bf16 weights into
 * w_bf16 + r S, and w_bf16 [nranks*S] bf16 is all-gathered in place, so every
 * rank ends with the full updated bf16 weights.  Wire bytes per parameter:
 * 4 (reduce-scatter) + 2 (all-gather) instead of 8 for an fp32 allreduce.
 * All buffers 16-byte aligned. */
attn_status_t attn_adam_step_sharded(attn_comm_t* c, const attn_adam_t* h, size_t n,
                                     float* g, float* w_shard, float* m_shard,
                                     float* v_shard, void* w_bf16, void* stream);

/* ---------------------------------------------------------------- NEXT-3
 * The model-parallel half of Fig. 3: the stacked-LSTM
 * encoder and decoder WITHOUT input feeding that produce
 * H_enc (the paper's S) and H_dec (H), the inputs of attn_softmax_fwd_bwd.
 * Forward only.  Cell (PyTorch gate order i, f, g, o; N1-N4):
 *   gates = W_ih x_t + W_hh h_{t-1} + b;  c_t = s(f) c_{t-1} + s(i) tanh(g);
 *   h_t = s(o) tanh(c_t).  Encoder: zero initial state, over all M steps;
 *   decoder layer l starts from encoder layer l's (h, c) at source step
 *   src_len[b] - 1, over all N steps.  Layer-step (l, t) depends only on
 *   (l, t-1) and (l-1, t): the kernels run that wavefront
 *   with SM groups in the role of the paper's GPUs. */
typedef struct {
  int32_t batch;      /* B <= 128 sentences (one 128-row MMA tile per step) */
  int32_t src_len;    /* M, padded source length */
  int32_t tgt_len;    /* N, padded target length */
  int32_t emb;        /* embedding size e (Table 1: 512), multiple of 64 */
  int32_t hidden;     /* hidden size h (Table 1: 1024), multiple of 64 */
  int32_t layers;     /* L in [1, 8] (Table 1: 4) */
  int32_t vocab_src, vocab_tgt;
} attn_lstm_shape_t;

/* Workspace bytes of attn_encoder_decoder_fwd (0 on an invalid shape). */
size_t attn_lstm_workspace_size(const attn_lstm_shape_t* s);
/* Bytes of one packed layer: bf16 [4 hidden][in + hidden]. */
size_t attn_lstm_packed_bytes(int in, int hidden);
/* Pack one layer for the kernels: W_ih [4h][in], W_hh [4h][h], b [4h] (bf16,
 * PyTorch layout: gate blocks i, f, g, o) -> W_packed [4h][in + h] bf16 with
 * row 4u + q = [W_ih | W_hh] row q h + u (gate-interleaved) and b_packed [4h]
 * fp32 likewise.  Device buffers, asynchronous on `stream`. */
attn_status_t attn_lstm_pack_layer(int in, int hidden, const void* W_ih, const void* W_hh,
                                   const void* b, void* W_packed, float* b_packed, void* stream);
/* Encoder-decoder forward.  src_ids [B][M], tgt_ids [B][N] int32 (device,
 * every id in [0, vocab)); src_lens_host [B] HOST (1 <= len <= M); E_src
 * [vocab_src][e], E_tgt [vocab_tgt][e] bf16; enc_W / dec_W: HOST arrays of
 * `layers` device pointers to packed layers (attn_lstm_pack_layer; layer 0
 * has in = e, the others in = h), enc_b / dec_b likewise (packed fp32 biases).
 * Outputs H_enc [B][M][h], H_dec [B][N][h] bf16 (the top layer's states at
 * every step).  Errors: ATTN_ERR_UNSUPPORTED for B > 128, sizes not multiples
 * of 64 or layers x (h / 32) CTAs beyond the SM count; ATTN_ERR_SHAPE for a
 * source length outside [1, M]. */
attn_status_t attn_encoder_decoder_fwd(
    const attn_lstm_shape_t* s, const int32_t* src_ids, const int32_t* tgt_ids,
    const int32_t* src_lens_host, const void* E_src, const void* E_tgt,
    const void* const* enc_W, const float* const* enc_b, const void* const* dec_W,
    const float* const* dec_b, void* H_enc, void* H_dec, void* workspace,
    size_t workspace_bytes, void* stream);

/* Training (the backward of the encoder-decoder, "the
 * alternation of data parallelism and model parallelism on the backward
 * process goes in a similar but opposite direction"):
 * attn_encoder_decoder_fwd_train is attn_encoder_decoder_fwd that also keeps,
 * in its (larger) workspace, every layer's states, cell states and gate
 * activations; attn_encoder_decoder_bwd then takes the stage's dH_enc / dH_dec
 * (bf16, e.g. the outputs of attn_softmax_fwd_bwd) and the forward's H_enc /
 * H_dec, runs the reverse wavefront (top layer first, t = T-1 down to 0; the
 * decoder before the encoder, whose layer-l state at src_len - 1 receives the
 * decoder's initial-state gradient) and writes per layer dW [4h][in + h] fp32
 * and db [4h] fp32 in the PACKED (gate-interleaved) order of
 * attn_lstm_pack_layer (row 4u + q = gate q of unit u; columns [0, in) the
 * W_ih part), and dE_src [vocab_src][e], dE_tgt [vocab_tgt][e] fp32 (the
 * embedding rows are summed with atomics: their summation order is not
 * fixed).  The same workspace must be passed to both calls. */
size_t attn_lstm_train_workspace_size(const attn_lstm_shape_t* s);
attn_status_t attn_encoder_decoder_fwd_train(
    const attn_lstm_shape_t* s, const int32_t* src_ids, const int32_t* tgt_ids,
    const int32_t* src_lens_host, const void* E_src, const void* E_tgt,
    const void* const* enc_W, const float* const* enc_b, const void* const* dec_W,
    const float* const* dec_b, void* H_enc, void* H_dec, void* workspace,
    size_t workspace_bytes, void* stream);
attn_status_t attn_encoder_decoder_bwd(
    const attn_lstm_shape_t* s, const int32_t* src_ids, const int32_t* tgt_ids,
    const int32_t* src_lens_host, const void* const* enc_W, const void* const* dec_W,
    const void* H_enc, const void* H_dec, const void* dH_enc, const void* dH_dec,
    float* const* dW_enc, float* const* db_enc, float* const* dW_dec, float* const* db_dec,
    float* dE_src, float* dE_tgt, void* workspace, size_t workspace_bytes, void* stream);

/* HybridNMTIF (the baseline model's input feeding, PAPER.md:75,
 * :99): the same encoder, and a decoder whose layer-0 input at step t is
 * [E_tgt[y_t] ; Htilde_{t-1}] (Htilde_{-1} = 0), where Htilde_t =
 * tanh(W_c [h_t ; C_t]) is Eq. 4 of the stage on the top-layer state h_t and
 * the attention context C_t over H_enc (Eqs. 1-3, dot score, src_len mask).
 * The steps therefore run one after another (one wavefront launch over the
 * layers per step, then the fused attention step).  dec_W[0] is packed with
 * in = emb + hidden.  Outputs H_enc [B][M][h], H_dec [B][N][h] and Htilde
 * [B][N][h] (bf16).  W_c [h][2h] bf16 as in attn_softmax_fwd_bwd.  M <= 128. */
size_t attn_lstm_if_workspace_size(const attn_lstm_shape_t* s);
attn_status_t attn_encoder_decoder_if_fwd(
    const attn_lstm_shape_t* s, const int32_t* src_ids, const int32_t* tgt_ids,
    const int32_t* src_lens_host, const void* E_src, const void* E_tgt,
    const void* const* enc_W, const float* const* enc_b, const void* const* dec_W,
    const float* const* dec_b, const void* W_c, void* H_enc, void* H_dec, void* Htilde,
    void* workspace, size_t workspace_bytes, void* stream);

/* MP -> DP hand-over ("the intermediate results of all hidden
 * states ... are distributed equally to 4 GPUs"): rank `root` holds `full`
 * [B_global][rows][hidden] bf16 (H_enc with rows = M, or H_dec with rows =
 * N); every rank receives its contiguous sentence shard (sizes differing by
 * at most one, lower ranks first) into `shard` [B_r][rows][hidden], by NCCL
 * point-to-point on `stream`.  `full` is read on the root only. */
attn_status_t attn_hidden_scatter(attn_comm_t* c, int root, int B_global, int rows, int hidden,
                                  const void* full, void* shard, void* stream);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* attn_last_error(void);

/* Library version string, e.g. "attnsm 0.1 sm_100a". */
const char* attn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ATTN_SOFTMAX_H */
