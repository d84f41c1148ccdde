"""fp64 CPU oracle for the attention-softmax stage (forward + backward).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_1909_00562_b200``) never imports, links or
executes anything under ``oracle/``; the two share no code.

What it computes is the plain definition of the right-hand (data-parallel) half
of Fig. 3 of arXiv 1909.00562 ("Hybrid Data-Model Parallel Training for
Sequence-to-Sequence RNN MT"), section 3.2, written out step by step in the
paper's order and notation, in float64, with a two-pass (max, then sum) softmax
and no fusion, chunking or online-LSE reformulation:

  Eq. 1  alpha = Softmax(alpha_hat)            (over source j)
  Eq. 2  alpha_hat = H^T W_alpha S             (W_alpha = I on
                                                                    the hot path,
                                                                    DESIGN.md R1)
  Eq. 3  C = alpha . S
  Eq. 4  H_c = tanh(W_c [H; C])
  Eq. 5  P = Softmax{F_c(H_c)},  F_c(x) = W_out x (no bias on
                                                     the hot path, R6; optional
                                                     b_out: F_c(x) = W_out x + b_out,
                                                     SPEC.md:171, NEXT-1)
  Eq. 6  P_i = P(y_i | y_<i, x); loss = scale * sum -log P_i(y_i)

The backward pass is the closed-form reverse-mode derivative of the above
(chain rule, step by step).

Storage convention (row-major, R4): H_dec [B,N,d], H_enc [B,M,d]
(the paper's column-stacked H, S transposed), W_c [d,2d] whose columns [0,d)
multiply H and [d,2d) multiply C (paper order [H;C], R5), W_out [V,d].

Every public function says which passage it follows.  Masking (R8): source
position j of sentence b takes part iff j < src_len[b]; alpha is exactly 0
elsewhere.  Target row (b,i) contributes to the loss iff i < tgt_len[b].

Parity pins: every function here is pinned by tests/test_oracle_pins.py (worked
examples E1-E5, invariants, central finite differences, torch float64 autograd
and library special cases).  No function is "parity unpinned".
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "attention_scores", "attention_weights", "context_vectors",
    "context_decoded", "vocab_logits", "log_sum_exp", "token_nll",
    "forward", "backward", "fwd_bwd", "decode_step",
]

F64 = np.float64


def _f64(x):
    return np.asarray(x, dtype=F64)


# --------------------------------------------------------------------------
# Forward, Eqs. 1-6
# --------------------------------------------------------------------------

def attention_scores(H_dec, H_enc, W_alpha=None):
    """Eq. 2: alpha_hat = H^T W_alpha S, per sentence.

    Row form: e[b,i,j] = q[b,i] . S[b,j] with q = H W_alpha (q = H when
    W_alpha is None, the "dot" score of the hot path, R1).
    Returns (e [B,N,M], q [B,N,d]).  No masking here (masking is Eq. 1's).
    """
    H = _f64(H_dec)
    S = _f64(H_enc)
    if W_alpha is None:
        q = H
    else:
        q = H @ _f64(W_alpha)          # h^T W_alpha as a row vector
    e = q @ np.swapaxes(S, 1, 2)       # [B,N,d] x [B,d,M]
    return e, q


def attention_weights(e, src_len):
    """Eq. 1: alpha = Softmax(alpha_hat) over source j.

    Two-pass softmax restricted to j < src_len[b] (reading R3, R8): first the
    row max over the unmasked positions, then exp and the sum.  Masked
    positions are exactly 0.
    """
    e = _f64(e)
    B, N, M = e.shape
    alpha = np.zeros_like(e)
    for b in range(B):
        L = int(src_len[b])
        if L < 1:
            raise ValueError(f"sentence {b}: src_len must be >= 1 (got {L})")
        x = e[b, :, :L]
        m = x.max(axis=1, keepdims=True)             # pass 1: max
        p = np.exp(x - m)
        alpha[b, :, :L] = p / p.sum(axis=1, keepdims=True)   # pass 2: sum
    return alpha


def context_vectors(alpha, H_enc):
    """Eq. 3: C_i = sum_j alpha_ij S_j (reading R4)."""
    return _f64(alpha) @ _f64(H_enc)


def context_decoded(H_dec, C, W_c):
    """Eq. 4: H_c = tanh(W_c [H; C]).

    Row form: z = h W_c[:, :d]^T + c W_c[:, d:]^T, H_c = tanh(z) (R5: the
    paper's concat order [H; C]).  Returns (z, H_c), both [B,N,d].
    """
    H = _f64(H_dec)
    C = _f64(C)
    W_c = _f64(W_c)
    d = H.shape[-1]
    z = H @ W_c[:, :d].T + C @ W_c[:, d:].T
    return z, np.tanh(z)


def vocab_logits(Hc_rows, W_out, b_out=None):
    """Eq. 5: F_c(H_c) = W_out h_c for each row (no bias on
    the hot path, R6); with b_out [V] the "liner function" F_c carries SPEC's
    bias: W_out h_c + b_out.

    Hc_rows [R,d] -> logits [R,V].
    """
    logits = _f64(Hc_rows) @ _f64(W_out).T
    if b_out is not None:
        logits = logits + _f64(b_out)[None, :]
    return logits


def log_sum_exp(logits):
    """Normaliser of the Eq. 5 softmax, two-pass: m = max_v l_v;
    lse = m + log sum_v exp(l_v - m).  logits [R,V] -> lse [R]."""
    logits = _f64(logits)
    m = logits.max(axis=1)
    return m + np.log(np.exp(logits - m[:, None]).sum(axis=1))


def token_nll(logits, lse, y):
    """Eq. 6: -log P_i(y_i) = lse_i - l_{i,y_i}."""
    rows = np.arange(len(y))
    return _f64(lse) - _f64(logits)[rows, np.asarray(y)]


def _valid_rows(tgt_len, B, N):
    """Row t = (b,i) is valid iff i < tgt_len[b] (R8).  Returns bool [B*N]."""
    valid = np.zeros((B, N), dtype=bool)
    for b in range(B):
        valid[b, : int(tgt_len[b])] = True
    return valid.reshape(-1)


def forward(H_dec, H_enc, src_len, tgt_len, tgt_ids, W_c, W_out, loss_scale,
            W_alpha=None, b_out=None):
    """Eqs. 1-6 in order.  Returns a dict of every intermediate (fp64)."""
    H = _f64(H_dec)
    S = _f64(H_enc)
    B, N, d = H.shape
    e, q = attention_scores(H, S, W_alpha)                     # Eq. 2
    alpha = attention_weights(e, src_len)                      # Eq. 1
    C = context_vectors(alpha, S)                              # Eq. 3
    z, Hc = context_decoded(H, C, W_c)                         # Eq. 4
    Hc_rows = Hc.reshape(B * N, d)
    logits = vocab_logits(Hc_rows, W_out, b_out)               # Eq. 5
    lse = log_sum_exp(logits)
    y = np.asarray(tgt_ids).reshape(-1)
    valid = _valid_rows(tgt_len, B, N)
    y_safe = np.where(valid, y, 0)     # padded ids are never read (R8)
    nll = token_nll(logits, lse, y_safe)                       # Eq. 6
    nll = np.where(valid, nll, 0.0)
    loss = float(loss_scale) * nll.sum()
    return dict(e=e, q=q, alpha=alpha, C=C, z=z, Hc=Hc, logits=logits,
                lse=lse, nll=nll, valid=valid, y=y_safe, loss=loss)


# --------------------------------------------------------------------------
# Backward: reverse-mode derivative of forward(), step by step
# (DP gradient sum semantics PAPER.md:121)
# --------------------------------------------------------------------------

def backward(H_dec, H_enc, src_len, W_c, W_out, loss_scale, fwd, W_alpha=None,
             b_out=None):
    """Gradients of loss w.r.t. H_dec, H_enc, W_c, W_out (and W_alpha, b_out).

    Step 8  dl_iv = scale (softmax(l_i)_v - [v = y_i]) on valid rows, else 0
    Step 9  dW_out = sum_rows dl_i^T hc_i ; dhc_i = sum_v dl_iv W_out[v]
            (b_out: db_out = sum_rows dl_i)
    Step 10 dz = dhc * (1 - hc^2) ; dW_c = sum_i dz_i [h_i ; c_i]^T
    Step 11 dh_i = W_c[:, :d]^T dz_i ; dc_i = W_c[:, d:]^T dz_i
    Step 12 dalpha_ij = dc_i . S_j ; D_i = sum_j alpha_ij dalpha_ij ;
            de_ij = alpha_ij (dalpha_ij - D_i)
    Step 13 dq_i = sum_j de_ij S_j ; dh_i += dq_i  (W_alpha: dh_i += W_alpha dq_i,
            dW_alpha = sum_i h_i dq_i^T)
    Step 14 dS_j = sum_i alpha_ij dc_i + sum_i de_ij q_i
    """
    H = _f64(H_dec)
    S = _f64(H_enc)
    W_c = _f64(W_c)
    W_out = _f64(W_out)
    B, N, d = H.shape
    alpha, C, Hc, q = fwd["alpha"], fwd["C"], fwd["Hc"], fwd["q"]
    logits, lse, valid, y = fwd["logits"], fwd["lse"], fwd["valid"], fwd["y"]

    # step 8
    P = np.exp(logits - lse[:, None])
    onehot = np.zeros_like(P)
    onehot[np.arange(len(y)), y] = 1.0
    dl = float(loss_scale) * (P - onehot)
    dl[~valid] = 0.0
    # step 9
    Hc_rows = Hc.reshape(B * N, d)
    dW_out = dl.T @ Hc_rows
    db_out = dl.sum(axis=0) if b_out is not None else None
    dHc = (dl @ W_out).reshape(B, N, d)
    # step 10
    dz = dHc * (1.0 - Hc * Hc)
    dz_rows = dz.reshape(B * N, d)
    dW_c = np.concatenate([dz_rows.T @ H.reshape(B * N, d),
                           dz_rows.T @ C.reshape(B * N, d)], axis=1)
    # step 11
    dH = dz @ W_c[:, :d]
    dC = dz @ W_c[:, d:]
    # step 12
    dalpha = dC @ np.swapaxes(S, 1, 2)
    D = (alpha * dalpha).sum(axis=2, keepdims=True)
    de = alpha * (dalpha - D)
    # step 13
    dq = de @ S
    dW_alpha = None
    if W_alpha is None:
        dH = dH + dq
    else:
        W_a = _f64(W_alpha)
        dH = dH + dq @ W_a.T
        dW_alpha = H.reshape(B * N, d).T @ dq.reshape(B * N, d)
    # step 14
    dS = np.swapaxes(alpha, 1, 2) @ dC + np.swapaxes(de, 1, 2) @ q
    return dict(dlogits=dl, dHc=dHc, dz=dz, dC=dC, dalpha=dalpha, de=de,
                dH_dec=dH, dH_enc=dS, dW_c=dW_c, dW_out=dW_out,
                dW_alpha=dW_alpha, db_out=db_out)


def fwd_bwd(H_dec, H_enc, src_len, tgt_len, tgt_ids, W_c, W_out, loss_scale,
            W_alpha=None, b_out=None):
    """The whole stage: forward (Eqs. 1-6) then backward.  Returns
    (fwd dict, bwd dict)."""
    fwd = forward(H_dec, H_enc, src_len, tgt_len, tgt_ids, W_c, W_out,
                  loss_scale, W_alpha, b_out)
    bwd = backward(H_dec, H_enc, src_len, W_c, W_out, loss_scale, fwd, W_alpha,
                   b_out)
    return fwd, bwd


# --------------------------------------------------------------------------
# NEXT-4: forward-only decoding step
# --------------------------------------------------------------------------

def decode_step(H_dec, H_enc, src_len, W_c, W_out, k, W_alpha=None, b_out=None):
    """One step of beam-search decoding on the stage (§4.4; the
    per-step output distribution of Eqs. 1-5): for each of
    the N live hypotheses of sentence b (rows H_dec[b, i], all attending over
    the same encoder states H_enc[b]), log P(v) = l_v - logsumexp(l) and its k
    best tokens, ordered by log-probability descending, ties by the lower
    token id (SPEC.md:541 determinism).  Returns (ids [B,N,k] int64,
    logp [B,N,k] fp64, lse [B,N] fp64)."""
    H = _f64(H_dec)
    B, N, d = H.shape
    e, _ = attention_scores(H, H_enc, W_alpha)                  # Eq. 2
    alpha = attention_weights(e, src_len)                       # Eq. 1
    C = context_vectors(alpha, H_enc)                           # Eq. 3
    _, Hc = context_decoded(H, C, W_c)                          # Eq. 4
    logits = vocab_logits(Hc.reshape(B * N, d), W_out, b_out)   # Eq. 5
    lse = log_sum_exp(logits)
    logp = logits - lse[:, None]
    V = logp.shape[1]
    ids = np.empty((B * N, k), np.int64)
    vals = np.empty((B * N, k))
    for r in range(B * N):
        order = np.lexsort((np.arange(V), -logp[r]))[:k]     # value desc, id asc
        ids[r] = order
        vals[r] = logp[r, order]
    return ids.reshape(B, N, k), vals.reshape(B, N, k), lse.reshape(B, N)
