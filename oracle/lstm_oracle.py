"""fp64 CPU oracle for the model-parallel half of Fig. 3 (NEXT-3): the
stacked-LSTM encoder and decoder that produce the hidden states S (= H_enc)
and H (= H_dec) the attention-softmax stage consumes.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu baseline may import this module; the product path never
imports, links or executes it, and the two share no code.

What it computes (§3.1-3.2; Table 1 PAPER.md:190-192 gives
the sizes: embedding 512, hidden 1024, 4 stacked LSTM layers):

* the proposed HybridNMT model REMOVES input feeding, so
  the decoder's first layer sees only the target word embedding, and every
  layer-step (l, t) depends only on (l, t-1) and (l-1, t) -- the "green arrow"
  wavefront of Fig. 3;
* each layer is the standard LSTM cell of Luong et al. (the baseline the paper
  builds on), with PyTorch's gate order (i, f, g, o):
      gates = W_ih x_t + W_hh h_{t-1} + b
      i = sigma(gates_i), f = sigma(gates_f), g = tanh(gates_g), o = sigma(gates_o)
      c_t = f * c_{t-1} + i * g,   h_t = o * tanh(c_t)
  (readings N1-N4 in DESIGN.md: one bias per layer, zero initial state for
  the encoder, the decoder layer l starts from the encoder layer l's state at
  the last REAL source position src_len[b] - 1, and the recurrences run over
  the padded lengths -- states past a sentence's end are computed but never
  read by the attention, whose mask excludes them);
* embeddings: x_t = E[y_t] (source and target tables);
* HybridNMTIF, encoder_decoder_if: the same model WITH the
  baseline's input feeding: the decoder's layer-0 input at
  step t is [E[y_t]; Htilde_{t-1}], Htilde_t = tanh(W_c [h_t; C_t]) from the
  attention over S at step t (Eqs. 1-4), Htilde_{-1} = 0.

Storage (row-major): ids [B, T] int; E [V, e]; W_ih[l] [4h, in_l] (in_0 = e,
else h); W_hh[l] [4h, h]; b[l] [4h]; outputs H [B, T, h] (the top layer, all
steps) and the per-layer final states.

Pinned by tests/test_lstm_oracle_pins.py: equality with torch.nn.LSTM in
float64 (an independent implementation of the same cell), the zero-weight and
bias-only closed forms, the decoder-initialisation rule; the input-feeding
decoder against torch.nn.LSTMCell + scaled_dot_product_attention in float64,
and reducing to the plain decoder when the feeding columns are zero.
"""
from __future__ import annotations

import numpy as np

__all__ = ["sigmoid", "lstm_cell", "lstm_stack", "encoder_decoder", "attention_step",
           "encoder_decoder_if", "lstm_stack_backward", "encoder_decoder_backward"]


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def lstm_cell(x, h, c, W_ih, W_hh, b):
    """One LSTM step for a batch (PAPER.md:75 baseline cell, gate order i, f, g, o).
    x [B, in], h / c [B, hd] -> (h', c')."""
    x = np.asarray(x, np.float64)
    h = np.asarray(h, np.float64)
    c = np.asarray(c, np.float64)
    gates = x @ np.asarray(W_ih, np.float64).T + h @ np.asarray(W_hh, np.float64).T + np.asarray(b, np.float64)
    hd = h.shape[1]
    i = sigmoid(gates[:, 0 * hd:1 * hd])
    f = sigmoid(gates[:, 1 * hd:2 * hd])
    g = np.tanh(gates[:, 2 * hd:3 * hd])
    o = sigmoid(gates[:, 3 * hd:4 * hd])
    c_new = f * c + i * g
    h_new = o * np.tanh(c_new)
    return h_new, c_new


def lstm_stack(X, weights, h0=None, c0=None, capture_at=None):
    """Stacked LSTM over all T steps, layer by layer (the order of evaluation
    does not change the result; the wavefront only reorders independent
    layer-steps).  X [B, T, in_0]; weights = [(W_ih, W_hh, b)] * L.
    h0 / c0: [L, B, hd] initial states (None = zeros).  capture_at: [B] step
    index whose states are returned per layer (None = the last step).
    Returns (H_top [B, T, hd], H_all [L, B, T, hd], h_cap [L, B, hd], c_cap [L, B, hd])."""
    X = np.asarray(X, np.float64)
    B, T, _ = X.shape
    L = len(weights)
    hd = np.asarray(weights[0][1]).shape[1]
    cap = np.full(B, T - 1) if capture_at is None else np.asarray(capture_at)
    H_all = np.zeros((L, B, T, hd))
    h_cap = np.zeros((L, B, hd))
    c_cap = np.zeros((L, B, hd))
    inp = X
    for l, (W_ih, W_hh, b) in enumerate(weights):
        h = np.zeros((B, hd)) if h0 is None else np.asarray(h0[l], np.float64).copy()
        c = np.zeros((B, hd)) if c0 is None else np.asarray(c0[l], np.float64).copy()
        for t in range(T):
            h, c = lstm_cell(inp[:, t, :], h, c, W_ih, W_hh, b)
            H_all[l, :, t, :] = h
            sel = cap == t
            h_cap[l, sel] = h[sel]
            c_cap[l, sel] = c[sel]
        inp = H_all[l]
    return H_all[L - 1], H_all, h_cap, c_cap


def encoder_decoder(src_ids, tgt_ids, src_len, E_src, E_tgt, enc_weights, dec_weights):
    """The encoder-decoder part of HybridNMT (no input feeding):
    S = encoder top-layer states for every source step, H = decoder top-layer
    states for every target step; decoder layer l starts from encoder layer
    l's state at source step src_len[b] - 1 (reading N3).
    Returns (S [B, M, hd], H [B, N, hd])."""
    E_src = np.asarray(E_src, np.float64)
    E_tgt = np.asarray(E_tgt, np.float64)
    Xs = E_src[np.asarray(src_ids)]
    Xt = E_tgt[np.asarray(tgt_ids)]
    S, _, h_fin, c_fin = lstm_stack(Xs, enc_weights, capture_at=np.asarray(src_len) - 1)
    H, _, _, _ = lstm_stack(Xt, dec_weights, h0=h_fin, c0=c_fin)
    return S, H


def attention_step(h, S, src_len, W_c):
    """Eqs. 1-4 for one decoder step of every sentence (dot
    score): e_j = h . S_j over j < src_len, alpha = softmax, C = sum_j alpha_j S_j,
    Htilde = tanh(W_c [h; C]) (W_c [d, 2d], columns [0, d) multiply h)."""
    h = np.asarray(h, np.float64)
    S = np.asarray(S, np.float64)
    W_c = np.asarray(W_c, np.float64)
    B, M, d = S.shape
    out = np.zeros((B, d))
    for b in range(B):
        L = int(src_len[b])
        e = S[b, :L] @ h[b]
        a = np.exp(e - e.max())
        a /= a.sum()
        C = a @ S[b, :L]
        out[b] = np.tanh(W_c[:, :d] @ h[b] + W_c[:, d:] @ C)
    return out


def encoder_decoder_if(src_ids, tgt_ids, src_len, E_src, E_tgt, enc_weights, dec_weights, W_c):
    """HybridNMTIF: the encoder of encoder_decoder, and a decoder
    with input feeding -- layer 0's input at step t is
    [E_tgt[y_t]; Htilde_{t-1}] (Htilde_{-1} = 0), Htilde_t = attention_step of
    the top-layer state.  Returns (S [B, M, hd], H [B, N, hd], Htilde [B, N, hd])."""
    E_src = np.asarray(E_src, np.float64)
    E_tgt = np.asarray(E_tgt, np.float64)
    Xs = E_src[np.asarray(src_ids)]
    S, _, h_fin, c_fin = lstm_stack(Xs, enc_weights, capture_at=np.asarray(src_len) - 1)
    B, N = np.asarray(tgt_ids).shape
    hd = S.shape[2]
    L = len(dec_weights)
    h = [h_fin[l].copy() for l in range(L)]
    c = [c_fin[l].copy() for l in range(L)]
    H = np.zeros((B, N, hd))
    Ht = np.zeros((B, N, hd))
    feed = np.zeros((B, hd))
    for t in range(N):
        x = np.concatenate([E_tgt[np.asarray(tgt_ids)[:, t]], feed], axis=1)
        for l, (W_ih, W_hh, b) in enumerate(dec_weights):
            h[l], c[l] = lstm_cell(x, h[l], c[l], W_ih, W_hh, b)
            x = h[l]
        H[:, t] = h[L - 1]
        feed = attention_step(h[L - 1], S, src_len, W_c)
        Ht[:, t] = feed
    return S, H, Ht


# ---------------------------------------------------------------- backward
def lstm_stack_backward(X, weights, dH_top, h0=None, c0=None, inject=None):
    """Reverse-mode derivative of lstm_stack (backpropagation through time, the
    plain chain rule of the cell, layer by layer from the top).  dH_top
    [B, T, hd]: gradient w.r.t. the top layer's states at every step.
    inject: optional (step [B], dh [L, B, hd], dc [L, B, hd]) added to layer
    l's (dh_t, dc_t) at t = step[b] (the decoder's initial-state gradients,
    which reach the encoder at source step src_len - 1).
    Returns (dX [B, T, in_0], [(dW_ih, dW_hh, db)] * L, dh0 [L, B, hd], dc0 [L, B, hd])."""
    X = np.asarray(X, np.float64)
    B, T, _ = X.shape
    L = len(weights)
    hd = np.asarray(weights[0][1]).shape[1]
    # forward again, keeping every activation
    inp = X
    acts = []
    for l, (W_ih, W_hh, b) in enumerate(weights):
        W_ih = np.asarray(W_ih, np.float64)
        W_hh = np.asarray(W_hh, np.float64)
        h = np.zeros((B, hd)) if h0 is None else np.asarray(h0[l], np.float64).copy()
        c = np.zeros((B, hd)) if c0 is None else np.asarray(c0[l], np.float64).copy()
        hs, cs, gs = [h], [c], []
        for t in range(T):
            z = inp[:, t] @ W_ih.T + h @ W_hh.T + np.asarray(b, np.float64)
            i, f = sigmoid(z[:, :hd]), sigmoid(z[:, hd:2 * hd])
            g, o = np.tanh(z[:, 2 * hd:3 * hd]), sigmoid(z[:, 3 * hd:])
            c = f * c + i * g
            h = o * np.tanh(c)
            hs.append(h)
            cs.append(c)
            gs.append((i, f, g, o))
        acts.append((inp, hs, cs, gs))
        inp = np.stack(hs[1:], axis=1)
    grads = [None] * L
    dh0 = np.zeros((L, B, hd))
    dc0 = np.zeros((L, B, hd))
    d_above = np.asarray(dH_top, np.float64)
    for l in range(L - 1, -1, -1):
        W_ih, W_hh, _ = (np.asarray(w, np.float64) for w in weights[l])
        xin, hs, cs, gs = acts[l]
        dW_ih = np.zeros_like(W_ih)
        dW_hh = np.zeros_like(W_hh)
        db = np.zeros(4 * hd)
        dx = np.zeros_like(xin)
        dh_next = np.zeros((B, hd))
        dc_next = np.zeros((B, hd))
        for t in range(T - 1, -1, -1):
            dh = d_above[:, t] + dh_next
            dc_in = dc_next.copy()
            if inject is not None:
                sel = np.asarray(inject[0]) == t
                dh[sel] += inject[1][l][sel]
                dc_in[sel] += inject[2][l][sel]
            i, f, g, o = gs[t]
            tc = np.tanh(cs[t + 1])
            dc = dc_in + dh * o * (1.0 - tc * tc)
            dz = np.concatenate([dc * g * i * (1 - i), dc * cs[t] * f * (1 - f),
                                 dc * i * (1 - g * g), dh * tc * o * (1 - o)], axis=1)
            dW_ih += dz.T @ xin[:, t]
            dW_hh += dz.T @ hs[t]
            db += dz.sum(0)
            dx[:, t] = dz @ W_ih
            dh_next = dz @ W_hh
            dc_next = dc * f
        grads[l] = (dW_ih, dW_hh, db)
        dh0[l], dc0[l] = dh_next, dc_next
        d_above = dx
    return d_above, grads, dh0, dc0


def encoder_decoder_backward(src_ids, tgt_ids, src_len, E_src, E_tgt, enc_weights, dec_weights,
                             dS, dH):
    """Gradients of encoder_decoder given dS = dL/dH_enc [B, M, hd] and
    dH = dL/dH_dec [B, N, hd] (what the attention-softmax stage returns):
    the decoder backward first; its initial-state gradients enter the encoder
    at source step src_len - 1 (reading N3); the embedding gradients sum the
    layer-0 input gradients per token id.  Returns dict with "enc" / "dec"
    [(dW_ih, dW_hh, db)] * L, "dE_src", "dE_tgt"."""
    E_src = np.asarray(E_src, np.float64)
    E_tgt = np.asarray(E_tgt, np.float64)
    src_ids = np.asarray(src_ids)
    tgt_ids = np.asarray(tgt_ids)
    Xs, Xt = E_src[src_ids], E_tgt[tgt_ids]
    cap = np.asarray(src_len) - 1
    _, _, h_fin, c_fin = lstm_stack(Xs, enc_weights, capture_at=cap)
    dXt, dec_g, dh0, dc0 = lstm_stack_backward(Xt, dec_weights, dH, h0=h_fin, c0=c_fin)
    dXs, enc_g, _, _ = lstm_stack_backward(Xs, enc_weights, dS, inject=(cap, dh0, dc0))
    dE_src = np.zeros_like(E_src)
    dE_tgt = np.zeros_like(E_tgt)
    np.add.at(dE_src, src_ids.reshape(-1), dXs.reshape(-1, dXs.shape[-1]))
    np.add.at(dE_tgt, tgt_ids.reshape(-1), dXt.reshape(-1, dXt.shape[-1]))
    return {"enc": enc_g, "dec": dec_g, "dE_src": dE_src, "dE_tgt": dE_tgt}
