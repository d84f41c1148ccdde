"""Pins of the encoder-decoder oracle (oracle/lstm_oracle.py, NEXT-3) against
things other than itself: torch.nn.LSTM in float64 (an independent
implementation of the same cell and stacking, PyTorch gate order i, f, g, o),
closed forms for zero / bias-only weights, and torch's packed-sequence
semantics for the decoder initialisation (reading N3: the encoder state at the
last real source position)."""
import numpy as np
import torch

from oracle import lstm_oracle as LO
from synthetic import CONFIGS, make_lstm_inputs


def _torch_lstm(ws, hd):
    L = len(ws)
    m = torch.nn.LSTM(input_size=ws[0][0].shape[1], hidden_size=hd, num_layers=L,
                      batch_first=True).double()
    with torch.no_grad():
        for l, (W_ih, W_hh, b) in enumerate(ws):
            getattr(m, f"weight_ih_l{l}").copy_(torch.from_numpy(np.asarray(W_ih, np.float64)))
            getattr(m, f"weight_hh_l{l}").copy_(torch.from_numpy(np.asarray(W_hh, np.float64)))
            getattr(m, f"bias_ih_l{l}").copy_(torch.from_numpy(np.asarray(b, np.float64)))
            getattr(m, f"bias_hh_l{l}").zero_()
    return m


def test_stack_equals_torch_lstm_float64():
    rng = np.random.default_rng(0)
    B, T, e, hd, L = 3, 7, 5, 6, 3
    ws = [(rng.uniform(-0.5, 0.5, (4 * hd, e if l == 0 else hd)), rng.uniform(-0.5, 0.5, (4 * hd, hd)),
           rng.uniform(-0.5, 0.5, 4 * hd)) for l in range(L)]
    X = rng.normal(size=(B, T, e))
    h0 = rng.normal(size=(L, B, hd)) * 0.3
    c0 = rng.normal(size=(L, B, hd)) * 0.3
    H, H_all, h_n, c_n = LO.lstm_stack(X, ws, h0=h0, c0=c0)
    m = _torch_lstm(ws, hd)
    with torch.no_grad():
        y, (hn, cn) = m(torch.from_numpy(X), (torch.from_numpy(h0), torch.from_numpy(c0)))
    assert np.allclose(H, y.numpy(), rtol=1e-12, atol=1e-14)
    assert np.allclose(h_n, hn.numpy(), rtol=1e-12, atol=1e-14)
    assert np.allclose(c_n, cn.numpy(), rtol=1e-12, atol=1e-14)


def test_zero_weights_give_zero_states():
    B, T, e, hd = 2, 4, 3, 5
    ws = [(np.zeros((4 * hd, e)), np.zeros((4 * hd, hd)), np.zeros(4 * hd)),
          (np.zeros((4 * hd, hd)), np.zeros((4 * hd, hd)), np.zeros(4 * hd))]
    H, _, h_n, c_n = LO.lstm_stack(np.ones((B, T, e)), ws)
    assert np.all(H == 0.0) and np.all(h_n == 0.0) and np.all(c_n == 0.0)


def test_bias_only_closed_form():
    """W = 0: every gate is its (constant) bias, so c_t = i g (1 - f^t) / (1 - f)
    (geometric series from c_0 = 0) and h_t = o tanh(c_t)."""
    hd, T = 4, 6
    b = np.array([0.3, -0.2, 1.1, 0.0, 0.5, 0.9, -0.4, 0.2, 0.7, -1.3, 0.25, 2.0, -0.1, 0.6, 1.5, -0.8])
    ws = [(np.zeros((4 * hd, 3)), np.zeros((4 * hd, hd)), b)]
    H, _, _, _ = LO.lstm_stack(np.zeros((1, T, 3)), ws)
    sg = lambda x: 1 / (1 + np.exp(-x))
    i, f, g, o = sg(b[0:4]), sg(b[4:8]), np.tanh(b[8:12]), sg(b[12:16])
    for t in range(T):
        c = i * g * (1 - f ** (t + 1)) / (1 - f)
        assert np.allclose(H[0, t], o * np.tanh(c), rtol=1e-13, atol=1e-15)


def test_decoder_starts_from_state_at_last_real_source_position():
    """Reading N3 against torch's packed sequences: the encoder run on each
    sentence's real prefix only (pack_padded_sequence) gives (h_n, c_n); the
    decoder started from them must give the oracle's H."""
    cfg = CONFIGS["small_f32"]
    inp = make_lstm_inputs(cfg, layers=2, emb=8)
    S, H = LO.encoder_decoder(inp["src_ids"], inp["tgt_ids"], inp["src_len"], inp["E_src"],
                              inp["E_tgt"], inp["enc"], inp["dec"])
    enc = _torch_lstm(inp["enc"], cfg.d)
    dec = _torch_lstm(inp["dec"], cfg.d)
    Xs = torch.from_numpy(np.asarray(inp["E_src"], np.float64)[inp["src_ids"]])
    Xt = torch.from_numpy(np.asarray(inp["E_tgt"], np.float64)[inp["tgt_ids"]])
    with torch.no_grad():
        packed = torch.nn.utils.rnn.pack_padded_sequence(
            Xs, torch.from_numpy(inp["src_len"].astype(np.int64)), batch_first=True, enforce_sorted=False)
        _, (hn, cn) = enc(packed)
        y, _ = dec(Xt, (hn, cn))
        s_full, _ = enc(Xs)
    assert np.allclose(H, y.numpy(), rtol=1e-11, atol=1e-13)
    # S (all source steps, padded positions included) = the unpacked run
    assert np.allclose(S, s_full.numpy(), rtol=1e-11, atol=1e-13)


def _torch_if(inp, cfg):
    """An independent float64 composition of HybridNMTIF: torch.nn.LSTM for the
    encoder (packed), torch.nn.LSTMCell per decoder layer, SDPA for Eqs. 1-3."""
    import torch.nn.functional as F
    enc = _torch_lstm(inp["enc"], cfg.d)
    Xs = torch.from_numpy(np.asarray(inp["E_src"], np.float64)[inp["src_ids"]])
    Et = torch.from_numpy(np.asarray(inp["E_tgt"], np.float64))
    W_c = torch.from_numpy(np.asarray(inp["W_c"], np.float64))
    lens = torch.from_numpy(inp["src_len"].astype(np.int64))
    with torch.no_grad():
        S, _ = enc(Xs)
        packed = torch.nn.utils.rnn.pack_padded_sequence(Xs, lens, batch_first=True, enforce_sorted=False)
        _, (hn, cn) = enc(packed)
        cells = []
        for (W_ih, W_hh, b) in inp["dec"]:
            cell = torch.nn.LSTMCell(W_ih.shape[1], cfg.d).double()
            cell.weight_ih.copy_(torch.from_numpy(np.asarray(W_ih, np.float64)))
            cell.weight_hh.copy_(torch.from_numpy(np.asarray(W_hh, np.float64)))
            cell.bias_ih.copy_(torch.from_numpy(np.asarray(b, np.float64)))
            cell.bias_hh.zero_()
            cells.append(cell)
        h = [hn[l].clone() for l in range(len(cells))]
        c = [cn[l].clone() for l in range(len(cells))]
        B, N = inp["tgt_ids"].shape
        mask = torch.arange(cfg.M)[None, :] < lens[:, None]
        feed = torch.zeros(B, cfg.d, dtype=torch.float64)
        Ht = []
        for t in range(N):
            x = torch.cat([Et[torch.from_numpy(inp["tgt_ids"][:, t].astype(np.int64))], feed], dim=1)
            for l, cell in enumerate(cells):
                h[l], c[l] = cell(x, (h[l], c[l]))
                x = h[l]
            C = F.scaled_dot_product_attention(h[-1][:, None, None, :], S[:, None], S[:, None],
                                               attn_mask=mask[:, None, None, :], scale=1.0)[:, 0, 0]
            feed = torch.tanh(torch.cat([h[-1], C], dim=1) @ W_c.T)
            Ht.append(feed)
    return torch.stack(Ht, 1).numpy()


def test_input_feeding_equals_torch_float64():
    cfg = CONFIGS["small_f32"]
    inp = make_lstm_inputs(cfg, layers=2, emb=8, input_feeding=True)
    _, _, Ht = LO.encoder_decoder_if(inp["src_ids"], inp["tgt_ids"], inp["src_len"], inp["E_src"],
                                     inp["E_tgt"], inp["enc"], inp["dec"], inp["W_c"])
    assert np.allclose(Ht, _torch_if(inp, cfg), rtol=1e-11, atol=1e-13)


def test_input_feeding_with_zero_feed_columns_is_the_plain_decoder():
    """W_ih[:, e:] = 0 cuts the feedback: H must equal the plain decoder's and
    Htilde_t the attention step of H_t (Eqs. 1-4 as the stage oracle computes them)."""
    from oracle import attn_softmax_oracle as AO
    cfg = CONFIGS["small_f32"]
    e = 8
    inp = make_lstm_inputs(cfg, layers=2, emb=e, input_feeding=True)
    W_ih, W_hh, b = inp["dec"][0]
    dec_plain = [(W_ih[:, :e], W_hh, b)] + list(inp["dec"][1:])
    W_ih0 = W_ih.copy()
    W_ih0[:, e:] = 0.0
    dec_zero = [(W_ih0, W_hh, b)] + list(inp["dec"][1:])
    S, H, Ht = LO.encoder_decoder_if(inp["src_ids"], inp["tgt_ids"], inp["src_len"], inp["E_src"],
                                     inp["E_tgt"], inp["enc"], dec_zero, inp["W_c"])
    S2, H2 = LO.encoder_decoder(inp["src_ids"], inp["tgt_ids"], inp["src_len"], inp["E_src"],
                                inp["E_tgt"], inp["enc"], dec_plain)
    assert np.allclose(H, H2, rtol=1e-12, atol=1e-14)
    B, N = inp["tgt_ids"].shape
    f, _ = AO.fwd_bwd(H, S, inp["src_len"], np.full(B, N, np.int32), np.zeros((B, N), np.int32),
                      inp["W_c"], np.zeros((5, cfg.d)), 1.0)
    assert np.allclose(Ht, f["Hc"].reshape(B, N, cfg.d), rtol=1e-12, atol=1e-14)


def test_encoder_decoder_backward_equals_torch_autograd():
    """The oracle's BPTT against torch float64 autograd through the same
    composition (embeddings, packed encoder, decoder started from the packed
    final states, arbitrary upstream gradients on S and H)."""
    cfg = CONFIGS["small_f32"]
    inp = make_lstm_inputs(cfg, layers=2, emb=8)
    rng = np.random.default_rng(3)
    dS = rng.normal(size=(cfg.B, cfg.M, cfg.d))
    dH = rng.normal(size=(cfg.B, cfg.N, cfg.d))
    got = LO.encoder_decoder_backward(inp["src_ids"], inp["tgt_ids"], inp["src_len"], inp["E_src"],
                                      inp["E_tgt"], inp["enc"], inp["dec"], dS, dH)
    enc = _torch_lstm(inp["enc"], cfg.d)
    dec = _torch_lstm(inp["dec"], cfg.d)
    Es = torch.tensor(np.asarray(inp["E_src"], np.float64), requires_grad=True)
    Et = torch.tensor(np.asarray(inp["E_tgt"], np.float64), requires_grad=True)
    src = torch.from_numpy(inp["src_ids"].astype(np.int64))
    tgt = torch.from_numpy(inp["tgt_ids"].astype(np.int64))
    lens = torch.from_numpy(inp["src_len"].astype(np.int64))
    Xs, Xt = Es[src], Et[tgt]
    S, _ = enc(Xs)
    packed = torch.nn.utils.rnn.pack_padded_sequence(Xs, lens, batch_first=True, enforce_sorted=False)
    _, (hn, cn) = enc(packed)
    H, _ = dec(Xt, (hn, cn))
    (S * torch.from_numpy(dS)).sum().add((H * torch.from_numpy(dH)).sum()).backward()
    for side, m in (("enc", enc), ("dec", dec)):
        for l, (dWi, dWh, db) in enumerate(got[side]):
            assert np.allclose(dWi, getattr(m, f"weight_ih_l{l}").grad.numpy(), rtol=1e-9, atol=1e-11), (side, l)
            assert np.allclose(dWh, getattr(m, f"weight_hh_l{l}").grad.numpy(), rtol=1e-9, atol=1e-11), (side, l)
            assert np.allclose(db, getattr(m, f"bias_ih_l{l}").grad.numpy(), rtol=1e-9, atol=1e-11), (side, l)
    assert np.allclose(got["dE_src"], Es.grad.numpy(), rtol=1e-9, atol=1e-11)
    assert np.allclose(got["dE_tgt"], Et.grad.numpy(), rtol=1e-9, atol=1e-11)
