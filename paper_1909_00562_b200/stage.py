"""Convenience wrapper over the C ABI: allocates the workspace and outputs
with PyTorch and calls attn_softmax_fwd_bwd.  No arithmetic happens here."""
from __future__ import annotations

import math
from typing import Optional

import torch

from . import binding

_TORCH_DTYPE = {"f32": torch.float32, "bf16": torch.bfloat16}


class NonFiniteLoss(RuntimeError):
    """The step's loss is NaN or inf (abort on a non-finite loss)."""


class AttnSoftmaxStage:
    """One GPU's shard of the data-parallel attention-softmax stage."""

    def __init__(self, B: int, N: int, M: int, d: int, V: int, dtype: str,
                 device: Optional[torch.device] = None):
        self.B, self.N, self.M, self.d, self.V, self.dtype = B, N, M, d, V, dtype
        self.tdtype = _TORCH_DTYPE[dtype]
        self.device = torch.device(device or "cuda")
        self.shape = binding.shape(B, N, M, d, V, dtype)
        nbytes = binding.attn_softmax_workspace_size(self.shape)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.views_meta = binding.attn_softmax_workspace_views(self.shape)

    def alloc_outputs(self, general_score: bool = False, bias: bool = False):
        dev, B, N, M, d, V = self.device, self.B, self.N, self.M, self.d, self.V
        out = dict(
            loss=torch.empty(1, dtype=torch.float32, device=dev),
            dH_dec=torch.empty(B, N, d, dtype=self.tdtype, device=dev),
            dH_enc=torch.empty(B, M, d, dtype=self.tdtype, device=dev),
            dW_c=torch.empty(d, 2 * d, dtype=torch.float32, device=dev),
            dW_out=torch.empty(V, d, dtype=torch.float32, device=dev))
        if general_score:
            out["dW_alpha"] = torch.empty(d, d, dtype=torch.float32, device=dev)
        if bias:
            out["db_out"] = torch.empty(V, dtype=torch.float32, device=dev)
        return out

    def __call__(self, H_dec, H_enc, src_len, tgt_len, tgt_ids, W_c, W_out,
                 loss_scale: float, out=None, comm=None, stream=None, W_alpha=None,
                 b_out=None, check_finite: bool = False):
        """W_alpha [d,d] (dtype of the stage) selects the Eq. 2 "general"
        score; None is the dot score of the hot path.
        b_out [V] adds the F_c bias of Eq. 5 (NEXT-1); out["db_out"] is its
        gradient.  check_finite reads the loss back (a host synchronisation)
        and raises NonFiniteLoss when it is NaN or inf."""
        if out is None:
            out = self.alloc_outputs(W_alpha is not None, b_out is not None)
        dWa = out.get("dW_alpha") if W_alpha is not None else None
        if b_out is None:
            binding.attn_softmax_fwd_bwd(
                self.shape, H_dec, H_enc, src_len, tgt_len, tgt_ids, W_c, W_out,
                loss_scale, out["loss"], out["dH_dec"], out["dH_enc"], out["dW_c"],
                out["dW_out"], self.workspace, comm=comm, stream=stream,
                W_alpha=W_alpha, dW_alpha=dWa)
        else:
            binding.attn_softmax_fwd_bwd_ex(
                self.shape, H_dec, H_enc, src_len, tgt_len, tgt_ids, W_c, W_out,
                loss_scale, out["loss"], out["dH_dec"], out["dH_enc"], out["dW_c"],
                out["dW_out"], self.workspace, comm=comm, stream=stream,
                W_alpha=W_alpha, dW_alpha=dWa, b_out=b_out, db_out=out["db_out"])
        if check_finite:
            loss = float(out["loss"].item())
            if not math.isfinite(loss):
                raise NonFiniteLoss(f"non-finite loss {loss} (B={self.B}, N={self.N}, M={self.M}, "
                                    f"d={self.d}, V={self.V}, {self.dtype})")
        return out

    def views(self):
        """Intermediates of the last call, as views into the workspace."""
        v, ws = self.views_meta, self.workspace
        T = self.B * self.N

        def view(off, n, dt):
            esz = torch.empty((), dtype=dt).element_size()
            return ws[off: off + n * esz].view(dt)

        return dict(
            alpha=view(v.alpha, T * v.alpha_ld, torch.float32).view(T, v.alpha_ld)[:, :self.M]
            .reshape(self.B, self.N, self.M),
            C=view(v.ctx, T * self.d, self.tdtype).view(self.B, self.N, self.d),
            Hc=view(v.hc, T * self.d, self.tdtype).view(self.B, self.N, self.d),
            lse=view(v.lse, T, torch.float32),
            nll=view(v.nll, T, torch.float32),
            vocab_chunk=int(v.vocab_chunk))


class DecodeStep:
    """Forward-only decoding step of the stage (NEXT-4): B sentences x N live
    hypotheses -> per hypothesis the k best next tokens and their
    log-probabilities (bf16 only)."""

    def __init__(self, B: int, N: int, M: int, d: int, V: int, k: int,
                 device: Optional[torch.device] = None):
        self.B, self.N, self.M, self.d, self.V, self.k = B, N, M, d, V, k
        self.device = torch.device(device or "cuda")
        self.shape = binding.shape(B, N, M, d, V, "bf16")
        nbytes = binding.attn_softmax_decode_workspace_size(self.shape)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)

    def __call__(self, H_dec, H_enc, src_len, W_c, W_out, W_alpha=None, b_out=None, stream=None):
        T = self.B * self.N
        ids = torch.empty(T, self.k, dtype=torch.int32, device=self.device)
        logp = torch.empty(T, self.k, dtype=torch.float32, device=self.device)
        lse = torch.empty(T, dtype=torch.float32, device=self.device)
        binding.attn_softmax_decode_step(self.shape, H_dec, H_enc, src_len, W_c, W_out, self.k,
                                         ids, logp, self.workspace, lse=lse, W_alpha=W_alpha,
                                         b_out=b_out, stream=stream)
        return ids.view(self.B, self.N, self.k), logp.view(self.B, self.N, self.k), \
            lse.view(self.B, self.N)


def to_device(inp: dict, dtype: str, device="cuda"):
    """numpy inputs from synthetic.make_inputs -> torch device tensors."""
    td = _TORCH_DTYPE[dtype]
    out = {}
    for k in ("H_dec", "H_enc", "W_c", "W_out", "W_alpha", "b_out"):
        if k in inp:
            out[k] = torch.from_numpy(inp[k]).to(device=device, dtype=td).contiguous()
    out["tgt_ids"] = torch.from_numpy(inp["tgt_ids"]).to(device=device, dtype=torch.int32).contiguous()
    out["src_len"] = inp["src_len"]
    out["tgt_len"] = inp["tgt_len"]
    return out


class EncoderDecoder:
    """NEXT-3: the stacked-LSTM encoder-decoder (no input feeding) that
    produces H_enc / H_dec for the stage (attn_encoder_decoder_fwd).  Holds
    the packed layer weights (attn_lstm_pack_layer) and the workspace."""

    def __init__(self, B: int, M: int, N: int, emb: int, hidden: int, layers: int,
                 vocab_src: int, vocab_tgt: int, device: Optional[torch.device] = None,
                 input_feeding: bool = False):
        """input_feeding=True: HybridNMTIF, the decoder's first
        layer sees [E_tgt[y_t]; Htilde_{t-1}] (its W_ih has emb + hidden columns)
        and the call also needs W_c and returns Htilde."""
        self.B, self.M, self.N, self.emb, self.hidden, self.layers = B, M, N, emb, hidden, layers
        self.input_feeding = input_feeding
        self.device = torch.device(device or "cuda")
        self.shape = binding.lstm_shape(B, M, N, emb, hidden, layers, vocab_src, vocab_tgt)
        n = (binding.attn_lstm_if_workspace_size if input_feeding else
             binding.attn_lstm_workspace_size)(self.shape)
        self.workspace = torch.empty(n, dtype=torch.uint8, device=self.device)
        self.enc_W = self.enc_b = self.dec_W = self.dec_b = None

    def _pack(self, layers, feed=False):
        Ws, bs = [], []
        for l, (W_ih, W_hh, b) in enumerate(layers):
            fin = (self.emb + (self.hidden if feed else 0)) if l == 0 else self.hidden
            Wp = torch.empty(4 * self.hidden, fin + self.hidden, dtype=torch.bfloat16, device=self.device)
            bp = torch.empty(4 * self.hidden, dtype=torch.float32, device=self.device)
            binding.attn_lstm_pack_layer(fin, self.hidden, W_ih, W_hh, b, Wp, bp)
            Ws.append(Wp)
            bs.append(bp)
        return Ws, bs

    def set_weights(self, enc_layers, dec_layers):
        """enc_layers / dec_layers: [(W_ih, W_hh, b)] bf16 device tensors (PyTorch layout)."""
        self.enc_W, self.enc_b = self._pack(enc_layers)
        self.dec_W, self.dec_b = self._pack(dec_layers, feed=self.input_feeding)

    def __call__(self, src_ids, tgt_ids, src_len, E_src, E_tgt, H_enc=None, H_dec=None, stream=None,
                 W_c=None, Htilde=None):
        if self.input_feeding:
            mk = lambda T: torch.empty(self.B, T, self.hidden, dtype=torch.bfloat16, device=self.device)
            H_enc = mk(self.M) if H_enc is None else H_enc
            H_dec = mk(self.N) if H_dec is None else H_dec
            Htilde = mk(self.N) if Htilde is None else Htilde
            binding.attn_encoder_decoder_if_fwd(self.shape, src_ids, tgt_ids, src_len, E_src, E_tgt,
                                                self.enc_W, self.enc_b, self.dec_W, self.dec_b, W_c,
                                                H_enc, H_dec, Htilde, self.workspace, stream=stream)
            return H_enc, H_dec, Htilde
        if H_enc is None:
            H_enc = torch.empty(self.B, self.M, self.hidden, dtype=torch.bfloat16, device=self.device)
        if H_dec is None:
            H_dec = torch.empty(self.B, self.N, self.hidden, dtype=torch.bfloat16, device=self.device)
        binding.attn_encoder_decoder_fwd(self.shape, src_ids, tgt_ids, src_len, E_src, E_tgt,
                                         self.enc_W, self.enc_b, self.dec_W, self.dec_b,
                                         H_enc, H_dec, self.workspace, stream=stream)
        return H_enc, H_dec


class EncoderDecoderTrainer(EncoderDecoder):
    """NEXT-3 training: the encoder-decoder forward that keeps its activations
    (attn_encoder_decoder_fwd_train) and the reverse-wavefront backward
    (attn_encoder_decoder_bwd) that turns the stage's dH_enc / dH_dec into the
    LSTM and embedding gradients.  dW / db come in the packed gate-interleaved
    order of attn_lstm_pack_layer (unpack_lstm_grad gives PyTorch's layout)."""

    def __init__(self, B, M, N, emb, hidden, layers, vocab_src, vocab_tgt, device=None):
        super().__init__(B, M, N, emb, hidden, layers, vocab_src, vocab_tgt, device=device)
        self.vocab_src, self.vocab_tgt = vocab_src, vocab_tgt
        self.workspace = torch.empty(binding.attn_lstm_train_workspace_size(self.shape),
                                     dtype=torch.uint8, device=self.device)

    def forward(self, src_ids, tgt_ids, src_len, E_src, E_tgt, stream=None):
        self.H_enc = torch.empty(self.B, self.M, self.hidden, dtype=torch.bfloat16, device=self.device)
        self.H_dec = torch.empty(self.B, self.N, self.hidden, dtype=torch.bfloat16, device=self.device)
        self.saved = (src_ids, tgt_ids, src_len)
        binding.attn_encoder_decoder_fwd_train(self.shape, src_ids, tgt_ids, src_len, E_src, E_tgt,
                                               self.enc_W, self.enc_b, self.dec_W, self.dec_b,
                                               self.H_enc, self.H_dec, self.workspace, stream=stream)
        return self.H_enc, self.H_dec

    def backward(self, dH_enc, dH_dec, stream=None):
        dev, L, hd = self.device, self.layers, self.hidden
        mk = lambda l: torch.empty(4 * hd, (self.emb if l == 0 else hd) + hd, dtype=torch.float32, device=dev)
        g = {"dW_enc": [mk(l) for l in range(L)], "dW_dec": [mk(l) for l in range(L)],
             "db_enc": [torch.empty(4 * hd, device=dev) for _ in range(L)],
             "db_dec": [torch.empty(4 * hd, device=dev) for _ in range(L)],
             "dE_src": torch.empty(self.vocab_src, self.emb, device=dev),
             "dE_tgt": torch.empty(self.vocab_tgt, self.emb, device=dev)}
        src_ids, tgt_ids, src_len = self.saved
        binding.attn_encoder_decoder_bwd(self.shape, src_ids, tgt_ids, src_len, self.enc_W, self.dec_W,
                                         self.H_enc, self.H_dec, dH_enc, dH_dec, g["dW_enc"], g["db_enc"],
                                         g["dW_dec"], g["db_dec"], g["dE_src"], g["dE_tgt"],
                                         self.workspace, stream=stream)
        return g


def unpack_lstm_grad(dW_packed, db_packed, in_dim: int, hidden: int):
    """Packed gate-interleaved (row 4u + q) -> PyTorch (W_ih [4h, in], W_hh [4h, h], b [4h])."""
    K = dW_packed.shape[1]
    W = dW_packed.reshape(hidden, 4, K).transpose(0, 1).reshape(4 * hidden, K)
    b = db_packed.reshape(hidden, 4).transpose(0, 1).reshape(4 * hidden)
    return W[:, :in_dim], W[:, in_dim:], b
