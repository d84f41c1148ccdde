"""Seeded synthetic inputs with the shapes of the paper's workloads.

Recipe:
  * H_dec, H_enc ~ N(0, sigma^2), sigma = (4/d)^(1/4), clipped to [-1, 1]
    (LSTM outputs lie in (-1, 1); the dot score then has std ~2, so the
    attention is neither uniform nor one-hot -- the paper has no 1/sqrt(d)
    scaling, reading R7).
  * W_c, W_out (and W_alpha) ~ U(-0.1, 0.1) (SPEC.md:273 init).
  * target ids y ~ U{4 .. V-1} (ids 0..3 reserved).
  * lengths: "full" (every sentence uses N, M), or ragged as each config says.
  * every value is drawn in fp32 and, for bf16 configs, rounded once to bf16
    (round-to-nearest-even); the oracle consumes those rounded values upcast
    to fp64, the GPU path the bf16 values themselves.
  * seeding is per sentence: lengths from default_rng([seed, b, 1]), data from
    default_rng([seed, b, 0]); weights from default_rng([seed, tag]).  A shard
    [b0, b1) therefore equals the matching slice of the global batch.
  * padded slots (i >= tgt_len, j >= src_len) hold ordinary random finite
    values, never zeros, so masking is exercised (R8, invariant I5).
"""
from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional, Sequence

import numpy as np

__all__ = ["Config", "CONFIGS", "round_bf16", "lengths", "make_inputs",
           "make_weights", "shard_range", "global_valid_tokens", "make_lstm_inputs"]


@dataclass(frozen=True)
class Config:
    name: str
    B: int          # sentences per GPU shard
    N: int          # padded target length
    M: int          # padded source length
    d: int          # hidden size
    V: int          # vocabulary size
    dtype: str      # "f32" | "bf16"
    seed: int
    lengths: str = "full"   # "full" | "ragged" | "ragged_src" | "fixed"
    src_len: Optional[tuple] = None   # used when lengths == "fixed"
    tgt_len: Optional[tuple] = None

    @property
    def T(self) -> int:
        return self.B * self.N

    def with_batch(self, B: int) -> "Config":
        return replace(self, B=B)


# BASELINE.json "configs" (C0..C4) plus parity-test shapes that span several
# tcgen05 tiles and ragged tails while the oracle still finishes in seconds.
CONFIGS = {
    # C0: tiny, fp32 (BASELINE.json configs[0])
    "tiny": Config("tiny", 2, 5, 5, 8, 50, "f32", 0),
    "tiny_ragged": Config("tiny_ragged", 2, 5, 5, 8, 50, "f32", 0, "fixed",
                          (5, 3), (5, 4)),
    # C1: paper-shaped (BASELINE.json configs[1]); C2 = C1 per GPU x {2,4,8}
    "paper": Config("paper", 128, 50, 50, 1024, 50000, "bf16", 1),
    # C3: large vocab (configs[3]), per GPU
    "large": Config("large", 256, 64, 64, 1024, 100000, "bf16", 3),
    # C4: long sentences with ragged source masks (configs[4]), per GPU
    "long": Config("long", 64, 120, 120, 2048, 64000, "bf16", 4, "ragged_src"),
    # parity-test shapes (not bench lines)
    "small_f32": Config("small_f32", 5, 13, 11, 40, 300, "f32", 5, "ragged"),
    "small": Config("small", 7, 37, 41, 256, 3001, "bf16", 6, "ragged"),
    "medium": Config("medium", 16, 50, 50, 512, 9000, "bf16", 7, "ragged"),
    # awkward shapes: d not a multiple of 256, N > 128 (two attention row
    # tiles per sentence), M not a multiple of 64, V tiny and odd
    "odd": Config("odd", 3, 130, 100, 320, 777, "bf16", 8, "ragged"),
    "odd_f32": Config("odd_f32", 3, 17, 9, 24, 77, "f32", 9, "ragged"),
    # boundary shapes of the bf16 path: one token of everything (d = one K
    # block, V below one 256-wide tile), and the largest source length
    # (M = 128, one attention tile) with full lengths
    "edge_min": Config("edge_min", 1, 1, 1, 64, 50, "bf16", 10, "full"),
    "edge_max_src": Config("edge_max_src", 2, 128, 128, 128, 300, "bf16", 11, "full"),
}


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (ties to even); returns fp32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def _sigma(d: int) -> float:
    return (4.0 / d) ** 0.25


def lengths(cfg: Config, b: int):
    """(src_len, tgt_len) of global sentence b."""
    if cfg.lengths == "full":
        return cfg.M, cfg.N
    if cfg.lengths == "fixed":
        return int(cfg.src_len[b]), int(cfg.tgt_len[b])
    rng = np.random.default_rng([cfg.seed, b, 1])
    if cfg.lengths == "ragged_src":
        # C4: sentence 0 has the maximum source length, sentence 1 the minimum
        s = int(rng.integers(1, cfg.M + 1))
        if b == 0:
            s = cfg.M
        elif b == 1:
            s = 1
        return s, cfg.N
    if cfg.lengths == "ragged":
        s = int(rng.integers(1, cfg.M + 1))
        t = int(rng.integers(0, cfg.N + 1))
        if b == 0:
            s, t = cfg.M, cfg.N          # one full sentence
        elif b == 1:
            s = 1                        # degenerate attention (E4)
        elif b == 2:
            t = 0                        # sentence without targets
        return s, t
    raise ValueError(f"unknown lengths mode {cfg.lengths!r}")


def global_valid_tokens(cfg: Config, B_global: int) -> int:
    return sum(lengths(cfg, b)[1] for b in range(B_global))


def make_weights(cfg: Config, with_alpha: bool = False, with_bias: bool = False):
    """W_c [d,2d], W_out [V,d] (and W_alpha [d,d], b_out [V]) ~ U(-0.1, 0.1)
    (b_out ~ U(-1, 1): wide enough that the bias visibly shapes the softmax)."""
    d, V = cfg.d, cfg.V
    W_c = np.random.default_rng([cfg.seed, 1001]).uniform(
        -0.1, 0.1, size=(d, 2 * d)).astype(np.float32)
    W_out = np.random.default_rng([cfg.seed, 1002]).uniform(
        -0.1, 0.1, size=(V, d)).astype(np.float32)
    out = dict(W_c=W_c, W_out=W_out)
    if with_alpha:
        out["W_alpha"] = np.random.default_rng([cfg.seed, 1003]).uniform(
            -0.1, 0.1, size=(d, d)).astype(np.float32)
    if with_bias:
        out["b_out"] = np.random.default_rng([cfg.seed, 1004]).uniform(
            -1.0, 1.0, size=(V,)).astype(np.float32)
    if cfg.dtype == "bf16":
        out = {k: round_bf16(v) for k, v in out.items()}
    return out


def make_inputs(cfg: Config, sentences: Optional[Sequence[int]] = None,
                with_weights: bool = True, with_alpha: bool = False,
                with_bias: bool = False):
    """Activations of the given global sentence ids (default: 0..B-1).

    Returns a dict of fp32 numpy arrays (bf16-representable for bf16
    configs) and int32 length / id arrays:
      H_dec [B,N,d], H_enc [B,M,d], src_len [B], tgt_len [B], tgt_ids [B,N]
    plus W_c, W_out (, W_alpha) when with_weights.
    """
    if sentences is None:
        sentences = range(cfg.B)
    sentences = list(sentences)
    B, N, M, d, V = len(sentences), cfg.N, cfg.M, cfg.d, cfg.V
    H_dec = np.empty((B, N, d), np.float32)
    H_enc = np.empty((B, M, d), np.float32)
    ids = np.empty((B, N), np.int32)
    src = np.empty(B, np.int32)
    tgt = np.empty(B, np.int32)
    sig = _sigma(d)
    for k, b in enumerate(sentences):
        src[k], tgt[k] = lengths(cfg, b)
        rng = np.random.default_rng([cfg.seed, b, 0])
        H_dec[k] = np.clip(rng.normal(0.0, sig, size=(N, d)), -1.0, 1.0)
        H_enc[k] = np.clip(rng.normal(0.0, sig, size=(M, d)), -1.0, 1.0)
        ids[k] = rng.integers(4, V, size=N)
    if cfg.dtype == "bf16":
        H_dec = round_bf16(H_dec)
        H_enc = round_bf16(H_enc)
    out = dict(H_dec=H_dec, H_enc=H_enc, src_len=src, tgt_len=tgt,
               tgt_ids=ids)
    if with_weights:
        out.update(make_weights(cfg, with_alpha, with_bias))
    return out


def shard_range(B_global: int, world: int, rank: int):
    """Contiguous sentence range of `rank`; sizes differ by at most one
    (split by sentence, never by decoder step)."""
    base, extra = divmod(B_global, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def make_lstm_inputs(cfg: Config, layers: int = 4, emb: Optional[int] = None,
                     sentences: Optional[Sequence[int]] = None, input_feeding: bool = False):
    """Inputs of the encoder-decoder part (NEXT-3; Table 1, PAPER.md:190-192:
    embedding 512, hidden 1024, 4 stacked LSTM layers): source / target ids
    [B, M] / [B, N] ~ U{4 .. V-1} (one vocabulary of size V for both sides),
    the config's lengths, embedding tables E_src / E_tgt [V, emb] and per
    layer (W_ih [4h, in], W_hh [4h, h], b [4h]) for the encoder and the
    decoder, all ~ U(-0.1, 0.1) (SPEC.md:273 init) and bf16-rounded for bf16
    configs.  emb defaults to h / 2 (512 for h = 1024).  input_feeding: the
    decoder's layer-0 W_ih has emb + h columns (HybridNMTIF), and W_c [h, 2h]
    (as make_weights) is included."""
    if sentences is None:
        sentences = range(cfg.B)
    sentences = list(sentences)
    B, N, M, h, V = len(sentences), cfg.N, cfg.M, cfg.d, cfg.V
    e = emb if emb is not None else max(16, h // 2)
    src_ids = np.empty((B, M), np.int32)
    tgt_ids = np.empty((B, N), np.int32)
    src = np.empty(B, np.int32)
    tgt = np.empty(B, np.int32)
    for k, b in enumerate(sentences):
        src[k], tgt[k] = lengths(cfg, b)
        rng = np.random.default_rng([cfg.seed, b, 2])
        src_ids[k] = rng.integers(4, V, size=M)
        tgt_ids[k] = rng.integers(4, V, size=N)

    def u(tag, shape):
        return np.random.default_rng([cfg.seed, tag]).uniform(-0.1, 0.1, size=shape).astype(np.float32)

    out = dict(src_ids=src_ids, tgt_ids=tgt_ids, src_len=src, tgt_len=tgt,
               E_src=u(2001, (V, e)), E_tgt=u(2002, (V, e)))
    for side, base in (("enc", 3000), ("dec", 4000)):
        ws = []
        for l in range(layers):
            fin = (e + (h if (input_feeding and side == "dec") else 0)) if l == 0 else h
            ws.append((u(base + 10 * l, (4 * h, fin)), u(base + 10 * l + 1, (4 * h, h)),
                       u(base + 10 * l + 2, (4 * h,))))
        out[side] = ws
    if input_feeding:
        out["W_c"] = make_weights(cfg)["W_c"]
    if cfg.dtype == "bf16":
        out["E_src"] = round_bf16(out["E_src"])
        out["E_tgt"] = round_bf16(out["E_tgt"])
        for side in ("enc", "dec"):
            out[side] = [tuple(round_bf16(w) for w in ws) for ws in out[side]]
    return out
