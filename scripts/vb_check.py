"""Development check of the persistent vocab backward: parity against the
fp64 oracle on small configs, determinism, then C1 timing (not the bench)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle import attn_softmax_oracle as O
from paper_1909_00562_b200 import binding
from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
from synthetic import CONFIGS, global_valid_tokens, make_inputs


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run(cfg, inp, scale, bias=False):
    st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
    dv = to_device(inp, cfg.dtype)
    out = st(dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"],
             dv["W_out"], scale, b_out=dv.get("b_out") if bias else None)
    torch.cuda.synchronize()
    return {k: (v.float().cpu().numpy() if torch.is_tensor(v) else v) for k, v in out.items()}, st


def parity(name, vc=0, budget=None, bias=False):
    cfg = CONFIGS[name] if isinstance(name, str) else name
    name = cfg.name
    if vc:
        binding.attn_softmax_set_option("vocab_chunk", vc)
    if budget:
        binding.attn_softmax_set_option("dl_budget_mb", budget)
    inp = make_inputs(cfg, with_bias=bias)
    scale = 1.0 / global_valid_tokens(cfg, cfg.B)
    g, st = run(cfg, inp, scale, bias)
    g2, _ = run(cfg, inp, scale, bias)
    f, b = O.fwd_bwd(inp["H_dec"], inp["H_enc"], inp["src_len"], inp["tgt_len"], inp["tgt_ids"],
                     inp["W_c"], inp["W_out"], scale, b_out=inp.get("b_out"))
    keys = ("dH_dec", "dH_enc", "dW_c", "dW_out") + (("db_out",) if bias else ())
    errs = {k: rel(g[k], b[k]) for k in keys}
    det = all(np.array_equal(g[k], g2[k]) for k in keys + ("loss",))
    print(f"{name} vc={st.views()['vocab_chunk']}: loss {abs(g['loss'][0]-f['loss'])/abs(f['loss']):.2e} "
          + " ".join(f"{k} {v:.2e}" for k, v in errs.items()) + f" deterministic={det}", flush=True)
    binding.attn_softmax_set_option("vocab_chunk", 0)
    binding.attn_softmax_set_option("dl_budget_mb", 96)


def timing(name="paper", n=10, **opts):
    cfg = CONFIGS[name]
    for k, v in opts.items():
        binding.attn_softmax_set_option(k, v)
    inp = make_inputs(cfg)
    scale = 1.0 / global_valid_tokens(cfg, cfg.B)
    st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
    dv = to_device(inp, cfg.dtype)
    out = st.alloc_outputs()
    args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"],
            dv["W_out"], scale)
    binding.attn_softmax_set_option("stage_events", 1)
    for _ in range(3):
        st(*args, out=out)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tot = 0.0
    stages = {}
    for i in range(n):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st(*args, out=out)
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
        for k, v in binding.attn_softmax_stage_times().items():
            stages[k] = stages.get(k, 0) + v / n
    binding.attn_softmax_set_option("stage_events", 0)
    ms = tot / n
    tok = int(inp["tgt_len"].sum())
    print(f"{name} {opts}: {ms:.3f} ms/step {tok / ms * 1e3 / 1e6:.3f} M tok/s loss "
          f"{out['loss'].item():.5f} vc {st.views()['vocab_chunk']} "
          + str({k: round(v, 4) for k, v in stages.items()}), flush=True)
    for k in opts:
        binding.attn_softmax_set_option(k, {"store_logits": 0, "vocab_bwd_persistent": 1,
                                            "dl_budget_mb": 96, "vocab_chunk": 0,
                                            "dl_buffers": 3, "vb_last_g2_first": 1,
                                            "vb_pair": 1, "vb_order": 1, "vb_fwd_fused": 0,
                                            "vb_wide": 1}.get(k, 0))


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "parity"):
        for nm in ("small", "medium", "odd", "edge_min", "edge_max_src"):
            parity(nm)
        parity("small", vc=256)
        parity("medium", vc=512)
        parity("odd", vc=256)
        parity("small", bias=True)
        parity("odd", vc=256, bias=True)
        binding.attn_softmax_set_option("vb_fwd_fused", 1)
        parity("small")
        parity("odd", vc=256, bias=True)
        parity("edge_min")
        binding.attn_softmax_set_option("vb_fwd_fused", 0)
    if what in ("wide",):   # 512-column G2 / G3 tiles (d % 512 == 0)
        from dataclasses import replace
        binding.attn_softmax_set_option("vb_wide", 1)
        parity("medium")
        parity("medium", vc=512)
        parity(replace(CONFIGS["small"], name="small_d1024", d=1024, V=3001))
        parity(replace(CONFIGS["small"], name="small_d1024_bias", d=1024, V=2500), vc=256, bias=True)
        parity(replace(CONFIGS["odd"], name="odd_d512", d=512, N=100, V=777), vc=256)
        for _ in range(2):
            timing()
            timing(vb_wide=0)
    if what in ("pair1",):
        binding.attn_softmax_set_option("vb_pair", 0)
        for nm in ("small", "medium", "odd"):
            parity(nm)
        binding.attn_softmax_set_option("vb_pair", 1)
    if what in ("all", "time"):
        timing()
        timing(vb_fwd_fused=1)
        for b in (72, 120):
            timing(dl_budget_mb=b)
        timing(store_logits=1)
        timing()
