"""Quick C1 timing of the stage (development aid, not the bench contract)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1909_00562_b200 import binding
from paper_1909_00562_b200.stage import AttnSoftmaxStage, to_device
from synthetic import CONFIGS, make_inputs, global_valid_tokens

name = sys.argv[1] if len(sys.argv) > 1 else "paper"
cfg = CONFIGS[name]
t0 = time.time()
inp = make_inputs(cfg)
print(f"inputs {time.time()-t0:.1f}s", flush=True)
if os.environ.get("ATTN_VC"):
    binding.attn_softmax_set_option("vocab_chunk", int(os.environ["ATTN_VC"]))
if os.environ.get("ATTN_PAIR"):
    binding.attn_softmax_set_option("cta_pair", int(os.environ["ATTN_PAIR"]))
if os.environ.get("ATTN_MCAST"):
    binding.attn_softmax_set_option("b_multicast", int(os.environ["ATTN_MCAST"]))
if os.environ.get("ATTN_WIDE"):
    binding.attn_softmax_set_option("wide_tiles", int(os.environ["ATTN_WIDE"]))
if os.environ.get("ATTN_MIXED"):
    binding.attn_softmax_set_option("mixed_tiles", int(os.environ["ATTN_MIXED"]))
if os.environ.get("ATTN_WIDEMC"):
    binding.attn_softmax_set_option("wide_multicast", int(os.environ["ATTN_WIDEMC"]))
if os.environ.get("ATTN_DBGEMM"):
    binding.attn_softmax_set_option("db_gemm", int(os.environ["ATTN_DBGEMM"]))
if os.environ.get("ATTN_SL"):
    binding.attn_softmax_set_option("store_logits", int(os.environ["ATTN_SL"]))
if os.environ.get("ATTN_NFAST"):
    binding.attn_softmax_set_option("n_fast", int(os.environ["ATTN_NFAST"]))
if os.environ.get("ATTN_SKIPEW"):
    binding.attn_softmax_set_option("debug_skip_dlogits", int(os.environ["ATTN_SKIPEW"]))
if os.environ.get("ATTN_PDL"):
    binding.attn_softmax_set_option("pdl", int(os.environ["ATTN_PDL"]))
if os.environ.get("ATTN_CTAS"):
    binding.attn_softmax_set_option("gemm_ctas", int(os.environ["ATTN_CTAS"]))
binding.attn_softmax_set_option("stage_events", int(os.environ.get("ATTN_EV", "1")))
st = AttnSoftmaxStage(cfg.B, cfg.N, cfg.M, cfg.d, cfg.V, cfg.dtype)
dv = to_device(inp, cfg.dtype)
scale = 1.0 / global_valid_tokens(cfg, cfg.B)
out = st.alloc_outputs(bias=bool(os.environ.get("ATTN_BIAS")))
args = (dv["H_dec"], dv["H_enc"], dv["src_len"], dv["tgt_len"], dv["tgt_ids"], dv["W_c"], dv["W_out"], scale)
kw = {}
if os.environ.get("ATTN_BIAS"):   # NEXT-1 F_c bias
    kw["b_out"] = to_device(make_inputs(cfg, with_bias=True), cfg.dtype)["b_out"]
for _ in range(3):
    st(*args, out=out, **kw)
torch.cuda.synchronize()
print("loss", out["loss"].item(), "vc", st.views()["vocab_chunk"], flush=True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
n = 10
for _ in range(n):
    st(*args, out=out, **kw)
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / n
tok = int(inp["tgt_len"].sum())
flops = tok * (6 * cfg.d * cfg.V + 12 * cfg.d * cfg.d + 12 * cfg.M * cfg.d)
st(*args, out=out, **kw)
if os.environ.get("ATTN_EV", "1") != "0":
    print({k: round(v, 4) for k, v in binding.attn_softmax_stage_times().items()})
print(f"{name}: {ms:.3f} ms/step, {tok/ms*1e3:.0f} tok/s, useful {flops/ms/1e9:.1f} TFLOP/s")
